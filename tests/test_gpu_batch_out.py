"""pf_parse_batch (the §8(b) batch entry point): caller-owned [B][max_humans]
device slots, per-call stream, no host synchronisation and no replay.  The
slots must hold exactly the poses the pooled path returns (pose_record
bytes), capacity overflows must land in the status words, and the maps may
be released as soon as the stream has consumed them (SPEC.md:250-258:
inputs are needed only for the call)."""
import pytest

torch = pytest.importorskip("torch")

import paper_2108_11826_b200 as pf  # noqa: E402
from support import synth  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def topo():
    return pf.load_topology("coco18")


def _maps(topo, scenes):
    conf, paf = synth.render_batch_gpu(scenes, topo, synth.SynthParams())
    return conf, paf


def _records(topo, poses_of, n):
    return [pf.pose_record(f, poses_of(f), topo) for f in range(n)]


@pytest.mark.parametrize("up", [1, 8])
def test_parse_into_equals_pooled_results(topo, up):
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(64)]
    conf, paf = _maps(topo, scenes)
    params = pf.ParserParams(upsample=up)
    eng = pf.PafParser(topo)
    eng.parse_tensors(conf, paf, 8, params)
    ref = eng.results()
    want = _records(topo, ref.poses, 64)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        slots = eng.parse_into(conf, paf, 8, params, max_humans=16)
    side.synchronize()
    slots.check()
    assert slots.status.tolist() == [0, -1]
    assert slots.n_humans.tolist() == [len(ref.poses(f)) for f in range(64)]
    assert _records(topo, slots.poses, 64) == want
    eng.close()


def test_parse_into_max_humans_overflow_is_reported(topo):
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(32)]
    conf, paf = _maps(topo, scenes)
    eng = pf.PafParser(topo)
    eng.parse_tensors(conf, paf, 8, pf.ParserParams())
    ref = eng.results()
    counts = [len(ref.poses(f)) for f in range(32)]
    first_over = next(f for f, c in enumerate(counts) if c > 1)
    slots = eng.parse_into(conf, paf, 8, pf.ParserParams(), max_humans=1)
    torch.cuda.synchronize()
    assert slots.status.tolist() == [pf._native.PF_ERR_CAPACITY, first_over]
    assert slots.n_humans.tolist() == counts                 # true counts, never truncated silently
    with pytest.raises(pf.CapacityError):
        slots.check()
    # the one slot written per frame holds the frame's best human
    view = pf.PoseSlots(slots.n_humans.clamp(max=1), slots.human_score, slots.n_parts, slots.kp_xy,
                        slots.kp_score, slots.kp_present, slots.status)
    for f in range(32):
        assert pf.pose_record(f, view.poses(f), topo) == pf.pose_record(f, ref.poses(f)[:1], topo)
    eng.close()


def test_parse_into_internal_capacity_is_reported(topo):
    conf, paf = _maps(topo, [synth.crowd_scene(3, 0), synth.crowd_scene(3, 1)])
    eng = pf.PafParser(topo, caps=dict(max_peaks_per_part=8))
    slots = eng.parse_into(conf, paf, 8, pf.ParserParams(), max_humans=64)
    torch.cuda.synchronize()
    assert slots.status.tolist()[0] == pf._native.PF_ERR_CAPACITY
    assert slots.status.tolist()[1] == 0
    assert slots.n_humans.tolist() == [0, 0]
    eng.close()


def test_parse_into_maps_only_needed_while_the_stream_runs(topo):
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(48)]
    conf, paf = _maps(topo, scenes)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    eng.parse_tensors(conf, paf, 8, params)
    want = _records(topo, eng.results().poses, 48)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        c2, p2 = conf.clone(), paf.clone()
        slots = eng.parse_into(c2, p2, 8, params, max_humans=16)
        del c2, p2                                            # released right after the call
        junk = [torch.full_like(conf, 7.0), torch.full_like(paf, -3.0)]   # reuse attempts
    side.synchronize()
    del junk
    slots.check()
    assert _records(topo, slots.poses, 48) == want
    eng.close()


def test_parse_into_contract_errors_before_work(topo):
    eng = pf.PafParser(topo)
    conf = torch.zeros(2, 19, 46, 82, device="cuda")
    with pytest.raises(pf.ContractError):
        eng.parse_into(conf, torch.zeros(2, 37, 46, 82, device="cuda"), 8, pf.ParserParams())
    with pytest.raises(pf.ConfigError):
        eng.parse_into(conf, torch.zeros(2, 38, 46, 82, device="cuda"), 8, pf.ParserParams(nms_window=4))
    with pytest.raises(pf.ContractError):
        eng.parse_into(conf, torch.zeros(2, 38, 46, 82, device="cuda"), 8, pf.ParserParams(), max_humans=-1)
    eng.close()
