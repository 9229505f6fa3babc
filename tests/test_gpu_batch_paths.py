"""Every batch-size path choice against the oracle: the Mode U NMS switches
from the one-kernel corner form to the scan + finish split at 256 frames,
the parse from the wide one-kernel form (at most one frame per SM) to the
split parse beyond; Mode R and Mode U, everyday and crowded frames mixed,
batch sizes on both sides of each boundary.  Each batch is parsed once and
a strided sample of its frames (always the first and the last) is compared
with the oracle byte for byte; the whole batch is also compared with the
split paths forced (PF_OPT_CORNER_SPLIT / PF_OPT_PARSE_SPLIT = 2)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402
from test_gpu_timed_configs import oracle_records  # noqa: E402

pytestmark = pytest.mark.gpu
SP = synth.SynthParams()


@pytest.fixture(scope="module")
def pool():
    topo = pf.load_topology("coco18")
    scenes = [synth.procedural_scene(31, s, 656, 368, SP) for s in range(288)]
    for k in range(0, 288, 24):                     # a crowded frame every 24
        scenes[k] = synth.crowd_scene(31, k)
    conf, paf = synth.render_batch_gpu(scenes, topo, SP)
    return topo, conf, paf


def _records(res, topo, n):
    return [pf.pose_record(f, res.poses(f), topo) for f in range(n)]


@pytest.mark.parametrize("up", [8, 1])
@pytest.mark.parametrize("n", [1, 31, 148, 149, 255, 256, 288])
def test_batch_size_paths_match_oracle_and_split(pool, n, up):
    topo, conf, paf = pool
    params = pf.ParserParams(upsample=up)
    eng = pf.PafParser(topo)
    eng.parse_tensors(conf[:n], paf[:n], 8, params)
    got = _records(eng.results(), topo, n)
    eng.ctx.set_option(_native.PF_OPT_CORNER_SPLIT, 2)
    eng.ctx.set_option(_native.PF_OPT_PARSE_SPLIT, 2)
    eng.parse_tensors(conf[:n], paf[:n], 8, params)
    assert _records(eng.results(), topo, n) == got
    eng.close()
    idx = sorted(set(list(range(0, n, max(1, n // 12))) + [n - 1]))
    c = conf[:n].cpu().numpy()
    p = paf[:n].cpu().numpy()
    assert [got[f] for f in idx] == oracle_records(c, p, topo, params, idx=idx)


def test_peak_ranking_forms_agree_on_crowded_frames():
    """k_parse_peaks ranks a frame's peaks with a warp per frame above 4
    frames per SM and with a 4-warp CTA per frame at or below: one batch
    just above the boundary (crowded frames every third) equals the same
    frames parsed in small batches, and its crowded frames equal the oracle."""
    topo = pf.load_topology("coco18")
    n = 4 * torch.cuda.get_device_properties(0).multi_processor_count + 8
    scenes = [synth.crowd_scene(57, s) if s % 3 == 0 else synth.procedural_scene(57, s, 656, 368, SP)
              for s in range(n)]
    conf, paf = synth.render_batch_gpu(scenes, topo, SP)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    eng.parse_tensors(conf, paf, 8, params)
    got = _records(eng.results(), topo, n)
    chunks = []
    for s in range(0, n, 100):
        eng.parse_tensors(conf[s:s + 100], paf[s:s + 100], 8, params)
        r = eng.results()
        chunks += [pf.pose_record(s + f, r.poses(f), topo) for f in range(min(100, n - s))]
    eng.close()
    assert chunks == got
    idx = [0, 3, n // 2 - (n // 2) % 3, n - 1 - (n - 1) % 3]
    c = conf.cpu().numpy()
    p = paf.cpu().numpy()
    assert [got[f] for f in idx] == oracle_records(c, p, topo, params, idx=idx)


def test_exact_list_handover_and_fallbacks(pool):
    """Split Mode U: k_corner_finish hands each plane's candidates to
    k_corner_exact (default); with the hand-over off, and with a list so short
    that most planes overflow it (their candidates are tested in the finish,
    the slots they had reserved are skipped), the poses are the same, and a
    sample equals the oracle."""
    topo, conf, paf = pool
    n = 288
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    out = []
    for opt in (0, -1, 700, 1):
        eng.ctx.set_option(_native.PF_OPT_EXACT_LIST, opt)
        eng.parse_tensors(conf[:n], paf[:n], 8, params)
        out.append(_records(eng.results(), topo, n))
    eng.close()
    assert out[1] == out[0] and out[2] == out[0] and out[3] == out[0]
    idx = [0, 24, 100, 287]
    c = conf[:n].cpu().numpy()
    p = paf[:n].cpu().numpy()
    assert [out[0][f] for f in idx] == oracle_records(c, p, topo, params, idx=idx)
