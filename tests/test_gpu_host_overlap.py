"""pf_parse_host with PF_OPT_HOST_OVERLAP: the NMS stage of chunk c+1 runs
beside the parse of chunk c on a second stream with two NMS slab sets.  The
poses must be byte-identical to the one-stream schedule, for the PAF read in
place and copied, across full and partial chunks, and equal the oracle."""
import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native
from support import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def maps():
    topo = pf.load_topology("coco18")
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(11, s, 656, 368, sp) for s in range(330)]   # 2 full chunks + 74
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    pin_conf = _native.PinnedArray(tuple(conf.shape))
    pin_paf = _native.PinnedArray(tuple(paf.shape))
    pin_conf.array[:] = conf.cpu().numpy()
    pin_paf.array[:] = paf.cpu().numpy()
    return topo, pin_conf, pin_paf


@pytest.mark.parametrize("up", [1, 8])
@pytest.mark.parametrize("zero_copy", [1, 0])
def test_host_overlap_equals_one_stream(maps, up, zero_copy):
    topo, pin_conf, pin_paf = maps
    params = pf.ParserParams(upsample=up)
    eng = pf.PafParser(topo)
    eng.ctx.set_option(_native.PF_OPT_PAF_ZERO_COPY, zero_copy)
    got = {}
    for ov in (0, 1):
        eng.ctx.set_option(_native.PF_OPT_HOST_OVERLAP, ov)
        for _ in range(2):                                 # second call reuses the slab sets
            got[ov] = eng.parse_arrays(pin_conf.array, pin_paf.array, 8, params).records(topo)
    assert got[1] == got[0]
    eng.close()
    # and the oracle on frames of every chunk
    for f in (0, 127, 128, 255, 256, 329):
        c = np.array(pin_conf.array[f]); p = np.array(pin_paf.array[f])
        want = (oracle.parse(c, p, topo, params, 8) if up == 1
                else oracle.parse_upsampled(c, p, topo, params, 8, up))
        rec = pf.pose_record(f, [pf.HumanPose(
            keypoints=tuple(None if k is None else pf.Keypoint(*k) for k in kps), score=s, n_parts=n)
            for s, n, kps in want.humans], topo)
        assert got[1][f] == rec, f
