"""The large-frame parse (k_parse_large, pf_large.cu): frames past the
shared-memory capacities of k_parse_frames — more than 32767 peaks per
frame, which the reference handles without limits (paf.py:100-109,
:231-289).  The context switches to it by itself when an automatic
capacity cannot grow on the usual path; PF_OPT_LARGE forces it."""

import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from conftest import record_of
from support import synth

pytestmark = pytest.mark.gpu

SP = synth.SynthParams()


def _oracle(conf, paf, topo, params, stride=8):
    if params.upsample == 1:
        return oracle.parse(conf, paf, topo, params, stride)
    return oracle.parse_upsampled(conf, paf, topo, params, stride, params.upsample)


@pytest.mark.parametrize("up", [1, 8])
def test_forced_large_path_equals_usual_path(topo, up):
    """Same peaks, connections (fp64 scores) and records as the usual
    (split / crowded) path on everyday and crowded frames, and as the oracle."""
    scenes = [synth.procedural_scene(7, s, 656, 368, SP) for s in range(30)] + \
             [synth.crowd_scene(44, s) for s in range(3)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=up)
    usual = pf.PafParser(topo, debug=True)
    got = usual.parse_arrays(conf, paf, 8, params)
    want_rec = [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))]
    want_pk = [usual.peaks(f) for f in range(len(scenes))]
    want_cn = [usual.connections(f) for f in range(len(scenes))]
    usual.close()
    large = pf.PafParser(topo, debug=True)
    large.ctx.set_option(pf._native.PF_OPT_LARGE, 1)
    large.set_timing(True)
    large.kernel_times(reset=True)
    got = large.parse_arrays(conf, paf, 8, params)
    assert "k_parse_large" in large.kernel_times(reset=True)
    assert [large.peaks(f) for f in range(len(scenes))] == want_pk
    assert [large.connections(f) for f in range(len(scenes))] == want_cn
    assert [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))] == want_rec
    for f in (0, 31):
        w = _oracle(conf[f], paf[f], topo, params)
        assert want_rec[f] == record_of(w.humans, topo, f)
    large.close()


def _noisy_frame(rng, h, w, n_noisy, people):
    """Parts 0-2 carry `people` three-part chains (Gaussian blobs, PAF
    corridors along limbs 0->1 and 1->2); parts 3.. are uniform noise."""
    K = 3 + n_noisy
    conf = np.zeros((K + 1, h, w), np.float32)
    paf = np.zeros((4, h, w), np.float32)
    yy, xx = np.mgrid[0:h, 0:w]
    for _ in range(people):
        c = rng.uniform(20, min(h, w) - 20, 2)
        pts = [c, c + rng.uniform(-12, 12, 2), None]
        pts[2] = pts[1] + rng.uniform(-12, 12, 2)
        for k, p in enumerate(pts):
            conf[k] = np.maximum(conf[k], np.exp(-((yy - p[0]) ** 2 + (xx - p[1]) ** 2) / 8.0).astype(np.float32))
        for l in range(2):
            a, b = pts[l], pts[l + 1]
            d = b - a
            n = np.hypot(*d)
            u = d / n
            t = ((yy - a[0]) * u[0] + (xx - a[1]) * u[1])
            perp = np.abs((yy - a[0]) * u[1] - (xx - a[1]) * u[0])
            m = (t >= -1) & (t <= n + 1) & (perp <= 1.5)
            paf[2 * l][m] = u[1]          # x component
            paf[2 * l + 1][m] = u[0]      # y component
    conf[3:K] = rng.random((n_noisy, h, w)).astype(np.float32)
    return conf, paf


@pytest.mark.parametrize("grid, up, n_noisy", [((200, 200), 1, 9), ((135, 240), 8, 12)])
def test_frame_with_more_than_32767_peaks(grid, up, n_noisy):
    """More than 32767 peaks in one frame (uniform-noise parts; the second case
    is a noise-like 1080p Mode U frame): the context outgrows the usual path's
    16-bit / shared-memory capacities, switches to k_parse_large and returns
    the oracle's peaks and poses instead of a CapacityError."""
    rng = np.random.default_rng(12)
    names = [f"p{k}" for k in range(3 + n_noisy)]
    topo = pf.SkeletonTopology.create(names, [(0, 1), (1, 2)])
    frames = [_noisy_frame(rng, grid[0], grid[1], n_noisy, 3) for _ in range(2)]
    conf = np.stack([f[0] for f in frames])
    paf = np.stack([f[1] for f in frames])
    params = pf.ParserParams(min_parts=2, upsample=up)
    e = pf.PafParser(topo, debug=True)
    e.set_timing(True)
    e.kernel_times(reset=True)
    got = e.parse_arrays(conf, paf, 8, params)
    assert "k_parse_large" in e.kernel_times(reset=True)
    for f in range(len(frames)):
        want = _oracle(conf[f], paf[f], topo, params)
        assert len(want.peaks) > 32767
        assert e.peaks(f) == want.peaks
        assert e.connections(f) == want.connections
        assert pf.pose_record(f, got.poses(f), topo) == record_of(want.humans, topo, f)
        assert got.frame_count[f] > 0
    # the switch is per call: the next (everyday) call runs the usual path again
    conf2, paf2 = conf.copy(), paf.copy()
    conf2[:, 3:] = 0.0
    e.kernel_times(reset=True)
    got = e.parse_arrays(conf2, paf2, 8, params)
    assert "k_parse_large" not in e.kernel_times(reset=True)
    for f in range(len(frames)):
        want = _oracle(conf2[f], paf2[f], topo, params)
        assert pf.pose_record(f, got.poses(f), topo) == record_of(want.humans, topo, f)
    e.close()
