"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden fixtures and the oracle, bit-exact — peaks, connections (fp64 scores),
person assignment, human scores and pose_record bytes."""

import json

import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from support import synth
from conftest import golden_path, record_of

pytestmark = pytest.mark.gpu

SP = synth.SynthParams()


@pytest.fixture(scope="module")
def eng(topo):
    e = pf.PafParser(topo, debug=True)
    yield e
    e.close()


def oracle_run(conf, paf, topo, params, stride=8):
    if params.upsample == 1 and params.blur_sigma == 0:
        return oracle.parse(conf, paf, topo, params, stride)
    taps = pf._native.gaussian_taps(params.blur_sigma) if params.blur_sigma > 0 else None
    return oracle.parse_upsampled(conf, paf, topo, params, stride, params.upsample, taps)


def assert_batch_matches(eng, topo, conf, paf, params, stride=8, stages=True):
    got = eng.parse_arrays(conf, paf, stride, params)
    for f in range(conf.shape[0]):
        want = oracle_run(conf[f], paf[f], topo, params, stride)
        if stages:
            assert eng.peaks(f) == want.peaks, f"frame {f} peaks"
            assert eng.connections(f) == want.connections, f"frame {f} connections"
        assert pf.pose_record(f, got.poses(f), topo) == record_of(want.humans, topo, f), f"frame {f}"
    return got


def render(scenes, topo):
    return synth.render_batch(scenes, topo, SP)


# ---------------------------------------------------------------- golden
@pytest.mark.parametrize("mode", ["R", "U"])
def test_reference_golden_frames(eng, topo, golden_frames, mode):
    data, recs = golden_frames
    names = [n for n in recs["names"] if mode == "R" or n in recs["U"]]
    conf = np.stack([data[f"{n}.conf"] for n in names])
    paf = np.stack([data[f"{n}.paf"] for n in names])
    params = pf.ParserParams(upsample=1 if mode == "R" else recs["up"])
    got = eng.parse_arrays(conf, paf, 8, params)
    for f, name in enumerate(names):
        pk, ps = data[f"{name}.{mode}.peaks"], data[f"{name}.{mode}.peak_scores"]
        assert eng.peaks(f) == [(int(a), int(b), int(c), float(s), q)
                                for q, ((a, b, c), s) in enumerate(zip(pk, ps))], name
        cn, cv = data[f"{name}.{mode}.conns"], data[f"{name}.{mode}.conn_vals"]
        assert eng.connections(f) == [(int(a), int(b), int(c), float(s), float(g))
                                      for (a, b, c), (s, g) in zip(cn, cv)], name
        assert pf.pose_record(0, got.poses(f), topo) == recs[mode][name], name


def test_nms_golden_maps():
    """nms_peaks on the reference's random / plateau / threshold-edge maps."""
    g = np.load(golden_path("nms_golden.npz"))
    one = pf.SkeletonTopology.create(["p"], [])
    e = pf.PafParser(one, debug=True)
    maps = g["maps"]
    off = 0
    for i in range(maps.shape[0]):
        conf = np.stack([maps[i], np.zeros_like(maps[i])])[None]
        paf = np.zeros((1, 0) + maps.shape[1:], np.float32)
        params = pf.ParserParams(conf_threshold=float(g["thresholds"][i]), nms_window=int(g["windows"][i]))
        e.parse_arrays(conf, paf, 1, params)
        n = int(g["counts"][i])
        want = [(0, int(c[0]), int(c[1]), float(s), q)
                for q, (c, s) in enumerate(zip(g["cells"][off:off + n], g["scores"][off:off + n]))]
        off += n
        assert e.peaks(0) == want, f"case {i}"
    off = 0
    for i in range(g["w5_maps"].shape[0]):
        m = g["w5_maps"][i]
        e.parse_arrays(np.stack([m, np.zeros_like(m)])[None], np.zeros((1, 0, 10, 10), np.float32), 1,
                       pf.ParserParams(nms_window=5))
        n = int(g["w5_counts"][i])
        want = [(0, int(c[0]), int(c[1]), float(s), q)
                for q, (c, s) in enumerate(zip(g["w5_cells"][off:off + n], g["w5_scores"][off:off + n]))]
        off += n
        assert e.peaks(0) == want
    e.close()


def test_score_limb_golden():
    """score_limb through the full pipeline: one limb, two single-cell peaks."""
    g = np.load(golden_path("score_golden.npz"))
    two = pf.SkeletonTopology.create(["a", "b"], [[0, 1]])
    e = pf.PafParser(two, debug=True)
    params = pf.ParserParams(good_fraction_min=0.0, min_parts=1, min_human_score=-1.0)
    checked = 0
    for fld, meta, vals in zip(g["fields"], g["meta"], g["vals"]):
        n, _limb, ai, aj, bi, bj = (int(v) for v in meta)
        if (ai, aj) == (bi, bj):
            continue
        conf = np.zeros((1, 3, n, n), np.float32)
        conf[0, 0, ai, aj] = 1.0
        conf[0, 1, bi, bj] = 1.0
        paf = fld[None, :, :n, :n].astype(np.float32)
        e.parse_arrays(conf, paf, 1, params)
        conns = e.connections(0)
        s, gd = float(vals[0]), float(vals[1])
        if s > 0.0:
            assert conns == [(0, 0, 1, s, gd)]
            checked += 1
        else:
            assert conns == []
    assert checked > 50
    e.close()


# ---------------------------------------------------------------- vs oracle
@pytest.mark.parametrize("up", [1, 8])
def test_procedural_frames(eng, topo, up):
    scenes = [synth.procedural_scene(7, s, 656, 368, SP) for s in range(24 if up == 1 else 8)]
    conf, paf = render(scenes, topo)
    assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up))


@pytest.mark.parametrize("up", [1, 8])
def test_crowded_frames(eng, topo, up):
    """40-person scenes: merges, part conflicts, slot-taken skips, min_parts drops,
    and > kCandSmem gated candidates (the global spill path)."""
    scenes = [synth.crowd_scene(3, s) for s in range(3 if up == 1 else 1)]
    conf, paf = render(scenes, topo)
    assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up))


@pytest.mark.parametrize("kw", [dict(nms_window=5), dict(nms_window=7), dict(nms_window=9),
                                dict(n_samples=2), dict(n_samples=17), dict(n_samples=40),
                                dict(conf_threshold=0.05), dict(conf_threshold=0.3), dict(conf_threshold=0.7),
                                dict(sample_dot_threshold=0.5), dict(good_fraction_min=0.5),
                                dict(good_fraction_min=1.0), dict(min_parts=1), dict(min_parts=12),
                                dict(min_human_score=0.0), dict(min_human_score=0.9)])
@pytest.mark.parametrize("up", [1, 8])
def test_param_variants(eng, topo, kw, up):
    scenes = [synth.procedural_scene(19, s, 656, 368, SP) for s in range(3)] + [synth.crowd_scene(5, 0)]
    conf, paf = render(scenes, topo)
    assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up, **kw))


@pytest.mark.parametrize("up", [2, 4])
def test_other_upsample_factors(eng, topo, up):
    scenes = [synth.procedural_scene(23, s, 656, 368, SP) for s in range(3)]
    conf, paf = render(scenes, topo)
    assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up))


def test_stride_and_odd_grid(eng, topo):
    # 45x37 grid, stride 8 -> 360x296 input; 1 person near the border
    scene = synth.GroundTruthScene(humans=(synth.procedural_scene(2, 0, 360, 296, SP).humans), input_w=360,
                                input_h=296)
    conf, paf = render([scene], topo)
    for up in (1, 2, 8):
        assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up))


def test_random_fields(topo):
    """Unstructured maps: many peaks, ties (quantised values), random PAFs,
    thousands of gated candidates per frame (spill slab), many merges."""
    rng = np.random.default_rng(77)
    conf = rng.random((4, 19, 12, 14)).astype(np.float32)
    conf[::2] = np.round(conf[::2] * 8) / 8
    paf = rng.uniform(-1, 1, (4, 38, 12, 14)).astype(np.float32)
    e = pf.PafParser(topo, debug=True, caps=dict(max_candidates=16384, max_humans_per_frame=1024))
    for up in (1, 4):
        assert_batch_matches(e, topo, conf, paf, pf.ParserParams(upsample=up, good_fraction_min=0.3,
                                                                  min_parts=2))
    e.close()


def test_corner_kernel_overflow_and_nonfinite(eng, topo):
    """Mode U corner kernel edge cases: an all-hot smooth frame (hot cells beyond
    the shared list -> whole-plane slow path), a noise part map (candidate list
    overflow), NaN / +inf / -inf sources; Mode R sees the same non-finite maps."""
    scenes = [synth.procedural_scene(41, s, 656, 368, SP) for s in range(4)]
    conf, paf = render(scenes, topo)
    K = topo.n_keypoints
    yy, xx = np.mgrid[0:conf.shape[2], 0:conf.shape[3]].astype(np.float32)
    conf[0, :K] = (0.55 + 0.35 * np.sin(xx / 3.0 + np.arange(K)[:, None, None]) * np.cos(yy / 4.0)).astype(np.float32)
    rng = np.random.default_rng(5)
    conf[1, 3] = rng.random(conf.shape[2:]).astype(np.float32)
    conf[1, 7] = np.round(rng.random(conf.shape[2:]) * 4).astype(np.float32) / 4   # ties
    for k, (i, j, v) in enumerate([(10, 20, np.nan), (11, 20, np.inf), (30, 40, -np.inf), (0, 0, np.nan),
                                   (45, 81, np.inf), (20, 60, np.nan)]):
        conf[2, k % K, i, j] = v
        conf[3, (3 * k) % K, (i + 7) % conf.shape[2], (j + 11) % conf.shape[3]] = v
    for up in (8, 1):
        assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up))


def test_blur_fused_kernels_vs_materialised(topo):
    """The fused upsample -> blur -> NMS kernels (2-D tiles for radius <= 8,
    the row kernel beyond) against the materialised path (resize -> blur
    rows / cols -> NMS over HBM maps) on 24 frames per sigma — peaks and
    records identical — and against the oracle on two of them."""
    scenes = [synth.procedural_scene(41, s, 656, 368, SP) for s in range(24)]
    conf, paf = render(scenes, topo)
    e = pf.PafParser(topo, debug=True)
    for sigma in (0.5, 1.0, 2.5, 3.0):
        params = pf.ParserParams(upsample=8, blur_sigma=sigma)
        e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 0)
        e.set_timing(True)
        e.kernel_times(reset=True)
        got = e.parse_arrays(conf, paf, 8, params)
        assert "k_up_blur_nms" in e.kernel_times(reset=True)
        e.set_timing(False)
        fused = [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))]
        peaks = [e.peaks(f) for f in range(len(scenes))]
        e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 1)
        got = e.parse_arrays(conf, paf, 8, params)
        assert [e.peaks(f) for f in range(len(scenes))] == peaks, sigma
        assert [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))] == fused, sigma
        for f in (0, 17):
            want = oracle_run(conf[f], paf[f], topo, params)
            assert peaks[f] == want.peaks, (sigma, f)
            assert fused[f] == record_of(want.humans, topo, f), (sigma, f)
    e.close()


def test_blur_cold_block_skip_edges(topo):
    """k_up_blur_tile skips blocks whose sources all lie in [0, thr (1 - 2^-10)):
    maps built around that bound (just below / at / above it, plateaus at the
    threshold, negative values, NaN) give the same peaks as the materialised
    path, which skips nothing."""
    rng = np.random.default_rng(5)
    thr = 0.1
    x = np.float32(thr) - np.float32(thr) * np.float32(2.0 ** -10)
    F, K, h, w = 6, topo.n_keypoints, 46, 82
    conf = np.zeros((F, K + 1, h, w), np.float32)
    base = [np.float32(x) * np.float32(0.999), np.nextafter(np.float32(x), np.float32(0)), np.float32(x),
            np.float32(thr), np.nextafter(np.float32(thr), np.float32(1))]
    for f in range(F):
        for k in range(K):
            v = base[(f + k) % len(base)]
            m = np.full((h, w), v, np.float32) * rng.uniform(0.97, 1.0, (h, w)).astype(np.float32)
            if (f + k) % 3 == 0:
                m[rng.integers(0, h), rng.integers(0, w)] = np.float32(thr) * 1.5      # one hot spot
            if (f + k) % 4 == 1:
                m[rng.integers(0, h), rng.integers(0, w)] = -0.5
            if (f + k) % 7 == 2:
                m[rng.integers(0, h), rng.integers(0, w)] = np.nan
            if (f + k) % 5 == 3:
                m[:] = np.float32(thr)                                               # plateau at thr
            conf[f, k] = m
    paf = np.zeros((F, 2 * topo.n_limbs, h, w), np.float32)
    e = pf.PafParser(topo, debug=True)
    for sigma in (1.0, 2.0):
        params = pf.ParserParams(upsample=8, blur_sigma=sigma)
        e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 0)
        e.parse_arrays(conf, paf, 8, params)
        fused = [e.peaks(f) for f in range(F)]
        e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 1)
        e.parse_arrays(conf, paf, 8, params)
        assert [e.peaks(f) for f in range(F)] == fused, sigma
        assert sum(len(p) for p in fused) > 0
    e.close()


def test_blur_paths(eng, topo):
    scenes = [synth.procedural_scene(29, s, 656, 368, SP) for s in range(2)]
    conf, paf = render(scenes, topo)
    for up, sigma in ((8, 1.0), (8, 2.5), (1, 0.8)):
        assert_batch_matches(eng, topo, conf, paf, pf.ParserParams(upsample=up, blur_sigma=sigma))


def test_materialised_and_generic_paths_agree(topo):
    scenes = [synth.procedural_scene(31, s, 656, 368, SP) for s in range(4)] + [synth.crowd_scene(8, 1)]
    conf, paf = render(scenes, topo)
    params = pf.ParserParams(upsample=8)
    e = pf.PafParser(topo, debug=True)
    ref = [pf.pose_record(f, p, topo) for f, p in enumerate(e.parse_arrays(conf, paf, 8, params).all_poses())]
    e.set_materialise(True)
    assert [pf.pose_record(f, p, topo) for f, p in enumerate(e.parse_arrays(conf, paf, 8, params).all_poses())] == ref
    e.set_materialise(False)
    e.ctx.set_option(pf._native.PF_OPT_GENERIC_FUSED, 1)
    assert [pf.pose_record(f, p, topo) for f, p in enumerate(e.parse_arrays(conf, paf, 8, params).all_poses())] == ref
    e.close()


# ---------------------------------------------------------------- API contract
def test_parse_drop_in(topo):
    """parse(maps, topo, params) returns HumanPose lists equal to the reference's."""
    scene = synth.procedural_scene(0, 1, 656, 368, SP)
    maps = synth.render_feature_maps(scene, topo, SP)
    poses = pf.parse(maps, topo, pf.ParserParams())
    want = oracle.parse(maps.conf.array, maps.paf.array, topo, pf.ParserParams(), 8)
    assert pf.pose_record(0, poses, topo) == record_of(want.humans, topo)
    assert all(isinstance(p, pf.HumanPose) for p in poses) and len(poses) == 3
    for p in poses:
        p.validate(input_w=656, input_h=368)


def test_parse_batch_equals_per_frame(topo):
    maps = [synth.render_feature_maps(synth.procedural_scene(4, s, 656, 368, SP), topo, SP) for s in range(5)]
    params = pf.ParserParams(upsample=8)
    batch = pf.parse_batch(maps, topo, params)
    single = [pf.parse(m, topo, params) for m in maps]
    assert [pf.pose_record(i, p, topo) for i, p in enumerate(batch)] == \
           [pf.pose_record(i, p, topo) for i, p in enumerate(single)]
    shuffled = pf.parse_batch(maps[::-1], topo, params)[::-1]
    assert [pf.pose_record(i, p, topo) for i, p in enumerate(shuffled)] == \
           [pf.pose_record(i, p, topo) for i, p in enumerate(single)]


def test_deterministic(eng, topo):
    conf, paf = render([synth.crowd_scene(4, s) for s in range(2)], topo)
    a = eng.parse_arrays(conf, paf, 8, pf.ParserParams(upsample=8))
    b = eng.parse_arrays(conf, paf, 8, pf.ParserParams(upsample=8))
    assert [pf.pose_record(f, a.poses(f), topo) for f in range(2)] == \
           [pf.pose_record(f, b.poses(f), topo) for f in range(2)]


def test_device_tensor_path(topo):
    import torch

    conf, paf = render([synth.procedural_scene(6, s, 656, 368, SP) for s in range(6)], topo)
    params = pf.ParserParams(upsample=8)
    e = pf.PafParser(topo)
    host = e.parse_arrays(conf, paf, 8, params)
    e.parse_tensors(torch.from_numpy(conf).cuda(), torch.from_numpy(paf).cuda(), 8, params)
    dev = e.results()
    assert [pf.pose_record(f, host.poses(f), topo) for f in range(6)] == \
           [pf.pose_record(f, dev.poses(f), topo) for f in range(6)]
    # native poses.jsonl of the whole batch == per-frame pose_record
    assert dev.records(topo, 40) == [pf.pose_record(40 + f, dev.poses(f), topo) for f in range(6)]
    assert e.launch_count() >= 4
    e.close()


@pytest.mark.parametrize("up", [1, 8])
def test_pinned_paf_read_in_place(topo, up):
    """pf_parse_host with pinned host maps: the PAF read in place over PCIe
    (PF_OPT_PAF_ZERO_COPY, default) gives the copied path's results and the
    oracle's, on procedural and crowded frames across several host chunks."""
    scenes = [synth.procedural_scene(12, s, 656, 368, SP) for s in range(5)] + [synth.crowd_scene(4, 0)]
    conf, paf = render(scenes, topo)
    reps = 46                                          # 276 frames: host chunks of 128, 128 and 20 frames
                                                       # (a partial chunk at the end)
    pc = pf._native.PinnedArray((len(scenes) * reps,) + conf.shape[1:])
    pp = pf._native.PinnedArray((len(scenes) * reps,) + paf.shape[1:])
    pc.array[:] = np.concatenate([conf] * reps)
    pp.array[:] = np.concatenate([paf] * reps)
    params = pf.ParserParams(upsample=up)
    e = pf.PafParser(topo)
    got = e.parse_arrays(pc.array, pp.array, 8, params)
    in_place = [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes) * reps)]
    e.ctx.set_option(pf._native.PF_OPT_PAF_ZERO_COPY, 0)
    got = e.parse_arrays(pc.array, pp.array, 8, params)
    copied = [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes) * reps)]
    e.close()
    assert in_place == copied
    for f in range(len(scenes)):
        want = oracle_run(conf[f], paf[f], topo, params)
        assert in_place[f] == record_of(want.humans, topo, f)
        assert in_place[f + len(scenes) * (reps - 1)].split(",", 1)[1] == in_place[f].split(",", 1)[1]
    pc.free()
    pp.free()


def test_empty_inputs(eng, topo):
    assert pf.parse_batch([], topo, pf.ParserParams()) == []
    zero = synth.render_feature_maps(synth.GroundTruthScene((), 64, 64), topo, SP)
    assert pf.parse(zero, topo, pf.ParserParams()) == []
    r = eng.parse_arrays(np.zeros((3, 19, 0, 0), np.float32), np.zeros((3, 38, 0, 0), np.float32), 8,
                         pf.ParserParams())
    assert r.n_frames == 3 and r.total_humans == 0
    tiny = np.zeros((1, 19, 1, 1), np.float32)
    tiny[0, :18] = 1.0
    r = eng.parse_arrays(tiny, np.ones((1, 38, 1, 1), np.float32), 8, pf.ParserParams(upsample=8))
    assert eng.peaks(0)[0][:3] == (0, 0, 0)


def test_errors_before_work(topo):
    maps = synth.render_feature_maps(synth.procedural_scene(0, 1, 656, 368, SP), topo, SP)
    with pytest.raises(pf.ConfigError):
        pf.parse(maps, topo, pf.ParserParams(nms_window=4))
    stub = pf.SkeletonTopology.create(["a", "b"], [[0, 1]])
    with pytest.raises(pf.ContractError):
        pf.parse(maps, stub, pf.ParserParams())
    e = pf.PafParser(topo)
    with pytest.raises(pf.ContractError):    # stride not divisible by upsample
        e.parse_arrays(maps.conf.array[None], maps.paf.array[None], 8, pf.ParserParams(upsample=3))
    e.close()


def test_capacity_errors_are_loud(topo):
    conf, paf = render([synth.crowd_scene(3, 0)], topo)
    e = pf.PafParser(topo, caps=dict(max_peaks_per_part=8))
    with pytest.raises(pf.CapacityError, match="max_peaks_per_part"):
        e.parse_arrays(conf, paf, 8, pf.ParserParams())
    e.close()
    e = pf.PafParser(topo, caps=dict(max_candidates=512))
    with pytest.raises(pf.CapacityError, match="max_candidates"):
        e.parse_arrays(conf, paf, 8, pf.ParserParams(upsample=8))
    e.close()
    e = pf.PafParser(topo, caps=dict(max_humans_total=3))
    with pytest.raises(pf.CapacityError):
        e.parse_arrays(conf, paf, 8, pf.ParserParams())
    e.close()


def _chain_fields(rng, K, h, w):
    """Adversarial part maps for the corner kernel's chain pre-filter: ramps
    (every interior cell chain-prunable), slopes near the 2^-16 M margin,
    exact plateaus / ties, saddles, checkerboards, huge and tiny magnitudes."""
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    f = []
    f.append(0.2 + 0.7 * xx / w)                                          # ramp right
    f.append(0.9 - 0.7 * yy / h)                                          # ramp up
    f.append(0.5 + 1e-5 * (xx - w / 2) ** 2 / w)                          # slopes ~ the margin
    f.append(0.5 + 2e-6 * np.sin(xx / 2) * np.cos(yy / 3))                # below the margin: exact path
    f.append(np.round(rng.random((h, w)) * 3) / 3 * 0.8 + 0.1)           # plateaus / ties
    f.append(0.5 + 0.3 * ((xx - w / 2) ** 2 - (yy - h / 2) ** 2) / (w * w))   # saddle
    f.append(0.4 + 0.2 * ((np.arange(h)[:, None] + np.arange(w)[None, :]) % 2))   # checkerboard
    f.append((0.5 + 0.4 * np.sin(xx / 4) * np.sin(yy / 5)) * 1e30)       # huge
    f.append((0.5 + 0.4 * np.sin(xx / 4) * np.sin(yy / 5)) * 1e-30)      # tiny (cold at thr 0.1)
    f.append(0.5 + 0.4 * np.exp(-((xx - 20.5) ** 2 + (yy - 10.25) ** 2) / 8)
             + 0.4 * np.exp(-((xx - 23.5) ** 2 + (yy - 10.25) ** 2) / 8))   # two close blobs: ridge
    f.append(np.full((h, w), 0.5))                                        # flat
    out = np.zeros((K, h, w), np.float32)
    for k in range(K):
        out[k] = f[k % len(f)]
    return out


@pytest.mark.parametrize("up", [2, 3, 8, 16])
def test_corner_chain_prefilter_is_exact(topo, up):
    """The chain pre-filter only removes cells that provably hold no peak: the
    corner kernel with and without it gives identical peaks, and both equal
    the oracle."""
    rng = np.random.default_rng(2024 + up)
    K = topo.n_keypoints
    h, w = 23, 41
    conf = np.zeros((3, K + 1, h, w), np.float32)
    for f in range(3):
        conf[f, :K] = _chain_fields(rng, K, h, w)
        conf[f, :K] = np.roll(conf[f, :K], f * 5, axis=0)
    conf[2, :K] = conf[2, :K] * np.float32(0.99) + rng.random((K, h, w)).astype(np.float32) * np.float32(0.01)
    paf = np.zeros((3, 38, h, w), np.float32)      # peaks are the subject; no limbs
    for thr in (0.1, 0.0):
        params = pf.ParserParams(upsample=up, conf_threshold=thr)
        e1 = pf.PafParser(topo, debug=True)
        runs = []
        for no_chain, split in ((0, 2), (1, 2), (0, 0), (1, 0)):
            # split 2: survivors classified by k_corner_finish; 0: one kernel
            e1.ctx.set_option(pf._native.PF_OPT_NO_CHAIN, no_chain)
            e1.ctx.set_option(pf._native.PF_OPT_CORNER_SPLIT, split)
            e1.parse_arrays(conf, paf, 48, params)      # stride divisible by every tested factor
            runs.append([e1.peaks(f) for f in range(3)])
        e1.close()
        with_chain = runs[0]
        assert all(r == with_chain for r in runs)
        if thr > 0 and up in (3, 8):
            for f in range(3):
                want = oracle_run(conf[f], paf[f], topo, params, 48)
                assert with_chain[f] == want.peaks, f"frame {f}"


@pytest.mark.parametrize("up", [1, 8])
def test_split_paths_agree(topo, up):
    """The split kernels (corner: scan + finish + crowded; parse: peaks + pair
    scoring over all frames + finish) give the one-kernel paths' peaks,
    connections and records on procedural, crowded and random frames."""
    rng = np.random.default_rng(99)
    scenes = [synth.procedural_scene(77, s, 656, 368, SP) for s in range(6)] + [synth.crowd_scene(11, s) for s in range(2)]
    conf, paf = render(scenes, topo)
    conf[5, :topo.n_keypoints] = rng.random(conf.shape[1:])[:topo.n_keypoints].astype(np.float32)   # noise part maps
    params = pf.ParserParams(upsample=up)
    e = pf.PafParser(topo, debug=True)
    out = []
    for corner_split, parse_split in ((2, 2), (0, 0), (2, 0), (0, 2)):   # 2: always split
        e.ctx.set_option(pf._native.PF_OPT_CORNER_SPLIT, corner_split)
        e.ctx.set_option(pf._native.PF_OPT_PARSE_SPLIT, parse_split)
        got = e.parse_arrays(conf, paf, 8, params)
        out.append(([e.peaks(f) for f in range(len(scenes))], [e.connections(f) for f in range(len(scenes))],
                    [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))]))
    e.close()
    assert all(o == out[0] for o in out)
    for f in (0, 6):
        want = oracle_run(conf[f], paf[f], topo, params)
        assert out[0][2][f] == record_of(want.humans, topo, f)


def test_large_maps_take_the_split_kernels(eng, topo):
    """135x240 maps (1080x1920 input): too large for the one-kernel corner
    form, so even a 2-frame batch runs k_nms_up_scan -> k_corner_finish; the
    peaks and records equal the oracle's and the materialised path's."""
    scenes = [synth.procedural_scene(31, s, 1920, 1080, SP) for s in range(2)]
    conf, paf = render(scenes, topo)
    assert conf.shape[2:] == (135, 240)
    params = pf.ParserParams(upsample=8)
    e = pf.PafParser(topo, debug=True)
    e.set_timing(True)
    e.kernel_times(reset=True)
    got = e.parse_arrays(conf, paf, 8, params)
    kt = e.kernel_times(reset=True)
    assert "k_nms_up_scan" in kt and "k_corner_finish" in kt, kt
    split = [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))]
    peaks = [e.peaks(f) for f in range(len(scenes))]
    e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 1)
    got = e.parse_arrays(conf, paf, 8, params)
    assert [pf.pose_record(f, got.poses(f), topo) for f in range(len(scenes))] == split
    assert [e.peaks(f) for f in range(len(scenes))] == peaks
    e.close()
    want = oracle_run(conf[0], paf[0], topo, params)
    assert split[0] == record_of(want.humans, topo, 0)
