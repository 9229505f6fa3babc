"""Parity on exactly the kernel paths the benchmark times.

The bench times C3 (256 crowded frames) and C5 (8192 frames), which take the
split kernels (``k_nms_up_scan`` -> ``k_corner_finish`` / ``k_corner_crowded``
and ``k_parse_peaks`` -> ``k_score_pairs`` -> ``k_parse_frames<true>``), and
C4 (32 frames of 135x240 maps: the split NMS kernels, the wide one-kernel
parse — at most one frame per SM), not the forms that small test batches
take.  Every frame here is
compared with the oracle (``paf.py:292-305`` composed with
``operators.py:79-107`` for Mode U), and the launch counters prove which
kernels ran.  Also: a 32-keypoint topology through the split parse (the
prefix of ``k_parse_peaks`` at K = 32) and the input-lifetime contract of
``parse_tensors`` when an automatic capacity grows and the call replays.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from conftest import record_of
from support import synth

pytestmark = pytest.mark.gpu
SP = synth.SynthParams()
THREADS = max(1, min(64, os.cpu_count() or 1))


def oracle_records(conf, paf, topo, params, stride=8, idx=None):
    idx = range(conf.shape[0]) if idx is None else idx

    def one(f):
        if params.upsample == 1:
            r = oracle.parse(conf[f], paf[f], topo, params, stride)
        else:
            r = oracle.parse_upsampled(conf[f], paf[f], topo, params, stride, params.upsample)
        return record_of(r.humans, topo, f)

    with ThreadPoolExecutor(THREADS) as ex:
        return list(ex.map(one, idx))


def device_parse(eng, conf, paf, params, stride=8):
    """The bench's call: device-resident maps through pf_parse_device."""
    import torch

    c = torch.from_numpy(conf).cuda()
    q = torch.from_numpy(paf).cuda()
    eng.ctx.kernel_times(reset=True)            # launch counters from here
    eng.parse_tensors(c, q, stride, params)
    res = eng.results()
    return res, {k: n for k, (_, n) in eng.ctx.kernel_times(reset=True).items()}


def records(res, topo, idx=None):
    idx = range(res.n_frames) if idx is None else idx
    return [pf.pose_record(f, res.poses(f), topo) for f in idx]


def test_c3_mode_u_256_crowded_split_path(topo):
    """BASELINE configs[2] exactly as timed: 256 crowded frames, Mode U."""
    scenes = [synth.crowd_scene(42, s) for s in range(256)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    device_parse(eng, conf, paf, params)              # automatic caps grow to the crowd
    res, launches = device_parse(eng, conf, paf, params)
    for k in ("k_nms_up_scan", "k_corner_finish", "k_corner_crowded", "k_parse_peaks", "k_score_pairs",
              "k_parse_frames"):
        assert launches.get(k, 0) >= 1, (k, launches)
    assert "k_nms_up_corner" not in launches
    assert records(res, topo) == oracle_records(conf, paf, topo, params)
    assert res.total_humans > 256 * 20
    eng.close()


def test_c3_mode_r_256_crowded_split_path(topo):
    scenes = [synth.crowd_scene(43, s) for s in range(256)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=1)
    eng = pf.PafParser(topo)
    device_parse(eng, conf, paf, params)
    res, launches = device_parse(eng, conf, paf, params)
    assert launches.get("k_score_pairs", 0) >= 1 and launches.get("k_nms_plane", 0) >= 1
    assert records(res, topo) == oracle_records(conf, paf, topo, params)
    eng.close()


@pytest.mark.parametrize("parse_split", [1, 2])
@pytest.mark.parametrize("people", [6, 40])
def test_c4_mode_u_batch32_split_path(topo, people, parse_split):
    """BASELINE configs[3] as timed: 32 frames of 135x240 maps, Mode U (-> 1080x1920):
    the split NMS kernels with the default (wide one-kernel) parse and with
    the split parse forced."""
    if people == 6:
        scenes = [synth.GroundTruthScene(synth.crowd_scene(9, s, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
                  for s in range(32)]
    else:
        scenes = [synth.crowd_scene(19, s, 1920, 1080, 40, (150.0, 300.0)) for s in range(32)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    assert conf.shape == (32, 19, 135, 240)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    eng.ctx.set_option(pf._native.PF_OPT_PARSE_SPLIT, parse_split)
    device_parse(eng, conf, paf, params)
    res, launches = device_parse(eng, conf, paf, params)
    assert launches.get("k_nms_up_scan", 0) >= 1, launches
    assert (launches.get("k_score_pairs", 0) >= 1) == (parse_split == 2), launches
    assert records(res, topo) == oracle_records(conf, paf, topo, params)
    eng.close()


def _chain_topology(k):
    names = [f"p{i}" for i in range(k)]
    return pf.SkeletonTopology.create(names, [(i, i + 1) for i in range(k - 1)])


def _chain_scenes(k, frames, seed, w=656, h=368):
    """Zig-zag chains of k keypoints, 1-4 per frame, ~14 px between joints."""
    rng = np.random.default_rng(seed)
    scenes = []
    for _ in range(frames):
        humans = []
        for _ in range(int(rng.integers(1, 5))):
            x0, y0 = rng.uniform(40, w - 40), rng.uniform(40, h - 40)
            ang = rng.uniform(0, 2 * np.pi)
            pts = []
            x, y = x0, y0
            for j in range(k):
                pts.append((float(np.clip(x, 0, w - 1e-3)), float(np.clip(y, 0, h - 1e-3))))
                ang += rng.uniform(-0.9, 0.9)
                x += 14.0 * np.cos(ang)
                y += 14.0 * np.sin(ang)
            humans.append(synth.GroundTruthHuman(tuple(pts)))
        scenes.append(synth.GroundTruthScene(tuple(humans), w, h))
    return scenes


@pytest.mark.parametrize("parse_split", [2, 1])
@pytest.mark.parametrize("k", [32, 31])
@pytest.mark.parametrize("up", [1, 8])
def test_max_keypoints_topology_split_parse(k, up, parse_split):
    """PF_MAX_KEYPOINTS = 32 parts through the split parse (forced) and the
    default (wide one-kernel) parse of 40 frames."""
    topo = _chain_topology(k)
    conf, paf = synth.render_batch(_chain_scenes(k, 40, 100 + k), topo, SP)
    params = pf.ParserParams(upsample=up, min_parts=4)
    eng = pf.PafParser(topo)
    eng.ctx.set_option(pf._native.PF_OPT_PARSE_SPLIT, parse_split)
    res, launches = device_parse(eng, conf, paf, params)
    assert (launches.get("k_parse_peaks", 0) >= 1) == (parse_split == 2), launches
    assert records(res, topo) == oracle_records(conf, paf, topo, params)
    assert res.total_humans >= 40
    eng.close()


def test_inputs_survive_capacity_replay(topo):
    """parse_tensors on non-contiguous maps whose crowd overflows the automatic
    capacities: the call replays inside results() from the .contiguous()
    temporaries, after the caller dropped its tensors and the caching
    allocator handed that memory to new tensors filled with garbage."""
    import torch

    scenes = [synth.crowd_scene(77, s) for s in range(40)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8)
    want = oracle_records(conf, paf, topo, params)
    eng = pf.PafParser(topo)     # fresh context: default (automatic) capacities
    # non-contiguous views: channels-last storage permuted back to NCHW
    c = torch.from_numpy(np.ascontiguousarray(conf.transpose(0, 2, 3, 1))).cuda().permute(0, 3, 1, 2)
    q = torch.from_numpy(np.ascontiguousarray(paf.transpose(0, 2, 3, 1))).cuda().permute(0, 3, 1, 2)
    assert not c.is_contiguous() and not q.is_contiguous()
    eng.parse_tensors(c, q, 8, params)
    del c, q
    junk = [torch.full((conf.size + paf.size,), float("nan"), device="cuda") for _ in range(4)]
    junk += [torch.full((conf.size,), 1.0, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    launched = eng.launch_count()
    res = eng.results()
    assert eng.launch_count() > launched          # the call was replayed with grown capacities
    del junk
    assert records(res, topo) == want
    eng.close()


@pytest.mark.parametrize("sigma", [1.0, 2.0])
def test_fused_blur_batch_vs_oracle_and_materialised(topo, sigma):
    """k_up_blur_nms (upsample -> blur -> 3x3 NMS fused, split parse at 40
    frames) against the oracle (bilinear_resize x8 -> blur_chw -> parse) on
    every frame, and against the materialised path (k_resize_planes ->
    k_blur_rows/cols -> k_nms_plane)."""
    scenes = [synth.procedural_scene(61, s, 656, 368, SP) for s in range(38)] + \
             [synth.crowd_scene(62, 0), synth.crowd_scene(62, 1)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8, blur_sigma=sigma)
    eng = pf.PafParser(topo)
    res, launches = device_parse(eng, conf, paf, params)
    assert launches.get("k_up_blur_nms", 0) >= 1, launches
    got = records(res, topo)
    taps = pf._native.gaussian_taps(sigma)

    def one(f):
        r = oracle.parse_upsampled(conf[f], paf[f], topo, params, 8, 8, taps)
        return record_of(r.humans, topo, f)

    with ThreadPoolExecutor(THREADS) as ex:
        want = list(ex.map(one, range(conf.shape[0])))
    assert got == want
    eng.set_materialise(True)
    mat, launches = device_parse(eng, conf, paf, params)
    assert launches.get("k_blur_rows", 0) >= 1 and "k_up_blur_nms" not in launches, launches
    assert records(mat, topo) == got
    eng.close()


def test_fused_blur_1080p_tiles(topo):
    """1080x1920 output (8 column tiles per plane) with blur, vs the oracle."""
    scenes = [synth.GroundTruthScene(synth.crowd_scene(91, s, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
              for s in range(2)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8, blur_sigma=1.5)
    eng = pf.PafParser(topo)
    res, launches = device_parse(eng, conf, paf, params)
    assert launches.get("k_up_blur_nms", 0) >= 1, launches
    taps = pf._native.gaussian_taps(1.5)
    want = [record_of(oracle.parse_upsampled(conf[f], paf[f], topo, params, 8, 8, taps).humans, topo, f)
            for f in range(2)]
    assert records(res, topo) == want
    eng.close()


def test_paf_sector_count_instrumentation(topo):
    """PF_OPT_COUNT_PAF (the bench's in-run count of the PAF bytes an in-place
    PAF moves): same results as the uninstrumented call, deterministic, and
    bounded by the frame's PAF sectors."""
    scenes = [synth.procedural_scene(71, s, 656, 368, SP) for s in range(48)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    want = records(eng.parse_arrays(conf, paf, 8, params), topo)
    eng.ctx.set_option(pf._native.PF_OPT_COUNT_PAF, 1)
    got = records(eng.parse_arrays(conf, paf, 8, params), topo)
    n1 = eng.ctx.paf_sectors()
    eng.parse_arrays(conf, paf, 8, params)
    n2 = eng.ctx.paf_sectors()
    eng.ctx.set_option(pf._native.PF_OPT_COUNT_PAF, 0)
    assert got == want
    assert n1 == n2 and 0 < n1 <= 48 * paf[0].nbytes // 32
    # every sampled pair touches at least 2 sectors (x and y channels)
    assert n1 * 32 / 48 > 1000
    eng.close()


@pytest.mark.parametrize("grid, patch", [((46, 82), 30), ((135, 240), 72)])
def test_crowded_plane_kernel_stress(topo, grid, patch):
    """k_corner_crowded on adversarial planes — uniform noise patches above
    the threshold (hundreds to thousands of hot cells, most of them
    non-monotone, hot-list / dense-list overflow on the 135x240 grid, which
    is also too large to stage in shared memory) and ties from quantised
    noise — against the materialised path (resize + plane NMS over HBM maps)
    through the split path (forced: 32 frames of 46x82 maps would take the
    one-kernel corner form by default)."""
    rng = np.random.default_rng(grid[0] + patch)
    F, K = 32, topo.n_keypoints
    h, w = grid
    conf = np.zeros((F, K + 1, h, w), np.float32)
    for f in range(3):
        for k in (0, 5, 11):
            y0, x0 = rng.integers(0, h - patch), rng.integers(0, w - patch)
            m = rng.random((patch, patch)).astype(np.float32)
            if k == 5:
                m = np.round(m * 4) / 4                  # plateaus and ties
            conf[f, k, y0:y0 + patch, x0:x0 + patch] = m
    paf = np.zeros((F, 2 * topo.n_limbs, h, w), np.float32)
    e = pf.PafParser(topo, debug=True)
    e.ctx.set_option(pf._native.PF_OPT_CORNER_SPLIT, 2)
    params = pf.ParserParams(upsample=8)
    e.set_timing(True)
    e.kernel_times(reset=True)
    e.parse_arrays(conf, paf, 8, params)
    kt = e.kernel_times(reset=True)
    assert "k_nms_up_scan" in kt and "k_corner_crowded" in kt, kt
    split = [e.peaks(f) for f in range(F)]
    e.ctx.set_option(pf._native.PF_OPT_MATERIALISE, 1)
    e.parse_arrays(conf, paf, 8, params)
    assert [e.peaks(f) for f in range(F)] == split
    assert sum(len(p) for p in split) > 1000
    e.close()
