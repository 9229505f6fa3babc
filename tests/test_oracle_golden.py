"""Pin the CPU oracle (oracle/pf_oracle.c) against fixtures the reference
itself produced (tests/golden/make_golden.py).  CPU only."""

import json
import math

import numpy as np
import pytest

import oracle
from conftest import golden_path, record_of


class P:
    conf_threshold = 0.10
    nms_window = 3
    n_samples = 10
    sample_dot_threshold = 0.05
    good_fraction_min = 0.8
    min_parts = 4
    min_human_score = 0.2

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)


def test_nms_matches_reference_nms_peaks():
    g = np.load(golden_path("nms_golden.npz"))
    off = 0
    for i, conf in enumerate(g["maps"]):
        n = int(g["counts"][i])
        want = [(int(c[0]), int(c[1]), float(s)) for c, s in
                zip(g["cells"][off:off + n], g["scores"][off:off + n])]
        off += n
        got = oracle.nms_peaks(conf, float(g["thresholds"][i]), int(g["windows"][i]))
        assert got == want, f"case {i}"


def test_nms_window5_matches_reference():
    g = np.load(golden_path("nms_golden.npz"))
    off = 0
    for i, conf in enumerate(g["w5_maps"]):
        n = int(g["w5_counts"][i])
        want = [(int(c[0]), int(c[1]), float(s)) for c, s in
                zip(g["w5_cells"][off:off + n], g["w5_scores"][off:off + n])]
        off += n
        assert oracle.nms_peaks(conf, 0.1, 5) == want


def test_nms_known_answers():
    z = np.zeros((8, 8), np.float32)
    assert oracle.nms_peaks(z, 0.1, 3) == []
    one = z.copy(); one[3, 4] = 1.0
    assert oracle.nms_peaks(one, 0.1, 3) == [(3, 4, 1.0)]                 # test_paf.py:41-48
    plat = z.copy(); plat[2:4, 2:4] = 0.7
    assert [c[:2] for c in oracle.nms_peaks(plat, 0.1, 3)] == [(2, 2)]     # test_paf.py:50-54
    s = z.copy(); s[1, 1] = 0.5; s[5, 5] = 0.9; s[1, 5] = 0.5
    assert [c[:2] for c in oracle.nms_peaks(s, 0.1, 3)] == [(5, 5), (1, 1), (1, 5)]  # :69-78


def test_score_limb_matches_reference(topo):
    g = np.load(golden_path("score_golden.npz"))
    for fld, meta, vals in zip(g["fields"], g["meta"], g["vals"]):
        n, limb, ai, aj, bi, bj = (int(v) for v in meta)
        paf = np.zeros((38, n, n), np.float32)
        cx, cy = topo.paf_channels[limb]
        paf[cx], paf[cy] = fld[0][:n, :n], fld[1][:n, :n]
        s, gd = oracle.score_limb(paf, topo, limb, (ai, aj), (bi, bj), 10, 0.05)
        assert (s, gd) == (float(vals[0]), float(vals[1]))     # bit-exact fp64


def test_greedy_matches_reference():
    with open(golden_path("greedy_golden.json")) as f:
        cases = json.load(f)
    for case in cases:
        cands = [tuple(c) for c in case["candidates"]]
        got = oracle.greedy_select(cands)
        assert [list(c) for c in got] == case["accepted"]


def test_python_sum_semantics():
    rng = np.random.default_rng(0)
    for _ in range(5000):
        n = int(rng.integers(1, 20))
        v = (rng.random(n) * 10.0 ** rng.integers(-5, 17, n)).tolist()
        if rng.random() < 0.3:
            v = [x * (-1) ** int(rng.integers(2)) for x in v]
        assert oracle.py_sum(v) == sum(v)
    assert oracle.py_sum([1e16, 1.0, -1e16]) == sum([1e16, 1.0, -1e16]) == 1.0


@pytest.mark.parametrize("mode", ["R", "U"])
def test_frames_stage_by_stage(topo, golden_frames, mode):
    data, recs = golden_frames
    params = P()
    checked = 0
    for name in recs["names"]:
        if mode not in ("R",) and name not in recs["U"]:
            continue
        conf, paf = data[f"{name}.conf"], data[f"{name}.paf"]
        if mode == "R":
            got = oracle.parse(conf, paf, topo, params, 8)
        else:
            got = oracle.parse_upsampled(conf, paf, topo, params, 8, recs["up"])
        pk, ps = data[f"{name}.{mode}.peaks"], data[f"{name}.{mode}.peak_scores"]
        assert [(p[0], p[1], p[2], p[3]) for p in got.peaks] == \
            [(int(a), int(b), int(c), float(s)) for (a, b, c), s in zip(pk, ps)], name
        cn, cv = data[f"{name}.{mode}.conns"], data[f"{name}.{mode}.conn_vals"]
        assert [(c[0], c[1], c[2], c[3], c[4]) for c in got.connections] == \
            [(int(a), int(b), int(c), float(s), float(gd)) for (a, b, c), (s, gd) in zip(cn, cv)], name
        assert record_of(got.humans, topo) == recs[mode][name], name
        checked += 1
    assert checked >= (9 if mode == "R" else 4)


def test_crowded_frames_exercise_merges(topo, golden_frames):
    """crowded scenes must reach the merge / conflict branches."""
    data, recs = golden_frames
    got = oracle.parse(data["C3_0.conf"], data["C3_0.paf"], topo, P(), 8)
    # more accepted connections than (humans-created) implies merges/appends happened
    assert len(got.connections) > 200 and len(got.humans) >= 20


def test_preprocess_matches_reference():
    import hashlib

    g = np.load(golden_path("preprocess_golden.npz"))
    for idx in range(4):
        img, want = g[f"case{idx}.img"], g[f"case{idx}.out"]
        got = oracle.preprocess(img, want.shape[1], want.shape[2])
        assert got.dtype == np.float32 and np.array_equal(got.view(np.uint32), want.view(np.uint32))
    big = np.random.default_rng(360640).integers(0, 256, size=(360, 640, 3), dtype=np.uint8)
    got = oracle.preprocess(big, 368, 656)
    assert hashlib.sha256(got.tobytes()).digest() == bytes(g["big.sha256"])


def test_resize_exact_copy_and_constant():
    rng = np.random.default_rng(1)
    x = rng.random((3, 6, 8)).astype(np.float32)
    assert np.array_equal(oracle.resize_chw(x, 6, 8), x)                   # operators.py:84-85
    c = np.full((2, 2, 3), 0.37, np.float32)
    assert np.allclose(oracle.resize_hwc(c, 4, 4), 0.37, atol=1e-7)       # test_operators.py:95-98


def test_blur_identity_and_normalised():
    x = np.random.default_rng(3).random((2, 9, 11)).astype(np.float32)
    assert np.array_equal(oracle.blur_chw(x, np.array([1.0])), x)
    const = np.full((1, 7, 7), 0.5, np.float32)
    taps = np.exp(-np.arange(-3, 4) ** 2 / 2.0)
    taps /= taps.sum()
    assert np.allclose(oracle.blur_chw(const, taps), 0.5, atol=1e-7)
