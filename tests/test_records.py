"""Native poses.jsonl formatting (pf_format_records / pf_format_float, SURVEY
§8(f) 3): byte-identical to the reference pose_record (operators.py:293-310),
i.e. json.dumps with CPython float repr.  Host-only: runs without a GPU."""

import ctypes
import json
import struct

import numpy as np
import pytest

import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native
from paper_2108_11826_b200.parser import format_records


def fmt(v: float) -> str:
    lib = _native.load_library()
    buf = ctypes.create_string_buffer(64)
    n = lib.pf_format_float(float(v), buf, 64)
    assert n > 0
    return buf.value.decode()


EDGE = [0.0, -0.0, 1.0, -1.0, 0.1, 0.2, 0.3, 1 / 3, 2 / 3, 1e-5, 1e-4, 9.999e-5, 0.0001, 0.001, 1e15, 1e16,
        9999999999999998.0, 1234567890123456.0, 12345678901234567.0, 5e-324, 2.2250738585072014e-308,
        1.7976931348623157e308, 123.0, 100.0, 0.5, 2.5e-7, 655.5, 367.0, 1e22, 1e23, float("inf"),
        float("-inf"), float("nan")]


def test_float_repr_edge_cases():
    for v in EDGE:
        assert fmt(v) == json.dumps(v), v


def test_float_repr_random_doubles():
    rng = np.random.default_rng(1234)
    bits = rng.integers(0, 2 ** 63, size=60000, dtype=np.int64)
    vals = [struct.unpack("<d", struct.pack("<q", int(b)))[0] for b in bits]
    vals += list(rng.random(30000) * 1000)
    vals += [float(np.float32(x)) for x in rng.random(30000)]            # keypoint scores are fp32
    vals += [float(x) + 0.5 for x in rng.integers(0, 656, 5000)]         # cell_to_pixel coordinates
    vals += list(10.0 ** rng.uniform(-8, 20, 20000))
    for v in vals:
        v = float(v)
        if v != v:
            continue
        assert fmt(v) == json.dumps(v), v           # json.dumps: repr() for finite floats


class _Fake:
    """A BatchResult-shaped SoA batch built on the host."""

    def __init__(self, rng, n_frames, k):
        counts = rng.integers(0, 5, n_frames).astype(np.int32)
        self.n_frames, self.n_keypoints = n_frames, k
        self.frame_count = counts
        self.frame_first = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
        total = int(counts.sum())
        self.total_humans = total
        self.human_score = rng.random(total) * 3
        self.human_n_parts = rng.integers(1, k + 1, total).astype(np.int32)
        self.kp_x = (rng.integers(0, 656, (total, k)) + 0.5 * rng.integers(0, 2, (total, k))).astype(np.float64)
        self.kp_y = rng.random((total, k)) * 368
        self.kp_score = rng.random((total, k)).astype(np.float32)
        self.kp_peak = np.where(rng.random((total, k)) < 0.3, -1, rng.integers(0, 500, (total, k))).astype(np.int32)

    def poses(self, f):
        out = []
        for h in range(self.frame_first[f], self.frame_first[f] + self.frame_count[f]):
            kps = tuple(None if self.kp_peak[h, k] < 0 else
                        pf.Keypoint(float(self.kp_x[h, k]), float(self.kp_y[h, k]), float(self.kp_score[h, k]))
                        for k in range(self.n_keypoints))
            out.append(pf.HumanPose(keypoints=kps, score=float(self.human_score[h]),
                                    n_parts=int(self.human_n_parts[h])))
        return out


@pytest.mark.parametrize("seq_base", [0, 1000])
def test_records_match_pose_record(seq_base):
    topo = pf.load_topology("coco18")
    rng = np.random.default_rng(7 + seq_base)
    fake = _Fake(rng, 200, topo.n_keypoints)
    got = format_records(fake, topo, seq_base)
    want = [pf.pose_record(seq_base + f, fake.poses(f), topo) for f in range(fake.n_frames)]
    assert got == want


def test_records_empty_batch():
    topo = pf.load_topology("coco18")
    fake = _Fake(np.random.default_rng(0), 0, topo.n_keypoints)
    assert format_records(fake, topo) == []


def test_records_non_ascii_part_names():
    # json.dumps(ensure_ascii=True) escapes by code point: é for U+00E9,
    # 中 for a BMP ideograph, a surrogate pair for U+1F600; control and
    # DEL characters as \u00XX; quotes and backslashes by their short forms
    names = ["nosé", "中心", "smile\U0001F600", "tab\tq\"b\\", "del\x7f", "ctl\x01",
             "ÿĀ߿ࠀ￿", "plain"]
    limbs = [(k, k + 1) for k in range(len(names) - 1)]
    topo = pf.SkeletonTopology.create(names, limbs)
    rng = np.random.default_rng(99)
    fake = _Fake(rng, 40, topo.n_keypoints)
    got = format_records(fake, topo, 5)
    want = [pf.pose_record(5 + f, fake.poses(f), topo) for f in range(fake.n_frames)]
    assert got == want
