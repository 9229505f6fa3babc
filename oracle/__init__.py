"""CPU oracle for the pose-parsing hot path — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``liborc.so`` (``pf_oracle.c``), a C restatement of the
reference ``poseflow`` path (``/root/reference/pkg/src/poseflow``):

* ``nms_peaks``      — ``paf.py:74-109``
* ``score_limb``     — ``paf.py:112-146``
* ``parse``          — ``paf.py:292-305`` (peaks, ``connect_limbs``
  ``paf.py:149-199``, ``assemble_humans`` ``paf.py:210-289``)
* ``parse_upsampled``— Mode U: ``operators.bilinear_resize``
  (``operators.py:79-107``) on every channel, then ``parse(stride/up)``
* ``resize_chw`` / ``resize_hwc`` / ``preprocess`` — ``operators.py:79-131``
  with ``formats.read_ppm``'s ``u8/255`` (``formats.py:116-117``)
* ``blur_chw``       — separable Gaussian, no reference (parity unpinned)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker
or the CPU baseline.  The product package never imports it.

Pinned by ``tests/test_oracle_golden.py`` against fixtures the reference
itself produced (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None


def build() -> str:
    """Compile liborc.so with the committed Makefile (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(os.path.join(_HERE, f)) for f in ("pf_oracle.c", "pf_oracle.h")
    ):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    c_int, c_double = ctypes.c_int, ctypes.c_double
    lib.orc_u8_to_f32.argtypes = [u8p, ctypes.c_int64, f32p]
    lib.orc_resize_chw.argtypes = [f32p, c_int, c_int, c_int, f32p, c_int, c_int]
    lib.orc_resize_hwc.argtypes = [f32p, c_int, c_int, c_int, f32p, c_int, c_int]
    lib.orc_preprocess.argtypes = [u8p, c_int, c_int, f32p, c_int, c_int]
    lib.orc_nms_peaks.argtypes = [f32p, c_int, c_int, c_double, c_int,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, c_int]
    lib.orc_score_limb.argtypes = [f32p, f32p, c_int, c_int, c_int, c_int, c_int, c_int,
                                   c_int, c_double, ctypes.POINTER(c_double),
                                   ctypes.POINTER(c_double)]
    lib.orc_score_limb.restype = None
    lib.orc_greedy_select.argtypes = [f64p, i32p, i32p, c_int, i32p]
    lib.orc_py_sum.argtypes = [f64p, c_int]
    lib.orc_py_sum.restype = c_double
    lib.orc_parse.argtypes = [f32p, f32p, c_int, c_int, i32p, i32p, c_int, c_int, c_int,
                              ctypes.c_void_p, ctypes.c_void_p]
    lib.orc_parse_upsampled.argtypes = [f32p, f32p, c_int, c_int, i32p, i32p, c_int, c_int,
                                        c_int, c_int, ctypes.c_void_p, c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]
    lib.orc_blur_chw.argtypes = [f32p, c_int, c_int, c_int, f64p, c_int]
    _lib = lib
    return lib


class _Params(ctypes.Structure):
    _fields_ = [
        ("conf_threshold", ctypes.c_double),
        ("nms_window", ctypes.c_int32),
        ("n_samples", ctypes.c_int32),
        ("sample_dot_threshold", ctypes.c_double),
        ("good_fraction_min", ctypes.c_double),
        ("min_parts", ctypes.c_int32),
        ("min_human_score", ctypes.c_double),
    ]


class _Result(ctypes.Structure):
    _fields_ = [
        ("n_peaks", ctypes.c_int32), ("peaks_cap", ctypes.c_int32),
        ("peak_part", ctypes.c_void_p), ("peak_i", ctypes.c_void_p),
        ("peak_j", ctypes.c_void_p), ("peak_score", ctypes.c_void_p),
        ("n_conns", ctypes.c_int32), ("conns_cap", ctypes.c_int32),
        ("conn_limb", ctypes.c_void_p), ("conn_a", ctypes.c_void_p),
        ("conn_b", ctypes.c_void_p), ("conn_score", ctypes.c_void_p),
        ("conn_good", ctypes.c_void_p),
        ("n_humans", ctypes.c_int32), ("humans_cap", ctypes.c_int32),
        ("n_keypoints", ctypes.c_int32),
        ("human_score", ctypes.c_void_p), ("human_n_parts", ctypes.c_void_p),
        ("kp_x", ctypes.c_void_p), ("kp_y", ctypes.c_void_p),
        ("kp_score", ctypes.c_void_p), ("kp_peak", ctypes.c_void_p),
    ]


@dataclass
class OracleParse:
    """Per-frame oracle output: stage intermediates plus humans.

    ``humans`` entries are ``(score, n_parts, keypoints)`` with ``keypoints``
    a K-tuple of ``None`` or ``(x, y, score)`` — the fields of the
    reference ``HumanPose`` (``types.py:208-214``).
    """

    peaks: List[Tuple[int, int, int, float, int]]       # (part, i, j, score, id)
    connections: List[Tuple[int, int, int, float, float]]  # (limb, id_a, id_b, score, good)
    humans: List[Tuple[float, int, Tuple[Optional[Tuple[float, float, float]], ...]]]


def _params(p) -> _Params:
    return _Params(float(p.conf_threshold), int(p.nms_window), int(p.n_samples),
                   float(p.sample_dot_threshold), float(p.good_fraction_min),
                   int(p.min_parts), float(p.min_human_score))


def _topo_arrays(topo):
    limbs = np.ascontiguousarray(np.asarray(topo.limbs, dtype=np.int32).reshape(-1, 2))
    ch = np.ascontiguousarray(np.asarray(topo.paf_channels, dtype=np.int32).reshape(-1, 2))
    return len(topo.keypoint_names), limbs.shape[0], limbs, ch


_ERRS = {1: "config", 2: "contract", 4: "alloc"}


def _run(fn_name, conf, paf, topo, params, extra, caps=(8192, 8192, 4096)):
    lib = _load()
    K, L, limbs, ch = _topo_arrays(topo)
    conf = np.ascontiguousarray(conf, dtype=np.float32)
    paf = np.ascontiguousarray(paf, dtype=np.float32)
    if paf.size == 0:
        paf = np.zeros((1,), np.float32)
    pc, cc, hc = caps
    bufs = dict(
        peak_part=np.zeros(pc, np.int32), peak_i=np.zeros(pc, np.int32),
        peak_j=np.zeros(pc, np.int32), peak_score=np.zeros(pc, np.float32),
        conn_limb=np.zeros(cc, np.int32), conn_a=np.zeros(cc, np.int32),
        conn_b=np.zeros(cc, np.int32), conn_score=np.zeros(cc, np.float64),
        conn_good=np.zeros(cc, np.float64),
        human_score=np.zeros(hc, np.float64), human_n_parts=np.zeros(hc, np.int32),
        kp_x=np.zeros(hc * K, np.float64), kp_y=np.zeros(hc * K, np.float64),
        kp_score=np.zeros(hc * K, np.float32), kp_peak=np.zeros(hc * K, np.int32),
    )
    res = _Result()
    res.peaks_cap, res.conns_cap, res.humans_cap = pc, cc, hc
    for k, v in bufs.items():
        setattr(res, k, v.ctypes.data)
    prm = _params(params)
    h, w = conf.shape[-2], conf.shape[-1]
    args = [conf, paf, K, L, limbs, ch, h, w] + list(extra) + [ctypes.byref(prm), ctypes.byref(res)]
    rc = getattr(lib, fn_name)(*args)
    if rc == 3:
        return _run(fn_name, conf, paf, topo, params, extra,
                    caps=(max(pc, res.n_peaks), max(cc, res.n_conns), max(hc, res.n_humans)))
    if rc:
        raise ValueError(f"oracle {fn_name} failed: {_ERRS.get(rc, rc)}")
    peaks = [(int(bufs["peak_part"][q]), int(bufs["peak_i"][q]), int(bufs["peak_j"][q]),
              float(bufs["peak_score"][q]), q) for q in range(res.n_peaks)]
    conns = [(int(bufs["conn_limb"][q]), int(bufs["conn_a"][q]), int(bufs["conn_b"][q]),
              float(bufs["conn_score"][q]), float(bufs["conn_good"][q]))
             for q in range(res.n_conns)]
    humans = []
    for q in range(res.n_humans):
        kps = []
        for k in range(K):
            o = q * K + k
            if bufs["kp_peak"][o] < 0:
                kps.append(None)
            else:
                kps.append((float(bufs["kp_x"][o]), float(bufs["kp_y"][o]),
                            float(bufs["kp_score"][o])))
        humans.append((float(bufs["human_score"][q]), int(bufs["human_n_parts"][q]), tuple(kps)))
    return OracleParse(peaks, conns, humans)


def parse(conf: np.ndarray, paf: np.ndarray, topo, params, stride: int) -> OracleParse:
    """Mode R oracle: ``paf.parse`` (paf.py:292-305) on [K+1,h,w] / [2L,h,w]."""
    return _run("orc_parse", conf, paf, topo, params, [int(stride)])


def parse_upsampled(conf, paf, topo, params, stride: int, up: int,
                    blur_taps: Optional[np.ndarray] = None) -> OracleParse:
    """Mode U oracle: bilinear_resize every channel by ``up`` then parse(stride/up)."""
    if blur_taps is None or len(blur_taps) <= 1:
        taps_ptr, r = None, 0
        taps = None
    else:
        taps = np.ascontiguousarray(blur_taps, dtype=np.float64)
        taps_ptr, r = taps.ctypes.data, (len(taps) - 1) // 2
    return _run("orc_parse_upsampled", conf, paf, topo, params,
                [int(stride), int(up), taps_ptr, r])


def nms_peaks(conf: np.ndarray, conf_threshold: float, nms_window: int):
    """``paf.nms_peaks`` cells and scores in output order: [(i, j, score)]."""
    lib = _load()
    conf = np.ascontiguousarray(conf, dtype=np.float32)
    h, w = conf.shape
    n = lib.orc_nms_peaks(conf, h, w, float(conf_threshold), int(nms_window), None, None, None, 0)
    oi = np.zeros(max(n, 1), np.int32)
    oj = np.zeros(max(n, 1), np.int32)
    os_ = np.zeros(max(n, 1), np.float32)
    lib.orc_nms_peaks(conf, h, w, float(conf_threshold), int(nms_window),
                      oi.ctypes.data, oj.ctypes.data, os_.ctypes.data, n)
    return [(int(oi[k]), int(oj[k]), float(os_[k])) for k in range(n)]


def score_limb(paf: np.ndarray, topo, limb: int, cell_a, cell_b, n_samples: int,
               sample_dot_threshold: float) -> Tuple[float, float]:
    lib = _load()
    cx, cy = topo.paf_channels[limb]
    px = np.ascontiguousarray(paf[cx], dtype=np.float32)
    py = np.ascontiguousarray(paf[cy], dtype=np.float32)
    s, g = ctypes.c_double(), ctypes.c_double()
    lib.orc_score_limb(px, py, px.shape[0], px.shape[1], int(cell_a[0]), int(cell_a[1]),
                       int(cell_b[0]), int(cell_b[1]), int(n_samples),
                       float(sample_dot_threshold), ctypes.byref(s), ctypes.byref(g))
    return s.value, g.value


def greedy_select(candidates):
    """``paf._greedy_select`` (paf.py:168-182): candidates are
    ``(id_a, id_b, score)``; returns the accepted ones in acceptance order."""
    lib = _load()
    n = len(candidates)
    sc = np.ascontiguousarray([c[2] for c in candidates] or [0.0], dtype=np.float64)
    ia = np.ascontiguousarray([c[0] for c in candidates] or [0], dtype=np.int32)
    ib = np.ascontiguousarray([c[1] for c in candidates] or [0], dtype=np.int32)
    out = np.zeros(max(n, 1), np.int32)
    m = lib.orc_greedy_select(sc, ia, ib, n, out)
    return [candidates[int(out[q])] for q in range(m)]


def py_sum(values: Sequence[float]) -> float:
    lib = _load()
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    return lib.orc_py_sum(arr if arr.size else np.zeros(1), int(arr.size))


def resize_chw(src: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    lib = _load()
    src = np.ascontiguousarray(src, dtype=np.float32)
    c, h, w = src.shape
    dst = np.empty((c, out_h, out_w), np.float32)
    rc = lib.orc_resize_chw(src, c, h, w, dst, out_h, out_w)
    if rc:
        raise ValueError("resize extents")
    return dst


def resize_hwc(src: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    lib = _load()
    src = np.ascontiguousarray(src, dtype=np.float32)
    h, w, c = src.shape
    dst = np.empty((out_h, out_w, c), np.float32)
    rc = lib.orc_resize_hwc(src, h, w, c, dst, out_h, out_w)
    if rc:
        raise ValueError("resize extents")
    return dst


def preprocess(src_u8: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    lib = _load()
    src = np.ascontiguousarray(src_u8, dtype=np.uint8)
    h, w, _ = src.shape
    dst = np.empty((3, out_h, out_w), np.float32)
    rc = lib.orc_preprocess(src, h, w, dst, out_h, out_w)
    if rc:
        raise ValueError("preprocess extents")
    return dst


def blur_chw(maps: np.ndarray, taps: np.ndarray) -> np.ndarray:
    lib = _load()
    out = np.ascontiguousarray(maps, dtype=np.float32).copy()
    taps = np.ascontiguousarray(taps, dtype=np.float64)
    c, h, w = out.shape
    lib.orc_blur_chw(out, c, h, w, taps, (len(taps) - 1) // 2)
    return out
