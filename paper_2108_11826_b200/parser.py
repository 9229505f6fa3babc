"""PAF pose parsing on B200 — drop-in for ``poseflow.paf`` (``paf.py``).

Public surface (reference lines in brackets):

* ``ParserParams``  [paf.py:34-54] — same seven fields, defaults and
  ``validate()`` errors, plus ``upsample`` (1 = parse the feature grid as
  the reference does; 8 = HyperPose-style x8 bilinear upsample first) and
  ``blur_sigma`` (0 = off).
* ``parse(maps, topo, params)`` [paf.py:292-305] — one frame, returns a new
  ``List[HumanPose]``; raises ``ConfigError``/``ContractError`` before any
  device work.  Pure and deterministic: the GPU result equals the reference's
  bit for bit (peaks, connections, assignment, scores).
* ``parse_batch`` / ``parse_arrays`` / ``PafParser.parse_device`` — the
  batched forms the GPU is built for (SoA results, lazy ``HumanPose``).

Every call goes through ``libpf_b200.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native
from .core import FeatureMaps, HumanPose, Keypoint, SkeletonTopology
from .errors import CapacityError, ConfigError, ContractError, DeviceError


@dataclass
class ParserParams:
    conf_threshold: float = 0.10
    nms_window: int = 3
    n_samples: int = 10
    sample_dot_threshold: float = 0.05
    good_fraction_min: float = 0.8
    min_parts: int = 4
    min_human_score: float = 0.2
    # B200-path extensions (not in the reference; defaults = reference behaviour)
    upsample: int = 1
    blur_sigma: float = 0.0

    def validate(self) -> None:
        # paf.py:44-54, same order and messages
        if self.nms_window < 3 or self.nms_window % 2 == 0:
            raise ConfigError("nms_window must be odd and >= 3")
        if self.n_samples < 2:
            raise ConfigError("n_samples must be >= 2")
        for name in ("conf_threshold", "sample_dot_threshold", "good_fraction_min"):
            value = getattr(self, name)
            if not (0.0 <= value <= 1.0):
                raise ConfigError(f"{name} must be in [0, 1], got {value}")
        if self.min_parts < 1:
            raise ConfigError("min_parts must be >= 1")
        if int(self.upsample) != self.upsample or self.upsample < 1:
            raise ConfigError("upsample must be an integer >= 1")
        if not (self.blur_sigma >= 0.0) or self.blur_sigma == float("inf"):
            raise ConfigError("blur_sigma must be finite and >= 0")

    def to_native(self) -> _native.PfParams:
        return _native.PfParams(float(self.conf_threshold), int(self.nms_window),
                                int(self.n_samples), float(self.sample_dot_threshold),
                                float(self.good_fraction_min), int(self.min_parts),
                                float(self.min_human_score), int(self.upsample),
                                float(self.blur_sigma))


def _params_of(params) -> ParserParams:
    """Accept our ParserParams or any object with the reference's fields."""
    if isinstance(params, ParserParams):
        return params
    return ParserParams(**{f: getattr(params, f) for f in (
        "conf_threshold", "nms_window", "n_samples", "sample_dot_threshold",
        "good_fraction_min", "min_parts", "min_human_score")},
        upsample=getattr(params, "upsample", 1), blur_sigma=getattr(params, "blur_sigma", 0.0))


class BatchResult:
    """Humans of a batch as structure-of-arrays (a copy of the C ABI's
    ``pf_results``); ``poses(f)`` materialises ``HumanPose`` objects lazily."""

    def __init__(self, res: _native.PfResults):
        n, total, k = res.n_frames, res.total_humans, res.n_keypoints
        self.n_frames, self.total_humans, self.n_keypoints = n, total, k

        def arr(ptr, count, dtype):
            if count <= 0:
                return np.zeros(0, dtype)
            return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)

        self.frame_first = arr(res.frame_first, n, np.int32)
        self.frame_count = arr(res.frame_count, n, np.int32)
        self.human_score = arr(res.human_score, total, np.float64)
        self.human_n_parts = arr(res.human_n_parts, total, np.int32)
        self.kp_x = arr(res.kp_x, total * k, np.float64).reshape(total, k)
        self.kp_y = arr(res.kp_y, total * k, np.float64).reshape(total, k)
        self.kp_score = arr(res.kp_score, total * k, np.float32).reshape(total, k)
        self.kp_peak = arr(res.kp_peak, total * k, np.int32).reshape(total, k)

    def poses(self, frame: int) -> List[HumanPose]:
        first, count = int(self.frame_first[frame]), int(self.frame_count[frame])
        out = []
        for h in range(first, first + count):
            kps = []
            for k in range(self.n_keypoints):
                if self.kp_peak[h, k] < 0:
                    kps.append(None)
                else:
                    kps.append(Keypoint(x=float(self.kp_x[h, k]), y=float(self.kp_y[h, k]),
                                        score=float(self.kp_score[h, k])))
            out.append(HumanPose(keypoints=tuple(kps), score=float(self.human_score[h]),
                                 n_parts=int(self.human_n_parts[h])))
        return out

    @classmethod
    def _from_block(cls, block: "_HostBlock", n: int, total: int, k: int) -> "BatchResult":
        """Views into a pinned block that pf_get_results_into filled (no copy);
        the block returns to its pool once every view of it is gone."""
        self = cls.__new__(cls)
        self.n_frames, self.total_humans, self.n_keypoints = n, total, k
        buf = block.buffer()
        off = block.offsets(n, block.capacity, k)

        def view(name, count, dtype):
            return np.frombuffer(buf, dtype=dtype, count=count, offset=off[name])

        self.frame_first = view("ff", n, np.int32)
        self.frame_count = view("fc", n, np.int32)
        self.human_score = view("hs", total, np.float64)
        self.human_n_parts = view("hn", total, np.int32)
        self.kp_x = view("kx", total * k, np.float64).reshape(total, k)
        self.kp_y = view("ky", total * k, np.float64).reshape(total, k)
        self.kp_score = view("ks", total * k, np.float32).reshape(total, k)
        self.kp_peak = view("kp", total * k, np.int32).reshape(total, k)
        return self

    def all_poses(self) -> List[List[HumanPose]]:
        return [self.poses(f) for f in range(self.n_frames)]

    def records(self, topo: SkeletonTopology, seq_base: int = 0) -> List[str]:
        """``pose_record(seq_base + f, poses(f), topo)`` for every frame, built
        natively from the SoA arrays (byte-identical; no HumanPose objects)."""
        return format_records(self, topo, seq_base)


class _HostBlock:
    """One pinned host block holding a parse_arrays result (pf_host_out)."""

    def __init__(self, pool: "_HostPool", ptr: int, nbytes: int, frames: int, capacity: int, k: int):
        self.pool, self.ptr, self.nbytes = pool, ptr, nbytes
        self.frames, self.capacity, self.k = frames, capacity, k

    @staticmethod
    def offsets(frames: int, capacity: int, k: int) -> dict:
        off, o = {}, 0
        for name, size in (("ff", 4 * frames), ("fc", 4 * frames), ("hs", 8 * capacity), ("hn", 4 * capacity),
                           ("kx", 8 * capacity * k), ("ky", 8 * capacity * k), ("ks", 4 * capacity * k),
                           ("kp", 4 * capacity * k)):
            off[name] = o
            o += (size + 63) & ~63
        off["_total"] = o
        return off

    def native(self) -> "_native.PfHostOut":
        off = self.offsets(self.frames, self.capacity, self.k)
        p = self.ptr
        return _native.PfHostOut(self.capacity, p + off["ff"], p + off["fc"], p + off["hs"], p + off["hn"],
                                 p + off["kx"], p + off["ky"], p + off["ks"], p + off["kp"])

    def buffer(self):
        """A fresh ctypes view of the block; the block goes back to the pool
        when it (and every numpy array built on it) is collected."""
        import weakref

        buf = (ctypes.c_char * self.nbytes).from_address(self.ptr)
        weakref.finalize(buf, self.pool.give, self.ptr, self.nbytes)
        return buf


class _HostPool:
    """Recycled pinned blocks for parse_arrays results (pf_host_alloc): the
    device-to-host copies land in the result's own memory (no host copy), and
    a block is reused only after its BatchResult and all views are gone."""

    def __init__(self, lib, keep: int = 3):
        self.lib, self.keep = lib, keep
        self.free: List[tuple] = []
        self.lock = threading.Lock()
        self.closed = False

    def take(self, frames: int, capacity: int, k: int) -> _HostBlock:
        need = _HostBlock.offsets(frames, capacity, k)["_total"]
        with self.lock:
            fit = [b for b in self.free if b[1] >= need]
            if fit:
                best = min(fit, key=lambda b: b[1])
                self.free.remove(best)
                ptr, nbytes = best
            else:
                nbytes = need
                ptr = self.lib.pf_host_alloc(nbytes)
                if not ptr:
                    raise DeviceError(f"pf_host_alloc({nbytes}) failed")
        return _HostBlock(self, ptr, nbytes, frames, capacity, k)

    def give(self, ptr: int, nbytes: int) -> None:
        with self.lock:
            if self.closed:                      # the parser is gone: nothing will reuse it
                self.lib.pf_host_free(ptr)
                return
            self.free.append((ptr, nbytes))
            while len(self.free) > self.keep:
                p, _ = min(self.free, key=lambda b: b[1])
                self.free.remove((p, _))
                self.lib.pf_host_free(p)


class PafParser:
    """A GPU parsing engine bound to one device (one ``pf_ctx``).

    Not reentrant; use one per thread (``parse()`` keeps a thread-local one).
    """

    def __init__(self, topo: SkeletonTopology, device: int = 0,
                 caps: Optional[dict] = None, debug: bool = False):
        c = _native.PfCaps(**(caps or {}))
        self.ctx = _native.Context(device, c)
        self.topo = topo
        self.ctx.set_topology(topo)
        self.device = device
        # the maps of the last parse_tensors call (including .contiguous()
        # temporaries): pf_get_results may replay the call from them when an
        # automatic capacity grows, so they stay alive until results() returns
        self._inflight = None
        self._host_pool = _HostPool(self.ctx.lib)
        self._host_cap = 0
        if debug:
            self.set_debug(True)

    def set_debug(self, enable: bool) -> None:
        self.ctx.check(self.ctx.lib.pf_set_debug(self.ctx.handle, 1 if enable else 0))

    def set_stream(self, stream_handle: int) -> None:
        self.ctx.check(self.ctx.lib.pf_set_stream(self.ctx.handle, ctypes.c_void_p(stream_handle)))

    def launch_count(self) -> int:
        return self.ctx.launch_count()

    def set_timing(self, enable: bool) -> None:
        self.ctx.set_option(_native.PF_OPT_TIMING, 1 if enable else 0)

    def set_materialise(self, enable: bool) -> None:
        """Force the unfused Mode U path (resize -> NMS through HBM)."""
        self.ctx.set_option(_native.PF_OPT_MATERIALISE, 1 if enable else 0)

    def kernel_times(self, reset: bool = False) -> dict:
        return self.ctx.kernel_times(reset)

    def _check_arrays(self, conf_shape, paf_shape, stride):
        k, n_l = self.topo.n_keypoints, self.topo.n_limbs
        if len(conf_shape) != 4 or conf_shape[1] != k + 1:
            raise ContractError(f"conf dims {tuple(conf_shape)} inconsistent with {k} keypoints")
        if len(paf_shape) != 4 or paf_shape[1] != 2 * n_l:
            raise ContractError(f"paf dims {tuple(paf_shape)} inconsistent with {n_l} limbs")
        if conf_shape[0] != paf_shape[0]:
            raise ContractError("conf and paf batch sizes differ")
        if tuple(conf_shape[2:]) != tuple(paf_shape[2:]):
            raise ContractError(f"conf grid {tuple(conf_shape[2:])} != paf grid {tuple(paf_shape[2:])}")
        if stride < 1:
            raise ContractError("stride must be >= 1")

    def parse_arrays(self, conf: np.ndarray, paf: np.ndarray, stride: int,
                     params: ParserParams) -> BatchResult:
        """Host arrays conf [B,K+1,H,W], paf [B,2L,H,W] (f32) -> BatchResult."""
        params = _params_of(params)
        params.validate()
        conf = np.ascontiguousarray(conf, dtype=np.float32)
        paf = np.ascontiguousarray(paf, dtype=np.float32)
        self._check_arrays(conf.shape, paf.shape, stride)
        p = params.to_native()
        b, _, h, w = conf.shape
        self.ctx.check(self.ctx.lib.pf_parse_host(
            self.ctx.handle, conf.ctypes.data if conf.size else None,
            paf.ctypes.data if paf.size else None, b, h, w, int(stride),
            ctypes.byref(p), None))
        return self._host_results(b)

    def _host_results(self, frames: int) -> BatchResult:
        """pf_get_results_into a pooled pinned block sized for the call."""
        k = self.topo.n_keypoints
        cap = max(self._host_cap, 4 * frames, 16)
        n_frames, total = ctypes.c_int32(), ctypes.c_int32()
        while True:
            block = self._host_pool.take(frames, cap, k)
            dst = block.native()
            rc = self.ctx.lib.pf_get_results_into(self.ctx.handle, ctypes.byref(dst), ctypes.byref(n_frames),
                                                  ctypes.byref(total))
            if rc == _native.PF_ERR_CAPACITY and total.value > cap:
                self._host_pool.give(block.ptr, block.nbytes)
                cap = self._host_cap = max(total.value, 2 * cap)
                continue
            if rc:
                self._host_pool.give(block.ptr, block.nbytes)
                self.ctx.check(rc)
            return BatchResult._from_block(block, n_frames.value, total.value, k)

    def parse_device(self, conf_ptr: int, paf_ptr: int, batch: int, grid_h: int, grid_w: int,
                     stride: int, params: ParserParams) -> None:
        """Asynchronous parse of device-resident maps (raw CUDA pointers, the
        FeatureMaps layout batched); collect with ``results()``.  The memory
        behind the pointers must stay valid until ``results()`` returns (a
        capacity grow replays the call from it); ``parse_tensors`` keeps its
        tensors alive itself."""
        self._inflight = None
        p = _params_of(params).to_native()
        self.ctx.check(self.ctx.lib.pf_parse_device(
            self.ctx.handle, ctypes.c_void_p(conf_ptr), ctypes.c_void_p(paf_ptr), int(batch),
            int(grid_h), int(grid_w), int(stride), ctypes.byref(p)))

    def parse_tensors(self, conf, paf, stride: int, params: ParserParams) -> None:
        """torch CUDA tensors [B,K+1,H,W] / [B,2L,H,W] on this engine's device;
        enqueued on torch's current stream."""
        import torch

        params = _params_of(params)
        params.validate()
        self._check_arrays(tuple(conf.shape), tuple(paf.shape), stride)
        if conf.dtype != torch.float32 or paf.dtype != torch.float32:
            raise ContractError("maps must be float32")
        if not (conf.is_cuda and paf.is_cuda):
            raise ContractError("parse_tensors needs CUDA tensors")
        conf = conf.contiguous()
        paf = paf.contiguous()
        self.set_stream(torch.cuda.current_stream(conf.device).cuda_stream)
        b, _, h, w = conf.shape
        self.parse_device(conf.data_ptr(), paf.data_ptr(), b, h, w, stride, params)
        self._inflight = (conf, paf)

    def parse_into(self, conf, paf, stride: int, params: ParserParams, max_humans: int = 64,
                   out: Optional["PoseSlots"] = None, stream=None) -> "PoseSlots":
        """The §8(b) batch entry point (``pf_parse_batch``): torch CUDA maps
        in, caller-owned device slots out (``PoseSlots``, allocated here
        unless ``out`` is given), enqueued on ``stream`` (default: torch's
        current stream) with no host synchronisation.  Valid once that stream
        reaches this point; the maps are needed only until then (no replay:
        capacity overflows land in ``out.status``)."""
        import torch

        params = _params_of(params)
        params.validate()
        self._check_arrays(tuple(conf.shape), tuple(paf.shape), stride)
        if conf.dtype != torch.float32 or paf.dtype != torch.float32:
            raise ContractError("maps must be float32")
        if not (conf.is_cuda and paf.is_cuda):
            raise ContractError("parse_into needs CUDA tensors")
        conf = conf.contiguous()
        paf = paf.contiguous()
        b, _, h, w = conf.shape
        if out is None:
            out = PoseSlots.empty(b, int(max_humans), self.topo.n_keypoints, conf.device)
        elif out.n_humans.shape[0] != b or out.kp_present.shape[2] != self.topo.n_keypoints:
            raise ContractError("output slots do not match the batch / keypoint count")
        st = stream if stream is not None else torch.cuda.current_stream(conf.device)
        p = params.to_native()
        native_out = out.native()
        self.ctx.check(self.ctx.lib.pf_parse_batch(
            self.ctx.handle, ctypes.c_void_p(conf.data_ptr()), ctypes.c_void_p(paf.data_ptr()), int(b),
            int(h), int(w), int(stride), ctypes.byref(p), ctypes.byref(native_out),
            ctypes.c_void_p(st.cuda_stream)))
        # the caching allocator must not reuse the maps before the stream is done with them
        conf.record_stream(st)
        paf.record_stream(st)
        return out

    def results(self) -> BatchResult:
        res = _native.PfResults()
        try:
            self.ctx.check(self.ctx.lib.pf_get_results(self.ctx.handle, ctypes.byref(res)))
            return BatchResult(res)
        finally:
            self._inflight = None

    def peaks(self, frame: int):
        """Debug capture: [(part, row, col, score, id)] in id order."""
        lib, h = self.ctx.lib, self.ctx.handle
        n = ctypes.c_int()
        self.ctx.check(lib.pf_get_peaks(h, frame, ctypes.byref(n), None, None, None, None))
        cnt = max(n.value, 1)
        part, row, col = (np.zeros(cnt, np.int32) for _ in range(3))
        score = np.zeros(cnt, np.float32)
        self.ctx.check(lib.pf_get_peaks(h, frame, ctypes.byref(n), part.ctypes.data,
                                        row.ctypes.data, col.ctypes.data, score.ctypes.data))
        return [(int(part[q]), int(row[q]), int(col[q]), float(score[q]), q)
                for q in range(n.value)]

    def connections(self, frame: int):
        """Debug capture: [(limb, id_a, id_b, score, good_fraction)]."""
        lib, h = self.ctx.lib, self.ctx.handle
        n = ctypes.c_int()
        self.ctx.check(lib.pf_get_connections(h, frame, ctypes.byref(n), None, None, None, None, None))
        cnt = max(n.value, 1)
        limb, ia, ib = (np.zeros(cnt, np.int32) for _ in range(3))
        sc, gd = np.zeros(cnt, np.float64), np.zeros(cnt, np.float64)
        self.ctx.check(lib.pf_get_connections(h, frame, ctypes.byref(n), limb.ctypes.data,
                                              ia.ctypes.data, ib.ctypes.data, sc.ctypes.data,
                                              gd.ctypes.data))
        return [(int(limb[q]), int(ia[q]), int(ib[q]), float(sc[q]), float(gd[q]))
                for q in range(n.value)]

    def close(self) -> None:
        with self._host_pool.lock:
            for ptr, _ in self._host_pool.free:
                self.ctx.lib.pf_host_free(ptr)
            self._host_pool.free.clear()
            self._host_pool.closed = True        # blocks of live results are freed when they die
        self.ctx.close()


class PoseSlots:
    """Caller-owned result slots of ``parse_into`` (torch device tensors,
    the ``pf_out`` SoA): frame f's humans in slots [f, :n_humans[f]], in
    the reference output order (paf.py:288)."""

    def __init__(self, n_humans, human_score, n_parts, kp_xy, kp_score, kp_present, status):
        self.n_humans, self.human_score, self.n_parts = n_humans, human_score, n_parts
        self.kp_xy, self.kp_score, self.kp_present, self.status = kp_xy, kp_score, kp_present, status

    @classmethod
    def empty(cls, batch: int, max_humans: int, n_keypoints: int, device) -> "PoseSlots":
        import torch

        if max_humans < 0:
            raise ContractError("max_humans must be >= 0")
        z = dict(device=device)
        return cls(torch.empty(batch, dtype=torch.int32, **z),
                   torch.empty(batch, max_humans, dtype=torch.float64, **z),
                   torch.empty(batch, max_humans, dtype=torch.int32, **z),
                   torch.empty(batch, max_humans, n_keypoints, 2, dtype=torch.float64, **z),
                   torch.empty(batch, max_humans, n_keypoints, dtype=torch.float32, **z),
                   torch.empty(batch, max_humans, n_keypoints, dtype=torch.uint8, **z),
                   torch.empty(2, dtype=torch.int32, **z))

    def native(self) -> "_native.PfOut":
        return _native.PfOut(int(self.human_score.shape[1]), self.n_humans.data_ptr(),
                             self.human_score.data_ptr(), self.n_parts.data_ptr(), self.kp_xy.data_ptr(),
                             self.kp_score.data_ptr(), self.kp_present.data_ptr(), self.status.data_ptr())

    def check(self) -> None:
        """Synchronise on the slots and raise CapacityError if a frame did not fit."""
        code, frame = (int(v) for v in self.status.cpu())
        if code == _native.PF_ERR_CAPACITY:
            raise CapacityError(f"frame {frame} exceeds a capacity of pf_parse_batch "
                                f"(max_humans {self.human_score.shape[1]} or an internal cap)")
        if code != 0:
            raise DeviceError(f"pf_parse_batch status {code}")

    def poses(self, frame: int) -> List[HumanPose]:
        """Host HumanPose list of one frame (reference types, types.py:208-230)."""
        n = int(self.n_humans[frame])
        sc = self.human_score[frame, :n].cpu().tolist()
        npart = self.n_parts[frame, :n].cpu().tolist()
        xy = self.kp_xy[frame, :n].cpu().tolist()
        ks = self.kp_score[frame, :n].cpu().tolist()
        pr = self.kp_present[frame, :n].cpu().tolist()
        return [HumanPose(keypoints=tuple(Keypoint(x=xy[i][k][0], y=xy[i][k][1], score=ks[i][k]) if pr[i][k] else None
                                          for k in range(len(pr[i]))),
                          score=sc[i], n_parts=npart[i]) for i in range(n)]


_tls = threading.local()
DEFAULT_DEVICE = 0


def default_parser(topo: SkeletonTopology, device: Optional[int] = None) -> PafParser:
    """Thread-local engine per device (contexts are not reentrant)."""
    dev = DEFAULT_DEVICE if device is None else int(device)
    cache = getattr(_tls, "parsers", None)
    if cache is None:
        cache = _tls.parsers = {}
    eng = cache.get(dev)
    if eng is None:
        eng = cache[dev] = PafParser(topo, device=dev)
    else:
        eng.topo = topo
        eng.ctx.set_topology(topo)
    return eng


def _stack_maps(maps_list: Sequence[FeatureMaps], topo: SkeletonTopology):
    strides = {m.stride for m in maps_list}
    grids = {m.grid_shape() for m in maps_list}
    if len(strides) != 1 or len(grids) != 1:
        raise ContractError("parse_batch needs frames with one grid shape and stride")
    conf = np.stack([m.conf.array for m in maps_list])
    paf = np.stack([m.paf.array for m in maps_list])
    return conf, paf, strides.pop()


def parse(maps: FeatureMaps, topo: SkeletonTopology, params) -> List[HumanPose]:
    """Drop-in for ``poseflow.paf.parse`` (paf.py:292-305), on the GPU."""
    params = _params_of(params)
    params.validate()          # ConfigError before any work (paf.py:295)
    maps.validate(topo)        # ContractError (paf.py:296)
    eng = default_parser(topo)
    conf = maps.conf.array[None]
    paf = maps.paf.array[None]
    return eng.parse_arrays(conf, paf, maps.stride, params).poses(0)


def parse_batch(maps_list: Sequence[FeatureMaps], topo: SkeletonTopology, params,
                device: Optional[int] = None) -> List[List[HumanPose]]:
    """``[parse(m, topo, params) for m in maps_list]`` in one GPU call."""
    params = _params_of(params)
    params.validate()
    for m in maps_list:
        m.validate(topo)
    if not maps_list:
        return []
    conf, paf, stride = _stack_maps(maps_list, topo)
    return default_parser(topo, device).parse_arrays(conf, paf, stride, params).all_poses()


def parse_arrays(conf: np.ndarray, paf: np.ndarray, stride: int, topo: SkeletonTopology,
                 params, device: Optional[int] = None) -> BatchResult:
    """Batched host arrays -> SoA ``BatchResult`` (no per-human objects)."""
    return default_parser(topo, device).parse_arrays(conf, paf, stride, params)


def format_records(res: "BatchResult", topo: SkeletonTopology, seq_base: int = 0) -> List[str]:
    """poses.jsonl lines of a batch (operators.py:293-310) via pf_format_records."""
    import ctypes

    lib = _native.load_library()
    names = [n.encode() for n in topo.keypoint_names]
    name_arr = (ctypes.c_char_p * len(names))(*names)
    k = res.n_keypoints

    def p(a):
        return a.ctypes.data_as(ctypes.c_void_p) if a.size else None

    xs = np.ascontiguousarray(res.kp_x).reshape(-1)
    ys = np.ascontiguousarray(res.kp_y).reshape(-1)
    ks = np.ascontiguousarray(res.kp_score).reshape(-1)
    kp = np.ascontiguousarray(res.kp_peak).reshape(-1)
    args = (res.n_frames, k, p(res.frame_first), p(res.frame_count), p(res.human_score), p(xs), p(ys), p(ks),
            p(kp), ctypes.cast(name_arr, ctypes.c_void_p), int(seq_base))
    n = lib.pf_format_records(*args, None, 0)
    if n < 0:
        raise ContractError("pf_format_records: bad arguments")
    buf = ctypes.create_string_buffer(int(n) + 1)
    lib.pf_format_records(*args, ctypes.cast(buf, ctypes.c_void_p), n)
    text = buf.raw[:n].decode()
    return text.split("\n")[:-1] if text else []
