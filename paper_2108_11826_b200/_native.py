"""ctypes binding of ``libpf_b200.so`` (the C ABI in ``include/pf_b200.h``).

The library is built in-tree (``csrc/Makefile``, driven by
``__graft_entry__.build()``).  There is no CPU fallback: if the library or
a CUDA device is missing, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import CapacityError, ConfigError, ContractError, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_B200_LIB: load another build of the same sources (A/B of build variants)
LIB_PATH = os.environ.get("PF_B200_LIB") or os.path.join(_HERE, "libpf_b200.so")

PF_OK, PF_ERR_CONFIG, PF_ERR_CONTRACT, PF_ERR_CAPACITY, PF_ERR_CUDA = 0, 1, 2, 3, 4
PF_MAX_KEYPOINTS, PF_MAX_LIMBS = 32, 64
PF_OPT_DEBUG, PF_OPT_TIMING, PF_OPT_MATERIALISE, PF_OPT_GENERIC_FUSED = 1, 2, 3, 4
PF_OPT_WIN_VARIANT = 5
PF_OPT_NO_CHAIN = 6
PF_OPT_PAF_ZERO_COPY = 8
PF_OPT_CORNER_SPLIT = 9
PF_OPT_PARSE_SPLIT = 10
PF_OPT_CONF_ZERO_COPY = 11
PF_OPT_PDL = 12
PF_OPT_COUNT_PAF = 13
PF_OPT_LARGE = 15
PF_OPT_HOST_OVERLAP = 16
PF_OPT_EXACT_LIST = 17
PF_N_KERNELS = 17

# every symbol include/pf_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTED_SYMBOLS = (
    "pf_abi_version", "pf_create", "pf_destroy", "pf_last_error", "pf_set_stream",
    "pf_use_own_stream",
    "pf_set_topology", "pf_validate_params", "pf_parse_device", "pf_parse_host",
    "pf_get_results", "pf_sync", "pf_set_debug", "pf_set_option", "pf_kernel_name",
    "pf_get_kernel_times", "pf_get_peaks", "pf_get_connections",
    "pf_preprocess_device", "pf_preprocess_f32_device", "pf_resize_device", "pf_host_alloc", "pf_host_free",
    "pf_launch_count", "pf_gaussian_taps", "pf_format_records", "pf_format_float", "pf_render_maps",
    "pf_overlay", "pf_get_paf_sectors", "pf_parse_batch", "pf_get_results_into",
)


class PfParams(ctypes.Structure):
    _fields_ = [
        ("conf_threshold", ctypes.c_double),
        ("nms_window", ctypes.c_int32),
        ("n_samples", ctypes.c_int32),
        ("sample_dot_threshold", ctypes.c_double),
        ("good_fraction_min", ctypes.c_double),
        ("min_parts", ctypes.c_int32),
        ("min_human_score", ctypes.c_double),
        ("upsample", ctypes.c_int32),
        ("blur_sigma", ctypes.c_double),
    ]


class PfCaps(ctypes.Structure):
    _fields_ = [
        ("max_peaks_per_part", ctypes.c_int32),
        ("max_peaks_per_frame", ctypes.c_int32),
        ("max_candidates", ctypes.c_int32),
        ("max_humans_per_frame", ctypes.c_int32),
        ("chunk_frames", ctypes.c_int32),
        ("max_humans_total", ctypes.c_int32),
    ]


class PfResults(ctypes.Structure):
    _fields_ = [
        ("n_frames", ctypes.c_int32),
        ("n_keypoints", ctypes.c_int32),
        ("total_humans", ctypes.c_int32),
        ("frame_first", ctypes.POINTER(ctypes.c_int32)),
        ("frame_count", ctypes.POINTER(ctypes.c_int32)),
        ("human_score", ctypes.POINTER(ctypes.c_double)),
        ("human_n_parts", ctypes.POINTER(ctypes.c_int32)),
        ("kp_x", ctypes.POINTER(ctypes.c_double)),
        ("kp_y", ctypes.POINTER(ctypes.c_double)),
        ("kp_score", ctypes.POINTER(ctypes.c_float)),
        ("kp_peak", ctypes.POINTER(ctypes.c_int32)),
    ]


class PfHostOut(ctypes.Structure):
    """pf_host_out: caller-owned host arrays for pf_get_results_into."""
    _fields_ = [
        ("capacity", ctypes.c_int32),
        ("frame_first", ctypes.c_void_p),
        ("frame_count", ctypes.c_void_p),
        ("human_score", ctypes.c_void_p),
        ("human_n_parts", ctypes.c_void_p),
        ("kp_x", ctypes.c_void_p),
        ("kp_y", ctypes.c_void_p),
        ("kp_score", ctypes.c_void_p),
        ("kp_peak", ctypes.c_void_p),
    ]


class PfOut(ctypes.Structure):
    """pf_out: caller-owned [B][max_humans] result slots (device pointers)."""
    _fields_ = [
        ("max_humans", ctypes.c_int32),
        ("n_humans", ctypes.c_void_p),
        ("human_score", ctypes.c_void_p),
        ("n_parts", ctypes.c_void_p),
        ("kp_xy", ctypes.c_void_p),
        ("kp_score", ctypes.c_void_p),
        ("kp_present", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the C ABI (no device work); raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"native library {path} not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        vp, i32, c_int = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
        lib.pf_abi_version.restype = c_int
        lib.pf_create.argtypes = [ctypes.POINTER(vp), c_int, ctypes.POINTER(PfCaps)]
        lib.pf_destroy.argtypes = [vp]
        lib.pf_destroy.restype = None
        lib.pf_last_error.argtypes = [vp]
        lib.pf_last_error.restype = ctypes.c_char_p
        lib.pf_set_stream.argtypes = [vp, vp]
        lib.pf_use_own_stream.argtypes = [vp]
        lib.pf_set_topology.argtypes = [vp, c_int, c_int, vp, vp]
        lib.pf_validate_params.argtypes = [ctypes.POINTER(PfParams)]
        lib.pf_parse_device.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int,
                                        ctypes.POINTER(PfParams)]
        lib.pf_parse_host.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int,
                                      ctypes.POINTER(PfParams), ctypes.POINTER(PfResults)]
        lib.pf_get_results.argtypes = [vp, ctypes.POINTER(PfResults)]
        lib.pf_get_results_into.argtypes = [vp, ctypes.POINTER(PfHostOut), ctypes.POINTER(i32),
                                            ctypes.POINTER(i32)]
        lib.pf_parse_batch.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, ctypes.POINTER(PfParams),
                                       ctypes.POINTER(PfOut), vp]
        lib.pf_sync.argtypes = [vp]
        lib.pf_set_debug.argtypes = [vp, c_int]
        lib.pf_set_option.argtypes = [vp, c_int, c_int]
        lib.pf_kernel_name.argtypes = [c_int]
        lib.pf_kernel_name.restype = ctypes.c_char_p
        lib.pf_get_kernel_times.argtypes = [vp, vp, vp, c_int]
        lib.pf_get_peaks.argtypes = [vp, c_int, ctypes.POINTER(c_int), vp, vp, vp, vp]
        lib.pf_get_connections.argtypes = [vp, c_int, ctypes.POINTER(c_int), vp, vp, vp, vp, vp]
        lib.pf_preprocess_device.argtypes = [vp, vp, c_int, c_int, c_int, vp, c_int, c_int]
        lib.pf_preprocess_f32_device.argtypes = [vp, vp, c_int, c_int, c_int, vp, c_int, c_int]
        lib.pf_resize_device.argtypes = [vp, vp, c_int, c_int, c_int, vp, c_int, c_int]
        lib.pf_host_alloc.argtypes = [ctypes.c_size_t]
        lib.pf_host_alloc.restype = vp
        lib.pf_host_free.argtypes = [vp]
        lib.pf_host_free.restype = None
        lib.pf_launch_count.argtypes = [vp]
        lib.pf_launch_count.restype = ctypes.c_int64
        lib.pf_format_records.argtypes = [c_int, c_int, vp, vp, vp, vp, vp, vp, vp, vp,
                                          ctypes.c_longlong, vp, ctypes.c_longlong]
        lib.pf_format_records.restype = ctypes.c_longlong
        lib.pf_format_float.argtypes = [ctypes.c_double, ctypes.c_char_p, c_int]
        lib.pf_render_maps.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, ctypes.c_double, ctypes.c_double,
                                       vp, vp]
        lib.pf_render_maps.restype = c_int
        lib.pf_overlay.argtypes = [vp, vp, vp, c_int, c_int, c_int, c_int, vp]
        lib.pf_overlay.restype = c_int
        lib.pf_format_float.restype = c_int
        lib.pf_gaussian_taps.argtypes = [ctypes.c_double, vp, c_int]
        lib.pf_get_paf_sectors.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
        del i32
        _lib = lib
        return lib


def gaussian_taps(sigma: float) -> np.ndarray:
    """The exact smoothing taps the library applies for ``blur_sigma``."""
    lib = load_library()
    buf = np.zeros(2 * 64 + 1, np.float64)
    r = lib.pf_gaussian_taps(float(sigma), buf.ctypes.data, buf.size)
    if r < 0:
        raise ConfigError(f"invalid blur_sigma {sigma}")
    return buf[: 2 * r + 1].copy()


def raise_for(code: int, message: str) -> None:
    if code == PF_OK:
        return
    if code == PF_ERR_CONFIG:
        raise ConfigError(message)
    if code == PF_ERR_CONTRACT:
        raise ContractError(message)
    if code == PF_ERR_CAPACITY:
        raise CapacityError(message)
    raise DeviceError(message or f"native call failed with status {code}")


class Context:
    """Owns one ``pf_ctx`` (device workspaces + stream) — not reentrant."""

    def __init__(self, device: int = 0, caps: "PfCaps | None" = None):
        self.lib = load_library()
        self.device = int(device)
        handle = ctypes.c_void_p()
        rc = self.lib.pf_create(ctypes.byref(handle), self.device,
                                ctypes.byref(caps) if caps is not None else None)
        if rc != PF_OK:
            msg = self.lib.pf_last_error(None)
            raise_for(rc, f"pf_create(device={self.device}): "
                          f"{msg.decode() if msg else f'status {rc}'}")
        self.handle = handle
        self._topo_key = None

    def check(self, rc: int) -> None:
        if rc != PF_OK:
            msg = self.lib.pf_last_error(self.handle)
            raise_for(rc, msg.decode() if msg else "")

    def set_topology(self, topo) -> None:
        key = (tuple(topo.keypoint_names), tuple(topo.limbs), tuple(topo.paf_channels))
        if key == self._topo_key:
            return
        limbs = np.ascontiguousarray(np.asarray(topo.limbs, dtype=np.int32).reshape(-1, 2))
        chans = np.ascontiguousarray(np.asarray(topo.paf_channels, dtype=np.int32).reshape(-1, 2))
        self.check(self.lib.pf_set_topology(self.handle, topo.n_keypoints, topo.n_limbs,
                                            limbs.ctypes.data, chans.ctypes.data))
        self._topo_key = key

    def launch_count(self) -> int:
        return int(self.lib.pf_launch_count(self.handle))

    def set_option(self, option: int, value: int) -> None:
        self.check(self.lib.pf_set_option(self.handle, int(option), int(value)))

    def paf_sectors(self) -> int:
        """Distinct 32-byte PAF sectors the last parse sampled (PF_OPT_COUNT_PAF on)."""
        n = ctypes.c_longlong()
        self.check(self.lib.pf_get_paf_sectors(self.handle, ctypes.byref(n)))
        return int(n.value)

    def kernel_times(self, reset: bool = False) -> dict:
        """{kernel name: (total ms, launches)} since the last reset (PF_OPT_TIMING)."""
        ms = np.zeros(PF_N_KERNELS, np.float64)
        n = np.zeros(PF_N_KERNELS, np.int64)
        self.check(self.lib.pf_get_kernel_times(self.handle, ms.ctypes.data, n.ctypes.data,
                                                1 if reset else 0))
        return {self.lib.pf_kernel_name(k).decode(): (float(ms[k]), int(n[k]))
                for k in range(PF_N_KERNELS) if n[k]}

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.pf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PinnedArray:
    """Page-locked host buffer exposed as a numpy array (pf_host_alloc)."""

    def __init__(self, shape, dtype=np.float32):
        self.lib = load_library()
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        self.ptr = self.lib.pf_host_alloc(max(nbytes, 1))
        if not self.ptr:
            raise DeviceError(f"pf_host_alloc({nbytes}) failed")
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self) -> None:
        if self.ptr:
            self.array = None
            self.lib.pf_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
