"""Operator-level API around the GPU path (reference: ``poseflow/operators.py``
and the plugin types of ``poseflow/dataflow.py:37-170``).

* ``Packet`` / ``OperatorSpec`` — same fields as ``dataflow.py:37-44`` /
  ``:145-170`` so the operators below slot into a poseflow pipeline.
* ``make_preprocess(input_w, input_h)`` [operators.py:114-131] —
  ``(Frame) -> (Frame, TensorF32[3,H,W])``; the resize/layout runs on the GPU
  (``pf_preprocess_f32_device``), bit-identical to the reference.
* ``make_postprocess(topo, params)`` [operators.py:147-157] —
  ``(Frame, FeatureMaps) -> (Frame, [HumanPose])`` through the GPU parser.
* ``make_batched_postprocess`` — the batched GPU stage of SURVEY.md §8(f)2:
  the reference batching operator (``accumulate_batch`` with ``linger_us``,
  ``batch_hist``, ``ctx.timed``, ``split_batch_results``; scheduler.py:55-131)
  around one ``parse_batch`` call per drained batch.
* ``preprocess_batch`` — u8 HWC frames -> f32 CHW on the device.
* ``bilinear_resize`` / ``hwc_to_chw`` [operators.py:79-111] and
  ``pose_record`` [operators.py:293-310].
"""

from __future__ import annotations

import ctypes
import json
import threading
from dataclasses import dataclass
from typing import Any, Callable, Iterator, List, Optional, Sequence

import numpy as np

from . import _native
from .core import Frame, HumanPose, SkeletonTopology, TensorF32
from .errors import ContractError
from .parser import ParserParams, _params_of, _stack_maps, default_parser, parse, parse_batch


@dataclass(frozen=True)
class Packet:
    seq_id: int
    ingest_ns: int
    payload: Any


@dataclass
class OperatorSpec:
    name: str
    kind: str  # "source" | "transform" | "sink"
    fn: Optional[Callable] = None
    runner: Optional[Callable] = None

    @staticmethod
    def source(name: str, make_iter: Callable[[], Iterator]) -> "OperatorSpec":
        return OperatorSpec(name=name, kind="source", fn=make_iter)

    @staticmethod
    def transform(name: str, fn: Callable[[Any], Any]) -> "OperatorSpec":
        return OperatorSpec(name=name, kind="transform", fn=fn)

    @staticmethod
    def sink(name: str, fn: Callable[[Any], None]) -> "OperatorSpec":
        return OperatorSpec(name=name, kind="sink", fn=fn)


# ---------------------------------------------------------------- device ops
_tls = threading.local()


def _ctx(device: int = 0) -> _native.Context:
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    if device not in cache:
        cache[device] = _native.Context(device)
    return cache[device]


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _native.DeviceError("no CUDA device visible (the GPU path has no CPU fallback)")
    return torch


def preprocess_batch(frames, out_h: int, out_w: int, device: int = 0):
    """u8 [B,h,w,3] (torch CUDA tensor or numpy) -> f32 [B,3,out_h,out_w] CUDA tensor.

    ``read_ppm``'s ``u8/255`` plus ``make_preprocess``'s resize/layout in one
    kernel (formats.py:116-117, operators.py:118-129).
    """
    torch = _torch()
    src = frames if isinstance(frames, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(frames))
    if src.dtype not in (torch.uint8, torch.float32):
        raise ContractError("frames must be uint8 (raw) or float32 (normalised) HWC")
    if src.dim() != 4 or src.shape[3] != 3:
        raise ContractError(f"frames must be [B, H, W, 3], got {tuple(src.shape)}")
    src = src.to(f"cuda:{device}", non_blocking=True).contiguous()
    b, h, w, _ = src.shape
    if h < 1 or w < 1:
        raise ContractError("zero-area frame")
    dst = torch.empty((b, 3, out_h, out_w), dtype=torch.float32, device=src.device)
    ctx = _ctx(device)
    ctx.check(ctx.lib.pf_set_stream(ctx.handle, ctypes.c_void_p(torch.cuda.current_stream(src.device).cuda_stream)))
    fn = ctx.lib.pf_preprocess_device if src.dtype == torch.uint8 else ctx.lib.pf_preprocess_f32_device
    ctx.check(fn(ctx.handle, ctypes.c_void_p(src.data_ptr()), b, h, w,
                 ctypes.c_void_p(dst.data_ptr()), out_h, out_w))
    return dst


def resize_planes(planes, out_h: int, out_w: int, device: int = 0):
    """bilinear_resize's 2-D branch per plane on the GPU: f32 [P,h,w] -> [P,out_h,out_w]."""
    torch = _torch()
    src = planes if isinstance(planes, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(planes, dtype=np.float32))
    if src.dtype != torch.float32 or src.dim() != 3:
        raise ContractError("planes must be float32 [P, h, w]")
    src = src.to(f"cuda:{device}").contiguous()
    p, h, w = src.shape
    if min(h, w, out_h, out_w) < 1:
        raise ContractError("resize requires positive extents")
    dst = torch.empty((p, out_h, out_w), dtype=torch.float32, device=src.device)
    ctx = _ctx(device)
    ctx.check(ctx.lib.pf_set_stream(ctx.handle, ctypes.c_void_p(torch.cuda.current_stream(src.device).cuda_stream)))
    ctx.check(ctx.lib.pf_resize_device(ctx.handle, ctypes.c_void_p(src.data_ptr()), p, h, w,
                                       ctypes.c_void_p(dst.data_ptr()), out_h, out_w))
    return dst


def bilinear_resize(image: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """operators.py:79-107 on the GPU for float32 [H,W] or [H,W,C] arrays."""
    if image.ndim not in (2, 3):
        raise ContractError("image must be [H, W] or [H, W, C]")
    in_h, in_w = image.shape[:2]
    if min(in_h, in_w, out_h, out_w) < 1:
        raise ContractError("resize requires positive extents")
    if (in_h, in_w) == (out_h, out_w):
        return image.copy()
    if image.dtype != np.float32:
        raise ContractError("GPU bilinear_resize computes float32 maps/images")
    planes = image[None] if image.ndim == 2 else np.transpose(image, (2, 0, 1))
    out = resize_planes(planes, out_h, out_w).cpu().numpy()
    return out[0] if image.ndim == 2 else np.ascontiguousarray(np.transpose(out, (1, 2, 0)))


def hwc_to_chw(image: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.moveaxis(image, 2, 0))


# ---------------------------------------------------------------- operators
def make_preprocess(input_w: int, input_h: int, latency_us: int = 0) -> OperatorSpec:
    """Resize to the network input extents and switch to channel-first (GPU)."""

    def fn(pkt: Packet) -> Packet:
        frame: Frame = pkt.payload
        img = frame.image.array
        if img.shape[0] < 1 or img.shape[1] < 1:
            raise ContractError("zero-area frame")
        if (img.shape[0], img.shape[1]) == (input_h, input_w):
            chw = hwc_to_chw(img)  # layout only, values untouched
        else:
            chw = preprocess_batch(img[None].astype(np.float32, copy=False), input_h, input_w)[0].cpu().numpy()
        return Packet(pkt.seq_id, pkt.ingest_ns, (frame, TensorF32(chw)))

    return OperatorSpec.transform("preprocess", fn)


def make_postprocess(topo: SkeletonTopology, params, latency_us: int = 0) -> OperatorSpec:
    """(frame, maps) -> (frame, poses) via the GPU parser."""
    params = _params_of(params)

    def fn(pkt: Packet) -> Packet:
        frame, maps = pkt.payload
        return Packet(pkt.seq_id, pkt.ingest_ns, (frame, parse(maps, topo, params)))

    return OperatorSpec.transform("postprocess", fn)


def _is_packet(item) -> bool:
    return hasattr(item, "seq_id") and hasattr(item, "payload")


def _is_end(item) -> bool:
    # the reference's channel sentinels (dataflow.py:26-37) by name; this
    # package never imports the reference
    return repr(item) == "END_OF_STREAM"


def accumulate_batch(ctx, in_ch, batch_max: int, linger_us: int = 0):
    """The reference batch former (scheduler.py:55-86): block for the first
    item, then drain without waiting up to ``batch_max`` — or keep waiting
    inside the ``linger_us`` window.  Returns (batch, saw_end)."""
    import time

    first = ctx.recv(in_ch)
    if _is_end(first):
        return [], True
    batch = [first]
    deadline = time.monotonic() + linger_us / 1e6 if linger_us else None
    while len(batch) < batch_max:
        item = ctx.try_recv(in_ch)
        if not _is_packet(item) and not _is_end(item):          # NO_ITEM
            if deadline is None:
                break
            remaining = deadline - time.monotonic()
            if remaining <= 0:
                break
            item = ctx.recv_timeout(in_ch, remaining)
            if not _is_packet(item) and not _is_end(item):
                break
        if _is_end(item):
            return batch, True
        batch.append(item)
    return batch, False


def split_batch_results(outputs: Sequence[Any], batch: Sequence[Packet]) -> List[Packet]:
    """Re-wrap one output per packet, checking count and ascending seq order
    exactly as the reference does (scheduler.py:89-105)."""
    from .errors import BackendError

    if len(outputs) != len(batch):
        raise BackendError(f"backend returned {len(outputs)} outputs for batch of {len(batch)} "
                           f"(seq_ids {[p.seq_id for p in batch]})")
    for prev, cur in zip(batch, batch[1:]):
        if cur.seq_id <= prev.seq_id:
            raise BackendError(f"batch seq_ids not ascending: {prev.seq_id} then {cur.seq_id}")
    return [Packet(seq_id=pkt.seq_id, ingest_ns=pkt.ingest_ns, payload=out) for pkt, out in zip(batch, outputs)]


def make_batched_postprocess(topo: SkeletonTopology, params, batch_max: int = 256, linger_us: int = 0,
                             device: int = 0, devices: Optional[Sequence[int]] = None,
                             name: str = "postprocess") -> OperatorSpec:
    """Batched GPU post-processing stage.

    ``runner(ctx, in_ch, out_ch)`` is the reference batching operator
    (``make_batching_operator``, scheduler.py:108-131) with the GPU parse as
    its backend call: ``accumulate_batch`` (block for one item, drain up to
    ``batch_max``, optional ``linger_us`` window), ``ctx.batch_hist[len] += 1``,
    the parse of the whole batch under ``ctx.timed`` (so the reference's
    ``PipelineStats`` charge it as busy time), ``split_batch_results`` (count
    and ascending-seq checks), then one packet per frame downstream.
    ``fn`` is the per-item form for sequential runs.  With ``devices`` (more
    than one entry) a batch is cut into contiguous shards parsed concurrently
    on those GPUs (``MultiDeviceParser``) and merged back in frame order.
    Outputs are identical for every batch composition and device count
    (parse is pure).
    """
    params = _params_of(params)
    params.validate()
    if batch_max < 1:
        raise ContractError("batch_max must be >= 1")
    if linger_us < 0:
        raise ContractError("linger_us must be >= 0")
    multi = None
    if devices is not None and len(devices) > 1:
        from .sharding import MultiDeviceParser

        multi = MultiDeviceParser(topo, devices)

    def backend_call(batch: Sequence[Packet]) -> List[Any]:
        maps = [p.payload[1] for p in batch]
        if multi is None:
            poses = parse_batch(maps, topo, params, device=device)
        else:
            for m in maps:
                m.validate(topo)
            conf, paf, stride = _stack_maps(maps, topo)
            poses = multi.parse_arrays(conf, paf, stride, params).all_poses()
        return [(p.payload[0], hp) for p, hp in zip(batch, poses)]

    def runner(ctx, in_ch, out_ch):
        while True:
            batch, saw_end = accumulate_batch(ctx, in_ch, batch_max, linger_us)
            if batch:
                hist = getattr(ctx, "batch_hist", None)
                if hist is not None:
                    hist[len(batch)] += 1
                timed = getattr(ctx, "timed", None)
                outputs = timed(backend_call, batch) if timed is not None else backend_call(batch)
                for pkt in split_batch_results(outputs, batch):
                    ctx.send(out_ch, pkt)
            if saw_end:
                out_ch.close()
                return

    def item_fn(pkt: Packet) -> Packet:
        return split_batch_results(backend_call([pkt]), [pkt])[0]

    return OperatorSpec(name=name, kind="transform", fn=item_fn, runner=runner)


def pose_record(seq_id: int, poses: Sequence[HumanPose], topo: SkeletonTopology) -> str:
    """One poses.jsonl line (operators.py:293-310): key order and float repr
    are part of the contract, so records are byte-comparable across engines."""
    humans = [
        {"score": float(pose.score),
         "keypoints": [{"part": topo.keypoint_names[k], "x": float(kp.x), "y": float(kp.y),
                        "score": float(kp.score)}
                       for k, kp in enumerate(pose.keypoints) if kp is not None]}
        for pose in poses
    ]
    return json.dumps({"frame_id": seq_id, "humans": humans}, separators=(",", ":"))
