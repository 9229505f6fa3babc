"""Pose overlay on the GPU: the reference's
``visualize`` (poseflow/operators.py:160-290) with the same signature and
pixels.  The host places keypoints (``_round_half_up`` of the scaled input
coordinates, operators.py:270-277), lists the primitives in the reference's
draw order (per pose: limbs in topology order, keypoint discs by part, the
optional score label) and expands label glyphs into points; the raster work
and the "later draws overwrite earlier ones" rule run on the device
(``pf_overlay``: draw-order atomicMax per pixel, then one colour write)."""

from __future__ import annotations

import colorsys
import ctypes
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .core import Frame, HumanPose, SkeletonTopology, TensorF32
from .errors import ContractError


@dataclass
class OverlayStyle:
    keypoint_radius: int = 3
    limb_thickness: int = 2
    score_label: bool = False

    def validate(self) -> None:
        if self.keypoint_radius < 1:
            raise ContractError("keypoint_radius must be >= 1")
        if self.limb_thickness < 1:
            raise ContractError("limb_thickness must be >= 1")


def part_color(part: int) -> Tuple[float, float, float]:
    """Deterministic per-part colour: golden-ratio hue stepping (operators.py:173-176)."""
    hue = (part * 0.6180339887498949) % 1.0
    return colorsys.hsv_to_rgb(hue, 0.85, 1.0)


# 3x5 label glyphs, row-major (operators.py:219-225)
_GLYPHS = {
    "0": "111101101101111", "1": "010110010010111", "2": "111001111100111",
    "3": "111001111001111", "4": "101101111001001", "5": "111100111001111",
    "6": "111100111101111", "7": "111001001001001", "8": "111101111101111",
    "9": "111101111001111", ".": "000000000000010",
}

PRIM_DTYPE = np.dtype([("frame", "<i4"), ("kind", "<i4"), ("x0", "<i4"), ("y0", "<i4"), ("x1", "<i4"),
                       ("y1", "<i4"), ("r", "<i4"), ("rgb", "<f4", (3,))])


def _round_half_up(v: float) -> int:
    return int(math.floor(v + 0.5))


def _primitives(frame: int, poses: Sequence[HumanPose], style: OverlayStyle, topo: SkeletonTopology,
                h: int, w: int, input_w: int, input_h: int) -> List[tuple]:
    scale_x = w / input_w
    scale_y = h / input_h
    out = []
    for pose in poses:
        pts: List[Optional[Tuple[int, int]]] = []
        for kp in pose.keypoints:
            if kp is None:
                pts.append(None)
            else:
                pts.append((_round_half_up((kp.x + 0.5) * scale_x - 0.5),
                            _round_half_up((kp.y + 0.5) * scale_y - 0.5)))
        for a, b in topo.limbs:
            if pts[a] is not None and pts[b] is not None:
                out.append((frame, 0, pts[a][0], pts[a][1], pts[b][0], pts[b][1], style.limb_thickness // 2,
                            part_color(b)))
        for part, pt in enumerate(pts):
            if pt is not None:
                out.append((frame, 1, pt[0], pt[1], 0, 0, style.keypoint_radius, part_color(part)))
        if style.score_label:
            anchor = next((pt for pt in pts if pt is not None), None)
            if anchor is not None:
                x, y = anchor[0] + style.keypoint_radius + 2, anchor[1]
                for ch in f"{pose.score:.2f}":
                    glyph = _GLYPHS.get(ch)
                    if glyph is None:
                        continue
                    for row in range(5):
                        for col in range(3):
                            if glyph[row * 3 + col] == "1":
                                out.append((frame, 1, x + col, y + row, 0, 0, 0, (1.0, 1.0, 1.0)))
                    x += 4
    return out


def visualize_batch(images: np.ndarray, poses_per_frame: Sequence[Sequence[HumanPose]], style: OverlayStyle,
                    topo: SkeletonTopology, input_w: int, input_h: int, device: int = 0) -> np.ndarray:
    """Overlay every frame's poses on a copy of its image: f32 [B, H, W, 3]."""
    import torch

    from .parser import default_parser

    style.validate()
    images = np.ascontiguousarray(images, dtype=np.float32)
    if images.ndim != 4 or images.shape[3] != 3:
        raise ContractError(f"images must be [B, H, W, 3], got {images.shape}")
    b, h, w, _ = images.shape
    if len(poses_per_frame) != b:
        raise ContractError("one pose list per frame")
    prims, first = [], [0]
    for f, poses in enumerate(poses_per_frame):
        prims.extend(_primitives(f, poses, style, topo, h, w, input_w, input_h))
        first.append(len(prims))
    arr = np.zeros(max(len(prims), 1), dtype=PRIM_DTYPE)
    for i, (fr, kind, x0, y0, x1, y1, r, rgb) in enumerate(prims):
        arr[i] = (fr, kind, x0, y0, x1, y1, r, rgb)
    dev = torch.device("cuda", device)
    img = torch.from_numpy(images).to(dev)
    prim_d = torch.from_numpy(arr.view(np.uint8)).to(dev)
    first_d = torch.tensor(first, dtype=torch.int32, device=dev)
    ctx = default_parser(topo, device).ctx
    ctx.check(ctx.lib.pf_set_stream(ctx.handle, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    ctx.check(ctx.lib.pf_overlay(ctx.handle, ctypes.c_void_p(prim_d.data_ptr()), ctypes.c_void_p(first_d.data_ptr()),
                                 len(prims), b, h, w, ctypes.c_void_p(img.data_ptr())))
    return img.cpu().numpy()


def visualize(frame: Frame, poses: Sequence[HumanPose], style: OverlayStyle, topo: SkeletonTopology,
              input_w: int, input_h: int) -> TensorF32:
    """Drop-in for ``poseflow.operators.visualize`` (operators.py:249-290)."""
    style.validate()
    img = frame.image.array.copy()
    if not poses:
        return TensorF32(img)
    out = visualize_batch(img[None], [poses], style, topo, input_w, input_h)
    return TensorF32(out[0])
