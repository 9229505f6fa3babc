"""Synthetic scenes and feature maps — TEST / BENCHMARK INPUT GENERATION.

Not product code: it lives outside ``paper_2108_11826_b200`` and only
``tests/``, ``bench.py``, ``__graft_entry__.smoke()`` and ``tools/`` use it.
It restates the reference's synthetic backend so the GPU box — where the
reference is absent — can produce the same inputs:

* ``SynthParams``          — ``synth.py:29-52``
* ``GroundTruthHuman/Scene`` — ``synth.py:55-90``
* ``render_feature_maps``  — ``synth.py:93-161`` (+ ``_paint_limb`` 164-183):
  max-blended Gaussians (sigma in cells) per part, background = 1 - max,
  unit limb vectors in a corridor, averaged where limbs overlap, clamped to
  unit length; computed in fp64, stored as fp32.  Same operation order as
  the reference, so on the same numpy the maps are bit-identical
  (``tests/test_host_api.py::TestSynth`` checks against reference-rendered
  maps, ``tests/golden/frames_golden.npz``).
* ``procedural_scene``     — ``synth.py:224-275`` (1-5 separated stick figures,
  ``default_rng([seed, seq])``), same RNG call sequence.
* ``crowd_scene``          — SURVEY.md §8(d) C3: 40 unseparated figures.

Not on the hot path: this only feeds tests and the benchmark.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from paper_2108_11826_b200.core import FeatureMaps, SkeletonTopology, TensorF32, pixel_to_cell
from paper_2108_11826_b200.errors import ConfigError, ContractError


@dataclass
class SynthParams:
    sigma_conf: float = 2.0
    paf_halfwidth: float = 1.0
    stride: int = 8
    service_delay_us: int = 0
    batch_overhead_us: int = 0
    per_item_us: int = 0
    max_batch: int = 32

    def validate(self) -> None:
        if self.sigma_conf <= 0:
            raise ConfigError("sigma_conf must be > 0")
        if self.paf_halfwidth <= 0:
            raise ConfigError("paf_halfwidth must be > 0")
        if self.stride < 1:
            raise ConfigError("stride must be >= 1")
        if self.max_batch < 1:
            raise ConfigError("max_batch must be >= 1")
        for name in ("service_delay_us", "batch_overhead_us", "per_item_us"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} must be >= 0")


@dataclass(frozen=True)
class GroundTruthHuman:
    keypoints: Tuple[Optional[Tuple[float, float]], ...]

    @property
    def n_present(self) -> int:
        return sum(kp is not None for kp in self.keypoints)


@dataclass(frozen=True)
class GroundTruthScene:
    humans: Tuple[GroundTruthHuman, ...]
    input_w: int
    input_h: int
    seed: int = 0

    def validate(self, n_keypoints: Optional[int] = None, min_parts: int = 1) -> None:
        for idx, hum in enumerate(self.humans):
            if n_keypoints is not None and len(hum.keypoints) != n_keypoints:
                raise ContractError(
                    f"human {idx} has {len(hum.keypoints)} keypoint slots, topology has {n_keypoints}")
            if hum.n_present < min_parts:
                raise ContractError(f"human {idx} has fewer than {min_parts} keypoints")
            for part, kp in enumerate(hum.keypoints):
                if kp is None:
                    continue
                if not (0 <= kp[0] < self.input_w and 0 <= kp[1] < self.input_h):
                    raise ContractError(
                        f"human {idx} keypoint {part} at ({kp[0]}, {kp[1]}) outside "
                        f"[0, {self.input_w}) x [0, {self.input_h})")


def _corridor(paf_sum, paf_count, limb, chans, ca, cb, halfwidth, rows, cols) -> None:
    """Accumulate one limb's unit vector over cells within ``halfwidth`` of
    the segment (reference ``_paint_limb``, synth.py:164-183)."""
    (ai, aj), (bi, bj) = ca, cb
    di, dj = bi - ai, bj - aj
    len_sq = di * di + dj * dj
    if len_sq == 0.0:
        return
    length = np.sqrt(len_sq)
    ux, uy = dj / length, di / length
    t = np.clip(((rows - ai) * di + (cols - aj) * dj) / len_sq, 0.0, 1.0)
    dist_sq = (rows - (ai + t * di)) ** 2 + (cols - (aj + t * dj)) ** 2
    inside = dist_sq <= halfwidth * halfwidth
    paf_sum[chans[0]][inside] += ux
    paf_sum[chans[1]][inside] += uy
    paf_count[limb][inside] += 1


def render_feature_maps(scene: GroundTruthScene, topo: SkeletonTopology, p: SynthParams,
                        frame_ref: int = 0) -> FeatureMaps:
    scene.validate(topo.n_keypoints)
    if scene.input_w % p.stride or scene.input_h % p.stride:
        raise ContractError("scene extents must be divisible by the stride")
    k = topo.n_keypoints
    gh, gw = scene.input_h // p.stride, scene.input_w // p.stride
    conf = np.zeros((k + 1, gh, gw), dtype=np.float64)
    paf_sum = np.zeros((2 * topo.n_limbs, gh, gw), dtype=np.float64)
    paf_count = np.zeros((topo.n_limbs, gh, gw), dtype=np.int32)
    rows = np.arange(gh, dtype=np.float64)[:, None]
    cols = np.arange(gw, dtype=np.float64)[None, :]
    inv = 1.0 / (2.0 * p.sigma_conf * p.sigma_conf)
    for hum in scene.humans:
        cells: List[Optional[Tuple[float, float]]] = [None] * k
        for part, kp in enumerate(hum.keypoints):
            if kp is None:
                continue
            ci, cj = pixel_to_cell(kp[0], kp[1], p.stride)
            cells[part] = (ci, cj)
            np.maximum(conf[part], np.exp(-((rows - ci) ** 2 + (cols - cj) ** 2) * inv),
                       out=conf[part])
        for limb, (a, b) in enumerate(topo.limbs):
            if cells[a] is not None and cells[b] is not None:
                _corridor(paf_sum, paf_count, limb, topo.paf_channels[limb], cells[a], cells[b],
                          p.paf_halfwidth, rows, cols)
    conf[k] = 1.0 - conf[:k].max(axis=0, initial=0.0)
    paf = np.zeros_like(paf_sum)
    for limb, (cx, cy) in enumerate(topo.paf_channels):
        hit = paf_count[limb] > 0
        if not hit.any():
            continue
        cnt = paf_count[limb][hit]
        vx = paf_sum[cx][hit] / cnt
        vy = paf_sum[cy][hit] / cnt
        mag = np.sqrt(vx * vx + vy * vy)
        big = mag > 1.0
        vx[big] /= mag[big]
        vy[big] /= mag[big]
        paf[cx][hit] = vx
        paf[cy][hit] = vy
    maps = FeatureMaps(conf=TensorF32.from_array(conf), paf=TensorF32.from_array(paf),
                       stride=p.stride, frame_ref=frame_ref)
    maps.validate(topo, scene.input_w, scene.input_h)
    return maps


# Canonical figure in figure-height units (x right, y down), same template
# as the reference (synth.py:190-209): nose, neck, r/l arm, r/l leg, eyes, ears.
CANONICAL_FIGURE: Tuple[Tuple[float, float], ...] = (
    (0.00, -0.40), (0.00, -0.25),
    (-0.15, -0.25), (-0.21, -0.09), (-0.25, 0.07),
    (0.15, -0.25), (0.21, -0.09), (0.25, 0.07),
    (-0.09, 0.05), (-0.11, 0.28), (-0.13, 0.50),
    (0.09, 0.05), (0.11, 0.28), (0.13, 0.50),
    (-0.14, -0.54), (0.14, -0.54), (-0.28, -0.46), (0.28, -0.46),
)
_ATTEMPTS = 300


_HEIGHTS = {1: (120.0, 170.0), 2: (100.0, 150.0), 3: (85.0, 130.0)}


def _heights(n: int) -> Tuple[float, float]:
    """Figure height range by crowd size (fewer people -> taller figures)."""
    return _HEIGHTS.get(max(n, 1), (70.0, 105.0))


def _min_dist(a: np.ndarray, b: np.ndarray) -> float:
    d = a[:, None, :] - b[None, :, :]
    return float(np.sqrt((d * d).sum(axis=2)).min())


def procedural_scene(seed: int, seq_id: int, input_w: int, input_h: int, params: SynthParams,
                     min_separation_px: Optional[float] = None) -> GroundTruthScene:
    """1-5 jittered, scaled, optionally mirrored figures with pairwise keypoint
    separation >= ``6 * sigma * stride`` (RNG call order of synth.py:224-275)."""
    if min_separation_px is None:
        min_separation_px = 6.0 * params.sigma_conf * params.stride
    rng = np.random.default_rng([int(seed), int(seq_id)])
    target = int(rng.integers(1, 6))
    lo, hi = _heights(target)
    hi = min(hi, min(input_h / 1.2, input_w / 0.75))
    lo = min(lo, 0.75 * hi)
    template = np.array(CANONICAL_FIGURE, dtype=np.float64)
    placed: List[np.ndarray] = []
    for _ in range(target):
        for _try in range(_ATTEMPTS):
            height = rng.uniform(lo, hi)
            flip = -1.0 if rng.random() < 0.5 else 1.0
            pts = template * height
            pts[:, 0] *= flip
            pts += rng.normal(0.0, 0.01 * height, size=pts.shape)
            mx = 0.32 * height
            cx = rng.uniform(mx, input_w - mx)
            cy = rng.uniform(0.58 * height, input_h - 0.54 * height)
            pts = pts + np.array([cx, cy])
            pts[:, 0] = np.clip(pts[:, 0], 0.0, input_w - 1e-3)
            pts[:, 1] = np.clip(pts[:, 1], 0.0, input_h - 1e-3)
            if all(_min_dist(pts, other) >= min_separation_px for other in placed):
                placed.append(pts)
                break
    humans = tuple(GroundTruthHuman(tuple((float(x), float(y)) for x, y in pts)) for pts in placed)
    return GroundTruthScene(humans=humans, input_w=input_w, input_h=input_h, seed=seed)


def crowd_scene(seed: int, frame: int, input_w: int = 656, input_h: int = 368,
                n_people: int = 40, height_range: Tuple[float, float] = (60.0, 110.0)
                ) -> GroundTruthScene:
    """SURVEY.md §8(d) C3 stress scene: ``n_people`` canonical figures, heights
    U(60, 110) px, random mirror, jitter N(0, 0.01 h), uniform centres, no
    separation, ``default_rng([seed, frame])``.  Overlaps exercise the
    merge / conflict / slot-taken branches of assemble_humans."""
    rng = np.random.default_rng([int(seed), int(frame)])
    template = np.array(CANONICAL_FIGURE, dtype=np.float64)
    humans = []
    for _ in range(n_people):
        height = rng.uniform(*height_range)
        pts = template * height
        if rng.random() < 0.5:
            pts[:, 0] *= -1.0
        pts += rng.normal(0.0, 0.01 * height, size=pts.shape)
        cx = rng.uniform(0.0, input_w)
        cy = rng.uniform(0.0, input_h)
        pts = pts + np.array([cx, cy])
        pts[:, 0] = np.clip(pts[:, 0], 0.0, input_w - 1e-3)
        pts[:, 1] = np.clip(pts[:, 1], 0.0, input_h - 1e-3)
        humans.append(GroundTruthHuman(tuple((float(x), float(y)) for x, y in pts)))
    return GroundTruthScene(humans=tuple(humans), input_w=input_w, input_h=input_h, seed=seed)


def render_batch(scenes, topo: SkeletonTopology, p: SynthParams):
    """Render scenes into stacked conf [B,K+1,H,W] and paf [B,2L,H,W] arrays."""
    maps = [render_feature_maps(s, topo, p, frame_ref=i) for i, s in enumerate(scenes)]
    return (np.stack([m.conf.array for m in maps]), np.stack([m.paf.array for m in maps]))


def render_batch_gpu(scenes, topo: SkeletonTopology, p: SynthParams, device: int = 0):
    """``render_batch`` on the GPU through the product's producer kernel
    (``paper_2108_11826_b200.producer.render_maps_gpu`` -> pf_render_maps,
    SURVEY.md §8(f) 1): torch CUDA tensors conf [B,K+1,H,W] and paf
    [B,2L,H,W].  Equal to the host renderer except where fp64 exp() differs
    from numpy's in the last bit and that decides an fp32 rounding."""
    from paper_2108_11826_b200.producer import render_maps_gpu

    p.validate()
    k = topo.n_keypoints
    if not scenes:
        raise ContractError("render_batch_gpu needs at least one scene")
    w0, h0 = scenes[0].input_w, scenes[0].input_h
    for s in scenes:
        s.validate(k)
        if (s.input_w, s.input_h) != (w0, h0):
            raise ContractError("render_batch_gpu needs scenes of one size")
    if w0 % p.stride or h0 % p.stride:
        raise ContractError("scene extents must be divisible by the stride")
    hmax = max(1, max(len(s.humans) for s in scenes))
    kp = np.full((len(scenes), hmax, k, 2), np.nan, dtype=np.float64)
    nh = np.zeros(len(scenes), dtype=np.int32)
    for f, s in enumerate(scenes):
        nh[f] = len(s.humans)
        for hh, hum in enumerate(s.humans):
            for part, xy in enumerate(hum.keypoints):
                if xy is not None:
                    kp[f, hh, part] = pixel_to_cell(xy[0], xy[1], p.stride)
    return render_maps_gpu(kp, nh, topo, h0 // p.stride, w0 // p.stride, p.sigma_conf, p.paf_halfwidth,
                           device=device)
