"""GPU-resident producer of feature maps.

``render_maps_gpu`` draws OpenPose-style confidence maps and part affinity
fields for given keypoint cells directly into device memory
(``pf_render_maps``): max-blended Gaussians per part with background
``1 - max``, and unit limb vectors in a corridor around each limb, averaged
where limbs overlap — the drawing rule of the reference's synthetic backend
(``synth.py:93-183``).  The maps feed ``PafParser.parse_tensors`` without a
host round trip, exactly like a network's output tensors would.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .core import SkeletonTopology
from .errors import ContractError


def render_maps_gpu(kp_cells: np.ndarray, n_humans: np.ndarray, topo: SkeletonTopology, grid_h: int,
                    grid_w: int, sigma: float, halfwidth: float, device: int = 0):
    """kp_cells f64 [F, Hmax, K, 2] (row, col) cells, NaN = missing keypoint;
    n_humans i32 [F].  Returns torch CUDA tensors conf [F,K+1,grid_h,grid_w]
    and paf [F,2L,grid_h,grid_w] (f32), rendered on ``device``."""
    import torch

    from .parser import default_parser

    kp_cells = np.ascontiguousarray(kp_cells, dtype=np.float64)
    n_humans = np.ascontiguousarray(n_humans, dtype=np.int32)
    if kp_cells.ndim != 4 or kp_cells.shape[2] != topo.n_keypoints or kp_cells.shape[3] != 2:
        raise ContractError(f"kp_cells must be [F, Hmax, {topo.n_keypoints}, 2], got {kp_cells.shape}")
    frames, hmax = kp_cells.shape[:2]
    if n_humans.shape != (frames,) or (n_humans < 0).any() or (n_humans > hmax).any():
        raise ContractError("n_humans must be [F] with 0 <= n <= Hmax")
    dev = torch.device("cuda", device)
    kp_d = torch.from_numpy(kp_cells).to(dev)
    nh_d = torch.from_numpy(n_humans).to(dev)
    conf = torch.empty((frames, topo.n_keypoints + 1, grid_h, grid_w), dtype=torch.float32, device=dev)
    paf = torch.empty((frames, 2 * topo.n_limbs, grid_h, grid_w), dtype=torch.float32, device=dev)
    ctx = default_parser(topo, device).ctx
    ctx.check(ctx.lib.pf_set_stream(ctx.handle, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    ctx.check(ctx.lib.pf_render_maps(ctx.handle, ctypes.c_void_p(kp_d.data_ptr()), ctypes.c_void_p(nh_d.data_ptr()),
                                     frames, hmax, grid_h, grid_w, float(sigma), float(halfwidth),
                                     ctypes.c_void_p(conf.data_ptr()), ctypes.c_void_p(paf.data_ptr())))
    torch.cuda.synchronize(dev)
    return conf, paf
