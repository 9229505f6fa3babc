"""Frame sharding across the GPUs of one node.

``parse`` is a pure per-frame function (paf.py:292-305), so a stream of
frames partitions into independent shards with no exchange step: rank r
parses its own contiguous block on its own GPU and the only collective is the
host-side gather of the compact results (JSONL records, ~KB per frame) in
``seq_id`` order — the order the reference sink requires
(operators.py:330-334).  Timing plumbing (max over ranks) also lives here.

One process per GPU (torchrun); ``torch.distributed`` carries only the
result gather and the timing reduction, never maps.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


def shard_bounds(n_frames: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of frame indices owned by ``rank``; blocks
    differ in size by at most one frame and cover [0, n_frames) exactly."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_indices(n_frames: int, rank: int, world: int, mode: str = "block") -> np.ndarray:
    """Frame indices of one rank: ``block`` (contiguous) or ``round_robin``."""
    if mode == "block":
        lo, hi = shard_bounds(n_frames, rank, world)
        return np.arange(lo, hi)
    if mode == "round_robin":
        return np.arange(rank, n_frames, world)
    raise ValueError(f"unknown shard mode {mode!r}")


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float) -> float:
    """The job's time is its slowest rank's (never wall clock of one rank)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    import torch

    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_records(local: Sequence[Tuple[int, str]], dst: int = 0) -> Optional[List[str]]:
    """Gather ``(seq_id, record)`` pairs of every rank to ``dst``, merged in
    ascending ``seq_id``; other ranks get None.  Duplicate seq ids are an error."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        merged = sorted(local)
    else:
        parts = [None] * dist.get_world_size() if dist.get_rank() == dst else None
        dist.gather_object(list(local), parts, dst=dst)
        if dist.get_rank() != dst:
            return None
        merged = sorted(x for part in parts for x in part)
    seqs = [s for s, _ in merged]
    if len(set(seqs)) != len(seqs):
        raise ValueError("duplicate seq_id across shards")
    return [r for _, r in merged]


def parse_shard(conf: np.ndarray, paf: np.ndarray, stride: int, topo, params, rank: int,
                world: int, parse_fn: Optional[Callable] = None, seq_base: int = 0,
                batch: int = 8192) -> List[Tuple[int, str]]:
    """Parse this rank's block of a [N,...] map stream; return (seq, record).

    ``parse_fn(conf_block, paf_block) -> list of per-frame pose lists`` defaults
    to the GPU parser on the current device.
    """
    from .pipeline_ops import pose_record

    lo, hi = shard_bounds(conf.shape[0], rank, world)
    if parse_fn is None:
        from .parser import default_parser

        def parse_fn(c, p):
            return default_parser(topo).parse_arrays(c, p, stride, params).all_poses()
    out = []
    for b0 in range(lo, hi, batch):
        b1 = min(hi, b0 + batch)
        for i, poses in zip(range(b0, b1), parse_fn(conf[b0:b1], paf[b0:b1])):
            out.append((seq_base + i, pose_record(seq_base + i, poses, topo)))
    return out


class MultiDeviceParser:
    """In-process frame sharding over several GPUs.

    One worker thread and one ``pf_ctx`` per entry of ``devices`` (contexts are
    not reentrant, so each stays on its own thread); a batch is cut into
    contiguous shards (``shard_bounds``), the shards run concurrently, and the
    results come back in frame order.  No maps move between GPUs and there is
    no collective: ``parse`` is pure per frame (paf.py:292-305).  The same
    device may appear more than once (two contexts on one GPU).
    """

    def __init__(self, topo, devices: Sequence[int], caps: Optional[dict] = None):
        from concurrent.futures import ThreadPoolExecutor

        if not devices:
            raise ValueError("MultiDeviceParser needs at least one device")
        self.topo = topo
        self.devices = [int(d) for d in devices]
        self._caps = caps
        self._pools = [ThreadPoolExecutor(max_workers=1) for _ in self.devices]
        self._engines = [None] * len(self.devices)

    def _engine(self, i: int):
        if self._engines[i] is None:
            from .parser import PafParser

            self._engines[i] = PafParser(self.topo, device=self.devices[i], caps=self._caps)
        return self._engines[i]

    def parse_arrays(self, conf: np.ndarray, paf: np.ndarray, stride: int, params) -> "ShardedResult":
        n, world = conf.shape[0], len(self.devices)

        def work(i: int):
            lo, hi = shard_bounds(n, i, world)
            if hi == lo:
                return lo, None
            return lo, self._engine(i).parse_arrays(conf[lo:hi], paf[lo:hi], stride, params)

        futures = [self._pools[i].submit(work, i) for i in range(world)]
        return ShardedResult(n, [f.result() for f in futures])

    def close(self) -> None:
        for i, pool in enumerate(self._pools):
            if self._engines[i] is not None:
                pool.submit(self._engines[i].close).result()
                self._engines[i] = None
            pool.shutdown()


class ShardedResult:
    """Frame-ordered view over the per-device ``BatchResult`` shards."""

    def __init__(self, n_frames: int, shards):
        self.n_frames = n_frames
        self._shards = [(lo, r) for lo, r in shards if r is not None]
        self.total_humans = sum(int(r.total_humans) for _, r in self._shards)

    def poses(self, frame: int):
        if not 0 <= frame < self.n_frames:
            raise IndexError(frame)
        for lo, r in reversed(self._shards):
            if frame >= lo:
                return r.poses(frame - lo)
        raise IndexError(frame)

    def all_poses(self):
        return [self.poses(f) for f in range(self.n_frames)]
