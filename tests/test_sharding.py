"""Multi-GPU path on CPU: frame sharding with gloo, world_size 2.

Each rank parses its shard (with the oracle standing in for the GPU — this is
a CPU test of the sharding / gather / timing plumbing); rank 0's merged JSONL
must equal the single-process result byte for byte."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2108_11826_b200 as pf
from support import synth
from paper_2108_11826_b200 import sharding


@pytest.mark.parametrize("n,world", [(0, 1), (1, 2), (7, 2), (8, 4), (8192, 8), (5, 8)])
def test_shard_bounds_partition(n, world):
    got = []
    for r in range(world):
        lo, hi = sharding.shard_bounds(n, r, world)
        assert 0 <= lo <= hi <= n
        got.extend(range(lo, hi))
    assert got == list(range(n))
    sizes = [np.subtract(*sharding.shard_bounds(n, r, world)[::-1]) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_round_robin():
    idx = [sharding.shard_indices(10, r, 3, "round_robin").tolist() for r in range(3)]
    assert sorted(sum(idx, [])) == list(range(10))


def _oracle_parse_fn(topo, params):
    import oracle

    def fn(conf, paf):
        out = []
        for c, p in zip(conf, paf):
            humans = oracle.parse(c, p, topo, params, 8).humans
            out.append([pf.HumanPose(tuple(None if k is None else pf.Keypoint(*k) for k in kps), s, n)
                        for s, n, kps in humans])
        return out
    return fn


def _inputs():
    topo = pf.load_topology("coco18")
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(11, s, 656, 368, sp) for s in range(6)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    return topo, conf, paf


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    topo, conf, paf = _inputs()
    params = pf.ParserParams()
    local = sharding.parse_shard(conf, paf, 8, topo, params, rank, world,
                                 parse_fn=_oracle_parse_fn(topo, params), seq_base=100)
    merged = sharding.gather_records(local)
    t = sharding.max_over_ranks(float(rank + 1))
    if rank == 0:
        with open(os.path.join(outdir, "merged.jsonl"), "w") as f:
            f.write("\n".join(merged) + "\n")
        with open(os.path.join(outdir, "tmax"), "w") as f:
            f.write(str(t))
    else:
        assert merged is None
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_matches_single_process(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    topo, conf, paf = _inputs()
    params = pf.ParserParams()
    single = sharding.parse_shard(conf, paf, 8, topo, params, 0, 1,
                                  parse_fn=_oracle_parse_fn(topo, params), seq_base=100)
    want = "\n".join(r for _, r in single) + "\n"
    assert (tmp_path / "merged.jsonl").read_text() == want
    assert float((tmp_path / "tmax").read_text()) == 2.0


def test_sharded_result_frame_order():
    """ShardedResult maps frame indices onto the per-device shards (host logic)."""
    from paper_2108_11826_b200.sharding import ShardedResult, shard_bounds

    class Fake:
        def __init__(self, lo, hi):
            self.lo, self.total_humans = lo, hi - lo

        def poses(self, f):
            return ["frame", self.lo + f]

    n, world = 11, 4
    shards = []
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        shards.append((lo, Fake(lo, hi) if hi > lo else None))
    res = ShardedResult(n, shards)
    assert [p[1] for p in res.all_poses()] == list(range(n))
    assert res.total_humans == n
    one = ShardedResult(1, [(0, Fake(0, 1)), (1, None), (1, None)])      # empty trailing shards
    assert one.poses(0) == ["frame", 0]
    import pytest

    with pytest.raises(IndexError):
        res.poses(n)
