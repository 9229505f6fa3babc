"""bench.py's multi-GPU plumbing on a CPU host: --gpus N with fewer devices
fails loudly instead of measuring one GPU, a WORLD_SIZE that disagrees with
--gpus is refused, and the reference arm under a 2-rank launch prints one
line from rank 0 (the other rank exits 0 without work)."""
import json
import os
import subprocess
import sys

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=600):
    e = dict(os.environ, CUDA_VISIBLE_DEVICES="", PYTHONDONTWRITEBYTECODE="1")
    e.update(env or {})
    return subprocess.run([sys.executable] + args, cwd=ROOT, env=e, capture_output=True, text=True,
                          timeout=timeout)


def test_more_gpus_than_devices_fails_loudly():
    p = _run([BENCH, "--gpus", "2", "--steps", "1", "--warmup", "0"])
    assert p.returncode != 0
    assert "only 0 CUDA device(s) visible" in p.stderr + p.stdout


def test_world_size_must_match_gpus():
    p = _run([BENCH, "--gpus", "1", "--steps", "1", "--warmup", "0"],
             env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 1" in p.stderr + p.stdout


def test_reference_arm_two_ranks_prints_one_line():
    p = _run(["-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29731", BENCH,
              "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--distinct", "8"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
