#!/usr/bin/env python
"""Pose-parsing throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[4], "C5"): a synthetic video stream at
368x656 — COCO-18 feature maps 19x46x82 + 38x46x82 f32 per frame, parsed with
the x8 bilinear upsample (Mode U) — sharded by frame across the GPUs of one
node with no collective (weak scaling: every GPU parses ``--frames`` distinct
frames per step).  ``value`` times ``pf_parse_device`` on device-resident
maps (per-kernel event timing OFF); the per-kernel split comes from a second
pass with PF_OPT_TIMING on.  ``e2e`` times ``pf_parse_host`` (the C ABI with
pinned host buffers: H2D of the maps and D2H of the humans inside the timed
region).  After the timed region the step's own output is checked against
the oracle on a strided sample of its frames (``parity``); a mismatch exits
non-zero.

  python bench.py [--gpus N --steps K --warmup W]          # B200 arm
  python bench.py --impl reference [...]                   # CPU reference arm

``--gpus N`` without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU).  The reference arm runs the genuine reference
(``poseflow`` installed in ``baseline/_ref``: ``operators.bilinear_resize`` x8
on every channel + ``paf.parse(stride=1)``) in one process per host core;
the C restatement in ``oracle/`` (kind "port") is timed beside it.  One JSON
line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "pose-parsing frames/sec @368x656 COCO-18 at 1/2/4/8 B200; % HBM roofline"
UNIT = "frames/s"
GRID_H, GRID_W, STRIDE, UP = 46, 82, 8, 8
K_PARTS, N_LIMBS = 18, 19
PLANE = GRID_H * GRID_W
CONF_FRAME_BYTES = (K_PARTS + 1) * PLANE * 4        # 286,672
PAF_FRAME_BYTES = 2 * N_LIMBS * PLANE * 4           # 573,344
# SURVEY.md §8(d) algorithmic bytes per frame
BYTES_FUSED_UN = K_PARTS * PLANE * 4                # 271,584: read low-res part maps once
BYTES_UPSAMPLE = K_PARTS * PLANE * 4 + K_PARTS * PLANE * 64 * 4   # 17,652,960: read low + write full (18 part ch)
BYTES_NMS_FULL = K_PARTS * PLANE * 64 * 4           # 17,381,376: read full-res part maps
BYTES_BLUR = 2 * K_PARTS * PLANE * 64 * 4           # 34,762,752: read + write full-res part maps


def ncu_traffic(kernel: str, frames_per_launch: float):
    """dram read+write bytes per launch of `kernel` from the committed ncu
    capture (profiles/<round>_traffic.json), scaled to this launch size."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except Exception:
            continue
        for name, val in d.items():
            if name != "frames_per_launch" and name.split("<")[0] == kernel:
                best = (val / d["frames_per_launch"]) * frames_per_launch
    return best


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_info():
    """Host CPU description for the CPU baselines (lscpu + os.cpu_count)."""
    info = {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keep = ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket", "Socket(s)",
                "NUMA node(s)", "CPU max MHz", "L3 cache")
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in keep and k.strip() not in info:
                info[k.strip()] = v.strip()
    except Exception as exc:   # noqa: BLE001
        info["lscpu"] = f"unavailable: {exc}"
    return info


def workload_config(args, world):
    """The workload both arms report (identical dict in both JSON lines)."""
    return {"workload": "C5 stream: synthetic 368x656 frames, 46x82 COCO-18 maps (19 conf + 38 paf), "
                        "x8 bilinear upsample (Mode U), 1-5 people per frame",
            "frames_per_gpu_step": args.frames, "mode": args.mode,
            "parallelism": f"frame-sharded x{world}, no collective",
            "l2": f"inputs {args.frames * (CONF_FRAME_BYTES + PAF_FRAME_BYTES) / 1e9:.2f} GB per GPU > 126 MB L2; "
                  f"no flush"}


# ------------------------------------------------------------------ inputs
def make_inputs(n_distinct: int, seed: int):
    import paper_2108_11826_b200 as pf
    from support import synth

    topo = pf.load_topology("coco18")
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(seed, s, GRID_W * STRIDE, GRID_H * STRIDE, sp)
              for s in range(n_distinct)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    return topo, conf, paf


def other_configs(dev, gpu):
    """BASELINE.json configs 1-4 (the parity configs) timed on the device
    with CUDA events, inputs resident: frames/s (timing off), then the kernel
    split in a separate pass.  Not part of the headline; rank 0, N=1."""
    import torch

    import paper_2108_11826_b200 as pf
    from support import synth

    topo = pf.load_topology("coco18")
    sp = synth.SynthParams()
    out = {}

    def timed(name, conf, paf, params, reps):
        eng = pf.PafParser(topo, device=gpu)
        c = torch.from_numpy(conf).to(dev)
        q = torch.from_numpy(paf).to(dev)
        for _ in range(2):
            eng.parse_tensors(c, q, STRIDE, params)
            eng.results()          # automatic capacities grow (and replay) here
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        s0.record()
        for _ in range(reps):
            eng.parse_tensors(c, q, STRIDE, params)
        s1.record()
        torch.cuda.synchronize(dev)
        ms = s0.elapsed_time(s1) / reps
        eng.set_timing(True)
        eng.kernel_times(reset=True)
        for _ in range(reps):
            eng.parse_tensors(c, q, STRIDE, params)
        kt = eng.kernel_times(reset=True)
        eng.set_timing(False)
        n = conf.shape[0]
        out[name] = {"frames": n, "ms_per_call": ms, "frames_per_s": n / (ms / 1e3),
                     "humans": int(eng.results().total_humans),
                     "kernels_ms": {k: v[0] / reps for k, v in kt.items()}}
        eng.close()
        return out[name]

    scene = synth.procedural_scene(0, 1, 656, 368, sp)
    conf, paf = synth.render_batch([scene], topo, sp)
    timed("C1 1 frame 3 people, Mode R", conf, paf, pf.ParserParams(upsample=1), 50)
    timed("C1 1 frame 3 people, Mode U", conf, paf, pf.ParserParams(upsample=8), 50)
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(64)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    timed("C2 64 frames 1-5 people, Mode U", conf, paf, pf.ParserParams(upsample=8), 20)
    scenes = [synth.crowd_scene(42, s) for s in range(256)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    timed("C3 256 crowded frames (40 people), Mode R", conf, paf, pf.ParserParams(upsample=1), 5)
    timed("C3 256 crowded frames (40 people), Mode U", conf, paf, pf.ParserParams(upsample=8), 5)
    scenes = [synth.GroundTruthScene(synth.crowd_scene(9, s, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
              for s in range(32)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    timed("C4 32 frames 1080x1920 (135x240 maps, 6 people), Mode U", conf, paf, pf.ParserParams(upsample=8), 5)
    # blur: C2's frames, x8 upsample then sigma = 1 (radius 3) Gaussian on the part maps
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(64)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    r = timed("C5 frames with blur sigma=1, 64 frames, Mode U", conf, paf,
              pf.ParserParams(upsample=8, blur_sigma=1.0), 10)
    peak, _ = measured_peaks()
    for k, ms in r["kernels_ms"].items():
        if k.startswith("k_blur") or k.startswith("k_up_blur"):
            gbs = BYTES_BLUR * 64 / (ms / 1e3) / 1e9
            r.setdefault("blur", {})[k] = {"bytes_per_frame": BYTES_BLUR, "achieved_gbs": gbs, "frac": gbs / peak,
                                           "bytes_kind": "SURVEY §8(d) G: read+write full-res part maps"}
    # C4 pre-processing: u8 1080x1920 frames -> f32 CHW (same size: layout + /255)
    frames = torch.randint(0, 256, (32, 1080, 1920, 3), dtype=torch.uint8, device=dev)
    for _ in range(2):
        pf.preprocess_batch(frames, 1080, 1920, device=gpu)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    s0.record()
    for _ in range(10):
        pf.preprocess_batch(frames, 1080, 1920, device=gpu)
    s1.record()
    torch.cuda.synchronize(dev)
    ms = s0.elapsed_time(s1) / 10
    nbytes = 32 * (1080 * 1920 * 3 + 3 * 1080 * 1920 * 4)
    out["C4 pre-processing 32 u8 frames 1080x1920 -> f32 CHW"] = {
        "frames": 32, "ms_per_call": ms, "frames_per_s": 32 / (ms / 1e3),
        "achieved_gbs": nbytes / (ms / 1e3) / 1e9, "bytes_per_frame": nbytes // 32,
        "note": "includes a torch.empty of the output per call"}
    return out


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ PCIe
def gpu_numa(gpu: int):
    """NUMA node and local CPUs of the GPU's PCIe slot (sysfs), for NUMA-local
    pinned host buffers."""
    try:
        import torch

        p = torch.cuda.get_device_properties(gpu)
        base = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(os.path.join(base, "numa_node")) as f:
            node = int(f.read().strip())
        with open(os.path.join(base, "local_cpulist")) as f:
            spec = f.read().strip()
    except Exception:
        return None, None
    cpus = set()
    for part in spec.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return node, cpus


def pinned_copy_peaks(dev, nbytes: int = 1 << 30):
    """Pinned host <-> device copy bandwidth (GB/s, best of 5 copies of
    ``nbytes``, CUDA events): the e2e leg's link ceiling."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, (a, b) in (("h2d", (dst, src)), ("d2h", (src, dst))):
        a.copy_(b, non_blocking=True)
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a.copy_(b, non_blocking=True)
            e1.record()
            torch.cuda.synchronize(dev)
            best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name] = best
    del src, dst
    return out


# ------------------------------------------------------------------ CPU legs
def cpu_oracle_run(conf, paf, topo, params, frames: int, threads: int, offset: int = 0):
    """Time the oracle (C restatement of the reference path) on `frames`
    frames spread over `threads` host threads (ctypes releases the GIL)."""
    import oracle

    idx = [(offset + i) % conf.shape[0] for i in range(frames)]

    def one(i):
        oracle.parse_upsampled(conf[i], paf[i], topo, params, STRIDE, UP)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, idx))
    return time.perf_counter() - t0


_REF_STATE = {}


def _ref_init(conf, paf):
    """Pool initializer: the genuine reference, imported from baseline/_ref."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from poseflow import topology  # noqa: F401

    _REF_STATE["conf"], _REF_STATE["paf"] = conf, paf


def _ref_parse_one(i):
    """One frame through the reference's own functions: Mode U is
    operators.bilinear_resize (operators.py:79-107) x8 on every channel, then
    paf.parse (paf.py:292-305) on FeatureMaps(stride=1)."""
    from poseflow import operators, paf as ref_paf
    from poseflow.topology import load_topology
    from poseflow.types import FeatureMaps, TensorF32

    topo = _REF_STATE.get("topo")
    if topo is None:
        topo = _REF_STATE["topo"] = load_topology("coco18")
    conf, paf = _REF_STATE["conf"][i], _REF_STATE["paf"][i]
    h, w = conf.shape[1:]
    cu = np.stack([operators.bilinear_resize(ch, h * UP, w * UP) for ch in conf])
    pu = np.stack([operators.bilinear_resize(ch, h * UP, w * UP) for ch in paf])
    maps = FeatureMaps(TensorF32.from_array(cu), TensorF32.from_array(pu), STRIDE // UP, i)
    return len(ref_paf.parse(maps, topo, ref_paf.ParserParams()))


class ReferencePool:
    """The genuine reference (pure Python + numpy, GIL-bound) in one process
    per host core, forked after the inputs exist."""

    def __init__(self, conf, paf, procs: int):
        import multiprocessing as mp

        self.procs = procs
        self.n = conf.shape[0]
        self.pool = mp.get_context("fork").Pool(procs, initializer=_ref_init, initargs=(conf, paf))

    def run(self, frames: int, offset: int = 0) -> float:
        idx = [(offset + i) % self.n for i in range(frames)]
        t0 = time.perf_counter()
        self.pool.map(_ref_parse_one, idx, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.terminate()
        self.pool.join()


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "poseflow"))


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on all host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    import paper_2108_11826_b200 as pf

    oracle.build()
    topo, conf, paf = make_inputs(min(args.distinct, 64), seed=5)
    params = pf.ParserParams(upsample=UP)
    cores = len(os.sched_getaffinity(0))
    host = host_info()
    # the C port beside it (all cores, threads)
    port_frames = max(2 * cores, 8)
    cpu_oracle_run(conf, paf, topo, params, port_frames, cores)
    tp = sum(cpu_oracle_run(conf, paf, topo, params, port_frames, cores, s * port_frames) for s in range(3))
    port = {"value": 3 * port_frames / tp, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{3 * port_frames} frames of the C5 stream, oracle/ C restatement, {cores} threads"}
    if reference_available():
        per_step = cores
        pool = ReferencePool(conf, paf, cores)
        for s in range(args.warmup):
            pool.run(per_step, s * per_step)
        t = 0.0
        for s in range(args.steps):
            t += pool.run(per_step, (args.warmup + s) * per_step)
        pool.close()
        kind = "reference"
        sample = (f"{per_step} frames/step of the C5 stream (procedural seed 5, 1-5 people, 64 distinct), genuine "
                  f"poseflow from baseline/_ref: operators.bilinear_resize x8 on all 57 channels + "
                  f"paf.parse(stride=1), {cores} processes")
    else:
        per_step = port_frames
        t = sum(cpu_oracle_run(conf, paf, topo, params, per_step, cores, s * per_step) for s in range(args.steps))
        kind = "port"
        sample = f"{per_step} frames/step, oracle/ C restatement (baseline/_ref missing), {cores} threads"
    value = per_step * args.steps / t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (procedural scenes, host renderer)",
        "config": workload_config(args, world),
        "sample_frames_per_step": per_step,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "host": host},
        "cpu_port": port,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def sum_over_ranks(value: int) -> int:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(value)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([int(value)], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    return int(t.item())


def check_parity(res, conf_d, paf_d, topo, params, n_check: int):
    """The timed step's own output against the oracle on a strided sample of
    its frames (pose_record bytes, operators.py:293-310)."""
    import oracle
    import paper_2108_11826_b200 as pf

    F = conf_d.shape[0]
    idx = sorted(set(np.linspace(0, F - 1, n_check).astype(int).tolist()))
    conf = conf_d[idx].cpu().numpy()
    paf = paf_d[idx].cpu().numpy()

    def one(j):
        r = oracle.parse_upsampled(conf[j], paf[j], topo, params, STRIDE, params.upsample) \
            if params.upsample > 1 else oracle.parse(conf[j], paf[j], topo, params, STRIDE)
        poses = [pf.HumanPose(keypoints=tuple(None if k is None else pf.Keypoint(*k) for k in kps),
                              score=s, n_parts=n) for s, n, kps in r.humans]
        return pf.pose_record(idx[j], poses, topo)

    with ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
        want = list(ex.map(one, range(len(idx))))
    got = [pf.pose_record(f, res.poses(f), topo) for f in idx]
    bad = [idx[j] for j in range(len(idx)) if got[j] != want[j]]
    return {"frames_checked": len(idx), "mismatches": len(bad), "first_mismatch": bad[:5],
            "humans_checked": int(sum(res.frame_count[f] for f in idx)),
            "sample": f"{len(idx)} frames evenly spaced over the timed step's {F}, oracle Mode U "
                      f"(bilinear_resize x8 + parse), pose_record bytes"}


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2108_11826_b200 as pf
    from paper_2108_11826_b200 import _native
    from paper_2108_11826_b200.sharding import max_over_ranks
    from support import synth

    ndev = torch.cuda.device_count()
    gpu = local_rank % ndev
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    numa_node, numa_cpus = gpu_numa(gpu)
    if numa_cpus and world > 1:
        try:      # pinned buffers are first-touched by this process: keep them on the GPU's NUMA node
            os.sched_setaffinity(0, numa_cpus & set(range(os.cpu_count() or 1)) or numa_cpus)
        except Exception:
            pass
    params = pf.ParserParams(upsample=UP if args.mode == "U" else 1)
    F = args.frames
    sp = synth.SynthParams()
    topo = pf.load_topology("coco18")
    # every frame distinct: F procedural scenes rendered on the GPU
    # (pf_render_maps, the GPU-resident producer); per-rank seeds
    scenes = [synth.procedural_scene(5 + 1000 * rank, s, GRID_W * STRIDE, GRID_H * STRIDE, sp) for s in range(F)]
    conf_d, paf_d = synth.render_batch_gpu(scenes, topo, sp, device=gpu)
    eng = pf.PafParser(topo, device=gpu)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (automatic capacities settle here)
    for _ in range(args.warmup):
        eng.parse_tensors(conf_d, paf_d, STRIDE, params)
    res = eng.results()
    torch.cuda.synchronize(dev)

    # ---- timed region: device-resident maps, per-kernel timing OFF ----
    eng.set_timing(False)
    clocks = ClockSampler(gpu)
    clocks.start()
    time.sleep(0.3)  # let the sampler attach
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = eng.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        eng.parse_tensors(conf_d, paf_d, STRIDE, params)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    launches = eng.launch_count() - launches0
    clk = clocks.stop()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))     # the job's time is its slowest rank's
    value = world * F * args.steps / (elapsed_ms / 1e3)
    res = eng.results()                                    # the last timed step's humans
    humans_per_step = int(res.total_humans)

    # ---- parity of the timed step (every rank checks its own frames) ----
    parity = check_parity(res, conf_d, paf_d, topo, params, args.parity_frames)
    parity["mismatches_all_ranks"] = sum_over_ranks(parity["mismatches"])
    parity["frames_checked_all_ranks"] = sum_over_ranks(parity["frames_checked"])

    # ---- per-kernel split: a separate pass with CUDA events around every launch ----
    split_steps = max(1, min(args.steps, args.split_steps))
    eng.set_timing(True)
    eng.kernel_times(reset=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(split_steps):
        eng.parse_tensors(conf_d, paf_d, STRIDE, params)
    s1.record(stream)
    torch.cuda.synchronize(dev)
    split_ms_per_step = s0.elapsed_time(s1) / split_steps
    ktimes = eng.kernel_times(reset=True)
    eng.set_timing(False)

    # ---- e2e: through the C ABI from pinned host memory ----
    copy_peak = pinned_copy_peaks(dev)
    E = min(args.e2e_frames, F)
    pin_conf = _native.PinnedArray((E, K_PARTS + 1, GRID_H, GRID_W))
    pin_paf = _native.PinnedArray((E, 2 * N_LIMBS, GRID_H, GRID_W))
    pin_conf.array[:] = conf_d[:E].cpu().numpy()     # the device step's frames, from host memory
    pin_paf.array[:] = paf_d[:E].cpu().numpy()
    for _ in range(max(1, args.warmup)):
        r = eng.parse_arrays(pin_conf.array, pin_paf.array, STRIDE, params)
    barrier()
    e2e_steps = min(args.steps, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):          # synchronous API: H2D + kernels + D2H of humans
        r = eng.parse_arrays(pin_conf.array, pin_paf.array, STRIDE, params)
    e2e_s_local = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s_local)
    e2e_value = world * E * e2e_steps / e2e_s
    # counted bytes: conf planes copied by the copy engine (K of K+1 planes;
    # the background plane is never read), the PAF sectors the parse kernel
    # reads in place — counted in-run by one instrumented call of the same
    # path (PF_OPT_COUNT_PAF: a bitmap of the 32-byte sectors sampled) — and
    # the humans read back
    h2d_conf = E * K_PARTS * PLANE * 4
    eng.ctx.set_option(_native.PF_OPT_COUNT_PAF, 1)
    r_count = eng.parse_arrays(pin_conf.array, pin_paf.array, STRIDE, params)
    paf_sectors = eng.ctx.paf_sectors()
    eng.ctx.set_option(_native.PF_OPT_COUNT_PAF, 0)
    h2d_paf = paf_sectors * 32
    counted_same = r_count.total_humans == r.total_humans
    d2h = E * 8 + 32 + r.total_humans * (8 + 4 + K_PARTS * (8 + 8 + 4 + 4))
    h2d = int(h2d_conf + h2d_paf)
    h2d_gbs = h2d * e2e_steps / e2e_s_local / 1e9

    # ---- unfused Mode U stages (materialised x8 maps through HBM) ----
    stages = {}
    peak_gbs, peak_kind = measured_peaks()
    if args.mode == "U" and not args.no_unfused:
        U = min(args.unfused_frames, F)
        eng.set_materialise(True)
        eng.set_timing(True)
        for _ in range(2):
            eng.parse_tensors(conf_d[:U], paf_d[:U], STRIDE, params)
        eng.kernel_times(reset=True)
        for _ in range(3):
            eng.parse_tensors(conf_d[:U], paf_d[:U], STRIDE, params)
        kt = eng.kernel_times(reset=True)
        eng.set_timing(False)
        eng.set_materialise(False)
        for name, per_frame in (("k_resize_planes", BYTES_UPSAMPLE), ("k_nms_plane", BYTES_NMS_FULL)):
            if name in kt:
                ms, n = kt[name]
                per_launch = ms / n
                frames_per_launch = U * 3 / n
                gbs = per_frame * frames_per_launch / (per_launch / 1e3) / 1e9
                stages[f"unfused.{name}"] = {
                    "ms_per_launch": per_launch, "frames_per_launch": frames_per_launch,
                    "bytes_per_frame": per_frame, "achieved_gbs": gbs,
                    "frac": gbs / peak_gbs}

    # ---- roofline of the dominant kernel (split pass) ----
    launches_per_step = {name: n / split_steps for name, (ms, n) in ktimes.items()}
    per_frame_bytes = {"k_nms_up": BYTES_FUSED_UN, "k_nms_up_win": BYTES_FUSED_UN,
                       "k_nms_up_corner": BYTES_FUSED_UN, "k_nms_up_scan": BYTES_FUSED_UN,
                       "k_nms_plane": BYTES_FUSED_UN}
    for name, (ms, n) in ktimes.items():
        frames_per_launch = F / launches_per_step[name]
        per_launch = ms / n
        stages[name] = {"ms_per_launch": per_launch, "launches": n,
                        "frames_per_launch": frames_per_launch,
                        "us_per_frame": per_launch * 1e3 / frames_per_launch,
                        "share_of_step": ms / split_steps / max(split_ms_per_step, 1e-9)}
        if name in per_frame_bytes:
            b = per_frame_bytes[name] * frames_per_launch
            stages[name].update({"bytes_per_launch": b, "bytes_kind": "algorithmic",
                                 "achieved_gbs": b / (per_launch / 1e3) / 1e9})
        else:
            t = ncu_traffic(name, frames_per_launch)
            stages[name].update({"bytes_per_launch": t, "bytes_kind": "ncu dram read+write (profiles/)",
                                 "achieved_gbs": t / (per_launch / 1e3) / 1e9 if t else None,
                                 "bound": "latency (gather + serial assembly)"})
    dominant = max(ktimes.items(), key=lambda kv: kv[1][0])[0] if ktimes else None
    roof = None
    if dominant:
        d = stages[dominant]
        traffic = ncu_traffic(dominant, d["frames_per_launch"])
        roof = {"kernel": dominant, "bound": "hbm", "achieved": d.get("achieved_gbs"),
                "peak": peak_gbs, "unit": "GB/s",
                "frac": (d["achieved_gbs"] / peak_gbs) if d.get("achieved_gbs") else None,
                "traffic": traffic, "peak_kind": peak_kind,
                "bytes_per_launch": d["bytes_per_launch"], "ms_per_launch": d["ms_per_launch"],
                "bytes_per_frame": per_frame_bytes.get(dominant, 0),
                "timing": f"CUDA events around every launch, separate pass of {split_steps} steps "
                          f"({split_ms_per_step:.3f} ms/step vs {elapsed_ms / args.steps:.3f} untimed)",
                "note": "algorithmic bytes = the low-res part maps the fused upsample+NMS must read "
                        "(SURVEY §8(d) 'fused U+N compulsory'); traffic = ncu dram read+write per launch"}
        fused = [k for k in ("k_nms_up_scan", "k_nms_up_corner", "k_corner_finish", "k_corner_crowded",
                             "k_nms_up_win", "k_nms_up") if k in stages]
        if fused:
            ms = sum(stages[k]["ms_per_launch"] * stages[k]["launches"] for k in fused) / split_steps
            b = BYTES_FUSED_UN * F
            roof["stage_upsample_nms"] = {"kernels": fused, "ms_per_step": ms,
                                          "achieved_gbs": b / (ms / 1e3) / 1e9,
                                          "frac": b / (ms / 1e3) / 1e9 / peak_gbs}
        step_bytes = F * BYTES_FUSED_UN + h2d_paf * F / E
        roof["step"] = {"compulsory_bytes_per_frame": step_bytes / F,
                        "floor_ms": step_bytes / (peak_gbs * 1e9) * 1e3,
                        "ms_per_step": elapsed_ms / args.steps,
                        "frac": (step_bytes / (peak_gbs * 1e9) * 1e3) / (elapsed_ms / args.steps),
                        "note": "conf part planes + the distinct 32-byte PAF sectors the line integral samples "
                                "(counted in-run, PF_OPT_COUNT_PAF)"}

    # ---- CPU baselines (rank 0, N == 1) ----
    cpu = cpu_port = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.build()
        cores = len(os.sched_getaffinity(0))
        conf_h = conf_d[:64].cpu().numpy()
        paf_h = paf_d[:64].cpu().numpy()
        frames = max(256, 16 * cores)
        t = cpu_oracle_run(conf_h, paf_h, topo, params, frames, cores)
        cpu_port = {"value": frames / t, "unit": UNIT, "cores": cores, "kind": "port",
                    "sample": f"{frames} frames of the same stream, oracle/ C restatement (bilinear_resize x8 on "
                              f"all 57 channels + parse), {cores} threads, {t:.2f} s wall"}
        host = host_info()
        if reference_available():
            pool = ReferencePool(conf_h, paf_h, cores)
            pool.run(cores)                         # fork + import warm-up
            n_ref = 2 * cores
            t = pool.run(n_ref, cores)
            pool.close()
            cpu = {"value": n_ref / t, "unit": UNIT, "cores": cores, "kind": "reference", "host": host,
                   "sample": f"{n_ref} frames of the same stream through the genuine poseflow (baseline/_ref): "
                             f"operators.bilinear_resize x8 on all 57 channels + paf.parse(stride=1), "
                             f"{cores} processes, {t:.2f} s wall"}
        else:
            cpu = dict(cpu_port, host=host)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (procedural scenes, rendered on the GPU by pf_render_maps)",
            "config": workload_config(args, world),
            "humans_per_step": humans_per_step,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "frames_per_step": E, "steps": e2e_steps,
                    "h2d_gbs": h2d_gbs, "pcie_peak_gbs": copy_peak["h2d"], "d2h_peak_gbs": copy_peak["d2h"],
                    "frac_of_pcie_peak": h2d_gbs / copy_peak["h2d"] if copy_peak["h2d"] else None,
                    "h2d_conf_copied": h2d_conf, "h2d_paf_read_in_place": h2d_paf,
                    "paf_bytes_per_frame": h2d_paf / E,
                    "paf_bytes_source": "distinct 32-byte PAF sectors sampled, counted in-run by an instrumented "
                                        "call of the same path (PF_OPT_COUNT_PAF)",
                    "instrumented_call_same_humans": counted_same,
                    "numa_node": numa_node,
                    "path": "pf_parse_host (pinned host maps: conf planes H2D by copy engine, PAF read "
                            "in place over PCIe by the parse kernel -> kernels -> D2H humans)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "cpu_port": cpu_port,
            "gpu_launches": launches,
            "clocks": clk,
            "stages": stages,
            "devices": {"rank0_gpu": gpu, "visible": ndev, "name": torch.cuda.get_device_name(gpu)},
        }
        if world == 1 and not args.no_configs:
            line["configs"] = other_configs(dev, gpu)
        print(json.dumps(line), flush=True)
    eng.close()
    if parity["mismatches_all_ranks"]:
        raise SystemExit(f"parity: {parity['mismatches_all_ranks']} frames of the timed step differ from "
                         f"the oracle")


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--split-steps", type=int, default=20, help="steps of the per-kernel timing pass")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--frames", type=int, default=8192, help="distinct frames per GPU per step")
    ap.add_argument("--distinct", type=int, default=64, help="host-rendered frames of the reference arm")
    ap.add_argument("--e2e-frames", type=int, default=8192, help="frames per e2e step (default: the device step)")
    ap.add_argument("--parity-frames", type=int, default=64, help="frames of the timed step checked vs the oracle")
    ap.add_argument("--unfused-frames", type=int, default=256)
    ap.add_argument("--mode", choices=("U", "R"), default="U")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config (C1-C4) timings")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1 or args.gpus < 1:
        ap.error("steps >= 1, warmup >= 0, gpus >= 1")

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "b200":
        # one process per GPU: re-launch under torch.distributed.run
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
        cmd += sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else os.environ.get("PF_BENCH_BACKEND", "nccl")
        if args.impl == "b200":
            import torch

            if torch.cuda.device_count() < world and backend == "nccl":
                sys.exit(f"bench.py: {world} ranks but {torch.cuda.device_count()} CUDA device(s)")
            torch.cuda.set_device(local_rank % torch.cuda.device_count())
        dist.init_process_group(backend=backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
