#!/usr/bin/env python
"""Pose-parsing throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[4], "C5"): a synthetic video stream at
368x656 — COCO-18 feature maps 19x46x82 + 38x46x82 f32 per frame, parsed with
the x8 bilinear upsample (Mode U) — sharded by frame across the GPUs of one
node with no collective (weak scaling: every GPU parses ``--frames`` frames
per step).  ``value`` times ``pf_parse_device`` on device-resident maps;
``e2e`` times ``pf_parse_host`` (the C ABI with pinned host buffers: H2D of
the maps and D2H of the humans inside the timed region).

  python bench.py [--gpus N --steps K --warmup W]          # B200 arm
  python bench.py --impl reference [...]                   # CPU reference arm

The reference (poseflow) is pure Python and cannot travel to the GPU box;
the reference arm runs the C restatement in oracle/ (kind "port") on all host
cores.  One JSON line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

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
            if name != "frames_per_launch" and name.split("<")[0].startswith(kernel):
                best = (val / d["frames_per_launch"]) * frames_per_launch
    return best


def paf_in_place_bytes():
    """PCIe read bytes per frame of the in-place (zero-copy) PAF reads of
    k_parse_frames, from the committed ncu capture (profiles/*_e2e_pcie.json)."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_e2e_pcie.json"))):
        try:
            with open(path) as f:
                best = (float(json.load(f)["paf_read_in_place_bytes_per_frame"]), os.path.basename(path))
        except Exception:
            continue
    return best


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ inputs
def make_inputs(n_distinct: int, seed: int):
    import paper_2108_11826_b200 as pf

    topo = pf.load_topology("coco18")
    sp = pf.SynthParams()
    scenes = [pf.procedural_scene(seed, s, GRID_W * STRIDE, GRID_H * STRIDE, sp)
              for s in range(n_distinct)]
    conf, paf = pf.synth.render_batch(scenes, topo, sp)
    return topo, conf, paf


def other_configs(dev, gpu):
    """BASELINE.json configs 1-4 (the parity configs) timed on the device
    with CUDA events, inputs resident: frames/s and the kernel split.  Not
    part of the headline; run after the timed region (rank 0, N=1)."""
    import torch

    import paper_2108_11826_b200 as pf

    topo = pf.load_topology("coco18")
    sp = pf.SynthParams()
    out = {}

    def timed(name, conf, paf, params, reps):
        eng = pf.PafParser(topo, device=gpu)
        c = torch.from_numpy(conf).to(dev)
        q = torch.from_numpy(paf).to(dev)
        for _ in range(2):
            eng.parse_tensors(c, q, STRIDE, params)
            eng.results()          # automatic capacities grow (and replay) here
        eng.set_timing(True)
        eng.kernel_times(reset=True)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        s0.record()
        for _ in range(reps):
            eng.parse_tensors(c, q, STRIDE, params)
        s1.record()
        torch.cuda.synchronize(dev)
        ms = s0.elapsed_time(s1) / reps
        kt = eng.kernel_times(reset=True)
        n = conf.shape[0]
        out[name] = {"frames": n, "ms_per_call": ms, "frames_per_s": n / (ms / 1e3),
                     "humans": int(eng.results().total_humans),
                     "kernels_ms": {k: v[0] / reps for k, v in kt.items()}}
        eng.close()

    scene = pf.procedural_scene(0, 1, 656, 368, sp)
    conf, paf = pf.synth.render_batch([scene], topo, sp)
    timed("C1 1 frame 3 people, Mode R", conf, paf, pf.ParserParams(upsample=1), 50)
    timed("C1 1 frame 3 people, Mode U", conf, paf, pf.ParserParams(upsample=8), 50)
    scenes = [pf.procedural_scene(7, s, 656, 368, sp) for s in range(64)]
    conf, paf = pf.synth.render_batch(scenes, topo, sp)
    timed("C2 64 frames 1-5 people, Mode U", conf, paf, pf.ParserParams(upsample=8), 20)
    scenes = [pf.crowd_scene(42, s) for s in range(256)]
    conf, paf = pf.synth.render_batch(scenes, topo, sp)
    timed("C3 256 crowded frames (40 people), Mode R", conf, paf, pf.ParserParams(upsample=1), 5)
    timed("C3 256 crowded frames (40 people), Mode U", conf, paf, pf.ParserParams(upsample=8), 5)
    scenes = [pf.GroundTruthScene(pf.crowd_scene(9, s, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
              for s in range(32)]
    conf, paf = pf.synth.render_batch(scenes, topo, sp)
    timed("C4 32 frames 1080x1920 (135x240 maps, 6 people), Mode U", conf, paf, pf.ParserParams(upsample=8), 5)
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


# ------------------------------------------------------------------ CPU legs
def cpu_oracle_run(conf, paf, topo, params, frames: int, threads: int):
    """Time the oracle (C restatement of the reference path) on `frames`
    frames spread over `threads` host threads (ctypes releases the GIL)."""
    import oracle

    idx = [i % conf.shape[0] for i in range(frames)]

    def one(i):
        oracle.parse_upsampled(conf[i], paf[i], topo, params, STRIDE, UP)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, idx))
    return time.perf_counter() - t0


def run_reference(args, rank, world):
    """--impl reference: the CPU reference path on all host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    import paper_2108_11826_b200 as pf

    oracle.build()
    topo, conf, paf = make_inputs(min(args.distinct, 64), seed=5)
    params = pf.ParserParams(upsample=UP)
    cores = os.cpu_count() or 1
    per_step = max(2 * cores, 8)
    for _ in range(args.warmup):
        cpu_oracle_run(conf, paf, topo, params, per_step, cores)
    t = 0.0
    for _ in range(args.steps):
        t += cpu_oracle_run(conf, paf, topo, params, per_step, cores)
    value = per_step * args.steps / t
    sample = (f"{per_step} frames/step of the C5 stream (procedural seed 5, 1-5 people), "
              f"Mode U oracle (bilinear_resize x8 of all 57 channels + parse) over {cores} threads")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C5 stream @368x656, 46x82 COCO-18 maps, x8 upsample (Mode U)",
                   "frames_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2108_11826_b200 as pf
    from paper_2108_11826_b200 import _native

    # one GPU per rank; ranks share devices only in the plumbing test (more
    # ranks than GPUs, PF_BENCH_BACKEND=gloo)
    gpu = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    params = pf.ParserParams(upsample=UP if args.mode == "U" else 1)
    F = args.frames
    if args.distinct >= F:
        # every frame distinct: F procedural scenes rendered on the GPU
        # (pf_render_maps, the GPU-resident producer); host copies of the
        # first frames feed the CPU baseline
        sp = pf.SynthParams()
        topo = pf.load_topology("coco18")
        scenes = [pf.procedural_scene(5 + 1000 * rank, s, GRID_W * STRIDE, GRID_H * STRIDE, sp) for s in range(F)]
        conf_d, paf_d = pf.synth.render_batch_gpu(scenes, topo, sp, device=gpu)
        conf_h = conf_d[:256].cpu().numpy()
        paf_h = paf_d[:256].cpu().numpy()
    else:
        topo, conf_h, paf_h = make_inputs(args.distinct, seed=5 + 1000 * rank)
        # device pool: `distinct` rendered frames tiled to F frames (F * 0.86 MB > L2)
        idx = torch.arange(F) % conf_h.shape[0]
        conf_d = torch.from_numpy(conf_h).to(dev)[idx.to(dev)].contiguous()
        paf_d = torch.from_numpy(paf_h).to(dev)[idx.to(dev)].contiguous()
    eng = pf.PafParser(topo, device=gpu)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up
    for _ in range(args.warmup):
        eng.parse_tensors(conf_d, paf_d, STRIDE, params)
    res = eng.results()
    humans_per_step = int(res.total_humans)
    torch.cuda.synchronize(dev)

    # ---- timed region: device-resident maps ----
    eng.set_timing(True)
    eng.kernel_times(reset=True)
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
    elapsed_ms = ev0.elapsed_time(ev1)
    ktimes = eng.kernel_times(reset=True)
    eng.set_timing(False)
    from paper_2108_11826_b200.sharding import max_over_ranks

    elapsed_ms = max_over_ranks(elapsed_ms)      # the job's time is its slowest rank's
    value = world * F * args.steps / (elapsed_ms / 1e3)

    # ---- e2e: through the C ABI from pinned host memory ----
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
    e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s)
    e2e_value = world * E * e2e_steps / e2e_s
    # conf: K of K+1 planes copied (the background plane is never read);
    # PAF: read in place from pinned host memory by k_parse_frames, so only
    # the sampled cells cross PCIe (ncu pcie__read_bytes, committed profile)
    paf_rd = paf_in_place_bytes()
    h2d_conf = E * K_PARTS * PLANE * 4
    h2d_paf = E * paf_rd[0] if paf_rd else E * PAF_FRAME_BYTES
    h2d = int(h2d_conf + h2d_paf)
    d2h = E * 8 + 32 + r.total_humans * (8 + 4 + K_PARTS * (8 + 8 + 4 + 4))

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

    # ---- roofline of the dominant kernel of the timed region ----
    chunk = 1024
    launches_per_step = {name: n / args.steps for name, (ms, n) in ktimes.items()}
    per_frame_bytes = {"k_nms_up": BYTES_FUSED_UN, "k_nms_up_win": BYTES_FUSED_UN,
                       "k_nms_up_corner": BYTES_FUSED_UN, "k_nms_up_scan": BYTES_FUSED_UN,
                       "k_nms_plane": BYTES_FUSED_UN}
    for name, (ms, n) in ktimes.items():
        frames_per_launch = F / launches_per_step[name]
        per_launch = ms / n
        stages[name] = {"ms_per_launch": per_launch, "launches": n,
                        "frames_per_launch": frames_per_launch,
                        "us_per_frame": per_launch * 1e3 / frames_per_launch,
                        "share_of_step": ms / max(elapsed_ms, 1e-9)}
        if name in per_frame_bytes:
            b = per_frame_bytes[name] * frames_per_launch
            stages[name].update({"bytes_per_launch": b, "bytes_kind": "algorithmic",
                                 "achieved_gbs": b / (per_launch / 1e3) / 1e9})
        else:
            # latency-bound gather (the line integral reads only the sampled PAF
            # cells): report its measured DRAM traffic, not a roofline
            t = ncu_traffic(name, frames_per_launch)
            stages[name].update({"bytes_per_launch": t, "bytes_kind": "ncu dram read+write",
                                 "achieved_gbs": t / (per_launch / 1e3) / 1e9 if t else None,
                                 "bound": "latency (gather + serial assembly)"})
    dominant = max(ktimes.items(), key=lambda kv: kv[1][0])[0] if ktimes else None
    roof = None
    if dominant:
        d = stages[dominant]
        traffic = args.traffic if args.traffic is not None else ncu_traffic(dominant, d["frames_per_launch"])
        roof = {"kernel": dominant, "bound": "hbm", "achieved": d["achieved_gbs"],
                "peak": peak_gbs, "unit": "GB/s",
                "frac": (d["achieved_gbs"] / peak_gbs) if d["achieved_gbs"] else None,
                "traffic": traffic, "peak_kind": peak_kind,
                "bytes_per_launch": d["bytes_per_launch"],
                "ms_per_launch": d["ms_per_launch"],
                "bytes_per_frame": per_frame_bytes.get(dominant, 0),
                "note": "algorithmic bytes = the low-res part maps the fused upsample+NMS must read "
                        "(SURVEY §8(d) 'fused U+N compulsory'); traffic = ncu dram read+write per launch"}
        # the fused upsample+NMS stage is two kernels when split (streaming +
        # survivor finish): report the stage as a whole too
        fused = [k for k in ("k_nms_up_scan", "k_nms_up_corner", "k_corner_finish", "k_corner_crowded", "k_nms_up_win",
                             "k_nms_up")
                 if k in stages]
        if fused:
            ms = sum(stages[k]["ms_per_launch"] * stages[k]["launches"] for k in fused) / args.steps
            b = BYTES_FUSED_UN * F
            roof["stage_upsample_nms"] = {"kernels": fused, "ms_per_step": ms, "achieved_gbs": b / (ms / 1e3) / 1e9,
                                          "frac": b / (ms / 1e3) / 1e9 / peak_gbs}

    # ---- CPU baseline (rank 0, N == 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        frames = max(256, 16 * cores)      # ~15-60 s of CPU work, a few s wall
        t = cpu_oracle_run(conf_h, paf_h, topo, params, frames, cores)
        cpu = {"value": frames / t, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{frames} frames of the same stream, Mode U oracle (C restatement of "
                         f"bilinear_resize x8 on all 57 channels + parse), {cores} threads, "
                         f"{t:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (procedural scenes, rendered on the GPU by pf_render_maps)",
            "config": {"workload": "C5 stream: synthetic 368x656 frames, 46x82 COCO-18 maps "
                                   "(19 conf + 38 paf), x8 bilinear upsample (Mode U), 1-5 people",
                       "frames_per_gpu_step": F, "distinct_frames": min(F, args.distinct),
                       "mode": args.mode, "parallelism": f"frame-sharded x{world}, no collective",
                       "l2": f"inputs {F * (CONF_FRAME_BYTES + PAF_FRAME_BYTES) / 1e9:.2f} GB/GPU > L2; no flush",
                       "humans_per_step": humans_per_step},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "frames_per_step": E, "steps": e2e_steps,
                    "h2d_gbs": h2d * e2e_steps * world / e2e_s / 1e9,
                    "h2d_conf_copied": h2d_conf, "h2d_paf_read_in_place": int(h2d_paf),
                    "h2d_paf_source": (f"ncu pcie__read_bytes of k_parse_frames, profiles/{paf_rd[1]}"
                                       if paf_rd else "whole PAF (no capture committed)"),
                    "path": "pf_parse_host (pinned host maps: conf planes H2D by copy engine, PAF read "
                            "in place over PCIe by the parse kernel -> kernels -> D2H humans)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk,
            "stages": stages,
        }
        if world == 1 and not args.no_configs:
            line["configs"] = other_configs(dev, gpu)
        print(json.dumps(line), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--frames", type=int, default=8192, help="frames per GPU per step")
    ap.add_argument("--distinct", type=int, default=8192,
                    help="distinct frames (>= --frames: all distinct, rendered on the GPU; else host-rendered, tiled)")
    ap.add_argument("--e2e-frames", type=int, default=8192, help="frames per e2e step (default: the device step)")
    ap.add_argument("--unfused-frames", type=int, default=256)
    ap.add_argument("--mode", choices=("U", "R"), default="U")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config (C1-C4) timings")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        ap.error("steps >= 1, warmup >= 0")

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else os.environ.get("PF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            import torch

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
