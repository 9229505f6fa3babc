"""Where the e2e time goes (dev tool): the conf copy alone (2-D pinned H2D in
128-frame chunks, as pf_parse_host issues it), pf_parse_host through ctypes
only, through parse_arrays (+ the BatchResult copy), with the PAF copied
instead of read in place, and the per-kernel device times of one e2e call."""
import ctypes
import sys
import time

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402

E = 8192
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(E)]
conf_d, paf_d = synth.render_batch_gpu(scenes, topo, sp)
pin_conf = _native.PinnedArray((E, 19, 46, 82))
pin_paf = _native.PinnedArray((E, 38, 46, 82))
pin_conf.array[:] = conf_d.cpu().numpy()
pin_paf.array[:] = paf_d.cpu().numpy()
del conf_d, paf_d
plane = 46 * 82 * 4
fr = 19 * plane
dst = torch.empty(2, 128, 19, 46, 82, device="cuda")
stream = torch.cuda.Stream()
base = pin_conf.array.ctypes.data


def copy_only(reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for ci, f0 in enumerate(range(0, E, 128)):
            d = dst[ci % 2].data_ptr()
            rt.cudaMemcpy2DAsync(d, fr, base + f0 * fr, fr, 18 * plane, 128,
                                 rt.cudaMemcpyKind.cudaMemcpyHostToDevice, stream.cuda_stream)
        stream.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


t = copy_only()
print(f"conf copy only: {t * 1e3:.2f} ms per {E} frames = {E * 18 * plane / t / 1e9:.1f} GB/s -> ceiling "
      f"{E / t:.0f} frames/s", flush=True)

params = pf.ParserParams(upsample=8)
eng = pf.PafParser(topo)
p = params.to_native()
res = _native.PfResults()


def raw_call():
    eng.ctx.check(eng.ctx.lib.pf_parse_host(eng.ctx.handle, pin_conf.array.ctypes.data,
                                            pin_paf.array.ctypes.data, E, 46, 82, 8, ctypes.byref(p),
                                            ctypes.byref(res)))


for label, fn in (("pf_parse_host (ctypes only)", raw_call),
                  ("parse_arrays (+ BatchResult copy)", lambda: eng.parse_arrays(pin_conf.array, pin_paf.array, 8, params))):
    for _ in range(2):
        fn()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    dt = (time.perf_counter() - t0) / 5
    print(f"{label}: {dt * 1e3:.2f} ms = {E / dt:.0f} frames/s", flush=True)

eng.ctx.set_option(_native.PF_OPT_PAF_ZERO_COPY, 0)
for _ in range(2):
    raw_call()
t0 = time.perf_counter()
for _ in range(3):
    raw_call()
dt = (time.perf_counter() - t0) / 3
print(f"PAF copied too: {dt * 1e3:.2f} ms = {E / dt:.0f} frames/s ({E * (18 * plane + 38 * plane) / dt / 1e9:.1f} GB/s)",
      flush=True)
eng.ctx.set_option(_native.PF_OPT_PAF_ZERO_COPY, 1)
eng.set_timing(True)
eng.kernel_times(reset=True)
raw_call()
kt = eng.kernel_times(reset=True)
print("kernel ms per e2e call:", {k: (round(v[0], 3), v[1]) for k, v in kt.items()}, flush=True)
