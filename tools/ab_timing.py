"""A/B: the C5 step (8192 GPU-rendered frames, Mode U) timed with CUDA events
around the whole step, per-kernel event timing OFF vs ON, with and without the
nvidia-smi sampler, plus options (PDL off etc.) given as NAME=VALUE args."""
import json
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from support import synth  # noqa: E402

topo = pf.load_topology("coco18")
sp = synth.SynthParams()
F = 8192
scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(F)]
conf, paf = synth.render_batch_gpu(scenes, topo, sp)
params = pf.ParserParams(upsample=8)
eng = pf.PafParser(topo)
for _ in range(3):
    eng.parse_tensors(conf, paf, 8, params)
eng.results()


def run(steps=30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.parse_tensors(conf, paf, 8, params)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


out = {}
for rep in range(2):
    eng.set_timing(False)
    out[f"off_{rep}"] = run()
    eng.set_timing(True)
    out[f"on_{rep}"] = run()
    eng.kernel_times(reset=True)
eng.set_timing(False)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                       stdout=subprocess.DEVNULL)
time.sleep(0.5)
out["off_sampler"] = run()
smi.terminate()
for arg in sys.argv[1:]:
    k, v = arg.split("=")
    eng.ctx.set_option(int(k), int(v))
    out[f"off_opt{k}={v}"] = run()
kt_eng = eng
kt_eng.set_timing(True)
kt_eng.kernel_times(reset=True)
run(10)
out["kernels_ms"] = {k: v[0] / 10 for k, v in kt_eng.kernel_times(reset=True).items()}
print(json.dumps(out))
