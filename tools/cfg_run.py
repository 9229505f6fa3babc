"""Run one BASELINE config a few times on device-resident maps (for ncu
captures and quick timings): c3u / c3r (256 crowded frames), blur (64 C2
frames, x8 + sigma 1), c4u (32 frames 1080p)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from support import synth  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
if name.startswith("c3"):
    scenes = [synth.crowd_scene(42, s) for s in range(256)]
    params = pf.ParserParams(upsample=8 if name == "c3u" else 1)
elif name == "blur":
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(64)]
    params = pf.ParserParams(upsample=8, blur_sigma=1.0)
elif name == "c4u":
    scenes = [synth.GroundTruthScene(synth.crowd_scene(9, s, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
              for s in range(32)]
    params = pf.ParserParams(upsample=8)
conf, paf = synth.render_batch_gpu(scenes, topo, sp)
eng = pf.PafParser(topo)
for kv in filter(None, __import__("os").environ.get("PF_OPTS", "").split(",")):   # e.g. PF_OPTS=9=0
    k, v = kv.split("=")
    eng.ctx.set_option(int(k), int(v))
for _ in range(2):
    eng.parse_tensors(conf, paf, 8, params)
    eng.results()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    eng.parse_tensors(conf, paf, 8, params)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
eng.set_timing(True)
eng.kernel_times(reset=True)
for _ in range(reps):
    eng.parse_tensors(conf, paf, 8, params)
kt = {k: round(v[0] / reps, 4) for k, v in eng.kernel_times(reset=True).items()}
print(json.dumps({"config": name, "frames": len(scenes), "ms": ms, "frames_per_s": len(scenes) / ms * 1e3,
                  "humans": eng.results().total_humans, "kernels_ms": kt}))
