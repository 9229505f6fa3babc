"""Minimal C5 driver for ncu captures: 8192 GPU-rendered frames, Mode U,
`steps` parse calls (argv[1], default 3) on device-resident maps."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from support import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(8192)]
conf, paf = synth.render_batch_gpu(scenes, topo, sp)
eng = pf.PafParser(topo)
for kv in filter(None, os.environ.get("PF_OPTS", "").split(",")):   # e.g. PF_OPTS=14=0
    k, v = kv.split("=")
    eng.ctx.set_option(int(k), int(v))
params = pf.ParserParams(upsample=8)
for _ in range(steps):
    eng.parse_tensors(conf, paf, 8, params)
print("humans", eng.results().total_humans)
