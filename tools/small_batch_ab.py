"""Small batches (C2: 64 frames, 1-5 people, Mode U; plus 32 and 128) under the
split / one-kernel path options (dev tool): us per call (CUDA events) and a
pose digest per setting."""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402

topo = pf.load_topology("coco18")
sp = synth.SynthParams()
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,64,128").split(",")]:
    scenes = [synth.procedural_scene(7, s, 656, 368, sp) for s in range(n)]
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    params = pf.ParserParams(upsample=8)
    for cs, ps in (((1, 1), (0, 1)) if len(sys.argv) > 2 else ((1, 1), (0, 1), (1, 0), (0, 0))):
        eng = pf.PafParser(topo)
        eng.ctx.set_option(_native.PF_OPT_CORNER_SPLIT, cs)
        eng.ctx.set_option(_native.PF_OPT_PARSE_SPLIT, ps)
        for _ in range(10):
            eng.parse_tensors(conf, paf, 8, params)
        r = eng.results()
        dg = hashlib.sha1("".join(pf.pose_record(f, r.poses(f), topo) for f in range(n)).encode()).hexdigest()[:10]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            eng.parse_tensors(conf, paf, 8, params)
        e1.record()
        torch.cuda.synchronize()
        eng.results()
        us = e0.elapsed_time(e1) / 200 * 1e3
        print(f"B{n} corner_split={cs} parse_split={ps}: {us:.1f} us/call  {n / us * 1e3:.0f}k frames/s  {dg}", flush=True)
        eng.close()
