"""PF_OPT_PDL masks on C3 Mode U and the C5 step (dev tool): ms per call and
a pose digest (must not change)."""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402

topo = pf.load_topology("coco18")
sp = synth.SynthParams()
work = {"c3u": [synth.crowd_scene(42, s) for s in range(256)],
        "c5": [synth.procedural_scene(5, s, 656, 368, sp) for s in range(8192)]}
masks = [int(m, 0) for m in (sys.argv[1:] or ["64", "65", "66", "68", "72", "80", "96", "127"])]
for name, scenes in work.items():
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    for m in masks:
        eng.ctx.set_option(_native.PF_OPT_PDL, m)
        for _ in range(3):
            eng.parse_tensors(conf, paf, 8, params)
        r = eng.results()
        dg = hashlib.sha1("".join(pf.pose_record(f, r.poses(f), topo) for f in range(0, len(scenes), 11)).encode()).hexdigest()[:10]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            eng.parse_tensors(conf, paf, 8, params)
        e1.record()
        torch.cuda.synchronize()
        eng.results()
        print(f"{name} pdl={m:#05x}: {e0.elapsed_time(e1) / reps:.4f} ms  {dg}", flush=True)
    eng.close()
    del conf, paf
