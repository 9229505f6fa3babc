import sys, time, torch
sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native
from support import synth
topo = pf.load_topology("coco18"); sp = synth.SynthParams()
for F, ov in ((64, 0), (8192, 0), (8192, 1024)):
    scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(F)]
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    eng.ctx.set_option(_native.PF_OPT_OVERLAP, ov)
    for _ in range(3): eng.parse_tensors(conf, paf, 8, params)
    eng.results(); torch.cuda.synchronize()
    # host enqueue time: GPU kept busy by a long sleep kernel first
    torch.cuda._sleep(int(2e9))
    t0 = time.perf_counter()
    for _ in range(10): eng.parse_tensors(conf, paf, 8, params)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(F, ov, "host us/call", round((t1 - t0) / 10 * 1e6, 1), flush=True)
    eng.results()
