"""Single-frame (C1) and small-batch call latency per library build (dev
tool): device-resident maps, CUDA events around 300 parse_tensors calls, per
kernel times from a timing pass.  python tools/c1_latency.py a.so b.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf
from support import synth
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
out = {}
for n in (1, 4, 16):
    scenes = [synth.procedural_scene(0, 1 + s, 656, 368, sp) for s in range(n)]
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    for up in (1, 8):
        params = pf.ParserParams(upsample=up)
        eng = pf.PafParser(topo)
        for _ in range(20):
            eng.parse_tensors(conf, paf, 8, params)
        rec = [pf.pose_record(f, eng.results().poses(f), topo) for f in range(n)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(300):
            eng.parse_tensors(conf, paf, 8, params)
        e1.record(); torch.cuda.synchronize()
        eng.results()
        eng.set_timing(True); eng.kernel_times(reset=True)
        for _ in range(50):
            eng.parse_tensors(conf, paf, 8, params)
        eng.results()
        kt = eng.kernel_times(reset=True)
        out[f"B{n} up{up}"] = {"us_per_call": round(e0.elapsed_time(e1) / 300 * 1e3, 1),
                               "kernels_us": {k: round(v[0] / v[1] * 1e3, 1) for k, v in kt.items()},
                               "digest": __import__("hashlib").sha1("".join(rec).encode()).hexdigest()[:10]}
        eng.close()
print("RESULT " + json.dumps(out))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, PF_B200_LIB=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    print(lib, line[0][7:] if line else "FAILED " + p.stderr[-1500:], flush=True)
