"""A/B of library builds (dev tool): for each .so given, a subprocess loads it
(PF_B200_LIB) and times the C5 step (8192 GPU-rendered frames, Mode U) and
C3 Mode U (256 crowded frames) per kernel (CUDA events, PF_OPT_TIMING),
plus a digest of the poses so the variants can be compared.
  python tools/lib_ab.py scratch_libs/a.so scratch_libs/b.so ..."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import hashlib, json, sys, torch
sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf
from support import synth
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
out = {}
import os
for name in os.environ.get("PF_AB_CFGS", "c5,c3u").split(","):
    if name == "c5":
        scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(8192)]
    else:
        scenes = [synth.crowd_scene(42, s) for s in range(256)]
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    params = pf.ParserParams(upsample=1 if name == "c3r" else 8)
    eng = pf.PafParser(topo)
    for _ in range(3):
        eng.parse_tensors(conf, paf, 8, params)
    r = eng.results()
    h = hashlib.sha1()
    for f in range(0, len(scenes), 7):
        h.update(pf.pose_record(f, r.poses(f), topo).encode())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if name == "c5" else 10
    e0.record()
    for _ in range(reps):
        eng.parse_tensors(conf, paf, 8, params)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    eng.results()
    eng.set_timing(True); eng.kernel_times(reset=True)
    for _ in range(reps):
        eng.parse_tensors(conf, paf, 8, params)
    eng.results()
    kt = eng.kernel_times(reset=True)
    out[name] = {"ms": round(ms, 4), "digest": h.hexdigest()[:12], "humans": r.total_humans,
                 "kernels": {k: round(v[0] / v[1], 4) for k, v in kt.items()}}
    eng.close()
    del conf, paf
print("RESULT " + json.dumps(out))
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, PF_B200_LIB=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    if not line:
        print(lib, "FAILED", p.stderr[-2000:], flush=True)
        continue
    print(lib, line[0][7:], flush=True)
