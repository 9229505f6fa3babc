"""Randomised parity sweep (dev tool, GPU): random scenes (procedural and
crowded), random ParserParams, random batch sizes across the path
boundaries, device and host entry points; sampled frames vs the oracle,
pose_record bytes.  python tools/fuzz_parity.py [seconds] [seed]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2108_11826_b200 as pf  # noqa: E402
from conftest import record_of  # noqa: E402
from support import synth  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
t0 = time.time()
cases = frames_checked = 0
fails = []
while time.time() - t0 < budget:
    n = int(rng.choice([1, 3, 17, 31, 64, 148, 149, 200, 256, 300, 620]))
    seed = int(rng.integers(1 << 30))
    scenes = []
    for s in range(n):
        if rng.random() < 0.08:
            scenes.append(synth.crowd_scene(seed, s))
        else:
            scenes.append(synth.procedural_scene(seed, s, 656, 368, sp))
    conf, paf = synth.render_batch_gpu(scenes, topo, sp)
    kw = dict(conf_threshold=float(rng.choice([0.05, 0.1, 0.2, 0.35])),
              nms_window=int(rng.choice([3, 3, 3, 5])),
              n_samples=int(rng.choice([5, 10, 10, 15])),
              sample_dot_threshold=float(rng.choice([0.0, 0.05, 0.2])),
              good_fraction_min=float(rng.choice([0.5, 0.8, 0.9])),
              min_parts=int(rng.choice([1, 3, 4, 6])),
              min_human_score=float(rng.choice([0.0, 0.2, 0.4])),
              upsample=int(rng.choice([1, 8, 8, 2, 4])))
    params = pf.ParserParams(**kw)
    eng = pf.PafParser(topo)
    host = rng.random() < 0.3
    if host:
        res = eng.parse_arrays(conf.cpu().numpy(), paf.cpu().numpy(), 8, params)
    else:
        eng.parse_tensors(conf, paf, 8, params)
        res = eng.results()
    eng.close()
    c, p = conf.cpu().numpy(), paf.cpu().numpy()
    idx = sorted(set(rng.choice(n, size=min(n, 4), replace=False).tolist() + [n - 1]))
    for f in idx:
        if params.upsample == 1:
            want = oracle.parse(c[f], p[f], topo, params, 8)
        else:
            want = oracle.parse_upsampled(c[f], p[f], topo, params, 8, params.upsample)
        got = pf.pose_record(f, res.poses(f), topo)
        if got != record_of(want.humans, topo, f):
            fails.append((n, seed, kw, host, f))
            print("MISMATCH", n, seed, kw, host, f, flush=True)
        frames_checked += 1
    cases += 1
print(f"cases {cases} frames checked {frames_checked} mismatches {len(fails)}", flush=True)
sys.exit(1 if fails else 0)
