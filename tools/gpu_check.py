"""Ad-hoc GPU-vs-oracle stage checker (development tool; uses the oracle as checker)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2108_11826_b200 as pf
from support import synth

topo = pf.load_topology("coco18")
sp = synth.SynthParams()

def rec(f, humans):
    return pf.pose_record(f, [pf.HumanPose(keypoints=tuple(None if k is None else pf.Keypoint(*k) for k in kps), score=s, n_parts=n) for s, n, kps in humans], topo)

def check(name, scenes, up, params=None, stride=8):
    params = params or pf.ParserParams(upsample=up)
    params.upsample = up
    conf, paf = synth.render_batch(scenes, topo, sp)
    eng = pf.PafParser(topo, debug=True)
    t0 = time.time()
    got = eng.parse_arrays(conf, paf, stride, params)
    bad = 0
    for f in range(len(scenes)):
        want = oracle.parse(conf[f], paf[f], topo, params, stride) if up == 1 else \
            oracle.parse_upsampled(conf[f], paf[f], topo, params, stride, up)
        gp = eng.peaks(f)
        if gp != want.peaks:
            print(name, f, "PEAKS differ", len(gp), len(want.peaks))
            s1, s2 = set(gp), set(want.peaks)
            print("  gpu-only", sorted(s1 - s2)[:5], " oracle-only", sorted(s2 - s1)[:5])
            bad += 1
            continue
        gc = eng.connections(f)
        if gc != want.connections:
            print(name, f, "CONNS differ", len(gc), len(want.connections))
            for a, b in zip(gc, want.connections):
                if a != b:
                    print("  first diff", a, b); break
            bad += 1
            continue
        a, b = pf.pose_record(f, got.poses(f), topo), rec(f, want.humans)
        if a != b:
            print(name, f, "HUMANS differ\n", a[:300], "\n", b[:300])
            bad += 1
    print(f"{name}: up={up} frames={len(scenes)} mismatching={bad} ({time.time()-t0:.1f}s)", flush=True)
    return bad

total = 0
total += check("procedural-R", [synth.procedural_scene(7, s, 656, 368, sp) for s in range(16)], 1)
total += check("procedural-U", [synth.procedural_scene(7, s, 656, 368, sp) for s in range(8)], 8)
total += check("crowd-R", [synth.crowd_scene(3, s) for s in range(2)], 1)
total += check("crowd-U", [synth.crowd_scene(3, s) for s in range(1)], 8)
print("TOTAL mismatching", total)
total += check("procedural-U-w5", [synth.procedural_scene(9, s, 656, 368, sp) for s in range(4)], 8, pf.ParserParams(nms_window=5))
total += check("procedural-U-w7", [synth.procedural_scene(9, s, 656, 368, sp) for s in range(2)], 8, pf.ParserParams(nms_window=7))
total += check("procedural-U-x4", [synth.procedural_scene(9, s, 656, 368, sp) for s in range(2)], 4)
print("TOTAL2 mismatching", total)
