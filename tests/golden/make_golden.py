#!/usr/bin/env python
"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only where the reference is importable (this build container:
PYTHONPATH=/root/reference/pkg/src); the GPU box has no /root/reference, so
the outputs are committed.  Every expected value below is produced by calling
the reference's own functions (poseflow, pure Python/numpy):

  nms_golden.npz       paf.nms_peaks            test_paf.py:56-97 recipes + threshold edges
  score_golden.npz     paf.score_limb           test_paf.py:124-153 recipes
  greedy_golden.json   paf._greedy_select       test_paf.py:189-204 recipe
  frames_golden.npz    synth.render_feature_maps + paf.parse (Mode R) and
                       operators.bilinear_resize x8 + paf.parse(stride=1) (Mode U),
                       with paf.nms_peaks / connect_limbs stage outputs
  preprocess_golden.npz  operators.make_preprocess (+ formats.read_ppm's u8/255)
  records_golden.json  operators.pose_record known answers

Usage:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("POSEFLOW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import poseflow  # noqa: E402  (the reference)
from poseflow import formats, operators  # noqa: E402
from poseflow.paf import ParserParams, Peak, _greedy_select, connect_limbs, nms_peaks, parse, score_limb  # noqa: E402
from poseflow.synth import GroundTruthHuman, GroundTruthScene, SynthParams, procedural_scene, render_feature_maps  # noqa: E402
from poseflow.topology import load_topology  # noqa: E402
from poseflow.types import FeatureMaps, TensorF32  # noqa: E402
from poseflow import oracles  # noqa: E402

import support.synth as our_synth  # noqa: E402  (crowd keypoints only: pure numpy)

TOPO = load_topology("coco18")
P = ParserParams()


def peaks_arrays(conf, params, K=None):
    """Reference peaks of every part channel, in id order."""
    K = conf.shape[0] - 1 if K is None else K
    out, nid = [], 0
    by_part = []
    for part in range(K):
        ps = nms_peaks(conf[part], params, part=part, id_base=nid)
        nid += len(ps)
        by_part.append(ps)
        out += [(p.part, p.cell[0], p.cell[1], p.score, p.id) for p in ps]
    return out, by_part


def gen_nms():
    maps, counts, cells, scores, windows, thrs = [], [], [], [], [], []

    def add(conf, params):
        ps = nms_peaks(conf, params)
        maps.append(conf.astype(np.float32))
        counts.append(len(ps))
        cells.extend(p.cell for p in ps)
        scores.extend(p.score for p in ps)
        windows.append(params.nms_window)
        thrs.append(params.conf_threshold)

    rng = np.random.default_rng(123)                 # test_paf.py:56-67
    for case in range(200):
        conf = rng.random((16, 16)).astype(np.float32)
        if case % 4 == 0:
            conf = np.round(conf * 8) / 8
        add(conf.astype(np.float32), P)
    rng = np.random.default_rng(7)                   # test_paf.py:90-97 (padded to 16x16 below)
    w5 = []
    for _ in range(20):
        w5.append(rng.random((10, 10)).astype(np.float32))
    # threshold edges: fp32 compare (numpy NEP 50) with thresholds that round
    # up (0.1) and down (0.7) in float32, and NaN / -0.0 cells
    rng = np.random.default_rng(99)
    edge = []
    for thr in (0.1, 0.7, 0.3, 0.0, 1.0):
        conf = rng.random((16, 16)).astype(np.float32) * 0.5
        conf[3, 3] = np.float32(thr)
        conf[8, 8] = np.nextafter(np.float32(thr), np.float32(0))
        conf[12, 4] = np.nextafter(np.float32(thr), np.float32(2))
        conf[5, 12] = np.float32(np.nan)
        conf[14, 14] = np.float32(-0.0)
        edge.append((conf, thr))
    for conf, thr in edge:
        add(conf, ParserParams(conf_threshold=thr))
    small = {"maps": np.stack(maps), "counts": np.array(counts), "cells": np.array(cells, dtype=np.int32).reshape(-1, 2),
             "scores": np.array(scores, dtype=np.float64), "windows": np.array(windows), "thresholds": np.array(thrs)}
    # window-5 set kept separately (10x10 maps)
    w5c, w5cells, w5s = [], [], []
    for conf in w5:
        ps = nms_peaks(conf, ParserParams(nms_window=5))
        w5c.append(len(ps))
        w5cells.extend(p.cell for p in ps)
        w5s.extend(p.score for p in ps)
    np.savez_compressed(os.path.join(HERE, "nms_golden.npz"), **small,
                        w5_maps=np.stack(w5), w5_counts=np.array(w5c),
                        w5_cells=np.array(w5cells, dtype=np.int32).reshape(-1, 2),
                        w5_scores=np.array(w5s, dtype=np.float64))


def gen_score():
    rows = []
    fields = []
    rng = np.random.default_rng(5)                   # test_paf.py:124-138
    for _ in range(100):
        paf = np.empty((38, 12, 12), dtype=np.float32)
        paf[:] = rng.uniform(-1, 1, size=(38, 1, 1))
        ca = (int(rng.integers(12)), int(rng.integers(12)))
        cb = (int(rng.integers(12)), int(rng.integers(12)))
        limb = int(rng.integers(19))
        pa, pb = Peak(1, ca, 1.0, 0), Peak(2, cb, 1.0, 1)
        s, g = score_limb(paf, TOPO, limb, pa, pb, P)
        cx, cy = TOPO.paf_channels[limb]
        fields.append(np.pad(np.stack([paf[cx], paf[cy]]), ((0, 0), (0, 8), (0, 8))))
        rows.append((12, limb, ca[0], ca[1], cb[0], cb[1], s, g))
    rng = np.random.default_rng(6)                   # test_paf.py:140-153
    for _ in range(100):
        paf = oracles.smooth_random_field((38, 20, 20), rng).astype(np.float32)
        ca = (int(rng.integers(20)), int(rng.integers(20)))
        cb = (int(rng.integers(20)), int(rng.integers(20)))
        limb = int(rng.integers(19))
        pa, pb = Peak(1, ca, 1.0, 0), Peak(2, cb, 1.0, 1)
        s, g = score_limb(paf, TOPO, limb, pa, pb, P)
        cx, cy = TOPO.paf_channels[limb]
        fields.append(np.stack([paf[cx], paf[cy]]))
        rows.append((20, limb, ca[0], ca[1], cb[0], cb[1], s, g))
    meta = np.array([r[:6] for r in rows], dtype=np.int32)
    vals = np.array([r[6:] for r in rows], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "score_golden.npz"), fields=np.stack(fields), meta=meta, vals=vals)


def gen_greedy():
    rng = np.random.default_rng(17)                  # test_paf.py:189-204
    cases = []
    for _ in range(200):
        n_a, n_b = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        cands = []
        for i in range(n_a):
            for j in range(n_b):
                score = float(rng.choice([0.2, 0.4, 0.6, 0.8, rng.random()]))
                cands.append((Peak(0, (0, i), 1.0, i), Peak(1, (5, j), 1.0, 100 + j), score, 1.0))
        got = _greedy_select(cands)
        cases.append({"candidates": [[a.id, b.id, s] for a, b, s, _ in cands],
                      "accepted": [[a.id, b.id, s] for a, b, s, _ in got]})
    with open(os.path.join(HERE, "greedy_golden.json"), "w") as f:
        json.dump(cases, f)


def upsampled(maps, up):
    c = maps.conf.array
    p = maps.paf.array
    h, w = c.shape[1:]
    cu = np.stack([operators.bilinear_resize(ch, h * up, w * up) for ch in c])
    pu = np.stack([operators.bilinear_resize(ch, h * up, w * up) for ch in p])
    return FeatureMaps(TensorF32.from_array(cu), TensorF32.from_array(pu), maps.stride // up, maps.frame_ref)


def stage_outputs(maps):
    peaks, by_part = peaks_arrays(maps.conf.array, P)
    conns = connect_limbs(by_part, maps.paf.array, TOPO, P)
    poses = parse(maps, TOPO, P)
    rec = operators.pose_record(0, poses, TOPO)
    return (np.array([p[:3] for p in peaks], dtype=np.int32).reshape(-1, 3),
            np.array([p[3] for p in peaks], dtype=np.float64),
            np.array([(c.limb, c.peak_a, c.peak_b) for c in conns], dtype=np.int32).reshape(-1, 3),
            np.array([(c.score, c.good_fraction) for c in conns], dtype=np.float64).reshape(-1, 2),
            rec)


def gen_frames():
    sp = SynthParams()
    scenes = [("C1", procedural_scene(0, 1, 656, 368, sp))]
    scenes += [(f"C2_{s}", procedural_scene(7, s, 656, 368, sp)) for s in range(6)]
    for fr in range(2):
        cs = our_synth.crowd_scene(3, fr)
        scenes.append((f"C3_{fr}", GroundTruthScene(
            humans=tuple(GroundTruthHuman(h.keypoints) for h in cs.humans), input_w=656, input_h=368)))
    up_names = {"C1", "C2_0", "C2_1", "C3_0"}
    out = {}
    names, records_r, records_u = [], {}, {}
    for name, scene in scenes:
        maps = render_feature_maps(scene, TOPO, sp)
        names.append(name)
        out[f"{name}.conf"] = maps.conf.array
        out[f"{name}.paf"] = maps.paf.array
        out[f"{name}.kps"] = np.array([[kp if kp is not None else (np.nan, np.nan) for kp in h.keypoints]
                                       for h in scene.humans], dtype=np.float64).reshape(-1, 18, 2)
        pk, ps, cn, cs_, rec = stage_outputs(maps)
        out[f"{name}.R.peaks"], out[f"{name}.R.peak_scores"] = pk, ps
        out[f"{name}.R.conns"], out[f"{name}.R.conn_vals"] = cn, cs_
        records_r[name] = rec
        if name in up_names:
            pk, ps, cn, cs_, rec = stage_outputs(upsampled(maps, 8))
            out[f"{name}.U.peaks"], out[f"{name}.U.peak_scores"] = pk, ps
            out[f"{name}.U.conns"], out[f"{name}.U.conn_vals"] = cn, cs_
            records_u[name] = rec
        print(name, len(scene.humans), "humans", flush=True)
    np.savez_compressed(os.path.join(HERE, "frames_golden.npz"), **out)
    with open(os.path.join(HERE, "frames_records.json"), "w") as f:
        json.dump({"names": names, "R": records_r, "U": records_u, "up": 8}, f, indent=0)
    # procedural keypoints for the synth-port check (scenes only; cheap)
    kp = {}
    for seed, seq in [(0, 1), (7, 0), (7, 5), (31, 3), (42, 10), (5, 100)]:
        sc = procedural_scene(seed, seq, 656, 368, sp)
        kp[f"{seed}_{seq}"] = [[list(k) for k in h.keypoints] for h in sc.humans]
    with open(os.path.join(HERE, "scenes_golden.json"), "w") as f:
        json.dump(kp, f)


def gen_preprocess():
    out = {}
    rng = np.random.default_rng(2024)
    cases = [((45, 80), (46, 82)), ((37, 61), (50, 70)), ((12, 20), (12, 20)), ((9, 7), (4, 5))]
    for idx, ((h, w), (oh, ow)) in enumerate(cases):
        img = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        want = prep(img, ow, oh)
        out[f"case{idx}.img"] = img
        out[f"case{idx}.out"] = want
    # full-size case: seeded input, only the digest of the expected output is stored
    big = np.random.default_rng(360640).integers(0, 256, size=(360, 640, 3), dtype=np.uint8)
    want = prep(big, 656, 368)
    out["big.sha256"] = np.frombuffer(hashlib.sha256(want.tobytes()).digest(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "preprocess_golden.npz"), **out)


def prep(img_u8, out_w, out_h):
    """Reference path: write a PPM, read it back (formats.read_ppm), preprocess."""
    buf = io.BytesIO()
    h, w, _ = img_u8.shape
    buf.write(f"P6\n{w} {h}\n255\n".encode())
    buf.write(img_u8.tobytes())
    buf.seek(0)
    image = formats.read_ppm(buf)
    frame = poseflow.Frame(seq_id=0, image=image, ingest_ns=0)
    pkt = operators.make_preprocess(out_w, out_h).fn(poseflow.Packet(0, 0, frame))
    return pkt.payload[1].array


def gen_records():
    from poseflow.types import HumanPose, Keypoint

    kps = [None] * 18
    kps[0] = Keypoint(x=1.5, y=2.5, score=0.75)
    kps[2] = Keypoint(x=3.0, y=4.0, score=0.5)
    pose = HumanPose(keypoints=tuple(kps), score=1.25, n_parts=2)
    kps2 = [None] * 18
    kps2[5] = Keypoint(x=655.0, y=0.0, score=float(np.float32(0.1)))
    pose2 = HumanPose(keypoints=tuple(kps2), score=0.30000000000000004, n_parts=1)
    recs = {"one": operators.pose_record(7, [pose], TOPO),
            "two": operators.pose_record(8, [pose, pose2], TOPO),
            "empty": operators.pose_record(3, [], TOPO)}
    with open(os.path.join(HERE, "records_golden.json"), "w") as f:
        json.dump(recs, f, indent=0)


if __name__ == "__main__":
    meta = {"numpy": np.__version__, "python": sys.version.split()[0], "reference": REF}
    with open(os.path.join(HERE, "GOLDEN_META.json"), "w") as f:
        json.dump(meta, f, indent=1)
    gen_nms()
    gen_score()
    gen_greedy()
    gen_records()
    gen_preprocess()
    gen_frames()
    print("golden fixtures written to", HERE)
