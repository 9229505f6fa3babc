"""BASELINE.json configurations at full size on the GPU.

Exact comparison with the oracle wherever the oracle finishes in seconds,
size-independent properties (determinism, batch / chunk invariance, shard
invariance) for the 8192-frame stream."""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from support import synth
from conftest import record_of

pytestmark = pytest.mark.gpu
SP = synth.SynthParams()
THREADS = max(1, min(32, os.cpu_count() or 1))


def oracle_records(conf, paf, topo, params, stride=8, up=1, idx=None):
    idx = range(conf.shape[0]) if idx is None else idx

    def one(f):
        if up == 1:
            r = oracle.parse(conf[f], paf[f], topo, params, stride)
        else:
            r = oracle.parse_upsampled(conf[f], paf[f], topo, params, stride, up)
        return record_of(r.humans, topo, f)

    with ThreadPoolExecutor(THREADS) as ex:
        return list(ex.map(one, idx))


def gpu_records(res, topo, idx=None):
    idx = range(res.n_frames) if idx is None else idx
    return [pf.pose_record(f, res.poses(f), topo) for f in idx]


def test_c1_single_frame_modes(topo):
    conf, paf = synth.render_batch([synth.procedural_scene(0, 1, 656, 368, SP)], topo, SP)
    e = pf.PafParser(topo)
    for up in (1, 8):
        params = pf.ParserParams(upsample=up)
        assert gpu_records(e.parse_arrays(conf, paf, 8, params), topo) == \
            oracle_records(conf, paf, topo, params, up=up)
    e.close()


def test_c2_batch64_mode_u(topo):
    scenes = [synth.procedural_scene(7, s, 656, 368, SP) for s in range(64)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    params = pf.ParserParams(upsample=8)
    e = pf.PafParser(topo)
    got = gpu_records(e.parse_arrays(conf, paf, 8, params), topo)
    assert got == oracle_records(conf, paf, topo, params, up=8)
    e.close()


def test_c3_crowded_batch256(topo):
    scenes = [synth.crowd_scene(42, s) for s in range(256)]
    conf, paf = synth.render_batch(scenes, topo, SP)
    e = pf.PafParser(topo)
    params = pf.ParserParams()
    assert gpu_records(e.parse_arrays(conf, paf, 8, params), topo) == oracle_records(conf, paf, topo, params)
    pu = pf.ParserParams(upsample=8)
    got = e.parse_arrays(conf[:4], paf[:4], 8, pu)
    assert gpu_records(got, topo) == oracle_records(conf[:4], paf[:4], topo, pu, up=8)
    e.close()


@pytest.mark.parametrize("people", [6, 40])
def test_c4_highres_1080p(topo, people):
    sp = synth.SynthParams()
    if people == 40:
        scene = synth.crowd_scene(9, 0, 1920, 1080, 40, (150.0, 300.0))
    else:
        scene = synth.GroundTruthScene(synth.crowd_scene(9, 1, 1920, 1080, 6, (300.0, 500.0)).humans, 1920, 1080)
    conf, paf = synth.render_batch([scene], topo, sp)
    assert conf.shape == (1, 19, 135, 240)
    e = pf.PafParser(topo)
    for up in (1, 8):
        params = pf.ParserParams(upsample=up)
        assert gpu_records(e.parse_arrays(conf, paf, 8, params), topo) == \
            oracle_records(conf, paf, topo, params, up=up)
    e.close()


def test_c4_preprocess_1080p():
    rng = np.random.default_rng(1080)
    frames = rng.integers(0, 256, size=(2, 1080, 1920, 3), dtype=np.uint8)
    got = pf.preprocess_batch(frames, 1080, 1920).cpu().numpy()
    for b in range(2):
        assert np.array_equal(got[b], oracle.preprocess(frames[b], 1080, 1920))
    got = pf.preprocess_batch(frames, 368, 656).cpu().numpy()
    assert np.array_equal(got[1], oracle.preprocess(frames[1], 368, 656))


def test_c5_stream_8192_properties(topo):
    """8192-frame stream: one call == four chunked calls == per-shard calls,
    repeatable, and an oracle spot check on 48 frames."""
    import torch

    scenes = [synth.procedural_scene(5, s, 656, 368, SP) for s in range(128)]
    conf_h, paf_h = synth.render_batch(scenes, topo, SP)
    idx = np.arange(8192) % 128
    conf = torch.from_numpy(conf_h).cuda()[torch.from_numpy(idx).cuda()].contiguous()
    paf = torch.from_numpy(paf_h).cuda()[torch.from_numpy(idx).cuda()].contiguous()
    params = pf.ParserParams(upsample=8)
    e = pf.PafParser(topo)
    e.parse_tensors(conf, paf, 8, params)
    full = e.results()
    e.parse_tensors(conf, paf, 8, params)
    again = e.results()
    assert np.array_equal(full.frame_count, again.frame_count)
    whole = [full.poses(f) for f in range(8192)]
    assert whole == [again.poses(f) for f in range(8192)]     # pool order may differ, frames may not
    for lo in range(0, 8192, 2048):
        e.parse_tensors(conf[lo:lo + 2048], paf[lo:lo + 2048], 8, params)
        part = e.results()
        for f in range(0, 2048, 97):
            assert part.poses(f) == whole[lo + f]
    # frames with the same content give the same poses wherever they sit in the stream
    for f in range(128, 8192, 311):
        assert whole[f] == whole[f % 128]
    spot = list(range(0, 128, 3))[:48]
    want = oracle_records(conf_h, paf_h, topo, params, up=8, idx=spot)
    assert [pf.pose_record(f, whole[f], topo) for f in spot] == want
    assert sum(full.frame_count) == full.total_humans > 8192
    e.close()
