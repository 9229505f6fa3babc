"""GPU pre-processing and resize kernels vs the reference fixtures and the
oracle (bit-exact fp32 outputs of the fp64 bilinear formula)."""

import collections
import hashlib

import numpy as np
import pytest

import oracle
import paper_2108_11826_b200 as pf
from support import synth
from conftest import golden_path

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def test_preprocess_reference_golden():
    g = np.load(golden_path("preprocess_golden.npz"))
    for idx in range(4):
        img, want = g[f"case{idx}.img"], g[f"case{idx}.out"]
        got = pf.preprocess_batch(img[None], want.shape[1], want.shape[2])[0].cpu().numpy()
        assert np.array_equal(bits(got), bits(want)), idx
    big = np.random.default_rng(360640).integers(0, 256, size=(360, 640, 3), dtype=np.uint8)
    got = pf.preprocess_batch(big[None], 368, 656)[0].cpu().numpy()
    assert hashlib.sha256(got.tobytes()).digest() == bytes(g["big.sha256"])


@pytest.mark.parametrize("shape,out", [((1080, 1920), (1080, 1920)), ((1080, 1920), (368, 656)),
                                       ((360, 640), (368, 656)), ((7, 5), (9, 11)), ((1, 1), (3, 2)),
                                       ((33, 17), (8, 8))])
def test_preprocess_batch_vs_oracle(shape, out):
    rng = np.random.default_rng(sum(shape) + sum(out))
    imgs = rng.integers(0, 256, size=(3,) + shape + (3,), dtype=np.uint8)
    got = pf.preprocess_batch(imgs, *out).cpu().numpy()
    for b in range(3):
        assert np.array_equal(bits(got[b]), bits(oracle.preprocess(imgs[b], *out)))


def test_preprocess_f32_frames_and_operator():
    rng = np.random.default_rng(5)
    img = (rng.integers(0, 256, size=(45, 80, 3)).astype(np.float32) / np.float32(255.0))
    got = pf.preprocess_batch(img[None], 46, 82)[0].cpu().numpy()
    want = np.transpose(oracle.resize_hwc(img, 46, 82), (2, 0, 1))
    assert np.array_equal(bits(got), bits(want))
    frame = pf.Frame(seq_id=4, image=pf.TensorF32.from_array(img), ingest_ns=7)
    out = pf.make_preprocess(82, 46).fn(pf.Packet(4, 7, frame))
    assert out.seq_id == 4 and np.array_equal(bits(out.payload[1].array), bits(want))
    same = pf.make_preprocess(80, 45).fn(pf.Packet(4, 7, frame))       # layout only
    assert np.array_equal(same.payload[1].array, np.transpose(img, (2, 0, 1)))


def test_preprocess_contract():
    with pytest.raises(pf.ContractError):
        pf.preprocess_batch(np.zeros((1, 0, 4, 3), np.uint8), 4, 4)
    with pytest.raises(pf.ContractError):
        pf.preprocess_batch(np.zeros((1, 4, 4, 4), np.uint8), 4, 4)


@pytest.mark.parametrize("src,out", [((46, 82), (368, 656)), ((135, 240), (1080, 1920)),
                                     ((5, 7), (5, 7)), ((9, 4), (2, 3)), ((4, 4), (7, 9))])
def test_resize_planes_vs_oracle(src, out):
    rng = np.random.default_rng(src[0] * 7 + out[1])
    planes = rng.random((3,) + src).astype(np.float32)
    got = pf.resize_planes(planes, *out).cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle.resize_chw(planes, *out)))


def test_bilinear_resize_api():
    rng = np.random.default_rng(2)
    img = rng.random((7, 5, 3)).astype(np.float32)
    got = pf.bilinear_resize(img, 4, 4)
    assert np.array_equal(bits(got), bits(oracle.resize_hwc(img, 4, 4)))
    plane = rng.random((6, 9)).astype(np.float32)
    assert np.array_equal(bits(pf.bilinear_resize(plane, 12, 3)),
                          bits(oracle.resize_chw(plane[None], 12, 3)[0]))
    assert np.array_equal(pf.bilinear_resize(img, 7, 5), img)
    with pytest.raises(pf.ContractError):
        pf.bilinear_resize(np.zeros((0, 4, 3), np.float32), 2, 2)


def test_batched_postprocess_operator(topo):
    sp = synth.SynthParams()
    maps = [synth.render_feature_maps(synth.procedural_scene(12, s, 656, 368, sp), topo, sp) for s in range(5)]
    op = pf.make_batched_postprocess(topo, pf.ParserParams(upsample=8), batch_max=3)
    one = pf.make_postprocess(topo, pf.ParserParams(upsample=8))
    pkts = [pf.Packet(s, 0, (None, m)) for s, m in enumerate(maps)]
    a = [op.fn(p).payload[1] for p in pkts]
    b = [one.fn(p).payload[1] for p in pkts]
    assert [pf.pose_record(i, x, topo) for i, x in enumerate(a)] == \
           [pf.pose_record(i, x, topo) for i, x in enumerate(b)]

    class Sentinel:                              # dataflow.py:26-37 channel sentinels
        def __init__(self, name):
            self.name = name

        def __repr__(self):
            return self.name

    END, NO_ITEM = Sentinel("END_OF_STREAM"), Sentinel("NO_ITEM")

    class Ctx:                                   # the reference runner protocol (dataflow.py:240-280)
        def __init__(self, items):
            self.items = list(items)
            self.out = []
            self.batch_hist = collections.Counter()
            self.busy = 0

        def recv(self, ch):
            return self.items.pop(0) if self.items else END

        def try_recv(self, ch):
            return self.items.pop(0) if self.items else NO_ITEM

        def send(self, ch, pkt):
            self.out.append(pkt)

        def timed(self, fn, *args):
            self.busy += 1
            return fn(*args)

    class Ch:
        closed = False

        def close(self):
            self.closed = True

    ctx, ch = Ctx(pkts), Ch()
    op.runner(ctx, None, ch)
    assert ch.closed and [p.seq_id for p in ctx.out] == list(range(5))
    assert dict(ctx.batch_hist) == {3: 1, 2: 1} and ctx.busy == 2      # batch_max 3: 3 + 2
    with pytest.raises(pf.BackendError):                                 # scheduler.py:96-101
        op.runner(Ctx([pkts[1], pkts[0]]), None, Ch())
    assert [pf.pose_record(p.seq_id, p.payload[1], topo) for p in ctx.out] == \
           [pf.pose_record(i, x, topo) for i, x in enumerate(b)]


def test_multi_device_parser_and_operator(topo):
    """In-process sharding: contiguous shards on several
    contexts (two on this one GPU, plus an empty shard) give the single-context
    results in frame order; the batched operator with ``devices`` likewise."""
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(21, s, 656, 368, sp) for s in range(7)] + [synth.crowd_scene(6, 0)]
    conf, paf = synth.render_batch(scenes, topo, sp)
    params = pf.ParserParams(upsample=8)
    single = pf.PafParser(topo).parse_arrays(conf, paf, 8, params)
    want = [pf.pose_record(f, single.poses(f), topo) for f in range(len(scenes))]
    for devices in ([0, 0], [0, 0, 0]):
        multi = pf.MultiDeviceParser(topo, devices)
        got = multi.parse_arrays(conf, paf, 8, params)
        assert got.total_humans == single.total_humans
        assert [pf.pose_record(f, p, topo) for f, p in enumerate(got.all_poses())] == want
        one = multi.parse_arrays(conf[:1], paf[:1], 8, params)     # shards 1 and 2 empty
        assert pf.pose_record(0, one.poses(0), topo) == want[0]
        multi.close()
    maps = [synth.render_feature_maps(s, topo, sp) for s in scenes[:5]]
    op = pf.make_batched_postprocess(topo, params, batch_max=4, devices=[0, 0])
    pkts = [pf.Packet(s, 0, (None, m)) for s, m in enumerate(maps)]
    got = [pf.pose_record(p.seq_id, op.fn(p).payload[1], topo) for p in pkts]
    assert got == want[:5]


def test_gpu_renderer_matches_host(topo):
    """pf_render_maps (GPU-resident producer) against the host renderer on
    procedural and crowded scenes: bit-identical except where fp64 exp()
    rounds differently from numpy's (then within 1 fp32 ulp), and the parse
    of both renderings gives the same records."""
    sp = synth.SynthParams()
    scenes = [synth.procedural_scene(3, s, 656, 368, sp) for s in range(6)] + [synth.crowd_scene(2, 0)]
    conf_h, paf_h = synth.render_batch(scenes, topo, sp)
    conf_g, paf_g = synth.render_batch_gpu(scenes, topo, sp)
    conf_g, paf_g = conf_g.cpu().numpy(), paf_g.cpu().numpy()
    assert np.array_equal(paf_g, paf_h)                      # sqrt / division only: exact
    diff = conf_g != conf_h
    assert diff.mean() < 1e-3
    assert np.all(np.abs(conf_g[diff].view(np.int32) - conf_h[diff].view(np.int32)) <= 1)
    e = pf.PafParser(topo)
    params = pf.ParserParams(upsample=8)
    a = e.parse_arrays(conf_h, paf_h, 8, params)
    ra = [pf.pose_record(f, a.poses(f), topo) for f in range(len(scenes))]
    b = e.parse_arrays(np.ascontiguousarray(conf_g), np.ascontiguousarray(paf_g), 8, params)
    rb = [pf.pose_record(f, b.poses(f), topo) for f in range(len(scenes))]
    e.close()
    if not diff.any():
        assert ra == rb
