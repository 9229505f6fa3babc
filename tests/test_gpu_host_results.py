"""parse_arrays results land in caller-owned pinned blocks (pf_get_results_into):
the same poses as the context-buffer path, valid after later calls, views
keep their block alive, and the block grows to the call's need."""
import numpy as np
import pytest

import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native
from support import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def frames():
    topo = pf.load_topology("coco18")
    sp = synth.SynthParams()
    a = synth.render_batch_gpu([synth.procedural_scene(3, s, 656, 368, sp) for s in range(200)], topo, sp)
    b = synth.render_batch_gpu([synth.procedural_scene(4, s, 656, 368, sp) for s in range(200)], topo, sp)
    return topo, [(c.cpu().numpy(), p.cpu().numpy()) for c, p in (a, b)]


def test_same_poses_as_context_buffers_and_stable_across_calls(frames):
    topo, ((ca, pa), (cb, pb)) = frames
    params = pf.ParserParams(upsample=8)
    eng = pf.PafParser(topo)
    r1 = eng.parse_arrays(ca, pa, 8, params)
    want1 = r1.records(topo)
    # the context-buffer path on the same maps
    import torch
    eng.parse_tensors(torch.from_numpy(ca).cuda(), torch.from_numpy(pa).cuda(), 8, params)
    assert eng.results().records(topo) == want1
    kx = r1.kp_x                                   # a view into r1's block
    kx_copy = kx.copy()
    del r1
    for _ in range(3):                             # later calls reuse freed blocks, never a live one
        r2 = eng.parse_arrays(cb, pb, 8, params)
    assert np.array_equal(kx, kx_copy)
    r3 = eng.parse_arrays(ca, pa, 8, params)
    assert r3.records(topo) == want1
    assert r2.records(topo) != want1
    eng.close()


def test_block_grows_to_the_call(frames):
    topo, _ = frames
    crowd = synth.render_batch_gpu([synth.crowd_scene(5, s) for s in range(6)], topo, synth.SynthParams())
    conf, paf = (t.cpu().numpy() for t in crowd)
    eng = pf.PafParser(topo)
    eng._host_cap = 1                               # force the grow-and-retry path
    r = eng.parse_arrays(conf, paf, 8, pf.ParserParams())
    assert r.total_humans > 24 and eng._host_cap >= r.total_humans
    eng2 = pf.PafParser(topo)
    import torch
    eng2.parse_tensors(torch.from_numpy(conf).cuda(), torch.from_numpy(paf).cuda(), 8, pf.ParserParams())
    assert r.records(topo) == eng2.results().records(topo)
    eng.close()
    eng2.close()


def test_results_into_reports_the_need(frames):
    topo, ((ca, pa), _) = frames
    import ctypes
    eng = pf.PafParser(topo)
    p = pf.ParserParams().to_native()
    eng.ctx.check(eng.ctx.lib.pf_parse_host(eng.ctx.handle, ca.ctypes.data, pa.ctypes.data, 16, 46, 82, 8,
                                            ctypes.byref(p), None))
    n, total = ctypes.c_int32(), ctypes.c_int32()
    dst = _native.PfHostOut(0, None, None, None, None, None, None, None, None)
    rc = eng.ctx.lib.pf_get_results_into(eng.ctx.handle, ctypes.byref(dst), ctypes.byref(n), ctypes.byref(total))
    assert rc == _native.PF_ERR_CAPACITY and n.value == 16 and total.value > 0
    eng.close()
