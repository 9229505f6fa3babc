"""e2e through pf_parse_host with and without PF_OPT_PAF_ZERO_COPY (dev tool):
identical poses required, wall-clock frames/s printed for each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native

topo, conf_h, paf_h = bench.make_inputs(256, 5)
E = int(os.environ.get("E2E_FRAMES", "2048"))
pin_conf = _native.PinnedArray((E,) + conf_h.shape[1:])
pin_paf = _native.PinnedArray((E,) + paf_h.shape[1:])
sel = np.arange(E) % conf_h.shape[0]
pin_conf.array[:] = conf_h[sel]
pin_paf.array[:] = paf_h[sel]
params = pf.ParserParams(upsample=8)
e = pf.PafParser(topo)
ref = None
for rep in range(2):
    for zc in (1, 3):        # 0: copy both, 1: PAF in place, 2: PAF and conf in place, 3: 1 + one-kernel parse
        e.ctx.set_option(_native.PF_OPT_PAF_ZERO_COPY, 1 if zc else 0)
        e.ctx.set_option(_native.PF_OPT_CONF_ZERO_COPY, 1 if zc == 2 else 0)
        e.ctx.set_option(_native.PF_OPT_PARSE_SPLIT, 0 if zc == 3 else 1)
        r = e.parse_arrays(pin_conf.array, pin_paf.array, 8, params)
        recs = [pf.pose_record(f, r.poses(f), topo) for f in range(0, E, 17)]
        if ref is None:
            ref = recs
        assert recs == ref, "zero copy changes the results"
        t0 = time.perf_counter()
        for _ in range(10):
            r = e.parse_arrays(pin_conf.array, pin_paf.array, 8, params)
        dt = time.perf_counter() - t0
        print(f"zero_copy={zc}: {10 * E / dt:.0f} frames/s", flush=True)
