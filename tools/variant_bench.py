"""Time the Mode U NMS kernel variants on the bench workload (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native
import bench

topo, conf_h, paf_h = bench.make_inputs(256, 5)
F = 8192
idx = torch.arange(F) % conf_h.shape[0]
conf = torch.from_numpy(conf_h).cuda()[idx.cuda()].contiguous()
paf = torch.from_numpy(paf_h).cuda()[idx.cuda()].contiguous()
params = pf.ParserParams(upsample=8)
e = pf.PafParser(topo)
ref = None
for variant in [int(v) for v in os.environ.get("VARIANTS", "2,4").split(",")]:
    e.ctx.set_option(_native.PF_OPT_WIN_VARIANT, variant)
    for _ in range(2):
        e.parse_tensors(conf, paf, 8, params)
    r = e.results()
    recs = [r.poses(f) for f in range(0, F, 37)]
    if ref is None: ref = recs
    assert recs == ref, f"variant {variant} differs"
    e.set_timing(True); e.kernel_times(reset=True)
    for _ in range(10):
        e.parse_tensors(conf, paf, 8, params)
    kt = e.kernel_times(reset=True); e.set_timing(False)
    print(variant, {k: round(v[0] / v[1], 3) for k, v in kt.items()}, flush=True)
