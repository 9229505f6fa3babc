"""A/B a pf_set_option knob on the bench workload (dev tool): identical poses
required, per-kernel CUDA-event times printed for each setting.

  OPT=6 VALUES=0,1 python tools/ab_options.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2108_11826_b200 as pf

opt = int(os.environ.get("OPT", "6"))
values = [int(v) for v in os.environ.get("VALUES", "0,1").split(",")]
topo, conf_h, paf_h = bench.make_inputs(int(os.environ.get("DISTINCT", "256")), 5)
F = 8192
idx = torch.arange(F) % conf_h.shape[0]
conf = torch.from_numpy(conf_h).cuda()[idx.cuda()].contiguous()
paf = torch.from_numpy(paf_h).cuda()[idx.cuda()].contiguous()
params = pf.ParserParams(upsample=int(os.environ.get("UP", "8")))
caps = dict(kv.split("=") for kv in os.environ["CAPS"].split(",")) if os.environ.get("CAPS") else {}
e = pf.PafParser(topo, caps={k: int(v) for k, v in caps.items()})
ref = None
for rep in range(2):
    for v in values:
        e.ctx.set_option(opt, v)
        for _ in range(2):
            e.parse_tensors(conf, paf, 8, params)
        r = e.results()
        recs = [pf.pose_record(f, r.poses(f), topo) for f in range(0, F, 31)]
        if ref is None:
            ref = recs
        assert recs == ref, f"option {opt}={v} changes the results"
        e.set_timing(True)
        e.kernel_times(reset=True)
        for _ in range(20):
            e.parse_tensors(conf, paf, 8, params)
        kt = e.kernel_times(reset=True)
        e.set_timing(False)
        print(f"opt {opt}={v}", {k: round(t[0] / t[1], 4) for k, t in kt.items()}, flush=True)
