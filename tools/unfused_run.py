"""Run the materialised Mode U path (k_resize_planes -> k_nms_plane) on the
bench workload, for ncu captures of the HBM-streaming kernels (dev tool).
Prints the frames each launch covers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2108_11826_b200 as pf

topo, conf_h, paf_h = bench.make_inputs(64, 5)
U = 256
idx = torch.arange(U) % conf_h.shape[0]
conf = torch.from_numpy(conf_h).cuda()[idx.cuda()].contiguous()
paf = torch.from_numpy(paf_h).cuda()[idx.cuda()].contiguous()
e = pf.PafParser(topo)
e.set_materialise(True)
e.set_timing(True)
e.parse_tensors(conf, paf, 8, pf.ParserParams(upsample=8))
kt = e.kernel_times(reset=True)
print({k: (U / n) for k, (ms, n) in kt.items()})
