"""Per-phase cycle breakdown of k_nms_up_corner (dev tool; needs a
-DPF_CORNER_PROF build loaded through PF_B200_LIB)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native

topo, conf_h, paf_h = bench.make_inputs(256, 5)
F = 8192
idx = torch.arange(F) % conf_h.shape[0]
conf = torch.from_numpy(conf_h).cuda()[idx.cuda()].contiguous()
paf = torch.from_numpy(paf_h).cuda()[idx.cuda()].contiguous()
params = pf.ParserParams(upsample=8)
e = pf.PafParser(topo)
lib = _native.load_library()
buf = (ctypes.c_ulonglong * 16)()
e.parse_tensors(conf, paf, 8, params)
lib.pf_corner_prof_read(buf, 1)
for _ in range(5):
    e.parse_tensors(conf, paf, 8, params)
lib.pf_corner_prof_read(buf, 1)
planes = buf[12]
names = ["A hot words", "sync1", "B hot list", "sync2", "C1b classify", "sync3", "C2 exact", "tail (sync4, redo, sync5, store, TMA issue)",
         "C1a prune", "sync C1", "TMA wait", "-"]
tot = sum(buf[k] for k in range(12))
for k in range(11):
    print(f"{names[k]:28s} {buf[k] / planes:9.0f} cycles/plane  {100 * buf[k] / tot:5.1f}%")
print("total cycles per plane per CTA", tot / planes)
print("per plane: hot cells %.1f, chain survivors %.1f, candidates %.1f" % (buf[13] / planes, buf[14] / planes, buf[15] / planes))
