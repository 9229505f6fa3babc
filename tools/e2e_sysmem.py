"""One pf_parse_host call on the bench's e2e workload (for an ncu capture of the
PCIe traffic of the zero-copy PAF reads; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_2108_11826_b200 as pf
from paper_2108_11826_b200 import _native

topo, conf_h, paf_h = bench.make_inputs(256, 5)
E = 2048
pin_conf = _native.PinnedArray((E,) + conf_h.shape[1:])
pin_paf = _native.PinnedArray((E,) + paf_h.shape[1:])
sel = np.arange(E) % conf_h.shape[0]
pin_conf.array[:] = conf_h[sel]
pin_paf.array[:] = paf_h[sel]
e = pf.PafParser(topo)
e.parse_arrays(pin_conf.array, pin_paf.array, 8, pf.ParserParams(upsample=8))
print("frames", E)
