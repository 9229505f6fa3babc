"""Survivor / cell / candidate statistics of k_corner_finish on the C5 step
(dev tool; needs a -DPF_FIN_PROF build loaded through PF_B200_LIB)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402

topo = pf.load_topology("coco18")
sp = synth.SynthParams()
scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(8192)]
conf, paf = synth.render_batch_gpu(scenes, topo, sp)
e = pf.PafParser(topo)
params = pf.ParserParams(upsample=8)
lib = _native.load_library()
buf = (ctypes.c_ulonglong * 16)()
e.parse_tensors(conf, paf, 8, params)
e.results()
lib.pf_corner_prof_read(buf, 1)
e.parse_tensors(conf, paf, 8, params)
e.results()
lib.pf_corner_prof_read(buf, 1)
planes = buf[12]
names = {0: "survivors", 1: "normal cells", 2: "partial cells", 3: "corner candidates", 4: "partial candidates",
         6: "partial ok=0", 7: "partial ok=1 (h)", 8: "partial ok=2 (v)"}
print("planes", planes)
for k, n in names.items():
    print(f"{n:20s} {buf[k] / planes:8.3f} per plane")
