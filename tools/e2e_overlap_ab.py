"""e2e (pf_parse_host, 8192 pinned frames of the bench stream) with
PF_OPT_HOST_OVERLAP off / on and the PAF in place / copied (dev tool):
frames/s and a digest of every frame's pose_record (must not change)."""
import hashlib
import sys
import time

sys.path.insert(0, ".")
import paper_2108_11826_b200 as pf  # noqa: E402
from paper_2108_11826_b200 import _native  # noqa: E402
from support import synth  # noqa: E402

E = 8192
topo = pf.load_topology("coco18")
sp = synth.SynthParams()
scenes = [synth.procedural_scene(5, s, 656, 368, sp) for s in range(E)]
conf_d, paf_d = synth.render_batch_gpu(scenes, topo, sp)
pin_conf = _native.PinnedArray((E, 19, 46, 82))
pin_paf = _native.PinnedArray((E, 38, 46, 82))
pin_conf.array[:] = conf_d.cpu().numpy()
pin_paf.array[:] = paf_d.cpu().numpy()
del conf_d, paf_d
params = pf.ParserParams(upsample=8)
eng = pf.PafParser(topo)
ref = None
import os
CS = [int(x) for x in os.environ.get("CORNER_SPLIT", "1").split(",")]
for zc in (1, 0):
    for ov in (0, 1):
      for cs in CS:
        eng.ctx.set_option(_native.PF_OPT_CORNER_SPLIT, cs)
        eng.ctx.set_option(_native.PF_OPT_PAF_ZERO_COPY, zc)
        eng.ctx.set_option(_native.PF_OPT_HOST_OVERLAP, ov)
        r = eng.parse_arrays(pin_conf.array, pin_paf.array, 8, params)
        dg = hashlib.sha1("".join(r.records(topo)).encode()).hexdigest()[:12]
        ref = ref or dg
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(3):
                eng.parse_arrays(pin_conf.array, pin_paf.array, 8, params)
            best = min(best, (time.perf_counter() - t0) / 3)
        print(f"paf_zero_copy={zc} host_overlap={ov} corner_split={cs}: {E / best:.0f} frames/s ({best * 1e3:.2f} ms)  digest {dg} "
              f"{'OK' if dg == ref else 'DIFFERS'}", flush=True)
