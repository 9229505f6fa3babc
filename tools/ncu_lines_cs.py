#!/usr/bin/env python
"""Per-source-line hot spots from `ncu --page source --csv --print-source cuda,sass`.

  python tools/ncu_lines_cs.py FILE.csv [N]
Prints the top-N CUDA source lines by warp-stall samples and by executed
warp instructions (file:line, samples, instructions, source)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname = None
hdr = None
recs = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samp = int(r[4])
        inst = int(r[7])
    except (ValueError, IndexError):
        continue
    recs.append((fname, r[0], samp, inst, r[1].strip()[:90]))
tot_s = sum(x[2] for x in recs) or 1
tot_i = sum(x[3] for x in recs) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
print("-- by stall samples")
for f, ln, s, i, src in sorted(recs, key=lambda x: -x[2])[:n]:
    print(f"{f}:{ln:>5} {100*s/tot_s:5.1f}% inst {100*i/tot_i:5.1f}%  {src}")
print("-- by instructions")
for f, ln, s, i, src in sorted(recs, key=lambda x: -x[3])[:n]:
    print(f"{f}:{ln:>5} {100*s/tot_s:5.1f}% inst {100*i/tot_i:5.1f}%  {src}")
