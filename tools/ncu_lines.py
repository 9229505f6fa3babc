"""Aggregate an ncu source page (--print-source cuda,sass) by CUDA source line."""
import csv, subprocess, sys, collections

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        key = (cur_file, int(r[0]))
    except ValueError:
        continue
    a = agg[key]
    num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
    a[0] += num(r[ii])
    a[1] += num(r[si])
    a[2] = r[1][:100]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti}, stall samples {ts}")
order = 0 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 1
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][order])[:top]:
    print(f"{v[1]/ts*100:5.1f}% stall {v[0]/ti*100:5.1f}% inst  {key[0]}:{key[1]}  {v[2]}")
