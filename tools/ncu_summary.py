"""Print headline metrics of every kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
ki, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate"]
for row in r[1:]:
    if row[mi] in want and pat in row[ki]:
        print(f"{row[ki][:28]:28s} | {row[mi]:36s} {row[vi]} {row[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
for v in rr[2:]:
    name = v[h.index("Kernel Name")]
    if pat not in name:
        continue
    stalls = []
    for i, col in enumerate(h):
        if col.startswith("smsp__average_warps_issue_stalled_") and col.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), col[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    dr = [v[i] for i, col in enumerate(h) if col in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
    print(name[:40], "dram read/write:", dr, "| top stalls:",
          ", ".join(f"{n}={x:.2f}" for x, n in sorted(stalls, reverse=True)[:6]))
