#!/usr/bin/env python
"""Summarise an ncu launch list + an ncu --set full report into profiles/.

  python tools/profile_summary.py ROUND LAUNCHES.csv FULL.ncu-rep FRAMES_PER_LAUNCH

  python tools/profile_summary.py --unfused ROUND UNFUSED.ncu-rep FRAMES
  python tools/profile_summary.py --e2e-pcie ROUND E2E_SYSMEM.csv FRAMES

Writes profiles/<ROUND>_launches.md, profiles/<ROUND>_ncu_full.md and
profiles/<ROUND>_traffic.json (dram bytes per launch of each profiled kernel,
read by bench.py for the roofline "traffic" field).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        us = float(r[vi].replace(",", "")) * UNITS[r[ui]]
        a = agg.setdefault(name, [0, 0.0, float("inf"), 0.0])
        a[0] += 1
        a[1] += us
        a[2] = min(a[2], us)
        a[3] = max(a[3], us)
    return agg


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m in want:
            if m in h:
                i = h.index(m)
                d[m] = (r[i], units[i])
        stalls = []
        for i, col in enumerate(h):
            if col.startswith("smsp__average_warps_issue_stalled_") and col.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), col[34:-23]))
                except ValueError:
                    pass
        d["stalls"] = sorted(stalls, reverse=True)[:6]
        res.append(d)
    return res


def to_bytes(v):
    val, unit = v
    return float(val.replace(",", "")) * BYTES.get(unit, 1)


# materialised Mode U kernels (tools/unfused_run.py): compulsory bytes per frame
UNFUSED_ALG = {"k_resize_planes": 18 * 46 * 82 * 4 + 18 * 368 * 656 * 4, "k_nms_plane": 18 * 368 * 656 * 4}


def unfused(rnd, rep, frames):
    """profiles/<rnd>_ncu_unfused.md from the --set full capture of tools/unfused_run.py."""
    path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_unfused.md")
    with open(path, "w") as f:
        f.write(f"# {rnd}: ncu --set full of the materialised Mode U kernels (first launch of each: {frames} frames "
                "= the 2 GiB workspace chunk)\n\n`python tools/unfused_run.py`.  Algorithmic bytes per frame: "
                f"resize = read 18 low-res part planes + write 18 x 368x656 f32 = {UNFUSED_ALG['k_resize_planes']:,} B; "
                f"NMS = read 18 x 368x656 f32 = {UNFUSED_ALG['k_nms_plane']:,} B.\n\n")
        seen = set()
        for d in full_metrics(rep):
            if d["kernel"] in seen or d["kernel"] not in UNFUSED_ALG:
                continue
            seen.add(d["kernel"])
            f.write(f"## {d['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
            for k, v in d.items():
                if k not in ("kernel", "stalls"):
                    f.write(f"| {k} | {v[0]} | {v[1]} |\n")
            rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
            us = float(d["gpu__time_duration.sum"][0].replace(",", "")) * UNITS[d["gpu__time_duration.sum"][1]]
            alg = UNFUSED_ALG[d["kernel"]]
            f.write(f"| dram read+write per frame | {(rd + wr) / frames:.0f} | byte |\n")
            f.write(f"| algorithmic bytes per frame | {alg} | byte |\n")
            f.write(f"| algorithmic GB/s (cold, serialised) | {alg * frames / us / 1e3:.0f} | GB/s |\n")
            f.write("\nTop stall reasons (warps per issue): " +
                    ", ".join(f"{n} {x:.2f}" for x, n in d["stalls"]) + "\n\n")
    print(open(path).read())


def e2e_pcie(rnd, csv_path, frames):
    """profiles/<rnd>_e2e_pcie.json from tools/e2e_sysmem.py under ncu (PCIe metrics)."""
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        m = agg.setdefault(name, collections.OrderedDict())
        m[r[mi]] = m.get(r[mi], 0.0) + float(r[vi].replace(",", ""))
    out = {"what": f"PCIe traffic of one pf_parse_host call ({frames} pinned frames of the bench e2e workload) "
                   "with the PAF read in place (PF_OPT_PAF_ZERO_COPY) by the one-kernel k_parse_frames",
           "command": "ncu --metrics syslts__d_sectors_fill_sysmem.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,"
                      "gpu__time_duration.sum python tools/e2e_sysmem.py", "frames": frames}
    out.update(agg)
    pk = agg.get("k_parse_frames", {})
    out["paf_read_in_place_bytes_per_frame"] = round(pk.get("pcie__read_bytes.sum", 0.0) / frames)
    out["paf_sysmem_sector_fill_bytes_per_frame"] = round(pk.get("syslts__d_sectors_fill_sysmem.sum", 0.0) * 32 / frames)
    out["paf_bytes_per_frame_if_copied"] = 38 * 46 * 82 * 4
    with open(os.path.join(ROOT, "profiles", f"{rnd}_e2e_pcie.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


def main():
    if sys.argv[1] == "--unfused":
        return unfused(sys.argv[2], sys.argv[3], int(sys.argv[4]))
    if sys.argv[1] == "--e2e-pcie":
        return e2e_pcie(sys.argv[2], sys.argv[3], int(sys.argv[4]))
    rnd, lpath, rep, frames = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    agg = launches(lpath)
    tot = sum(a[1] for a in agg.values())
    with open(os.path.join(prof, f"{rnd}_launches.md"), "w") as f:
        f.write(f"# {rnd}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)\n\n")
        f.write("Cold-cache, serialised per-launch times of every kernel in a short bench run "
                "(device-resident step, e2e chunks and the unfused comparison); compare SHARES, not absolutes.\n\n")
        f.write("| kernel | launches | total ms | mean ms | min ms | max ms | share |\n|---|---|---|---|---|---|---|\n")
        for k, (n, t, lo, hi) in agg.items():
            f.write(f"| {k} | {n} | {t/1e3:.3f} | {t/n/1e3:.3f} | {lo/1e3:.3f} | {hi/1e3:.3f} | {t/tot*100:.1f}% |\n")
    met = full_metrics(rep)
    traffic = {"frames_per_launch": frames}
    with open(os.path.join(prof, f"{rnd}_ncu_full.md"), "w") as f:
        f.write(f"# {rnd}: ncu --set full (one launch each, {frames} frames per launch)\n\n")
        for d in met:
            f.write(f"## {d['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
            for k, v in d.items():
                if k in ("kernel", "stalls"):
                    continue
                f.write(f"| {k} | {v[0]} | {v[1]} |\n")
            rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
            f.write(f"| dram read+write per frame | {(rd + wr) / frames:.0f} | byte |\n")
            f.write("\nTop stall reasons (warps per issue): " +
                    ", ".join(f"{n} {x:.2f}" for x, n in d["stalls"]) + "\n\n")
            traffic[d["kernel"]] = rd + wr
    with open(os.path.join(prof, f"{rnd}_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print(open(os.path.join(prof, f"{rnd}_launches.md")).read())
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
