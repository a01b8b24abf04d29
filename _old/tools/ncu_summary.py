"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py <tag> <launches.csv> <full.ncu-rep>[,<more.ncu-rep>...]

Writes profiles/<tag>_launches.csv (per-kernel aggregate of the launch list),
profiles/<tag>_kernels.json (selected metrics of the full capture per launch)
and profiles/<tag>_summary.md.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_active.avg",
]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    start = rows.index(hdr) + 1
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    return agg


def full_table(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]].split("(")[0]}
        for m in METRICS:
            if m in idx:
                v = d[idx[m]].replace(",", "")
                try:
                    rec[m] = float(v)
                except ValueError:
                    rec[m] = v
                rec[m + ":unit"] = units[idx[m]]
        st = {}
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[idx[k]] or 0)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        rec["stall_top"] = {k: round(100 * v / tot, 1)
                            for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        res.append(rec)
    return res


def main():
    tag, launches, rep = sys.argv[1:4]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    agg = launch_table(launches)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as fh:
        fh.write("kernel,launches,total_us,share\n")
        for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{k},{n},{us:.1f},{us / tot:.4f}\n")
    full = [r for one in rep.split(",") for r in full_table(one)]
    with open(os.path.join(ROOT, "profiles", f"{tag}_kernels.json"), "w") as fh:
        json.dump(full, fh, indent=1)
    lines = [f"# ncu summary {tag}", "", "## Launch list (ncu, cold cache, serialised)", "",
             "| kernel | launches | total us | share |", "| --- | --- | --- | --- |"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
        lines.append(f"| {k} | {n} | {us:.0f} | {100 * us / tot:.1f}% |")
    lines += ["", "## Full-set capture (per launch)", "",
              "| kernel | us | DRAM MB (r+w) | DMMA pipe % | FP64 pipe % | DRAM % | warps % | issue % | regs | top stalls |",
              "| --- | --- | --- | --- | --- | --- | --- | --- | --- | --- |"]
    for r in full:
        us = r.get("gpu__time_duration.sum", 0)
        us *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
               "msecond": 1e3}.get(r.get("gpu__time_duration.sum:unit"), 1.0)
        dr = (r.get("dram__bytes_read.sum", 0) or 0) + (r.get("dram__bytes_write.sum", 0) or 0)
        unit = r.get("dram__bytes_read.sum:unit", "byte")
        mb = dr * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
        lines.append("| {} | {:.1f} | {:.1f} | {} | {} | {} | {} | {} | {} | {} |".format(
            r["kernel"], us, mb,
            r.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "-"),
            r.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "-"),
            r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "-"),
            r.get("sm__warps_active.avg.pct_of_peak_sustained_active", "-"),
            r.get("smsp__issue_active.avg.pct_of_peak_sustained_active", "-"),
            r.get("launch__registers_per_thread", "-"),
            ", ".join(f"{k} {v}%" for k, v in list(r["stall_top"].items())[:3])))
    with open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
