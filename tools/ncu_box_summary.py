#!/usr/bin/env python
"""Summarise `ncu --set full` reports ON THE GPU BOX (the .ncu-rep files are too large to bring
back): per report, the key raw metrics, the top issue-stall reasons and the hottest SASS lines
(warp-stall samples) as small text files; the reports are then removed.

  python tools/ncu_box_summary.py <dir>      (writes <dir>/<name>.summary.txt, deletes <name>.ncu-rep)
"""
import csv
import glob
import io
import os
import subprocess
import sys

KEY = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
       "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
       "lts__t_bytes.sum", "l1tex__t_bytes.sum", "lts__t_sector_hit_rate.pct",
       "smsp__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu(path, page):
    return subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout


def summarise(rep):
    out = []
    rows = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    if len(rows) < 3:
        return "no data\n"
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        out.append("## " + r[hdr.index("Kernel Name")][:160])
        for m in KEY:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"   {m:60s} {r[i]} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i].replace(",", "")), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        out.append("   stalls (warps per issue-active cycle): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:7]))
    src = list(csv.reader(io.StringIO(ncu(rep, "source"))))
    hdr = next((x for x in src if x and x[0] == "Address"), None)
    if hdr:
        i0 = src.index(hdr)
        si = hdr.index("Warp Stall Sampling (All Samples)")
        lines = [x for x in src[i0 + 1:] if len(x) == len(hdr) and x[si].isdigit()]
        tot = sum(int(x[si] or 0) for x in lines) or 1
        lines.sort(key=lambda x: -int(x[si] or 0))
        out.append(f"   hottest SASS (share of {tot} warp-stall samples):")
        for x in lines[:25]:
            out.append(f"     {100 * int(x[si] or 0) / tot:5.1f}%  {x[1].strip()[:90]}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    d = sys.argv[1]
    for rep in sorted(glob.glob(os.path.join(d, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        with open(os.path.join(d, name + ".summary.txt"), "w") as f:
            f.write(summarise(rep))
        os.remove(rep)
