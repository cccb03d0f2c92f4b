#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rNN_ncu_full.txt
  python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep <size> > profiles/traffic.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__occupancy_limit_registers",
           "smsp__inst_executed_pipe_fp64.sum"]

CLASS = {"icwy_update": "ortho_update", "icwy_dots": "ortho_dots", "matvec_kernel": "matvec",
         "mrep_interior": "mrep_fit", "sweep_kernel": "precond_solve", "combine": "combine",
         "arnoldi_fused": "arnoldi_fused"}


def short(name):
    return name.split("(")[0].replace("void ", "").split("::")[-1]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        agg[short(r[ki])][0] += 1
        agg[short(r[ki])][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none), {path}")
    print(f"# {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.2f} ms total (cold-cache, serialised)")
    print(f"{'kernel':42s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:42s} {c:8d} {t / 1e6:10.2f} {100 * t / tot:6.1f}%")


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(path):
    hdr, units, rows = raw(path)
    print(f"# ncu --set full summary of {path}")
    for r in rows:
        print("## " + short(r[hdr.index("Kernel Name")]))
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"   {m:60s} {r[i]} {units[i]}")


def traffic(path, size):
    hdr, units, rows = raw(path)
    res = {}
    for r in rows:
        nm = short(r[hdr.index("Kernel Name")])
        cls = next((v for k, v in CLASS.items() if k in nm), None)
        if cls is None:
            continue
        def val(m):
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            u = units[i]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        tr = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        res.setdefault(cls, []).append(tr)
    print(json.dumps({"size": size, "per_launch_dram_bytes": res}, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2])
    elif mode == "full":
        full(sys.argv[2])
    else:
        traffic(sys.argv[2], int(sys.argv[3]))
