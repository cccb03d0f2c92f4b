#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/abm2
mkdir -p $O
python tools/kbench.py mrep 26 32 1 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file $O/r02.csv python tools/kbench.py mrep 26 32 1 1 > /dev/null 2>&1
PSP_LIB=build/r01/libpspgmres.so ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file $O/r01.csv python tools/kbench.py mrep 26 32 1 1 > /dev/null 2>&1
for f in r01 r02; do echo "== $f"; python - $O/$f.csv <<'PY'
import csv, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; k=h.index("Kernel Name"); m=h.index("Metric Name"); v=h.index("Metric Value"); idx=h.index("ID")
d={}
for r in rows[1:]:
    d.setdefault((r[idx], r[k][:60]), {})[r[m]]=r[v]
for (i,kn),mm in list(d.items())[:40]:
    print(i, kn, mm)
PY
done
