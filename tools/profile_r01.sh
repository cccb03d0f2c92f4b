#!/bin/bash
# Round-1 profiling call (run under gpurun): plain run, then the ncu launch list and one full
# capture of the dominant kernel (icwy_update_kernel) and of icwy_dots / mrep for context.
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"icwy_update|icwy_dots|matvec_kernel|mrep_interior" -s 40 -c 8 \
    -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
