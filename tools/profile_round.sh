#!/bin/bash
# Round profiling call (run under gpurun): the plain bench line, then the ncu launch list of the
# same step command and one --set full capture of the top kernels of a C4 512^3 step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc $?"
PCMD="python tools/prof_step.py 512 1 1 16"
$PCMD > gpurun_out/prof_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fused_tma|icwy_dots|icwy_update|march4|mrep_tma|tile_map|factor_pass" \
    -s 60 -c 8 -o gpurun_out/prof_full $PCMD > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
