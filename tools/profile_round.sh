#!/bin/bash
# Round profiling call (run under gpurun): the plain bench line, then the ncu launch list of the
# same step command and --set full captures of the top kernels of a C4 512^3 step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc $?"
PCMD="python tools/prof_step.py 512 1 1 16"
$PCMD > gpurun_out/prof_step.log 2>&1 || exit 1
# one capture per kernel class: fused pass k = 10 (KMAX 12) and a split-column step's fused part
# (launch 20), the split-column dots / update passes, the MREP streaming and fit kernels
i=0
for sel in "fused_tma:10:2" "fused_tma:20:1" "icwy_dots:5:1" "icwy_update:5:1" "mrep_tma:0:1" "mrep_fitsum:0:1"; do
  k=${sel%%:*}; rest=${sel#*:}; s=${rest%%:*}; c=${rest#*:}
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c \
      -o gpurun_out/prof_full_$i $PCMD > gpurun_out/ncu_full_$i.log 2>&1
  echo "full $k rc $?"
  i=$((i+1))
done
