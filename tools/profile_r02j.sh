#!/bin/bash
# late-r02 profiling call: fresh `ncu --set full` captures of the kernels changed since
# profile_r02.sh (the resident solve, the fused pass with per-axis stencil accumulators) and the
# bench step's launch list; summarised on the box.  Output: gpurun_out/r02j/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02j
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
  python tools/ncu_box_summary.py $O > /dev/null 2>&1
  tail -c 2000 $O/$name.log > $O/$name.logtail; rm -f $O/$name.log
}
python tools/cfg_step.py c1 1 1 1 > $O/c1_res.txt 2>&1 || exit 1
python tools/cfg_step.py c2 2 1 2 > $O/c2_res.txt 2>&1 || exit 1
python tools/prof_step.py 512 1 1 16 > $O/prof_step.txt 2>&1 || exit 1
run resident_c1 resident 0 1 python tools/cfg_step.py c1 1 1 1
run resident_c2 resident 0 1 python tools/cfg_step.py c2 1 1 2
PCMD="python tools/prof_step.py 512 1 1 16"
run fused_k3 fused_tma 2 1 $PCMD
run fused_k10 fused_tma 9 1 $PCMD
run fused_k14 fused_tma 13 1 $PCMD
run fused_hyb fused_tma 20 1 $PCMD
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep"
$CMD > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_raw.csv $CMD > $O/ncu_launches.log 2>&1
echo "launches rc $?"
python tools/ncu_summary.py launches $O/launches_raw.csv > $O/launches.txt 2>&1; rm -f $O/launches_raw.csv
du -sh $O; ls $O
