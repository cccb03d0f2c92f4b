#!/bin/bash
# r02n profiling call: ncu captures of the late-r02 kernels (warp-range sweep d = 3 with its final
# knobs, the KMAX 6 / 10 / 14 fused passes) and the bench step's launch list.  Output: gpurun_out/r02n/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${PROF_OUT:-r02n}
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
  python tools/ncu_box_summary.py $O > /dev/null 2>&1
  tail -c 2000 $O/$name.log > $O/$name.logtail; rm -f $O/$name.log
}
run wsweep_d3 wsweep 0 4 python tools/kbench.py solve 26 3 3
PCMD="python tools/prof_step.py 512 1 1 16"
run fused_k5 fused_tma 4 1 $PCMD
run fused_k9 fused_tma 8 1 $PCMD
run fused_k13 fused_tma 12 1 $PCMD
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep"
$CMD > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_raw.csv $CMD > $O/ncu_launches.log 2>&1
echo "launches rc $?"
python tools/ncu_summary.py launches $O/launches_raw.csv > $O/launches.txt 2>&1; rm -f $O/launches_raw.csv
du -sh $O; ls $O
