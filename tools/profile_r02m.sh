#!/bin/bash
# r02m profiling call: `ncu --set full` captures of the warp-range banded sweeps and the
# cooperative factor pass (C5 sizes, n = 2^26, d = 3), summarised on the box.  Output: gpurun_out/r02m/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${PROF_OUT:-r02m}
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
  python tools/ncu_box_summary.py $O > /dev/null 2>&1
  tail -c 2000 $O/$name.log > $O/$name.logtail; rm -f $O/$name.log
}
python tools/kbench.py solve 26 3 3 > $O/kbench_solve3.txt 2>&1 || exit 1
run factor_d3 factor_pass 0 1 python tools/kbench.py solve 26 3 3
run wsweep_d3 wsweep 0 4 python tools/kbench.py solve 26 3 3
run wsweep_d1 wsweep 0 2 python tools/kbench.py solve 26 1 3
run factor_d1 factor_pass 0 1 python tools/kbench.py solve 26 1 3
run factor_d4 factor_pass 0 1 python tools/kbench.py solve 26 4 3
${PROF_EXTRA:-true}
du -sh $O; ls $O
