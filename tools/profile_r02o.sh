#!/bin/bash
# r02o profiling call: ncu captures of the final build's banded factor (d = 3) and MREP (C5
# d = 3: sums + fit), summarised on the box.  Output: gpurun_out/r02o/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${PROF_OUT:-r02o}
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
  python tools/ncu_box_summary.py $O > /dev/null 2>&1
  tail -c 2000 $O/$name.log > $O/$name.logtail; rm -f $O/$name.log
}
run factor_d3 factor_pass 0 1 python tools/kbench.py solve 26 3 3
run mrep_d3 "mrep_tma|mrep_fitsum" 0 4 python tools/kbench.py mrep 26 32 3 2
du -sh $O; ls $O
