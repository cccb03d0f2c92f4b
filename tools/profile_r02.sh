#!/bin/bash
# r02 profiling call: one `ncu --set full` capture per hot kernel (each program exits 0 without
# ncu first), summarised ON the box (tools/ncu_box_summary.py; the reports themselves are too
# large to bring back), and the bench's ncu launch list.  Output: gpurun_out/r02/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
  python tools/ncu_box_summary.py $O > /dev/null 2>&1
  tail -c 2000 $O/$name.log > $O/$name.logtail; rm -f $O/$name.log
}
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; tail -15 $O/pytest.log
python tools/kbench.py matvec 512 5 > $O/kb_matvec.txt 2>&1 || exit 1
for d in 1 2 3 4; do python tools/kbench.py solve 26 $d 5 > $O/kb_solve$d.txt 2>&1 || exit 1; done
python tools/kbench.py mrep 27 32 3 3 > $O/kb_mrep3.txt 2>&1 || exit 1
python tools/prof_step.py 512 1 1 16 > $O/prof_step.txt 2>&1 || exit 1
python tools/cfg_step.py c1 1 1 2 > $O/c1_res.txt 2>&1 || exit 1
python tools/cfg_step.py c2 2 1 2 > $O/c2_res.txt 2>&1 || exit 1
python tools/cfg_step.py c4 1 1 0 0 1 512 > $O/c4_cg.txt 2>&1 || exit 1
run matvec_march4 march4 1 1 python tools/kbench.py matvec 512 2
for d in 1 3 4; do
  run solve_d$d "tile_" 4 4 python tools/kbench.py solve 26 $d 1
done
run factor_d3 factor_pass 0 2 python tools/kbench.py solve 26 3 1
run mrep_sums mrep_tma 0 1 python tools/kbench.py mrep 27 32 3 1
run mrep_fit mrep_fitsum 0 1 python tools/kbench.py mrep 27 32 3 1
PCMD="python tools/prof_step.py 512 1 1 16"
run fused_k3 fused_tma 2 1 $PCMD
run fused_k6 fused_tma 5 1 $PCMD
run fused_k10 fused_tma 9 1 $PCMD
run fused_k14 fused_tma 13 1 $PCMD
run fused_hyb fused_tma 20 1 $PCMD
run icwy_dots icwy_dots 5 1 $PCMD
run icwy_update icwy_update 5 1 $PCMD
run update_combine update_combine 0 1 $PCMD
run ring_mrep_sums mrep_tma 0 1 $PCMD
run ring_mrep_fit mrep_fitsum 0 2 $PCMD
run resident_c1 resident 0 1 python tools/cfg_step.py c1 1 1 2
run resident_c2 resident 0 1 python tools/cfg_step.py c2 1 1 2
run cg_dir cg_dir4 3 1 python tools/cfg_step.py c4 1 1 0 0 1 512
run cg_update cg_update 3 1 python tools/cfg_step.py c4 1 1 0 0 1 512
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep"
$CMD > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_raw.csv $CMD > $O/ncu_launches.log 2>&1
echo "launches rc $?"
python tools/ncu_summary.py launches $O/launches_raw.csv > $O/launches.txt 2>&1; rm -f $O/launches_raw.csv
du -sh $O; ls $O
