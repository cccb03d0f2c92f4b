#!/bin/bash
# r02 profiling call: the bench's ncu launch list and one `ncu --set full` capture per hot kernel
# (each program exits 0 without ncu first).  Reports land in gpurun_out/r02/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, kernel regex, skip, count, command...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 $NCU -k regex:$k -s $s -c $c -o $O/$name "$@" > $O/$name.log 2>&1
  echo "$name rc $?"
}
timeout 900 python -m pytest tests/test_gpu_cg.py tests/test_gpu_parity.py -q -k "f1 or cg or resident or determinism" > $O/pytest_sel.log 2>&1; tail -5 $O/pytest_sel.log
# plain runs first (exit 0 without ncu)
python tools/kbench.py matvec 512 5 > $O/kb_matvec.txt 2>&1 || exit 1
python tools/kbench.py solve 26 3 5 > $O/kb_solve3.txt 2>&1 || exit 1
python tools/kbench.py mrep 27 32 3 3 > $O/kb_mrep3.txt 2>&1 || exit 1
python tools/prof_step.py 512 1 1 16 > $O/prof_step.txt 2>&1 || exit 1
python tools/cfg_step.py c1 1 1 2 > $O/c1_res.txt 2>&1 || exit 1
python tools/cfg_step.py c2 2 1 2 > $O/c2_res.txt 2>&1 || exit 1
python tools/cfg_step.py c4 1 1 0 0 1 512 > $O/c4_cg.txt 2>&1 || exit 1
# the stencil (march4), the banded sweeps and factor (d = 3), the MREP split kernels
run matvec_march4 march4 1 1 python tools/kbench.py matvec 512 2
for d in 1 2 3 4; do
  python tools/kbench.py solve 26 $d 2 > $O/kb_solve$d.txt 2>&1
  run solve_d$d "tile_" 4 4 python tools/kbench.py solve 26 $d 1
done
run factor_d3 factor_pass 0 2 python tools/kbench.py solve 26 3 1
run mrep_sums mrep_tma 0 1 python tools/kbench.py mrep 27 32 3 1
run mrep_fit mrep_fitsum 0 1 python tools/kbench.py mrep 27 32 3 1
# the C4 step: fused passes k = 3 (KMAX 4), 6 (KMAX 8), 10 (KMAX 12), 14 (KMAX 16), a split-column
# step's fused part, the split passes, the last-step combine, the C4 ring MREP (scaled probes)
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
# f2 resident solve (C1, one CTA; C2, cooperative grid) and f4 CG passes at 512^3
run resident_c1 resident 0 1 python tools/cfg_step.py c1 1 1 2
run resident_c2 resident 0 1 python tools/cfg_step.py c2 1 1 2
run cg_dir cg_dir4 3 1 python tools/cfg_step.py c4 1 1 0 0 1 512
run cg_update cg_update 3 1 python tools/cfg_step.py c4 1 1 0 0 1 512
# the bench's launch list (same step command, timed run first)
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep"
$CMD > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1
echo "launches rc $?"
ls $O | head -80
