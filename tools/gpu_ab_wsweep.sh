#!/bin/bash
# warp-range banded sweeps: parity tests, then solve times (n = 2^26, d = 1..4) for the default
# build, register-capped builds (PSP_WSWEEP_MINB) and the tile kernels (PSP_SOLVE_BLOCK=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${AB_OUT:-wsweep}
mkdir -p $O
[ -n "$AB_NOTEST" ] || timeout 900 python -m pytest tests -m gpu -q -x -k "banded or multirank_banded or precond_multirank or free_running_c1 or c5_full" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for i in $(seq ${AB_REPS:-2}); do
for v in base ${AB_VARIANTS:-w3 w4} blk; do
  case $v in
    base) E="" ;;
    blk) E="PSP_SOLVE_BLOCK=1" ;;
    *) E="PSP_LIB=build/$v/libpspgmres.so" ;;
  esac
  for d in 1 2 3 4; do echo "$v: $(env $E timeout 300 python tools/kbench.py solve 26 $d 10 2>&1 | grep 'solve n')"; done
done
done 2>&1 | tee $O/ab.log
