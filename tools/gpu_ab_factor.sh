#!/bin/bash
# banded factor: parity tests, then factor / solve times (n = 2^26, d = 1..4) for the default
# build (cooperative staging), build variants (PSP_LIB) and the per-thread copies (PSP_FACTOR_NOCOOP)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${AB_OUT:-factor}
mkdir -p $O
[ -n "$AB_NOTEST" ] || timeout 900 python -m pytest tests -m gpu -q -x -k "banded or multirank_banded or precond_multirank or free_running_c1 or c5_full or f1" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for i in $(seq ${AB_REPS:-2}); do
for v in base ${AB_VARIANTS:-pf2 t32 pf2t32} nocoop; do
  case $v in
    base) E="" ;;
    nocoop) E="PSP_FACTOR_NOCOOP=1" ;;
    *) E="PSP_LIB=build/$v/libpspgmres.so" ;;
  esac
  for d in 1 2 3 4; do echo "$v: $(env $E timeout 300 python tools/kbench.py solve 26 $d 10 2>&1 | grep 'factor n')"; done
done
done 2>&1 | tee $O/ab.log
