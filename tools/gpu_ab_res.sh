#!/bin/bash
# resident solve: parity tests + C1/C2 step times, this build vs build/${AB_VARIANTS:-prev}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests -m gpu -q -x -k "resident" 2>&1 | tail -2
for i in 1 2; do
for v in base ${AB_VARIANTS:-prev}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "$v c1: $(env $L timeout 300 python tools/cfg_step.py c1 5 1 1 2>&1 | tail -1 | cut -c1-200)"
  echo "$v c2: $(env $L timeout 300 python tools/cfg_step.py c2 20 1 2 2>&1 | tail -1 | cut -c1-120)"
done
done
