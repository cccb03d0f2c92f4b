#!/bin/bash
# MREP parity tests, then ring / raw MREP timings against build variants (same box)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
[ -n "$AB_NOTEST" ] || timeout 900 python -m pytest tests -m gpu -q -x -k "mrep or MREP or determinism or ridge or fit or stream or c5" 2>&1 | tail -2
for i in $(seq ${AB_REPS:-2}); do
for v in base ${AB_VARIANTS:-fitnopf}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "$v: $(env $L timeout 300 python tools/kbench.py mrepring 512 5 2>&1 | tail -1)"
  for d in 2 3 4; do echo "$v: $(env $L timeout 300 python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"; done
done
done
