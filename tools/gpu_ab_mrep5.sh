#!/bin/bash
# MREP parity + determinism tests, then ring / raw MREP timings against build/prevm (same box)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x -k "mrep or MREP or determinism or ridge or fit or stream or c5" 2>&1 | tail -2
for i in 1 2; do
for v in base prevm; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "$v: $(env $L timeout 300 python tools/kbench.py mrepring 512 5 2>&1 | tail -1) | $(env $L timeout 300 python tools/kbench.py mrep 26 32 3 3 2>&1 | tail -1)"
done
done
