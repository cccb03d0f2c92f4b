#!/bin/bash
# MREP variants on the C4 ring (512^3, m = 32, d = 3) and on the raw path (n = 2^26)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for v in base ${AB_VARIANTS:-c32 lb5 lb5c32}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "$v: $(env $L timeout 300 python tools/kbench.py mrepring 512 5 2>&1 | tail -1) | $(env $L timeout 300 python tools/kbench.py mrep 26 32 3 3 2>&1 | tail -1)"
done
done
