#!/bin/bash
# banded solve build variants (PSP_LIB), n = 2^26, d = 1..4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for v in base ${AB_VARIANTS:-sr12 sr16}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  for d in 1 2 3 4; do echo "$v: $(env $L timeout 300 python tools/kbench.py solve 26 $d 10 2>&1 | grep solve)"; done
done
done
