#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for d in 2 3; do
  echo "base d=$d: $(python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"
  for v in c8 c32 nst4 fit1; do echo "$v d=$d: $(PSP_LIB=build/$v/libpspgmres.so python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"; done
done
done
