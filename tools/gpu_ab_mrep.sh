#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/abm
mkdir -p $O
for i in 1 2; do
for d in 1 3; do
  echo "r02 d=$d: $(python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"
  echo "r01 d=$d: $(PSP_LIB=build/r01/libpspgmres.so python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"
done
done
python tools/cfg_step.py c1 5 1 2 | tail -1
