#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for d in 2 3 4; do
  echo "chol d=$d: $(python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"
  echo "ldl  d=$d: $(PSP_MREP_LDL=1 python tools/kbench.py mrep 26 32 $d 3 2>&1 | tail -1)"
done
done
PSP_MREP_LDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mrep" 2>&1 | tail -3
PSP_MREP_LDL=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "c5" 2>&1 | tail -3
