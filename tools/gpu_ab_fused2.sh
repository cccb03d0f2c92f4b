#!/bin/bash
# bench-mode per-k times (fused_kmax 16, split-column steps above) for build variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for v in base ${AB_VARIANTS:-s3}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "== $v"; env $L timeout 300 python tools/kstep.py 512 4 1 16 ${SPLIT:-16} 2>&1 | tail -2
done
done
