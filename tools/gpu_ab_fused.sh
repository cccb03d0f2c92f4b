#!/bin/bash
# A/B of fused-pass build variants (PSP_LIB): per-k step times at 512^3 (tools/kstep.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for v in base ${AB_VARIANTS:-u2 u4 s3 u4s3 u2s3}; do
  if [ $v = base ]; then L=""; else L="PSP_LIB=build/$v/libpspgmres.so"; fi
  echo "== $v"; env $L timeout 300 python tools/kstep.py 512 4 2>&1 | tail -2
done
done
