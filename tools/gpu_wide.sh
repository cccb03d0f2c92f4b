#!/bin/bash
# single-pass wide steps (k > 16) vs the split-column steps, 512^3, same box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
  echo "== hyb (bench default)"; timeout 300 python tools/kstep.py 512 4 1 16 16 2>&1 | tail -2
  KSTEP_VARIANTS="default,PSP_FUSED_WIDE=1,PSP_FUSED_WIDE=2" timeout 600 python tools/kstep.py 512 4 1 30 16 2>&1 | tail -6
done
