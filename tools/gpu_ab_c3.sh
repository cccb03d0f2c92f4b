#!/bin/bash
# 2-D fused pass KMAX granularity: lockstep parity on the 2-D cases, then C3 / C2 host-driven
# step times with and without the KMAX 4 / 12 instantiations (PSP_FUSED_COARSE) on one box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
[ -n "$AB_NOTEST" ] || timeout 1200 python -m pytest tests -m gpu -q -x -k "lockstep and (C2 or C3 or C1)" 2>&1 | tail -2
for i in 1 2; do
  for v in fine coarse; do
    if [ $v = coarse ]; then E="PSP_FUSED_COARSE=1"; else E=""; fi
    echo "$v c3: $(env $E timeout 600 python tools/cfg_step.py c3 2 1 0 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
