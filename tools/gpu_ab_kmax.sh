#!/bin/bash
# fused pass KMAX granularity: lockstep parity, then per-k step times (KMAX 4/6/8/10/12/14/16 vs
# the coarse 4/8/12/16 mapping, PSP_FUSED_COARSE) at 512^3 on one box, the bench's policy
# (fused steps 2..16)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
[ -n "$AB_NOTEST" ] || timeout 1200 python -m pytest tests -m gpu -q -x -k "lockstep or fused or cycle_invariants or determinism" 2>&1 | tail -2
KSTEP_VARIANTS="${KV:-default,PSP_FUSED_COARSE=1,default,PSP_FUSED_COARSE=1}" timeout 900 python tools/kstep.py 512 4 2 16 2>&1 | tail -12
