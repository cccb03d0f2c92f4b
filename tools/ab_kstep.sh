#!/bin/bash
# Same-box A/B of per-k Arnoldi step times: in-tree library vs paper_1308_5626_b200/libpspgmres_old.so
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${1:-2}); do
  for L in libpspgmres libpspgmres_old; do
    echo "== $L"; PSP_LIB=paper_1308_5626_b200/$L.so timeout 300 python tools/kstep.py ${2:-512} 4 2 16 2>&1 | tail -2
  done
done
