#!/bin/bash
# Same-box A/B: run a kbench command against the in-tree library and a comparison build
# (paper_1308_5626_b200/libpspgmres_old.so), alternating, REPS times.
#   bash tools/ab.sh "solve 26 3 10" 2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${2:-2}); do
  for L in libpspgmres libpspgmres_old; do
    echo "== $L"; PSP_LIB=paper_1308_5626_b200/$L.so timeout 300 python tools/kbench.py $1
  done
done
