#!/bin/bash
# MREP streaming kernel: two rows a thread (default) vs one (PSP_MREP_SUMS1): MREP parity tests,
# then C4-ring and C5 raw timings on one box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
[ -n "$AB_NOTEST" ] || timeout 900 python -m pytest tests -m gpu -q -x -k "mrep or MREP or determinism or ridge or fit or stream or c5 or lockstep_128" 2>&1 | tail -2
for i in 1 2; do
for v in two one; do
  if [ $v = one ]; then E="PSP_MREP_SUMS1=1"; else E=""; fi
  echo "$v: $(env $E timeout 300 python tools/kbench.py mrepring 512 5 2>&1 | tail -1)"
  for dm in "16 3" "32 2" "32 3" "32 4" "64 3"; do set -- $dm; echo "$v: $(env $E timeout 300 python tools/kbench.py mrep 26 $1 $2 3 2>&1 | tail -1)"; done
done
done
