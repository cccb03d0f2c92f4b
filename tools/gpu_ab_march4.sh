#!/bin/bash
# march4 stencil A/B at 512^3 (kbench matvec): builds (PSP_LIB) and z-chunk lengths (PSP_MARCH4_ZC)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
[ -n "$AB_NOTEST" ] || timeout 600 python -m pytest tests -m gpu -q -x -k "matvec" 2>&1 | tail -2
for i in $(seq ${AB_REPS:-2}); do
for v in base ${AB_VARIANTS:-l2pf} zc32 zc64 zc128; do
  case $v in
    base) E="" ;;
    zc*) E="PSP_MARCH4_ZC=${v#zc}" ;;
    *) E="PSP_LIB=build/$v/libpspgmres.so" ;;
  esac
  echo "$v: $(env $E timeout 300 python tools/kbench.py matvec 512 20 2>&1 | grep '^matvec 512')"
done
done
