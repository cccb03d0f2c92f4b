cd "${GRAFT_REPO_ROOT:-/root/repo}"
for d in 2 3 4; do PSP_LIB=build/v1/libpspgmres.so timeout 120 python tools/kbench.py mrep 26 32 $d 3; done
