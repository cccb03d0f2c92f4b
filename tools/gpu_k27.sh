cd "${GRAFT_REPO_ROOT:-/root/repo}"
for d in 1 3 4; do timeout 120 python tools/kbench.py mrep 26 32 $d 3; done
for d in 1 3 4; do PSP_LIB=build/v1/libpspgmres.so timeout 120 python tools/kbench.py mrep 26 32 $d 3; done
