cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PSP_LIB=build/v1/libpspgmres.so
timeout 120 python tools/kbench.py mrep 24 32 3 3 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:mrep_tma -s 1 -c 1 -o gpurun_out/prof_mrep3 python tools/kbench.py mrep 24 32 3 3 > gpurun_out/ncu_mrep3.log 2>&1
unset PSP_LIB
python tools/kbench.py matvec 512 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 -o gpurun_out/prof_matvec4 python tools/kbench.py matvec 512 3 > gpurun_out/ncu_matvec4.log 2>&1
echo ok
