cd "${GRAFT_REPO_ROOT:-/root/repo}"
python tools/kbench.py matvec 512 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 -o gpurun_out/prof_matvec3 python tools/kbench.py matvec 512 3 > gpurun_out/ncu_matvec3.log 2>&1
timeout 120 python tools/kbench.py mrep 24 32 3 3 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:mrep_tma -s 1 -c 1 -o gpurun_out/prof_mrep2 python tools/kbench.py mrep 24 32 3 3 > gpurun_out/ncu_mrep2.log 2>&1
tail -1 gpurun_out/ncu_matvec3.log gpurun_out/ncu_mrep2.log
