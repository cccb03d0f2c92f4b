cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python tools/kbench.py mrep 24 32 3 3 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:mrep_tma -s 1 -c 1 -o gpurun_out/prof_mrep4 python tools/kbench.py mrep 24 32 3 3 > gpurun_out/ncu_mrep4.log 2>&1
echo done
