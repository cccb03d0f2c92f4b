cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python tools/kbench.py solve 24 3 3 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 2 -o gpurun_out/prof_sweep python tools/kbench.py solve 24 3 3 > gpurun_out/ncu_sweep.log 2>&1
echo done
