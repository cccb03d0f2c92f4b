cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python tools/prof_step.py 512 1 1 16 > gpurun_out/prof_step.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tma -s 2 -c 1 -o gpurun_out/prof_fk4 python tools/prof_step.py 512 1 1 16 > gpurun_out/ncu_fk4.log 2>&1
echo done
