cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python tools/prof_step.py 512 1 1 > gpurun_out/prof_step.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_tma -c 40 --csv --log-file gpurun_out/fused_launches.csv python tools/prof_step.py 512 1 1 > gpurun_out/ncu_fl.log 2>&1
echo done
