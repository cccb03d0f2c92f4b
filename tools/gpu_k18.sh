cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python tools/kbench.py solve 27 3 2 > /dev/null && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tile_" -c 12 --csv --log-file gpurun_out/solve_launches.csv python tools/kbench.py solve 27 3 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"tile_apply" -s 1 -c 1 -o gpurun_out/prof_apply python tools/kbench.py solve 24 3 2 > /dev/null 2>&1
echo done
