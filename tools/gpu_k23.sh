cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python tools/kbench.py solve 24 3 2 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:factor_pass -s 1 -c 2 -o gpurun_out/prof_factor python tools/kbench.py solve 24 3 2 > gpurun_out/ncu_factor.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum -k regex:factor_pass --csv python tools/kbench.py solve 24 3 2 2>/dev/null | grep -c factor_pass
