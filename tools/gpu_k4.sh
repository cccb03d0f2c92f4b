cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -v -x --timeout 120 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "PASS|FAIL|Timeout|rc " gpurun_out/pytest_gpu.log | tail -30
timeout 120 python tools/kbench.py mrep 24 32 3 3 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:mrep_tma -s 1 -c 1 -o gpurun_out/prof_mrep python tools/kbench.py mrep 24 32 3 3 > gpurun_out/ncu_mrep.log 2>&1
tail -2 gpurun_out/ncu_mrep.log
