cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|rc " gpurun_out/pytest_gpu.log | tail -4
for d in 1 2 3 4; do timeout 120 python tools/kbench.py mrep 26 32 $d 3; done
