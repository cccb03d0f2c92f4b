cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|rc " gpurun_out/pytest_gpu.log | tail -4
timeout 600 python tools/paper_f1.py gpurun_out/f1.json > gpurun_out/f1.log 2>&1; cat gpurun_out/f1.log
