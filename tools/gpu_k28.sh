cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 --timeout-method=thread -k "matvec or lockstep or multirank" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|rc " gpurun_out/pytest_gpu.log | tail -4
python tools/kbench.py matvec 512 20
PSP_MARCH3=1 python tools/kbench.py matvec 512 20
