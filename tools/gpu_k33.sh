cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_multirank.py -m gpu -q --timeout 200 --timeout-method=thread 2>&1 | grep -E "passed|failed|FAILED"; done
