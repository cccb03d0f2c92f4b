#!/bin/bash
# r02 second call: GPU tests (parity log), then C1 / C2 step timings host-driven vs resident.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/parity_log.jsonl
PSP_PARITY_LOG=$PWD/gpurun_out/parity_log.jsonl timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
rm -f gpurun_out/cfg.jsonl
for args in "c1 5 1 0" "c1 5 1 1" "c2 20 1 0" "c2 20 1 2" "c2 20 1 0 2" "c2 20 1 2 2"; do
  timeout 300 python tools/cfg_step.py $args >> gpurun_out/cfg.jsonl 2>> gpurun_out/cfg.err
done
cat gpurun_out/cfg.jsonl
