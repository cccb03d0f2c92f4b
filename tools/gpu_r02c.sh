#!/bin/bash
# r02 third call: GPU tests (parity log), C1 / C2 resident timings, PSP-CG vs GMRES at C4 sizes.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/parity_log.jsonl
PSP_PARITY_LOG=$PWD/gpurun_out/parity_log.jsonl timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
rm -f gpurun_out/cfg.jsonl
for args in "c1 5 1 1" "c2 20 1 2" "c4 3 1 0 0 0 512" "c4 3 1 0 0 1 512"; do
  timeout 600 python tools/cfg_step.py $args >> gpurun_out/cfg.jsonl 2>> gpurun_out/cfg.err
done
cat gpurun_out/cfg.jsonl; tail -5 gpurun_out/cfg.err
