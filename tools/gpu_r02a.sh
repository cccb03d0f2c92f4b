#!/bin/bash
# r02 first call: GPU tests with the parity-floor log, smoke, the bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/lscpu.txt 2>&1
rm -f gpurun_out/parity_log.jsonl
PSP_PARITY_LOG=$PWD/gpurun_out/parity_log.jsonl timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
