cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|rc " gpurun_out/pytest_gpu.log | tail -4
python tools/kbench.py matvec 512 10
BENCH_ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c5" bash tools/gpu_bench.sh 2>&1 | head -12
timeout 300 python tools/prof_step.py 512 1 1 > gpurun_out/prof_step.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"icwy_dots|icwy_update" -s 20 -c 2 -o gpurun_out/prof_ortho python tools/prof_step.py 512 1 1 > gpurun_out/ncu_ortho.log 2>&1
echo done
