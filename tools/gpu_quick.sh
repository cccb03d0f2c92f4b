#!/bin/bash
# quick GPU check: gpu tests + bench (no ncu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3 --no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
python - <<'PY'
import json
try:
    l=json.loads(open('gpurun_out/bench.json').readline())
    print('value',l['value'],'ms/step',l['ms_per_step'],'iters',l['iterations_per_step'],'clk',l['clocks'])
    for k,v in l['kernels'].items(): print(k, round(v['ms'],1), v['launches'], round(v['GBps'] or 0), round(v['share'],3))
except Exception as e: print('bench parse failed', e)
PY
