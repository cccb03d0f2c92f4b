cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|rc " gpurun_out/pytest_gpu.log | tail -4
timeout 300 python tools/prof_step.py 512 1 1 30 > gpurun_out/prof_step.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_tma -c 30 --csv --log-file gpurun_out/fused_launches.csv python tools/prof_step.py 512 1 1 30 > gpurun_out/ncu_fl.log 2>&1
for cfg in "--fused 1" "--fused 1 --fused-kmin 3 --fused-kmax 16"; do
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c5 $cfg > gpurun_out/bench_cfg.json 2> gpurun_out/bench_cfg.err
python - "$cfg" <<'PY'
import json,sys
try:
    l=json.loads(open('gpurun_out/bench_cfg.json').readline())
    print(sys.argv[1], '| value',round(l['value']/1e9,2),'G ms/step',round(l['ms_per_step'],1),'iters',l['iterations_per_step'],'clk',l['clocks']['sm_mhz'])
    for k,v in l['kernels'].items(): print('    ',k, round(v['ms'],1), v['launches'], round(v['GBps'] or 0), round(v['share'],3))
except Exception as e: print(sys.argv[1], 'failed', e, open('gpurun_out/bench_cfg.err').read()[-800:])
PY
done
