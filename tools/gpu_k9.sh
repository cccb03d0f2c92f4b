cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; grep -E "passed|failed|FAIL|Error|Timeout|rc " gpurun_out/pytest_gpu.log | tail -12
for f in 0 1; do
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --fused $f > gpurun_out/bench_f$f.json 2> gpurun_out/bench_f$f.err
python - $f <<'PY'
import json,sys
f=sys.argv[1]
try:
    l=json.loads(open(f'gpurun_out/bench_f{f}.json').readline())
    print('fused',f,'value',round(l['value']/1e9,2),'G','ms/step',round(l['ms_per_step'],1),'iters',l['iterations_per_step'],'clk',l['clocks']['sm_mhz'],l['clocks']['reasons'])
    for k,v in l['kernels'].items(): print('  ',k, round(v['ms'],1), v['launches'], round(v['GBps'] or 0), round(v['share'],3))
except Exception as e: print('bench parse failed', e, open(f'gpurun_out/bench_f{f}.err').read()[-2000:])
PY
done
timeout 300 python tools/prof_step.py 512 1 1 > gpurun_out/prof_step.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tma -s 15 -c 1 -o gpurun_out/prof_fused6 python tools/prof_step.py 512 1 1 > gpurun_out/ncu_fused6.log 2>&1
echo ncu done
