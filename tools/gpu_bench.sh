cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench.json').readline())
print('value',round(l['value']/1e9,2),'G ms/step',round(l['ms_per_step'],1),'iters',l['iterations_per_step'],'clk',l['clocks'])
print('roofline', {k: l['roofline'][k] for k in ('kernel','achieved','frac')})
print('e2e', l.get('e2e')); print('cpu', l.get('cpu_baseline'))
for k,v in l['kernels'].items(): print('  ',k, round(v['ms'],1), v['launches'], round(v['GBps'] or 0), round(v['share'],3))
print(json.dumps(l.get('kernel_rooflines'), indent=0)[:1500])
print(json.dumps(l.get('c5'))[:1500])
PY
