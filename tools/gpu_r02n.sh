#!/bin/bash
# r02n: the -m gpu suite + smoke, the full bench line, then ncu captures of the late-r02
# kernels and the launch list (tools/profile_r02n.sh).  Output: gpurun_out/r02n/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02n
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02n/bench.json"))
print({k: d[k] for k in ("value", "ms_per_step", "gpu_launches")}, "roofline", d["roofline"]["frac"], "clocks", d["clocks"])
print("c5", json.dumps(d.get("c5"))[:800])
PY
PROF_OUT=r02n bash tools/profile_r02n.sh
