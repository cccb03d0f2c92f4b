#!/bin/bash
# r02o: the -m gpu suite + smoke, the full bench line, then ncu captures of the final build.s
# factor and MREP kernels (tools/profile_r02o.sh).  Output: gpurun_out/r02o/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02o
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02o/bench.json"))
print({k: d[k] for k in ("value", "ms_per_step", "gpu_launches")}, "roofline", d["roofline"]["frac"], "clocks", d["clocks"])
print("c5", json.dumps(d.get("c5"))[:800])
PY
PROF_OUT=r02o bash tools/profile_r02o.sh
