#!/bin/bash
# r02i: the -m gpu suite + smoke, then the full bench line (default args)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${R02_OUT:-r02i}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
R02_OUT=${R02_OUT:-r02i} python - <<'PY'
import json
import os
d = json.load(open("gpurun_out/%s/bench.json" % os.environ.get("R02_OUT", "r02i")))
print({k: d[k] for k in ("value", "ms_per_step", "gpu_launches")})
print("instr", d["instrumented_region"]["ms_per_step"], "roofline", d["roofline"]["frac"], d["roofline"]["kernel"])
print("e2e", d["e2e"]["value"], "solve_only", d["solve_only"]["value"], "clocks", d["clocks"])
print("configs", json.dumps(d.get("configs"))[:1500])
PY
tail -3 $O/bench.err
