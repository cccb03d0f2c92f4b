#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02h
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -8 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python - <<'PY'
import torch
from paper_1308_5626_b200 import inputs, pspgmres as P
for size in (128, 512):
    prob = inputs.c4(n=size, steps=1)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=P.default_opts(max_cycles=2, m_max=prob.m_max))
    b = torch.as_tensor(prob.u0).cuda(); x = torch.zeros_like(b)
    ctx.psp_solve(b, b, x)
    rep = ctx.psp_mrep_fit()
    print(size, {k: rep[k] for k in ("mrep_rows_ridge", "mrep_rows_fallback", "mrep_rows_nondominant", "mrep_gate_accepted")})
    ctx.close()
PY
