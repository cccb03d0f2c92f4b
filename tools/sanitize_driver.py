"""Small drivers of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): python tools/sanitize_driver.py <case>.  Sizes are tiny: the tools replay every
access."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

case = sys.argv[1]
torch.cuda.set_device(0)


def steps(prob, k, **kw):
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, **kw)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = torch.as_tensor(prob.u0).cuda()
    reps = [ctx.psp_step(u, u) for _ in range(k)]
    torch.cuda.synchronize()
    ctx.close()
    return [r["iterations"] for r in reps]


C4r = lambda: inputs.Problem("C4re", inputs.OperatorSpec(3, "cell_diff", (34, 19, 23), 1e-3 / 400,
                                                          field=np.exp(np.random.default_rng(5).standard_normal(34 * 19 * 23))),
                             np.random.default_rng(6).uniform(-1, 1, 34 * 19 * 23), 30, 1e-8, 3, 2, 32, 1000)
if case == "fused":          # every step one fused pass (TMA / mbarrier pipelines), the split MREP
    print(steps(C4r(), 2, fused=2, fused_kmin=0, fused_kmax=32, resident=0))
elif case == "hybrid":       # split-column steps + the fused last-step combine
    print(steps(C4r(), 2, fused=2, fused_kmin=0, fused_kmax=2, fused_split_cols=2, resident=0))
elif case == "resident":     # f2: one CTA (C1 with the accepted tridiagonal N) and a cooperative grid
    print(steps(inputs.c1(n=256, steps=2), 2, resident=2))
    print(steps(inputs.c2(n=64, d=1, steps=1), 1, resident=2))
elif case == "cg":           # f4: the fused direction pass (nx % 4 == 0) and the generic passes
    print(steps(inputs.c4(n=16, steps=2), 2, method=P.PSP_METHOD_CG))
    print(steps(inputs.c1(n=256, steps=2), 2, method=P.PSP_METHOD_CG))
elif case == "stream":       # f3: streaming MREP
    print(steps(inputs.c1(n=256, steps=2), 2, mrep_stream=1, reset_history_per_step=1, resident=0))
elif case == "c5":           # MREP (TMA + generic kernels), banded factor and solve, n = 5003
    for d in (1, 3):
        g = inputs.c5_numpy(5003, 16, d, seed=1)
        px = torch.as_tensor(g["px"]).cuda()
        py = torch.as_tensor(g["py"]).cuda()
        f = P.psp_mrep_fit_raw(px, py, d)
        st, lu = P.psp_banded_factor_raw(f["bands"], d)
        z = P.psp_banded_solve_raw(lu, d, torch.as_tensor(g["v"]).cuda())
        torch.cuda.synchronize()
        print(d, f["gate_accepted"], st, float(z.abs().max()))
else:
    raise SystemExit(f"unknown case {case}")
