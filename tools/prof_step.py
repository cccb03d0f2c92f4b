"""Run C4-recipe time steps at a given size (profiling driver; not the bench)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1308_5626_b200 import inputs, pspgmres as P

size = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fused = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kmax = int(sys.argv[4]) if len(sys.argv) > 4 else 30
prob = inputs.c4(n=size, steps=steps)
opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, fused=fused, fused_kmin=0, fused_kmax=kmax)
ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
u = torch.as_tensor(prob.u0).cuda()
for s in range(steps):
    r = ctx.psp_step(u, u)
    print("step", s, "iterations", r["iterations"], "converged", r["converged"], flush=True)
torch.cuda.synchronize()
