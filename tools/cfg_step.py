"""Time-step timings of a BASELINE config (C1/C2/C3/C4) with the ring/fused path on or off.

  python tools/cfg_step.py c3 [steps=3] [fused=1]      (prints ms per step and iterations)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fused = int(sys.argv[3]) if len(sys.argv) > 3 else 1
prob = getattr(inputs, name)()
opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, fused=fused)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=s)
    u = torch.as_tensor(prob.u0).cuda()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
its = []
e0.record(s)
for _ in range(steps):
    its.append(ctx.psp_step(u, u)["iterations"])
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
n = prob.op.rows
print(f"{name} fused={fused}: {ms:.1f} ms/step, iterations {its}, {n * sum(its) / (ms * steps / 1e3):.3e} unknown-it/s")
ctx.close()
