"""Time-step timings of a BASELINE config (C1/C2/C3/C4): the host-driven cycle (fused / ring /
split passes) against the device-resident solve (f2, resident.cu).

  python tools/cfg_step.py c1 [steps=5] [fused=1] [resident=1] [d=0 (config's)] [method=0|1 (CG)] [n=...]
(prints ms per step (CUDA events), the per-step iterations and unknown-iterations/s; the first
line is the config's own step count from a fresh context, so step 1 -- the long one -- counts)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fused = int(sys.argv[3]) if len(sys.argv) > 3 else 1
resident = int(sys.argv[4]) if len(sys.argv) > 4 else 1
kw = {}
if len(sys.argv) > 5 and int(sys.argv[5]) > 0:
    kw["d"] = int(sys.argv[5])
method = int(sys.argv[6]) if len(sys.argv) > 6 else 0     # 0 GMRES, 1 CG (f4)
if len(sys.argv) > 7:
    kw["n"] = int(sys.argv[7])
prob = getattr(inputs, name)(**kw)
n = prob.op.rows
opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, fused=fused, resident=resident, method=method)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=s)
    u = torch.as_tensor(prob.u0).cuda()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
its, per = [], []
e0.record(s)
for _ in range(steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    its.append(ctx.psp_step(u, u)["iterations"])
    b.record(s)
    per.append((a, b))
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
out = dict(config=name, fused=fused, resident=resident, method=method, n=n, d=prob.d, ms_per_step=ms, iterations=its,
           step_ms=[a.elapsed_time(b) for a, b in per], unknown_it_per_s=n * sum(its) / (ms * steps / 1e3),
           launches=ctx.psp_launch_count())
print(json.dumps(out))
ctx.close()
