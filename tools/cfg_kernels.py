"""Kernel-class table of a BASELINE config's time step (opts.timing = 2): summed CUDA-event time
per class against the step's device time -- the difference is host gaps (launch latency, the
per-step reads of R(k)).

  python tools/cfg_kernels.py c3 [steps=2]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = getattr(inputs, name)()
s = torch.cuda.Stream()
opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, timing=2)
with torch.cuda.stream(s):
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=s)
    u = torch.as_tensor(prob.u0).cuda()
    ctx.psp_step(u, u)                     # warm-up
    ctx.psp_kernel_stats(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    reps = [ctx.psp_step(u, u) for _ in range(steps)]
    e1.record(s)
torch.cuda.synchronize()
t = e0.elapsed_time(e1)
ks = ctx.psp_kernel_stats(reset=True)
tot = sum(v["ms"] for v in ks.values())
print(f"{name}: {t / steps:.2f} ms a step, iterations {[r['iterations'] for r in reps]}, kernel classes {tot / steps:.2f} ms "
      f"({100 * tot / t:.1f} %), launches {ctx.psp_launch_count()}")
for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"  {k:14s} {v['ms'] / steps:8.2f} ms  {v['launches'] // steps:6d} launches  "
              f"{v['bytes'] / (v['ms'] / 1e3) / 1e9 if v['ms'] else 0:7.0f} GB/s")
ctx.close()
