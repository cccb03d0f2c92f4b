"""Per-k Arnoldi-step times (CUDA events on the context stream) for the C4 recipe: one
cycle_begin, then psp_arnoldi_step(k) for k = 1..restart, over a few cycles; prints the median
ms per k.  Variants (KSTEP_VARIANTS="default,PSP_FUSED_TILE=1,...") set environment knobs read per launch.

  python tools/kstep.py [size=512] [cycles=3] [fused_kmin=1] [fused_kmax=30] [fused_split_cols=16]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kmin = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kmax = int(sys.argv[4]) if len(sys.argv) > 4 else 30
split_cols = int(sys.argv[5]) if len(sys.argv) > 5 else 16
prob = inputs.c4(n=size, steps=1)
s = torch.cuda.Stream()
opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, fused=1, fused_kmin=kmin, fused_kmax=kmax,
                      fused_split_cols=split_cols)
with torch.cuda.stream(s):
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=1e-30, opts=opts, stream=s)
    b = torch.as_tensor(prob.u0).cuda()
    x = torch.zeros_like(b)
torch.cuda.synchronize()
R = prob.restart
ev = [torch.cuda.Event(enable_timing=True) for _ in range(R + 2)]
variants = os.environ.get("KSTEP_VARIANTS", "default").split(",")
set_keys = set()
for var in variants:
    # variant "default" or "NAME=VAL+NAME2=VAL2" (environment knobs read per launch)
    for key in [k for k in os.environ if k.startswith("PSP_") and k != "PSP_LIB"] + list(set_keys):
        os.environ.pop(key, None)
    if var != "default":
        for kv in var.split("+"):
            name, val = kv.split("=")
            os.environ[name] = val
            set_keys.add(name)
    times = np.zeros((cycles, R + 1))
    for c in range(cycles):
        ev[0].record(s)
        ctx.psp_cycle_begin(b, x)
        ev[1].record(s)
        for k in range(1, R + 1):
            ctx.psp_arnoldi_step(k)
            ev[k + 1].record(s)
        torch.cuda.synchronize()
        ctx.psp_cycle_end(R, x)
        times[c] = [ev[i].elapsed_time(ev[i + 1]) for i in range(R + 1)]
    med = np.median(times[1:] if cycles > 1 else times, axis=0)
    print(f"{var}: total {med.sum():.2f} ms/cycle  begin {med[0]:.2f}")
    print(f"{var}: per k " + " ".join(f"{k}:{med[k]:.2f}" for k in range(1, R + 1)), flush=True)
ctx.close()
