"""march4s (PSP_MARCH4S=BY) against march4: bitwise equal outputs on C4-like grids (ragged y
blocks, record copies), and per-variant times at 512^3 (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P

for dims in ((64, 37, 20), (128, 50, 9), (512, 512, 512)):
    nx, ny, nz = dims
    fld = np.exp(np.random.default_rng(1).standard_normal(nx * ny * nz))
    for kind in ("cell_diff", "const_diff"):
        op = inputs.OperatorSpec(3, kind, dims, 1e-3 / 400, field=fld if kind != "const_diff" else None)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = P.Context(op, d=3, restart=30, tol=1e-8, opts=P.default_opts(m_max=4), stream=s)
            x = torch.randn(nx * ny * nz, dtype=torch.float64, device="cuda")
            outs = {}
            for var in ("0", "6", "14"):
                os.environ["PSP_MARCH4S"] = var
                y = torch.empty_like(x)
                ctx.psp_matvec(x, y, record=False)
                torch.cuda.synchronize()
                outs[var] = y.clone()
                if dims[0] == 512:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    for _ in range(3):
                        ctx.psp_matvec(x, y, record=False)
                    e0.record(s)
                    for _ in range(20):
                        ctx.psp_matvec(x, y, record=False)
                    e1.record(s)
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / 20
                    print(f"{kind} {dims} march4s={var}: {ms:.3f} ms  {24 * x.numel() / ms / 1e6:.0f} GB/s", flush=True)
            os.environ["PSP_MARCH4S"] = "0"
            for var in ("6", "14"):
                eq = torch.equal(outs["0"], outs[var])
                print(f"{kind} {dims} march4s={var} bitwise == march4: {eq}", flush=True)
                assert eq
        ctx.close()
        del x
        torch.cuda.empty_cache()
