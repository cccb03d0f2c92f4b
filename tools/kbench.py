"""Per-kernel microbenchmarks through the C ABI (profiling driver; not the bench).

  python tools/kbench.py matvec [size=512] [reps=20]
  python tools/kbench.py mrep   [log2n=27] [m=32] [d=3] [reps=5]
  python tools/kbench.py solve  [log2n=27] [d=3] [reps=10]
  python tools/kbench.py mrepring [size=512] [reps=5]   (psp_mrep_fit on a C4 context's full ring)

Times with CUDA events on the launching stream (after a warm-up launch) and prints GB/s at the
algorithmic bytes of DESIGN.md section 6.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1308_5626_b200 import inputs, pspgmres as P


def timed(fn, reps, stream):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def matvec(size=512, reps=20):
    n = size
    kappa = torch.rand(n ** 3, dtype=torch.float64) + 0.5
    op = inputs.OperatorSpec(ndim=3, kind="cell_diff", n=(n, n, n), dt=1e-6, field=kappa.numpy())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = P.Context(op, d=3, restart=30, tol=1e-8, opts=P.default_opts(m_max=4), stream=s)
        x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
    ms = timed(lambda: ctx.psp_matvec(x, y, record=False), reps, s)
    print(f"matvec {size}^3: {ms:.3f} ms  {24 * n ** 3 / ms / 1e6:.0f} GB/s (24 B/row)")
    ms = timed(lambda: ctx.psp_matvec(x, y, record=True), reps, s)
    # record = matvec with the probe copy (32 B/row) + a copy of the probe to y (16 B/row)
    print(f"matvec+record {size}^3: {ms:.3f} ms  {48 * n ** 3 / ms / 1e6:.0f} GB/s (48 B/row incl. copy-out)")
    ctx.close()


def mrep(log2n=27, m=32, d=3, reps=5):
    n = 1 << log2n
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    px = torch.randn((m, n), generator=g, device="cuda", dtype=torch.float64)
    py = torch.randn((m, n), generator=g, device="cuda", dtype=torch.float64)
    scratch = P.raw_scratch(n, d)
    s = torch.cuda.current_stream()
    ms = timed(lambda: P.psp_mrep_fit_raw(px, py, d, scratch=scratch, want_kind=False), reps, s)
    b = 16 * m + 8 * (2 * d + 1)
    print(f"mrep n=2^{log2n} m={m} d={d}: {ms:.3f} ms  {n / ms / 1e6:.2f} G rows/s  {b * n / ms / 1e6:.0f} GB/s ({b} B/row)")


def solve(log2n=27, d=3, reps=10):
    n = 1 << log2n
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    bands = torch.rand((2 * d + 1, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    bands[d] = bands.abs().sum(0) + 1.0
    v = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    scratch = P.raw_scratch(n, d)
    st, lu = P.psp_banded_factor_raw(bands, d, scratch=scratch)
    z = torch.empty_like(v)
    s = torch.cuda.current_stream()
    ms = timed(lambda: P.psp_banded_solve_raw(lu, d, v, scratch=scratch, out=z), reps, s)
    b = 8 * (2 * d + 5)
    print(f"banded solve n=2^{log2n} d={d}: {ms:.3f} ms  {n / ms / 1e6:.2f} G rows/s  {b * n / ms / 1e6:.0f} GB/s ({b} B/row)")
    msf = timed(lambda: P.psp_banded_factor_raw(bands, d, scratch=scratch), 3, s)
    bf = 16 * (2 * d + 1)
    print(f"banded factor n=2^{log2n} d={d}: {msf:.3f} ms  {bf * n / msf / 1e6:.0f} GB/s ({bf} B/row)")


def mrepring(size=512, reps=5):
    prob = inputs.c4(n=size, steps=1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol,
                        opts=P.default_opts(max_cycles=2, m_max=prob.m_max), stream=s)
        b = torch.as_tensor(prob.u0).cuda()
        x = torch.zeros_like(b)
        ctx.psp_solve(b, b, x)                   # two cycles: a full probe ring
    torch.cuda.synchronize()
    ms = timed(lambda: ctx.psp_mrep_fit(), reps, s)
    n = size ** 3
    bb = 16 * prob.m_max + 8 * (2 * prob.d + 1)
    print(f"mrep ring {size}^3 m={prob.m_max} d={prob.d}: {ms:.3f} ms  {n / ms / 1e6:.2f} G rows/s  "
          f"{bb * n / ms / 1e6:.0f} GB/s ({bb} B/row)")
    ctx.close()


if __name__ == "__main__":
    what = sys.argv[1]
    args = [int(a) for a in sys.argv[2:]]
    {"matvec": matvec, "mrep": mrep, "solve": solve, "mrepring": mrepring}[what](*args)
