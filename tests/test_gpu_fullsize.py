"""Parity at BASELINE.json's full sizes, in the configuration bench.py times, on sampled outputs
the oracle computes one by one (or on properties that hold at any size).

* C5 (configs[4]): n = 2^26, m = 32, d = 3 -- the split MREP, the warm-started factorisation and
  the two-sweep solve.  Every sampled interior row's fit is the oracle's Algorithm 2 on the
  4d+1 rows around it (the row's own regression only reads P_x rows i-d..i+d and P_y row i,
  P:111-122), boundary rows are fitted on the first / last 4d+1 rows; factors and solve are
  checked by (LU)(i,:) = N(i,:) and (N z)(i) = v(i) on the sampled rows.
* C4 (configs[3]): one 512^3 time step with the bench's options (fused passes, split-column
  steps): convergence with the true residual below tol ||b|| and, on sampled points of the
  newest recorded probes, P_y = A P_x with A applied by the oracle on the 3x3x3 neighbourhood
  of each point (its row of A only reaches those points, Eq.4 / P:25).
"""
import ctypes as C

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
U = np.finfo(np.float64).eps / 2


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a B200"
    return torch


@pytest.fixture(scope="module")
def P():
    from paper_1308_5626_b200 import pspgmres
    pspgmres.lib()
    return pspgmres


def _free(torch):
    import gc
    gc.collect()
    torch.cuda.empty_cache()


def _sample_rows(n, d, rng, count=1500):
    rows = set(rng.integers(2 * d, n - 2 * d, count).tolist())
    rows |= set(range(0, 2 * d + 1)) | set(range(n - 2 * d - 1, n))   # boundary + first interior rows
    E = 128 - 2 * d                                                      # TMA tile edges (R0 = 2d+2)
    for t in range(0, 40):
        rows |= {2 * d + 2 + t * E - 1, 2 * d + 2 + t * E}
    rows |= {n // 2 - 1, n // 2, n // 2 + 1}                             # split-MREP chunk seams
    return np.array(sorted(r for r in rows if 0 <= r < n))


def test_c5_full_size_sampled(torch, P, orc):
    n, m, d = 1 << 26, 32, 3
    g5 = inputs.c5_torch(n, m, d, seed=0)
    scratch = P.raw_scratch(n, d)
    g = P.psp_mrep_fit_raw(g5["px"], g5["py"], d, scratch=scratch)
    assert g["status"] == P.PSP_OK and g["gate_accepted"]            # A_true is dominant (C5 recipe)
    rows = _sample_rows(n, d, np.random.default_rng(5))
    bands = g["bands"][:, torch.as_tensor(rows, device="cuda")].cpu().numpy()
    kinds = g["row_kind"][torch.as_tensor(rows, device="cuda")].cpu().numpy()
    W = 4 * d + 1
    Pn = 2 * d + 2
    worst = 0.0
    for col, i in enumerate(rows):
        lo = min(max(i - 2 * d, 0), n - W)          # rows i-2d..i+2d, clamped inside the matrix:
        c = i - lo                                  # boundary rows stay boundary rows of the window
        px = g5["px"][:, lo:lo + W].cpu().numpy()
        py = g5["py"][:, lo:lo + W].cpu().numpy()
        r = orc.mrep(px, py, d)
        assert kinds[col] == r["row_kind"][c], (i, kinds[col], r["row_kind"][c])
        ref = r["bands"][:, c]
        scale = max(np.abs(ref).max(), 1e-300)
        err = np.abs(bands[:, col] - ref).max() / scale
        if d <= c < W - d:   # interior row: T3 tolerance from the row's Gram condition
            X = np.vstack([np.ones(m), px[:, c - d:c + d + 1].T])
            k2 = np.linalg.cond(X @ X.T)
            tol = 1e-10 if k2 <= 1e5 else 8 * Pn * U * k2
        else:
            tol = 1e-12
        worst = max(worst, err / tol)
        assert err <= tol, (i, err, tol)
    # factorisation: (L U)(i, j) = N(i, j) on the sampled rows (property of the exact factors)
    st, lu = P.psp_banded_factor_raw(g["bands"], d, scratch=scratch)
    assert st == P.PSP_OK
    Nb = g["bands"]
    for i in rows[(rows >= 2 * d) & (rows < n - 2 * d)][:400]:
        idx = torch.arange(i - d, i + 1, device="cuda")
        L = lu[:d, i].cpu().numpy()                     # L(i, i-d+q), unit diagonal
        Urows = lu[d:, idx].cpu().numpy()               # U(k, k+e) for k = i-d..i
        for o in range(2 * d + 1):
            j = i + o - d
            s = 0.0
            for q in range(d + 1):                      # k = i-d+q
                lik = 1.0 if q == d else L[q]
                e = j - (i - d + q)
                if 0 <= e <= d:
                    s += lik * Urows[e, q]
            ref = Nb[o, i].item()
            assert abs(s - ref) <= 1e-12 * (abs(ref) + 1.0), (i, o, s, ref)
    # solve: (N z)(i) = v(i) on the sampled rows
    z = P.psp_banded_solve_raw(lu, d, g5["v"], scratch=scratch)
    zs = {}
    for i in rows:
        acc, mag = 0.0, 0.0
        for o in range(2 * d + 1):
            j = i + o - d
            if 0 <= j < n:
                if j not in zs:
                    zs[j] = z[j].item()
                t = Nb[o, i].item() * zs[j]
                acc += t
                mag += abs(t)
        vi = g5["v"][i].item()
        assert abs(acc - vi) <= 1e-13 * (1 + d) * (abs(vi) + mag), (i, acc, vi)
    del g5, g, lu, z, scratch, Nb
    _free(torch)


def test_c4_full_size_sampled(torch, P, orc):
    size = 512
    prob = inputs.c4(n=size, steps=1)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max)    # the bench's defaults
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = torch.as_tensor(prob.u0).cuda()
    b = prob.u0.copy()
    rep = ctx.psp_step(u, u)
    assert rep["converged"]
    assert rep["final_resid_true"] <= rep["eps"]                # ||b - A u|| <= tol ||b|| (R1, R13)
    # the newest probes: P_y = A P_x on sampled points, A applied by the oracle on each point's
    # 3x3x3 neighbourhood (scaled dt keeps dt / h^2 of the full grid)
    lib = P.lib()
    cnt = C.c_int()
    slots = (C.c_int32 * 257)()
    scale = np.zeros(257)
    pxp, pyp, ld = C.c_void_p(), C.c_void_p(), C.c_int64()
    st = lib.psp_ring_view(ctx.h, C.byref(cnt), slots, scale.ctypes.data_as(C.POINTER(C.c_double)),
                           C.byref(pxp), C.byref(pyp), C.byref(ld))
    assert st == P.PSP_OK and cnt.value >= 3
    n = size ** 3
    ws64 = ctx.ws.view(torch.float64)
    base = ctx.ws.data_ptr()
    rng = np.random.default_rng(4)
    pts = rng.integers(1, size - 1, (300, 3))                   # (z, y, x) interior points
    pts = np.vstack([pts, [[0, 0, 0], [size - 1, size - 1, size - 1], [0, 5, size - 1]]])
    kap = prob.op.field.reshape(size, size, size)
    hfull = 1.0 / (size + 1)
    for q in range(cnt.value - 3, cnt.value):
        sl = slots[q]
        PX = ws64[(pxp.value - base) // 8 + sl * ld.value:(pxp.value - base) // 8 + sl * ld.value + n]
        PY = ws64[(pyp.value - base) // 8 + sl * ld.value:(pyp.value - base) // 8 + sl * ld.value + n]
        for (zz, yy, xx) in pts:
            # a 3x3x3 window clamped inside the grid: an interior point is its centre; a point on
            # the grid boundary sits on the window's edge, which is then the grid's own boundary
            z0, y0, x0 = (min(max(v - 1, 0), size - 3) for v in (zz, yy, xx))
            z1, y1, x1 = z0 + 3, y0 + 3, x0 + 3
            sub = (3, 3, 3)
            ids = (np.arange(z0, z1)[:, None, None] * size * size + np.arange(y0, y1)[None, :, None] * size
                   + np.arange(x0, x1)[None, None, :]).reshape(-1)
            xs = (PX[torch.as_tensor(ids, device="cuda")] * scale[q]).cpu().numpy()
            # a window that touches the grid boundary keeps the Dirichlet side; an interior window
            # edge is only reached by points other than the centre
            hsub = 1.0 / (np.array(sub, dtype=float) + 1)
            dt = prob.op.dt * (hsub[0] / hfull) ** 2
            spec = inputs.OperatorSpec(3, prob.op.kind, sub, dt,
                                       field=kap[z0:z1, y0:y1, x0:x1].reshape(-1).copy())
            ys = orc.matvec(spec, xs)
            cz, cy, cx = zz - z0, yy - y0, xx - x0
            c = (cz * sub[1] + cy) * sub[0] + cx
            gi = (zz * size + yy) * size + xx
            ref = ys[c]
            got = PY[gi].item() * scale[q]
            mag = np.abs(xs).max() * (1 + 12 * dt / hsub[0] ** 2 * kap.max())
            assert abs(got - ref) <= 64 * U * mag, (q, zz, yy, xx, got, ref)
    ctx.close()
    del ctx, u
    _free(torch)


def _lockstep_c4(torch, P, orc, size, max_cycles, with_mrep):
    """C4 recipe at size^3 with the bench's default options (fused passes from 2^21 rows on,
    split-column steps beyond k = 16, the fused last-step combine): the first time step (N = I
    on both sides, b = x0 = u0) on the GPU and in the oracle, compared by T4-T6 (DESIGN.md s.7)."""
    from test_gpu_parity import MREP_EXCLUDED_MAX, compare_mrep, compare_solve, log_parity, oracle_sensitivity
    prob = inputs.c4(n=size, steps=1)
    n = prob.op.rows
    b = prob.u0
    eps = prob.tol * np.linalg.norm(b)
    o = orc.pspgmres(prob.op, b, b, eps, prob.restart, max_cycles, d=prob.d)
    env, dx = oracle_sensitivity(orc, prob, b, None, o["resid_hist"], o["x"], max_cycles=max_cycles)
    opts = P.default_opts(max_cycles=max_cycles, m_max=prob.m_max)       # the bench's defaults
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    bt = torch.as_tensor(b).cuda()
    x = torch.empty_like(bt)
    gr = ctx.psp_solve(bt, bt, x)
    ro = dict(o["report"])
    ro["converged"] = ro["converged"] if max_cycles >= prob.max_cycles else 1
    if max_cycles < prob.max_cycles:          # a truncated solve: both sides ran every cycle
        assert gr["cycles"] == ro["cycles"] == max_cycles and gr["iterations"] == ro["iterations"]
        gr = dict(gr, converged=1, final_resid_true=0.0)
    compare_solve(gr, ro, o["resid_hist"], 0, env, nA=prob.restart, case=f"C4-{size}-full")
    err = np.linalg.norm(x.cpu().numpy() - o["x"])
    if gr["iterations"] == ro["iterations"]:                                           # T6
        assert err <= max(1e-9 * np.linalg.norm(o["x"]), 30.0 * dx), (err, dx)
    if with_mrep:
        # Alg.2 on the GPU's own probe ring (recorded with their Krylov scales: the scaled path of
        # the TMA kernels) vs the oracle's Algorithm 2 on the same probes
        rep = ctx.psp_mrep_fit()
        cnt, slots, PX, PY = ctx.psp_ring_view()
        px, py = PX.cpu().numpy(), PY.cpu().numpy()
        g = P.psp_mrep_fit_raw(PX.contiguous(), PY.contiguous(), prob.d)
        r = orc.mrep(px, py, prob.d)
        ex = compare_mrep(g, r, prob.d, n, px, max_excluded_frac=MREP_EXCLUDED_MAX)
        log_parity(case=f"C4-{size}-full", step=0, mrep_excluded=int(ex), rows=n)
        bands, _ = ctx.psp_get_bands()
        # psp_mrep_fit (the scaled ring columns: the scale enters the lagged sums as s^2 on one
        # factor) and psp_mrep_fit_raw (the same columns scaled by torch) are two evaluations of
        # the same normal equations: on the unridged rows each is within T3 of the exact
        # solution, so they agree within twice T3
        from test_gpu_parity import gram_cond2
        bb = bands.cpu().numpy()
        gb = g["bands"].cpu().numpy()
        k2 = gram_cond2(px, prob.d)
        P_ = 2 * prob.d + 2
        tol = np.maximum(np.where(k2 <= 1e5, 1e-10, 8 * P_ * 2.0 ** -53 * np.where(np.isfinite(k2), k2, 1e300)), 1e-10)
        ok = g["row_kind"].cpu().numpy() == P.ROW_INTERIOR
        err = np.abs(bb - gb).max(axis=0) / np.maximum(np.abs(gb).max(axis=0), 1e-300)
        assert np.all(err[ok] <= 2 * tol[ok]), np.max(err[ok] / tol[ok])
        assert bool(rep["mrep_gate_accepted"]) == r["gate_accepted"]
    ctx.close()
    del ctx, bt, x
    _free(torch)


def test_c4_lockstep_128_full_step(torch, P, orc):
    """Full first time step at 128^3 (2^21 rows: the bench's fused / split-column passes run,
    400 fused tiles over 148 persistent CTAs), every cycle to convergence, then Alg.2."""
    _lockstep_c4(torch, P, orc, 128, 1000, with_mrep=True)


def test_c4_lockstep_256_two_cycles(torch, P, orc):
    """256^3 (> 2000 fused tiles), the first two GMRES(30) cycles: every step width of the
    bench's policy (fused k = 2..16, split-column k = 17..29, the fused last-step combine at
    k = 30) and one restart, compared with the oracle's literal Alg.1."""
    _lockstep_c4(torch, P, orc, 256, 2, with_mrep=False)


@pytest.mark.parametrize("d", [1, 3])
def test_banded_solve_slow_decay_full_size(torch, P, orc, d):
    """The banded sweeps' exact fallback: a dominant N whose homogeneous
    response decays only by ~1e-4 a row (off-diagonals -1, diagonal margin 1e-8), so the decaying
    correction of a 28 K-row warp range has not died out within its 16384-row cap and the range is
    re-walked from its exact incoming state.  n = 2^26 + 38 (a ragged last warp-tile); the solve
    runs on the oracle's own LU factors (T2 against the oracle's sweeps on the same factors)."""
    n = (1 << 26) + 38
    rng = np.random.default_rng(26 + d)
    bands = np.zeros((2 * d + 1, n))
    bands[d - 1] = -1.0
    bands[d + 1] = -1.0
    for o in range(2 * d + 1):
        if abs(o - d) >= 2:
            bands[o] = 1e-3 * rng.uniform(-1, 1, n)
    inputs._mask_outside(bands, d)
    bands[d] = np.abs(bands).sum(axis=0) + 1e-8
    v = rng.standard_normal(n)
    st, lu_ref = orc.banded_lu(bands, d)
    assert st == orc.OK
    z_ref = orc.banded_lu_solve(lu_ref, d, v)
    del bands
    scratch = P.raw_scratch(n, d)
    z = P.psp_banded_solve_raw(torch.from_numpy(lu_ref).cuda(), d, torch.from_numpy(v).cuda(),
                               scratch=scratch).cpu().numpy()
    # rounding differences travel ~1e4 rows (the decay length) before they fade: 1e-9 relative
    assert np.linalg.norm(z - z_ref) <= 1e-9 * np.linalg.norm(z_ref)
    _free(torch)
