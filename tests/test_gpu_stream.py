"""GPU parity of f3, the streaming MREP ("obtained progressively"; R32-R33):
every recorded probe is added to the rows' lagged sums as it is produced and the fit reads only
the sums.  Compared with the oracle's literal Algorithm 2 on the same probes (the window of every
probe since the previous fit = the oracle's ring with reset_history and no capacity limit)."""
import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

pytestmark = pytest.mark.gpu


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


def dev(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("d,m", [(1, 6), (2, 19), (3, 40), (4, 12)])
def test_streamed_fit_matches_algorithm2(torch, P, orc, d, m):
    """m probes recorded through psp_matvec(record) (more than the ring holds when m > m_max):
    the streamed fit equals Alg.2 on all m probes (T3, per-row Gram conditioning)."""
    from test_gpu_parity import gram_cond2
    op = inputs.OperatorSpec(3, "cell_diff", (24, 11, 7), 2e-3,
                             field=np.exp(np.random.default_rng(d).standard_normal(24 * 11 * 7)))
    n = op.rows
    opts = P.default_opts(m_max=8, mrep_stream=1, gate=0)
    ctx = P.Context(op, d=d, restart=4, tol=1e-8, opts=opts)
    rng = np.random.default_rng(10 + d)
    px = rng.standard_normal((m, n))
    py = np.stack([orc.matvec(op, x) for x in px])
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for x in px:
        ctx.psp_matvec(dev(torch, x), y, record=True)
    rep = ctx.psp_mrep_fit()
    assert rep["mrep_ran"] == 1
    bands, ident = ctx.psp_get_bands()
    g = bands.cpu().numpy()
    r = orc.mrep(px, py, d)
    k2 = gram_cond2(px, d)
    scale = np.maximum(np.abs(r["bands"]).max(axis=0), 1e-300)
    err = np.abs(g - r["bands"]).max(axis=0) / scale
    P_ = 2 * d + 2
    tol = np.maximum(np.where(k2 <= 1e5, 1e-10, 8 * P_ * 2.0 ** -53 * np.where(np.isfinite(k2), k2, 1e300)), 1e-10)
    interior = (r["row_kind"] == orc.ROW_INTERIOR)
    assert np.all(err[interior] <= tol[interior]), np.max(err[interior] / tol[interior])
    bnd = r["row_kind"] == orc.ROW_BOUNDARY          # R33: one-pass centred moments
    assert np.all(err[bnd] <= 1e-9), np.max(err[bnd])
    assert rep["mrep_rows_ridge"] == r["rows_ridge"]
    # the window restarts after a fit: fewer than 2d+2 new probes -> SAMPLES, N unchanged
    ctx.psp_matvec(dev(torch, px[0]), y, record=True)
    rep2 = ctx.psp_mrep_fit()
    assert rep2["mrep_status"] == P.PSP_E_SAMPLES
    ctx.close()


@pytest.mark.parametrize("mode", ["split", "ring"])
def test_streaming_driver_c1(torch, P, orc, mode):
    """C1 through psp_step with the streaming fit: the oracle driver with the per-step window
    (reset_history, unbounded ring); same iteration counts (T5), gate decisions, and the fitted
    interior rows equal to A's (PN4 closed form)."""
    prob = inputs.c1()
    kw = dict(fused=0) if mode == "split" else dict(fused=2)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, mrep_stream=1, reset_history_per_step=1,
                          resident=0, **kw)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = dev(torch, prob.u0)
    reps = [ctx.psp_step(u, u) for _ in range(prob.steps)]
    r = orc.time_steps(prob.op, prob.u0, prob.steps, prob.restart, prob.max_cycles, prob.tol, prob.d, 4096,
                       reset_history=True)
    for s, (gr, orr) in enumerate(zip(reps, r["reports"])):
        assert abs(gr["iterations"] - orr["solve"]["iterations"]) <= 1, (s, gr["iterations"], orr["solve"]["iterations"])
        assert gr["converged"] == 1
        assert gr["precond_identity"] == int(orr["precond_was_identity"])
        assert bool(gr["mrep_gate_accepted"]) == orr["mrep"]["gate_accepted"]
    bands, ident = ctx.psp_get_bands()
    rr = 1e-3 * 1025.0 ** 2
    ref = np.array([-rr, 1 + 2 * rr, -rr])[:, None]
    if not ident:
        assert np.max(np.abs(bands.cpu().numpy()[:, 1:-1] - ref)) <= 1e-9 * (1 + 2 * rr)
    ctx.close()
