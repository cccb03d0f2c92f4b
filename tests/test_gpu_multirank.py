"""The multi-rank path (slab decomposition, halo exchange, all-reduced Arnoldi scalars,
partitioned MREP and banded solve) on ONE B200 through the loopback communicator: each rank is a
context driven by its own host thread and stream; collectives meet at a host barrier (no kernel
waits on another rank).  Results are compared with the single-rank GPU path and the oracle."""
import threading

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


def run_ranks(P, nranks, fn):
    """fn(rank, comm) in nranks threads; returns the per-rank results (re-raises failures)."""
    comms = P.psp_comm_loopback_create(nranks)
    out = [None] * nranks
    err = [None] * nranks

    def body(r):
        try:
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        P.psp_comm_destroy(c)
    for e in err:
        if e is not None:
            raise e
    return out


def multi_steps(torch, P, prob, nranks, steps, opts_kw=None):
    def fn(rank, comm):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, **(opts_kw or {}))
            ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts, stream=s,
                            comm=comm, nranks=nranks, rank=rank)
            u = torch.as_tensor(prob.u0[ctx.row0:ctx.row0 + ctx.n]).cuda()
            reps = [ctx.psp_step(u, u) for _ in range(steps)]
            bands, ident = ctx.psp_get_bands()
            s.synchronize()
            res = dict(u=u.cpu().numpy(), reps=reps, bands=bands.cpu().numpy(), ident=ident, row0=ctx.row0)
            ctx.close()
        return res
    parts = run_ranks(P, nranks, fn)
    u = np.concatenate([p["u"] for p in parts])
    bands = np.concatenate([p["bands"] for p in parts], axis=1)
    return dict(u=u, parts=parts, reps=parts[0]["reps"], bands=bands, ident=parts[0]["ident"])


def single_steps(torch, P, prob, steps, opts_kw=None):
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, **(opts_kw or {}))
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = torch.as_tensor(prob.u0).cuda()
    reps = [ctx.psp_step(u, u) for _ in range(steps)]
    bands, ident = ctx.psp_get_bands()
    out = dict(u=u.cpu().numpy(), reps=reps, bands=bands.cpu().numpy(), ident=ident)
    ctx.close()
    return out


@pytest.mark.parametrize("nranks", [2, 3])
def test_matvec_halo_bitwise(torch, P, nranks):
    # the stencil reads the neighbour planes from the halo: bitwise equal to one rank
    prob = inputs.c4(n=14, steps=1)
    x = np.random.default_rng(0).standard_normal(prob.op.rows)
    ctx1 = P.Context(prob.op, d=3, restart=4, tol=1e-8)
    xt = torch.as_tensor(x).cuda()
    y1 = torch.empty_like(xt)
    ctx1.psp_matvec(xt, y1)
    ref = y1.cpu().numpy()

    def fn(rank, comm):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = P.Context(prob.op, d=3, restart=4, tol=1e-8, stream=s, comm=comm, nranks=nranks, rank=rank)
            xl = torch.as_tensor(x[ctx.row0:ctx.row0 + ctx.n]).cuda()
            yl = torch.empty_like(xl)
            ctx.psp_matvec(xl, yl)
            s.synchronize()
            return yl.cpu().numpy()
    y = np.concatenate(run_ranks(P, nranks, fn))
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("nranks", [2, 3])
def test_c4_multirank_vs_single(torch, P, orc, nranks):
    prob = inputs.Problem("C4s", inputs.OperatorSpec(3, "cell_diff", (20, 18, 16), 2e-4,
                                                     field=np.exp(np.random.default_rng(5).standard_normal(20 * 18 * 16))),
                          np.random.default_rng(6).uniform(-1, 1, 20 * 18 * 16), 30, 1e-8, 3, 2, 32, 1000)
    m = multi_steps(torch, P, prob, nranks, 2)
    s = single_steps(torch, P, prob, 2)
    for rm, rs in zip(m["reps"], s["reps"]):
        assert rm["cycles"] == rs["cycles"] and abs(rm["iterations"] - rs["iterations"]) <= 1
        L = min(rm["resid_len"], rs["resid_len"])
        beta = rs["beta_history"][0]
        # reductions are summed per slab then across ranks: rounding-level differences (T4 floor)
        first = min(L, prob.restart)
        assert np.all(np.abs(rm["resid_history"][:first] - rs["resid_history"][:first])
                      <= 1e-8 * rs["resid_history"][:first] + 1e-10 * beta)
        assert rm["final_resid_true"] <= 1.05 * rm["eps"]
        assert bool(rm["mrep_gate_accepted"]) == bool(rs["mrep_gate_accepted"])
    # every rank reports the same thing
    for p in m["parts"][1:]:
        assert [r["iterations"] for r in p["reps"]] == [r["iterations"] for r in m["reps"]]
    # against the oracle: both solve the same implicit-Euler steps to tol
    r = orc.time_steps(prob.op, prob.u0, 2, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max)
    # A = I + dt K with K symmetric positive semi-definite, so ||A^-1|| <= 1 and two solutions
    # whose residuals are each below tol ||b|| differ by <= 2 tol ||b|| per step; the factor
    # ||A|| (Gershgorin) is slack for residual estimates vs true residuals
    h = 1.0 / 21
    normA = 1 + 12 * prob.op.dt * prob.op.field.max() / h ** 2
    assert np.linalg.norm(m["u"] - r["u"]) <= 2 * 2 * prob.tol * normA * np.linalg.norm(prob.u0)
    assert abs(m["reps"][0]["iterations"] - r["reports"][0]["solve"]["iterations"]) <= 1


@pytest.mark.parametrize("nranks", [2, 4])
def test_c1_multirank_banded_path(torch, P, orc, nranks):
    # 1-D C1: the fitted tridiagonal N is accepted -> partitioned MREP (halo rows), the gate on
    # all-reduced statistics, the partitioned banded LU and the two-pass look-back solve
    prob = inputs.c1(steps=3)
    m = multi_steps(torch, P, prob, nranks, 3)
    r = orc.time_steps(prob.op, prob.u0, 3, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max)
    for rm, ro in zip(m["reps"], r["reports"]):
        assert rm["cycles"] == ro["solve"]["cycles"]
        assert abs(rm["iterations"] - ro["solve"]["iterations"]) <= 1
        assert rm["precond_identity"] == int(ro["precond_was_identity"])
        assert bool(rm["mrep_gate_accepted"]) == ro["mrep"]["gate_accepted"]
    assert m["reps"][1]["precond_identity"] == 0 and m["reps"][1]["iterations"] <= 3
    rr = 1e-3 * 1025.0 ** 2
    ref = np.array([-rr, 1 + 2 * rr, -rr])[:, None]
    assert np.max(np.abs(m["bands"][:, 1:-1] - ref)) <= 1e-9 * (1 + 2 * rr)
    kappa = 1 + 4 * rr
    assert np.linalg.norm(m["u"] - r["u"]) <= kappa * 2 * prob.tol * np.linalg.norm(r["u"]) * 1.1


@pytest.mark.parametrize("nranks,d", [(2, 1), (3, 2), (2, 4)])
def test_banded_precond_multirank(torch, P, orc, nranks, d):
    # install the same dominant banded N on 1 and on nranks ranks; N^-1 v must agree (T2)
    n = 3000 + 7
    g5 = inputs.c5_numpy(n, 2 * d + 2, d, seed=4)
    bands, v = g5["bands"], g5["v"]
    op = inputs.OperatorSpec(1, "const_diff", (n,), 1e-6)
    st, lu = orc.banded_lu(bands, d)
    z_ref = orc.banded_lu_solve(lu, d, v)

    def fn(rank, comm):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = P.Context(op, d=d, restart=4, tol=1e-8, stream=s, comm=comm, nranks=nranks, rank=rank)
            bl = torch.as_tensor(np.ascontiguousarray(bands[:, ctx.row0:ctx.row0 + ctx.n])).cuda()
            assert ctx.psp_set_bands(bl)
            vl = torch.as_tensor(v[ctx.row0:ctx.row0 + ctx.n]).cuda()
            zl = torch.empty_like(vl)
            ctx.psp_precond_apply(vl, zl)
            s.synchronize()
            return zl.cpu().numpy()
    z = np.concatenate(run_ranks(P, nranks, fn))
    assert np.linalg.norm(z - z_ref) <= 1e-12 * np.linalg.norm(z_ref)


FUSED_MODES = {"fused": dict(fused=2, fused_kmin=0, fused_kmax=32, resident=0),
               "ring": dict(fused=2, resident=0),
               "hybrid": dict(fused=2, fused_kmin=0, fused_kmax=2, fused_split_cols=2, resident=0)}


@pytest.mark.parametrize("mode", list(FUSED_MODES))
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("case", ["C4s", "C2s"])
def test_fused_ring_on_slabs(torch, P, orc, mode, nranks, case):
    """The ring-resident fused / split-column passes on z-slabs (y-slabs in 2-D): every ring column
    carries ghost planes, refreshed after each pass by one plane exchange each way, so a sharded
    Arnoldi step streams the same bytes per row as one GPU's.  Against the single-rank run of the
    same mode: T5, the first cycle to T4's floor, the true residual; and against the oracle."""
    if case == "C4s":
        prob = inputs.Problem("C4s", inputs.OperatorSpec(3, "cell_diff", (20, 18, 16), 2e-4,
                                                         field=np.exp(np.random.default_rng(5).standard_normal(20 * 18 * 16))),
                              np.random.default_rng(6).uniform(-1, 1, 20 * 18 * 16), 30, 1e-8, 3, 2, 32, 1000)
    else:
        prob = inputs.c2(n=64, d=1, steps=2)
    kw = FUSED_MODES[mode]
    m = multi_steps(torch, P, prob, nranks, 2, kw)
    s = single_steps(torch, P, prob, 2, kw)
    for st, (rm, rs) in enumerate(zip(m["reps"], s["reps"])):
        assert abs(rm["iterations"] - rs["iterations"]) <= 1
        assert rm["final_resid_true"] <= 1.05 * rm["eps"]
        assert bool(rm["mrep_gate_accepted"]) == bool(rs["mrep_gate_accepted"])
        if st > 0:      # later steps start from slightly different u (T5 only, as free-running parity)
            continue
        L = min(rm["resid_len"], rs["resid_len"], prob.restart)
        beta = rs["beta_history"][0]
        dR = np.abs(rm["resid_history"][:L] - rs["resid_history"][:L])
        q = dR / (1e-8 * rs["resid_history"][:L] + 1e-11 * beta)           # T4, the first cycle
        w = int(np.argmax(q))
        assert np.all(q <= 1), (w, q[w], rm["resid_history"][max(0, w - 2):w + 3], rs["resid_history"][max(0, w - 2):w + 3])
    for p in m["parts"][1:]:
        assert [r["iterations"] for r in p["reps"]] == [r["iterations"] for r in m["reps"]]
    r = orc.time_steps(prob.op, prob.u0, 2, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max)
    assert abs(m["reps"][0]["iterations"] - r["reports"][0]["solve"]["iterations"]) <= 1
    assert np.linalg.norm(m["u"] - s["u"]) <= 4 * prob.tol * np.linalg.norm(prob.u0) * 50
