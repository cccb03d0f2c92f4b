"""GPU parity of f4, PSP-CG (readings R27-R31), against the oracle's orc_pcg and
its CG time-step driver on the same seeded inputs.  Runs on a B200 only."""
import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

pytestmark = pytest.mark.gpu

T4_FLOOR = 1e-11     # x beta_0, as GMRES's first cycle (T4)
T4_ENV = 128.0       # x the oracle's own response to a 1e-15 perturbation of x0 (CG has no
                     # restarts: rounding differences grow along the whole iteration)


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


def cg_env(orc, prob, b, N_used, ho):
    """The oracle CG's own response to a 1e-15 relative perturbation of x0 (running max of the
    relative change of R(k)) and its solution change."""
    lu = None
    if N_used is not None:
        st, lu = orc.banded_lu(N_used, prob.d)
        assert st == orc.OK
    x0 = b * (1.0 + 1e-15 * np.random.default_rng(11).standard_normal(len(b)))
    eps = prob.tol * np.linalg.norm(b)
    rp = orc.pcg(prob.op, b, x0, eps, prob.restart * prob.max_cycles, d=prob.d, lu=lu)
    hp = rp["resid_hist"]
    L = min(len(hp), len(ho))
    env = np.maximum.accumulate(np.abs(hp[:L] - ho[:L]) / np.maximum(ho[:L], 1e-300))
    env = np.concatenate([env, np.full(max(0, len(ho) - L), env[-1] if L else 1.0)])
    return env, rp["x"]


def compare_cg(gr, o, ho, env, u_g, u_o, dx, s):
    assert abs(gr["iterations"] - o["iterations"]) <= 1, (s, gr["iterations"], o["iterations"])   # T5
    assert gr["converged"] == 1 and o["converged"] == 1
    assert gr["matvecs"] == gr["iterations"] + 1
    hg = gr["resid_history"]
    L = min(len(hg), len(ho))
    b0 = gr["r0"]
    tol = 1e-8 * ho[:L] + T4_FLOOR * b0 + T4_ENV * env[:L] * ho[:L]                       # T4
    q = np.abs(hg[:L] - ho[:L]) / tol
    w = int(np.argmax(q)) if L else 0
    assert np.all(q <= 1), (s, q[w], w, hg[max(0, w - 2):w + 3], ho[max(0, w - 2):w + 3])
    assert gr["final_resid_true"] <= 1.05 * gr["eps"]
    err = np.linalg.norm(u_g - u_o)
    if gr["iterations"] == o["iterations"]:                                                 # T6
        assert err <= max(1e-9 * np.linalg.norm(u_o), T4_ENV * dx), (s, err, dx)


CASES = [
    ("C1", lambda: inputs.c1(steps=3), 3),                                   # 1-D: generic passes, N accepted
    ("C2-64-d1", lambda: inputs.c2(n=64, d=1, steps=2), 2),                  # 2-D: generic passes
    ("C4-16", lambda: inputs.c4(n=16, steps=2), 2),                          # 3-D nx % 4 == 0: fused direction pass
    ("C4-ragged", lambda: inputs.Problem("C4r", inputs.OperatorSpec(3, "cell_diff", (22, 17, 13), 1e-3 / 400,
                                                                     field=np.exp(np.random.default_rng(2).standard_normal(22 * 17 * 13))),
                                         np.random.default_rng(3).uniform(-1, 1, 22 * 17 * 13), 30, 1e-8, 3, 2, 32, 1000), 2),
    ("C4-march4", lambda: inputs.Problem("C4m", inputs.OperatorSpec(3, "cell_diff", (36, 20, 27), 1e-3 / 400,
                                                                     field=np.exp(np.random.default_rng(4).standard_normal(36 * 20 * 27))),
                                         np.random.default_rng(5).uniform(-1, 1, 36 * 20 * 27), 30, 1e-8, 3, 2, 32, 1000), 2),
]


@pytest.mark.parametrize("name,mk,steps", CASES, ids=[c[0] for c in CASES])
def test_cg_lockstep_parity(torch, P, orc, name, mk, steps):
    """Each time step on identical inputs: the GPU CG solves from the oracle's u^s with the oracle's
    N_s (installed through psp_set_bands), compared by T4-T6; the GPU's own MREP + symmetrisation
    + SPD gate on the oracle's probe ring agrees with the oracle's decision."""
    prob = mk()
    n = prob.op.rows
    drv = orc.Driver(prob.op, n, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max, method=orc.METHOD_CG)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, method=P.PSP_METHOD_CG)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = prob.u0.copy()
    for s in range(steps):
        r = drv.step(u)
        acc = ctx.psp_set_bands(None if r["N_used"] is None else dev(torch, r["N_used"]))
        assert acc == (r["N_used"] is not None)
        b = dev(torch, u)
        x = torch.empty_like(b)
        gr = ctx.psp_solve(b, b, x)
        env, xp = cg_env(orc, prob, u, r["N_used"], r["resid_hist"])
        compare_cg(gr, r["solve"], r["resid_hist"], env, x.cpu().numpy(), r["u"], np.linalg.norm(xp - r["u"]), s)
        u = r["u"]
    ctx.close()


def test_cg_free_running_c1(torch, P, orc):
    """The whole CG driver on the GPU (its own probes, fit, symmetric part, gate) vs the oracle's:
    step 1 (N = I) to T4-T6, later steps to T5 with the same gate decisions, and the fitted
    interior rows of N_s equal to A's (the C1 operator is exactly tridiagonal, PN4)."""
    prob = inputs.c1()
    r = orc.time_steps(prob.op, prob.u0, prob.steps, prob.restart, prob.max_cycles, prob.tol, prob.d, prob.m_max,
                       method=orc.METHOD_CG)
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, method=P.PSP_METHOD_CG)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    u = dev(torch, prob.u0)
    reps = [ctx.psp_step(u, u) for _ in range(prob.steps)]
    for s, (gr, orr) in enumerate(zip(reps, r["reports"])):
        o = orr["solve"]
        assert abs(gr["iterations"] - o["iterations"]) <= 1, (s, gr["iterations"], o["iterations"])
        assert gr["converged"] == 1 and gr["final_resid_true"] <= 1.05 * gr["eps"]
        assert gr["precond_identity"] == int(orr["precond_was_identity"])
        assert bool(gr["mrep_gate_accepted"]) == orr["mrep"]["gate_accepted"]
    assert reps[1]["precond_identity"] == 0 and reps[1]["iterations"] <= 5
    bands, ident = ctx.psp_get_bands()
    rr = 1e-3 * 1025.0 ** 2
    ref = np.array([-rr, 1 + 2 * rr, -rr])[:, None]
    assert not ident and np.max(np.abs(bands.cpu().numpy()[:, 2:-2] - ref)) <= 1e-9 * (1 + 2 * rr)
    kappa = 1 + 4 * rr
    assert np.linalg.norm(u.cpu().numpy() - r["u"]) <= kappa * 2 * prob.tol * np.linalg.norm(r["u"]) * prob.steps
    # the probe ring holds unit-norm (p, A p) pairs (R28), plus each step's (x0, A x0) probe
    cnt, slots, PX, PY = ctx.psp_ring_view()
    nrm = PX.norm(dim=1).cpu().numpy()
    assert np.sum(~np.isclose(nrm, 1.0, rtol=1e-12)) <= prob.steps
    ctx.close()


def test_cg_full_size_128(torch, P, orc):
    """C4 recipe at 128^3 (2^21 rows, the bench's fused direction pass): the first time step of
    PSP-CG (N = I) against the oracle's CG, T4-T6."""
    prob = inputs.c4(n=128, steps=1)
    b = prob.u0
    eps = prob.tol * np.linalg.norm(b)
    o = orc.pcg(prob.op, b, b, eps, prob.restart * prob.max_cycles, d=prob.d)
    env, xp = cg_env(orc, prob, b, None, o["resid_hist"])
    opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, method=P.PSP_METHOD_CG)
    ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
    bt = dev(torch, b)
    x = torch.empty_like(bt)
    gr = ctx.psp_solve(bt, bt, x)
    compare_cg(gr, o["report"], o["resid_hist"], env, x.cpu().numpy(), o["x"], np.linalg.norm(xp - o["x"]), 0)
    ctx.close()


def test_cg_determinism(torch, P):
    prob = inputs.c4(n=16, steps=1)
    outs = []
    for _ in range(2):
        opts = P.default_opts(max_cycles=prob.max_cycles, m_max=prob.m_max, method=P.PSP_METHOD_CG)
        ctx = P.Context(prob.op, d=prob.d, restart=prob.restart, tol=prob.tol, opts=opts)
        u = dev(torch, prob.u0)
        rep = ctx.psp_step(u, u)
        outs.append((u.cpu().numpy(), rep["resid_history"].copy()))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
