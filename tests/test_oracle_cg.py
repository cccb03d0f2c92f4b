"""Pins of the f4 oracle: PSP with conjugate gradients ("can be readily applied to all
Krylov subspace methods"; readings R27-R31 of DESIGN.md).

Independent checks: the dense solve, finite termination on a matrix with three distinct
eigenvalues, the Galerkin optimality of every iterate (x_k minimises the A-norm error over the
preconditioned Krylov space, built here with numpy from a dense A), an exact preconditioner,
probe accounting, the symmetric part N_s against a dense transpose, the SPD gate, and the
closed-form implicit-Euler decay of a sine mode through the CG driver.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense(orc, op):
    n = op.rows
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        A[:, j] = orc.matvec(op, e)
    return A


def dense_bands(bands, d):
    n = bands.shape[1]
    N = np.zeros((n, n))
    for o in range(2 * d + 1):
        for i in range(n):
            j = i + o - d
            if 0 <= j < n:
                N[i, j] = bands[o, i]
    return N


def spd_cases():
    rng = np.random.default_rng(3)
    return [
        ("c1-64", inputs.OperatorSpec(1, "const_diff", (64,), 1e-3)),
        ("c2-12", inputs.OperatorSpec(2, "const_diff", (12, 9), 3e-3)),
        ("c4-6", inputs.OperatorSpec(3, "cell_diff", (6, 5, 4), 2e-3, field=np.exp(rng.standard_normal(120)))),
    ]


@pytest.mark.parametrize("name,op", spd_cases(), ids=[c[0] for c in spd_cases()])
def test_pcg_matches_dense_solve(orc, name, op):
    A = dense(orc, op)
    assert np.allclose(A, A.T, atol=1e-12 * np.abs(A).max())          # the SPD configs (O1)
    b = np.random.default_rng(1).standard_normal(op.rows)
    xs = np.linalg.solve(A, b)
    eps = 1e-12 * np.linalg.norm(b)
    r = orc.pcg(op, b, np.zeros_like(b), eps, 10 * op.rows)
    assert r["report"]["converged"] == 1
    # ||x - x*|| <= ||A^-1|| ||b - A x|| and ||A^-1|| <= 1 for A = I + dt K, K >= 0
    assert np.linalg.norm(r["x"] - xs) <= 1.5 * max(r["report"]["final_resid_true"], eps)
    assert r["report"]["final_resid_true"] <= 1.01 * eps + 1e-14 * np.linalg.norm(b) * np.abs(A).max()


def test_three_distinct_eigenvalues_terminate(orc):
    # CG terminates in at most (number of distinct eigenvalues) steps in exact arithmetic
    n = 30
    diag = np.tile([1.0, 2.0, 5.0], n // 3)
    op = inputs.dia_operator(diag[None, :], 0)
    b = np.random.default_rng(2).standard_normal(n)
    r = orc.pcg(op, b, np.zeros(n), 1e-12 * np.linalg.norm(b), 50)
    assert r["report"]["converged"] == 1 and r["report"]["iterations"] <= 3


@pytest.mark.parametrize("precond", [False, True])
def test_galerkin_optimality_of_every_iterate(orc, precond):
    """CG with an SPD M: x_k = x0 + K_k y minimises ||x - x*||_A over the Krylov space
    K_k = span{M^-1 r0, (M^-1 A) M^-1 r0, ...}, i.e. y solves (K'AK) y = K' r0.  The optimum is
    formed here by numpy on a dense A and a dense M; the oracle's x after exactly k iterations
    must equal it."""
    op = spd_cases()[2][1]
    A = dense(orc, op)
    n = op.rows
    b = np.random.default_rng(5).standard_normal(n)
    x0 = 0.1 * np.random.default_rng(6).standard_normal(n)
    lu = None
    Minv = np.eye(n)
    if precond:
        d = 1
        g = inputs.c5_numpy(n, 4, d, seed=9)
        Ns = orc.sym_bands(g["bands"], d)
        assert orc.gate_spd(Ns, d)
        st, lu = orc.banded_lu(Ns, d)
        assert st == orc.OK
        Minv = np.linalg.inv(dense_bands(Ns, d))
    r0 = b - A @ x0
    K = [Minv @ r0]
    for k in range(1, 7):
        res = orc.pcg(op, b, x0, 0.0, k, d=1, lu=lu)
        assert res["report"]["iterations"] == k
        Kk = np.stack(K, axis=1)
        y = np.linalg.solve(Kk.T @ A @ Kk, Kk.T @ r0)
        xopt = x0 + Kk @ y
        e = res["x"] - xopt
        assert np.sqrt(e @ A @ e) <= 1e-9 * np.sqrt(xopt @ A @ xopt), k
        # R(k) is the recursive residual of x_k: equals ||b - A x_opt|| to rounding
        assert res["resid_hist"][-1] == pytest.approx(np.linalg.norm(b - A @ xopt), rel=1e-7)
        K.append(Minv @ (A @ K[-1]))


def test_identity_and_exact_preconditioner(orc):
    n = 40
    op = inputs.dia_operator(np.ones((1, n)), 0)
    b = np.arange(1.0, n + 1)
    r = orc.pcg(op, b, np.zeros(n), 1e-12, 10)
    assert r["report"]["iterations"] == 1 and np.allclose(r["x"], b, rtol=0, atol=1e-13)
    # M = A (the C1 operator is exactly tridiagonal): z0 = A^-1 r0 -> one iteration
    c1 = inputs.OperatorSpec(1, "const_diff", (n,), 1e-3)
    A = dense(orc, c1)
    bands = np.zeros((3, n))
    for o in range(3):
        for i in range(n):
            j = i + o - 1
            if 0 <= j < n:
                bands[o, i] = A[i, j]
    st, lu = orc.banded_lu(bands, 1)
    b2 = np.random.default_rng(0).standard_normal(n)
    r = orc.pcg(c1, b2, np.zeros(n), 1e-10 * np.linalg.norm(b2), 10, d=1, lu=lu)
    assert r["report"]["iterations"] == 1
    assert np.linalg.norm(r["x"] - np.linalg.solve(A, b2)) <= 1e-10 * np.linalg.norm(b2)


def test_probe_accounting(orc):
    op = spd_cases()[0][1]
    n = op.rows
    ring = orc.Ring(n, 256)
    b = np.random.default_rng(4).standard_normal(n)
    r = orc.pcg(op, b, np.zeros(n), 1e-10 * np.linalg.norm(b), 200, ring=ring)
    assert ring.count == r["report"]["matvecs"] == r["report"]["iterations"] + 1
    px, py = ring.columns()
    A = dense(orc, op)
    assert np.allclose(py, px @ A.T, rtol=0, atol=1e-12 * np.abs(py).max())     # y = A x (R28)
    assert np.array_equal(px[0], np.zeros(n))                                     # the x0 probe


@pytest.mark.parametrize("d", [1, 2, 3])
def test_sym_bands_is_dense_symmetric_part(orc, d):
    n = 23
    bands = np.random.default_rng(d).uniform(-1, 1, (2 * d + 1, n))
    inputs._mask_outside(bands, d)
    N = dense_bands(bands, d)
    S = dense_bands(orc.sym_bands(bands, d), d)
    assert np.array_equal(S, 0.5 * (N + N.T))


def test_gate_spd(orc):
    d, n = 1, 10
    bands = np.zeros((3, n))
    bands[0, 1:] = -0.4
    bands[2, :-1] = -0.4
    bands[1] = 1.0
    assert orc.gate_spd(bands, d)                  # dominant, positive diagonal -> SPD
    neg = bands.copy()
    neg[1, 4] = -1.0
    assert orc.gate_dominant(neg, d) and not orc.gate_spd(neg, d)
    weak = bands.copy()
    weak[1, 4] = 0.8
    assert not orc.gate_spd(weak, d)


@pytest.mark.parametrize("k", [1, 7, 300])
def test_cg_driver_sine_mode_decay(orc, k):
    # the closed-form implicit-Euler factor of a sine mode (PN5 golden values) through the CG driver
    g = json.load(open(os.path.join(GOLD, "implicit_euler_decay.json")))["c1_grid"]
    p = inputs.c1()
    x = np.arange(1, 1025) / 1025.0
    u0 = np.sin(k * np.pi * x)
    r = orc.time_steps(p.op, u0, 1, restart=30, max_cycles=10, tol=1e-10, d=1, m_max=64, method=orc.METHOD_CG)
    f = g["factors"][g["modes"].index(k)]
    assert r["reports"][0]["solve"]["converged"] and r["reports"][0]["solve"]["iterations"] <= 5
    assert np.max(np.abs(r["u"] - f * u0)) <= 1e-12


def test_cg_driver_c1_psp_active(orc):
    # C1 with CG: step 1 plain CG, the fitted N (symmetrised, SPD-gated) accepted for step 2,
    # which then converges in a handful of iterations (A N_s^-1 = I + low rank near the ends)
    p = inputs.c1()
    r = orc.time_steps(p.op, p.u0, 3, p.restart, p.max_cycles, p.tol, p.d, p.m_max, method=orc.METHOD_CG)
    reps = r["reports"]
    assert all(s["solve"]["converged"] for s in reps)
    assert reps[0]["precond_was_identity"] and not reps[1]["precond_was_identity"]
    assert reps[1]["solve"]["iterations"] <= 5 < reps[0]["solve"]["iterations"]
    rr = 1e-3 * 1025.0 ** 2
    assert np.max(np.abs(r["bands"][:, 2:-2] - np.array([-rr, 1 + 2 * rr, -rr])[:, None])) <= 1e-9 * (1 + 2 * rr)
    # each step solves the implicit-Euler system to tol: compare with the GMRES driver's u
    g = orc.time_steps(p.op, p.u0, 3, p.restart, p.max_cycles, p.tol, p.d, p.m_max)
    kappa = 1 + 4 * rr
    assert np.linalg.norm(r["u"] - g["u"]) <= kappa * 2 * p.tol * np.linalg.norm(g["u"]) * 3
