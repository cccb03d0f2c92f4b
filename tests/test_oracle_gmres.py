"""Pins of oracle O3: literal Algorithm 1 (PSPGMRES) -- PN3.

Independent checks: dense solves, brute-force Krylov least squares via numpy.linalg.lstsq,
the dense-QR residual of the Hessenberg least-squares problem, the Arnoldi relation and
orthogonality of the stored basis, the minimal-polynomial property, the Givens worked
example (golden), probe accounting.
"""
import json
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


def diag_op(values):
    values = np.asarray(values, dtype=np.float64)
    return inputs.dia_operator(values[None, :], 0)


def test_identity_one_iteration(orc):
    # A = I, b = [1,2,3], x0 = 0 -> 1 iteration, x = b
    op = diag_op(np.ones(3))
    r = orc.pspgmres(op, [1.0, 2.0, 3.0], np.zeros(3), eps=1e-14, n_A=5, n_r=2)
    assert r["report"]["iterations"] == 1 and r["report"]["converged"] == 1
    assert np.allclose(r["x"], [1, 2, 3], rtol=0, atol=1e-14)


def test_three_eigenvalues_three_iterations(orc):
    # minimal polynomial of degree 3 -> at most 3 iterations, matches a dense solve
    vals = np.tile([1.0, 2.0, 3.0], 10)
    op = diag_op(vals)
    b = np.random.default_rng(0).standard_normal(30)
    r = orc.pspgmres(op, b, np.zeros(30), eps=1e-10 * np.linalg.norm(b), n_A=10, n_r=1)
    assert r["report"]["iterations"] <= 3 and r["report"]["converged"]
    assert np.allclose(r["x"], b / vals, rtol=0, atol=1e-9)


def test_givens_345_golden(orc):
    g = json.load(open(os.path.join(GOLD, "givens_345.json")))
    # A e1 = 3 e1 + 4 e2, b = e1, x0 = 0: H(1,1) = 3, H(2,1) = 4 (pre-rotation)
    n = 4
    bands = np.zeros((3, n))
    bands[1] = 1.0
    bands[1, 0] = g["H11"]
    bands[0, 1] = g["H21"]      # A(1,0)
    op = inputs.dia_operator(bands, 1)
    b = np.zeros(n)
    b[0] = 1.0
    r = orc.pspgmres(op, b, np.zeros(n), eps=1e-300, n_A=1, n_r=1, trace=True)
    t = r["trace"]
    assert t["Hraw"][0, 0] == g["H11"] and t["Hraw"][1, 0] == g["H21"]
    assert t["H"][0, 0] == pytest.approx(g["gamma"], abs=1e-15) and t["H"][1, 0] == 0.0
    assert t["C"][0] == pytest.approx(g["C1"], abs=1e-15) and t["S"][0] == pytest.approx(g["S1"], abs=1e-15)
    assert np.allclose(t["G"], g["G_after"], rtol=0, atol=1e-15)
    assert r["resid_hist"][0] == pytest.approx(g["R1"], abs=1e-15)


def _krylov_min_residual(Aop, r0, k):
    """min_y || r0 - Aop K_k y || with K_k = [r0, Aop r0, ..., Aop^{k-1} r0] (brute force)."""
    K = [r0 / np.linalg.norm(r0)]
    for _ in range(k - 1):
        w = Aop @ K[-1]
        K.append(w / np.linalg.norm(w))
    K = np.array(K).T
    M = Aop @ K
    y, *_ = np.linalg.lstsq(M, r0, rcond=None)
    return np.linalg.norm(r0 - M @ y)


@pytest.mark.parametrize("precond", [False, True])
def test_residual_history_is_krylov_minimum(orc, precond):
    # PN3: R(k) of one cycle = brute-force minimal residual over the (right-preconditioned)
    # Krylov space A N^-1 K_k(A N^-1, r0), k <= 8
    op, _ = inputs.seven_diagonal(60, seed=2, margin=0.3)
    A = dense(orc, op)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(60)
    x0 = rng.standard_normal(60)
    lu = None
    Ninv = np.eye(60)
    if precond:
        nb = np.zeros((3, 60))
        nb[1] = np.diag(A)
        nb[0, 1:] = np.diag(A, -1)
        nb[2, :-1] = np.diag(A, 1)
        st, lu = orc.banded_lu(nb, 1)
        assert st == orc.OK
        Nd = np.diag(nb[1]) + np.diag(nb[0, 1:], -1) + np.diag(nb[2, :-1], 1)
        Ninv = np.linalg.inv(Nd)
    r = orc.pspgmres(op, b, x0, eps=1e-300, n_A=8, n_r=1, d=1, lu=lu)
    r0 = b - A @ x0
    assert r["beta_hist"][0] == pytest.approx(np.linalg.norm(r0), rel=1e-14)
    for k in range(1, 9):
        ref = _krylov_min_residual(A @ Ninv, r0, k)
        assert abs(r["resid_hist"][k - 1] - ref) <= 1e-10 * np.linalg.norm(r0), k
    # the solution formed at the cycle end is x0 + N^-1 Z: its true residual is R(8)
    assert np.linalg.norm(b - A @ r["x"]) == pytest.approx(r["resid_hist"][7], rel=1e-8)


def test_hessenberg_ls_residual_and_arnoldi_relation(orc):
    # AC7 / S:155: |G(k+1)| = dense-QR least-squares residual of beta e1 - Hbar q;
    # Arnoldi relation A V_k = V_{k+1} Hbar_k (pre-rotation); ||I - V'V|| <= 1e-10
    p = inputs.c4(n=8, steps=1)
    A = dense(orc, p.op)
    b = p.u0
    n_A = 12
    r = orc.pspgmres(p.op, b, np.zeros_like(b), eps=1e-300, n_A=n_A, n_r=1, trace=True)
    t = r["trace"]
    V, Hbar = t["V"], t["Hraw"]
    beta = r["beta_hist"][0]
    for k in range(1, n_A + 1):
        e1 = np.zeros(k + 1)
        e1[0] = beta
        q, *_ = np.linalg.lstsq(Hbar[:k + 1, :k], e1, rcond=None)
        assert abs(np.linalg.norm(e1 - Hbar[:k + 1, :k] @ q) - r["resid_hist"][k - 1]) <= 1e-12 * beta
    lhs = A @ V[:, :n_A]
    rhs = V @ Hbar
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.abs(lhs).max()
    assert np.max(np.abs(V.T @ V - np.eye(n_A + 1))) <= 1e-10
    # residual monotone within a cycle
    h = r["resid_hist"]
    assert np.all(np.diff(h) <= 1e-12 * beta)


def test_restarted_solve_matches_dense(orc):
    # AC1: restarted GMRES(5) reaches eps on a dominant system; x vs numpy.linalg.solve
    op, b = inputs.seven_diagonal(80, seed=4)
    A = dense(orc, op)
    eps = 1e-10 * np.linalg.norm(b)
    r = orc.pspgmres(op, b, np.zeros(80), eps=eps, n_A=5, n_r=500)
    rep = r["report"]
    assert rep["converged"] and rep["cycles"] > 1
    assert rep["final_resid_true"] <= 1.01 * eps
    xref = np.linalg.solve(A, b)
    assert np.linalg.norm(r["x"] - xref) <= np.linalg.cond(A) * 1e-10 * np.linalg.norm(xref)
    # probe accounting: one probe per cycle start + one per inner iteration
    assert rep["matvecs"] == rep["cycles"] + rep["iterations"]


def test_identity_precond_equivalence(orc):
    # AC2 / S:167: explicit N = I factors give the same iterates as the identity path
    op, b = inputs.seven_diagonal(50, seed=5)
    eye = np.zeros((3, 50))
    eye[1] = 1.0
    _, lu = orc.banded_lu(eye, 1)
    r1 = orc.pspgmres(op, b, np.zeros(50), eps=1e-9, n_A=7, n_r=100)
    r2 = orc.pspgmres(op, b, np.zeros(50), eps=1e-9, n_A=7, n_r=100, d=1, lu=lu)
    assert r1["report"]["iterations"] == r2["report"]["iterations"]
    assert np.max(np.abs(r1["resid_hist"] - r2["resid_hist"])) <= 1e-12 * r1["beta_hist"][0]
    assert np.max(np.abs(r1["x"] - r2["x"])) <= 1e-12 * np.abs(r1["x"]).max()


def test_exact_x0_zero_iterations(orc):
    # S:164 / R3: b = A x0 -> 0 iterations, x = x0
    op, _ = inputs.seven_diagonal(30, seed=6)
    x0 = np.random.default_rng(2).standard_normal(30)
    b = orc.matvec(op, x0)
    r = orc.pspgmres(op, b, x0, eps=1e-8, n_A=5, n_r=3)
    assert r["report"]["iterations"] == 0 and r["report"]["converged"]
    assert np.array_equal(r["x"], x0)


def test_probe_ring_records_operator_pairs(orc):
    # every recorded pair satisfies P_y = A P_x; FIFO eviction
    p = inputs.c1(n=64)
    ring = orc.Ring(64, 16)
    r = orc.pspgmres(p.op, p.u0, p.u0, eps=1e-10 * np.linalg.norm(p.u0), n_A=10, n_r=50, ring=ring)
    assert ring.count == min(16, r["report"]["matvecs"])
    px, py = ring.columns()
    for c in range(ring.count):
        assert np.array_equal(orc.matvec(p.op, px[c]), py[c])


def test_ring_eviction_order(orc):
    ring = orc.Ring(2, 2)
    for v in (1.0, 2.0, 3.0):
        ring.record(np.full(2, v), np.full(2, -v))
    px, py = ring.columns()
    assert ring.count == 2 and px[0, 0] == 2.0 and px[1, 0] == 3.0 and py[1, 0] == -3.0


def test_breakdown_identity_k1(orc):
    # A = N = I, k = 1 -> H(2,1) = 0: lucky breakdown, converged
    op = diag_op(np.ones(5))
    b = np.arange(1.0, 6.0)
    r = orc.pspgmres(op, b, np.zeros(5), eps=0.0, n_A=4, n_r=2, trace=True)
    assert r["report"]["iterations"] == 1 and r["report"]["converged"]
    assert r["trace"]["Hraw"][1, 0] == 0.0
    assert np.allclose(r["x"], b, rtol=0, atol=1e-14)


def test_noconv_status(orc):
    op, b = inputs.seven_diagonal(40, seed=8)
    r = orc.pspgmres(op, b, np.zeros(40), eps=1e-30, n_A=2, n_r=3)
    assert r["status"] == orc.E_NOCONV and not r["report"]["converged"] and r["report"]["cycles"] == 3
