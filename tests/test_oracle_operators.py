"""Pins of oracle O1 (A = I - dt L, Eq.4, applied matrix-free P:30) -- PN1.

Each check is independent of the oracle's own formula: closed-form eigenvalues of the
discrete Dirichlet Laplacian, the energy identity summed over faces (not rows), symmetry,
reduction to a textbook special case, linearity.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sine_mode(n_axes, ks):
    """Dirichlet sine mode prod_a sin(k_a pi x_a) on the interior grid (x fastest)."""
    grids = [np.sin(k * np.pi * np.arange(1, n + 1) / (n + 1)) for n, k in zip(n_axes, ks)]
    u = grids[0]
    for g in grids[1:]:
        u = np.multiply.outer(g, u)  # new axis is slower
    return u.reshape(-1)


def closed_form_eig(n_axes, ks, dt, nu):
    lam = 0.0
    for n, k in zip(n_axes, ks):
        h = 1.0 / (n + 1)
        lam += 4.0 * nu / (h * h) * math.sin(k * math.pi * h / 2) ** 2
    return 1.0 + dt * lam


@pytest.mark.parametrize("n_axes,ks,dt,nu", [
    ((1024,), (1,), 1e-3, 1.0),
    ((1024,), (300,), 1e-3, 1.0),
    ((64, 48), (3, 7), 2e-4, 0.7),
    ((12, 10, 9), (2, 1, 5), 1e-3, 1.3),
])
def test_const_diff_sine_mode_eigenvalue(orc, n_axes, ks, dt, nu):
    op = inputs.OperatorSpec(ndim=len(n_axes), kind="const_diff", n=n_axes, dt=dt, nu=nu)
    phi = sine_mode(n_axes, ks)
    y = orc.matvec(op, phi)
    lam = closed_form_eig(n_axes, ks, dt, nu)
    assert np.max(np.abs(y - lam * phi)) <= 1e-12 * lam * np.max(np.abs(phi))


def test_dt_zero_is_identity(orc):
    rng = np.random.default_rng(1)
    for kind, extra in [("const_diff", {}), ("cell_diff", {"field": rng.uniform(0.5, 2, 60)}),
                        ("cell_advdiff", {"field": rng.uniform(0.5, 2, 60), "c": (1.0, 0.5, 0)})]:
        op = inputs.OperatorSpec(ndim=2, kind=kind, n=(10, 6), dt=0.0, **extra)
        x = rng.standard_normal(60)
        assert np.array_equal(orc.matvec(op, x), x)


def test_interior_rows_annihilate_constants(orc):
    # the second difference annihilates constants on interior rows
    op = inputs.OperatorSpec(ndim=1, kind="const_diff", n=(50,), dt=1e-3)
    y = orc.matvec(op, np.ones(50))
    assert np.allclose(y[1:-1], 1.0, rtol=0, atol=1e-12)
    assert y[0] > 1.0 and y[-1] > 1.0


def dense(orc, op):
    n = op.rows
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        A[:, j] = orc.matvec(op, e)
    return A


@pytest.mark.parametrize("n_axes", [(9,), (7, 5), (5, 4, 3)])
def test_cell_diff_symmetric_and_energy_identity(orc, n_axes):
    rng = np.random.default_rng(2)
    N = int(np.prod(n_axes))
    kappa = np.exp(rng.standard_normal(N))
    dt = 3e-3
    op = inputs.OperatorSpec(ndim=len(n_axes), kind="cell_diff", n=n_axes, dt=dt, field=kappa)
    A = dense(orc, op)
    assert np.allclose(A, A.T, rtol=0, atol=1e-12 * np.abs(A).max())
    # energy identity, summed over FACES: x'Ax = |x|^2 + dt sum_faces kappa_f (x_c - x_nb)^2 / h^2
    x = rng.standard_normal(N)
    K = kappa.reshape(n_axes[::-1])
    X = x.reshape(n_axes[::-1])
    energy = float(x @ x)
    for a in range(len(n_axes)):
        ax = len(n_axes) - 1 - a  # numpy axis of grid axis a
        h = 1.0 / (n_axes[a] + 1)
        kf = 0.5 * (np.take(K, range(0, K.shape[ax] - 1), axis=ax) + np.take(K, range(1, K.shape[ax]), axis=ax))
        dx = np.diff(X, axis=ax)
        energy += dt / h ** 2 * float(np.sum(kf * dx * dx))
        # two boundary faces per line, kappa_f = kappa_c, neighbour value 0
        first = np.take(X, [0], axis=ax)
        last = np.take(X, [X.shape[ax] - 1], axis=ax)
        energy += dt / h ** 2 * float(np.sum(np.take(K, [0], axis=ax) * first ** 2)
                                      + np.sum(np.take(K, [K.shape[ax] - 1], axis=ax) * last ** 2))
    assert abs(float(x @ A @ x) - energy) <= 1e-11 * energy


def test_cell_diff_constant_field_reduces_to_const_diff(orc):
    rng = np.random.default_rng(3)
    n_axes = (8, 7, 6)
    N = int(np.prod(n_axes))
    x = rng.standard_normal(N)
    a = inputs.OperatorSpec(ndim=3, kind="cell_diff", n=n_axes, dt=1e-3, field=np.full(N, 1.7))
    b = inputs.OperatorSpec(ndim=3, kind="const_diff", n=n_axes, dt=1e-3, nu=1.7)
    ya, yb = orc.matvec(a, x), orc.matvec(b, x)
    assert np.max(np.abs(ya - yb)) <= 1e-12 * np.max(np.abs(yb))


def test_advdiff_pure_upwind_is_bidiagonal(orc):
    # nu = 0, c = (c_x, 0): A = I + dt c_x/h (I - S_west): textbook first-order upwind
    n_axes = (6, 5)
    N = 30
    cx = 0.8
    op = inputs.OperatorSpec(ndim=2, kind="cell_advdiff", n=n_axes, dt=0.01, field=np.zeros(N), c=(cx, 0.0, 0.0))
    A = dense(orc, op)
    h = 1.0 / 7
    ref = np.eye(N) * (1 + 0.01 * cx / h)
    for g in range(N):
        if g % 6 > 0:
            ref[g, g - 1] = -0.01 * cx / h
    assert np.allclose(A, ref, rtol=0, atol=1e-13)


def test_advdiff_diffusive_part_matches_cell_diff(orc):
    rng = np.random.default_rng(4)
    n_axes = (9, 8)
    N = 72
    nu = rng.uniform(0.5, 1.5, N)
    x = rng.standard_normal(N)
    a = inputs.OperatorSpec(ndim=2, kind="cell_advdiff", n=n_axes, dt=2e-3, field=nu, c=(0.0, 0.0, 0.0))
    b = inputs.OperatorSpec(ndim=2, kind="cell_diff", n=n_axes, dt=2e-3, field=nu)
    assert np.max(np.abs(orc.matvec(a, x) - orc.matvec(b, x))) <= 1e-12 * np.max(np.abs(orc.matvec(b, x)))


def test_c3_rows_dominant_by_exactly_one(orc):
    p = inputs.c3(n=32)
    A = dense(orc, p.op)
    off = np.abs(A).sum(axis=1) - np.abs(np.diag(A))
    margin = (np.diag(A) - off).reshape(32, 32)
    tol = 1e-9 * np.abs(A).max()
    # interior rows: dominant by exactly 1 (every face coupling appears once on each side)
    assert np.allclose(margin[1:-1, 1:-1], 1.0, rtol=0, atol=tol)
    # boundary rows keep the boundary-face terms on the diagonal only: strictly more dominant
    assert np.all(margin >= 1.0 - tol)


def test_linearity(orc):
    # apply(a x + b y) = a apply(x) + b apply(y) to 1e-12
    rng = np.random.default_rng(5)
    p = inputs.c4(n=10, steps=1)
    x, y = rng.standard_normal(1000), rng.standard_normal(1000)
    lhs = orc.matvec(p.op, 2.5 * x - 0.75 * y)
    rhs = 2.5 * orc.matvec(p.op, x) - 0.75 * orc.matvec(p.op, y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_dia_operator_matches_dense(orc):
    op, _ = inputs.seven_diagonal(20, seed=1)
    A = dense(orc, op)
    B = np.zeros((20, 20))
    for o in range(7):
        for i in range(20):
            j = i + o - 3
            if 0 <= j < 20:
                B[i, j] = op.bands[o, i]
    assert np.array_equal(A, B)


def test_c1_grid_convention(orc):
    # P:25 with h = 1/(n+1): C1's dt/h^2 = 1e-3 * 1025^2 = 1050.625 (BASELINE C1 "approx 1050")
    p = inputs.c1()
    e = np.zeros(1024)
    e[500] = 1.0
    y = orc.matvec(p.op, e)
    assert y[500] == pytest.approx(1 + 2 * 1050.625, rel=1e-14)
    assert y[499] == pytest.approx(-1050.625, rel=1e-14)


def test_closed_form_worked_values_golden():
    g = json.load(open(os.path.join(GOLD, "implicit_euler_decay.json")))
    c1 = g["c1_grid"]
    for k, f in zip(c1["modes"], c1["factors"]):
        assert 1.0 / closed_form_eig((c1["n"],), (k,), c1["dt"], 1.0) == pytest.approx(f, abs=c1["abs_tol"])
    c2 = g["c2_grid"]
    h = 1.0 / (c2["n"] + 1)
    assert 1.0 / closed_form_eig((c2["n"], c2["n"]), tuple(c2["mode"]), c2["dt_over_h2"] * h * h, 1.0) == \
        pytest.approx(c2["factor"], abs=c2["abs_tol"])
