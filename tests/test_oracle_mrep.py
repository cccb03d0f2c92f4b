"""Pins of oracle O4: MREP, literal Algorithm 2 -- PN4.

Independent checks: exact recovery of a banded A (regression is exact when the truth lies in
the model class), the KKT / normal-equation optimality of every interior row computed with
numpy, linear-fit worked examples (golden), the [1,0,3,0] recovery (golden), permutation
invariance, sample-count and degenerate cases.
"""
import json
import os

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def banded_apply(bands, d, X):
    """rows of X are vectors; returns A X' as rows (independent numpy construction)."""
    n = bands.shape[1]
    A = np.zeros((n, n))
    for o in range(2 * d + 1):
        for i in range(n):
            j = i + o - d
            if 0 <= j < n:
                A[i, j] = bands[o, i]
    return X @ A.T, A


@pytest.mark.parametrize("d,m", [(1, 4), (1, 13), (2, 6), (3, 8), (3, 32), (4, 40)])
def test_exact_recovery(orc, d, m):
    # AC3 / S:234: banded A (half-bandwidth <= d), m >= 2d+2 generic probes -> interior rows = A
    n = 60
    g = inputs.c5_numpy(n, m, d, seed=1)
    py, A = banded_apply(g["bands"], d, g["px"])
    r = orc.mrep(g["px"], py, d)
    assert r["status"] == orc.OK
    for i in range(d, n - d):
        row = A[i, i - d:i + d + 1]
        # accuracy attainable by the normal equations: ~ eps * kappa(Gram) (T3)
        tol = max(1e-12, 1e-14 * r["kappa_est"][i]) * np.abs(row).max()
        if r["row_kind"][i] == orc.ROW_INTERIOR_RIDGE:
            continue   # (only at m = 2d+2 can a random square design be that ill-conditioned)
        assert r["row_kind"][i] == orc.ROW_INTERIOR
        assert np.max(np.abs(r["bands"][:, i] - row)) <= tol, i
        assert abs(r["intercept"][i]) <= tol
    if m >= 4 * d + 4:
        assert np.all(r["row_kind"][d:n - d] == orc.ROW_INTERIOR)
        assert np.max(r["kappa_est"][d:n - d]) < 1e6
    # boundary rows: diagonal only
    for i in list(range(d)) + list(range(n - d, n)):
        assert r["row_kind"][i] == orc.ROW_BOUNDARY
        assert np.count_nonzero(r["bands"][:, i]) <= 1


def test_spec_tridiagonal_basis_probes(orc):
    # tridiagonal dominant A, n = 12, probes = 12 basis vectors + ones (m = 13)
    n = 12
    rng = np.random.default_rng(3)
    bands = rng.uniform(-1, 1, (3, n))
    bands[0, 0] = bands[2, -1] = 0
    bands[1] = np.abs(bands[0]) + np.abs(bands[2]) + 1
    px = np.vstack([np.eye(n), np.ones(n)])
    py, A = banded_apply(bands, 1, px)
    r = orc.mrep(px, py, 1)
    for i in range(1, n - 1):
        assert np.max(np.abs(r["bands"][:, i] - A[i, i - 1:i + 2])) <= 1e-8
        assert abs(r["intercept"][i]) <= 1e-8


def test_insufficient_samples(orc):
    # S:213 / R19: m < 2d+2 -> insufficient samples
    g = inputs.c5_numpy(20, 3, 1)
    assert orc.mrep(g["px"], g["py"], 1)["status"] == orc.E_SAMPLES
    g = inputs.c5_numpy(20, 7, 3)
    assert orc.mrep(g["px"], g["py"], 3)["status"] == orc.E_SAMPLES


@pytest.mark.parametrize("d,m", [(1, 8), (2, 16), (3, 32)])
def test_kkt_optimality_every_interior_row(orc, d, m):
    # P:122 normal equations: X*(y - X*' beta) = 0 for every interior row (noisy data, no truth)
    n = 50
    rng = np.random.default_rng(d * 10 + m)
    px = rng.standard_normal((m, n))
    py = rng.standard_normal((m, n))
    r = orc.mrep(px, py, d)
    for i in range(d, n - d):
        Xs = np.vstack([np.ones(m), px[:, i - d:i + d + 1].T])
        beta = np.concatenate([[r["intercept"][i]], r["bands"][:, i]])
        grad = Xs @ (py[:, i] - Xs.T @ beta)
        assert np.max(np.abs(grad)) <= 1e-11 * np.linalg.norm(Xs) * np.linalg.norm(py[:, i]), i


def _boundary_row_case(orc, xs, ys):
    m = len(xs)
    n, d = 5, 1
    rng = np.random.default_rng(0)
    px = rng.standard_normal((m, n))
    py = rng.standard_normal((m, n))
    px[:, 0] = xs
    py[:, 0] = ys
    return orc.mrep(px, py, d)


def test_linear_fit_golden(orc):
    g = json.load(open(os.path.join(GOLD, "linear_fit_examples.json")))
    pad = [0.5, -0.25, 2.0, 1.0]   # extra samples keep m >= 2d+2 while the fitted row is exact
    for case in g["cases"]:
        xs = case["xs"] + ([1.0] * 4 if case.get("zero_variance") else pad)
        if case.get("zero_variance"):
            ys = case["ys"] + [4.0] * 4
        else:
            ys = case["ys"] + [case["beta0"] + case["beta1"] * v for v in pad]
        r = _boundary_row_case(orc, xs, ys)
        if case.get("zero_variance"):
            assert r["row_kind"][0] == orc.ROW_FALLBACK_ZEROVAR and r["bands"][1, 0] == 1.0
        elif case["beta1"] == 0.0:
            # fitted slope 0 is a zero diagonal: R18 turns the row into an identity row,
            # the intercept of the fit is still reported
            assert r["row_kind"][0] == orc.ROW_FALLBACK_SMALLDIAG
            assert r["intercept"][0] == pytest.approx(case["beta0"], abs=1e-13)
        else:
            assert r["row_kind"][0] == orc.ROW_BOUNDARY
            assert r["bands"][1, 0] == pytest.approx(case["beta1"], abs=1e-14)
            assert r["intercept"][0] == pytest.approx(case["beta0"], abs=1e-13)


def test_coefficient_recovery_golden(orc):
    g = json.load(open(os.path.join(GOLD, "mrep_coefficient_recovery.json")))
    d = g["d"]
    n, m = 9, 10
    rng = np.random.default_rng(5)
    px = rng.standard_normal((m, n))
    py = rng.standard_normal((m, n))
    i = 4
    coef = g["coefficients"]
    py[:, i] = coef[0] + sum(coef[1 + a] * px[:, i - d + a] for a in range(2 * d + 1))
    r = orc.mrep(px, py, d)
    got = [r["intercept"][i]] + list(r["bands"][:, i])
    assert np.max(np.abs(np.array(got) - coef)) <= g["tol"]


def test_zero_response(orc):
    # S:230
    rng = np.random.default_rng(6)
    px = rng.standard_normal((12, 20))
    r = orc.mrep(px, np.zeros((12, 20)), 2)
    assert np.all(r["bands"][:, 2:18] == 0) and np.all(r["intercept"][2:18] == 0)


def test_permutation_invariance(orc):
    # relabelling probes leaves N unchanged (to rounding)
    g = inputs.c5_numpy(40, 16, 2, seed=3)
    perm = np.random.default_rng(0).permutation(16)
    a = orc.mrep(g["px"], g["py"], 2)
    b = orc.mrep(g["px"][perm], g["py"][perm], 2)
    assert np.max(np.abs(a["bands"] - b["bands"])) <= 1e-12 * np.abs(a["bands"]).max()
    # the `order` argument (ring slots) is the same permutation mechanism
    c = orc.mrep(g["px"][perm], g["py"][perm], 2, order=list(np.argsort(perm)))
    assert np.array_equal(a["bands"], c["bands"])


def test_rank_deficient_uses_ridge(orc):
    # duplicate probe columns -> rank-deficient Gram -> ridge path, finite, flagged
    rng = np.random.default_rng(7)
    base = rng.standard_normal((3, 20))
    px = np.vstack([base, base, base])      # m = 9 >= 4 samples but rank 3 < 4 unknowns
    py = 2.0 * px
    r = orc.mrep(px, py, 1)
    assert r["status"] == orc.OK and r["rows_ridge"] > 0
    assert np.all(np.isfinite(r["bands"]))
    assert np.all(r["row_kind"][1:19] != orc.ROW_INTERIOR)


def test_small_diagonal_fallback(orc):
    # R18 / S:243: |N(i,i)| < 1e-12 max|N(j,j)| -> identity row
    g = inputs.c5_numpy(30, 12, 1, seed=4)
    py, A = banded_apply(g["bands"], 1, g["px"])
    # make row 10's true diagonal tiny
    py[:, 10] = g["bands"][0, 10] * g["px"][:, 9] + 1e-20 * g["px"][:, 10] + g["bands"][2, 10] * g["px"][:, 11]
    r = orc.mrep(g["px"], py, 1)
    assert r["row_kind"][10] == orc.ROW_FALLBACK_SMALLDIAG
    assert list(r["bands"][:, 10]) == [0.0, 1.0, 0.0]
    assert r["rows_fallback"] == 1


def test_c5_recipe_statistical_recovery(orc):
    # PN4 (C5): noise 1e-8 -> |beta - A_true| <~ 5e-8/sqrt(m)-scale per coefficient
    d, m = 2, 32
    g = inputs.c5_numpy(200, m, d, seed=2)
    r = orc.mrep(g["px"], g["py"], d)
    err = np.abs(r["bands"][:, d:200 - d] - g["bands"][:, d:200 - d])
    assert err.max() <= 1e-7
    assert r["gate_accepted"]


def hadamard8():
    """Sylvester Hadamard matrix of order 8: rows mutually orthogonal, row 0 all ones, every other
    row sums to zero."""
    H = np.array([[1.0]])
    for _ in range(3):
        H = np.block([[H, H], [H, -H]])
    return H


@pytest.mark.parametrize("a2,ridged", [(3e-7, True), (1e-7, True), (1e-3, False)])
def test_ridge_branch_closed_form(orc, a2, ridged):
    """R17 / S:226 pinned by a closed form.  With orthogonal, zero-sum probe rows (Hadamard rows
    scaled by a_j) the interior row's Gram is diagonal, G = diag(8, 8a_0^2, 8a_1^2, 8a_2^2), so
    its Cholesky factor is diag(sqrt(G_jj)), the condition estimate is exactly
    (max L_jj / min L_jj)^2 = max G_jj / min G_jj, and the ridge solution of G + lambda I is
    beta_j = r_j / (G_jj + lambda) with lambda = 1e-10 trace(G) / (2d+2) -- no solver involved.
    A tiny a_2 puts the estimate above 1e12 and the shrinkage r_j / (G_jj + lambda) visibly
    below the unridged r_j / G_jj (a wrong lambda, an unsquared estimate or a missing retry
    fails); a_2 = 1e-3 stays below 1e12 (no ridge, the exact coefficients)."""
    d, m = 1, 8
    H = hadamard8()
    a = np.array([1.0, 0.5, a2])
    px = np.zeros((m, 3))
    for j in range(3):
        px[:, j] = a[j] * H[1 + j]
    beta_true = np.array([0.25, -1.5, 4.0, 2.0])   # intercept, N(1,0), N(1,1), N(1,2)
    py = np.zeros((m, 3))
    py[:, 1] = beta_true[0] + px @ beta_true[1:]
    py[:, 0] = 3.0 * px[:, 0]                        # boundary rows: exact linear fits
    py[:, 2] = -2.0 * px[:, 2]
    r = orc.mrep(px, py, d)
    g = np.array([8.0, 8.0 * a[0] ** 2, 8.0 * a[1] ** 2, 8.0 * a[2] ** 2])
    kap = g.max() / g.min()
    assert r["kappa_est"][1] == pytest.approx(kap, rel=1e-12)
    rhs = g * beta_true                              # r = G beta_true (consistent data)
    if ridged:
        assert kap > 1e12
        lam = 1e-10 * g.sum() / (2 * d + 2)
        expect = rhs / (g + lam)
        assert r["row_kind"][1] == orc.ROW_INTERIOR_RIDGE and r["rows_ridge"] == 1
        assert expect[3] < 0.9 * beta_true[3]        # the shrinkage is visible in the test
    else:
        assert kap < 1e12
        expect = beta_true
        assert r["row_kind"][1] == orc.ROW_INTERIOR and r["rows_ridge"] == 0
    # r_j = sum_c x_jc y_c cancels from terms of size |x_j| |y|: the attainable error of beta_j is
    # ~ m u sum_c |x_jc y_c| / (G_jj + lambda)
    X = np.vstack([np.ones(m), px.T])
    tol = 16 * 2.0 ** -53 * (np.abs(X) @ np.abs(py[:, 1])) / (g + (lam if ridged else 0.0)) + 1e-13 * np.abs(expect)
    got = np.concatenate([[r["intercept"][1]], r["bands"][:, 1]])
    assert np.all(np.abs(got - expect) <= tol), (got, expect, tol)
    assert r["bands"][1, 0] == pytest.approx(3.0, rel=1e-14) and r["bands"][1, 2] == pytest.approx(-2.0, rel=1e-14)


def test_ridge_matches_pseudo_inverse_on_row_space(orc):
    """for an exactly rank-deficient, consistent design the ridge solution of R17 equals
    the minimum-norm least-squares solution G^+ r (numpy's SVD pseudo-inverse of the design)
    up to O(lambda / sigma_min^2) = O(1e-10) on the row space; its null-space component is 0."""
    rng = np.random.default_rng(7)
    d, n = 1, 20
    base = rng.standard_normal((3, n))
    px = np.vstack([base, base, base])              # m = 9, rank-3 column space in 4 unknowns
    truth = np.array([0.3, -1.0, 2.5, 0.7])
    py = np.zeros_like(px)
    for i in range(1, n - 1):
        py[:, i] = truth[0] + px[:, i - 1:i + 2] @ truth[1:]
    r = orc.mrep(px, py, d)
    for i in range(1, n - 1):
        X = np.hstack([np.ones((9, 1)), px[:, i - 1:i + 2]])
        mn = np.linalg.pinv(X) @ py[:, i]           # minimum-norm least squares (SVD)
        got = np.concatenate([[r["intercept"][i]], r["bands"][:, i]])
        assert r["row_kind"][i] in (orc.ROW_INTERIOR_RIDGE,)
        # S:231's 1e-6, or the normal equations' attainable accuracy 8 P u kappa_2(G + lambda I)
        # (T3) when that is larger: the ridged Gram has kappa ~ trace / lambda ~ 1e10
        G = X.T @ X
        Gl = G + 1e-10 * np.trace(G) / 4 * np.eye(4)
        tol = max(1e-6, 8 * 4 * 2.0 ** -53 * np.linalg.cond(Gl))
        assert np.linalg.norm(got - mn) <= tol * np.linalg.norm(mn), i
        # null space of X: no component of the ridge solution there
        _, s, vt = np.linalg.svd(X)
        null = vt[np.sum(s > 1e-10 * s[0]):]
        assert np.all(np.abs(null @ got) <= tol * np.linalg.norm(mn))
