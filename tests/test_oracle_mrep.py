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
