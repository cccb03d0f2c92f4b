"""Pins of oracle O2: the banded solve N z = v (P:30 Thomas, P:161 d > 1) -- PN2."""
import json
import os

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def to_dense(bands, d):
    n = bands.shape[1]
    A = np.zeros((n, n))
    for o in range(2 * d + 1):
        for i in range(n):
            j = i + o - d
            if 0 <= j < n:
                A[i, j] = bands[o, i]
    return A


def dominant_bands(n, d, seed, margin=1.0):
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1, 1, (2 * d + 1, n))
    b[d] = 0
    for o in range(2 * d + 1):
        for i in range(n):
            if not 0 <= i + o - d < n:
                b[o, i] = 0
    b[d] = np.abs(b).sum(axis=0) + margin
    return b


def test_tridiag_worked_example_golden(orc):
    g = json.load(open(os.path.join(GOLD, "tridiag_worked_example.json")))
    st, z = orc.thomas(g["sub"], g["diag"], g["sup"], g["rhs"])
    assert st == orc.OK
    assert np.allclose(z, g["solution"], rtol=0, atol=1e-15)
    bands = np.array([g["sub"], g["diag"], g["sup"]])
    st, lu = orc.banded_lu(bands, 1)
    assert st == orc.OK
    assert np.allclose(orc.banded_lu_solve(lu, 1, np.array(g["rhs"])), g["solution"], rtol=0, atol=1e-15)


def test_scaled_identity(orc):
    # N = 3 I, rhs = ones -> ones/3 ; S:274 identity -> rhs
    for d in (1, 2, 4):
        bands = np.zeros((2 * d + 1, 9))
        bands[d] = 3.0
        st, lu = orc.banded_lu(bands, d)
        assert st == orc.OK
        assert np.array_equal(orc.banded_lu_solve(lu, d, np.ones(9)), np.full(9, 1.0 / 3.0))
    st, z = orc.thomas(np.zeros(3), np.ones(3), np.zeros(3), np.array([7.0, 8.0, 9.0]))
    assert st == orc.OK and list(z) == [7.0, 8.0, 9.0]


@pytest.mark.parametrize("d", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [10, 57, 200])
def test_banded_lu_vs_dense_solve(orc, d, n):
    # PN2: dense LU (numpy.linalg.solve) for n <= 200
    bands = dominant_bands(n, d, seed=100 * d + n)
    v = np.random.default_rng(n).standard_normal(n)
    st, lu = orc.banded_lu(bands, d)
    assert st == orc.OK
    z = orc.banded_lu_solve(lu, d, v)
    ref = np.linalg.solve(to_dense(bands, d), v)
    assert np.linalg.norm(z - ref) <= 1e-13 * np.linalg.norm(ref)
    # residual
    assert np.linalg.norm(orc.banded_matvec(bands, d, z) - v) <= 1e-13 * np.linalg.norm(v)


@pytest.mark.parametrize("d", [1, 3])
def test_lu_factors_reconstruct(orc, d):
    n = 40
    bands = dominant_bands(n, d, seed=7)
    st, lu = orc.banded_lu(bands, d)
    assert st == orc.OK
    Lf = np.eye(n)
    Uf = np.zeros((n, n))
    for o in range(2 * d + 1):
        for i in range(n):
            j = i + o - d
            if 0 <= j < n:
                (Lf if o < d else Uf)[i, j] = lu[o, i]
    A = to_dense(bands, d)
    assert np.max(np.abs(Lf @ Uf - A)) <= 1e-14 * np.abs(A).max() * n


def test_lu_d1_is_thomas_bitwise(orc):
    # LU(d=1) identical to Thomas
    n = 300
    bands = dominant_bands(n, 1, seed=3, margin=0.1)
    v = np.random.default_rng(0).standard_normal(n)
    st, z_t = orc.thomas(bands[0], bands[1], bands[2], v)
    st2, lu = orc.banded_lu(bands, 1)
    assert st == st2 == orc.OK
    assert np.array_equal(z_t, orc.banded_lu_solve(lu, 1, v))


def test_zero_pivot_is_singular(orc):
    # S:276
    bands = np.array([[0.0, 1.0, 1.0], [0.0, 2.0, 2.0], [1.0, 1.0, 0.0]])
    st, _ = orc.thomas(bands[0], bands[1], bands[2], np.ones(3))
    assert st == orc.E_SINGULAR
    st, _ = orc.banded_lu(bands, 1)
    assert st == orc.E_SINGULAR


def test_factor_once_solve_many(orc):
    # two solves against one factorization == two independent factor+solve runs
    bands = dominant_bands(80, 2, seed=9)
    st, lu = orc.banded_lu(bands, 2)
    rng = np.random.default_rng(1)
    v1, v2 = rng.standard_normal(80), rng.standard_normal(80)
    z1, z2 = orc.banded_lu_solve(lu, 2, v1), orc.banded_lu_solve(lu, 2, v2)
    _, lu2 = orc.banded_lu(bands, 2)
    assert np.array_equal(z1, orc.banded_lu_solve(lu2, 2, v1)) and np.array_equal(z2, orc.banded_lu_solve(lu2, 2, v2))


def test_gate_dominance(orc):
    d = 2
    bands = dominant_bands(30, d, seed=11, margin=1e-3)
    assert orc.gate_dominant(bands, d)
    b2 = bands.copy()
    b2[d, 17] = np.abs(b2[:, 17]).sum() - np.abs(b2[d, 17])  # exactly equal: not strict
    assert not orc.gate_dominant(b2, d)
    # out-of-matrix corner entries are ignored
    b3 = bands.copy()
    b3[0, 0] = 1e9
    assert orc.gate_dominant(b3, d)


def test_c5_recipe_dominant(orc):
    g = inputs.c5_numpy(500, 16, 3)
    assert orc.gate_dominant(g["bands"], 3)
