"""Pins of oracle O5: the implicit-Euler time-step driver (Eq.3-4) -- PN5."""
import json
import math
import os

import numpy as np
import pytest

from paper_1308_5626_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def decay(n_axes, ks, dt, nu=1.0):
    lam = sum(4.0 * nu * (n + 1) ** 2 * math.sin(k * math.pi / (2 * (n + 1))) ** 2 for n, k in zip(n_axes, ks))
    return 1.0 / (1.0 + dt * lam)


@pytest.mark.parametrize("k", [1, 7, 300])
def test_sine_mode_decay_c1_grid(orc, k):
    # AC8 / S:340: one step of a discrete sine mode scales it by the closed-form factor
    g = json.load(open(os.path.join(GOLD, "implicit_euler_decay.json")))["c1_grid"]
    p = inputs.c1()
    x = np.arange(1, 1025) / 1025.0
    u0 = np.sin(k * np.pi * x)
    r = orc.time_steps(p.op, u0, 1, restart=30, max_cycles=10, tol=1e-10, d=1, m_max=64)
    f = g["factors"][g["modes"].index(k)]
    # an eigenvector: one Krylov step up to the rounding of R_bar = u - A u (cancellation
    # amplified by ||A|| ~ 4200), so a couple of steps at most
    assert r["reports"][0]["solve"]["converged"] and r["reports"][0]["solve"]["iterations"] <= 5
    assert np.max(np.abs(r["u"] - f * u0)) <= 1e-12


def test_c2_modes_multi_step_closed_form(orc):
    # C2 recipe at 64^2: u^s = sum_j a_j f_j^s phi_j (R26)
    p = inputs.c2(n=64, d=1, steps=3)
    n = 64
    x = np.arange(1, n + 1) / (n + 1)
    r = orc.time_steps(p.op, p.u0, 3, restart=40, max_cycles=100, tol=1e-12, d=1, m_max=64)
    exact = np.zeros((n, n))
    for a, pp, qq in zip(p.meta["a"], p.meta["p"], p.meta["q"]):
        f = decay((n, n), (pp, qq), p.op.dt)
        exact += a * f ** 3 * np.outer(np.sin(qq * np.pi * x), np.sin(pp * np.pi * x))
    assert np.max(np.abs(r["u"] - exact.reshape(-1))) <= 1e-10 * np.abs(exact).max()


def test_c2_worked_value_golden(orc):
    g = json.load(open(os.path.join(GOLD, "implicit_euler_decay.json")))["c2_grid"]
    h = 1.0 / (g["n"] + 1)
    assert decay((g["n"], g["n"]), g["mode"], g["dt_over_h2"] * h * h) == pytest.approx(g["factor"], abs=g["abs_tol"])


def test_c1_psp_active_rank_bound_and_closed_form_N(orc):
    # PN4 (C1 closed form after step 1): interior rows of N = (-r, 1+2r, -r), r = dt/h^2;
    # PN5 (rank bound): A N^-1 = I + rank-2d boundary perturbation -> <= 2d+1 iterations
    p = inputs.c1()
    r = orc.time_steps(p.op, p.u0, p.steps, p.restart, p.max_cycles, p.tol, p.d, p.m_max)
    reps = r["reports"]
    assert all(s["solve"]["converged"] for s in reps)
    assert reps[0]["precond_was_identity"] and all(not s["precond_was_identity"] for s in reps[1:])
    assert all(s["mrep"]["gate_accepted"] for s in reps)
    assert all(s["solve"]["iterations"] <= 2 * p.d + 1 for s in reps[1:])
    assert reps[0]["solve"]["iterations"] > 10 * reps[1]["solve"]["iterations"]
    rr = 1e-3 * 1025.0 ** 2
    b = r["bands"]
    interior = b[:, 1:-1]
    ref = np.array([-rr, 1 + 2 * rr, -rr])[:, None]
    assert np.max(np.abs(interior - ref)) <= 1e-9 * (1 + 2 * rr)
    # boundary rows: diagonal only
    assert b[0, 0] == 0 and b[2, 0] == 0 and b[0, -1] == 0 and b[2, -1] == 0
    # every step solves Eq.4: true residual <= eps (R13)
    for s in reps:
        assert s["solve"]["final_resid_true"] <= 1.05 * s["solve"]["eps"]


def test_step_solution_vs_dense_solve(orc):
    p = inputs.c4(n=6, steps=2)
    n = p.op.rows
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1
        A[:, j] = orc.matvec(p.op, e)
    r = orc.time_steps(p.op, p.u0, 2, restart=30, max_cycles=100, tol=1e-12, d=3, m_max=32)
    u2 = np.linalg.solve(A, np.linalg.solve(A, p.u0))
    assert np.linalg.norm(r["u"] - u2) <= 1e-10 * np.linalg.norm(u2)


def test_steps1_is_plain_gmres(orc):
    # S:347
    p = inputs.c3(n=24)
    r1 = orc.time_steps(p.op, p.u0, 1, p.restart, p.max_cycles, p.tol, p.d, p.m_max)
    eps = p.tol * np.linalg.norm(p.u0)
    r2 = orc.pspgmres(p.op, p.u0, p.u0, eps, p.restart, p.max_cycles)
    assert np.array_equal(r1["u"], r2["x"])
    assert r1["reports"][0]["solve"]["iterations"] == r2["report"]["iterations"]


def test_reset_history_flag(orc):
    p = inputs.c1(n=128)
    a = orc.time_steps(p.op, p.u0, 2, 10, 2000, 1e-10, 1, 64, reset_history=True)
    b = orc.time_steps(p.op, p.u0, 2, 10, 2000, 1e-10, 1, 64, reset_history=False)
    assert a["ring"].count <= 64 and b["ring"].count == 64
    assert a["reports"][1]["solve"]["converged"] and b["reports"][1]["solve"]["converged"]


def test_gate_rejects_nondominant_fit_3d(orc):
    # R21: the 3-D variable-kappa operator is not banded within d; fitted rows are generally not
    # dominant, the gate keeps N = I and the step still converges
    p = inputs.c4(n=10, steps=2)
    r = orc.time_steps(p.op, p.u0, 2, p.restart, p.max_cycles, p.tol, p.d, p.m_max)
    assert r["reports"][0]["mrep_ran"]
    assert all(s["solve"]["converged"] for s in r["reports"])
    if not r["reports"][0]["mrep"]["gate_accepted"]:
        assert r["reports"][1]["precond_was_identity"]
