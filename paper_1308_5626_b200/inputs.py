"""Seeded synthetic inputs for the PSP-GMRES hot path (configs C1..C5 of BASELINE.json).

This module is the ONLY code shared by the CUDA path and the oracle: it generates input
data (grids, coefficient fields, initial states, probe sets) and holds none of the
method's arithmetic (no operator apply, no Krylov, no regression, no solve).  The recipes
are stated in DESIGN.md ("Input recipe"); they follow SURVEY.md section 8(d).

An operator is described by ``OperatorSpec`` (the data of A = I - dt*L, Eq.4); both
sides apply it with their own code.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field as dc_field

import numpy as np


@dataclass
class OperatorSpec:
    ndim: int
    kind: str                       # 'const_diff' | 'cell_diff' | 'cell_advdiff' | 'dia'
    n: tuple                        # interior points per axis, n[0] = nx (fastest)
    dt: float
    nu: float = 1.0                 # constant diffusivity (const_diff)
    c: tuple = (0.0, 0.0, 0.0)      # upwind velocity (cell_advdiff), c_a >= 0
    field: np.ndarray | None = None  # kappa / nu at the points, flat, length rows
    dA: int = 0                     # half-bandwidth (dia)
    bands: np.ndarray | None = None  # (2dA+1, rows) DIA bands (dia): bands[o, i] = A(i, i+o-dA)

    @property
    def rows(self) -> int:
        return int(np.prod(self.n))

    @property
    def h(self) -> tuple:
        return tuple(1.0 / (na + 1) for na in self.n)


@dataclass
class Problem:
    name: str
    op: OperatorSpec
    u0: np.ndarray                  # flat, length rows
    restart: int                    # n_A
    tol: float                      # eps = tol * ||b|| (R1)
    d: int                          # MREP half-bandwidth
    steps: int
    m_max: int
    max_cycles: int                 # n_r (R9)
    meta: dict = dc_field(default_factory=dict)


def _grid_1d(n: int) -> np.ndarray:
    h = 1.0 / (n + 1)
    return np.arange(1, n + 1, dtype=np.float64) * h


# ------------------------------------------------------------------------------------------
# C1: 1-D heat, n = 1024, dt = 1e-3 (dt/h^2 = 1050.625), u0 = sin(pi x) + 0.1 U(-1,1), seed 0
# ------------------------------------------------------------------------------------------
def c1(n: int = 1024, dt: float = 1e-3, steps: int = 5) -> Problem:
    rng = np.random.default_rng(0)
    x = _grid_1d(n)
    u0 = np.sin(np.pi * x) + 0.1 * rng.uniform(-1.0, 1.0, n)
    op = OperatorSpec(ndim=1, kind="const_diff", n=(n,), dt=dt, nu=1.0)
    return Problem("C1", op, u0, restart=30, tol=1e-10, d=1, steps=steps, m_max=64, max_cycles=10000)


# ------------------------------------------------------------------------------------------
# C2: 2-D heat 512^2, dt = 100 h^2, u0 = sum of 8 Dirichlet sine modes (R26), seed [0,2]
# ------------------------------------------------------------------------------------------
def c2(n: int = 512, d: int = 1, steps: int = 20) -> Problem:
    rng = np.random.default_rng([0, 2])
    a = rng.standard_normal(8)
    p = rng.integers(1, 33, 8)
    q = rng.integers(1, 33, 8)
    x = _grid_1d(n)
    X = x[None, :]
    Y = x[:, None]
    u0 = np.zeros((n, n))
    for j in range(8):
        u0 += a[j] * np.sin(p[j] * np.pi * X) * np.sin(q[j] * np.pi * Y)
    h = 1.0 / (n + 1)
    op = OperatorSpec(ndim=2, kind="const_diff", n=(n, n), dt=100.0 * h * h, nu=1.0)
    return Problem("C2", op, u0.reshape(-1), restart=40, tol=1e-10, d=d, steps=steps, m_max=64,
                   max_cycles=1000, meta=dict(a=a, p=p, q=q))


# ------------------------------------------------------------------------------------------
# C3: 2-D advection-diffusion 2048^2, nu = 1 + 0.5 sin(2 pi x) cos(2 pi y), c = (1, 0.5),
#     dt = 1e-4, u0 = Gaussian bump (width 0.1, centre (1/2,1/2)) + 1e-2 N(0,1), seed [0,3]
# ------------------------------------------------------------------------------------------
def c3(n: int = 2048, dt: float = 1e-4, steps: int = 10) -> Problem:
    rng = np.random.default_rng([0, 3])
    x = _grid_1d(n)
    X = x[None, :]
    Y = x[:, None]
    nu = 1.0 + 0.5 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
    u0 = np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * 0.1 ** 2)) + 1e-2 * rng.standard_normal((n, n))
    op = OperatorSpec(ndim=2, kind="cell_advdiff", n=(n, n), dt=dt, c=(1.0, 0.5, 0.0),
                      field=np.ascontiguousarray(nu.reshape(-1)))
    return Problem("C3", op, np.ascontiguousarray(u0.reshape(-1)), restart=50, tol=1e-9, d=2, steps=steps,
                   m_max=64, max_cycles=1000)


# ------------------------------------------------------------------------------------------
# C4: 3-D variable-kappa diffusion 512^3; kappa = exp(g), g a Gaussian random field with
#     covariance exp(-r^2 / (2 l^2)), l = 8 cells, normalised to mean 0 / std 1;
#     dt * max(kappa) / h^2 = 50; u0 = U(-1,1); seed [0,4].  Axes (z, y, x), x fastest.
# ------------------------------------------------------------------------------------------
def c4_field(n: int, ell: float = 8.0, seed=(0, 4)):
    """Returns (kappa, u0) as flat float64 arrays of n^3 (x fastest)."""
    import scipy.fft as sfft
    rng = np.random.default_rng(list(seed))
    w = rng.standard_normal((n, n, n))
    workers = max(1, os.cpu_count() or 1)
    wh = sfft.rfftn(w, workers=workers)
    del w
    kz = np.fft.fftfreq(n)[:, None, None]
    ky = np.fft.fftfreq(n)[None, :, None]
    kx = np.fft.rfftfreq(n)[None, None, :]
    filt = np.exp(-(math.pi ** 2) * ell * ell * (kz * kz + ky * ky + kx * kx))
    wh *= filt
    del filt
    g = sfft.irfftn(wh, s=(n, n, n), workers=workers)
    del wh
    g -= g.mean()
    g /= g.std()
    kappa = np.exp(g).reshape(-1)
    del g
    u0 = rng.uniform(-1.0, 1.0, (n, n, n)).reshape(-1)
    return kappa, u0


def c4(n: int = 512, steps: int = 10, m_max: int = 32) -> Problem:
    kappa, u0 = c4_field(n)
    h = 1.0 / (n + 1)
    dt = 50.0 * h * h / float(kappa.max())
    op = OperatorSpec(ndim=3, kind="cell_diff", n=(n, n, n), dt=dt, field=kappa)
    return Problem("C4", op, u0, restart=30, tol=1e-8, d=3, steps=steps, m_max=m_max, max_cycles=1000)


# ------------------------------------------------------------------------------------------
# C5: MREP + banded-solve sweep.  A_true banded (half-bandwidth d), off-diagonals U(-1,1)
#     (zero outside the matrix), diagonal = sum |off| + 1; P_x = N(0,1) (m x n, row c = probe
#     column c); P_y = A_true P_x + 1e-8 N(0,1); v = N(0,1).
# ------------------------------------------------------------------------------------------
def _mask_outside(bands: np.ndarray, d: int) -> np.ndarray:
    n = bands.shape[1]
    i = np.arange(n)
    for o in range(2 * d + 1):
        j = i + o - d
        bands[o, (j < 0) | (j >= n)] = 0.0
    return bands


def c5_numpy(n: int, m: int, d: int, seed: int = 0):
    """Small-n C5 instance on the host (numpy PCG64).  Returns dict(bands, px, py, v)."""
    rng = np.random.default_rng([0, 5, seed, n, m, d])
    bands = rng.uniform(-1.0, 1.0, (2 * d + 1, n))
    bands[d] = 0.0
    _mask_outside(bands, d)
    bands[d] = np.abs(bands).sum(axis=0) + 1.0
    px = rng.standard_normal((m, n))
    py = np.zeros((m, n))
    for o in range(2 * d + 1):      # synthesis of P_y from the known A_true (input recipe)
        s = o - d
        lo, hi = max(0, -s), min(n, n - s)
        py[:, lo:hi] += bands[o, lo:hi] * px[:, lo + s:hi + s]
    py += 1e-8 * rng.standard_normal((m, n))
    v = rng.standard_normal(n)
    return dict(bands=bands, px=px, py=py, v=v)


def c5_torch(n: int, m: int, d: int, seed: int = 0, device="cuda"):
    """Large-n C5 instance generated on the device (torch Philox, seeded).  Same recipe."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f64 = torch.float64
    bands = torch.rand((2 * d + 1, n), generator=g, device=device, dtype=f64) * 2.0 - 1.0
    bands[d] = 0.0
    i = torch.arange(n, device=device)
    for o in range(2 * d + 1):
        j = i + o - d
        bands[o][(j < 0) | (j >= n)] = 0.0
    bands[d] = bands.abs().sum(dim=0) + 1.0
    px = torch.randn((m, n), generator=g, device=device, dtype=f64)
    py = torch.empty((m, n), device=device, dtype=f64)
    for c in range(m):
        yc = bands[d] * px[c]
        for o in range(2 * d + 1):
            s = o - d
            if s == 0:
                continue
            lo, hi = max(0, -s), min(n, n - s)
            yc[lo:hi] += bands[o, lo:hi] * px[c, lo + s:hi + s]
        py[c] = yc
    py += 1e-8 * torch.randn((m, n), generator=g, device=device, dtype=f64)
    v = torch.randn((n,), generator=g, device=device, dtype=f64)
    return dict(bands=bands, px=px, py=py, v=v)


# ------------------------------------------------------------------------------------------
# f1 (the paper's own experiment): seven-diagonal random diagonally dominant A,
# rhs = [1..n] (off-diagonals U(-1,1), diagonal = row |off| sum + margin)
# ------------------------------------------------------------------------------------------
def seven_diagonal(n: int, seed: int = 0, margin: float = 1.0):
    rng = np.random.default_rng([0, 7, seed, n])
    dA = 3
    bands = rng.uniform(-1.0, 1.0, (2 * dA + 1, n))
    bands[dA] = 0.0
    _mask_outside(bands, dA)
    bands[dA] = np.abs(bands).sum(axis=0) + margin
    op = OperatorSpec(ndim=1, kind="dia", n=(n,), dt=0.0, dA=dA, bands=bands)
    b = np.arange(1, n + 1, dtype=np.float64)
    return op, b


def dia_operator(bands: np.ndarray, dA: int) -> OperatorSpec:
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    return OperatorSpec(ndim=1, kind="dia", n=(bands.shape[1],), dt=0.0, dA=dA, bands=bands)


def small(name: str, n: int, **kw) -> Problem:
    """Reduced-size instance of a config recipe (parity cases)."""
    if name == "C1":
        return c1(n=n, **kw)
    if name == "C2":
        return c2(n=n, **kw)
    if name == "C3":
        return c3(n=n, **kw)
    if name == "C4":
        return c4(n=n, **kw)
    raise KeyError(name)
