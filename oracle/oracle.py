"""ctypes marshalling for liboracle.so (oracle.c).  TEST INFRASTRUCTURE ONLY.

Argument marshalling only; every number is computed in oracle.c.  Operators are passed as
any object with attributes ``ndim, kind, n, dt, nu, c, field, dA, bands`` (the input
descriptions of ``paper_1308_5626_b200.inputs`` qualify) -- this module imports nothing
from the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

OK, E_ARG, E_DIM, E_SAMPLES, E_RANK, E_SINGULAR, E_NONFINITE, E_NOCONV = range(8)
ROW_INTERIOR, ROW_INTERIOR_RIDGE, ROW_BOUNDARY, ROW_FALLBACK_RANK, ROW_FALLBACK_ZEROVAR, \
    ROW_FALLBACK_SMALLDIAG = range(6)
_KINDS = {"const_diff": 0, "cell_diff": 1, "cell_advdiff": 2, "dia": 3}

_dp = C.POINTER(C.c_double)


class _Operator(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("kind", C.c_int32), ("n", C.c_int64 * 3), ("dt", C.c_double),
                ("nu", C.c_double), ("c", C.c_double * 3), ("field", _dp), ("dA", C.c_int32),
                ("pad_", C.c_int32), ("bands", _dp)]


class _Ring(C.Structure):
    _fields_ = [("n", C.c_int64), ("cap", C.c_int32), ("count", C.c_int32), ("head", C.c_int32),
                ("pad_", C.c_int32), ("px", _dp), ("py", _dp)]


class _SolveReport(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("cycles", C.c_int32),
                ("matvecs", C.c_int32), ("precond_applies", C.c_int32), ("status", C.c_int32),
                ("hist_len", C.c_int32), ("beta_len", C.c_int32), ("r0", C.c_double),
                ("final_resid_est", C.c_double), ("final_resid_true", C.c_double), ("eps", C.c_double)]


class _Trace(C.Structure):
    _fields_ = [("V", _dp), ("Hraw", _dp), ("H", _dp), ("G", _dp), ("C", _dp), ("S", _dp),
                ("k_last", C.c_int32), ("pad_", C.c_int32)]


class _MrepReport(C.Structure):
    _fields_ = [("rows_ridge", C.c_int64), ("rows_fallback", C.c_int64), ("status", C.c_int32),
                ("gate_accepted", C.c_int32), ("max_abs_diag", C.c_double)]


class _StepOpts(C.Structure):
    _fields_ = [("restart", C.c_int32), ("max_cycles", C.c_int32), ("tol", C.c_double), ("d", C.c_int32),
                ("m_max", C.c_int32), ("reset_history", C.c_int32), ("gate", C.c_int32), ("method", C.c_int32),
                ("pad_", C.c_int32)]


METHOD_GMRES, METHOD_CG = 0, 1


class _StepReport(C.Structure):
    _fields_ = [("solve", _SolveReport), ("mrep", _MrepReport), ("precond_was_identity", C.c_int32),
                ("mrep_ran", C.c_int32)]


_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, -O2 -ffp-contract=off, R23)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter", "-o", _SO, src, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.orc_op_rows.restype = C.c_int64
        L.orc_op_rows.argtypes = [C.POINTER(_Operator)]
        L.orc_matvec.argtypes = [C.POINTER(_Operator), _dp, _dp]
        L.orc_thomas.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, _dp]
        L.orc_banded_lu.argtypes = [C.c_int64, C.c_int, _dp, _dp]
        L.orc_banded_lu_solve.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp]
        L.orc_banded_lu_solve.restype = None
        L.orc_banded_matvec.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp]
        L.orc_banded_matvec.restype = None
        L.orc_gate_dominant.argtypes = [C.c_int64, C.c_int, _dp]
        L.orc_pspgmres.argtypes = [C.POINTER(_Operator), _dp, _dp, _dp, C.c_int, _dp, C.c_double, C.c_int,
                                   C.c_int, C.POINTER(_Ring), C.POINTER(_SolveReport), _dp, C.c_int, _dp,
                                   C.c_int, C.POINTER(_Trace)]
        L.orc_pcg.argtypes = [C.POINTER(_Operator), _dp, _dp, _dp, C.c_int, _dp, C.c_double, C.c_int,
                              C.POINTER(_Ring), C.POINTER(_SolveReport), _dp, C.c_int]
        L.orc_sym_bands.argtypes = [C.c_int64, C.c_int, _dp, _dp]
        L.orc_sym_bands.restype = None
        L.orc_gate_spd.argtypes = [C.c_int64, C.c_int, _dp]
        L.orc_mrep.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.c_int64, C.POINTER(C.c_int), C.c_int, _dp, _dp,
                               C.POINTER(C.c_uint8), _dp, C.POINTER(_MrepReport)]
        L.orc_time_steps.argtypes = [C.POINTER(_Operator), _dp, C.c_int, C.POINTER(_StepOpts),
                                     C.POINTER(_Ring), _dp, _dp, C.POINTER(C.c_int), C.POINTER(_StepReport),
                                     _dp, C.c_int]
        L.orc_ring_record.argtypes = [C.POINTER(_Ring), _dp, _dp]
        L.orc_ring_record.restype = None
        L.orc_ring_slot.argtypes = [C.POINTER(_Ring), C.c_int]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _op(spec):
    """Build the C operator struct; returns (struct, keepalive)."""
    o = _Operator()
    o.ndim = int(spec.ndim)
    o.kind = _KINDS[spec.kind]
    n = list(spec.n) + [1] * (3 - len(spec.n))
    for a in range(3):
        o.n[a] = int(n[a])
    o.dt = float(spec.dt)
    o.nu = float(getattr(spec, "nu", 0.0) or 0.0)
    c = list(getattr(spec, "c", None) or [0.0, 0.0, 0.0]) + [0.0] * 3
    for a in range(3):
        o.c[a] = float(c[a])
    keep = []
    fld = getattr(spec, "field", None)
    if fld is not None:
        fld = _f64(np.asarray(fld).reshape(-1))
        keep.append(fld)
        o.field = _p(fld)
    bands = getattr(spec, "bands", None)
    if bands is not None:
        bands = _f64(np.asarray(bands))
        keep.append(bands)
        o.bands = _p(bands)
        o.dA = int(spec.dA)
    return o, keep


def op_rows(spec) -> int:
    o, _k = _op(spec)
    return int(lib().orc_op_rows(C.byref(o)))


def matvec(spec, x):
    o, _k = _op(spec)
    x = _f64(np.asarray(x).reshape(-1))
    y = np.empty_like(x)
    st = lib().orc_matvec(C.byref(o), _p(x), _p(y))
    assert st == OK
    return y


def thomas(sub, diag, sup, v):
    sub, diag, sup, v = (_f64(a) for a in (sub, diag, sup, v))
    z = np.empty_like(v)
    st = lib().orc_thomas(len(v), _p(sub), _p(diag), _p(sup), _p(v), _p(z))
    return st, z


def banded_lu(bands, d):
    bands = _f64(bands)
    n = bands.shape[1]
    lu = np.zeros_like(bands)
    st = lib().orc_banded_lu(n, d, _p(bands), _p(lu))
    return st, lu


def banded_lu_solve(lu, d, v):
    lu = _f64(lu)
    v = _f64(v)
    z = np.empty_like(v)
    lib().orc_banded_lu_solve(len(v), d, _p(lu), _p(v), _p(z))
    return z


def banded_matvec(bands, d, x):
    bands = _f64(bands)
    x = _f64(x)
    y = np.empty_like(x)
    lib().orc_banded_matvec(len(x), d, _p(bands), _p(x), _p(y))
    return y


def gate_dominant(bands, d) -> bool:
    bands = _f64(bands)
    return bool(lib().orc_gate_dominant(bands.shape[1], d, _p(bands)))


class Ring:
    """FIFO probe ring (R20) held in numpy arrays: px/py are (cap, n) row-major = column-major n x cap."""

    def __init__(self, n: int, cap: int):
        self.px = np.zeros((cap, n))
        self.py = np.zeros((cap, n))
        self.s = _Ring()
        self.s.n, self.s.cap, self.s.count, self.s.head = n, cap, 0, 0
        self.s.px, self.s.py = _p(self.px), _p(self.py)

    @property
    def count(self):
        return self.s.count

    def order(self):
        return [(self.s.head + c) % self.s.cap for c in range(self.s.count)]

    def columns(self):
        """(P_x, P_y) as (m, n) arrays, oldest -> newest."""
        o = self.order()
        return self.px[o], self.py[o]

    def record(self, x, y):
        x, y = _f64(x), _f64(y)
        lib().orc_ring_record(C.byref(self.s), _p(x), _p(y))


def _report(r: _SolveReport) -> dict:
    return {k: getattr(r, k) for k, _ in _SolveReport._fields_}


def pspgmres(spec, b, x0, eps, n_A, n_r, d=1, lu=None, ring: Ring | None = None, trace=False,
             hist_cap=None):
    """Literal Algorithm 1.  Returns dict(x, report, resid_hist, beta_hist[, trace arrays])."""
    o, _k = _op(spec)
    b = _f64(np.asarray(b).reshape(-1))
    x0 = _f64(np.asarray(x0).reshape(-1))
    n = len(b)
    x = np.empty_like(b)
    hist_cap = hist_cap or n_A * n_r
    hist = np.zeros(hist_cap)
    betas = np.zeros(n_r)
    rep = _SolveReport()
    tr = None
    arrs = {}
    if trace:
        tr = _Trace()
        arrs = dict(V=np.zeros((n_A + 1, n)), Hraw=np.zeros((n_A, n_A + 1)), H=np.zeros((n_A, n_A + 1)),
                    G=np.zeros(n_A + 1), C=np.zeros(n_A), S=np.zeros(n_A))
        for k_, a in arrs.items():
            setattr(tr, k_, _p(a))
    lu_a = _f64(lu) if lu is not None else None
    st = lib().orc_pspgmres(C.byref(o), _p(b), _p(x0), _p(x), d, _p(lu_a), float(eps), n_A, n_r,
                            C.byref(ring.s) if ring is not None else None, C.byref(rep), _p(hist), hist_cap,
                            _p(betas), n_r, C.byref(tr) if tr is not None else None)
    out = dict(status=st, x=x, report=_report(rep), resid_hist=hist[:min(rep.hist_len, hist_cap)],
               beta_hist=betas[:min(rep.beta_len, n_r)])
    if trace:
        # column-major (n_A+1) x n_A stored as (n_A, n_A+1) rows -> transpose to (n_A+1, n_A)
        out["trace"] = dict(V=arrs["V"].T.copy(), Hraw=arrs["Hraw"].T.copy(), H=arrs["H"].T.copy(),
                            G=arrs["G"], C=arrs["C"], S=arrs["S"], k_last=tr.k_last)
    return out


def pcg(spec, b, x0, eps, max_iters, d=1, lu=None, ring: Ring | None = None, hist_cap=None):
    """f4: preconditioned CG with probe recording (orc_pcg, readings R27-R31).  lu = LU factors of the
    (symmetric) preconditioner, None for M = I.  Returns dict(x, report, resid_hist)."""
    o, _k = _op(spec)
    b = _f64(np.asarray(b).reshape(-1))
    x0 = _f64(np.asarray(x0).reshape(-1))
    x = np.empty_like(b)
    hist_cap = hist_cap or max_iters
    hist = np.zeros(hist_cap)
    rep = _SolveReport()
    lu_a = _f64(lu) if lu is not None else None
    st = lib().orc_pcg(C.byref(o), _p(b), _p(x0), _p(x), d, _p(lu_a), float(eps), int(max_iters),
                       C.byref(ring.s) if ring is not None else None, C.byref(rep), _p(hist), hist_cap)
    return dict(status=st, x=x, report=_report(rep), resid_hist=hist[:min(rep.hist_len, hist_cap)])


def sym_bands(bands, d):
    """R29: N_s = (N + N^T) / 2 in DIA storage."""
    bands = _f64(bands)
    out = np.zeros_like(bands)
    lib().orc_sym_bands(bands.shape[1], d, _p(bands), _p(out))
    return out


def gate_spd(bands, d) -> bool:
    bands = _f64(bands)
    return bool(lib().orc_gate_spd(bands.shape[1], d, _p(bands)))


def mrep(px, py, d, order=None):
    """Literal Algorithm 2.  px, py: (m, n) arrays (row c = probe column c, oldest -> newest
    unless ``order`` gives the slot of each column)."""
    px = _f64(px)
    py = _f64(py)
    m, n = px.shape
    if order is not None:
        m = len(order)
        order_a = (C.c_int * m)(*order)
    else:
        order_a = None
    bands = np.zeros((2 * d + 1, n))
    icpt = np.zeros(n)
    kind = np.zeros(n, dtype=np.uint8)
    kap = np.zeros(n)
    rep = _MrepReport()
    st = lib().orc_mrep(n, m, _p(px), _p(py), n, order_a, d, _p(bands), _p(icpt),
                        kind.ctypes.data_as(C.POINTER(C.c_uint8)), _p(kap), C.byref(rep))
    return dict(status=st, bands=bands, intercept=icpt, row_kind=kind, kappa_est=kap,
                rows_ridge=rep.rows_ridge, rows_fallback=rep.rows_fallback, gate_accepted=bool(rep.gate_accepted),
                max_abs_diag=rep.max_abs_diag)


class Driver:
    """O5 one step at a time, keeping the ring and N across calls (for lockstep parity)."""

    def __init__(self, spec, n, restart, max_cycles, tol, d, m_max, reset_history=False, gate=True,
                 method=METHOD_GMRES):
        self.spec = spec
        self.n = n
        self.d = d
        self.ring = Ring(n, m_max)
        self.bands = np.zeros((2 * d + 1, n))
        self.lu = np.zeros((2 * d + 1, n))
        self.ident = C.c_int(1)
        self.opts = _StepOpts(restart, max_cycles, float(tol), d, m_max, int(reset_history), int(gate), int(method))
        self.hist_cap = restart * max_cycles

    def step(self, u):
        """Returns dict(u_next, report, N_used=(bands copy or None for I), resid_hist)."""
        o, _k = _op(self.spec)
        uu = _f64(np.asarray(u).reshape(-1)).copy()
        n_used = None if self.ident.value else self.bands.copy()
        rep = (_StepReport * 1)()
        hist = np.zeros(self.hist_cap)
        st = lib().orc_time_steps(C.byref(o), _p(uu), 1, C.byref(self.opts), C.byref(self.ring.s), _p(self.bands),
                                  _p(self.lu), C.byref(self.ident), rep, _p(hist), self.hist_cap)
        r = rep[0]
        sr = _report(r.solve)
        return dict(status=st, u=uu, N_used=n_used, solve=sr, resid_hist=hist[:sr["hist_len"]].copy(),
                    mrep=dict(rows_ridge=r.mrep.rows_ridge, rows_fallback=r.mrep.rows_fallback,
                              gate_accepted=bool(r.mrep.gate_accepted)),
                    precond_was_identity=bool(r.precond_was_identity), mrep_ran=bool(r.mrep_ran))


def time_steps(spec, u0, steps, restart, max_cycles, tol, d, m_max, reset_history=False, gate=True,
               hist_cap=None, method=METHOD_GMRES):
    """O5: the implicit-Euler driver.  Returns dict(u, reports, resid_hist, bands, is_identity)."""
    o, _k = _op(spec)
    u = _f64(np.asarray(u0).reshape(-1)).copy()
    n = len(u)
    assert m_max <= 4096
    ring = Ring(n, m_max)
    bands = np.zeros((2 * d + 1, n))
    lu = np.zeros((2 * d + 1, n))
    ident = C.c_int(1)
    reps = (_StepReport * steps)()
    hist_cap = hist_cap or restart * max_cycles * steps
    hist = np.zeros(hist_cap)
    opts = _StepOpts(restart, max_cycles, float(tol), d, m_max, int(reset_history), int(gate), int(method))
    st = lib().orc_time_steps(C.byref(o), _p(u), steps, C.byref(opts), C.byref(ring.s), _p(bands), _p(lu),
                              C.byref(ident), reps, _p(hist), hist_cap)
    reports = []
    used = 0
    for s in range(steps):
        r = reps[s]
        sr = _report(r.solve)
        reports.append(dict(solve=sr, mrep=dict(rows_ridge=r.mrep.rows_ridge, rows_fallback=r.mrep.rows_fallback,
                                                status=r.mrep.status, gate_accepted=bool(r.mrep.gate_accepted),
                                                max_abs_diag=r.mrep.max_abs_diag),
                            precond_was_identity=bool(r.precond_was_identity), mrep_ran=bool(r.mrep_ran),
                            resid_hist=hist[used:used + sr["hist_len"]].copy()))
        used += sr["hist_len"]
    return dict(status=st, u=u, reports=reports, bands=bands, is_identity=bool(ident.value), ring=ring)
