"""ctypes binding of libpspgmres (include/pspgmres.h).  Argument marshalling only.

Every numeric step of the hot path runs in the library's sm_100a kernels; this module turns
torch tensors into device pointers, numpy arrays into host pointers, and C structs into
dicts.  PyTorch supplies device memory (the workspace is a torch uint8 tensor) and the CUDA
stream.  There is no fallback: if libpspgmres.so is missing or the GPU is absent, ``lib()``
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSP_LIB: tuning experiments only (an alternative build of the same sources)
LIB_PATH = os.environ.get("PSP_LIB") or os.path.join(_HERE, "libpspgmres.so")

# ---- enums (include/pspgmres.h) ----
PSP_OK, PSP_E_ARG, PSP_E_DIM, PSP_E_SAMPLES, PSP_E_RANK, PSP_E_SINGULAR, PSP_E_NONFINITE, \
    PSP_E_NOCONV, PSP_E_CUDA, PSP_E_NCCL, PSP_E_NOMEM = range(11)
PSP_OP_CONST_DIFF, PSP_OP_CELL_DIFF, PSP_OP_CELL_ADVDIFF, PSP_OP_DIA = range(4)
PSP_TOL_REL_B, PSP_TOL_ABS = 0, 1
PSP_MGS_1REDUCE, PSP_MGS_LITERAL = 0, 1
PSP_METHOD_GMRES, PSP_METHOD_CG = 0, 1
PSP_FLAG_CONVERGED, PSP_FLAG_BREAKDOWN, PSP_FLAG_NONFINITE = 1, 2, 4
PSP_KC_COUNT = 14
ROW_INTERIOR, ROW_INTERIOR_RIDGE, ROW_BOUNDARY, ROW_FALLBACK_RANK, ROW_FALLBACK_ZEROVAR, \
    ROW_FALLBACK_SMALLDIAG = range(6)
KIND_CODES = {"const_diff": PSP_OP_CONST_DIFF, "cell_diff": PSP_OP_CELL_DIFF,
              "cell_advdiff": PSP_OP_CELL_ADVDIFF, "dia": PSP_OP_DIA}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class psp_grid(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("pad_", C.c_int32), ("n", C.c_int64 * 3)]


class psp_stencil(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dA", C.c_int32), ("nu", C.c_double), ("c", C.c_double * 3),
                ("d_field", _vp), ("d_bands", _vp)]


class psp_opts(C.Structure):
    _fields_ = [("max_cycles", C.c_int32), ("tol_mode", C.c_int32), ("m_max", C.c_int32),
                ("reset_history_per_step", C.c_int32), ("ortho", C.c_int32), ("gate", C.c_int32),
                ("timing", C.c_int32), ("fused", C.c_int32), ("fused_kmin", C.c_int32),
                ("fused_kmax", C.c_int32), ("fused_split_cols", C.c_int32), ("resident", C.c_int32),
                ("method", C.c_int32), ("mrep_stream", C.c_int32)]


class psp_report(C.Structure):
    _fields_ = [("status", C.c_int32), ("converged", C.c_int32), ("iterations", C.c_int32),
                ("cycles", C.c_int32), ("matvecs", C.c_int32), ("precond_applies", C.c_int32),
                ("precond_identity", C.c_int32), ("resid_cap", C.c_int32), ("resid_len", C.c_int32),
                ("beta_cap", C.c_int32), ("beta_len", C.c_int32), ("mrep_ran", C.c_int32),
                ("mrep_status", C.c_int32), ("mrep_gate_accepted", C.c_int32),
                ("mrep_rows_ridge", C.c_int64), ("mrep_rows_fallback", C.c_int64),
                ("mrep_rows_nondominant", C.c_int64), ("r0", C.c_double), ("eps", C.c_double),
                ("final_resid_est", C.c_double), ("final_resid_true", C.c_double),
                ("mrep_max_abs_diag", C.c_double), ("t_solve_ms", C.c_double), ("t_mrep_ms", C.c_double),
                ("t_factor_ms", C.c_double), ("h_resid_history", _dp), ("h_beta_history", _dp),
                ("resid_verified", C.c_int32), ("pad_", C.c_int32)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, C.c_size_t, C.c_int)
SENDRECV_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _dp, C.c_size_t, _dp, _dp, C.c_size_t)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _dp, C.c_size_t)


class psp_host_transport(C.Structure):
    _fields_ = [("user", _vp), ("allreduce", ALLREDUCE_FN), ("sendrecv", SENDRECV_FN), ("allgather", ALLGATHER_FN)]


class psp_mrep_info(C.Structure):
    _fields_ = [("rows_ridge", C.c_int64), ("rows_fallback", C.c_int64), ("rows_nondominant", C.c_int64),
                ("max_abs_diag", C.c_double), ("gate_accepted", C.c_int32), ("status", C.c_int32)]


class PspError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libpspgmres status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libpspgmres.so.  Fails loudly: there is no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(or `make`) -- libpspgmres has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "psp_default_opts": (None, [P(psp_opts)]),
        "psp_workspace_bytes": (C.c_int, [P(psp_grid), P(psp_stencil), C.c_int, C.c_int, P(psp_opts), _vp,
                                           P(C.c_size_t)]),
        "psp_create": (C.c_int, [P(psp_grid), P(psp_stencil), C.c_double, C.c_int, C.c_int, C.c_double,
                                 P(psp_opts), _vp, C.c_size_t, _vp, _vp, P(_vp)]),
        "psp_destroy": (C.c_int, [_vp]),
        "psp_local_rows": (C.c_int, [_vp, P(C.c_int64), P(C.c_int64)]),
        "psp_matvec": (C.c_int, [_vp, _vp, _vp, C.c_int]),
        "psp_precond_apply": (C.c_int, [_vp, _vp, _vp]),
        "psp_cycle_begin": (C.c_int, [_vp, _vp, _vp, P(C.c_double)]),
        "psp_arnoldi_step": (C.c_int, [_vp, C.c_int, P(C.c_double), P(C.c_int)]),
        "psp_cycle_end": (C.c_int, [_vp, C.c_int, _vp]),
        "psp_solve": (C.c_int, [_vp, _vp, _vp, _vp, P(psp_report)]),
        "psp_mrep_fit": (C.c_int, [_vp, P(psp_report)]),
        "psp_step": (C.c_int, [_vp, _vp, _vp, P(psp_report)]),
        "psp_raw_scratch_bytes": (C.c_int, [C.c_int64, C.c_int, P(C.c_size_t)]),
        "psp_mrep_fit_raw": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, C.c_int64, P(C.c_int32), C.c_int, _vp, _vp,
                                       _vp, _vp, _vp, C.c_size_t, _vp, P(psp_mrep_info)]),
        "psp_banded_factor_raw": (C.c_int, [_vp, C.c_int64, C.c_int, _vp, _vp, C.c_size_t, _vp]),
        "psp_banded_solve_raw": (C.c_int, [_vp, C.c_int64, C.c_int, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
        "psp_set_bands": (C.c_int, [_vp, _vp, P(C.c_int)]),
        "psp_get_bands": (C.c_int, [_vp, _vp, P(C.c_int)]),
        "psp_inject_fault_rows": (C.c_int, [_vp, P(C.c_int64), C.c_int, P(C.c_int)]),
        "psp_ring_view": (C.c_int, [_vp, P(C.c_int), P(C.c_int32), _dp, P(_vp), P(_vp), P(C.c_int64)]),
        "psp_ring_reset": (C.c_int, [_vp]),
        "psp_get_hessenberg": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp]),
        "psp_get_basis": (C.c_int, [_vp, C.c_int, P(_vp), P(C.c_double)]),
        "psp_launch_count": (C.c_int, [_vp, P(C.c_int64)]),
        "psp_kernel_stats": (C.c_int, [_vp, _dp, _dp, P(C.c_int64), C.c_int]),
        "psp_set_timing": (C.c_int, [_vp, C.c_int]),
        "psp_kernel_class_name": (C.c_char_p, [C.c_int]),
        "psp_status_str": (C.c_char_p, [C.c_int]),
        "psp_last_error": (C.c_char_p, [_vp]),
        "psp_version": (C.c_char_p, []),
        "psp_comm_unique_id": (C.c_int, [_vp]),
        "psp_comm_init": (C.c_int, [_vp, C.c_int, C.c_int, P(_vp)]),
        "psp_comm_loopback_create": (C.c_int, [C.c_int, P(_vp)]),
        "psp_comm_host_create": (C.c_int, [P(psp_host_transport), C.c_int, C.c_int, P(_vp)]),
        "psp_comm_destroy": (C.c_int, [_vp]),
        "psp_comm_selftest": (C.c_int, [_vp, _vp]),
        "psp_partition": (C.c_int, [P(psp_grid), C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                    P(C.c_int64)]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("PSP_LIB") and not hasattr(L, name):
            continue                    # an older build under A/B (tools/): bind what it has
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["psp_default_opts", "psp_workspace_bytes", "psp_create", "psp_destroy", "psp_local_rows",
            "psp_matvec", "psp_precond_apply", "psp_cycle_begin", "psp_arnoldi_step", "psp_cycle_end",
            "psp_solve", "psp_mrep_fit", "psp_step", "psp_raw_scratch_bytes", "psp_mrep_fit_raw",
            "psp_banded_factor_raw", "psp_banded_solve_raw", "psp_set_bands", "psp_get_bands", "psp_inject_fault_rows",
            "psp_ring_view",
            "psp_ring_reset", "psp_get_hessenberg", "psp_get_basis", "psp_launch_count", "psp_kernel_stats",
            "psp_set_timing",
            "psp_kernel_class_name", "psp_status_str",
            "psp_last_error", "psp_version", "psp_comm_unique_id", "psp_comm_init", "psp_comm_loopback_create",
            "psp_comm_host_create", "psp_comm_destroy", "psp_comm_selftest", "psp_partition"]


def psp_partition(n_axes, nranks, rank):
    """(row0, nrows, slab0, slab_len) of rank's slab (pure host function of the library)."""
    g = make_grid(n_axes)
    out = [C.c_int64() for _ in range(4)]
    _check(lib().psp_partition(C.byref(g), nranks, rank, *[C.byref(o) for o in out]))
    return tuple(o.value for o in out)


def psp_comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().psp_comm_unique_id(buf))
    return bytes(buf)


def psp_comm_init(uid: bytes, nranks: int, rank: int):
    h = _vp()
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check(lib().psp_comm_init(buf, nranks, rank, C.byref(h)))
    return h


def psp_comm_loopback_create(nranks: int):
    arr = (_vp * nranks)()
    _check(lib().psp_comm_loopback_create(nranks, arr))
    return [_vp(a) for a in arr]


class TorchDistTransport:
    """The host collectives of psp_comm_host_create carried by torch.distributed on CPU tensors (a
    gloo process group): argument marshalling only -- the library stages device data through
    pinned host buffers around each call.  Keep the object alive while the communicator lives
    (it owns the ctypes callbacks)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._ops = [dist.ReduceOp.SUM, dist.ReduceOp.MAX, dist.ReduceOp.MIN]
        self._cbs = (ALLREDUCE_FN(self._allreduce), SENDRECV_FN(self._sendrecv), ALLGATHER_FN(self._allgather))
        self.struct = psp_host_transport(None, *self._cbs)

    @staticmethod
    def _t(ptr, count):
        import torch
        return torch.from_numpy(np.ctypeslib.as_array(ptr, shape=(count,)))

    def _allreduce(self, user, buf, count, op):
        try:
            self.dist.all_reduce(self._t(buf, count), op=self._ops[op], group=self.group)
            return 0
        except Exception:  # noqa: BLE001 -- a failed collective is PSP_E_NCCL in the library
            return 1

    def _sendrecv(self, user, send_lo, recv_lo, n_lo, send_hi, recv_hi, n_hi):
        try:
            reqs = []
            if n_lo:
                reqs.append(self.dist.isend(self._t(send_lo, n_lo), self.rank - 1, group=self.group))
                reqs.append(self.dist.irecv(self._t(recv_lo, n_lo), self.rank - 1, group=self.group))
            if n_hi:
                reqs.append(self.dist.isend(self._t(send_hi, n_hi), self.rank + 1, group=self.group))
                reqs.append(self.dist.irecv(self._t(recv_hi, n_hi), self.rank + 1, group=self.group))
            for r in reqs:
                r.wait()
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _allgather(self, user, send, recv, count):
        try:
            out = self._t(recv, count * self.world)
            self.dist.all_gather(list(out.split(count)), self._t(send, count).clone(), group=self.group)
            return 0
        except Exception:  # noqa: BLE001
            return 1


def psp_comm_host_create(transport: TorchDistTransport, nranks: int, rank: int):
    h = _vp()
    _check(lib().psp_comm_host_create(C.byref(transport.struct), nranks, rank, C.byref(h)))
    return h


def psp_comm_destroy(h):
    lib().psp_comm_destroy(h)


def psp_comm_selftest(h, stream=None):
    """Every collective of the hot path on small device buffers, checked against closed forms
    (collective: every rank calls it).  Returns the status (PSP_OK on success)."""
    sp = _vp(stream.cuda_stream) if stream is not None else None
    return lib().psp_comm_selftest(h, sp)


def _check(st, ctx=None, allow=(PSP_OK,)):
    if st not in allow:
        msg = lib().psp_last_error(ctx).decode()
        raise PspError(st, msg)
    return st


def _ptr(t):
    """device pointer of a torch CUDA tensor (or None)."""
    if t is None:
        return None
    assert t.is_cuda, "libpspgmres takes device tensors"
    assert t.is_contiguous()
    return t.data_ptr()


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def default_opts(**kw) -> psp_opts:
    o = psp_opts()
    lib().psp_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, int(v))
    return o


def make_grid(n_axes) -> psp_grid:
    g = psp_grid()
    g.ndim = len(n_axes)
    for a in range(3):
        g.n[a] = int(n_axes[a]) if a < len(n_axes) else 1
    return g


def make_stencil(op, d_field=None, d_bands=None) -> psp_stencil:
    s = psp_stencil()
    s.kind = KIND_CODES[op.kind]
    s.dA = int(getattr(op, "dA", 0) or 0)
    s.nu = float(getattr(op, "nu", 1.0) or 0.0)
    c = list(getattr(op, "c", (0, 0, 0)) or (0, 0, 0)) + [0.0] * 3
    for a in range(3):
        s.c[a] = float(c[a])
    s.d_field = _ptr(d_field)
    s.d_bands = _ptr(d_bands)
    return s


def report_dict(r: psp_report, hist=None, betas=None) -> dict:
    out = {k: getattr(r, k) for k, _ in psp_report._fields_ if not k.startswith("h_")}
    if hist is not None:
        out["resid_history"] = hist[:min(r.resid_len, r.resid_cap)].copy()
    if betas is not None:
        out["beta_history"] = betas[:min(r.beta_len, r.beta_cap)].copy()
    return out


class Context:
    """Owns a psp_ctx and its torch workspace.  Methods map 1:1 onto the C ABI."""

    def __init__(self, op, d, restart, tol, opts: psp_opts | None = None, device="cuda", stream=None,
                 hist_cap=1 << 16, comm=None, nranks=1, rank=0, field_local=None):
        """comm: a psp_comm handle (None: one rank).  With nranks > 1 the context owns rank's
        psp_partition slab: vectors passed to it are local rows [row0, row0 + n); the coefficient
        field is sliced from op.field unless field_local (a local CUDA tensor) is given."""
        import torch
        self.torch = torch
        self.op = op
        self.nranks, self.rank = nranks, rank
        self.row0, self.n, _, _ = psp_partition(op.n, nranks, rank)
        self.d = d
        self.restart = restart
        self.device = torch.device(device)
        self.stream = stream
        self._field = None
        self._bands = None
        if field_local is not None:
            self._field = field_local
        elif op.field is not None:
            f = np.asarray(op.field, dtype=np.float64).reshape(-1)[self.row0:self.row0 + self.n]
            self._field = torch.as_tensor(np.ascontiguousarray(f)).to(self.device)
        if op.kind == "dia":
            self._bands = torch.as_tensor(np.asarray(op.bands, dtype=np.float64)).to(self.device).contiguous()
        self.grid = make_grid(op.n)
        self.stencil = make_stencil(op, self._field, self._bands)
        self.opts = opts if opts is not None else default_opts()
        self.comm = comm
        nbytes = C.c_size_t(0)
        _check(lib().psp_workspace_bytes(C.byref(self.grid), C.byref(self.stencil), d, restart,
                                         C.byref(self.opts), comm, C.byref(nbytes)))
        self.ws_bytes = nbytes.value
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        h = _vp()
        _check(lib().psp_create(C.byref(self.grid), C.byref(self.stencil), float(op.dt), d, restart, float(tol),
                                C.byref(self.opts), self.ws.data_ptr(), self.ws_bytes, _stream_ptr(stream), comm,
                                C.byref(h)))
        self.h = h
        self.hist = np.zeros(hist_cap)
        self.betas = np.zeros(hist_cap)

    def close(self):
        if self.h:
            lib().psp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _report(self):
        r = psp_report()
        r.h_resid_history = self.hist.ctypes.data_as(_dp)
        r.resid_cap = len(self.hist)
        r.h_beta_history = self.betas.ctypes.data_as(_dp)
        r.beta_cap = len(self.betas)
        return r

    # ---- the C ABI, same names ----
    def psp_matvec(self, x, y, record=False):
        _check(lib().psp_matvec(self.h, _ptr(x), _ptr(y), int(record)), self.h)

    def psp_precond_apply(self, v, z):
        _check(lib().psp_precond_apply(self.h, _ptr(v), _ptr(z)), self.h)

    def psp_cycle_begin(self, b, x0):
        beta = C.c_double()
        _check(lib().psp_cycle_begin(self.h, _ptr(b), _ptr(x0), C.byref(beta)), self.h)
        return beta.value

    def psp_arnoldi_step(self, k):
        r = C.c_double()
        f = C.c_int()
        _check(lib().psp_arnoldi_step(self.h, k, C.byref(r), C.byref(f)), self.h)
        return r.value, f.value

    def psp_cycle_end(self, k, x):
        _check(lib().psp_cycle_end(self.h, k, _ptr(x)), self.h)

    def psp_solve(self, b, x0, x):
        r = self._report()
        st = lib().psp_solve(self.h, _ptr(b), _ptr(x0), _ptr(x), C.byref(r))
        _check(st, self.h, allow=(PSP_OK, PSP_E_NOCONV))
        return report_dict(r, self.hist, self.betas)

    def psp_mrep_fit(self):
        r = self._report()
        st = lib().psp_mrep_fit(self.h, C.byref(r))
        _check(st, self.h, allow=(PSP_OK, PSP_E_SAMPLES))
        return report_dict(r)

    def psp_step(self, u_n, u_np1):
        r = self._report()
        st = lib().psp_step(self.h, _ptr(u_n), _ptr(u_np1), C.byref(r))
        _check(st, self.h, allow=(PSP_OK, PSP_E_NOCONV))
        return report_dict(r, self.hist, self.betas)

    def psp_set_bands(self, bands):
        acc = C.c_int()
        _check(lib().psp_set_bands(self.h, _ptr(bands), C.byref(acc)), self.h)
        return bool(acc.value)

    def psp_inject_fault_rows(self, rows):
        arr = (C.c_int64 * len(rows))(*[int(r) for r in rows])
        acc = C.c_int()
        _check(lib().psp_inject_fault_rows(self.h, arr, len(rows), C.byref(acc)), self.h)
        return bool(acc.value)

    def psp_get_bands(self):
        out = self.torch.empty((2 * self.d + 1, self.n), dtype=self.torch.float64, device=self.device)
        ident = C.c_int()
        _check(lib().psp_get_bands(self.h, _ptr(out), C.byref(ident)), self.h)
        return out, bool(ident.value)

    def psp_ring_view(self):
        """(count, slots, P_x, P_y): the recorded probes oldest -> newest as new (count, n) tensors
        (each column times its recorded scale)."""
        cnt = C.c_int()
        slots = (C.c_int32 * 257)()
        scale = np.zeros(257)
        px, py = _vp(), _vp()
        ld = C.c_int64()
        _check(lib().psp_ring_view(self.h, C.byref(cnt), slots, scale.ctypes.data_as(_dp), C.byref(px),
                                   C.byref(py), C.byref(ld)), self.h)
        base = self.ws.data_ptr()
        phys = self.opts.m_max + 1
        t = self.torch
        ws64 = self.ws.view(t.float64)
        L = ld.value                     # column stride (multi-rank columns carry ghost planes)
        PXr = ws64[(px.value - base) // 8:(px.value - base) // 8 + (phys - 1) * L + self.n].as_strided((phys, self.n), (L, 1))
        PYr = ws64[(py.value - base) // 8:(py.value - base) // 8 + (phys - 1) * L + self.n].as_strided((phys, self.n), (L, 1))
        m = cnt.value
        sl = list(slots[:m])
        sc = t.tensor(scale[:m], dtype=t.float64, device=self.device)[:, None]
        return m, sl, PXr[sl] * sc, PYr[sl] * sc

    def psp_ring_reset(self):
        _check(lib().psp_ring_reset(self.h), self.h)

    def psp_get_hessenberg(self):
        nA = self.restart
        H = np.zeros(nA * (nA + 1))
        Hraw = np.zeros(nA * (nA + 1))
        G = np.zeros(nA + 1)
        Cc = np.zeros(nA)
        S = np.zeros(nA)
        _check(lib().psp_get_hessenberg(self.h, H.ctypes.data_as(_dp), Hraw.ctypes.data_as(_dp),
                                        G.ctypes.data_as(_dp), Cc.ctypes.data_as(_dp), S.ctypes.data_as(_dp)), self.h)
        return dict(H=H.reshape(nA, nA + 1).T.copy(), Hraw=Hraw.reshape(nA, nA + 1).T.copy(), G=G, C=Cc, S=S)

    def psp_get_basis(self, j):
        """V(:,j) as a new tensor (stored column times its lagged normalisation)."""
        p = _vp()
        sc = C.c_double()
        _check(lib().psp_get_basis(self.h, j, C.byref(p), C.byref(sc)), self.h)
        base = self.ws.data_ptr()
        off = (p.value - base) // 8
        return self.ws.view(self.torch.float64)[off:off + self.n] * sc.value

    def psp_launch_count(self):
        v = C.c_int64()
        _check(lib().psp_launch_count(self.h, C.byref(v)), self.h)
        return v.value

    def psp_set_timing(self, level):
        _check(lib().psp_set_timing(self.h, int(level)), self.h)

    def psp_kernel_stats(self, reset=True):
        """{class name: dict(ms, bytes, launches)} (needs opts.timing >= 2)."""
        K = PSP_KC_COUNT
        ms = np.zeros(K)
        by = np.zeros(K)
        cnt = (C.c_int64 * K)()
        _check(lib().psp_kernel_stats(self.h, ms.ctypes.data_as(_dp), by.ctypes.data_as(_dp), cnt, int(reset)),
               self.h)
        return {lib().psp_kernel_class_name(k).decode(): dict(ms=float(ms[k]), bytes=float(by[k]),
                                                             launches=int(cnt[k])) for k in range(K)}


def raw_scratch(n, d, device="cuda"):
    import torch
    b = C.c_size_t()
    _check(lib().psp_raw_scratch_bytes(n, d, C.byref(b)))
    return torch.zeros(b.value, dtype=torch.uint8, device=device)


def psp_mrep_fit_raw(px, py, d, order=None, scratch=None, stream=None, want_kind=True):
    """px, py: (cap, n) CUDA tensors (row = probe column).  Returns dict of tensors + info."""
    import torch
    cap, n = px.shape
    m = len(order) if order is not None else cap
    order_a = (C.c_int32 * m)(*order) if order is not None else None
    bands = torch.empty((2 * d + 1, n), dtype=torch.float64, device=px.device)
    icpt = torch.empty(n, dtype=torch.float64, device=px.device)
    kind = torch.empty(n, dtype=torch.uint8, device=px.device) if want_kind else None
    kap = torch.empty(n, dtype=torch.float64, device=px.device) if want_kind else None
    if scratch is None:
        scratch = raw_scratch(n, d, px.device)
    info = psp_mrep_info()
    st = lib().psp_mrep_fit_raw(_ptr(px), _ptr(py), n, m, n, order_a, d, _ptr(bands), _ptr(icpt), _ptr(kind),
                                _ptr(kap), scratch.data_ptr(), scratch.numel(), _stream_ptr(stream), C.byref(info))
    _check(st, None, allow=(PSP_OK, PSP_E_SAMPLES))
    return dict(status=st, bands=bands, intercept=icpt, row_kind=kind, kappa_est=kap,
                rows_ridge=info.rows_ridge, rows_fallback=info.rows_fallback,
                rows_nondominant=info.rows_nondominant, gate_accepted=bool(info.gate_accepted),
                max_abs_diag=info.max_abs_diag)


def psp_banded_factor_raw(bands, d, scratch=None, stream=None):
    import torch
    n = bands.shape[1]
    lu = torch.zeros_like(bands)
    if scratch is None:
        scratch = raw_scratch(n, d, bands.device)
    st = lib().psp_banded_factor_raw(_ptr(bands), n, d, _ptr(lu), scratch.data_ptr(), scratch.numel(),
                                     _stream_ptr(stream))
    _check(st, None, allow=(PSP_OK, PSP_E_SINGULAR))
    return st, lu


def psp_banded_solve_raw(lu, d, v, x0=None, scratch=None, stream=None, out=None):
    import torch
    n = lu.shape[1]
    z = out if out is not None else torch.empty_like(v)
    if scratch is None:
        scratch = raw_scratch(n, d, lu.device)
    _check(lib().psp_banded_solve_raw(_ptr(lu), n, d, _ptr(v), _ptr(x0), _ptr(z), scratch.data_ptr(),
                                      scratch.numel(), _stream_ptr(stream)))
    return z
