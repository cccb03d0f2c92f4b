/*
 * pspgmres.h -- C ABI of libpspgmres, the B200 (sm_100a) hot path of PSP-GMRES
 * (arXiv 1308.5626, "Progressive Statistical Preconditioning").
 *
 * Citations: "P:n" = line n of the paper text; "S:n" = line n of SPEC.md;
 * "Alg.1 l.N" = Algorithm 1 line N (algorithm2e numbering); "Rnn" = a reading of
 * the paper listed in DESIGN.md section 3.
 *
 * Conventions for every entry point
 *   - All floating point is IEEE FP64.  "d_" = device pointer, "h_" = host pointer.
 *   - A grid vector is lexicographic, x fastest: g = i + nx*(j + ny*k).
 *     Probe (P_x, P_y) and Krylov (V) matrices are column-major, one contiguous column per
 *     vector.  Banded matrices use DIA storage band[o*n + i] = N(i, i+o-d), o = 0..2d
 *     (entries addressing columns outside 0..n-1 are ignored / written as 0).
 *   - Every call is stream-ordered on the stream given to psp_create (a cudaStream_t passed
 *     as void*).  Calls that return host values synchronise that stream.
 *   - The caller owns every buffer it passes (vectors, fields, the workspace, host report
 *     arrays).  The library owns the context and never allocates device memory after
 *     psp_create: everything lives in the caller's workspace (sized by psp_workspace_bytes).
 *     It allocates a few hundred bytes of pinned host memory for device->host scalars.
 *   - Errors: every function returns psp_status and never throws; psp_last_error() gives
 *     the message.  CUDA failures (PSP_E_CUDA) are sticky: the context must be destroyed.
 *   - A context is single-writer.  The factorisation of N is immutable
 *     between fits.
 */
#ifndef PSPGMRES_H
#define PSPGMRES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PSP_OK = 0,
  PSP_E_ARG = 1,        /* bad configuration                         */
  PSP_E_DIM = 2,        /* dimension / contract violation         */
  PSP_E_SAMPLES = 3,    /* MREP with m < 2d+2 samples (R19)                          */
  PSP_E_RANK = 4,       /* rank-deficient fit -- rows fall back, the call succeeds   */
  PSP_E_SINGULAR = 5,   /* singular projection / zero pivot                  */
  PSP_E_NONFINITE = 6,  /* non-finite value, partial report                         */
  PSP_E_NOCONV = 7,     /* n_r restart cycles exhausted, full report             */
  PSP_E_CUDA = 8,       /* CUDA runtime failure (sticky)                                    */
  PSP_E_NCCL = 9,       /* NCCL failure (sticky)                                            */
  PSP_E_NOMEM = 10      /* workspace too small                                              */
} psp_status;

typedef struct psp_ctx psp_ctx;   /* opaque, host side, owned by the library                 */
typedef struct psp_comm psp_comm; /* opaque wrapper of an ncclComm_t; NULL = one GPU          */

/* Grid of interior points (R24: x_i = i*h, h = 1/(n+1) per axis, u = 0 outside). */
typedef struct {
  int32_t ndim;   /* 1, 2 or 3                                                              */
  int32_t pad_;
  int64_t n[3];   /* GLOBAL interior points per axis, n[0] = nx (fastest); unused axes = 1  */
} psp_grid;

/* Operator kinds of A = I - dt*L (Eq.4), applied matrix-free (R24). */
enum {
  PSP_OP_CONST_DIFF = 0,   /* L = nu * Laplacian, central second differences (C1, C2)       */
  PSP_OP_CELL_DIFF = 1,    /* L = div(kappa grad), arithmetic-mean faces (C4)               */
  PSP_OP_CELL_ADVDIFF = 2, /* L = -c.grad + div(nu grad), first-order upwind, c_a >= 0 (C3) */
  PSP_OP_DIA = 3           /* A given as a DIA banded matrix (tests; the paper's P:142 case) */
};

typedef struct {
  int32_t kind;            /* PSP_OP_*                                                      */
  int32_t dA;              /* half-bandwidth of a PSP_OP_DIA operator                        */
  double nu;               /* constant diffusivity (CONST_DIFF)                             */
  double c[3];             /* upwind velocity per axis (CELL_ADVDIFF), each >= 0            */
  const double* d_field;   /* kappa / nu at the points of THIS rank's rows (CELL_*), device  */
  const double* d_bands;   /* (2dA+1) x n_loc DIA bands of A (PSP_OP_DIA), device            */
} psp_stencil;

enum { PSP_TOL_REL_B = 0, PSP_TOL_ABS = 1 };       /* eps = tol*||b|| (R1) or eps = tol    */
enum { PSP_MGS_1REDUCE = 0, PSP_MGS_LITERAL = 1 }; /* R11                                   */
/* PSP_METHOD_CG (f4; R27-R31): preconditioned conjugate gradients (Hestenes-Stiefel) for
 * symmetric positive definite A (C1, C2, C4), at most restart * max_cycles iterations; the
 * probes are (p_k, A p_k) / ||p_k|| (plus (x0, A x0)); the preconditioner is the symmetric part
 * N_s = (N + N^T) / 2 of the fitted N, accepted when every row is strictly diagonally dominant
 * with a positive diagonal (so N_s is SPD).  One rank. */
enum { PSP_METHOD_GMRES = 0, PSP_METHOD_CG = 1 };

typedef struct {
  int32_t max_cycles;              /* n_r (R9); default 1000                                */
  int32_t tol_mode;                /* PSP_TOL_*; default PSP_TOL_REL_B                      */
  int32_t m_max;                   /* probe ring capacity (R20); default 64                 */
  int32_t reset_history_per_step;  /* clear the ring at every psp_step; default 0   */
  int32_t ortho;                   /* PSP_MGS_*; default PSP_MGS_1REDUCE                    */
  int32_t gate;                    /* apply the R21 dominance gate; default 1               */
  int32_t timing;                  /* record per-phase CUDA-event times in the report       */
  int32_t fused;                   /* with N = I and ICWY MGS, keep the Krylov basis in the  */
                                   /* probe ring (no probe copies) and run steps              */
                                   /* fused_kmin <= k <= fused_kmax as one fused pass         */
                                   /* (update + matvec + dots, DESIGN.md s.6), the other      */
                                   /* steps as update / matvec / dots passes on the ring;     */
                                   /* 1 (default): fused passes from 2^21 rows on (below,     */
                                   /* their per-plane cost dominates); 2: at any size         */
  int32_t fused_kmin;              /* first step run as a fused pass; default 2               */
  int32_t fused_kmax;              /* last step run as a fused pass; default 16 (wider steps  */
                                   /* hold more basis tiles than shared memory stages well)   */
  int32_t fused_split_cols;        /* steps k > fused_kmax: the newest fused_split_cols       */
                                   /* (1..16) basis columns through the fused pass, the older */
                                   /* k - fused_split_cols through an update pass and a dots  */
                                   /* pass (DESIGN.md s.6); 0 = three separate passes;        */
                                   /* default 16                                              */
  int32_t resident;                /* f2: run the whole solve (every restart cycle, the R(k)  */
                                   /* tests and the restarts) as one persistent device-resident */
                                   /* kernel, no host round trip per step (resident.cu):      */
                                   /* 0 off; 1 (default) for single-rank ICWY solves of up to  */
                                   /* 2^20 rows with n_A <= 64 (a banded N: up to 16384 rows); */
                                   /* 2 whenever supported                                    */
  int32_t method;                  /* PSP_METHOD_*: the Krylov method of psp_solve / psp_step */
                                   /* (f4: "readily applied to all Krylov subspace       */
                                   /* methods"); default PSP_METHOD_GMRES                     */
  int32_t mrep_stream;             /* f3: streaming MREP ("obtained progressively"): each */
                                   /* recorded probe is added to every row's 4d+4 lagged sums */
                                   /* as it is produced, and psp_mrep_fit fits from the sums  */
                                   /* of every probe since the previous fit (the window of    */
                                   /* reset_history_per_step, no m_max cap); one rank; the    */
                                   /* device-resident solve is not used.  Default 0 (the ring) */
} psp_opts;

/* Report of one solve / step.  Arrays are caller-owned host buffers (may be NULL). */
typedef struct {
  int32_t status;                  /* psp_status of the call                                */
  int32_t converged;               /* finish-flag set                                */
  int32_t iterations;              /* inner iterations, all cycles                         */
  int32_t cycles;                  /* restart cycles run                                   */
  int32_t matvecs;                 /* recorded probes                               */
  int32_t precond_applies;         /* banded solves (0 when N = I)                   */
  int32_t precond_identity;        /* the solve ran with N = I                              */
  int32_t resid_cap, resid_len;    /* R(k) history: capacity / entries written              */
  int32_t beta_cap, beta_len;      /* beta per cycle                                 */
  int32_t mrep_ran;                /* the fit ran (m >= 2d+2)                               */
  int32_t mrep_status;
  int32_t mrep_gate_accepted;      /* fitted N installed for the next step (R21)            */
  int64_t mrep_rows_ridge, mrep_rows_fallback, mrep_rows_nondominant;
  double r0;                       /* beta of the first cycle                               */
  double eps;                      /* absolute tolerance used (R1)                          */
  double final_resid_est;          /* last R(k)                                            */
  double final_resid_true;         /* ||b - A x|| recomputed (R13)                          */
  double mrep_max_abs_diag;
  double t_solve_ms, t_mrep_ms, t_factor_ms;   /* CUDA-event times (opts.timing)           */
  double* h_resid_history;         /* resid_cap entries                                    */
  double* h_beta_history;          /* beta_cap entries                                     */
  int32_t resid_verified;          /* final_resid_true <= eps: the explicit check that backs   */
                                   /* `converged` (R13); `converged` itself is the      */
                                   /* paper's finish-flag (R(k) <= eps or breakdown)  */
  int32_t pad_;
} psp_report;

/* MREP row kinds (same meaning as the oracle's, defined independently). */
enum {
  PSP_ROW_INTERIOR = 0, PSP_ROW_INTERIOR_RIDGE = 1, PSP_ROW_BOUNDARY = 2,
  PSP_ROW_FALLBACK_RANK = 3, PSP_ROW_FALLBACK_ZEROVAR = 4, PSP_ROW_FALLBACK_SMALLDIAG = 5
};

/* psp_arnoldi_step flags */
enum { PSP_FLAG_CONVERGED = 1, PSP_FLAG_BREAKDOWN = 2, PSP_FLAG_NONFINITE = 4 };

/* ---------------------------------------------------------------------------------------- */
/* Communicator (one process per GPU, NCCL over NVLink/NVSwitch).                            */
/* ---------------------------------------------------------------------------------------- */
/* nccl_unique_id: the 128-byte ncclUniqueId broadcast by the caller (rank 0 creates it with
 * psp_comm_unique_id).  Collective over nranks processes.  *out is owned by the library.
 * nranks = 1 with an id builds a one-rank NCCL communicator (the NCCL bindings exercised on one
 * GPU: psp_comm_selftest); with a NULL id a one-rank handle without NCCL. */
psp_status psp_comm_unique_id(void* h_id_128);
psp_status psp_comm_init(const void* h_nccl_unique_id, int nranks, int rank, psp_comm** out);
/* Self-test of a communicator (any backend): every collective the hot path uses -- all-reduce
 * sum / max / min, all-gather, the neighbour send/recv of the slab halos -- on small device
 * buffers allocated here, with rank-dependent values, checked on the host against their closed
 * forms.  Collective: every rank calls it (loopback: from its own thread).  stream: a
 * cudaStream_t (NULL = the legacy stream).  PSP_OK, PSP_E_NCCL on a wrong value (the message
 * names the collective) or a failed call, PSP_E_CUDA on an allocation / copy failure. */
psp_status psp_comm_selftest(psp_comm* comm, void* stream);
/* Test backend: nranks communicators of an in-process group (out: nranks handles) whose ranks
 * live on ONE device, each driven by its own host thread; every collective synchronises the
 * caller's stream, meets the other ranks at a host barrier and moves data with cudaMemcpy, so
 * no kernel ever waits on another rank.  Same call sequence and results as NCCL ranks. */
psp_status psp_comm_loopback_create(int nranks, psp_comm** out);
/* Process-level backend: one process per rank, the collectives carried by the caller's own
 * transport (e.g. torch.distributed over gloo) on HOST buffers.  Every callback is collective
 * over the nranks processes and returns 0 on success; the library synchronises the stream and
 * stages device data through pinned host memory around each call (host-mediated: no kernel ever
 * waits on another rank).  allreduce: in place, op 0 sum / 1 max / 2 min, the same result on
 * every rank.  sendrecv: send_lo goes to rank-1, whose send_hi arrives in recv_lo, and
 * symmetrically with rank+1; the pointers of a missing neighbour are NULL with count 0.
 * allgather: recv = the count values of rank 0, then rank 1, ... */
typedef struct {
  void* user;
  int (*allreduce)(void* user, double* h_buf, size_t count, int op);
  int (*sendrecv)(void* user, const double* h_send_lo, double* h_recv_lo, size_t n_lo, const double* h_send_hi,
                  double* h_recv_hi, size_t n_hi);
  int (*allgather)(void* user, const double* h_send, double* h_recv, size_t count);
} psp_host_transport;
psp_status psp_comm_host_create(const psp_host_transport* transport, int nranks, int rank, psp_comm** out);
psp_status psp_comm_destroy(psp_comm* comm);

/* The slab decomposition of a multi-rank context: contiguous blocks of the slowest
 * grid axis (z for 3-D, y for 2-D, the index for 1-D), balanced to within one plane, in global
 * lexicographic order.  Rank `rank` of `nranks` owns rows [row0, row0 + nrows), i.e. planes
 * [slab0, slab0 + slab_len) of that axis.  Pure host function.  PSP_E_DIM if a rank would get
 * no plane. */
psp_status psp_partition(const psp_grid* grid, int nranks, int rank, int64_t* row0, int64_t* nrows,
                         int64_t* slab0, int64_t* slab_len);

/* ---------------------------------------------------------------------------------------- */
/* Context lifecycle.                                                                        */
/* ---------------------------------------------------------------------------------------- */
void psp_default_opts(psp_opts* opts);

/* Bytes of device workspace psp_create needs for this problem on this rank. */
psp_status psp_workspace_bytes(const psp_grid* grid, const psp_stencil* stencil, int d,
                               int restart, const psp_opts* opts, const psp_comm* comm,
                               size_t* bytes);

/* Create a solver for (I - dt L) u^{n+1} = u^n (Eq.4).
 *   grid, stencil: the operator (stencil->d_field / d_bands must outlive the context);
 *   dt: time step; d: MREP half-bandwidth (1..4; P:30 d = 1 tridiagonal); restart: n_A;
 *   tol: see opts->tol_mode; opts: NULL = defaults; d_workspace/ws_bytes: caller-owned device
 *   memory of at least psp_workspace_bytes (256-byte aligned); stream: cudaStream_t;
 *   comm: NULL for one GPU.  N starts as I.
 * Multi-rank (comm with nranks > 1): every rank calls psp_create with the same GLOBAL grid; the
 * context owns the psp_partition slab of its rank, and d_field, every vector argument of the
 * calls below and the workspace are this rank's LOCAL rows.  All calls are then collective
 * (same calls, same order on every rank) and the reports are identical on every rank.  DIA
 * operators and the fused pass are single-rank only.
 * Errors: PSP_E_ARG (bad d, restart, tol, kind), PSP_E_DIM (grid), PSP_E_NOMEM. */
psp_status psp_create(const psp_grid* grid, const psp_stencil* stencil, double dt, int d,
                      int restart, double tol, const psp_opts* opts, void* d_workspace,
                      size_t ws_bytes, void* stream, psp_comm* comm, psp_ctx** out);
psp_status psp_destroy(psp_ctx* ctx);
/* This rank's contiguous row block [row0, row0 + nrows) of the global lexicographic order. */
psp_status psp_local_rows(const psp_ctx* ctx, int64_t* row0, int64_t* nrows);

/* ---------------------------------------------------------------------------------------- */
/* The steps of the hot path.                                                                */
/* ---------------------------------------------------------------------------------------- */
/* y = A x = (I - dt L) x, matrix-free "residual computation" (Eq.4).  x, y: n_loc.
 * record != 0 appends (x, y) to the probe ring as one column pair. */
psp_status psp_matvec(psp_ctx* ctx, const double* d_x, double* d_y, int record);

/* z = N^{-1} v with the current N (identity before the first accepted fit): the
 * preconditioner solve of Alg.1 l.10 and l.42 ("Thomas algorithm").
 * Banded unpivoted LU (R21 makes it breakdown-free), z and v may not alias. */
psp_status psp_precond_apply(psp_ctx* ctx, const double* d_v, double* d_z);

/* Alg.1 l.4-7: record the probe (X0, A X0), R_bar = b - A X0, beta = ||R_bar||,
 * V(:,1) = R_bar / beta, G(1) = beta.  h_beta receives beta (synchronises). */
psp_status psp_cycle_begin(psp_ctx* ctx, const double* d_b, const double* d_x0, double* h_beta);

/* Alg.1 l.9-36 for inner iteration k (1-based, 1 <= k <= restart):
 * Y_k = N^{-1} V(:,k) recorded as P_x(:,i); A Y_k recorded as P_y(:,i); MGS (R11) into
 * H(1..k+1,k); V(:,k+1) (R4 breakdown rule); Givens update; R(k) = |G(k+1)| into
 * *h_resid_k; *h_flags = PSP_FLAG_* (CONVERGED when R(k) <= eps).  Synchronises. */
psp_status psp_arnoldi_step(psp_ctx* ctx, int k, double* h_resid_k, int* h_flags);

/* Alg.1 l.38-43: Q = H^{-1} G on the leading k x k triangle (R6), Z = sum Q_j V_j,
 * x = X0 + N^{-1} Z, and X0 <- x for the next cycle. */
psp_status psp_cycle_end(psp_ctx* ctx, int k, double* d_x);

/* Algorithm 1 in full: x = PSPGMRES(A, b, N, eps, n_A, x0, n_r) with probe
 * recording, then the true residual (R13).  rep may be NULL.  Returns PSP_E_NOCONV when n_r
 * cycles run out (x holds the last iterate). */
psp_status psp_solve(psp_ctx* ctx, const double* d_b, const double* d_x0, double* d_x,
                     psp_report* rep);

/* Algorithm 2 on the probe ring (oldest -> newest, R20), then R18, the R21 gate
 * and the banded LU factorisation of the accepted N (a9).  Rejection or a failed
 * factorisation installs N = I.  PSP_E_SAMPLES if m < 2d+2 (N unchanged).
 * Uses the Krylov basis storage as scratch (4d+4 <= restart+1): call it between solves, as
 * the time-step driver does. */
psp_status psp_mrep_fit(psp_ctx* ctx, psp_report* rep);

/* One implicit-Euler step (Eq.3-4; a10): b = u_n, x0 = u_n (R2),
 * u_np1 = PSPGMRES(...) with the current N, then psp_mrep_fit for the next step.
 * u_n and u_np1 may alias. */
psp_status psp_step(psp_ctx* ctx, const double* d_u_n, double* d_u_np1, psp_report* rep);

/* ---------------------------------------------------------------------------------------- */
/* Stateless kernels (C5 sweep) and test hooks.                                              */
/* ---------------------------------------------------------------------------------------- */
typedef struct {
  int64_t rows_ridge, rows_fallback, rows_nondominant;
  double max_abs_diag;
  int32_t gate_accepted;   /* every row strictly diagonally dominant after R18 (R21)        */
  int32_t status;
} psp_mrep_info;

/* Scratch bytes for psp_mrep_fit_raw / psp_banded_factor_raw / psp_banded_solve_raw
 * (includes (4d+4) x n doubles of lagged-sum rows for the MREP fit). */
psp_status psp_raw_scratch_bytes(int64_t n, int d, size_t* bytes);

/* Alg.2 on caller probe columns: column c (oldest -> newest) of P_x / P_y starts at
 * d_Px + h_order[c]*ld (h_order NULL: c*ld), n rows.  Outputs: d_bands (2d+1) x n,
 * d_intercept n (may be NULL), d_row_kind n (PSP_ROW_*, may be NULL), d_kappa n
 * (Cholesky condition estimate R17, 0 on boundary rows, may be NULL).  Applies R18 and
 * evaluates (does not act on) the R21 gate.  Synchronises (fills *info). */
psp_status psp_mrep_fit_raw(const double* d_Px, const double* d_Py, int64_t n, int m,
                            int64_t ld, const int32_t* h_order, int d, double* d_bands,
                            double* d_intercept, uint8_t* d_row_kind, double* d_kappa,
                            void* d_scratch, size_t scratch_bytes, void* stream,
                            psp_mrep_info* info);

/* Unpivoted banded LU of N (Doolittle; Thomas for d = 1): d_lu (2d+1) x n, o < d ->
 * L(i, i+o-d) (unit diagonal implied), o >= d -> U(i, i+o-d).  PSP_E_SINGULAR on a pivot
 * |U(i,i)| < 1e-300 or growth > 1e100.  Synchronises. */
psp_status psp_banded_factor_raw(const double* d_bands, int64_t n, int d, double* d_lu,
                                 void* d_scratch, size_t scratch_bytes, void* stream);
/* z = N^{-1} v from the factors (forward then backward sweep).  d_x0 != NULL: z = x0 + N^{-1}v. */
psp_status psp_banded_solve_raw(const double* d_lu, int64_t n, int d, const double* d_v,
                                const double* d_x0, double* d_z, void* d_scratch,
                                size_t scratch_bytes, void* stream);

/* Install N (DIA, (2d+1) x n_loc) as the preconditioner for the next solve: applies the R21
 * gate when opts.gate, then factors.  *h_accepted = 1 if installed, 0 if N = I.
 * d_bands == NULL installs N = I. */
psp_status psp_set_bands(psp_ctx* ctx, const double* d_bands, int* h_accepted);
/* Fault injection (SPEC AC10): zero rows h_rows[0..count) (local indices) of the current
 * N's bands and re-install it through the R21 gate and the factorisation (as psp_set_bands):
 * the corrupted N is rejected (gate) or fails the factorisation (zero pivot), N := I and
 * *h_accepted = 0 -- the identity fallback of S:281 / S:345.  Test hook. */
psp_status psp_inject_fault_rows(psp_ctx* ctx, const int64_t* h_rows, int count, int* h_accepted);
/* Copy the current N into d_bands_out ((2d+1) x n_loc); *h_is_identity = 1 when N = I. */
psp_status psp_get_bands(const psp_ctx* ctx, double* d_bands_out, int* h_is_identity);
/* Probe ring view: the c-th oldest recorded probe (c < *h_count) is
 *   P_x(:,c) = h_scale[c] * (*d_px + h_slots[c]*ld)[0..n_loc),  P_y(:,c) likewise with *d_py
 * (the fused path stores probes unnormalised with their Krylov scale).  Host arrays h_slots /
 * h_scale of at least m_max entries; any output may be NULL.  Synchronises for h_scale. */
psp_status psp_ring_view(const psp_ctx* ctx, int* h_count, int32_t* h_slots, double* h_scale,
                         const double** d_px, const double** d_py, int64_t* ld);
psp_status psp_ring_reset(psp_ctx* ctx);
/* Hessenberg state of the current cycle: H ((restart+1) x restart col-major, rotated),
 * Hraw (same, before rotation), G (restart+1), C, S (restart).  Any pointer may be NULL. */
psp_status psp_get_hessenberg(const psp_ctx* ctx, double* h_H, double* h_Hraw, double* h_G,
                              double* h_C, double* h_S);
/* Krylov column V(:,j), 1 <= j <= restart+1, of the current cycle: the columns are stored
 * unnormalised (lagged normalisation), V(:,j) = *h_scale * (*d_vj)[0..n_loc).  h_scale may be
 * NULL.  Synchronises when h_scale is requested. */
psp_status psp_get_basis(const psp_ctx* ctx, int j, const double** d_vj, double* h_scale);
/* Kernel launches issued by this context so far (the bench's gpu_launches). */
psp_status psp_launch_count(const psp_ctx* ctx, int64_t* h_launches);

/* Per-kernel-class CUDA-event timing (opts.timing >= 2 records an event pair on the context's
 * stream around every launch of the hot path).  Classes PSP_KC_*; for each class: summed
 * device milliseconds, summed ALGORITHMIC bytes (the bytes the method
 * must move, not the DRAM traffic) and launch count since the last reset.  Synchronises. */
enum {
  PSP_KC_MATVEC = 0, PSP_KC_PRECOND = 1, PSP_KC_ORTHO_DOTS = 2, PSP_KC_ORTHO_UPDATE = 3,
  PSP_KC_MGS_LITERAL = 4, PSP_KC_NORMALIZE = 5, PSP_KC_COMBINE = 6, PSP_KC_RESIDUAL = 7,
  PSP_KC_MREP = 8, PSP_KC_FACTOR = 9, PSP_KC_OTHER = 10, PSP_KC_FUSED = 11, PSP_KC_RESIDENT = 12,
  PSP_KC_CG = 13, PSP_KC_COUNT = 14
};
psp_status psp_kernel_stats(psp_ctx* ctx, double* h_ms, double* h_bytes, int64_t* h_launches,
                            int reset);
/* Change opts.timing of a live context (0 none, 1 the report's t_solve / t_mrep / t_factor, 2 also
 * the per-kernel-class event pairs above): a measurement can time its headline region without
 * the per-launch events and a second region with them.  PSP_E_ARG for a level outside 0..2;
 * pending per-class records are kept until psp_kernel_stats flushes them.  No GPU work. */
psp_status psp_set_timing(psp_ctx* ctx, int level);
const char* psp_kernel_class_name(int klass);

const char* psp_status_str(psp_status s);
const char* psp_last_error(const psp_ctx* ctx);   /* ctx may be NULL: last global error */
const char* psp_version(void);

#ifdef __cplusplus
}
#endif
#endif
