/*
 * oracle.h -- the CPU oracle of the PSP-GMRES hot path (arXiv 1308.5626).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product (paper_1308_5626_b200/, include/pspgmres.h) never includes,
 * links or calls anything in this directory, and this directory never
 * includes anything from the product.
 *
 * Plain, slow, single-threaded IEEE FP64 C99, built with -O2 -ffp-contract=off
 * (reading R23 of DESIGN.md: every sum is sequential, left to right, in index
 * order; no FMA contraction).  Citations: "P:n" = line n of the paper text
 * (PAPER.md), "S:n" = line n of SPEC.md, "Alg.1 l.N" = Algorithm 1 line N
 * (algorithm2e numbering), "Rnn" = a reading listed in DESIGN.md.
 *
 * Layout: a grid vector is lexicographic, x fastest: g = i + nx*(j + ny*k).
 * Probe and Krylov matrices are column-major (one contiguous column of n per
 * vector).  Banded matrices use DIA storage band[o*n + i] = N(i, i+o-d),
 * o = 0..2d (entries addressing columns outside 0..n-1 are ignored).
 */
#ifndef PSP_ORACLE_H
#define PSP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (same meaning as the product's, defined independently) ---- */
enum {
  ORC_OK = 0, ORC_E_ARG = 1, ORC_E_DIM = 2, ORC_E_SAMPLES = 3, ORC_E_RANK = 4,
  ORC_E_SINGULAR = 5, ORC_E_NONFINITE = 6, ORC_E_NOCONV = 7
};

/* ---- O1: operators A = I - dt*L (Eq.4), applied matrix-free ---- */
enum {
  ORC_OP_CONST_DIFF = 0,   /* L = nu * sum_a d^2/dx_a^2, 2nd-order central (C1, C2)          */
  ORC_OP_CELL_DIFF = 1,    /* L = div(kappa grad), arithmetic-mean faces (C4)                 */
  ORC_OP_CELL_ADVDIFF = 2, /* L = -c.grad + div(nu grad), 1st-order upwind, c_a >= 0 (C3)     */
  ORC_OP_DIA = 3           /* A given explicitly as a banded matrix (DIA), for tests and f1   */
};

typedef struct {
  int32_t ndim;       /* 1, 2 or 3                                                          */
  int32_t kind;       /* ORC_OP_*                                                           */
  int64_t n[3];       /* interior points per axis, n[0] = nx (fastest); unused axes = 1      */
  double dt;          /* time step                                                          */
  double nu;          /* constant diffusivity (CONST_DIFF)                                  */
  double c[3];        /* upwind velocity per axis (CELL_ADVDIFF), each >= 0                 */
  const double* field;/* kappa or nu sampled at the grid points (CELL_*), length N          */
  int32_t dA;         /* half-bandwidth of the DIA operator                                 */
  int32_t pad_;
  const double* bands;/* DIA operator bands, (2dA+1) x N                                    */
} orc_operator;

int64_t orc_op_rows(const orc_operator* A);
/* y = A x.  Returns ORC_OK or ORC_E_ARG. */
int orc_matvec(const orc_operator* A, const double* x, double* y);

/* ---- O2: banded solve ("Thomas algorithm") ---- */
int orc_thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* v, double* z);
/* Doolittle LU without pivoting in DIA storage: lu[o*n+i], o<d -> L(i,i+o-d) (unit
 * diagonal implied), o>=d -> U(i,i+o-d).  ORC_E_SINGULAR if |U(i,i)| < 1e-300 or any
 * |entry| > 1e100. */
int orc_banded_lu(int64_t n, int d, const double* bands, double* lu);
void orc_banded_lu_solve(int64_t n, int d, const double* lu, const double* v, double* z);
void orc_banded_matvec(int64_t n, int d, const double* bands, const double* x, double* y);
/* R21: 1 iff every row is strictly diagonally dominant. */
int orc_gate_dominant(int64_t n, int d, const double* bands);

/* ---- probe history: FIFO ring of (P_x, P_y) columns ---- */
typedef struct {
  int64_t n;      /* rows                                                   */
  int32_t cap;    /* m_max                                                  */
  int32_t count;  /* columns held (m)                                       */
  int32_t head;   /* slot of the oldest column                              */
  int32_t pad_;
  double* px;     /* n x cap, column-major, caller-owned                     */
  double* py;     /* n x cap                                                */
} orc_ring;
void orc_ring_record(orc_ring* ring, const double* x, const double* y);
/* slot of the c-th oldest column, c = 0..count-1 */
int orc_ring_slot(const orc_ring* ring, int c);

/* ---- O3: PSP-GMRES, literal Algorithm 1 ---- */
typedef struct {
  int32_t converged, iterations, cycles, matvecs, precond_applies, status;
  int32_t hist_len, beta_len;
  double r0, final_resid_est, final_resid_true, eps;
} orc_solve_report;

/* optional per-solve trace of the LAST cycle (any pointer may be NULL) */
typedef struct {
  double* V;      /* n x (n_A+1): Krylov basis of the last cycle            */
  double* Hraw;   /* (n_A+1) x n_A column-major: H(:,k) before rotation     */
  double* H;      /* (n_A+1) x n_A: H after rotation (upper triangular)     */
  double* G;      /* n_A+1                                                  */
  double* C;      /* n_A                                                    */
  double* S;      /* n_A                                                    */
  int32_t k_last; /* k of the last cycle                                    */
  int32_t pad_;
} orc_trace;

/* x <- PSPGMRES(A, b, N, eps, n_A, x0, n_r).  lu = banded LU factors of N (NULL: N = I,
 * S:178).  ring (may be NULL) receives every recorded probe.  resid_hist receives R(k)
 * for every inner iteration of every cycle (R12), beta_hist the ||R_bar|| of every cycle. */
int orc_pspgmres(const orc_operator* A, const double* b, const double* x0, double* x,
                 int d, const double* lu, double eps, int n_A, int n_r, orc_ring* ring,
                 orc_solve_report* rep, double* resid_hist, int hist_cap,
                 double* beta_hist, int beta_cap, orc_trace* trace);

/* ---- O4: MREP, literal Algorithm 2 ---- */
enum {
  ORC_ROW_INTERIOR = 0,         /* interior multi-regression, unridged              */
  ORC_ROW_INTERIOR_RIDGE = 1,   /* interior multi-regression after the ridge retry  */
  ORC_ROW_BOUNDARY = 2,         /* first/last d rows, simple linear fit              */
  ORC_ROW_FALLBACK_RANK = 3,    /* ridge retry failed -> identity row  */
  ORC_ROW_FALLBACK_ZEROVAR = 4, /* boundary row with zero regressor variance */
  ORC_ROW_FALLBACK_SMALLDIAG = 5/* |N(i,i)| < 1e-12 max|N(j,j)| -> identity (R18)    */
};
typedef struct {
  int64_t rows_ridge, rows_fallback;
  int32_t status, gate_accepted;
  double max_abs_diag;
} orc_mrep_report;

/* px/py: n x m column matrices with column stride ld; column c (oldest -> newest) lives at
 * slot order[c] (order NULL: slot c).  Outputs: bands (2d+1) x n, intercept n, row_kind n,
 * kappa_est n (condition estimate of the interior Gram, 0 elsewhere); any may be NULL except
 * bands.  Returns ORC_E_SAMPLES if m < 2d+2 (R19), bands untouched. */
int orc_mrep(int64_t n, int m, const double* px, const double* py, int64_t ld, const int* order,
             int d, double* bands, double* intercept, uint8_t* row_kind, double* kappa_est,
             orc_mrep_report* rep);

/* ---- f4: PSP with conjugate gradients (the method "can be readily applied to all
 * Krylov subspace methods"; readings R27-R31 of DESIGN.md) ---- */
/* R29: the symmetric part N_s = (N + N^T) / 2 of a DIA banded N: sym[o*n+i] = (N(i,i+o-d) +
 * N(i+o-d,i)) / 2, the second term read from band 2d-o of row i+o-d. */
void orc_sym_bands(int64_t n, int d, const double* bands, double* sym);
/* R29: 1 iff every row of the (symmetric) bands is strictly diagonally dominant with a
 * positive diagonal -- then N_s is symmetric positive definite (Gershgorin). */
int orc_gate_spd(int64_t n, int d, const double* bands);
/* R27/R28/R30: preconditioned CG (Hestenes-Stiefel) with M = the banded matrix whose LU factors
 * are lu (NULL: M = I):  r = b - A x0 (the probe (x0, A x0) is recorded, as Alg.1 l.4),
 * z = M^-1 r, p = z, rho = r'z; for k = 1..max_iters: q = A p (the probe (p, q)/||p|| is
 * recorded: unit-norm like Alg.1's Krylov probes, so Alg.2's intercept row is commensurate),
 * pq = p'q (pq <= 0 or non-finite: A or M not SPD -> ORC_E_SINGULAR), alpha = rho / pq,
 * x += alpha p, r -= alpha q, R(k) = ||r|| (history; R(k) <= eps stops), z = M^-1 r,
 * rho' = r'z, p = z + (rho'/rho) p.  Then the true residual ||b - A x|| (R13).  cycles = 1;
 * ORC_E_NOCONV after max_iters. */
int orc_pcg(const orc_operator* A, const double* b, const double* x0, double* x, int d, const double* lu,
            double eps, int max_iters, orc_ring* ring, orc_solve_report* rep, double* resid_hist,
            int hist_cap);

/* ---- O5: time-step driver (Eq.3-4; "next time step") ---- */
enum { ORC_METHOD_GMRES = 0, ORC_METHOD_CG = 1 };
typedef struct {
  int32_t restart;          /* n_A                                                  */
  int32_t max_cycles;       /* n_r (CG: at most n_A * n_r iterations, R31)          */
  double tol;               /* eps = tol * ||b||_2 (R1)                             */
  int32_t d;                /* MREP half-bandwidth                                  */
  int32_t m_max;            /* ring capacity                                        */
  int32_t reset_history;    /* clear the ring at the start of every step     */
  int32_t gate;             /* apply R21 (1) or accept any factorable N (0)          */
  int32_t method;           /* ORC_METHOD_*: the Krylov method of the step (f4)      */
  int32_t pad_;
} orc_step_opts;

typedef struct {
  orc_solve_report solve;
  orc_mrep_report mrep;
  int32_t precond_was_identity;  /* N used in this step's solve was I              */
  int32_t mrep_ran;              /* the fit ran after this step (m >= 2d+2)         */
} orc_step_report;

/* Advance u through `steps` implicit-Euler steps.  u (n) is updated in place.  ring is
 * caller-owned (cap = m_max).  bands_N / lu_N (each (2d+1) x n) hold the current N and its
 * factors; *n_is_identity says whether N = I (N_0 = I).  reports: steps entries. */
int orc_time_steps(const orc_operator* A, double* u, int steps, const orc_step_opts* opt,
                   orc_ring* ring, double* bands_N, double* lu_N, int* n_is_identity,
                   orc_step_report* reports, double* resid_hist, int hist_cap);

#ifdef __cplusplus
}
#endif
#endif
