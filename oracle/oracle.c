/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle of the PSP-GMRES hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the CUDA product.
 *
 * Everything here follows the paper (arXiv 1308.5626, PAPER.md) step by step, in its
 * order and notation, with the readings R1..R26 of DESIGN.md where it is silent.
 * Single-threaded IEEE FP64, compiled with -O2 -ffp-contract=off; every reduction is a
 * sequential left-to-right loop in index order (R23).
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   orc_matvec          closed-form sine-mode eigenvalues, dense assembly, symmetry (PN1)
 *   orc_banded_lu*      dense LU via numpy, tridiag(-1,2,-1) worked example, LU(d=1)=Thomas (PN2)
 *   orc_pspgmres        dense solve, brute-force Krylov least squares, dense-QR residual,
 *                       Arnoldi relation, orthogonality, minimal polynomial (PN3)
 *   orc_mrep            exact recovery of banded A, KKT optimality, linear-fit examples (PN4)
 *   orc_time_steps      closed-form implicit-Euler decay of a sine mode; rank bound (PN5)
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* small vector helpers (sequential sums, R23)                                           */
/* ------------------------------------------------------------------------------------ */
static double dot(int64_t n, const double* x, const double* y) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
static double norm2(int64_t n, const double* x) { return sqrt(dot(n, x, x)); }
static void copy(int64_t n, const double* x, double* y) { memcpy(y, x, (size_t)n * sizeof(double)); }

/* ------------------------------------------------------------------------------------ */
/* O1. Operators: y = A x = (I - dt L) x   (Eq.4), matrix-free.            */
/* Grid: interior points x_i = i*h, h = 1/(n+1) per axis, u = 0 outside (R24).          */
/* ------------------------------------------------------------------------------------ */
int64_t orc_op_rows(const orc_operator* A) {
  int64_t n = 1;
  for (int a = 0; a < A->ndim; ++a) n *= A->n[a];
  return n;
}

/* value of x at the neighbour of point g along axis a in direction dir (+1/-1); 0 outside */
static int nb_index(const orc_operator* A, const int64_t idx[3], int a, int dir, int64_t* g_out) {
  int64_t j = idx[a] + dir;
  if (j < 0 || j >= A->n[a]) return 0;
  int64_t q[3] = {idx[0], idx[1], idx[2]};
  q[a] = j;
  *g_out = q[0] + A->n[0] * (q[1] + A->n[1] * q[2]);
  return 1;
}

int orc_matvec(const orc_operator* A, const double* x, double* y) {
  const int64_t N = orc_op_rows(A);
  if (A->kind == ORC_OP_DIA) {
    orc_banded_matvec(N, A->dA, A->bands, x, y);
    return ORC_OK;
  }
  if (A->ndim < 1 || A->ndim > 3) return ORC_E_ARG;
  double inv_h[3], inv_h2[3];
  for (int a = 0; a < 3; ++a) {
    double h = 1.0 / (double)(A->n[a] + 1);
    inv_h[a] = 1.0 / h;
    inv_h2[a] = 1.0 / (h * h);
  }
  for (int64_t g = 0; g < N; ++g) {
    int64_t idx[3];
    idx[0] = g % A->n[0];
    idx[1] = (g / A->n[0]) % A->n[1];
    idx[2] = g / (A->n[0] * A->n[1]);
    double Lx = 0.0; /* (L x)_g */
    for (int a = 0; a < A->ndim; ++a) {
      for (int dir = -1; dir <= 1; dir += 2) {
        int64_t gn;
        int inside = nb_index(A, idx, a, dir, &gn);
        double xn = inside ? x[gn] : 0.0; /* Dirichlet 0 outside */
        if (A->kind == ORC_OP_CONST_DIFF) {
          /* central second difference nu (x_{g-e} - 2 x_g + x_{g+e}) / h^2, split per face */
          Lx += A->nu * (xn - x[g]) * inv_h2[a];
        } else {
          /* face coefficient: arithmetic mean inside, the cell value on the boundary face */
          double kf = inside ? 0.5 * (A->field[g] + A->field[gn]) : A->field[g];
          Lx += kf * (xn - x[g]) * inv_h2[a];
        }
      }
      if (A->kind == ORC_OP_CELL_ADVDIFF) {
        /* first-order upwind for c_a >= 0: -c_a (x_g - x_{g-e_a}) / h */
        int64_t gw;
        double xw = nb_index(A, idx, a, -1, &gw) ? x[gw] : 0.0;
        Lx += -A->c[a] * (x[g] - xw) * inv_h[a];
      }
    }
    y[g] = x[g] - A->dt * Lx;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------ */
/* O2. Banded solve ("solved efficiently in O(n) FLOPs using Thomas algorithm";   */
/* P:161 for d > 1).  Unpivoted.                                   */
/* ------------------------------------------------------------------------------------ */
int orc_thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* v, double* z) {
  /* w_1 = b_1; l_i = a_i / w_{i-1}; w_i = b_i - l_i c_{i-1}; y_i = v_i - l_i y_{i-1};
   * z_n = y_n / w_n; z_i = (y_i - c_i z_{i+1}) / w_i */
  double* w = (double*)malloc((size_t)n * sizeof(double));
  double* y = (double*)malloc((size_t)n * sizeof(double));
  int st = ORC_OK;
  w[0] = diag[0];
  y[0] = v[0];
  if (fabs(w[0]) < 1e-300) st = ORC_E_SINGULAR;
  for (int64_t i = 1; i < n && st == ORC_OK; ++i) {
    double l = sub[i] / w[i - 1];
    w[i] = diag[i] - l * sup[i - 1];
    y[i] = v[i] - l * y[i - 1];
    if (fabs(w[i]) < 1e-300) st = ORC_E_SINGULAR;
  }
  if (st == ORC_OK) {
    z[n - 1] = y[n - 1] / w[n - 1];
    for (int64_t i = n - 2; i >= 0; --i) z[i] = (y[i] - sup[i] * z[i + 1]) / w[i];
  }
  free(w);
  free(y);
  return st;
}

#define BAND(b, n, o, i) ((b)[(int64_t)(o) * (n) + (i)])

void orc_banded_matvec(int64_t n, int d, const double* bands, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int o = 0; o <= 2 * d; ++o) {
      int64_t j = i + o - d;
      if (j < 0 || j >= n) continue;
      s += BAND(bands, n, o, i) * x[j];
    }
    y[i] = s;
  }
}

int orc_banded_lu(int64_t n, int d, const double* bands, double* lu) {
  /* Doolittle, row by row: L(i,j) for j < i, then U(i,j) for j >= i, all within the band.
   * L(i,j) = (N(i,j) - sum_{k<j} L(i,k) U(k,j)) / U(j,j);  U(i,j) = N(i,j) - sum_{k<i} L(i,k) U(k,j)
   * with k restricted to the band (k >= i-d and k >= j-d). */
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = (i - d > 0 ? i - d : 0); j < i; ++j) {
      double s = BAND(bands, n, j - i + d, i);
      int64_t k0 = (j - d > i - d ? j - d : i - d);
      if (k0 < 0) k0 = 0;
      for (int64_t k = k0; k < j; ++k) s -= BAND(lu, n, k - i + d, i) * BAND(lu, n, j - k + d, k);
      BAND(lu, n, j - i + d, i) = s / BAND(lu, n, d, j);
    }
    for (int64_t j = i; j <= i + d && j < n; ++j) {
      double s = BAND(bands, n, j - i + d, i);
      int64_t k0 = (j - d > i - d ? j - d : i - d);
      if (k0 < 0) k0 = 0;
      for (int64_t k = k0; k < i; ++k) s -= BAND(lu, n, k - i + d, i) * BAND(lu, n, j - k + d, k);
      BAND(lu, n, j - i + d, i) = s;
    }
    if (fabs(BAND(lu, n, d, i)) < 1e-300) return ORC_E_SINGULAR;
    for (int o = 0; o <= 2 * d; ++o) {
      int64_t j = i + o - d;
      if (j < 0 || j >= n) { BAND(lu, n, o, i) = 0.0; continue; }
      double e = BAND(lu, n, o, i);
      if (!(fabs(e) <= 1e100)) return ORC_E_SINGULAR; /* growth / non-finite */
    }
  }
  return ORC_OK;
}

void orc_banded_lu_solve(int64_t n, int d, const double* lu, const double* v, double* z) {
  /* forward: y_i = v_i - sum_{j=i-d}^{i-1} L(i,j) y_j ; backward: z_i = (y_i - sum U(i,j) z_j)/U(i,i) */
  double* y = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    double s = v[i];
    for (int64_t j = (i - d > 0 ? i - d : 0); j < i; ++j) s -= BAND(lu, n, j - i + d, i) * y[j];
    y[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t j = i + 1; j <= i + d && j < n; ++j) s -= BAND(lu, n, j - i + d, i) * z[j];
    z[i] = s / BAND(lu, n, d, i);
  }
  free(y);
}

int orc_gate_dominant(int64_t n, int d, const double* bands) {
  /* R21: every row strictly diagonally dominant: |n_ii| > sum_{j != i} |n_ij| */
  for (int64_t i = 0; i < n; ++i) {
    double off = 0.0;
    for (int o = 0; o <= 2 * d; ++o) {
      int64_t j = i + o - d;
      if (o == d || j < 0 || j >= n) continue;
      off += fabs(BAND(bands, n, o, i));
    }
    if (!(fabs(BAND(bands, n, d, i)) > off)) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------------------ */
/* Probe history ("the result is stored in the i-th column of matrix P_y"),        */
/* FIFO ring of capacity m_max across solves (R20).                          */
/* ------------------------------------------------------------------------------------ */
void orc_ring_record(orc_ring* r, const double* x, const double* y) {
  int slot;
  if (r->count < r->cap) {
    slot = (r->head + r->count) % r->cap;
    r->count += 1;
  } else {
    slot = r->head; /* evict the oldest */
    r->head = (r->head + 1) % r->cap;
  }
  copy(r->n, x, r->px + (int64_t)slot * r->n);
  copy(r->n, y, r->py + (int64_t)slot * r->n);
}
int orc_ring_slot(const orc_ring* r, int c) { return (r->head + c) % r->cap; }

/* ------------------------------------------------------------------------------------ */
/* O3. PSP-GMRES: Algorithm 1, line by line.                                  */
/* ------------------------------------------------------------------------------------ */
static void precond_solve(int64_t n, int d, const double* lu, const double* v, double* z) {
  if (lu == NULL) copy(n, v, z); /* N = I: the identity path skips the solve */
  else orc_banded_lu_solve(n, d, lu, v, z);
}

#define HM(H, ld, r, c) ((H)[(int64_t)(c) * (ld) + (r)]) /* column-major (n_A+1) x n_A */

int orc_pspgmres(const orc_operator* A, const double* b, const double* x0_in, double* x,
                 int d, const double* lu, double eps, int n_A, int n_r, orc_ring* ring,
                 orc_solve_report* rep, double* resid_hist, int hist_cap,
                 double* beta_hist, int beta_cap, orc_trace* trace) {
  const int64_t n = orc_op_rows(A);
  const int ldh = n_A + 1;
  memset(rep, 0, sizeof(*rep));
  rep->eps = eps;
  if (n_A < 1 || n_r < 1 || !(eps >= 0.0)) { rep->status = ORC_E_ARG; return ORC_E_ARG; }

  double* X0 = (double*)malloc((size_t)n * sizeof(double));
  double* V = (double*)calloc((size_t)n * (size_t)(n_A + 1), sizeof(double));
  double* H = (double*)calloc((size_t)ldh * (size_t)n_A, sizeof(double));
  double* G = (double*)calloc((size_t)n_A + 1, sizeof(double));
  double* C = (double*)calloc((size_t)n_A, sizeof(double));
  double* S = (double*)calloc((size_t)n_A, sizeof(double));
  double* Q = (double*)calloc((size_t)n_A, sizeof(double));
  double* U = (double*)malloc((size_t)n * sizeof(double));
  double* Y = (double*)malloc((size_t)n * sizeof(double));
  double* W = (double*)malloc((size_t)n * sizeof(double));
  double* Z = (double*)malloc((size_t)n * sizeof(double));
  double* Rb = (double*)malloc((size_t)n * sizeof(double));
  int status = ORC_OK;
  int finish = 0;

  copy(n, x0_in, X0);
  for (int l = 1; l <= n_r; ++l) {                          /* l.3 */
    /* l.4: P_x(:,i) <- X0, P_y(:,i) <- A X0 */
    orc_matvec(A, X0, W);
    if (ring) orc_ring_record(ring, X0, W);
    rep->matvecs += 1;
    /* l.5: R_bar <- B - P_y(:,i) */
    for (int64_t t = 0; t < n; ++t) Rb[t] = b[t] - W[t];
    /* l.6-7: V(:,1) <- R_bar/||R_bar||, G(1) <- ||R_bar|| */
    double beta = norm2(n, Rb);
    if (rep->beta_len < beta_cap && beta_hist) beta_hist[rep->beta_len] = beta;
    rep->beta_len += 1;
    if (l == 1) rep->r0 = beta;
    rep->cycles += 1;
    if (!isfinite(beta)) { status = ORC_E_NONFINITE; break; }
    if (beta <= eps) { /* R3: already converged, return X0 after 0 iterations */
      finish = 1;
      rep->final_resid_est = beta;
      if (trace) trace->k_last = 0;
      break;
    }
    memset(V, 0, sizeof(double) * (size_t)n * (size_t)(n_A + 1));
    memset(H, 0, sizeof(double) * (size_t)ldh * (size_t)n_A);
    memset(G, 0, sizeof(double) * (size_t)(n_A + 1));
    for (int64_t t = 0; t < n; ++t) V[t] = Rb[t] / beta;
    G[0] = beta;

    int k;       /* current inner iteration, 1-based as in the paper */
    int kdone = 0;
    for (k = 1; k <= n_A; ++k) {                            /* l.8 */
      double* Vk = V + (int64_t)(k - 1) * n;
      G[k] = 0.0;                                           /* l.9: G(k+1) <- 0 */
      precond_solve(n, d, lu, Vk, Y);                       /* l.10: Y_k <- N^-1 V(:,k) */
      if (lu) rep->precond_applies += 1;
      orc_matvec(A, Y, W);                                  /* l.11: P_y(:,i) <- A Y_k */
      if (ring) orc_ring_record(ring, Y, W);                /*              P_x(:,i) <- Y_k   */
      rep->matvecs += 1;
      copy(n, W, U);                                        /* l.12: U_k <- P_y(:,i) */
      for (int j = 1; j <= k; ++j) {                        /* l.13-16: MGS */
        const double* Vj = V + (int64_t)(j - 1) * n;
        double h = dot(n, Vj, U);
        HM(H, ldh, j - 1, k - 1) = h;
        for (int64_t t = 0; t < n; ++t) U[t] = U[t] - h * Vj[t];
      }
      double hk1 = norm2(n, U);                             /* l.17: H(k+1,k) <- ||U_k|| */
      HM(H, ldh, k, k - 1) = hk1;
      if (!isfinite(hk1)) { status = ORC_E_NONFINITE; break; }
      /* R4: breakdown if H(k+1,k) <= 1e-14 ||H(1:k+1,k)|| (before rotation) */
      double colnorm = 0.0;
      for (int j = 0; j <= k; ++j) colnorm += HM(H, ldh, j, k - 1) * HM(H, ldh, j, k - 1);
      colnorm = sqrt(colnorm);
      int breakdown = !(hk1 > 1e-14 * colnorm);
      double* Vk1 = V + (int64_t)k * n;
      if (!breakdown)                                       /* l.18: V(:,k+1) <- U_k/H(k+1,k) */
        for (int64_t t = 0; t < n; ++t) Vk1[t] = U[t] / hk1;
      /* (breakdown: V(:,k+1) stays 0) */
      if (trace && trace->Hraw)
        for (int j = 0; j <= k; ++j) trace->Hraw[(int64_t)(k - 1) * ldh + j] = HM(H, ldh, j, k - 1);
      for (int j = 1; j <= k - 1; ++j) {                    /* l.19-23: old rotations */
        double delta = HM(H, ldh, j - 1, k - 1);
        HM(H, ldh, j - 1, k - 1) = delta * C[j - 1] + S[j - 1] * HM(H, ldh, j, k - 1);
        HM(H, ldh, j, k - 1) = -delta * S[j - 1] + C[j - 1] * HM(H, ldh, j, k - 1);
      }
      {                                                     /* l.24-28: new rotation, R10 */
        double a = HM(H, ldh, k - 1, k - 1), bb = HM(H, ldh, k, k - 1);
        double gamma = sqrt(a * a + bb * bb);
        if (gamma == 0.0) { C[k - 1] = 1.0; S[k - 1] = 0.0; breakdown = 1; }
        else { C[k - 1] = a / gamma; S[k - 1] = bb / gamma; }
        HM(H, ldh, k - 1, k - 1) = gamma;
        HM(H, ldh, k, k - 1) = 0.0;
      }
      {                                                     /* l.29-31 */
        double delta = G[k - 1];
        G[k - 1] = C[k - 1] * delta + S[k - 1] * G[k];
        G[k] = -S[k - 1] * delta + C[k - 1] * G[k];
      }
      double Rk = fabs(G[k]);                               /* l.32: R(k) <- |G(k+1)| */
      if (resid_hist && rep->hist_len < hist_cap) resid_hist[rep->hist_len] = Rk;
      rep->hist_len += 1;
      rep->iterations += 1;
      rep->final_resid_est = Rk;
      kdone = k;
      if (Rk <= eps || breakdown) {                         /* l.33-36, R4, R5 */
        finish = 1;
        break;
      }
    }
    if (status != ORC_OK) break;
    k = kdone;                                              /* R8: k = n_A without a break */
    /* l.38: Q <- H^-1 G on the leading k x k upper triangle (R6) */
    for (int j = k; j >= 1; --j) {
      double s = G[j - 1];
      for (int t = j + 1; t <= k; ++t) s -= HM(H, ldh, j - 1, t - 1) * Q[t - 1];
      double piv = HM(H, ldh, j - 1, j - 1);
      if (piv == 0.0) { status = ORC_E_SINGULAR; break; }
      Q[j - 1] = s / piv;
    }
    if (status != ORC_OK) break;
    /* l.39-41: Z_k <- Z_k + Q(j) V(:,j), Z_k = 0 at cycle start (R7) */
    for (int64_t t = 0; t < n; ++t) Z[t] = 0.0;
    for (int j = 1; j <= k; ++j) {
      const double* Vj = V + (int64_t)(j - 1) * n;
      for (int64_t t = 0; t < n; ++t) Z[t] = Z[t] + Q[j - 1] * Vj[t];
    }
    /* l.42: X <- X0 + N^-1 Z_k */
    precond_solve(n, d, lu, Z, Y);
    if (lu) rep->precond_applies += 1;
    for (int64_t t = 0; t < n; ++t) x[t] = X0[t] + Y[t];
    copy(n, x, X0);                                         /* l.43: X0 <- X */
    if (trace) {                                            /* (trace of the last cycle) */
      trace->k_last = k;
      if (trace->V) copy(n * (int64_t)(n_A + 1), V, trace->V);
      if (trace->H) copy((int64_t)ldh * n_A, H, trace->H);
      if (trace->G) copy(n_A + 1, G, trace->G);
      if (trace->C) copy(n_A, C, trace->C);
      if (trace->S) copy(n_A, S, trace->S);
    }
    /* l.44: clean G, V, H, C, S  (done at the top of the next cycle) */
    if (finish) break;                                      /* l.45-48 */
  }
  if (status == ORC_OK || status == ORC_E_NOCONV) {
    copy(n, X0, x); /* X holds the last X0 (also covers the R3 early exit) */
    /* R13: explicit true residual ||b - A x|| with one unrecorded matvec */
    orc_matvec(A, x, W);
    for (int64_t t = 0; t < n; ++t) Rb[t] = b[t] - W[t];
    rep->final_resid_true = norm2(n, Rb);
    rep->converged = finish;
    if (!finish) status = ORC_E_NOCONV;
  }
  rep->status = status;
  free(X0); free(V); free(H); free(G); free(C); free(S); free(Q);
  free(U); free(Y); free(W); free(Z); free(Rb);
  return status;
}

/* ------------------------------------------------------------------------------------ */
/* O4. MREP: Algorithm 2, literal per-row normal equations.           */
/* ------------------------------------------------------------------------------------ */

/* Cholesky of the p x p SPD matrix G (row-major), no pivoting (R17).  Returns 0 on
 * failure (a pivot^2 <= 0 or non-finite), else 1 and the factor in L (row-major). */
static int cholesky(int p, const double* G, double* L) {
  memset(L, 0, sizeof(double) * (size_t)p * (size_t)p);
  for (int j = 0; j < p; ++j) {
    double s = G[j * p + j];
    for (int k = 0; k < j; ++k) s -= L[j * p + k] * L[j * p + k];
    if (!(s > 0.0) || !isfinite(s)) return 0;
    L[j * p + j] = sqrt(s);
    for (int i = j + 1; i < p; ++i) {
      double t = G[i * p + j];
      for (int k = 0; k < j; ++k) t -= L[i * p + k] * L[j * p + k];
      L[i * p + j] = t / L[j * p + j];
    }
  }
  return 1;
}
static void cholesky_solve(int p, const double* L, const double* r, double* beta) {
  double z[16];
  for (int i = 0; i < p; ++i) {
    double s = r[i];
    for (int k = 0; k < i; ++k) s -= L[i * p + k] * z[k];
    z[i] = s / L[i * p + i];
  }
  for (int i = p - 1; i >= 0; --i) {
    double s = z[i];
    for (int k = i + 1; k < p; ++k) s -= L[k * p + i] * beta[k];
    beta[i] = s / L[i * p + i];
  }
}

static void set_identity_row(int64_t n, int d, double* bands, int64_t i) {
  for (int o = 0; o <= 2 * d; ++o) BAND(bands, n, o, i) = (o == d) ? 1.0 : 0.0;
}

int orc_mrep(int64_t n, int m, const double* px, const double* py, int64_t ld, const int* order,
             int d, double* bands, double* intercept, uint8_t* row_kind, double* kappa_est,
             orc_mrep_report* rep) {
  orc_mrep_report dummy;
  if (!rep) rep = &dummy;
  memset(rep, 0, sizeof(*rep));
  if (d < 1 || d > 7 || n < 2 * d + 1) { rep->status = ORC_E_DIM; return ORC_E_DIM; }
  if (m < 2 * d + 2) { rep->status = ORC_E_SAMPLES; return ORC_E_SAMPLES; }          /* R19 */
  const int p = 2 * d + 2;
  const double** xcol = (const double**)malloc(sizeof(double*) * (size_t)m);
  const double** ycol = (const double**)malloc(sizeof(double*) * (size_t)m);
  for (int c = 0; c < m; ++c) {
    int s = order ? order[c] : c;
    xcol[c] = px + (int64_t)s * ld;
    ycol[c] = py + (int64_t)s * ld;
  }
  double G[256], L[256], r[16], beta[16], xs[16];

  for (int64_t i = 0; i < n; ++i) {
    for (int o = 0; o <= 2 * d; ++o) BAND(bands, n, o, i) = 0.0;
    if (kappa_est) kappa_est[i] = 0.0;
    if (i < d || i >= n - d) {
      /* (beta0, beta1) <- linear fit(P_x(i,:), P_y(i,:)); N(i,i) <- beta1.
       * R16: two-pass centred OLS. */
      double mx = 0.0, my = 0.0;
      for (int c = 0; c < m; ++c) { mx += xcol[c][i]; my += ycol[c][i]; }
      mx /= (double)m;
      my /= (double)m;
      double sxx = 0.0, sxy = 0.0;
      for (int c = 0; c < m; ++c) {
        double dx = xcol[c][i] - mx, dy = ycol[c][i] - my;
        sxx += dx * dx;
        sxy += dx * dy;
      }
      if (sxx < 1e-300) { /* zero variance -> N(i,i) := 1, flagged */
        set_identity_row(n, d, bands, i);
        if (intercept) intercept[i] = 0.0;
        if (row_kind) row_kind[i] = ORC_ROW_FALLBACK_ZEROVAR;
        rep->rows_fallback += 1;
      } else {
        double b1 = sxy / sxx;
        BAND(bands, n, d, i) = b1;
        if (intercept) intercept[i] = my - b1 * mx;
        if (row_kind) row_kind[i] = ORC_ROW_BOUNDARY;
      }
      continue;
    }
    /* P_x* = [1 ... 1; P_x(i-d,:); ...; P_x(i+d,:)], P_y* = P_y(i,:)
     * P:122:     N* = (P_x* P_x*')^-1 P_x* P_y*'   (normal equations, columns oldest -> newest) */
    memset(G, 0, sizeof(G));
    memset(r, 0, sizeof(r));
    for (int c = 0; c < m; ++c) {
      xs[0] = 1.0;
      for (int a = 0; a <= 2 * d; ++a) xs[1 + a] = xcol[c][i - d + a];
      double yc = ycol[c][i];
      for (int a = 0; a < p; ++a) {
        for (int bq = 0; bq < p; ++bq) G[a * p + bq] += xs[a] * xs[bq];
        r[a] += xs[a] * yc;
      }
    }
    /* R17: Cholesky; condition estimate (max L_jj / min L_jj)^2; one ridge retry */
    int ok = cholesky(p, G, L);
    double kap = 0.0;
    if (ok) {
      double lmax = L[0], lmin = L[0];
      for (int j = 1; j < p; ++j) {
        double v = L[j * p + j];
        if (v > lmax) lmax = v;
        if (v < lmin) lmin = v;
      }
      kap = (lmax / lmin) * (lmax / lmin);
    }
    if (kappa_est) kappa_est[i] = ok ? kap : INFINITY;
    int kind = ORC_ROW_INTERIOR;
    if (!ok || kap > 1e12) {
      double tr = 0.0;
      for (int j = 0; j < p; ++j) tr += G[j * p + j];
      double lambda = 1e-10 * tr / (double)p;
      for (int j = 0; j < p; ++j) G[j * p + j] += lambda;
      ok = cholesky(p, G, L);
      kind = ORC_ROW_INTERIOR_RIDGE;
      rep->rows_ridge += 1;
    }
    if (!ok) { /* rank-deficient even with the ridge -> identity row */
      set_identity_row(n, d, bands, i);
      if (intercept) intercept[i] = 0.0;
      if (row_kind) row_kind[i] = ORC_ROW_FALLBACK_RANK;
      rep->rows_fallback += 1;
      continue;
    }
    cholesky_solve(p, L, r, beta);
    /* P:124-127 with R14: N(i, i+j-d-2) <- N*(j), j = 2..2d+2 (1-based), i.e. band o = j-2 */
    for (int o = 0; o <= 2 * d; ++o) BAND(bands, n, o, i) = beta[1 + o];
    if (intercept) intercept[i] = beta[0]; /* R15: reported, never installed */
    if (row_kind) row_kind[i] = (uint8_t)kind;
  }
  /* R18: rows whose |N(i,i)| < 1e-12 max_j |N(j,j)| become identity rows */
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double v = fabs(BAND(bands, n, d, i));
    if (v > mx) mx = v;
  }
  rep->max_abs_diag = mx;
  for (int64_t i = 0; i < n; ++i) {
    if (fabs(BAND(bands, n, d, i)) < 1e-12 * mx) {
      set_identity_row(n, d, bands, i);
      if (row_kind) row_kind[i] = ORC_ROW_FALLBACK_SMALLDIAG;
      rep->rows_fallback += 1;
    }
  }
  rep->gate_accepted = orc_gate_dominant(n, d, bands);
  free(xcol);
  free(ycol);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------ */
/* f4. PSP with conjugate gradients ("the methodology can be readily applied to all   */
/* Krylov subspace methods"); readings R27-R31.                                           */
/* ------------------------------------------------------------------------------------ */
void orc_sym_bands(int64_t n, int d, const double* bands, double* sym) {
  /* R29: N_s(i, j) = (N(i, j) + N(j, i)) / 2, j = i + o - d; N(j, i) = band 2d - o of row j */
  for (int o = 0; o <= 2 * d; ++o) {
    for (int64_t i = 0; i < n; ++i) {
      int64_t j = i + o - d;
      if (j < 0 || j >= n) { BAND(sym, n, o, i) = 0.0; continue; }
      BAND(sym, n, o, i) = 0.5 * (BAND(bands, n, o, i) + BAND(bands, n, 2 * d - o, j));
    }
  }
}

int orc_gate_spd(int64_t n, int d, const double* bands) {
  /* R29: positive diagonal and strict diagonal dominance => symmetric positive definite */
  for (int64_t i = 0; i < n; ++i) {
    if (!(BAND(bands, n, d, i) > 0.0)) return 0;
  }
  return orc_gate_dominant(n, d, bands);
}

int orc_pcg(const orc_operator* A, const double* b, const double* x0, double* x, int d, const double* lu,
            double eps, int max_iters, orc_ring* ring, orc_solve_report* rep, double* resid_hist,
            int hist_cap) {
  const int64_t n = orc_op_rows(A);
  memset(rep, 0, sizeof(*rep));
  rep->eps = eps;
  double* r = (double*)malloc((size_t)n * sizeof(double));
  double* z = (double*)malloc((size_t)n * sizeof(double));
  double* p = (double*)malloc((size_t)n * sizeof(double));
  double* q = (double*)malloc((size_t)n * sizeof(double));
  double* w = (double*)malloc((size_t)n * sizeof(double));
  int status = ORC_OK, finish = 0;
  copy(n, x0, x);
  orc_matvec(A, x, q);                                  /* the probe (x0, A x0), as Alg.1 l.4 */
  if (ring) orc_ring_record(ring, x, q);
  rep->matvecs = 1;
  rep->cycles = 1;
  for (int64_t t = 0; t < n; ++t) r[t] = b[t] - q[t];   /* r = b - A x0 */
  double rn = norm2(n, r);
  rep->r0 = rn;
  rep->final_resid_est = rn;
  if (!isfinite(rn)) status = ORC_E_NONFINITE;
  else if (rn <= eps) finish = 1;                       /* R3 */
  double rho = 0.0;
  if (status == ORC_OK && !finish) {
    precond_solve(n, d, lu, r, z);                      /* z = M^-1 r */
    if (lu) rep->precond_applies += 1;
    copy(n, z, p);                                      /* p = z */
    rho = dot(n, r, z);
  }
  for (int k = 1; status == ORC_OK && !finish && k <= max_iters; ++k) {
    orc_matvec(A, p, q);                                /* q = A p */
    rep->matvecs += 1;
    if (ring) {                                         /* R28: the probe (p, A p) / ||p||     */
      double pn = norm2(n, p);
      for (int64_t t = 0; t < n; ++t) { z[t] = p[t] / pn; w[t] = q[t] / pn; }
      orc_ring_record(ring, z, w);
    }
    double pq = dot(n, p, q);
    if (!isfinite(pq)) { status = ORC_E_NONFINITE; break; }
    if (!(pq > 0.0)) { status = ORC_E_SINGULAR; break; } /* R30: A (or M) not SPD */
    double alpha = rho / pq;
    for (int64_t t = 0; t < n; ++t) x[t] = x[t] + alpha * p[t];
    for (int64_t t = 0; t < n; ++t) r[t] = r[t] - alpha * q[t];
    double Rk = norm2(n, r);                            /* R(k): the recursive residual */
    if (resid_hist && rep->hist_len < hist_cap) resid_hist[rep->hist_len] = Rk;
    rep->hist_len += 1;
    rep->iterations += 1;
    rep->final_resid_est = Rk;
    if (!isfinite(Rk)) { status = ORC_E_NONFINITE; break; }
    if (Rk <= eps) { finish = 1; break; }
    precond_solve(n, d, lu, r, z);                      /* z = M^-1 r */
    if (lu) rep->precond_applies += 1;
    double rho1 = dot(n, r, z);
    double beta = rho1 / rho;
    rho = rho1;
    for (int64_t t = 0; t < n; ++t) p[t] = z[t] + beta * p[t];
  }
  if (status == ORC_OK) {
    orc_matvec(A, x, q);                                /* R13: true residual, not recorded */
    for (int64_t t = 0; t < n; ++t) r[t] = b[t] - q[t];
    rep->final_resid_true = norm2(n, r);
    rep->converged = finish;
    if (!finish) status = ORC_E_NOCONV;
  }
  rep->status = status;
  free(r); free(z); free(p); free(q); free(w);
  return status;
}

/* ------------------------------------------------------------------------------------ */
/* O5. Time-step driver: N_1 = I; u^{n+1} = PSPGMRES(A, u^n, N_n, ...); N_{n+1} = MREP.  */
/* (Eq.3-4; "used as a preconditioner ... for the next time step").       */
/* ------------------------------------------------------------------------------------ */
int orc_time_steps(const orc_operator* A, double* u, int steps, const orc_step_opts* opt,
                   orc_ring* ring, double* bands_N, double* lu_N, int* n_is_identity,
                   orc_step_report* reports, double* resid_hist, int hist_cap) {
  const int64_t n = orc_op_rows(A);
  const int d = opt->d;
  double* b = (double*)malloc((size_t)n * sizeof(double));
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* fit = (double*)malloc((size_t)n * (size_t)(2 * d + 1) * sizeof(double));
  int hist_used = 0;
  int worst = ORC_OK;
  for (int s = 0; s < steps; ++s) {
    orc_step_report* R = &reports[s];
    memset(R, 0, sizeof(*R));
    if (opt->reset_history) { ring->count = 0; ring->head = 0; }
    copy(n, u, b);                                 /* b := u^n (Eq.4 right-hand side) */
    double eps = opt->tol * norm2(n, b);           /* R1 */
    R->precond_was_identity = *n_is_identity;
    int st;
    if (opt->method == ORC_METHOD_CG)                /* f4: PSP-CG (R27-R31) */
      st = orc_pcg(A, b, u, x, d, *n_is_identity ? NULL : lu_N, eps, opt->restart * opt->max_cycles, ring,
                   &R->solve, resid_hist ? resid_hist + hist_used : NULL,
                   resid_hist ? hist_cap - hist_used : 0);
    else
      st = orc_pspgmres(A, b, u, x, d, *n_is_identity ? NULL : lu_N, eps, opt->restart,
                        opt->max_cycles, ring, &R->solve,
                        resid_hist ? resid_hist + hist_used : NULL,
                        resid_hist ? hist_cap - hist_used : 0, NULL, 0, NULL);
    if (resid_hist) hist_used += (R->solve.hist_len < hist_cap - hist_used ? R->solve.hist_len : hist_cap - hist_used);
    if (st == ORC_E_NONFINITE || st == ORC_E_SINGULAR || st == ORC_E_ARG) { worst = st; break; }
    if (st != ORC_OK && worst == ORC_OK) worst = st;
    copy(n, x, u);                                 /* u^{n+1} */
    /* MREP for the next step, then R18 + the gate R21, then factor */
    if (ring->count >= 2 * d + 2) {
      int order[4096];
      int m = ring->count;
      for (int c = 0; c < m; ++c) order[c] = orc_ring_slot(ring, c);
      int mst = orc_mrep(n, m, ring->px, ring->py, n, order, d, fit, NULL, NULL, NULL, &R->mrep);
      R->mrep_ran = (mst == ORC_OK);
      if (mst == ORC_OK && opt->method == ORC_METHOD_CG) {
        /* R29: CG needs a symmetric positive definite preconditioner: N_s = (N + N^T) / 2,
         * gated by positive-diagonal strict dominance */
        double* sym = (double*)malloc((size_t)n * (size_t)(2 * d + 1) * sizeof(double));
        orc_sym_bands(n, d, fit, sym);
        copy(n * (int64_t)(2 * d + 1), sym, fit);
        free(sym);
        R->mrep.gate_accepted = orc_gate_spd(n, d, fit);
      }
      int accept = (mst == ORC_OK) && (R->mrep.gate_accepted || !opt->gate);
      if (accept) {
        if (orc_banded_lu(n, d, fit, lu_N) == ORC_OK) {
          copy(n * (int64_t)(2 * d + 1), fit, bands_N);
          *n_is_identity = 0;
        } else {
          accept = 0;
        }
      }
      R->mrep.gate_accepted = accept;
      if (!accept) *n_is_identity = 1;
    }
  }
  free(b);
  free(x);
  free(fit);
  return worst;
}
