// resident.cu -- f2: the whole restarted PSP-GMRES solve (Alg.1) as ONE
// persistent kernel, for the small and L2-resident systems (C1 1-D n = 1024, C2 2-D 512^2, the
// paper's own n <= 700 seven-diagonal family) whose host-driven cycle is bound by launch latency
// and the per-step device->host read of R(k) (~20 us a step).
//
// Every CTA owns a contiguous block of rows and replicates the O(n_A^2) scalar state of the cycle
// (Hessenberg, Givens rotations, G, the ICWY L matrix, the lagged normalisations) in shared
// memory; the grid meets only at the reductions.  An Arnoldi step is two grid-wide reductions:
//   [A] probe Y_k = N^{-1}(alpha_k V_k) -> P_x, w = A Y_k -> P_y (l.10-12), the inner products
//       s_j = V_j'w and l_j = V_j'V_k (one-reduction MGS, R11), reduced; every CTA solves
//       (I + L) h = s for H(1..k, k) (l.13-16);
//   [B] U = w - sum_j h_j V_j -> V(:,k+1) (stored unnormalised), ||U||^2, reduced; every CTA
//       applies the Givens update (l.17-32) and tests R(k) <= eps (l.33) -- identical inputs,
//       identical decisions, no broadcast needed.
// Reductions are deterministic (fixed partition, fixed summation order, the same in every CTA),
// so results are bitwise reproducible.  The grid barrier is a monotone arrival counter
// (cooperative launch: every CTA is co-resident).  One CTA (n <= 4096): barriers are
// __syncthreads() only.  A banded N (accepted by the gate, R21) is applied by one thread's
// sequential forward / backward sweeps (P:30's Thomas recurrence for d = 1), so it is offered only
// to one-CTA problems (n <= kResidentSeqRows).
//
// Same arithmetic as the host-driven split path (icwy_dots / icwy_update / combine kernels of
// krylov.cu, up to the association of the reductions): T4-T6 parity with the oracle holds in the
// same tolerances (tests/test_gpu_parity.py, mode "resident").
#include <math.h>

#include "givens.cuh"
#include "internal.h"
#include "stencil_row.cuh"

namespace psp {
namespace {

constexpr int RT = 512;          // threads per CTA
constexpr int RMAX = 8;          // rows per thread (n <= grid * RT * RMAX)
constexpr int RW = RT / 32;

struct ResArgs {
  Stencil st;
  const double* b;
  double* X0;                    // in: x0; out: the last iterate (l.43)
  double* V;                     // (nA+1) columns of ldv: V(:,j) unnormalised, scale alpha_j
  int64_t ldv;
  double* ring_px;
  double* ring_py;
  double* slot_scale;
  int ring_cap, ring_phys, ring_head, ring_count;
  const double* lu;              // banded LU factors of N (NULL: N = I)
  int d;
  double* y;                     // n: sweep intermediate (N != I)
  double* z;                     // n: Z of the cycle end (N != I)
  int nA, max_cycles;
  int tol_abs;
  double tol;
  int64_t chunk;                 // rows per CTA
  double* partials;              // [2][grid][2 nA + 2]: double-buffered (a CTA may write reduction
                                 // r+1's partial while a slower one still reads reduction r's)
  unsigned long long* bar;       // arrival counter (zeroed before the launch)
  double* hist;                  // R(k) of every inner iteration (hist_cap)
  int hist_cap;
  double* betas;                 // beta per cycle (beta_cap)
  int beta_cap;
  double* out;                   // summary, see enum
  DevState ds;                   // global mirror of the scalar state (test hooks)
};
enum { O_ITER = 0, O_CYCLES, O_MATVECS, O_PAPPLY, O_FINISH, O_STATUS, O_R0, O_EPS, O_EST, O_TRUE, O_HLEN,
       O_BLEN, O_HEAD, O_COUNT, O_N };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// transposing butterfly: v[0..7] per lane -> lane l holds the warp sum of v[l & 7]
__device__ __forceinline__ double butterfly8(double (&v)[8], int lane) {
#pragma unroll
  for (int m = 4, h = 4; m >= 1; m >>= 1, h >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double send = up ? v[j] : v[j + h];
      const double keep = up ? v[j + h] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  double r = v[0];
  r += __shfl_xor_sync(0xffffffffu, r, 8);
  r += __shfl_xor_sync(0xffffffffu, r, 16);
  return r;
}

// the cooperative grid is at most one CTA per SM: 148 on B200 -> five rounds of 32 (host-checked)
constexpr int kCtaRounds = 5;

// grid barrier: monotone arrival counter, epoch e -> wait for grid * e arrivals
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long& epoch) {
  __syncthreads();
  if (gridDim.x > 1) {
    epoch += 1;
    if (threadIdx.x == 0) {
      const unsigned long long target = epoch * gridDim.x;
      __threadfence();
      atomicAdd(bar, 1ull);
      unsigned long long v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      } while (v < target);
      __threadfence();
    }
    __syncthreads();
  }
}

// loads of data written in this launch: L2 only across CTAs, L1-cached within the one CTA
template <int M>
__device__ __forceinline__ double ldm(const double* p) { return M == 2 ? *p : __ldcg(p); }

// (A x)_g for the operator kinds of the context, x written in this launch (M: ld's policy)
// not inlined: the kernel evaluates rows in unrolled per-thread loops, and nine inlined stencil
// variants per row would make the kernel megabytes of code (instruction-fetch bound)
template <int M>
__device__ __noinline__ double arow(const Stencil& st, const double* x, int64_t g, int i, int j, int k, double& xc) {
  if (st.kind == PSP_OP_DIA) {
    xc = ldm<M>(x + g);
    return dia_row<M>(st, x, g);
  }
  switch (st.kind * 4 + st.ndim) {
    case PSP_OP_CONST_DIFF * 4 + 1: return stencil_row<PSP_OP_CONST_DIFF, 1, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CONST_DIFF * 4 + 2: return stencil_row<PSP_OP_CONST_DIFF, 2, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CONST_DIFF * 4 + 3: return stencil_row<PSP_OP_CONST_DIFF, 3, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CELL_DIFF * 4 + 1: return stencil_row<PSP_OP_CELL_DIFF, 1, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CELL_DIFF * 4 + 2: return stencil_row<PSP_OP_CELL_DIFF, 2, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CELL_DIFF * 4 + 3: return stencil_row<PSP_OP_CELL_DIFF, 3, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CELL_ADVDIFF * 4 + 1: return stencil_row<PSP_OP_CELL_ADVDIFF, 1, M>(st, x, i, j, k, g, xc);
    case PSP_OP_CELL_ADVDIFF * 4 + 2: return stencil_row<PSP_OP_CELL_ADVDIFF, 2, M>(st, x, i, j, k, g, xc);
    default: return stencil_row<PSP_OP_CELL_ADVDIFF, 3, M>(st, x, i, j, k, g, xc);
  }
}

// (A x) at this thread's rows g_q = gb + q T (q < R, g_q < r1) -> y[q], with x_g -> xc[q]:
// every load of the R rows is issued (predicated) before any face is evaluated, then the faces
// in stencil_row's order and arithmetic (bitwise its result).  One rank only (the resident solve):
// a neighbour outside the grid is the Dirichlet zero, never a halo plane.
template <int KIND, int NDIM, int M, int R, int T>
__device__ __forceinline__ void rows_eval(const Stencil& st, const double* __restrict__ x, int64_t gb, int64_t r1,
                                          double (&y)[R], double (&xc)[R]) {
  constexpr bool cell = KIND != PSP_OP_CONST_DIFF;
  constexpr int NB = 2 * NDIM;
  const double* __restrict__ f = st.field;
  const unsigned unx = (unsigned)st.nx, uny = (unsigned)st.ny;
  const int64_t strides[3] = {1, st.nx, st.nx * st.ny};
  double xn[R][NB], fn[R][NB], fc[R];
  bool in[R][NB];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int64_t g = gb + (int64_t)q * T;
    const bool valid = g < r1;
    const unsigned ug = valid ? (unsigned)g : 0u;
    const unsigned ci = NDIM == 1 ? ug : ug % unx;
    const unsigned cj = NDIM == 1 ? 0u : (NDIM == 2 ? ug / unx : (ug / unx) % uny);
    const unsigned ck = NDIM == 3 ? ug / (unx * uny) : 0u;
    const unsigned cc[3] = {ci, cj, ck};
    const int64_t ext[3] = {st.nx, st.ny, st.nz};
    xc[q] = valid ? ldx<M>(x + g) : 0.0;
    fc[q] = (cell && valid) ? __ldg(f + g) : 0.0;
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
#pragma unroll
      for (int dd = 0; dd < 2; ++dd) {                 // dd 0: -1 (w / s / b), 1: +1 (e / n / t)
        const int nb = 2 * a + dd;
        const bool ok = valid && (dd == 0 ? cc[a] > 0u : (int64_t)cc[a] + 1 < ext[a]);
        const int64_t gn = g + (dd == 0 ? -strides[a] : strides[a]);
        in[q][nb] = ok;
        xn[q][nb] = ok ? ldx<M>(x + gn) : 0.0;
        fn[q][nb] = (cell && ok) ? __ldg(f + gn) : 0.0;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const double c0 = xc[q];
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
#pragma unroll
      for (int dd = 0; dd < 2; ++dd) {
        const int nb = 2 * a + dd;
        const double kf = cell ? (in[q][nb] ? 0.5 * (fc[q] + fn[q][nb]) : fc[q]) : 1.0;
        acc = fma(st.s[a] * kf, c0 - xn[q][nb], acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[a], c0 - xn[q][2 * a], acc);
    }
    y[q] = c0 + acc;
  }
}

// the R rows of rows_eval for the context's operator kind (one body per kind and dimension; not
// inlined: three call sites of nine variants would be megabytes of code).  y, xc: R doubles.
template <int M, int R, int T>
__device__ __noinline__ void arow_rows(const Stencil& st, const double* x, int64_t gb, int64_t r1, double* y,
                                       double* xc) {
  constexpr int G = R < 4 ? R : 4;                  // rows a group (more would spill the loads)
#pragma unroll 1
  for (int g0 = 0; g0 < R; g0 += G) {
    const int64_t gg = gb + (int64_t)g0 * T;
    double yy[G], xx[G];
    switch (st.kind * 4 + st.ndim) {
      case PSP_OP_CONST_DIFF * 4 + 1: rows_eval<PSP_OP_CONST_DIFF, 1, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CONST_DIFF * 4 + 2: rows_eval<PSP_OP_CONST_DIFF, 2, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CONST_DIFF * 4 + 3: rows_eval<PSP_OP_CONST_DIFF, 3, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CELL_DIFF * 4 + 1: rows_eval<PSP_OP_CELL_DIFF, 1, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CELL_DIFF * 4 + 2: rows_eval<PSP_OP_CELL_DIFF, 2, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CELL_DIFF * 4 + 3: rows_eval<PSP_OP_CELL_DIFF, 3, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CELL_ADVDIFF * 4 + 1: rows_eval<PSP_OP_CELL_ADVDIFF, 1, M, G, T>(st, x, gg, r1, yy, xx); break;
      case PSP_OP_CELL_ADVDIFF * 4 + 2: rows_eval<PSP_OP_CELL_ADVDIFF, 2, M, G, T>(st, x, gg, r1, yy, xx); break;
      default: rows_eval<PSP_OP_CELL_ADVDIFF, 3, M, G, T>(st, x, gg, r1, yy, xx); break;
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      y[g0 + q] = yy[q];
      xc[g0 + q] = xx[q];
    }
  }
}

// N^{-1} v by the sequential recurrences of the factors (O2's order of operations):
// y_i = v_i - sum_{j<i} L(i,j) y_j, z_i = (y_i - sum_{j>i} U(i,j) z_j) / U(i,i).  One thread.
// vs: v is scaled by vs on the fly.  z may alias v (v is consumed by the forward sweep).
__device__ void seq_solve(const double* lu, int64_t n, int d, const double* v, double vs, double* y, double* z,
                          const double* add) {
  for (int64_t i = 0; i < n; ++i) {
    double s = vs * v[i];
    for (int o = 0; o < d; ++o) {
      const int64_t j = i + o - d;
      if (j >= 0) s -= __ldg(lu + (int64_t)o * n + i) * y[j];
    }
    y[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int o = d + 1; o <= 2 * d; ++o) {
      const int64_t j = i + o - d;
      if (j < n) s -= __ldg(lu + (int64_t)o * n + i) * z[j];
    }
    z[i] = s / __ldg(lu + (int64_t)d * n + i);
  }
  if (add)
    for (int64_t i = 0; i < n; ++i) z[i] = add[i] + z[i];
}

// N^{-1} (vs v) for d = 1 (tridiagonal: P:30's Thomas recurrence) by the whole CTA: both
// sweeps are first-order affine recurrences, y_i = v_i - l_i y_{i-1} and
// z_i = y_i / u_i - (c_i / u_i) z_{i+1}; each thread composes the map of its chunk of rows, a
// block-wide scan (Hillis-Steele over the RT chunk maps, in shared memory) gives every chunk its
// incoming state, and each thread re-walks its chunk from it.  Equal to the sequential sweeps in
// exact arithmetic (composition of affine maps is associative).  y: n-vector scratch; z may
// alias v (v is consumed by the forward sweep).  sm2: 2 RT doubles.
template <int T>
__device__ void scan_solve_d1(const double* lu, int64_t n, const double* v, double vs, double* y, double* z,
                              double* sm2) {
  const int t = threadIdx.x;
  const int64_t L = (n + T - 1) / T;
  const int64_t i0 = t * L, i1 = (i0 + L < n) ? i0 + L : n;
  const double* lo = lu;              // band 0: L(i, i-1)
  const double* dg = lu + n;          // band 1: U(i, i)
  const double* up = lu + 2 * n;      // band 2: U(i, i+1)
  double* A = sm2;
  double* B = sm2 + T;
  // forward: y_i = a_i y_{i-1} + b_i, a_i = -l_i, b_i = vs v_i; chunk map y_out = A y_in + B
  double ca = 1.0, cb = 0.0;
  for (int64_t i = i0; i < i1; ++i) {
    const double ai = (i > 0) ? -__ldg(lo + i) : 0.0, bi = vs * v[i];
    ca = ai * ca;
    cb = fma(ai, cb, bi);
  }
  A[t] = ca;
  B[t] = cb;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {          // inclusive scan: (A,B)_t <- (A,B)_t o (A,B)_{t-off}
    double na = A[t], nb = B[t];
    if (t >= off) { nb = fma(A[t], B[t - off], B[t]); na = A[t] * A[t - off]; }
    __syncthreads();
    A[t] = na;
    B[t] = nb;
    __syncthreads();
  }
  double yin = (t > 0) ? B[t - 1] : 0.0;            // y_{i0-1} (the state entering the chunk)
  for (int64_t i = i0; i < i1; ++i) {
    const double ai = (i > 0) ? -__ldg(lo + i) : 0.0;
    yin = fma(ai, yin, vs * v[i]);
    y[i] = yin;
  }
  __syncthreads();
  // backward: z_i = e_i z_{i+1} + f_i, e_i = -c_i / u_i, f_i = y_i / u_i, from the last row
  ca = 1.0;
  cb = 0.0;
  for (int64_t i = i1 - 1; i >= i0; --i) {
    const double ui = __ldg(dg + i);
    const double ei = (i + 1 < n) ? -__ldg(up + i) / ui : 0.0, fi = y[i] / ui;
    ca = ei * ca;
    cb = fma(ei, cb, fi);
  }
  const int tr = T - 1 - t;                        // reversed order: chunk T-1 first
  A[tr] = ca;
  B[tr] = cb;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    double na = A[t], nb = B[t];
    if (t >= off) { nb = fma(A[t], B[t - off], B[t]); na = A[t] * A[t - off]; }
    __syncthreads();
    A[t] = na;
    B[t] = nb;
    __syncthreads();
  }
  double zin = (tr > 0) ? B[tr - 1] : 0.0;          // z_{i1} (the state entering from above)
  for (int64_t i = i1 - 1; i >= i0; --i) {
    const double ui = __ldg(dg + i);
    const double ei = (i + 1 < n) ? -__ldg(up + i) / ui : 0.0;
    zin = fma(ei, zin, y[i] / ui);
    z[i] = zin;
  }
  __syncthreads();
}

#ifdef PSP_RES_PROFILE
// phase timer (instrumented builds only): cycles from mark q-1 to mark q summed into out[16 + q]
#define PROF_MARK(q)                                                        \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      const long long now = clock64();                                      \
      if ((q) > 0) a.out[16 + (q)] += (double)(now - prof_t);               \
      prof_t = now;                                                         \
    }                                                                       \
  } while (0)
#else
#define PROF_MARK(q) do {} while (0)
#endif

template <int M, int R, int T>
__global__ void __launch_bounds__(T, 1) resident_kernel(ResArgs a) {
  constexpr int TW = T / 32;
#ifdef PSP_RES_PROFILE
  long long prof_t = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int q = 16; q < 24; ++q) a.out[q] = 0.0;
#endif
  extern __shared__ __align__(16) double sm[];
  const int nA = a.nA, ld = nA + 1, PV = 2 * nA + 2;
  double* H = sm;                       // (nA+1) x nA, rotated in place
  double* Lm = H + (size_t)ld * nA;     // (nA+1) x (nA+1)
  double* Gv = Lm + (size_t)ld * ld;    // nA+1
  double* Cv = Gv + ld;                 // nA
  double* Sv = Cv + nA;                 // nA
  double* al = Sv + nA;                 // nA+1
  double* Qv = al + ld;                 // nA
  double* rs = Qv + nA;                 // nA (R(k) of the cycle)
  double* sc = rs + nA;                 // SC_NSCAL
  double* red = sc + SC_NSCAL;          // [TW][PV] (also the 2 T doubles of the block scans)
  const int REDN = TW * PV > 2 * T ? TW * PV : 2 * T;
  double* tot = red + REDN;             // PV
  DevState S;                           // the replicated scalar state (givens_update's view)
  S.H = H;
  S.Hraw = a.ds.Hraw;                   // identical writes from every CTA (test hook)
  S.G = Gv;
  S.C = Cv;
  S.S = Sv;
  S.Q = Qv;
  S.Lm = Lm;
  S.alpha = al;
  S.scal = sc;
  S.resid = rs;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t n = a.st.n;
  const int64_t r0 = (int64_t)blockIdx.x * a.chunk;
  const int64_t r1 = (r0 + a.chunk < n) ? r0 + a.chunk : n;
  const bool lead = blockIdx.x == 0 && t == 0;
  const bool seqN = a.lu != nullptr;    // one CTA (host-checked)
  unsigned long long epoch = 0;
  unsigned nred = 0;                    // grid reductions so far (partials buffer parity)
  int head = a.ring_head, count = a.ring_count;
  auto ring_next = [&]() -> int {       // R20: FIFO of capacity ring_cap over ring_phys slots
    const int slot = (head + count) % a.ring_phys;
    if (count < a.ring_cap) count += 1;
    else head = (head + 1) % a.ring_phys;
    return slot;
  };
  auto V = [&](int j) -> double* { return a.V + (int64_t)j * a.ldv; };   // 0-based column

  // deterministic grid sum of nv per-thread values given by f(j, q) summed over this thread's
  // rows: block butterflies -> red -> this CTA's tot -> partials -> every CTA sums the grid's
  // partials in CTA order -> tot (valid in every thread after the call)
  // w0 (one CTA): the totals are formed by warp 0 and valid only there (its caller consumes
  // them in warp 0 and meets the block at its own barrier) -- one __syncthreads fewer
  // the totals of the warp partials in red (red_finish) -- see grid_reduce
  auto red_finish = [&](int nv, bool w0) {
    if (gridDim.x > 1) PROF_MARK(6);                  // (instrumented: the local work)
    __syncthreads();
    if (w0 && gridDim.x == 1) {
      if (warp == 0) {
        for (int j = lane; j < nv; j += 32) {
          double s = 0.0;
          for (int w = 0; w < TW; ++w) s += red[w * PV + j];
          tot[j] = s;
        }
        __syncwarp();
      }
      return;
    }
    for (int j = t; j < nv; j += T) {
      double s = 0.0;
      for (int w = 0; w < TW; ++w) s += red[w * PV + j];
      tot[j] = s;
    }
    if (gridDim.x > 1) {
      double* part = a.partials + (size_t)(nred & 1u) * gridDim.x * PV;
      nred += 1;
      __syncthreads();
      for (int j = t; j < nv; j += T) __stcg(part + (int64_t)blockIdx.x * PV + j, tot[j]);
      grid_sync(a.bar, epoch);
      PROF_MARK(7);                                   // (instrumented: CTA totals + the grid barrier)
      // values j = warp + TW q: every lane sums CTAs lane, lane + 32, ... for up to 4 values at
      // once (independent loads in flight), then a warp butterfly; fixed order in every CTA
      // (kCtaRounds rounds of 32 CTAs: every load of a value set is issued before the adds, which
      // keep the CTA order c = lane, lane + 32, ...; a partial written by another SM is an L2
      // round trip, so a dependent load per round was most of the reduction, r02 profile)
      for (int j0 = warp; j0 < nv; j0 += 4 * TW) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        double x4[kCtaRounds][4];
#pragma unroll
        for (int rr = 0; rr < kCtaRounds; ++rr) {
          const int c = lane + 32 * rr;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = j0 + q * TW;
            x4[rr][q] = (c < (int)gridDim.x && j < nv) ? ldm<M>(part + (int64_t)c * PV + j) : 0.0;
          }
        }
#pragma unroll
        for (int rr = 0; rr < kCtaRounds; ++rr) {
          if (lane + 32 * rr < (int)gridDim.x) {
#pragma unroll
            for (int q = 0; q < 4; ++q) s4[q] += x4[rr][q];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double sv = warp_sum(s4[q]);
          if (lane == 0 && j0 + q * TW < nv) tot[j0 + q * TW] = sv;
        }
      }
    }
    __syncthreads();
  };
  auto grid_reduce = [&](int nv, auto&& f, bool w0 = false) {
    for (int j0 = 0; j0 < nv; j0 += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (j0 + q < nv) ? f(j0 + q) : 0.0;
      const double r = butterfly8(v, lane);
      if (lane < 8 && j0 + lane < nv) red[warp * PV + j0 + lane] = r;
    }
    red_finish(nv, w0);
  };

  // this thread's rows: r0 + t + q T, q < R; with few rows a thread their grid coordinates are
  // kept (no integer divisions in the step), else recomputed per use (registers)
  double w[R];
  constexpr bool PRE = R <= 2;
  int ci0[PRE ? R : 1], cj0[PRE ? R : 1], ck0[PRE ? R : 1];
#pragma unroll
  for (int q = 0; q < (PRE ? R : 1); ++q) {
    const int64_t g = r0 + t + (int64_t)q * T;
    ci0[q] = (int)(g % a.st.nx);
    cj0[q] = (int)((g / a.st.nx) % a.st.ny);
    ck0[q] = (int)(g / (a.st.nx * a.st.ny));
  }
  // (32-bit: the resident solve's n < 2^31 -- a 64-bit division is an out-of-line call)
  const unsigned unx = (unsigned)a.st.nx, uny = (unsigned)a.st.ny;
  auto ug = [&](int q) { return (unsigned)(r0 + t + (int64_t)q * T); };
  auto ci = [&](int q) { return PRE ? ci0[q] : (int)(ug(q) % unx); };
  auto cj = [&](int q) { return PRE ? cj0[q] : (int)((ug(q) / unx) % uny); };
  auto ck = [&](int q) { return PRE ? ck0[q] : (int)(ug(q) / (unx * uny)); };
  int iters = 0, cycles = 0, matvecs = 0, papply = 0, hlen = 0, blen = 0, status = 0;
  bool finish = false;
  double r0v = 0.0, est = 0.0, eps;
  if (a.tol_abs) {
    eps = a.tol;
  } else {                                             // R1: eps = tol ||b||
    grid_reduce(1, [&](int) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int64_t g = r0 + t + (int64_t)q * T;
        if (g < r1) { const double bv = __ldg(a.b + g); s = fma(bv, bv, s); }
      }
      return s;
    });
    eps = a.tol * sqrt(tot[0]);
  }
  if (t == 0) sc[SC_EPS] = eps;
  __syncthreads();

  for (int l = 1; l <= a.max_cycles; ++l) {            // l.3
    // ---- l.4-7: probe (X0, A X0); R_bar = B - A X0 -> V(:,1); beta ----
    int slot = ring_next();
    double* px = a.ring_px + (int64_t)slot * n;
    double* py = a.ring_py + (int64_t)slot * n;
    if (lead) a.slot_scale[slot] = 1.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t g = r0 + t + (int64_t)q * T;
      w[q] = 0.0;
      if (g < r1) {
        double xc;
        const double y = arow<M>(a.st, a.X0, g, ci(q), cj(q), ck(q), xc);
        __stcs(px + g, xc);                              // probes: evict-first (V stays in L2)
        __stcs(py + g, y);
        const double rr = __ldg(a.b + g) - y;
        V(0)[g] = rr;
        w[q] = rr;
      }
    }
    grid_reduce(1, [&](int) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) s = fma(w[q], w[q], s);
      return s;
    });
    const double beta = sqrt(tot[0]);
    matvecs += 1;
    cycles += 1;
    if (lead && blen < a.beta_cap) a.betas[blen] = beta;
    blen += 1;
    if (l == 1) r0v = beta;
    if (!isfinite(beta)) { status = PSP_E_NONFINITE; break; }
    if (beta <= eps) { finish = true; est = beta; break; }   // R3
    if (t == 0) {
      for (int q = 0; q <= nA; ++q) Gv[q] = 0.0;     // l.44 "clean"
      Gv[0] = beta;                                    // l.7
      al[0] = 1.0 / beta;                              // V(:,1) = R_bar / beta (l.6), lagged
    }
    __syncthreads();
    int kdone = 0;
    for (int k = 1; k <= nA; ++k) {                  // l.8
      // ---- [A] l.10-12: Y_k = N^{-1} V(:,k) -> P_x, A Y_k -> P_y; l.13-16's inner products ----
      PROF_MARK(0);
      slot = ring_next();
      px = a.ring_px + (int64_t)slot * n;
      py = a.ring_py + (int64_t)slot * n;
      if (lead) a.slot_scale[slot] = 1.0;
      const double ak = al[k - 1];
      const double* Vk = V(k - 1);
      if (seqN) {                                      // one CTA: the sweeps of P:30 (d = 1: a
        if (a.d == 1) {                                // block scan of the affine recurrences)
          scan_solve_d1<T>(a.lu, n, Vk, ak, a.y, px, red);
        } else {
          if (t == 0) seq_solve(a.lu, n, a.d, Vk, ak, a.y, px, nullptr);
          __syncthreads();
        }
        papply += 1;
      }
      double vk[R];
      if (a.st.kind != PSP_OP_DIA) {                   // every row's loads in flight together
        double yr[R], xr[R];
        arow_rows<M, R, T>(a.st, seqN ? px : Vk, r0 + t, r1, yr, xr);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int64_t g = r0 + t + (int64_t)q * T;
          w[q] = 0.0;
          vk[q] = 0.0;
          if (g < r1) {
            if (seqN) {
              w[q] = yr[q];
              vk[q] = ldm<M>(Vk + g);
            } else {                                   // N = I: Y_k = alpha_k V(:,k)
              vk[q] = xr[q];
              w[q] = ak * yr[q];
              __stcs(px + g, ak * xr[q]);               // probes: evict-first (V stays in L2)
            }
            __stcs(py + g, w[q]);
          }
        }
      } else {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int64_t g = r0 + t + (int64_t)q * T;
        w[q] = 0.0;
        vk[q] = 0.0;
        if (g < r1) {
          double xc;
          if (seqN) {
            w[q] = arow<M>(a.st, px, g, ci(q), cj(q), ck(q), xc);
            vk[q] = ldm<M>(Vk + g);
          } else {                                     // N = I: Y_k = alpha_k V(:,k)
            const double y = arow<M>(a.st, Vk, g, ci(q), cj(q), ck(q), xc);
            vk[q] = xc;
            w[q] = ak * y;
            px[g] = ak * xc;
          }
          py[g] = w[q];
        }
      }
      }
      matvecs += 1;
      // s_j = V_j' w (j < k) at [0, k), l_j = V_j' V_k (j < k-1) at [k, 2k-1) (EPI_DOTS layout)
      PROF_MARK(1);
      // one load of V_j for both of its products, eight columns (all their loads in flight) a
      // round; the per-thread values and the butterfly / warp-sum order are grid_reduce's
      for (int j0 = 0; j0 < k; j0 += 8) {
        double vs[8], vl[8];
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8) {
          const int j = j0 + q8;
          double ss = 0.0, sl = 0.0;
          if (j < k) {
            const double* Vj = V(j);
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const int64_t g = r0 + t + (int64_t)q * T;
              if (g < r1) {
                const double x = ldm<M>(Vj + g);
                ss = fma(x, w[q], ss);
                sl = fma(x, vk[q], sl);
              }
            }
          }
          vs[q8] = ss;
          vl[q8] = (j < k - 1) ? sl : 0.0;
        }
        const double rs = butterfly8(vs, lane);
        const double rl = butterfly8(vl, lane);
        if (lane < 8 && j0 + lane < k) red[warp * PV + j0 + lane] = rs;
        if (lane < 8 && j0 + lane < k - 1) red[warp * PV + k + j0 + lane] = rl;
      }
      red_finish(2 * k - 1, true);
      PROF_MARK(2);
      if (warp == 0) {                                 // (I + L) h = s (R11), as EPI_DOTS, by warp 0:
        double* Lrow = Lm + (int64_t)(k - 1) * ld;     // right-looking -- lane i holds s_i (and
        for (int jb = lane; jb < k - 1; jb += 32) Lrow[jb] = al[jb] * ak * tot[k + jb];   // s_{i+32})
        __syncwarp();
        double s0 = lane < k ? al[lane] * tot[lane] : 0.0;
        double s1 = lane + 32 < k ? al[lane + 32] * tot[lane + 32] : 0.0;
        for (int jb = 0; jb < k; ++jb) {               // h_jb final: broadcast, update the rest
          const double hj = __shfl_sync(0xffffffffu, jb < 32 ? s0 : s1, jb & 31);
          if (lane > jb && lane < k) s0 = fma(-Lm[(int64_t)lane * ld + jb], hj, s0);
          if (lane + 32 > jb && lane + 32 < k) s1 = fma(-Lm[(int64_t)(lane + 32) * ld + jb], hj, s1);
        }
        double* Hc = H + (int64_t)(k - 1) * ld;
        if (lane < k) Hc[lane] = s0;
        if (lane + 32 < k) Hc[lane + 32] = s1;
      }
      __syncthreads();
      PROF_MARK(3);
      // ---- [B] l.13-17: U = w - sum_j h_j alpha_j V_j -> V(:,k+1); H(k+1,k) = ||U|| ----
      {
        const double* Hc = H + (int64_t)(k - 1) * ld;
        double* Vn = V(k);
        // columns outer, this thread's rows inner: R independent chains (each row's in j order),
        // the loads of JC columns issued before their FMAs (one load round trip per JC columns)
        constexpr int JC = R <= 2 ? 8 : (R <= 4 ? 4 : 2);
        int j = 0;
        for (; j + JC <= k; j += JC) {
          double x[JC][R];
#pragma unroll
          for (int jj = 0; jj < JC; ++jj) {
            const double* Vj = V(j + jj);
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const int64_t g = r0 + t + (int64_t)q * T;
              x[jj][q] = (g < r1) ? ldm<M>(Vj + g) : 0.0;
            }
          }
#pragma unroll
          for (int jj = 0; jj < JC; ++jj) {
            const double cj = -(Hc[j + jj] * al[j + jj]);
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const int64_t g = r0 + t + (int64_t)q * T;
              if (g < r1) w[q] = fma(cj, x[jj][q], w[q]);
            }
          }
        }
        for (; j < k; ++j) {
          const double cj = -(Hc[j] * al[j]);
          const double* Vj = V(j);
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int64_t g = r0 + t + (int64_t)q * T;
            if (g < r1) w[q] = fma(cj, ldm<M>(Vj + g), w[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int64_t g = r0 + t + (int64_t)q * T;
          if (g < r1) Vn[g] = w[q];
          else w[q] = 0.0;
        }
      }
      grid_reduce(1, [&](int) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) s = fma(w[q], w[q], s);
        return s;
      }, true);
      if (t == 0) {
        H[(int64_t)(k - 1) * ld + k] = sqrt(tot[0]);  // l.17
        PROF_MARK(4);
        givens_update(S, k, nA);                      // l.18-32 (R4 breakdown, R10)
      }
      __syncthreads();
      PROF_MARK(5);
      const double R = sc[SC_RK];
      const int flags = (int)sc[SC_FLAGS];
      if (lead && hlen < a.hist_cap) a.hist[hlen] = R;
      hlen += 1;
      iters += 1;
      est = R;
      kdone = k;
      if (flags & PSP_FLAG_NONFINITE) { status = PSP_E_NONFINITE; break; }
      if (flags & (PSP_FLAG_CONVERGED | PSP_FLAG_BREAKDOWN)) { finish = true; break; }   // l.33-36
    }
    if (status != 0) break;
    // ---- l.38-43: Q = H^{-1} G (R6); X = X0 + N^{-1} sum_j Q_j V_j; X0 <- X ----
    if (t == 0) {
      int bad = 0;
      for (int j = kdone; j >= 1; --j) {
        double s = Gv[j - 1];
        for (int q = j + 1; q <= kdone; ++q) s -= H[(int64_t)(q - 1) * ld + (j - 1)] * Qv[q - 1];
        const double piv = H[(int64_t)(j - 1) * ld + (j - 1)];
        if (piv == 0.0) { bad = 1; Qv[j - 1] = 0.0; continue; }
        Qv[j - 1] = s / piv;
      }
      sc[SC_STATUS] = bad ? (double)PSP_E_SINGULAR : 0.0;
    }
    __syncthreads();
    if (sc[SC_STATUS] != 0.0) { status = PSP_E_SINGULAR; break; }
    double* zdst = seqN ? a.z : a.X0;
    {
      double zz[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int64_t g = r0 + t + (int64_t)q * T;
        zz[q] = (g < r1 && !seqN) ? ldm<M>(a.X0 + g) : 0.0;
      }
      for (int j = 0; j < kdone; ++j) {            // (as the update: R chains, each in j order)
        const double cj = Qv[j] * al[j];
        const double* Vj = V(j);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int64_t g = r0 + t + (int64_t)q * T;
          if (g < r1) zz[q] = fma(cj, ldm<M>(Vj + g), zz[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int64_t g = r0 + t + (int64_t)q * T;
        if (g < r1) zdst[g] = zz[q];
      }
    }
    if (seqN) {
      __syncthreads();
      // l.42: X = X0 + N^{-1} Z (Z consumed by the forward sweep, then reused for N^{-1} Z)
      if (a.d == 1) {
        scan_solve_d1<T>(a.lu, n, a.z, 1.0, a.y, a.z, red);
        for (int64_t i = t; i < n; i += T) a.X0[i] = a.X0[i] + a.z[i];
      } else if (t == 0) {
        seq_solve(a.lu, n, a.d, a.z, 1.0, a.y, a.z, nullptr);
        for (int64_t i = 0; i < n; ++i) a.X0[i] = a.X0[i] + a.z[i];
      }
      papply += 1;
    }
    grid_sync(a.bar, epoch);                           // X0 complete before the next probe
    if (finish) break;                                 // l.45-48
  }
  // ---- R13: true residual ||b - A x|| (one unrecorded matvec) ----
  double tr = 0.0;
  if (status == 0) {
    grid_reduce(1, [&](int) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int64_t g = r0 + t + (int64_t)q * T;
        if (g < r1) {
          double xc;
          const double rr = __ldg(a.b + g) - arow<M>(a.st, a.X0, g, ci(q), cj(q), ck(q), xc);
          s = fma(rr, rr, s);
        }
      }
      return s;
    });
    tr = sqrt(tot[0]);
  }
  if (lead) {
    double* o = a.out;
    o[O_ITER] = iters;
    o[O_CYCLES] = cycles;
    o[O_MATVECS] = matvecs;
    o[O_PAPPLY] = papply;
    o[O_FINISH] = finish ? 1.0 : 0.0;
    o[O_STATUS] = status;
    o[O_R0] = r0v;
    o[O_EPS] = eps;
    o[O_EST] = est;
    o[O_TRUE] = tr;
    o[O_HLEN] = hlen;
    o[O_BLEN] = blen;
    o[O_HEAD] = head;
    o[O_COUNT] = count;
  }
  if (blockIdx.x == 0) {                               // the scalar state for the test hooks
    for (int q = t; q < ld * nA; q += T) a.ds.H[q] = H[q];
    for (int q = t; q < ld * ld; q += T) a.ds.Lm[q] = Lm[q];
    for (int q = t; q < ld; q += T) { a.ds.G[q] = Gv[q]; a.ds.alpha[q] = al[q]; }
    for (int q = t; q < nA; q += T) { a.ds.C[q] = Cv[q]; a.ds.S[q] = Sv[q]; a.ds.Q[q] = Qv[q]; a.ds.resid[q] = rs[q]; }
  }
}

size_t res_smem(int nA) {
  const size_t ld = nA + 1, PV = 2 * nA + 2;
  const size_t redn = RW * PV > 2 * RT ? RW * PV : 2 * RT;
  return (ld * nA + ld * ld + ld + nA + nA + ld + nA + nA + SC_NSCAL + redn + PV) * 8;
}

}  // namespace

// one CTA per SM, at most 32 kCtaRounds (the partials readback's unrolled rounds)
static int max_grid() { return device_sms() < 32 * kCtaRounds ? device_sms() : 32 * kCtaRounds; }

bool resident_supported(int64_t n, int nA, bool banded_n) {
  if (nA > kResidentMaxRestart) return false;
  if (banded_n && n > kResidentSeqRows) return false;
  if (res_smem(nA) > 200 * 1024) return false;
  const int64_t per_cta = (int64_t)RT * RMAX;
  return n <= per_cta * max_grid();
}

int resident_grid(int64_t n, bool banded_n) {
  if (banded_n || n <= kResidentOneCtaRows) return 1;
  int64_t g = (n + RT - 1) / RT;                       // about one row per thread
  const int64_t need = (n + (int64_t)RT * RMAX - 1) / ((int64_t)RT * RMAX);
  if (g > max_grid()) g = max_grid();
  if (g < need) g = need;
  return (int)g;
}

size_t resident_scratch_doubles(int nA, int grid) { return (size_t)2 * grid * (2 * nA + 2); }

int launch_resident(const ResidentCall& c, cudaStream_t s) {
  ResArgs a;
  a.st = c.st;
  a.b = c.b;
  a.X0 = c.X0;
  a.V = c.V;
  a.ldv = c.ldv;
  a.ring_px = c.ring_px;
  a.ring_py = c.ring_py;
  a.slot_scale = c.slot_scale;
  a.ring_cap = c.ring_cap;
  a.ring_phys = c.ring_phys;
  a.ring_head = c.ring_head;
  a.ring_count = c.ring_count;
  a.lu = c.lu;
  a.d = c.d;
  a.y = c.y;
  a.z = c.z;
  a.nA = c.nA;
  a.max_cycles = c.max_cycles;
  a.tol_abs = c.tol_abs;
  a.tol = c.tol;
  const int grid = c.grid;
  a.chunk = (c.st.n + grid - 1) / grid;
  a.partials = c.partials;
  a.bar = c.bar;
  a.hist = c.hist;
  a.hist_cap = c.hist_cap;
  a.betas = c.betas;
  a.beta_cap = c.beta_cap;
  a.out = c.out;
  a.ds = c.ds;
  const size_t smem = res_smem(c.nA);
  const int dev = device_ordinal();
  thread_local size_t attr[kMaxDev] = {};
  if (attr[dev] < smem) {
    if (cudaFuncSetAttribute(resident_kernel<1, RMAX, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(resident_kernel<1, 4, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(resident_kernel<2, RMAX, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(resident_kernel<2, 2, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 1;
    attr[dev] = smem;
  }
  cudaMemsetAsync(c.bar, 0, sizeof(unsigned long long), s);
  void* args[] = {&a};
  if (grid > 1) {
    // at most four rows a thread (C2: 1772 rows a CTA): the register tile of four rows keeps
    // more column loads in flight than eight mostly idle ones
    const void* kern = a.chunk <= 4 * RT ? (const void*)resident_kernel<1, 4, RT> : (const void*)resident_kernel<1, RMAX, RT>;
    if (cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(RT), args, smem, s) != cudaSuccess)
      return 1;
  } else if (c.st.n <= 2 * RT) {
    // one CTA, two rows a thread (C1; measured against four warps with eight rows a thread:
    // 27 ms against 49 ms for C1's first step -- the per-row work is latency, not issue)
    resident_kernel<2, 2, RT><<<1, RT, smem, s>>>(a);
  } else {
    resident_kernel<2, RMAX, RT><<<1, RT, smem, s>>>(a);   // one CTA: L1-cached loads, no grid barrier
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace psp
