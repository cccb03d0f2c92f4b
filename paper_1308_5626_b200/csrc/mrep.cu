// mrep.cu -- K3: MREP, Algorithm 2, the per-row multi-regression that fits the
// banded N with P_y ~ N P_x, plus R18 and the R21 gate statistics.
//
// Interior rows: the normal equations (P_x* P_x*') N* = P_x* P_y*' with
// P_x* = [1; P_x(i-d,:); ...; P_x(i+d,:)].  The Gram entries are lagged cross products of
// neighbouring rows,
//     G_i[1+a][1+b] = C_{b-a}(i-d+a),  C_l(r) = sum_c P_x(r,c) P_x(r+l,c),
//     G_i[0][1+a]   = S(i-d+a),        S(r)   = sum_c P_x(r,c),   G_i[0][0] = m,
//     rhs_i[1+a]    = D_{a-d}(i),      D_l(i) = sum_c P_x(i+l,c) P_y(i,c),  rhs_i[0] = sum_c P_y(i,c)
// so each thread accumulates 4d+4 running sums for its own row (one FMA per sum per probe,
// columns oldest -> newest exactly as the oracle's per-row Gram), exchanges C and S with its
// 2d neighbours through shared memory, and solves its (2d+2)^2 system by Cholesky in
// registers (R17: condition estimate, one ridge retry, identity-row fallback).
//
// HBM-bound: per row 16m bytes of probes read once (P_x rows of the 2d-row halo come from the
// shared-memory tile) + 8(2d+1) bytes of bands written.  Blocks of 256 threads own 256 rows of
// sums and emit 256-2d rows (the 2d halo rows are recomputed by the neighbour block).
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "internal.h"

#ifndef PSP_MREP_NST
#define PSP_MREP_NST 3    // TMA stages of PSP_MREP_TCB probe columns each
#endif
#ifndef PSP_MREP_MINB
#define PSP_MREP_MINB 2   // resident blocks per SM of the TMA MREP kernel
#endif

namespace psp {
namespace {

constexpr int TPB = 256;
constexpr int CB = 12;         // probe columns staged per shared-memory round
constexpr int kMaxM = 256;     // probe columns supported

struct Cols {
  const double* px;            // column c of P_x at px + slot[c]*ld
  const double* py;
  const double* scale;         // per slot: the probe is scale[slot] * column (NULL: 1)
  const double* hlo;           // multi-rank: P_x rows row0-d..row0-1, [c*d + q] (NULL: none)
  const double* hhi;           //   and rows row0+n..row0+n+d-1
  int64_t grow0, gN;           // global index of local row 0; global rows
  int hd;                      // halo depth (= d)
  int64_t ld;
  int32_t slot[kMaxM];
  __device__ double sc(int c) const { return scale ? __ldg(scale + slot[c]) : 1.0; }
  // raw P_x(local row rr, column c) for rr in [-hd, n + hd); 0 beyond the global matrix
  __device__ double xraw(int c, int64_t rr, int64_t n) const {
    if (rr >= 0 && rr < n) return __ldg(px + (int64_t)slot[c] * ld + rr);
    if (rr < 0 && rr >= -hd && hlo) return __ldg(hlo + (int64_t)c * hd + (rr + hd));
    if (rr >= n && rr < n + hd && hhi) return __ldg(hhi + (int64_t)c * hd + (rr - n));
    return 0.0;
  }
};

template <int D>
__device__ __forceinline__ double band_abs_off_sum(const double (&row)[2 * D + 1], int64_t i, int64_t n) {
  double off = 0.0;
#pragma unroll
  for (int o = 0; o <= 2 * D; ++o) {
    const int64_t j = i + o - D;
    if (o == D || j < 0 || j >= n) continue;
    off += fabs(row[o]);
  }
  return off;
}

// Interior-row fit.  Writes bands / intercept / kind / kappa for rows d <= r < n-d and the
// per-block gate statistics.
// packed lower-triangular index (row a >= col b)
__host__ __device__ constexpr int pk(int a, int b) { return a * (a + 1) / 2 + b; }

// Gram of row r (thread t) from the lagged sums in shared memory:
// G[0][0] = m, G[1+a][0] = S(r-d+a), G[1+b][1+a] = C_{b-a}(r-d+a) (b >= a); + lambda on the diagonal
template <int D>
__device__ __forceinline__ void assemble(double (&A)[(2 * D + 2) * (2 * D + 3) / 2], const double* ex,
                                         int64_t TS, int t, int m, double lambda) {
  A[pk(0, 0)] = (double)m + lambda;
#pragma unroll
  for (int a = 0; a <= 2 * D; ++a) {
    A[pk(1 + a, 0)] = ex[(2 * D + 1) * TS + (t - D + a)];
#pragma unroll
    for (int b = a; b <= 2 * D; ++b) A[pk(1 + b, 1 + a)] = ex[(b - a) * TS + (t - D + a)];
    A[pk(1 + a, 1 + a)] += lambda;
  }
}

// in-place Cholesky of the packed P x P matrix (R17); false on a pivot^2 <= 0 or non-finite.
// Stores 1 / L_jj on the diagonal (one division per column; the solves multiply by it: each
// multiply-by-reciprocal adds at most one rounding, inside T3's 8 P u kappa_2(G) bound) and
// returns max_j L_jj, min_j L_jj for the condition estimate.  Straight-line (no early exit), so
// the packed matrix stays in registers.
// compile-time loop: f(std::integral_constant<int, i>) for i in [B, E) (forces full unrolling
// of the small dense kernels below; a rolled loop would index the packed Gram at run time and
// send it to local memory)
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// 1/sqrt(s) for s > 0: the hardware approximation refined by three Newton steps (each doubles
// the correct bits; within ~1 ulp).  Unlike sqrt() and '/', it has no out-of-line special-case
// path, whose call would force the packed Gram out of registers around every pivot.
__device__ __forceinline__ double rsqrt_nr(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double h = 0.5 * s;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = y * fma(-h * y, y, 1.5);
  return y;
}

// in-place Cholesky of the packed P x P matrix (R17); false on a pivot^2 <= 0 or non-finite.
// Stores 1/L_jj on the diagonal (the solves multiply by it: each product adds at most one
// rounding, inside T3's 8 P u kappa_2(G) bound) and returns max_j L_jj and max_j 1/L_jj for
// the condition estimate (max L_jj / min L_jj)^2 = (max L_jj * max 1/L_jj)^2.
template <int P>
__device__ __forceinline__ bool chol_packed(double (&A)[P * (P + 1) / 2], double& lmax, double& imax) {
  bool ok = true;
  static_for<0, P>([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    double s = A[pk(j, j)];
    static_for<0, j>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      s -= A[pk(j, k)] * A[pk(j, k)];
    });
    ok = ok && (s > 0.0) && isfinite(s);
    const double sv = ok ? s : 1.0;
    const double inv = rsqrt_nr(sv);               // 1 / L_jj
    const double ljj = sv * inv;                   // L_jj
    lmax = (j == 0) ? ljj : fmax(lmax, ljj);
    imax = (j == 0) ? inv : fmax(imax, inv);
    A[pk(j, j)] = inv;
    static_for<j + 1, P>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      double u = A[pk(i, j)];
      static_for<0, j>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        u -= A[pk(i, k)] * A[pk(j, k)];
      });
      A[pk(i, j)] = u * inv;
    });
  });
  return ok;
}

// 1/s for s > 0: the hardware approximation refined by two Newton steps (~23 -> 46 -> 92 bits)
__device__ __forceinline__ double rcp_nr(double s) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
#pragma unroll
  for (int it = 0; it < 2; ++it) y = fma(y, fma(-s, y, 1.0), y);
  return y;
}

// The same factorisation as LDL^T (G = L D L^T, L unit lower; L_chol = L sqrt(D)): no square
// roots on the critical path, one reciprocal a column.  Stores 1/D_jj on the diagonal and the
// strictly-lower L; the condition estimate (max L_jj / min L_jj)^2 of R17 is max D / min D =
// dmax * imax.  Failure (R17): a pivot D_jj <= 0 or non-finite.
template <int P>
__device__ __forceinline__ bool ldl_packed(double (&A)[P * (P + 1) / 2], double& dmax, double& imax) {
  bool ok = true;
  double dv[P];
  static_for<0, P>([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    double w[j > 0 ? j : 1];                       // w_k = L_jk D_k
    static_for<0, j>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      w[k] = A[pk(j, k)] * dv[k];
    });
    double sj = A[pk(j, j)];
    static_for<0, j>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      sj -= A[pk(j, k)] * w[k];
    });
    ok = ok && (sj > 0.0) && isfinite(sj);
    const double sv = ok ? sj : 1.0;
    const double inv = rcp_nr(sv);
    dv[j] = sv;
    dmax = (j == 0) ? sv : fmax(dmax, sv);
    imax = (j == 0) ? inv : fmax(imax, inv);
    A[pk(j, j)] = inv;
    static_for<j + 1, P>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      double u = A[pk(i, j)];
      static_for<0, j>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        u -= A[pk(i, k)] * w[k];
      });
      A[pk(i, j)] = u * inv;
    });
  });
  return ok;
}

// Gate statistics of one block: max|diag|, max|diag| over non-dominant rows, min|diag|,
// rows ridged, rows fallen back, rows non-dominant (R18 / R21)
struct GateStats {
  double v[6] = {0.0, 0.0, INFINITY, 0.0, 0.0, 0.0};
};

// The fit of one interior row from the exchanged lagged sums: Gram assembly,
// Cholesky + condition estimate + one ridge retry (R17), solve, band install (R14, R15),
// diagnostics and gate statistics.  ex: (2D+2) x TS sums of the tile's rows; t: this row's
// index in the tile; r: local row; gr: global row.
// LDL: the LDL^T form of the factorisation (ldl_packed) instead of Cholesky (chol_packed)
template <int D, bool LDL = false>
__device__ __forceinline__ void fit_row(const double* ex, int64_t TS, int t, int m, double Tsum, const double (&Dl)[2 * D + 1],
                                        int64_t r, int64_t n, int64_t gr, int64_t gN, MrepOut out, GateStats& g) {
  constexpr int P = 2 * D + 2;
  constexpr int NP = P * (P + 1) / 2;
  double A[NP];
  double lmax = 0.0, imax = 0.0, kap = INFINITY, lambda = 0.0;
  bool ok = false;
  int kind = PSP_ROW_INTERIOR;
#pragma unroll 1
  for (int attempt = 0; attempt < 2; ++attempt) {  // one code copy for the try and the retry
    assemble<D>(A, ex, TS, t, m, lambda);
    ok = LDL ? ldl_packed<P>(A, lmax, imax) : chol_packed<P>(A, lmax, imax);
    if (attempt == 0) {
      kap = ok ? (LDL ? lmax * imax : (lmax * imax) * (lmax * imax)) : INFINITY;
      if (ok && kap <= 1e12) break;
      // S:226 ridge retry on G + lambda I
      double tr = (double)m;
#pragma unroll
      for (int a = 0; a <= 2 * D; ++a) tr += ex[0 * TS + (t - D + a)];   // diag = C_0(r-d+a)
      lambda = (1e-10 / (double)P) * tr;
      kind = PSP_ROW_INTERIOR_RIDGE;
      g.v[3] += 1.0;
    }
  }
  double row[2 * D + 1];
  double icpt = 0.0;
  if (!ok) {                                      // identity row
    kind = PSP_ROW_FALLBACK_RANK;
    g.v[4] += 1.0;
#pragma unroll
    for (int o = 0; o <= 2 * D; ++o) row[o] = (o == D) ? 1.0 : 0.0;
  } else {
    double z[P];
    // Cholesky: (L L^T) x = b, each triangle scaled by 1/L_ii;  LDL: unit triangles, 1/D_ii once
    static_for<0, P>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      double sum = (i == 0) ? Tsum : Dl[i > 0 ? i - 1 : 0];
      static_for<0, i>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        sum -= A[pk(i, k)] * z[k];
      });
      z[i] = LDL ? sum : sum * A[pk(i, i)];
    });
    if (LDL) {
#pragma unroll
      for (int i = 0; i < P; ++i) z[i] *= A[pk(i, i)];
    }
    static_for<0, P>([&](auto ic) {
      constexpr int i = P - 1 - decltype(ic)::value;
      double sum = z[i];
      static_for<i + 1, P>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        sum -= A[pk(k, i)] * z[k];
      });
      z[i] = LDL ? sum : sum * A[pk(i, i)];
    });
    icpt = z[0];                                  // R15: reported, never installed
#pragma unroll
    for (int o = 0; o <= 2 * D; ++o) row[o] = z[1 + o];  // R14: N(i, i+o-d) = N*(o+2)
  }
#pragma unroll
  for (int o = 0; o <= 2 * D; ++o) out.bands[(int64_t)o * n + r] = row[o];
  if (out.intercept) out.intercept[r] = icpt;
  if (out.kind) out.kind[r] = (uint8_t)kind;
  if (out.kappa) out.kappa[r] = kap;
  const double ad = fabs(row[D]);
  g.v[0] = fmax(g.v[0], ad);
  g.v[2] = fmin(g.v[2], ad);
  if (!(ad > band_abs_off_sum<D>(row, gr, gN))) { g.v[5] += 1.0; g.v[1] = fmax(g.v[1], ad); }
}

// Merge a block's gate statistics into result[0..5]: max / min of non-negative doubles through
// their bit patterns (order-preserving), counts as exact integer adds -> order-independent.
__device__ void merge_stats(GateStats& g, double* red /* 8 warps x 6 */, double* result) {
  const int t = threadIdx.x, nw = blockDim.x / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    g.v[0] = fmax(g.v[0], __shfl_xor_sync(0xffffffffu, g.v[0], o));
    g.v[1] = fmax(g.v[1], __shfl_xor_sync(0xffffffffu, g.v[1], o));
    g.v[2] = fmin(g.v[2], __shfl_xor_sync(0xffffffffu, g.v[2], o));
    g.v[3] += __shfl_xor_sync(0xffffffffu, g.v[3], o);
    g.v[4] += __shfl_xor_sync(0xffffffffu, g.v[4], o);
    g.v[5] += __shfl_xor_sync(0xffffffffu, g.v[5], o);
  }
  if ((t & 31) == 0)
    for (int q = 0; q < 6; ++q) red[(t >> 5) * 6 + q] = g.v[q];
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < nw; ++w) {
      g.v[0] = fmax(g.v[0], red[w * 6 + 0]);
      g.v[1] = fmax(g.v[1], red[w * 6 + 1]);
      g.v[2] = fmin(g.v[2], red[w * 6 + 2]);
      g.v[3] += red[w * 6 + 3];
      g.v[4] += red[w * 6 + 4];
      g.v[5] += red[w * 6 + 5];
    }
    unsigned long long* ru = reinterpret_cast<unsigned long long*>(result);
    if (g.v[0] > 0.0) atomicMax(ru + 0, (unsigned long long)__double_as_longlong(g.v[0]));
    if (g.v[1] > 0.0) atomicMax(ru + 1, (unsigned long long)__double_as_longlong(g.v[1]));
    if (g.v[2] < INFINITY) atomicMin(ru + 2, (unsigned long long)__double_as_longlong(g.v[2]));
    if (g.v[3] != 0.0) atomicAdd(result + 3, g.v[3]);
    if (g.v[4] != 0.0) atomicAdd(result + 4, g.v[4]);
    if (g.v[5] != 0.0) atomicAdd(result + 5, g.v[5]);
  }
}

// Generic interior-row kernel (any row range, multi-rank halos): thread t accumulates the sums
// of row r = i0 - D + t of a 256-row tile that emits rows [i0, i0 + 256 - 2D).  It fits the rows
// of [a0, a1) and [b0, b1) (tiles start at a0 / b0; emission is clipped to the range) -- the
// rows the TMA kernel below does not take, or every row.
template <int D>
__global__ void __launch_bounds__(TPB, 1) mrep_interior_kernel(Cols cols, int m, int64_t n, int64_t a0, int64_t a1,
                                                               int64_t b0, int64_t b1, MrepOut out, MrepScratch sc) {
  constexpr int TILE = TPB + 3 * D;                 // rows [i0-2D, i0-D+TPB+2D)
  constexpr int64_t E = TPB - 2 * D;
  __shared__ double xs[CB][TILE];
  __shared__ double ex[(2 * D + 2) * TPB];
  __shared__ double red[TPB / 32 * 6];
  const int t = threadIdx.x;
  GateStats gs;
  const int64_t na = a1 > a0 ? (a1 - a0 + E - 1) / E : 0;
  const int64_t nbt = b1 > b0 ? (b1 - b0 + E - 1) / E : 0;
  for (int64_t q = blockIdx.x; q < na + nbt; q += gridDim.x) {
  const int64_t i0 = q < na ? a0 + q * E : b0 + (q - na) * E;
  const int64_t rend = q < na ? a1 : b1;            // emission stops at the range end
  const int64_t r = i0 - D + t;                     // the row this thread accumulates for
  const int64_t tile0 = i0 - 2 * D;

  double Cl[2 * D + 1], Dl[2 * D + 1], Ssum = 0.0, Tsum = 0.0;
#pragma unroll
  for (int l = 0; l <= 2 * D; ++l) { Cl[l] = 0.0; Dl[l] = 0.0; }

  const bool rvalid = (r >= 0 && r < n);
  for (int c0 = 0; c0 < m; c0 += CB) {
    const int cn = (m - c0) < CB ? (m - c0) : CB;
    double yv[CB];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc)                 // this row's P_y samples of the chunk
      yv[cc] = (cc < cn && rvalid) ? cols.sc(c0 + cc) * __ldg(cols.py + (int64_t)cols.slot[c0 + cc] * cols.ld + r) : 0.0;
    __syncthreads();
    for (int cc = 0; cc < cn; ++cc) {
      const double scx = cols.sc(c0 + cc);
      for (int qq = t; qq < TILE; qq += TPB) xs[cc][qq] = scx * cols.xraw(c0 + cc, tile0 + qq, n);
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
      if (cc >= cn) break;
      const double* xr = &xs[cc][t + D];            // xr[l] = P_x(r + l), l in [-D, 2D]
      const double x0 = xr[0];
      Ssum += x0;
      Tsum += yv[cc];
#pragma unroll
      for (int l = 0; l <= 2 * D; ++l) Cl[l] = fma(x0, xr[l], Cl[l]);
#pragma unroll
      for (int l = 0; l <= 2 * D; ++l) Dl[l] = fma(xr[l - D], yv[cc], Dl[l]);
    }
  }
  // exchange C_l(r), S(r) with the neighbours ((2D+2) x TPB doubles)
  __syncthreads();
#pragma unroll
  for (int l = 0; l <= 2 * D; ++l) ex[l * TPB + t] = Cl[l];
  ex[(2 * D + 1) * TPB + t] = Ssum;
  __syncthreads();

  const int64_t gr = cols.grow0 + r;                 // global row (multi-rank slabs)
  const bool emit = (t >= D && t < TPB - D) && r >= 0 && r < n && r < rend && gr >= D && gr < cols.gN - D;
  if (emit) fit_row<D>(ex, TPB, t, m, Tsum, Dl, r, n, gr, cols.gN, out, gs);
  }  // tiles
  merge_stats(gs, red, sc.result);
}

// ------------------------------------------------------------------------------------------
// TMA-pipelined interior kernel (the bulk of the rows).  Same tiles and per-row arithmetic as
// the generic kernel (thread t accumulates sum row s0 + t, s0 = i0 - D, of the 256-row tile that
// emits [i0, i0 + 256 - 2D)), but the probe columns are staged by one thread with
// cp.async.bulk (1-D TMA bulk copies) into an NST-deep ring of shared-memory stages of CB
// columns each -- P_x rows [s0 - D, s0 + 256 + 2D) and P_y rows [s0, s0 + 256), widened to
// 16-byte boundaries -- with completion on one mbarrier per stage.  HBM reads run ahead of the
// FMAs and of the per-row Cholesky phase without holding registers, and a warp's shared-memory
// reads are 32 consecutive doubles (conflict-free).  All columns must share the 16-byte
// alignment parity (sx, sy; checked on the host, else the generic kernel runs everything).
// ------------------------------------------------------------------------------------------
constexpr int TT = 128;        // threads (= sum rows) per tile of the TMA kernel
#ifndef PSP_MREP_CHUNKS
#define PSP_MREP_CHUNKS 16    // row chunks of the split MREP (fits overlap the next chunk's sums)
#endif
#ifndef PSP_MREP_SUMS_LB
#define PSP_MREP_SUMS_LB 4    // launch bound (blocks per SM) of the streaming kernel: its register cap
#endif
#ifndef PSP_MREP_SUMS_BPS
#define PSP_MREP_SUMS_BPS 3   // streaming blocks per SM of a chunked split MREP (a fit block beside)
#endif
#ifndef PSP_MREP_LASTFULL
#define PSP_MREP_LASTFULL 1  // the last chunk's fit kernel on the full grid
#endif
#ifndef PSP_MREP_FIT_MINB
#define PSP_MREP_FIT_MINB 2   // resident blocks per SM of the split MREP's fit kernel
#endif
#ifndef PSP_MREP_TCB
#define PSP_MREP_TCB 8    // probe columns per stage (measured: 8 x 3 stages beats 4 x 4 at d = 3)
#endif
constexpr int TCB = PSP_MREP_TCB;   // probe columns per stage
constexpr int TNST = PSP_MREP_NST;   // stages

template <int D>
struct TmaCfg {
  static constexpr int PXW = ((TT + 3 * D + 2) + 1) / 2 * 2;    // P_x stage row (doubles)
  static constexpr int PYW = TT + 2;                             // P_y stage row
  static constexpr int STAGE = TCB * (PXW + PYW);                // doubles per stage
  static constexpr size_t SMEM = (size_t)TNST * STAGE * 8 + (size_t)(2 * D + 2) * TT * 8 + 16 * TNST;
  static constexpr size_t SMEM_SUMS = (size_t)TNST * STAGE * 8 + 16 * TNST;   // no exchange buffer
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct TmaCols {
  const double* px;
  const double* py;
  int64_t ld;
  int sx, sy;                  // row shift of the P_x / P_y segments in a stage (0 / 1)
  int32_t slot[kMaxM];
};

// SUMS = true: the streaming half only -- every sum row of the tile (the D halo rows on each
// side included; overlapping tiles write identical values) goes to sc.sums, and
// mrep_fitsum_kernel fits the rows afterwards at its own occupancy.
template <int D, bool SUMS>
__global__ void __launch_bounds__(TT, SUMS ? PSP_MREP_SUMS_LB : PSP_MREP_MINB) mrep_tma_kernel(TmaCols cols, const double* __restrict__ scale,
                                                                      int m, int64_t n, int64_t gN, int64_t grow0,
                                                                      int64_t R0, int64_t ntile, MrepOut out,
                                                                      MrepScratch sc) {
  using Cfg = TmaCfg<D>;
  constexpr int E = TT - 2 * D;                    // rows emitted per tile
  constexpr int LX = ((TT + 3 * D) + 1) & ~1;      // P_x segment length (shift 0) ...
  constexpr int LX1 = ((TT + 3 * D + 1) + 1) & ~1; //   ... and with shift 1
  constexpr int LY = TT, LY1 = TT + 2;
  extern __shared__ __align__(16) double sm[];
  double* stages = sm;                             // [TNST][TCB x PXW | TCB x PYW]
  double* ex = sm + TNST * Cfg::STAGE;             // [(2D+2)][TT]: C_l, S of the tile's rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(ex + (SUMS ? 0 : (2 * D + 2) * TT));
  __shared__ double scs[kMaxM];                    // per-column probe scale
  __shared__ double red[TT / 32 * 6];
  __shared__ int s_unit;
  const int t = threadIdx.x;
  if (t == 0) s_unit = 1;
  __syncthreads();
  for (int c = t; c < m; c += TT) {
    scs[c] = scale ? scale[cols.slot[c]] : 1.0;
    if (scs[c] != 1.0) s_unit = 0;
  }
  if (t == 0) {
    for (int q = 0; q < TNST; ++q) mbar_init(bars + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool unit = s_unit != 0;                   // every recorded probe scale is 1

  const int lx = cols.sx ? LX1 : LX, ly = cols.sy ? LY1 : LY;
  const int nch = (m + TCB - 1) / TCB;             // the last chunk may be partial
  // 32-bit load counters with incremental (tile, chunk, stage) indices: a 64-bit division in
  // the loop is an out-of-line call whose ABI would push the packed Gram to local memory
  const int my_tiles = (int)((ntile - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int total = my_tiles * nch;
  int is_tq = 0, is_ch = 0, is_stg = 0;            // the next load to issue (thread 0)
  auto issue_next = [&]() {                        // thread 0: stage the columns of the next load
    const int64_t tile = blockIdx.x + (int64_t)is_tq * gridDim.x;
    double* st = stages + (size_t)is_stg * Cfg::STAGE;
    const int64_t s0 = R0 + tile * E - D;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int ncols = (m - is_ch * TCB) < TCB ? (m - is_ch * TCB) : TCB;
    mbar_expect_tx(bars + is_stg, 8u * (unsigned)(ncols * (lx + ly)));
#pragma unroll
    for (int cc = 0; cc < TCB; ++cc) {
      const int c = is_ch * TCB + cc;
      if (c >= m) break;
      const double* bxp = cols.px + (int64_t)cols.slot[c] * cols.ld;
      const double* byp = cols.py + (int64_t)cols.slot[c] * cols.ld;
      bulk_g2s(st + cc * Cfg::PXW, bxp + (s0 - D - cols.sx), 8u * lx, bars + is_stg);
      bulk_g2s(st + TCB * Cfg::PXW + cc * Cfg::PYW, byp + (s0 - cols.sy), 8u * ly, bars + is_stg);
    }
    if (++is_ch == nch) { is_ch = 0; ++is_tq; }
    if (++is_stg == TNST) is_stg = 0;
  };
  if (t == 0)
    for (int q = 0; q < total && q < TNST; ++q) issue_next();

  GateStats gs;
  double Cl[2 * D + 1], Dl[2 * D + 1], Ssum = 0.0, Tsum = 0.0;
  const int xo = cols.sx + t, yo = cols.sy + t;    // this row's offsets in a stage row
  int stg = 0, ch = 0, tq = 0;
  unsigned phase = 0;                              // parity bit per stage
  for (int q = 0; q < total; ++q) {
    if (ch == 0) {
#pragma unroll
      for (int l = 0; l <= 2 * D; ++l) { Cl[l] = 0.0; Dl[l] = 0.0; }
      Ssum = Tsum = 0.0;
    }
    mbar_wait(bars + stg, (phase >> stg) & 1u);
    phase ^= 1u << stg;
    const double* st = stages + (size_t)stg * Cfg::STAGE;
    const int ccn = (m - ch * TCB) < TCB ? (m - ch * TCB) : TCB;   // columns in this chunk
    if (unit) {
#pragma unroll
      for (int cc = 0; cc < TCB; ++cc) {
        if (cc >= ccn) break;                      // uniform
        const double* xr = st + cc * Cfg::PXW + xo;  // xr[k] = P_x(r - D + k), r = s0 + t
        double xw[3 * D + 1];
#pragma unroll
        for (int k = 0; k < 3 * D + 1; ++k) xw[k] = xr[k];
        const double yv = st[TCB * Cfg::PXW + cc * Cfg::PYW + yo];
        const double x0 = xw[D];
        Ssum += x0;
        Tsum += yv;
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) Cl[l] = fma(x0, xw[D + l], Cl[l]);
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) Dl[l] = fma(xw[l], yv, Dl[l]);
      }
    } else {
      // scaled probes (s x, s y): the scale enters the products once, as s^2 on one factor
      // (2 multiplies a column instead of 3d+2; equal to the scaled sums up to rounding)
      const int c0 = ch * TCB;
#pragma unroll
      for (int cc = 0; cc < TCB; ++cc) {
        if (cc >= ccn) break;                      // uniform
        const double sc = scs[c0 + cc], s2 = sc * sc;   // (no s^2 table: its 2 KB of shared memory
        const double* xr = st + cc * Cfg::PXW + xo;      //  cost a resident block per SM)
        double xw[3 * D + 1];
#pragma unroll
        for (int k = 0; k < 3 * D + 1; ++k) xw[k] = xr[k];
        const double yr = st[TCB * Cfg::PXW + cc * Cfg::PYW + yo];
        const double x0 = xw[D];
        Ssum = fma(sc, x0, Ssum);
        Tsum = fma(sc, yr, Tsum);
        const double ax = s2 * x0, by = s2 * yr;
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) Cl[l] = fma(ax, xw[D + l], Cl[l]);
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) Dl[l] = fma(xw[l], by, Dl[l]);
      }
    }
    __syncthreads();                               // every thread is done with stage stg
    if (t == 0 && q + TNST < total) issue_next();
    if (++stg == TNST) stg = 0;
    if (SUMS && ch == nch - 1) {
      const int64_t tile = blockIdx.x + (int64_t)tq * gridDim.x;
      const int64_t r = R0 + tile * E - D + t;
      const int64_t ns = sc.sums_n;
      if (r >= 0 && r < n) {
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) sc.sums[(int64_t)l * ns + r] = Cl[l];
        sc.sums[(int64_t)(2 * D + 1) * ns + r] = Ssum;
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) sc.sums[(int64_t)(2 * D + 2 + l) * ns + r] = Dl[l];
        sc.sums[(int64_t)(4 * D + 3) * ns + r] = Tsum;
      }
      ch = 0;
      ++tq;
    } else if (!SUMS && ch == nch - 1) {
      // exchange C_l, S of the tile's TT sum rows, then fit the emitted rows
#pragma unroll
      for (int l = 0; l <= 2 * D; ++l) ex[l * TT + t] = Cl[l];
      ex[(2 * D + 1) * TT + t] = Ssum;
      __syncthreads();
      const int64_t tile = blockIdx.x + (int64_t)tq * gridDim.x;
      const int64_t r = R0 + tile * E - D + t;
      if (t >= D && t < TT - D) fit_row<D>(ex, TT, t, m, Tsum, Dl, r, n, grow0 + r, gN, out, gs);
      __syncthreads();                             // ex is rewritten by the next tile
      ch = 0;
      ++tq;
    } else {
      ++ch;
    }
  }
  if (!SUMS) merge_stats(gs, red, sc.result);
}

// ------------------------------------------------------------------------------------------
// Warp-specialised MREP (d >= 2): the streaming and the fitting run in the same persistent CTA on
// different warps.  Warps 0-3 (the sum group, thread t = sum row t of a 128-row tile) consume
// the TMA stage ring exactly as mrep_tma_kernel and, at the end of a tile, hand its 4d+4 lagged
// sums per row to a double-buffered shared-memory exchange (mbarriers ex_full / ex_empty) and go
// straight on with the next tile's columns; warps 4-7 (the fit group, thread f = emitted row
// f + d) assemble each row's Gram from the exchange and solve it (fit_row: Cholesky, R17 ridge
// retry, R14 install) while the next tile streams.  The lagged sums never leave the SM: HBM sees
// only the probes and the bands (568 B a row at m = 32, d = 3).  One CTA per SM (the fit's
// register budget sets the occupancy).  MEASURED AND NOT THE DEFAULT (PSP_MREP_WS=1 selects
// it): with one warp per scheduler the sum group cannot hide the FP64 / shared-memory latency of
// the lagged sums, so the stream stalls (n = 2^27, m = 32, d = 3: 45.4 ms against the split
// path's 26.7 ms; d = 2 at 2^26: 20.6 against 8.8 ms; r02d).  Giving the sum group more warps
// needs a register split between the groups (setmaxnreg) that the fit's ~220 registers a
// thread leave no room for.
// ------------------------------------------------------------------------------------------
#ifndef PSP_MREP_WS_NST
#define PSP_MREP_WS_NST 6     // TMA stages of the warp-specialised kernel (more bytes in flight)
#endif
constexpr int WNST = PSP_MREP_WS_NST;

template <int D>
struct WsCfg {
  static constexpr int STAGE = TmaCfg<D>::STAGE;
  static constexpr int EXR = 4 * D + 4;                                  // exchange rows (sums)
  static constexpr size_t SMEM = (size_t)WNST * STAGE * 8 + (size_t)2 * EXR * TT * 8 + 16 * WNST + 64;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int D>
__global__ void __launch_bounds__(2 * TT, 1) mrep_ws_kernel(TmaCols cols, const double* __restrict__ scale, int m,
                                                           int64_t n, int64_t gN, int64_t grow0, int64_t R0,
                                                           int64_t ntile, MrepOut out, MrepScratch sc) {
  using Cfg = WsCfg<D>;
  constexpr int E = TT - 2 * D;                    // rows emitted per tile
  constexpr int LX = ((TT + 3 * D) + 1) & ~1;
  constexpr int LX1 = ((TT + 3 * D + 1) + 1) & ~1;
  constexpr int LY = TT, LY1 = TT + 2;
  constexpr int EXR = Cfg::EXR;
  extern __shared__ __align__(16) double sm[];
  double* stages = sm;                             // [WNST][TCB x PXW | TCB x PYW]
  double* exb = sm + WNST * TmaCfg<D>::STAGE;      // [2][EXR][TT]: C_0..C_2D, S, D_0..D_2D, T
  uint64_t* bars = reinterpret_cast<uint64_t*>(exb + 2 * EXR * TT);
  uint64_t* ex_full = bars + WNST;
  uint64_t* ex_empty = ex_full + 2;
  __shared__ double scs[kMaxM];
  __shared__ double scs2[kMaxM];
  __shared__ double red[2 * TT / 32 * 6];
  __shared__ int s_unit;
  const int t = threadIdx.x;
  const bool sums = t < TT;
  if (t == 0) s_unit = 1;
  __syncthreads();
  for (int c = t; c < m; c += 2 * TT) {
    scs[c] = scale ? scale[cols.slot[c]] : 1.0;
    scs2[c] = scs[c] * scs[c];
    if (scs[c] != 1.0) s_unit = 0;
  }
  if (t == 0) {
    for (int q = 0; q < WNST; ++q) mbar_init(bars + q, 1);
    for (int q = 0; q < 2; ++q) {
      mbar_init(ex_full + q, TT);
      mbar_init(ex_empty + q, TT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool unit = s_unit != 0;
  const int nch = (m + TCB - 1) / TCB;
  const int my_tiles = (int)((ntile - blockIdx.x + gridDim.x - 1) / gridDim.x);
  GateStats gs;
  if (sums) {
    // ---- the sum group: TMA issue (thread 0) + lagged sums, as mrep_tma_kernel ----
    const int lx = cols.sx ? LX1 : LX, ly = cols.sy ? LY1 : LY;
    const int total = my_tiles * nch;
    int is_tq = 0, is_ch = 0, is_stg = 0;
    auto issue_next = [&]() {
      const int64_t tile = blockIdx.x + (int64_t)is_tq * gridDim.x;
      double* st = stages + (size_t)is_stg * TmaCfg<D>::STAGE;
      const int64_t s0 = R0 + tile * E - D;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int ncols = (m - is_ch * TCB) < TCB ? (m - is_ch * TCB) : TCB;
      mbar_expect_tx(bars + is_stg, 8u * (unsigned)(ncols * (lx + ly)));
#pragma unroll
      for (int cc = 0; cc < TCB; ++cc) {
        const int c = is_ch * TCB + cc;
        if (c >= m) break;
        const double* bxp = cols.px + (int64_t)cols.slot[c] * cols.ld;
        const double* byp = cols.py + (int64_t)cols.slot[c] * cols.ld;
        bulk_g2s(st + cc * TmaCfg<D>::PXW, bxp + (s0 - D - cols.sx), 8u * lx, bars + is_stg);
        bulk_g2s(st + TCB * TmaCfg<D>::PXW + cc * TmaCfg<D>::PYW, byp + (s0 - cols.sy), 8u * ly, bars + is_stg);
      }
      if (++is_ch == nch) { is_ch = 0; ++is_tq; }
      if (++is_stg == WNST) is_stg = 0;
    };
    if (t == 0)
      for (int q = 0; q < total && q < WNST; ++q) issue_next();
    double Cl[2 * D + 1], Dl[2 * D + 1], Ssum = 0.0, Tsum = 0.0;
    const int xo = cols.sx + t, yo = cols.sy + t;
    int stg = 0, ch = 0, tq = 0;
    unsigned phase = 0;
    for (int q = 0; q < total; ++q) {
      if (ch == 0) {
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) { Cl[l] = 0.0; Dl[l] = 0.0; }
        Ssum = Tsum = 0.0;
      }
      mbar_wait(bars + stg, (phase >> stg) & 1u);
      phase ^= 1u << stg;
      const double* st = stages + (size_t)stg * TmaCfg<D>::STAGE;
      const int ccn = (m - ch * TCB) < TCB ? (m - ch * TCB) : TCB;
      const int c0 = ch * TCB;
#pragma unroll
      for (int cc = 0; cc < TCB; ++cc) {
        if (cc >= ccn) break;
        const double* xr = st + cc * TmaCfg<D>::PXW + xo;
        double xw[3 * D + 1];
#pragma unroll
        for (int k = 0; k < 3 * D + 1; ++k) xw[k] = xr[k];
        const double yr = st[TCB * TmaCfg<D>::PXW + cc * TmaCfg<D>::PYW + yo];
        const double x0 = xw[D];
        if (unit) {
          Ssum += x0;
          Tsum += yr;
#pragma unroll
          for (int l = 0; l <= 2 * D; ++l) Cl[l] = fma(x0, xw[D + l], Cl[l]);
#pragma unroll
          for (int l = 0; l <= 2 * D; ++l) Dl[l] = fma(xw[l], yr, Dl[l]);
        } else {
          const double scv = scs[c0 + cc], s2 = scs2[c0 + cc];
          Ssum = fma(scv, x0, Ssum);
          Tsum = fma(scv, yr, Tsum);
          const double ax = s2 * x0, by = s2 * yr;
#pragma unroll
          for (int l = 0; l <= 2 * D; ++l) Cl[l] = fma(ax, xw[D + l], Cl[l]);
#pragma unroll
          for (int l = 0; l <= 2 * D; ++l) Dl[l] = fma(xw[l], by, Dl[l]);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TT) : "memory");   // the sum group is done with stage stg
      if (t == 0 && q + WNST < total) issue_next();
      if (++stg == WNST) stg = 0;
      if (ch == nch - 1) {
        // hand the tile's sums to the fit group (buffer tq & 1, its (tq >> 1)-th use)
        const int b = tq & 1;
        mbar_wait(ex_empty + b, ((tq >> 1) & 1u) ^ 1u);
        double* ex = exb + (size_t)b * EXR * TT;
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) ex[l * TT + t] = Cl[l];
        ex[(2 * D + 1) * TT + t] = Ssum;
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) ex[(2 * D + 2 + l) * TT + t] = Dl[l];
        ex[(4 * D + 3) * TT + t] = Tsum;
        mbar_arrive(ex_full + b);
        ch = 0;
        ++tq;
      } else {
        ++ch;
      }
    }
  } else {
    // ---- the fit group: one thread per emitted row of the tile handed over ----
    const int f = t - TT;
    for (int tq = 0; tq < my_tiles; ++tq) {
      const int b = tq & 1;
      mbar_wait(ex_full + b, (tq >> 1) & 1u);
      const double* ex = exb + (size_t)b * EXR * TT;
      const int64_t tile = blockIdx.x + (int64_t)tq * gridDim.x;
      const int tr = f + D;                        // this thread's row in the tile
      if (f < E) {
        const int64_t r = R0 + tile * E - D + tr;
        double Dl[2 * D + 1];
#pragma unroll
        for (int l = 0; l <= 2 * D; ++l) Dl[l] = ex[(2 * D + 2 + l) * TT + tr];
        const double Tsum = ex[(4 * D + 3) * TT + tr];
        fit_row<D>(ex, TT, tr, m, Tsum, Dl, r, n, grow0 + r, gN, out, gs);
      }
      mbar_arrive(ex_empty + b);
    }
  }
  merge_stats(gs, red, sc.result);
}

// The fitting half of the split MREP: one thread per row r in [r0, r1), its Gram from the
// lagged sums of rows r-D..r+D in sc.sums (rows of neighbouring tiles: L2 / L1 hits).
template <int D, bool LDL = false>
__global__ void __launch_bounds__(TT, PSP_MREP_FIT_MINB) mrep_fitsum_kernel(int m, int64_t n, int64_t gN, int64_t grow0,
                                                                         int64_t r0, int64_t r1, MrepOut out,
                                                                         MrepScratch sc) {
  __shared__ double red[TT / 32 * 6];
  GateStats gs;
  const int64_t ns = sc.sums_n;
  for (int64_t r = r0 + (int64_t)blockIdx.x * TT + threadIdx.x; r < r1; r += (int64_t)gridDim.x * TT) {
    double Dl[2 * D + 1];
#pragma unroll
    for (int l = 0; l <= 2 * D; ++l) Dl[l] = sc.sums[(int64_t)(2 * D + 2 + l) * ns + r];
    const double Tsum = sc.sums[(int64_t)(4 * D + 3) * ns + r];
    fit_row<D, LDL>(sc.sums + (r - D), ns, D, m, Tsum, Dl, r, n, grow0 + r, gN, out, gs);
  }
  merge_stats(gs, red, sc.result);
}

template <int D>
void launch_tma(const TmaCols& tc, const double* scale, int m, int64_t n, int64_t gN, int64_t grow0, int64_t R0,
                int64_t ntile, MrepOut out, MrepScratch sc, int nb, cudaStream_t s) {
  const size_t smem = TmaCfg<D>::SMEM;
  const int dev = device_ordinal();
  thread_local bool attr[kMaxDev] = {};
  if (!attr[dev]) {
    cudaFuncSetAttribute(mrep_tma_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(mrep_tma_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TmaCfg<D>::SMEM_SUMS);
    attr[dev] = true;
  }
  const int sms = device_sms();
  const int64_t E = TT - 2 * D;
  if (D >= 2 && getenv("PSP_MREP_WS")) {
    // the warp-specialised fused kernel (measured and not the default: at one CTA a SM the four
    // sum warps cannot hide the FP64 latency of the lagged sums -- n = 2^27, m = 32, d = 3:
    // 45.4 ms against the split path's 26.7 ms, r02d)
    thread_local bool wattr[kMaxDev] = {};
    if (!wattr[dev]) {
      cudaFuncSetAttribute(mrep_ws_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WsCfg<D>::SMEM);
      wattr[dev] = true;
    }
    const int64_t g = ntile < sms ? ntile : sms;
    mrep_ws_kernel<D><<<(unsigned)g, 2 * TT, WsCfg<D>::SMEM, s>>>(tc, scale, m, n, gN, grow0, R0, ntile, out, sc);
    return;
  }
  if (sc.sums != nullptr && sc.sums_n >= n && D >= 2) {
    // split: stream + lagged sums, then the fits.  d <= 3: the rows go in PSP_MREP_CHUNKS
    // chunks and the fits of chunk c run on a second stream beside the sums of chunk c+1 (the
    // streaming kernel at 3 blocks per SM, so one fit block per SM fits beside it); d = 4 (the
    // fit spills at that occupancy): one chunk, the streaming kernel at full occupancy.
    // Measured n = 2^26, m = 32: d = 2 9.8 -> 8.9 ms, d = 3 11.3 -> 10.7 ms by the overlap.
    constexpr int K = D <= 3 ? PSP_MREP_CHUNKS : 1;
    // the fit side stream and its events: per host thread and device
    thread_local cudaStream_t s2s[kMaxDev] = {};
    thread_local cudaEvent_t evs[kMaxDev][K + 1];
    thread_local int occs[kMaxDev] = {};
    cudaStream_t& s2 = s2s[dev];
    cudaEvent_t* ev = evs[dev];
    if (s2 == nullptr) {
      cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
      for (int q = 0; q <= K; ++q) cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming);
    }
    int& occ = occs[dev];
    if (!occ) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mrep_tma_kernel<D, true>, TT, TmaCfg<D>::SMEM_SUMS);
      if (occ < 1) occ = 1;
    }
    const int64_t g1max = sms * (int64_t)(K > 1 && occ > PSP_MREP_SUMS_BPS ? PSP_MREP_SUMS_BPS : occ);
    const int64_t per = (ntile + K - 1) / K;
    for (int c = 0; c < K; ++c) {
      const int64_t t0 = c * per, t1 = (t0 + per < ntile) ? t0 + per : ntile;
      if (t1 <= t0) break;
      const int64_t R0c = R0 + t0 * E;
      const int g1 = (int)((t1 - t0) < g1max ? (t1 - t0) : g1max);
      mrep_tma_kernel<D, true><<<g1, TT, TmaCfg<D>::SMEM_SUMS, s>>>(tc, scale, m, n, gN, grow0, R0c, t1 - t0, out,
                                                                   sc);
      cudaEventRecord(ev[c], s);
      cudaStreamWaitEvent(s2, ev[c], 0);
      const int64_t rows = (t1 - t0) * E;
      // beside the sums: one block per SM; the last chunk's fits run alone (no sums beside them):
      // every resident block
      const bool last = (c == K - 1) || (t1 >= ntile);
      const int64_t g2max = (K > 1 && !(PSP_MREP_LASTFULL && last)) ? sms : sms * PSP_MREP_FIT_MINB;
      const int64_t g2 = (rows + TT - 1) / TT < g2max ? (rows + TT - 1) / TT : g2max;
      static const bool ldl = getenv("PSP_MREP_LDL") != nullptr;   // A/B knob (the LDL^T fit)
      if (ldl) mrep_fitsum_kernel<D, true><<<(int)g2, TT, 0, s2>>>(m, n, gN, grow0, R0c, R0c + rows, out, sc);
      else mrep_fitsum_kernel<D><<<(int)g2, TT, 0, s2>>>(m, n, gN, grow0, R0c, R0c + rows, out, sc);
    }
    cudaEventRecord(ev[K], s2);
    cudaStreamWaitEvent(s, ev[K], 0);
  } else {
    // one full wave at the kernel's occupancy (a partial second wave of a persistent grid leaves
    // SMs idle for a third of the launch)
    thread_local int occn[kMaxDev] = {};
    if (!occn[dev]) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occn[dev], mrep_tma_kernel<D, false>, TT, smem);
      if (occn[dev] < 1) occn[dev] = 1;
    }
    const int64_t g = (int64_t)occn[dev] * sms < ntile ? (int64_t)occn[dev] * sms : ntile;
    (void)nb;
    mrep_tma_kernel<D, false><<<(unsigned)g, TT, smem, s>>>(tc, scale, m, n, gN, grow0, R0, ntile, out, sc);
  }
}

// Boundary rows, R16 two-pass centred OLS, one thread per row.
__global__ void mrep_boundary_kernel(Cols cols, int m, int64_t n, int d, MrepOut out,
                                     MrepScratch sc) {
  __shared__ double st[64][6];
  const int t = threadIdx.x;
  double v[6] = {0.0, 0.0, INFINITY, 0.0, 0.0, 0.0};
  // global boundary rows g < d and g >= gN - d that this rank owns (local i = g - grow0)
  const int64_t g = (t < d) ? t : (cols.gN - 2 * d + t);
  const int64_t i = g - cols.grow0;
  if (t < 2 * d && i >= 0 && i < n) {
    double mx = 0.0, my = 0.0;
    for (int c = 0; c < m; ++c) {
      mx += cols.sc(c) * cols.px[(int64_t)cols.slot[c] * cols.ld + i];
      my += cols.sc(c) * cols.py[(int64_t)cols.slot[c] * cols.ld + i];
    }
    mx /= (double)m;
    my /= (double)m;
    double sxx = 0.0, sxy = 0.0;
    for (int c = 0; c < m; ++c) {
      const double dx = cols.sc(c) * cols.px[(int64_t)cols.slot[c] * cols.ld + i] - mx;
      const double dy = cols.sc(c) * cols.py[(int64_t)cols.slot[c] * cols.ld + i] - my;
      sxx += dx * dx;
      sxy += dx * dy;
    }
    double b1, b0;
    int kind;
    if (sxx < 1e-300) { b1 = 1.0; b0 = 0.0; kind = PSP_ROW_FALLBACK_ZEROVAR; v[4] = 1.0; }
    else { b1 = sxy / sxx; b0 = my - b1 * mx; kind = PSP_ROW_BOUNDARY; }
    for (int o = 0; o <= 2 * d; ++o) out.bands[(int64_t)o * n + i] = (o == d) ? b1 : 0.0;
    if (out.intercept) out.intercept[i] = b0;
    if (out.kind) out.kind[i] = (uint8_t)kind;
    if (out.kappa) out.kappa[i] = 0.0;
    v[0] = fabs(b1);
    v[2] = fabs(b1);
    // a diagonal-only row is dominant iff its diagonal is nonzero
    if (!(fabs(b1) > 0.0)) { v[1] = fabs(b1); v[5] = 1.0; }
  }
  for (int q = 0; q < 6; ++q) st[t][q] = v[q];
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < 64; ++w) {
      v[0] = fmax(v[0], st[w][0]);
      v[1] = fmax(v[1], st[w][1]);
      v[2] = fmin(v[2], st[w][2]);
      v[3] += st[w][3];
      v[4] += st[w][4];
      v[5] += st[w][5];
    }
    for (int q = 0; q < 6; ++q) sc.result[q] = v[q];
  }
}

// R18: rows with |N(i,i)| < 1e-12 max_j |N(j,j)| become identity rows.  Runs only
// when the fit kernel found such a row (result[6]); counts them into result[4].
__global__ void mrep_patch_kernel(int64_t n, int d, MrepOut out, MrepScratch sc) {
  if (sc.result[6] == 0.0) return;
  const double thr = 1e-12 * sc.result[0];
  double cnt = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (fabs(out.bands[(int64_t)d * n + i]) < thr) {
      for (int o = 0; o <= 2 * d; ++o) out.bands[(int64_t)o * n + i] = (o == d) ? 1.0 : 0.0;
      if (out.kind) out.kind[i] = PSP_ROW_FALLBACK_SMALLDIAG;
      cnt += 1.0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt != 0.0) atomicAdd(sc.result + 8, cnt);  // exact integers
}

__global__ void mrep_pack_kernel(Cols cols, int m, int64_t n, int d, double* send) {
  // send[0 .. m*d): rows 0..d-1 (for rank-1), send[m*d ..): rows n-d..n-1 (for rank+1), raw
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * m * d; q += gridDim.x * blockDim.x) {
    const int side = q / (m * d), c = (q / d) % m, k = q % d;
    const int64_t rr = side == 0 ? k : n - d + k;
    send[q] = __ldg(cols.px + (int64_t)cols.slot[c] * cols.ld + rr);
  }
}

// multi-rank: R18 / R21 decisions from the all-reduced statistics
__global__ void mrep_decide_kernel(MrepScratch sc) {
  const double* a = sc.result;
  const double thr = 1e-12 * a[0];
  sc.result[6] = (a[2] < thr) ? 1.0 : 0.0;
  sc.result[7] = (a[5] == 0.0 || a[1] < thr) ? 1.0 : 0.0;
}

// R21 on a given N (psp_set_bands): rows that are not strictly diagonally dominant, summed in band
// order as the fit kernels do, counted into *count (exact integer adds: order-free)
__global__ void gate_count_kernel(const double* __restrict__ bands, int64_t n, int d, int64_t grow0, int64_t gN,
                                  double* count, int spd) {
  double cnt = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double off = 0.0;
    for (int o = 0; o <= 2 * d; ++o) {
      const int64_t j = grow0 + i + o - d;
      if (o == d || j < 0 || j >= gN) continue;
      off += fabs(bands[(int64_t)o * n + i]);
    }
    const double dg = bands[(int64_t)d * n + i];
    if (!(fabs(dg) > off) || (spd && !(dg > 0.0))) cnt += 1.0;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt != 0.0) atomicAdd(count, cnt);
}

}  // namespace

// ------------------------------------------------------------------------------------------
// f3: streaming MREP (the probe data are "obtained progressively").  Each recorded probe
// (x, y) (scale sc: the probe is sc * column) adds its terms to every row's lagged sums, in the
// recording order (oldest -> newest, as the ring's column order):
//   C_l(r) += x_r x_{r+l} (l = 0..2d),  S(r) += x_r,  D_l(i) += x_{i-d+l} y_i (l = 0..2d),  T(i) += y_i
// (x = 0 outside the matrix), the layout mrep_fitsum_kernel reads.  Bytes per row and probe:
// x, y read, 4d+4 sums read and written = 16 + 16(4d+4).
// ------------------------------------------------------------------------------------------
namespace {
template <int D>
__global__ void __launch_bounds__(256) mrep_accumulate_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                              const double* scale, int slot, int64_t n,
                                                              double* __restrict__ sums, int64_t ns, int first) {
  const double sc = scale ? __ldg(scale + slot) : 1.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double xw[3 * D + 1];                                      // x_{r-D .. r+2D}
#pragma unroll
    for (int q = 0; q < 3 * D + 1; ++q) {
      const int64_t rr = r - D + q;
      xw[q] = (rr >= 0 && rr < n) ? sc * __ldg(x + rr) : 0.0;
    }
    const double yv = sc * __ldg(y + r), x0 = xw[D];
#pragma unroll
    for (int l = 0; l <= 2 * D; ++l) {
      double* p = sums + (int64_t)l * ns + r;
      *p = first ? x0 * xw[D + l] : fma(x0, xw[D + l], *p);
    }
    double* ps = sums + (int64_t)(2 * D + 1) * ns + r;
    *ps = first ? x0 : *ps + x0;
#pragma unroll
    for (int l = 0; l <= 2 * D; ++l) {
      double* p = sums + (int64_t)(2 * D + 2 + l) * ns + r;
      *p = first ? xw[l] * yv : fma(xw[l], yv, *p);
    }
    double* pt = sums + (int64_t)(4 * D + 3) * ns + r;
    *pt = first ? yv : *pt + yv;
  }
}

// Boundary rows from the sums: the centred OLS slope from the row's moments,
// sxx = C_0 - S^2/m, sxy = D_d - S T/m (R33: one-pass centred moments; the two-pass form of R16
// needs the probes themselves); sxx < 1e-300 -> N(i,i) := 1, flagged.  Writes result[0..5].
__global__ void mrep_boundary_sums_kernel(const double* __restrict__ sums, int64_t ns, int m, int64_t n, int d,
                                          MrepOut out, MrepScratch sc) {
  __shared__ double st[64][6];
  const int t = threadIdx.x;
  double v[6] = {0.0, 0.0, INFINITY, 0.0, 0.0, 0.0};
  const int64_t i = (t < d) ? t : (n - 2 * d + t);
  if (t < 2 * d && i >= 0 && i < n) {
    const double S = sums[(int64_t)(2 * d + 1) * ns + i], T = sums[(int64_t)(4 * d + 3) * ns + i];
    const double C0 = sums[i], Dd = sums[(int64_t)(2 * d + 2 + d) * ns + i];
    const double mx = S / (double)m, my = T / (double)m;
    const double sxx = C0 - S * mx, sxy = Dd - S * my;
    double b1, b0;
    int kind;
    if (sxx < 1e-300) { b1 = 1.0; b0 = 0.0; kind = PSP_ROW_FALLBACK_ZEROVAR; v[4] = 1.0; }
    else { b1 = sxy / sxx; b0 = my - b1 * mx; kind = PSP_ROW_BOUNDARY; }
    for (int o = 0; o <= 2 * d; ++o) out.bands[(int64_t)o * n + i] = (o == d) ? b1 : 0.0;
    if (out.intercept) out.intercept[i] = b0;
    if (out.kind) out.kind[i] = (uint8_t)kind;
    if (out.kappa) out.kappa[i] = 0.0;
    v[0] = fabs(b1);
    v[2] = fabs(b1);
    if (!(fabs(b1) > 0.0)) { v[1] = fabs(b1); v[5] = 1.0; }
  }
  for (int q = 0; q < 6; ++q) st[t][q] = v[q];
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < 64; ++w) {
      v[0] = fmax(v[0], st[w][0]);
      v[1] = fmax(v[1], st[w][1]);
      v[2] = fmin(v[2], st[w][2]);
      v[3] += st[w][3];
      v[4] += st[w][4];
      v[5] += st[w][5];
    }
    for (int q = 0; q < 6; ++q) sc.result[q] = v[q];
  }
}
}  // namespace

void launch_mrep_accumulate(const double* x, const double* y, const double* scale, int slot, int64_t n, int d,
                            double* sums, int64_t ns, int first, cudaStream_t s) {
  int64_t nb = (n + 255) / 256;
  if (nb > 16 * device_sms()) nb = 16 * device_sms();
  const unsigned g = (unsigned)(nb < 1 ? 1 : nb);
  switch (d) {
    case 1: mrep_accumulate_kernel<1><<<g, 256, 0, s>>>(x, y, scale, slot, n, sums, ns, first); break;
    case 2: mrep_accumulate_kernel<2><<<g, 256, 0, s>>>(x, y, scale, slot, n, sums, ns, first); break;
    case 3: mrep_accumulate_kernel<3><<<g, 256, 0, s>>>(x, y, scale, slot, n, sums, ns, first); break;
    default: mrep_accumulate_kernel<4><<<g, 256, 0, s>>>(x, y, scale, slot, n, sums, ns, first); break;
  }
}

void mrep_fit_sums(int m, int64_t n, int d, MrepOut out, MrepScratch sc, cudaStream_t s) {
  cudaMemsetAsync(sc.result, 0, 16 * sizeof(double), s);
  mrep_boundary_sums_kernel<<<1, 64, 0, s>>>(sc.sums, sc.sums_n, m, n, d, out, sc);
  const int64_t rows = n - 2 * d;
  if (rows > 0) {
    int64_t g = (rows + TT - 1) / TT;
    if (g > (int64_t)PSP_MREP_FIT_MINB * device_sms()) g = (int64_t)PSP_MREP_FIT_MINB * device_sms();
    switch (d) {
      case 1: mrep_fitsum_kernel<1><<<(unsigned)g, TT, 0, s>>>(m, n, n, 0, d, n - d, out, sc); break;
      case 2: mrep_fitsum_kernel<2><<<(unsigned)g, TT, 0, s>>>(m, n, n, 0, d, n - d, out, sc); break;
      case 3: mrep_fitsum_kernel<3><<<(unsigned)g, TT, 0, s>>>(m, n, n, 0, d, n - d, out, sc); break;
      default: mrep_fitsum_kernel<4><<<(unsigned)g, TT, 0, s>>>(m, n, n, 0, d, n - d, out, sc); break;
    }
  }
  mrep_decide_kernel<<<1, 1, 0, s>>>(sc);
  int pb = (int)((n + 255) / 256);
  if (pb > 8 * device_sms()) pb = 8 * device_sms();
  mrep_patch_kernel<<<pb, 256, 0, s>>>(n, d, out, sc);
}

void launch_gate_count(const double* bands, int64_t n, int d, int64_t grow0, int64_t gN, double* count,
                       cudaStream_t s, int spd) {
  cudaMemsetAsync(count, 0, sizeof(double), s);
  int64_t nb = (n + 255) / 256;
  if (nb > 8 * device_sms()) nb = 8 * device_sms();
  gate_count_kernel<<<(unsigned)(nb < 1 ? 1 : nb), 256, 0, s>>>(bands, n, d, grow0, gN, count, spd);
}

namespace {
// R29: N_s(i, i+o-d) = (N(i, i+o-d) + N(i+o-d, i)) / 2, the second term from band 2d-o of row i+o-d
__global__ void sym_bands_kernel(const double* __restrict__ b, double* __restrict__ sym, int64_t n, int d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int o = 0; o <= 2 * d; ++o) {
      const int64_t j = i + o - d;
      sym[(int64_t)o * n + i] = (j < 0 || j >= n) ? 0.0 : 0.5 * (b[(int64_t)o * n + i] + b[(int64_t)(2 * d - o) * n + j]);
    }
  }
}
}  // namespace

void launch_sym_bands(const double* bands, double* sym, int64_t n, int d, cudaStream_t s) {
  int64_t nb = (n + 255) / 256;
  if (nb > 8 * device_sms()) nb = 8 * device_sms();
  sym_bands_kernel<<<(unsigned)(nb < 1 ? 1 : nb), 256, 0, s>>>(bands, sym, n, d);
}

int mrep_launch(const double* px, const double* py, const double* slot_scale, int64_t ld,
                const int32_t* slots, int m, int64_t n, int d, MrepOut out, MrepScratch sc,
                cudaStream_t s, MrepMulti mm) {
  const bool multi = mm.comm && mm.comm->nranks > 1;
  Cols cols;
  cols.px = px;
  cols.py = py;
  cols.scale = slot_scale;
  cols.ld = ld;
  cols.hlo = cols.hhi = nullptr;
  cols.hd = d;
  cols.grow0 = multi ? mm.row0 : 0;
  cols.gN = multi ? mm.gN : n;
  for (int c = 0; c < m && c < kMaxM; ++c) cols.slot[c] = slots ? slots[c] : c;
  if (multi) {
    // the d P_x rows beyond each end of this rank's block (Alg.2's P_x(i-d..i+d,:))
    mrep_pack_kernel<<<4, 256, 0, s>>>(cols, m, n, d, mm.send);
    const size_t cnt = (size_t)m * d;
    if (mm.comm->sendrecv(mm.send, mm.recv, cnt, mm.send + cnt, mm.recv + cnt, cnt, s)) return 1;
    cols.hlo = mm.comm->rank > 0 ? mm.recv : nullptr;
    cols.hhi = mm.comm->rank < mm.comm->nranks - 1 ? mm.recv + cnt : nullptr;
  }
  cudaMemsetAsync(sc.result, 0, 16 * sizeof(double), s);
  mrep_boundary_kernel<<<1, 64, 0, s>>>(cols, m, n, d, out, sc);   // writes result[0..5]
  // rows [R0, R1) go to the TMA kernel (tiles of TT - 2d emitted rows whose P_x / P_y rows,
  // widened by one row for 16-byte alignment, lie inside this rank's block), the rest to the
  // generic kernel
  const int64_t Et = TT - 2 * d;
  const int64_t R0 = 2 * d + 2;
  int64_t ntile = (n - 1 - 3 * d - R0) >= 0 ? (n - 1 - 3 * d - R0) / Et : 0;
  // the TMA kernel needs every column's P_x (and P_y) segments to share a 16-byte parity
  int sxp = -1, syp = -1;
  bool uniform = true;
  for (int c = 0; c < m && c < kMaxM; ++c) {
    const uintptr_t ax = (uintptr_t)(px + (int64_t)cols.slot[c] * ld);
    const uintptr_t ay = (uintptr_t)(py + (int64_t)cols.slot[c] * ld);
    const int px_par = (int)((ax >> 3) & 1), py_par = (int)(((ay >> 3) + (uintptr_t)(R0 - d)) & 1);
    if (sxp < 0) { sxp = px_par; syp = py_par; }
    uniform = uniform && px_par == sxp && py_par == syp && (ax & 7) == 0 && (ay & 7) == 0;
  }
  if (ntile < 1 || m > kMaxM || !uniform) ntile = 0;
  const int64_t R1 = ntile > 0 ? R0 + ntile * Et : n;
  const int64_t a0 = 0, a1 = ntile > 0 ? R0 : n, b0 = R1, b1 = ntile > 0 ? n : n;
  {
    const int64_t E = TPB - 2 * d;
    const int64_t nt = (a1 - a0 + E - 1) / E + (b1 > b0 ? (b1 - b0 + E - 1) / E : 0);
    const int nb = (int)(nt < kMrepMaxBlocks ? (nt > 0 ? nt : 1) : kMrepMaxBlocks);
    switch (d) {
      case 1: mrep_interior_kernel<1><<<nb, TPB, 0, s>>>(cols, m, n, a0, a1, b0, b1, out, sc); break;
      case 2: mrep_interior_kernel<2><<<nb, TPB, 0, s>>>(cols, m, n, a0, a1, b0, b1, out, sc); break;
      case 3: mrep_interior_kernel<3><<<nb, TPB, 0, s>>>(cols, m, n, a0, a1, b0, b1, out, sc); break;
      default: mrep_interior_kernel<4><<<nb, TPB, 0, s>>>(cols, m, n, a0, a1, b0, b1, out, sc); break;
    }
  }
  if (ntile > 0) {
    TmaCols tc;
    tc.px = px;
    tc.py = py;
    tc.ld = ld;
    tc.sx = sxp;
    tc.sy = syp;
    for (int c = 0; c < m; ++c) tc.slot[c] = cols.slot[c];
    const int64_t nbmax = 4 * (int64_t)device_sms();
    const int nb = (int)(ntile < nbmax ? ntile : nbmax);
    switch (d) {
      case 1: launch_tma<1>(tc, slot_scale, m, n, cols.gN, cols.grow0, R0, ntile, out, sc, nb, s); break;
      case 2: launch_tma<2>(tc, slot_scale, m, n, cols.gN, cols.grow0, R0, ntile, out, sc, nb, s); break;
      case 3: launch_tma<3>(tc, slot_scale, m, n, cols.gN, cols.grow0, R0, ntile, out, sc, nb, s); break;
      default: launch_tma<4>(tc, slot_scale, m, n, cols.gN, cols.grow0, R0, ntile, out, sc, nb, s); break;
    }
  }
  if (multi) {
    // R18 needs the global max |N(i,i)|, R21 the global non-dominant statistics
    if (mm.comm->allreduce(sc.result + 0, 2, 1, s)) return 1;  // max |diag|, max over non-dominant
    if (mm.comm->allreduce(sc.result + 2, 1, 2, s)) return 1;  // min |diag|
    if (mm.comm->allreduce(sc.result + 3, 3, 0, s)) return 1;  // counts
  }
  mrep_decide_kernel<<<1, 1, 0, s>>>(sc);
  int pb = (int)((n + 255) / 256);
  if (pb > 8 * device_sms()) pb = 8 * device_sms();
  mrep_patch_kernel<<<pb, 256, 0, s>>>(n, d, out, sc);
  if (multi && mm.comm->allreduce(sc.result + 8, 1, 0, s)) return 1;  // rows patched by R18
  return 0;
}

}  // namespace psp
