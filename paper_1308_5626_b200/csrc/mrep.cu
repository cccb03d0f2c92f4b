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

#include "internal.h"

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

__device__ __forceinline__ double band_abs_off_sum(const double* row /*2d+1 coeffs*/, int d,
                                                   int64_t i, int64_t n) {
  double off = 0.0;
  for (int o = 0; o <= 2 * d; ++o) {
    int64_t j = i + o - d;
    if (o == d || j < 0 || j >= n) continue;
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
                                         int t, int m, double lambda) {
  A[pk(0, 0)] = (double)m + lambda;
#pragma unroll
  for (int a = 0; a <= 2 * D; ++a) {
    A[pk(1 + a, 0)] = ex[(2 * D + 1) * TPB + (t - D + a)];
#pragma unroll
    for (int b = a; b <= 2 * D; ++b) A[pk(1 + b, 1 + a)] = ex[(b - a) * TPB + (t - D + a)];
    A[pk(1 + a, 1 + a)] += lambda;
  }
}

// in-place Cholesky of the packed P x P matrix (R17); false on a pivot^2 <= 0 or non-finite
template <int P>
__device__ __forceinline__ bool chol_packed(double (&A)[P * (P + 1) / 2]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double s = A[pk(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= A[pk(j, k)] * A[pk(j, k)];
    if (!(s > 0.0) || !isfinite(s)) return false;
    const double ljj = sqrt(s);
    A[pk(j, j)] = ljj;
#pragma unroll
    for (int i = j + 1; i < P; ++i) {
      double u = A[pk(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) u -= A[pk(i, k)] * A[pk(j, k)];
      A[pk(i, j)] = u / ljj;
    }
  }
  return true;
}

template <int D>
__global__ void __launch_bounds__(TPB, 2) mrep_interior_kernel(Cols cols, int m, int64_t n,
                                                               MrepOut out, MrepScratch sc) {
  constexpr int P = 2 * D + 2;
  constexpr int NP = P * (P + 1) / 2;
  constexpr int TILE = TPB + 3 * D;                 // rows [i0-2D, i0-D+TPB+2D)
  __shared__ double xs[CB][TILE];
  __shared__ double ex[(2 * D + 2) * TPB];
  __shared__ double red[TPB / 32][6];
  const int t = threadIdx.x;
  double maxdiag = 0.0, maxdiag_nd = 0.0, mindiag = INFINITY, nridge = 0.0, nfb = 0.0, nnd = 0.0;
  const int64_t ntiles = (n + (TPB - 2 * D) - 1) / (TPB - 2 * D);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const int64_t i0 = tile * (TPB - 2 * D);
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
      for (int q = t; q < TILE; q += TPB) xs[cc][q] = scx * cols.xraw(c0 + cc, tile0 + q, n);
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
  const bool emit = (t >= D && t < TPB - D) && r >= 0 && r < n && gr >= D && gr < cols.gN - D;
  if (emit) {
    double A[NP];
    assemble<D>(A, ex, t, m, 0.0);
    bool ok = chol_packed<P>(A);
    double kap = INFINITY;
    if (ok) {
      double lmax = A[pk(0, 0)], lmin = A[pk(0, 0)];
#pragma unroll
      for (int j = 1; j < P; ++j) {
        lmax = fmax(lmax, A[pk(j, j)]);
        lmin = fmin(lmin, A[pk(j, j)]);
      }
      kap = (lmax / lmin) * (lmax / lmin);
    }
    int kind = PSP_ROW_INTERIOR;
    if (!ok || kap > 1e12) {                        // S:226 ridge retry on G + lambda I
      double tr = (double)m;
#pragma unroll
      for (int a = 0; a <= 2 * D; ++a) tr += ex[0 * TPB + (t - D + a)];   // diag = C_0(r-d+a)
      const double lambda = 1e-10 * tr / (double)P;
      assemble<D>(A, ex, t, m, lambda);
      ok = chol_packed<P>(A);
      kind = PSP_ROW_INTERIOR_RIDGE;
      nridge += 1.0;
    }
    double row[2 * D + 1];
    double icpt = 0.0;
    if (!ok) {                                      // identity row
      kind = PSP_ROW_FALLBACK_RANK;
      nfb += 1.0;
#pragma unroll
      for (int o = 0; o <= 2 * D; ++o) row[o] = (o == D) ? 1.0 : 0.0;
    } else {
      double z[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double s = (i == 0) ? Tsum : Dl[i - 1];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= A[pk(i, k)] * z[k];
        z[i] = s / A[pk(i, i)];
      }
#pragma unroll
      for (int i = P - 1; i >= 0; --i) {
        double s = z[i];
#pragma unroll
        for (int k = i + 1; k < P; ++k) s -= A[pk(k, i)] * z[k];
        z[i] = s / A[pk(i, i)];
      }
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
    maxdiag = fmax(maxdiag, ad);
    mindiag = fmin(mindiag, ad);
    if (!(ad > band_abs_off_sum(row, D, gr, cols.gN))) { nnd += 1.0; maxdiag_nd = fmax(maxdiag_nd, ad); }
  }
  }  // tiles
  // block reduction of the gate statistics (max, max, min, sum, sum, sum)
  double v[6] = {maxdiag, maxdiag_nd, mindiag, nridge, nfb, nnd};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v[0] = fmax(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
    v[1] = fmax(v[1], __shfl_xor_sync(0xffffffffu, v[1], o));
    v[2] = fmin(v[2], __shfl_xor_sync(0xffffffffu, v[2], o));
    v[3] += __shfl_xor_sync(0xffffffffu, v[3], o);
    v[4] += __shfl_xor_sync(0xffffffffu, v[4], o);
    v[5] += __shfl_xor_sync(0xffffffffu, v[5], o);
  }
  if ((t & 31) == 0)
    for (int q = 0; q < 6; ++q) red[t >> 5][q] = v[q];
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < TPB / 32; ++w) {
      v[0] = fmax(v[0], red[w][0]);
      v[1] = fmax(v[1], red[w][1]);
      v[2] = fmin(v[2], red[w][2]);
      v[3] += red[w][3];
      v[4] += red[w][4];
      v[5] += red[w][5];
    }
    for (int q = 0; q < 6; ++q) sc.partials[(int64_t)q * gridDim.x + blockIdx.x] = v[q];
  }
  // last block: fold in the boundary rows (result[0..5] written by the boundary kernel) and
  // evaluate R18 / R21
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (t == 0) {
    unsigned tk = atomicAdd(sc.ticket, 1u);
    s_last = (tk == gridDim.x - 1);
    if (s_last) *sc.ticket = 0u;
  }
  __syncthreads();
  if (s_last && t == 0) {
    __threadfence();
    volatile double* pp = sc.partials;
    volatile double* res = sc.result;
    double a[6] = {res[0], res[1], res[2], res[3], res[4], res[5]};
    for (unsigned b = 0; b < gridDim.x; ++b) {
      a[0] = fmax(a[0], pp[0 * gridDim.x + b]);
      a[1] = fmax(a[1], pp[1 * gridDim.x + b]);
      a[2] = fmin(a[2], pp[2 * gridDim.x + b]);
      a[3] += pp[3 * gridDim.x + b];
      a[4] += pp[4 * gridDim.x + b];
      a[5] += pp[5 * gridDim.x + b];
    }
    for (int q = 0; q < 6; ++q) res[q] = a[q];
    // R18 threshold and the R21 decision: every non-dominant row must be patched to identity
    const double thr = 1e-12 * a[0];
    res[6] = (a[2] < thr) ? 1.0 : 0.0;                       // some row needs the R18 patch
    res[7] = (a[5] == 0.0 || a[1] < thr) ? 1.0 : 0.0;        // gate accepted (R21)
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

// The real entry point (api.cpp): column base pointers + slot order.
int mrep_blocks(int64_t n, int d) {
  int64_t t = (n + (TPB - 2 * d) - 1) / (TPB - 2 * d);
  return (int)(t < kMrepMaxBlocks ? t : kMrepMaxBlocks);
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

}  // namespace

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
  mrep_boundary_kernel<<<1, 64, 0, s>>>(cols, m, n, d, out, sc);
  const int nb = mrep_blocks(n, d);  // grid-stride over row tiles
  switch (d) {
    case 1: mrep_interior_kernel<1><<<nb, TPB, 0, s>>>(cols, m, n, out, sc); break;
    case 2: mrep_interior_kernel<2><<<nb, TPB, 0, s>>>(cols, m, n, out, sc); break;
    case 3: mrep_interior_kernel<3><<<nb, TPB, 0, s>>>(cols, m, n, out, sc); break;
    default: mrep_interior_kernel<4><<<nb, TPB, 0, s>>>(cols, m, n, out, sc); break;
  }
  if (multi) {
    // R18 needs the global max |N(i,i)|, R21 the global non-dominant statistics
    if (mm.comm->allreduce(sc.result + 0, 2, 1, s)) return 1;  // max |diag|, max over non-dominant
    if (mm.comm->allreduce(sc.result + 2, 1, 2, s)) return 1;  // min |diag|
    if (mm.comm->allreduce(sc.result + 3, 3, 0, s)) return 1;  // counts
    mrep_decide_kernel<<<1, 1, 0, s>>>(sc);
  }
  int pb = (int)((n + 255) / 256);
  if (pb > 148 * 8) pb = 148 * 8;
  mrep_patch_kernel<<<pb, 256, 0, s>>>(n, d, out, sc);
  if (multi && mm.comm->allreduce(sc.result + 8, 1, 0, s)) return 1;  // rows patched by R18
  return 0;
}

}  // namespace psp
