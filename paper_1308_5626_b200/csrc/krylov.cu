// krylov.cu -- K2 (Gram-Schmidt), K5 (Givens / back-substitution) and the vector passes of
// Algorithm 1.
//
// Lagged normalisation: the Krylov columns are stored unnormalised, V(:,j) = alpha_j * Vs(:,j)
// with alpha_j = 1/||R_bar|| (j = 1) or 1/H(j,j-1) kept on the device; every
// reader folds alpha_j into its coefficient, so line 18's division costs no pass over memory.
//
// Every reduction is deterministic: a fixed grid of blocks writes one partial per block, and
// the last block to finish (atomic ticket) sums the partials in a fixed order.  Bitwise
// run-to-run determinism follows.  The last block also runs the O(k) scalar epilogue
// (Givens rotation, triangular solves) on one thread, so an Arnoldi step costs no extra
// launch for its scalar work.
//
// Streaming kernels keep RPT rows per thread in registers (rows t + TPB*i of a TPB*RPT tile)
// and walk the k basis vectors in chunks of JC, so each thread has JC*RPT independent 8-byte
// loads in flight: enough bytes in flight per SM to cover the HBM latency.
#include <math.h>

#include "cg.cuh"
#include "givens.cuh"
#include "internal.h"
#include "reduce.cuh"

namespace psp {
namespace {

constexpr int TPB = kRedThreads;  // 256
constexpr int kWarps = TPB / 32;
constexpr int RPT = 8;            // rows per thread in the register-tiled passes
constexpr int TILE = TPB * RPT;   // 2048 rows
constexpr int JC = 4;             // basis vectors per chunk

// ------------------------------------------------------------------------------------------
// Scalar epilogues of the reductions (one thread), from the totals tot[]
// ------------------------------------------------------------------------------------------
__device__ void updcomb_tail(DevState ds, int k, int nA, double tt);

__device__ void epilogue(int kind, DevState ds, int k, int nA, int j, int slot, const double* tot) {
  const int ld = nA + 1;
  if (kind == EPI_FUSED) {                        // multi-rank fused ring step (givens.cuh)
    fused_tail(ds, k, nA, tot, ds.slot_scale, slot);
    return;
  }
  if (kind == EPI_UPDCOMB) {                      // multi-rank last step of a ring cycle
    updcomb_tail(ds, k, nA, tot[0]);
    return;
  }
  if (kind >= EPI_CG_START) {                     // f4 (cg.cuh); j = 1: N = I
    cg_epilogue(kind, ds, slot, j, tot);
    return;
  }
  switch (kind) {
    case EPI_NORM:
      ds.scal[slot] = sqrt(tot[0]);
      break;
    case EPI_RESIDUAL: {  // Alg.1 l.5-7
      const double beta = sqrt(tot[0]);
      ds.scal[SC_BETA] = beta;
      for (int q = 0; q <= nA; ++q) ds.G[q] = 0.0;  // l.44 "clean"
      ds.G[0] = beta;                                // l.7
      ds.alpha[0] = (beta > 0.0 && isfinite(beta)) ? 1.0 / beta : 0.0;
      break;
    }
    case EPI_MGS:  // l.14: H(j,k) = V(:,j)' U
      ds.H[(int64_t)(k - 1) * ld + (j - 1)] = ds.alpha[j - 1] * tot[0];
      break;
    case EPI_MGS_FINAL:
    case EPI_UPDATE:  // l.17: H(k+1,k) = ||U||, then Givens (l.19-32)
      ds.H[(int64_t)(k - 1) * ld + k] = sqrt(tot[0]);
      givens_update(ds, k, nA);
      break;
    case EPI_DOTS:
    case EPI_DOTS_RAW: {  // ICWY: the new row of L and (I + L) h = s (R11)
      const double ak = ds.alpha[k - 1];
      double* Lrow = ds.Lm + (int64_t)(k - 1) * ld;
      for (int jb = 0; jb < k - 1; ++jb) Lrow[jb] = ds.alpha[jb] * ak * tot[k + jb];
      double* Hc = ds.H + (int64_t)(k - 1) * ld;
      for (int jb = 0; jb < k; ++jb) {  // s_j = alpha_j V_j'w (raw w: alpha_j alpha_k V_j'w~)
        double h = (kind == EPI_DOTS_RAW) ? ds.alpha[jb] * ak * tot[jb] : ds.alpha[jb] * tot[jb];
        const double* Lr = ds.Lm + (int64_t)jb * ld;
        for (int c = 0; c < jb; ++c) h -= Lr[c] * Hc[c];
        Hc[jb] = h;
      }
      break;
    }
    case EPI_HYB: {  // split-column ring step k (j = J): as the fused pass's epilogue (fused.cu)
      // columns [0, J): tot = [s_0..s_J, l_0..l_{J-1}] of the dots pass (s_J = u'w~);
      // columns [J, k): ds.rpart = [t_J..t_{k-1}, l_J..l_{k-1}, t_u, nu] of the fused pass
      const int J = j, kk = k - J;
      const double* hb = ds.rpart + kHybOff;
      const double t_u = hb[2 * kk], s_nu = hb[2 * kk + 1];
      ds.H[(int64_t)(k - 1) * ld + k] = sqrt(s_nu);  // l.17: H(k+1,k) = ||U_k||
      givens_update(ds, k, nA);                       // l.19-32, sets alpha[k] (0 on breakdown)
      if (k >= nA) break;
      const double an = ds.alpha[k];
      double* Lrow = ds.Lm + (int64_t)k * ld;        // the new row of L (R11)
      for (int jb = 0; jb < k; ++jb) Lrow[jb] = ds.alpha[jb] * an * (jb < J ? tot[J + 1 + jb] : hb[kk + jb - J]);
      double* Hc = ds.H + (int64_t)k * ld;           // (I + L) h = s for step k+1
      for (int jb = 0; jb <= k; ++jb) {
        double h = (jb < k) ? ds.alpha[jb] * an * (jb < J ? tot[jb] : hb[jb - J]) : an * an * t_u;
        const double* Lr = ds.Lm + (int64_t)jb * ld;
        for (int c = 0; c < jb; ++c) h -= Lr[c] * Hc[c];
        Hc[jb] = h;
      }
      break;
    }
  }
}

// last block, thread 0: run the epilogue, or (multi-rank) park this rank's totals in rpart for
// the host's all-reduce, after which launch_epilogue runs the same epilogue on every rank
__device__ void finish_scalar(const DevState& ds, int kind, int k, int nA, int j, int slot,
                              const double* tot, int nv) {
  if (ds.multi) {
    for (int v = 0; v < nv; ++v) ds.rpart[v] = tot[v];
  } else {
    epilogue(kind, ds, k, nA, j, slot, tot);
  }
}

__global__ void epilogue_kernel(int kind, DevState ds, int k, int nA, int j, int slot) {
  epilogue(kind, ds, k, nA, j, slot, ds.rpart);
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(TPB) norm_kernel(const double* __restrict__ x, int64_t n,
                                                   DevState ds, int slot) {
  __shared__ double sm[kWarps];
  double a[1] = {0.0};
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    double v = x[r];
    a[0] = fma(v, v, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_AUX)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_NORM, 0, 0, 0, slot, &t, 1);
  }
}

__global__ void __launch_bounds__(TPB) diff_norm_kernel(const double* __restrict__ b,
                                                        const double* __restrict__ y, int64_t n,
                                                        DevState ds, int slot) {
  __shared__ double sm[kWarps];
  double a[1] = {0.0};
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    double v = b[r] - y[r];
    a[0] = fma(v, v, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_AUX)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_NORM, 0, 0, 0, slot, &t, 1);
  }
}

// Alg.1 l.5-7: R_bar = B - P_y(:,i) -> V(:,1) (unnormalised), beta = ||R_bar||,
// G(1) = beta, alpha_1 = 1/beta (l.6).
__global__ void __launch_bounds__(TPB) residual_kernel(const double* __restrict__ b,
                                                       const double* __restrict__ y,
                                                       double* __restrict__ v, int64_t n,
                                                       DevState ds, int nA) {
  __shared__ double sm[kWarps];
  double a[1] = {0.0};
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    double t = b[r] - y[r];
    v[r] = t;
    a[0] = fma(t, t, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_RESIDUAL, 0, nA, 0, 0, &t, 1);
  }
}

__global__ void copy_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    y[r] = x[r];
}

// ------------------------------------------------------------------------------------------
// Literal MGS (Alg.1 l.13-16), one grid pass per j:
//   U <- src - H(j-1,k) V(:,j-1)   (the update of step j-1, lagged into this pass)
//   H(j,k) <- V(:,j)' U
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(TPB) mgs_literal_kernel(const double* src, double* U,
                                                          const double* __restrict__ Vprev,
                                                          const double* __restrict__ Vj, int j,
                                                          int k, int nA, int64_t n, DevState ds) {
  __shared__ double sm[kWarps];
  const int ld = nA + 1;
  const double hprev = Vprev ? ds.H[(int64_t)(k - 1) * ld + (j - 2)] * ds.alpha[j - 2] : 0.0;
  double a[1] = {0.0};
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    double u = src[r];
    if (Vprev) u = fma(-hprev, Vprev[r], u);
    U[r] = u;
    a[0] = fma(Vj[r], u, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_MGS, k, nA, j, 0, &t, 1);
  }
  (void)ld;
}

// U <- U - H(k,k) V(:,k) ; H(k+1,k) = ||U|| (l.17) ; Givens (l.19-32)
__global__ void __launch_bounds__(TPB) mgs_literal_final_kernel(double* __restrict__ U,
                                                                const double* __restrict__ Vk,
                                                                int k, int nA, int64_t n,
                                                                DevState ds) {
  __shared__ double sm[kWarps];
  const int ld = nA + 1;
  const double h = ds.H[(int64_t)(k - 1) * ld + (k - 1)] * ds.alpha[k - 1];
  double a[1] = {0.0};
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    double u = fma(-h, Vk[r], U[r]);
    U[r] = u;
    a[0] = fma(u, u, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_MGS_FINAL, k, nA, 0, 0, &t, 1);
  }
}

// ------------------------------------------------------------------------------------------
// ICWY one-reduction MGS (R11; the Swirydowicz-Langou-Ananthan-Yang-Thomas 2020 form):
// the MGS coefficients satisfy (I + L) h = V'w with L = strictly-lower part of V'V, exactly
// the sequential MGS recurrence h_j = V_j'w - sum_{i<j} (V_j'V_i) h_i.
// Pass A: s_j = V_j'w (j <= k) and l_j = V_k'V_j (j < k, the new row of L) in one pass over
// the k+1 vectors; the last block solves (I + L) h = s into H(1..k, k).
// ------------------------------------------------------------------------------------------
template <int C, bool FULL>
__device__ __forceinline__ void dots_chunk(const double* const* cp, int j0,
                                           const double (&wr)[RPT], const double (&qr)[RPT],
                                           int64_t n, int64_t r0, int lane, int k, double* acc) {
  double as[C], al[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    as[c] = 0.0;
    al[c] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double* __restrict__ vj = cp[j0 + c];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t r = r0 + (int64_t)TPB * i;
      const double v = (FULL || r < n) ? vj[r] : 0.0;
      as[c] = fma(v, wr[i], as[c]);
      al[c] = fma(v, qr[i], al[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double s1 = warp_sum(as[c]);
    const double s2 = warp_sum(al[c]);
    if (lane == 0) {
      acc[j0 + c] += s1;
      acc[k + j0 + c] += s2;
    }
  }
}

template <bool FULL>
__device__ __forceinline__ void dots_tile(const double* const* cp,
                                          const double* __restrict__ w, int k, int64_t n,
                                          int64_t r0, int lane, double* acc) {
  const double* __restrict__ qk = cp[k - 1];
  double wr[RPT], qr[RPT];
  double sk = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int64_t r = r0 + (int64_t)TPB * i;
    wr[i] = (FULL || r < n) ? w[r] : 0.0;
    qr[i] = (FULL || r < n) ? qk[r] : 0.0;
    sk = fma(qr[i], wr[i], sk);
  }
  int j0 = 0;
  for (; j0 + JC <= k - 1; j0 += JC) dots_chunk<JC, FULL>(cp, j0, wr, qr, n, r0, lane, k, acc);
  for (; j0 < k - 1; ++j0) dots_chunk<1, FULL>(cp, j0, wr, qr, n, r0, lane, k, acc);
  sk = warp_sum(sk);
  if (lane == 0) acc[k - 1] += sk;
}
__global__ void __launch_bounds__(TPB) icwy_dots_kernel(Basis V,
                                                        const double* __restrict__ w, int k,
                                                        int nA, int64_t n, int w_raw, DevState ds,
                                                        const double* last, int kstep) {
  // last != NULL: column k-1 is `last` (the split-column step's new u), and the epilogue is
  // EPI_HYB of step kstep with J = k-1 columns from here
  __shared__ double accw[kWarps][2 * kMaxRestart];
  __shared__ const double* cp[kMaxRestart + 1];   // V(:,j) resolved once (ring slots)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, t = threadIdx.x;
  for (int q = t; q < k; q += TPB) cp[q] = (last != nullptr && q == k - 1) ? last : V.col(q);
  __syncthreads();
  const int nv = 2 * k - 1;  // s_0..s_{k-1} at [0,k), l_0..l_{k-2} at [k, 2k-1)
  for (int q = lane; q < 2 * k; q += 32) accw[warp][q] = 0.0;
  __syncwarp();
  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int64_t nfull = n / TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TILE + t;
    if (tile < nfull) dots_tile<true>(cp, w, k, n, r0, lane, accw[warp]);
    else dots_tile<false>(cp, w, k, n, r0, lane, accw[warp]);
  }
  __syncthreads();
  const int nb = gridDim.x;
  for (int q = t; q < nv; q += TPB) {
    double s = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) s += accw[w2][q];
    ds.partials[(int64_t)q * nb + blockIdx.x] = s;
  }
  if (finish_block(ds.tickets + TK_MAIN)) {
    __shared__ double tot[2 * kMaxRestart];
    for (int q = warp; q < nv; q += kWarps) {
      double s = 0.0;
      for (int b = lane; b < nb; b += 32) s += ((volatile double*)ds.partials)[(int64_t)q * nb + b];
      s = warp_sum(s);
      if (lane == 0) tot[q] = s;
    }
    __syncthreads();
    if (t == 0) {
      if (last != nullptr) finish_scalar(ds, EPI_HYB, kstep, nA, k - 1, 0, tot, nv);
      else finish_scalar(ds, w_raw ? EPI_DOTS_RAW : EPI_DOTS, k, nA, 0, 0, tot, nv);
    }
  }
}

// Pass B tile: URPT rows per thread, UJC basis vectors per chunk (URPT*UJC = 32 loads in
// flight per thread); bounds checks only in the last, partial tile.
constexpr int URPT = 4;
constexpr int UJC = 8;
constexpr int UTILE = TPB * URPT;

template <bool FULL>
__device__ __forceinline__ void update_tile(const double* const* cp, const double* w, double wsc, double* U,
                                            const double* hs, int k, int64_t n, int64_t r0,
                                            double& acc) {
  double u[URPT];
#pragma unroll
  for (int i = 0; i < URPT; ++i) {
    const int64_t r = r0 + (int64_t)TPB * i;
    u[i] = (w != nullptr && (FULL || r < n)) ? wsc * w[r] : 0.0;
  }
  int jb = 0;
  for (; jb + UJC <= k; jb += UJC) {
    double v[UJC][URPT];
#pragma unroll
    for (int c = 0; c < UJC; ++c)
#pragma unroll
      for (int i = 0; i < URPT; ++i) {
        const int64_t r = r0 + (int64_t)TPB * i;
        v[c][i] = (FULL || r < n) ? cp[jb + c][r] : 0.0;
      }
#pragma unroll
    for (int c = 0; c < UJC; ++c)
#pragma unroll
      for (int i = 0; i < URPT; ++i) u[i] = fma(-hs[jb + c], v[c][i], u[i]);
  }
  for (; jb < k; ++jb) {
    double v[URPT];
#pragma unroll
    for (int i = 0; i < URPT; ++i) {
      const int64_t r = r0 + (int64_t)TPB * i;
      v[i] = (FULL || r < n) ? cp[jb][r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < URPT; ++i) u[i] = fma(-hs[jb], v[i], u[i]);
  }
#pragma unroll
  for (int i = 0; i < URPT; ++i) {
    const int64_t r = r0 + (int64_t)TPB * i;
    if (FULL || r < n) {
      U[r] = u[i];
      acc = fma(u[i], u[i], acc);
    }
  }
}

// Pass B: U = w - sum_j h_j alpha_j V_j (sequential in j, as the MGS updates), H(k+1,k) =
// ||U||, then the Givens update of column k.
__global__ void __launch_bounds__(TPB) icwy_update_kernel(Basis V, const double* __restrict__ w,
                                                          const double* ws,
                                                          double* __restrict__ U, int k, int nA,
                                                          int64_t n, DevState ds, int ncols) {
  // ncols < k: the partial update of a split-column step (columns [0, ncols) only, no epilogue)
  __shared__ double hs[kMaxRestart];
  __shared__ double sm[kWarps];
  __shared__ const double* cp[kMaxRestart + 1];
  const int ld = nA + 1, t = threadIdx.x;
  for (int q = t; q < ncols; q += TPB) {
    hs[q] = ds.H[(int64_t)(k - 1) * ld + q] * ds.alpha[q];
    cp[q] = V.col(q);
  }
  __syncthreads();
  const double wsc = ws ? *ws : 1.0;  // scale of w (the fused path stores A u unnormalised)
  double a[1] = {0.0};
  const int64_t ntiles = (n + UTILE - 1) / UTILE;
  const int64_t nfull = n / UTILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * UTILE + t;
    if (tile < nfull) update_tile<true>(cp, w, wsc, U, hs, ncols, n, r0, a[0]);
    else update_tile<false>(cp, w, wsc, U, hs, ncols, n, r0, a[0]);
  }
  if (ncols < k) return;
  block_sum<1>(a, sm);
  if (t == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double tt = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (t == 0) finish_scalar(ds, EPI_UPDATE, k, nA, 0, 0, &tt, 1);
  }
}

// l.38-42: Q = H^{-1} G (R6, every block recomputes the k x k back-substitution
// redundantly: identical inputs, identical result), out = base + sum_j Q_j alpha_j V_j.
__global__ void __launch_bounds__(TPB) combine_kernel(Basis V, int k, int nA, const double* base,
                                                      double* out, int64_t n, DevState ds) {
  __shared__ double qs[kMaxRestart];
  __shared__ double qa[kMaxRestart];
  __shared__ const double* cp[kMaxRestart + 1];
  __shared__ int bad;
  for (int q = threadIdx.x; q < k; q += TPB) cp[q] = V.col(q);
  if (threadIdx.x == 0) {
    const int ld = nA + 1;
    bad = 0;
    for (int j = k; j >= 1; --j) {
      double s = ds.G[j - 1];
      for (int t = j + 1; t <= k; ++t) s -= ds.H[(int64_t)(t - 1) * ld + (j - 1)] * qs[t - 1];
      const double piv = ds.H[(int64_t)(j - 1) * ld + (j - 1)];
      if (piv == 0.0) { bad = 1; qs[j - 1] = 0.0; continue; }
      qs[j - 1] = s / piv;
    }
    for (int j = 0; j < k; ++j) qa[j] = -qs[j] * ds.alpha[j];  // update_tile subtracts
    if (blockIdx.x == 0) {
      for (int j = 0; j < k; ++j) ds.Q[j] = qs[j];
      ds.scal[SC_STATUS] = bad ? (double)PSP_E_SINGULAR : 0.0;
    }
  }
  __syncthreads();
  // out = base - sum_j qa_j V_j with qa = -Q alpha (the register-tiled update pass)
  const int64_t ntiles = (n + UTILE - 1) / UTILE;
  const int64_t nfull = n / UTILE;
  double unused = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * UTILE + threadIdx.x;
    if (tile < nfull) update_tile<true>(cp, base, 1.0, out, qa, k, n, r0, unused);
    else update_tile<false>(cp, base, 1.0, out, qa, k, n, r0, unused);
  }
}

// ------------------------------------------------------------------------------------------
// The last step of a full ring cycle (k = n_A, N = I) fused with the cycle's combine (l.38-43).
// The least-squares solution of the cycle is R y = g (R the rotated H).  Before the last Givens
// rotation is known (it needs ||U_k||), y is already fixed up to its last entry:
// y_{1:k-1} = a - y_k b, a = R_{k-1}^{-1} g'_{1:k-1}, b = R_{k-1}^{-1} h'_{1:k-1} (h' = column k
// after rotations 1..k-1; rows 1..k-1 of column k are untouched by rotation k).  So
// Z = sum_j y_j V_j = Z0 + y_k Z1 with Z0 = sum_{j<k} a_j V_j, Z1 = V_k - sum_{j<k} b_j V_j, and
// one pass over the basis forms U_k (its norm), X0 + Z0 and Z1 together; the cycle end is
// then X = (X0 + Z0) + y_k Z1.  Equal to Q = H^{-1}G (R6) and the combine in exact arithmetic.
// ------------------------------------------------------------------------------------------
__global__ void combine_prep_kernel(DevState ds, int k, int nA) {
  // one thread: c0_j = a_j alpha_j, c1_j = -b_j alpha_j (j < k-1), c1_{k-1} = alpha_{k-1} into
  // ds.rpart[0, k) / [k, 2k); rpart[2k] = 1 on a zero pivot of R_{k-1} (R6)
  const int ld = nA + 1;
  double hp[kMaxRestart + 1], a[kMaxRestart], b[kMaxRestart];   // hp[0..k]
  const double* Hk = ds.H + (int64_t)(k - 1) * ld;   // column k, MGS coefficients (unrotated)
  for (int j = 0; j <= k; ++j) hp[j] = Hk[j];
  for (int j = 1; j <= k - 1; ++j) {                 // rotations 1..k-1 (as givens_update)
    const double delta = hp[j - 1];
    hp[j - 1] = delta * ds.C[j - 1] + ds.S[j - 1] * hp[j];
    hp[j] = -delta * ds.S[j - 1] + ds.C[j - 1] * hp[j];
  }
  int bad = 0;
  for (int j = k - 1; j >= 1; --j) {                 // back-substitution on R_{k-1}
    double sa = ds.G[j - 1], sb = hp[j - 1];
    for (int t = j + 1; t <= k - 1; ++t) {
      const double r = ds.H[(int64_t)(t - 1) * ld + (j - 1)];
      sa -= r * a[t - 1];
      sb -= r * b[t - 1];
    }
    const double piv = ds.H[(int64_t)(j - 1) * ld + (j - 1)];
    if (piv == 0.0) { bad = 1; a[j - 1] = b[j - 1] = 0.0; continue; }
    a[j - 1] = sa / piv;
    b[j - 1] = sb / piv;
  }
  for (int j = 0; j < k - 1; ++j) {
    ds.rpart[j] = a[j] * ds.alpha[j];
    ds.rpart[k + j] = -b[j] * ds.alpha[j];
  }
  ds.rpart[k - 1] = 0.0;
  ds.rpart[2 * k - 1] = ds.alpha[k - 1];
  ds.rpart[2 * k] = bad ? 1.0 : 0.0;
}

constexpr int CRPT = 4;                               // rows per thread (register tile)
constexpr int CTILE = TPB * CRPT;

template <bool FULL>
__device__ __forceinline__ void update_combine_tile(const double* const* cp, const double* w, double wsc,
                                                    const double* x0, double* z0, double* z1,
                                                    const double* hs, const double* c0, const double* c1,
                                                    int k, int64_t n, int64_t r0, double& acc) {
  double u[CRPT], p[CRPT], q[CRPT];
#pragma unroll
  for (int i = 0; i < CRPT; ++i) {
    const int64_t r = r0 + (int64_t)TPB * i;
    const bool in = FULL || r < n;
    u[i] = in ? wsc * w[r] : 0.0;
    p[i] = in ? x0[r] : 0.0;
    q[i] = 0.0;
  }
  constexpr int CJ = 4;                               // columns per chunk: 16 loads in flight
  int jb = 0;
  for (; jb + CJ <= k; jb += CJ) {
    double v[CJ][CRPT];
#pragma unroll
    for (int c = 0; c < CJ; ++c)
#pragma unroll
      for (int i = 0; i < CRPT; ++i) {
        const int64_t r = r0 + (int64_t)TPB * i;
        v[c][i] = (FULL || r < n) ? cp[jb + c][r] : 0.0;
      }
#pragma unroll
    for (int c = 0; c < CJ; ++c) {
      const double hj = hs[jb + c], aj = c0[jb + c], bj = c1[jb + c];
#pragma unroll
      for (int i = 0; i < CRPT; ++i) {
        u[i] = fma(-hj, v[c][i], u[i]);
        p[i] = fma(aj, v[c][i], p[i]);
        q[i] = fma(bj, v[c][i], q[i]);
      }
    }
  }
  for (; jb < k; ++jb) {
    double v[CRPT];
#pragma unroll
    for (int i = 0; i < CRPT; ++i) {
      const int64_t r = r0 + (int64_t)TPB * i;
      v[i] = (FULL || r < n) ? cp[jb][r] : 0.0;
    }
    const double hj = hs[jb], aj = c0[jb], bj = c1[jb];
#pragma unroll
    for (int i = 0; i < CRPT; ++i) {
      u[i] = fma(-hj, v[i], u[i]);
      p[i] = fma(aj, v[i], p[i]);
      q[i] = fma(bj, v[i], q[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < CRPT; ++i) {
    const int64_t r = r0 + (int64_t)TPB * i;
    if (FULL || r < n) {
      z0[r] = p[i];
      z1[r] = q[i];
      acc = fma(u[i], u[i], acc);
    }
  }
}

// U_k = alpha_k w~_k - sum_j h_j alpha_j V_j (only ||U_k|| is kept), z0 = X0 + Z0, z1 = Z1; the
// last block: H(k+1,k), Givens (l.17-32), then Q = H^{-1}G (R6) with y_k -> ds.scal[SC_TMP].
__device__ void updcomb_tail(DevState ds, int k, int nA, double tt) {
  const int ld = nA + 1;
  epilogue(EPI_UPDATE, ds, k, nA, 0, 0, &tt);       // H(k+1,k) = ||U||, Givens of column k
  // Q = H^{-1} G (R6), as combine_kernel
  int bad = ds.rpart[2 * k] != 0.0;
  for (int j = k; j >= 1; --j) {
    double sv = ds.G[j - 1];
    for (int q = j + 1; q <= k; ++q) sv -= ds.H[(int64_t)(q - 1) * ld + (j - 1)] * ds.Q[q - 1];
    const double piv = ds.H[(int64_t)(j - 1) * ld + (j - 1)];
    if (piv == 0.0) { bad = 1; ds.Q[j - 1] = 0.0; continue; }
    ds.Q[j - 1] = sv / piv;
  }
  ds.scal[SC_TMP] = ds.Q[k - 1];                    // y_k
  ds.scal[SC_STATUS] = bad ? (double)PSP_E_SINGULAR : 0.0;
}

__global__ void __launch_bounds__(TPB) update_combine_kernel(Basis V, const double* __restrict__ w,
                                                             const double* ws, const double* __restrict__ x0,
                                                             double* __restrict__ z0, double* __restrict__ z1,
                                                             int k, int nA, int64_t n, DevState ds) {
  __shared__ double hs[kMaxRestart], c0[kMaxRestart], c1[kMaxRestart];
  __shared__ double sm[kWarps];
  __shared__ const double* cp[kMaxRestart + 1];
  const int ld = nA + 1, t = threadIdx.x;
  for (int q = t; q < k; q += TPB) {
    hs[q] = ds.H[(int64_t)(k - 1) * ld + q] * ds.alpha[q];
    c0[q] = ds.rpart[q];
    c1[q] = ds.rpart[k + q];
    cp[q] = V.col(q);
  }
  __syncthreads();
  const double wsc = ws ? *ws : 1.0;
  double a[1] = {0.0};
  const int64_t ntiles = (n + CTILE - 1) / CTILE;
  const int64_t nfull = n / CTILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * CTILE + t;
    if (tile < nfull) update_combine_tile<true>(cp, w, wsc, x0, z0, z1, hs, c0, c1, k, n, r0, a[0]);
    else update_combine_tile<false>(cp, w, wsc, x0, z0, z1, hs, c0, c1, k, n, r0, a[0]);
  }
  block_sum<1>(a, sm);
  if (t == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double tt = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (t == 0) {
      if (ds.multi) ds.rpart[0] = tt;                 // (c0 / c1 were read; rpart[2k] stays)
      else updcomb_tail(ds, k, nA, tt);
    }
  }
  (void)ld;
}

// cycle end after update_combine_kernel: x = z0 + y_k z1
__global__ void __launch_bounds__(TPB) combine_finish_kernel(const double* __restrict__ z0,
                                                             const double* __restrict__ z1, double* __restrict__ x,
                                                             int64_t n, DevState ds) {
  const double yk = ds.scal[SC_TMP];
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB)
    x[r] = fma(yk, z1[r], z0[r]);
}

// ------------------------------------------------------------------------------------------
// f4: PSP-CG passes (readings R27-R31; oracle/oracle.c orc_pcg for the recurrences)
// ------------------------------------------------------------------------------------------
// r = b - A x0 (y = A x0 was recorded as the probe of x0); r'r
__global__ void __launch_bounds__(TPB) cg_start_kernel(const double* __restrict__ b, const double* __restrict__ y,
                                                       double* __restrict__ r, int64_t n, DevState ds) {
  __shared__ double sm[kWarps];
  double a[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    const double t = b[i] - y[i];
    r[i] = t;
    a[0] = fma(t, t, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_CG_START, 0, 0, 1, 0, &t, 1);
  }
}

// p = z + beta p_old (R27); p_old == NULL: p = z (the first direction)
__global__ void __launch_bounds__(TPB) cg_pupdate_kernel(const double* __restrict__ z, const double* __restrict__ pold,
                                                         double* __restrict__ p, int64_t n, DevState ds) {
  const double beta = ds.scal[SC_BETACG];
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB)
    p[i] = pold ? fma(beta, pold[i], z[i]) : z[i];
}

// p'q and p'p of the direction just applied -> alpha and the slot's probe scale
__global__ void __launch_bounds__(TPB) cg_dirdots_kernel(const double* __restrict__ p, const double* __restrict__ q,
                                                         int64_t n, int slot, DevState ds) {
  __shared__ double sm[kWarps * 2];
  double a[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    const double pv = p[i];
    a[0] = fma(pv, q[i], a[0]);
    a[1] = fma(pv, pv, a[1]);
  }
  block_sum<2>(a, sm);
  if (threadIdx.x == 0) {
    ds.partials[blockIdx.x] = a[0];
    ds.partials[gridDim.x + blockIdx.x] = a[1];
  }
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t[2];
    t[0] = reduce_partials(ds.partials, 0, gridDim.x, sm);
    t[1] = reduce_partials(ds.partials, 1, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_CG_DIR, 0, 0, 1, slot, t, 2);
  }
}

// x += alpha p, r -= alpha q; r'r
__global__ void __launch_bounds__(TPB) cg_update_kernel(double* __restrict__ x, const double* __restrict__ p,
                                                        const double* __restrict__ q, double* __restrict__ r, int64_t n,
                                                        int identity, DevState ds) {
  __shared__ double sm[kWarps];
  const double alpha = ds.scal[SC_ALPHA];
  double a[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    x[i] = fma(alpha, p[i], x[i]);
    const double rv = fma(-alpha, q[i], r[i]);
    r[i] = rv;
    a[0] = fma(rv, rv, a[0]);
  }
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_CG_UPD, 0, 0, identity, 0, &t, 1);
  }
}

// r'z (N != I)
__global__ void __launch_bounds__(TPB) cg_rz_kernel(const double* __restrict__ r, const double* __restrict__ z,
                                                    int64_t n, DevState ds) {
  __shared__ double sm[kWarps];
  double a[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB)
    a[0] = fma(r[i], z[i], a[0]);
  block_sum<1>(a, sm);
  if (threadIdx.x == 0) ds.partials[blockIdx.x] = a[0];
  if (finish_block(ds.tickets + TK_MAIN)) {
    double t = reduce_partials(ds.partials, 0, gridDim.x, sm);
    if (threadIdx.x == 0) finish_scalar(ds, EPI_CG_RHO, 0, 0, 0, 0, &t, 1);
  }
}

inline int grid_for(int64_t n, int cap) {
  int64_t b = (n + TPB - 1) / TPB;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}
inline int tiles_grid(int64_t n, int cap) {
  int64_t b = (n + TILE - 1) / TILE;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_norm(const double* x, int64_t n, DevState ds, int slot, const RedCfg& rc, cudaStream_t s) {
  norm_kernel<<<rc.nblocks, TPB, 0, s>>>(x, n, ds, slot);
}
void launch_diff_norm(const double* b, const double* y, int64_t n, DevState ds, int slot,
                      const RedCfg& rc, cudaStream_t s) {
  diff_norm_kernel<<<rc.nblocks, TPB, 0, s>>>(b, y, n, ds, slot);
}
void launch_residual(const double* b, const double* y, double* v, int64_t n, int nA, DevState ds,
                     const RedCfg& rc, cudaStream_t s) {
  residual_kernel<<<rc.nblocks, TPB, 0, s>>>(b, y, v, n, ds, nA);
}
void launch_copy(const double* x, double* y, int64_t n, cudaStream_t s) {
  copy_kernel<<<grid_for(n, 8 * device_sms()), TPB, 0, s>>>(x, y, n);
}
void launch_mgs_literal(const double* src, double* U, const double* Vprev, const double* Vj,
                        int j, int k, int nA, int64_t n, DevState ds, const RedCfg& rc,
                        cudaStream_t s) {
  mgs_literal_kernel<<<rc.nblocks, TPB, 0, s>>>(src, U, Vprev, Vj, j, k, nA, n, ds);
}
void launch_mgs_literal_final(double* U, const double* Vk, int k, int nA, int64_t n,
                              DevState ds, const RedCfg& rc, cudaStream_t s) {
  mgs_literal_final_kernel<<<rc.nblocks, TPB, 0, s>>>(U, Vk, k, nA, n, ds);
}
// one full wave: the resident blocks per SM of a kernel (a partial second wave of a
// grid-stride kernel leaves SMs idle for up to a third of the launch)
template <typename K>
int wave_blocks(K kernel, int cap) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, TPB, 0) != cudaSuccess || per < 1) per = 1;
  const int b = per * device_sms();
  return b < cap ? b : cap;
}

void launch_icwy_dots(Basis V, const double* w, int k, int nA, int64_t n, int w_raw,
                      DevState ds, const RedCfg& rc, cudaStream_t s) {
  thread_local int waves[kMaxDev] = {};
  int& wave = waves[device_ordinal()];
  if (!wave) wave = wave_blocks(icwy_dots_kernel, rc.nblocks);
  icwy_dots_kernel<<<tiles_grid(n, wave), TPB, 0, s>>>(V, w, k, nA, n, w_raw, ds, nullptr, 0);
}
void launch_icwy_dots_hyb(Basis V, const double* w, const double* u, int J, int k, int nA, int64_t n,
                          DevState ds, const RedCfg& rc, cudaStream_t s) {
  thread_local int waves[kMaxDev] = {};
  int& wave = waves[device_ordinal()];
  if (!wave) wave = wave_blocks(icwy_dots_kernel, rc.nblocks);
  icwy_dots_kernel<<<tiles_grid(n, wave), TPB, 0, s>>>(V, w, J + 1, nA, n, 1, ds, u, k);
}
void launch_icwy_update(Basis V, const double* w, const double* ws, double* U, int k,
                        int nA, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s, int ncols) {
  thread_local int waves[kMaxDev] = {};
  int& wave = waves[device_ordinal()];
  if (!wave) wave = wave_blocks(icwy_update_kernel, rc.nblocks);
  int64_t ub = (n + UTILE - 1) / UTILE;
  if (ub > wave) ub = wave;
  icwy_update_kernel<<<(int)(ub < 1 ? 1 : ub), TPB, 0, s>>>(V, w, ws, U, k, nA, n, ds, ncols < 0 ? k : ncols);
}
void launch_cg_start(const double* b, const double* y, double* r, int64_t n, DevState ds, const RedCfg& rc,
                     cudaStream_t s) {
  cg_start_kernel<<<rc.nblocks, TPB, 0, s>>>(b, y, r, n, ds);
}
void launch_cg_pupdate(const double* z, const double* pold, double* p, int64_t n, DevState ds, cudaStream_t s) {
  cg_pupdate_kernel<<<grid_for(n, 8 * device_sms()), TPB, 0, s>>>(z, pold, p, n, ds);
}
void launch_cg_dirdots(const double* p, const double* q, int64_t n, int slot, DevState ds, const RedCfg& rc,
                       cudaStream_t s) {
  cg_dirdots_kernel<<<rc.nblocks, TPB, 0, s>>>(p, q, n, slot, ds);
}
void launch_cg_update(double* x, const double* p, const double* q, double* r, int64_t n, int identity,
                      DevState ds, const RedCfg& rc, cudaStream_t s) {
  cg_update_kernel<<<rc.nblocks, TPB, 0, s>>>(x, p, q, r, n, identity, ds);
}
void launch_cg_rz(const double* r, const double* z, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s) {
  cg_rz_kernel<<<rc.nblocks, TPB, 0, s>>>(r, z, n, ds);
}
void launch_epilogue(int kind, DevState ds, int k, int nA, int j, int slot, cudaStream_t s) {
  epilogue_kernel<<<1, 1, 0, s>>>(kind, ds, k, nA, j, slot);
}
void launch_update_combine(Basis V, const double* w, const double* ws, const double* x0, double* z0, double* z1,
                           int k, int nA, int64_t n, DevState ds, const RedCfg& rc, cudaStream_t s) {
  combine_prep_kernel<<<1, 1, 0, s>>>(ds, k, nA);
  thread_local int waves[kMaxDev] = {};
  int& wave = waves[device_ordinal()];
  if (!wave) wave = wave_blocks(update_combine_kernel, rc.nblocks);
  int64_t ub = (n + CTILE - 1) / CTILE;
  if (ub > wave) ub = wave;
  update_combine_kernel<<<(int)(ub < 1 ? 1 : ub), TPB, 0, s>>>(V, w, ws, x0, z0, z1, k, nA, n, ds);
}
void launch_combine_finish(const double* z0, const double* z1, double* x, int64_t n, DevState ds, cudaStream_t s) {
  int64_t b = (n + TPB - 1) / TPB;
  if (b > 8 * device_sms()) b = 8 * device_sms();
  combine_finish_kernel<<<(int)(b < 1 ? 1 : b), TPB, 0, s>>>(z0, z1, x, n, ds);
}
void launch_combine(Basis V, int k, int nA, const double* base, double* out,
                    int64_t n, DevState ds, cudaStream_t s) {
  thread_local int waves[kMaxDev] = {};
  int& wave = waves[device_ordinal()];
  if (!wave) wave = wave_blocks(combine_kernel, 8 * device_sms());
  int64_t cb = (n + UTILE - 1) / UTILE;
  if (cb > wave) cb = wave;
  combine_kernel<<<(int)(cb < 1 ? 1 : cb), TPB, 0, s>>>(V, k, nA, base, out, n, ds);
}

}  // namespace psp
