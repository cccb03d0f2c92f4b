// fused.cu -- the single-pass Arnoldi step for N = I (the gate's decision on C2-C4, R21).
//
// With N = I the preconditioner solve is the identity, Y_k = V_k, and one grid pass
// can finish step k and start step k+1 (Alg.1 l.13-18 then l.10-16 of the next k):
//   u      = alpha_k w~_k - sum_{j<=k} h_j alpha_j V_j       (MGS update of step k, ICWY form, R11)
//   w~     = A u                                            (the matrix-free matvec)
//   t_j    = V_j' w~, t_u = u' w~, l_j = V_j' u, nu = u' u   (every inner product step k+1 needs)
// u is stored as V_{k+1} (it IS the probe P_x of step k+1, so it lives in the probe ring slot)
// and w~ as the probe P_y, both unnormalised with the scale alpha_{k+1} = 1/sqrt(nu) recorded
// per ring slot (lagged normalisation).  The last block then applies the Givens rotation of
// column k (l.19-32) and solves (I + L) h = s for step k+1's MGS coefficients.
//
// Bytes per row and step: k basis columns + w~_k + kappa read, u + w~ written = 8(k+4), against
// 8(2k+7) for separate matvec / dots / update passes.
//
// Work layout: a block owns a TX x TY column of the grid and marches a chunk of planes along the
// slowest axis (2-D grids march y, 1-D grids are a single line).  Every thread owns one point of
// the tile plus its one-point halo ring (TX*TY interior threads + NH halo threads): per plane it
// issues all its loads at once (the k basis values, w~_k and kappa) and computes U at its point;
// the halo is recomputed from the L2-resident basis instead of exchanged.  Then w~ = A u on the
// previous plane from three U planes in shared memory, and that plane's dot products against
// V_j(p-1), which the interior threads parked in shared memory (Vsave) one plane earlier.
#include <math.h>

#include "givens.cuh"
#include "internal.h"

namespace psp {
namespace {

template <int TX, int TY>
struct Tile {
  static constexpr bool HASY = TY > 1;               // y halo rows (3-D tiles)
  static constexpr int HX = TX + 2, HY = HASY ? TY + 2 : TY, HP = HX * HY;
  static constexpr int NI = TX * TY;                 // interior points
  static constexpr int NH = HP - NI;                 // halo points
  static constexpr int THREADS = ((NI + NH + 31) / 32) * 32;
  // interior point i -> halo-tile index
  __device__ static int interior_h(int i) { return (i / TX + (HASY ? 1 : 0)) * HX + (i % TX + 1); }
  // halo point h -> halo-tile coordinates
  __device__ static void halo_xy(int h, int& hx, int& hy) {
    if (!HASY) { hx = (h == 0) ? 0 : HX - 1; hy = 0; return; }
    if (h < HX) { hx = h; hy = 0; return; }
    h -= HX;
    if (h < HX) { hx = h; hy = HY - 1; return; }
    h -= HX;
    if (h < TY) { hx = 0; hy = 1 + h; return; }
    h -= TY;
    hx = HX - 1;
    hy = 1 + h;
  }
};

struct FusedArgs {
  Stencil st;          // 3-D view (1-D / 2-D mapped to nx x 1 x nz)
  Basis V;             // V(:,1..k) (raw, scales ds.alpha)
  int k;               // step being finished; 0 = cycle-start pass (u = src, no update)
  int nA;
  const double* src;   // w~_k (raw, scale ds.alpha[k-1]); k = 0: V_1 raw (R_bar)
  double* dstx;        // u -> ring P_x slot of step k+1 (unused when k = 0)
  double* dsty;        // w~ -> ring P_y slot of step k+1
  double* slot_scale;  // per-slot probe scale
  int dst_slot;
  int zchunk;          // planes per block along the march axis
  DevState ds;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int KIND, int TX, int TY, int KMAX>
__global__ void __launch_bounds__(Tile<TX, TY>::THREADS, (KMAX <= 16 ? 2 : 1)) fused_arnoldi_kernel(FusedArgs a) {
  using T = Tile<TX, TY>;
  constexpr int HX = T::HX, HP = T::HP, NI = T::NI, NH = T::NH, NT = T::THREADS;
  constexpr int YOFF = T::HASY ? HX : 0;             // halo-tile stride of a y step
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr int NW = NT / 32;
  constexpr int JPW = (KMAX + NW - 1) / NW;  // basis vectors per warp in the dot phase
  extern __shared__ double smem[];
  double* Up = smem;                 // [3][HP]  u planes (ring)
  double* Kp = Up + 3 * HP;          // [3][HP]  kappa planes (cell kinds)
  double* Wt = Kp + 3 * HP;          // [NI]     w~ of the previous plane (interior)
  double* Vsave = Wt + NI;           // [KMAX][NI] V_j of the previous plane (interior)
  __shared__ double hs[KMAX];
  __shared__ const double* colp[KMAX];   // V(:,j) base pointers (ring slots resolved once)
  __shared__ double accs[2 * KMAX + 2];
  __shared__ double red[NW][2];
  __shared__ double tot[2 * KMAX + 2];
  __shared__ bool s_last;

  const Stencil& st = a.st;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int k = a.k;
  const int ld = a.nA + 1;
  if (t < k) hs[t] = a.ds.H[(int64_t)(k - 1) * ld + t] * a.ds.alpha[t];
  if (t < KMAX) colp[t] = (t < k) ? a.V.col(t) : a.src;
  const double wsc = (k >= 1) ? a.ds.alpha[k - 1] : 1.0;
  __syncthreads();

  // tile position
  const int64_t tiles_x = (st.nx + TX - 1) / TX;
  const int64_t tiles_y = (st.ny + TY - 1) / TY;
  int64_t b = blockIdx.x;
  const int64_t tx_i = b % tiles_x;
  b /= tiles_x;
  const int64_t ty_i = b % tiles_y;
  const int64_t zc_i = b / tiles_y;
  const int64_t x0 = tx_i * TX, y0 = ty_i * TY;
  const int64_t z0 = zc_i * a.zchunk;
  const int64_t z1 = (z0 + a.zchunk < st.nz) ? z0 + a.zchunk : st.nz;

  // this thread's point: interior (t < NI) or halo (NI <= t < NI + NH)
  const bool interior = t < NI;
  const bool active = t < NI + NH;
  int hx = 0, hy = 0, hidx = 0;
  if (interior) {
    hidx = T::interior_h(t);
    hx = t % TX + 1;
    hy = t / TX + (T::HASY ? 1 : 0);
  } else if (active) {
    T::halo_xy(t - NI, hx, hy);
    hidx = hy * HX + hx;
  }
  const int64_t gx = x0 - 1 + hx, gy = y0 + hy - (T::HASY ? 1 : 0);
  const bool in_grid = active && gx >= 0 && gx < st.nx && gy >= 0 && gy < st.ny;
  const int64_t gcol = gx + st.nx * gy;   // index within a plane

  double nu = 0.0, tu = 0.0;          // u'u and u'w~ over this thread's interior points
  double at[JPW], al[JPW];            // t_j and l_j partials for the warp's basis vectors
#pragma unroll
  for (int q = 0; q < JPW; ++q) { at[q] = 0.0; al[q] = 0.0; }
  const int64_t plane = st.nx * st.ny;

  const int64_t p_begin = (z0 > 0) ? z0 - 1 : 0;
  for (int64_t p = p_begin; p <= z1; ++p) {
    const bool have_p = p < st.nz;               // U(p) exists (else Dirichlet 0 beyond the grid)
    const int slot = (int)(p % 3);
    double vr[KMAX];
    // ---- U(p) at this thread's point: every load of the plane issued together ----
    if (have_p && active) {
      double u = 0.0;
      if (in_grid) {
        const int64_t g = gcol + plane * p;
        const double s0 = __ldg(a.src + g);
        if (cell) Kp[slot * HP + hidx] = __ldg(st.field + g);
        if (k == 0) {
          u = s0;
        } else {
#pragma unroll
          for (int j = 0; j < KMAX; ++j) vr[j] = (j < k) ? __ldg(colp[j] + g) : 0.0;
          u = wsc * s0;
#pragma unroll
          for (int j = 0; j < KMAX; ++j)
            if (j < k) u = fma(-hs[j], vr[j], u);
        }
        if (interior && p >= z0 && p < z1) {
          if (k > 0) a.dstx[g] = u;
          nu = fma(u, u, nu);
        }
      }
      Up[slot * HP + hidx] = u;
    }
    __syncthreads();
    // ---- w~ = A u on plane q = p-1 ----
    const int64_t q = p - 1;
    const bool do_q = (q >= z0) && (q < z1);
    if (do_q && interior) {
      const int qs = (int)(q % 3);
      double w = 0.0;
      if (in_grid) {
        const double* Uq = Up + qs * HP;
        const double* Kq = Kp + qs * HP;
        const double xc = Uq[hidx];
        const double fc = cell ? Kq[hidx] : 0.0;
        double acc = 0.0;
        auto face = [&](double xn, double fn, bool inside, double s) {
          const double kf = cell ? (inside ? 0.5 * (fc + fn) : fc) : 1.0;
          acc = fma(s * kf, xc - xn, acc);
        };
        {  // x neighbours
          const bool inw = gx > 0, ine = gx + 1 < st.nx;
          const double xw = Uq[hidx - 1], xe = Uq[hidx + 1];
          face(xw, cell ? Kq[hidx - 1] : 0.0, inw, st.s[0]);
          face(xe, cell ? Kq[hidx + 1] : 0.0, ine, st.s[0]);
          if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[0], xc - xw, acc);
        }
        if (T::HASY) {  // y neighbours
          const bool ins = gy > 0, inn = gy + 1 < st.ny;
          const double xs = Uq[hidx - YOFF], xn = Uq[hidx + YOFF];
          face(xs, cell ? Kq[hidx - YOFF] : 0.0, ins, st.s[1]);
          face(xn, cell ? Kq[hidx + YOFF] : 0.0, inn, st.s[1]);
          if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[1], xc - xs, acc);
        }
        if (st.nz > 1) {  // z neighbours (the march axis)
          const bool inb = q > 0, int_ = q + 1 < st.nz;
          const int sb = (int)((q + 2) % 3), stp = (int)((q + 1) % 3);
          const double xb = inb ? Up[sb * HP + hidx] : 0.0;
          const double xt = int_ ? Up[stp * HP + hidx] : 0.0;
          face(xb, cell && inb ? Kp[sb * HP + hidx] : 0.0, inb, st.s[2]);
          face(xt, cell && int_ ? Kp[stp * HP + hidx] : 0.0, int_, st.s[2]);
          if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[2], xc - xb, acc);
        }
        w = xc + acc;
        a.dsty[gcol + plane * q] = w;
        tu = fma(xc, w, tu);
      }
      Wt[t] = w;
    }
    __syncthreads();
    // ---- dots of plane q against V_j(q) (parked in Vsave one plane ago) ----
    if (do_q && k > 0) {
      const double* Uq = Up + (int)(q % 3) * HP;
#pragma unroll
      for (int jj = 0; jj < JPW; ++jj) {
        const int j = warp + NW * jj;
        if (j < k) {
          const double* vs = Vsave + (int64_t)j * NI;
          double s1 = 0.0, s2 = 0.0;
          for (int pt = lane; pt < NI; pt += 32) {
            const double v = vs[pt];
            s1 = fma(v, Wt[pt], s1);
            s2 = fma(v, Uq[T::interior_h(pt)], s2);
          }
          at[jj] += s1;
          al[jj] += s2;
        }
      }
    }
    __syncthreads();
    // ---- park V_j(p) for the next plane's dots ----
    if (have_p && k > 0 && interior && p >= z0 && p < z1) {
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < k) Vsave[(int64_t)j * NI + t] = in_grid ? vr[j] : 0.0;
    }
  }

  // ---- block reduction: [t_0..t_{k-1}, l_0..l_{k-1}, t_u, nu] ----
#pragma unroll
  for (int jj = 0; jj < JPW; ++jj) {
    const int j = warp + NW * jj;
    const double s1 = warp_sum(at[jj]);
    const double s2 = warp_sum(al[jj]);
    if (lane == 0 && j < k) {
      accs[j] = s1;
      accs[KMAX + j] = s2;
    }
  }
  nu = warp_sum(nu);
  tu = warp_sum(tu);
  if (lane == 0) {
    red[warp][0] = tu;
    red[warp][1] = nu;
  }
  __syncthreads();
  const int nv = 2 * k + 2;
  const int nb = gridDim.x;
  if (t == 0) {
    double s_tu = 0.0, s_nu = 0.0;
    for (int w = 0; w < NW; ++w) {
      s_tu += red[w][0];
      s_nu += red[w][1];
    }
    accs[2 * KMAX] = s_tu;
    accs[2 * KMAX + 1] = s_nu;
  }
  __syncthreads();
  for (int v = t; v < nv; v += NT) {
    const double val = (v < k) ? accs[v] : (v < 2 * k ? accs[KMAX + v - k] : accs[2 * KMAX + (v - 2 * k)]);
    a.ds.partials[(int64_t)v * nb + blockIdx.x] = val;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    const unsigned tk = atomicAdd(a.ds.tickets + TK_MAIN, 1u);
    s_last = (tk == (unsigned)nb - 1);
    if (s_last) a.ds.tickets[TK_MAIN] = 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // totals in a fixed order (one warp per value)
  for (int v = warp; v < nv; v += NW) {
    double s = 0.0;
    for (int bb = lane; bb < nb; bb += 32) s += ((volatile double*)a.ds.partials)[(int64_t)v * nb + bb];
    s = warp_sum(s);
    if (lane == 0) tot[v] = s;
  }
  __syncthreads();
  if (t != 0) return;
  DevState& ds = a.ds;
  const int ldl = a.nA + 1;
  const double t_u = tot[2 * k], s_nu = tot[2 * k + 1];
  double an;  // alpha of u = V_{k+1}
  if (k >= 1) {
    ds.H[(int64_t)(k - 1) * ld + k] = sqrt(s_nu);  // l.17: H(k+1,k) = ||U_k||
    givens_update(ds, k, a.nA);                    // l.19-32, sets alpha[k] (0 on breakdown)
    an = ds.alpha[k];
  } else {
    an = ds.alpha[0];                              // 1/beta from the residual kernel (l.6)
  }
  a.slot_scale[a.dst_slot] = an;
  if (k >= a.nA) return;
  // MGS coefficients of step k+1 (column index k): (I + L) h = s (R11)
  double* Lrow = ds.Lm + (int64_t)k * ldl;
  for (int j = 0; j < k; ++j) Lrow[j] = ds.alpha[j] * an * tot[k + j];
  double* Hc = ds.H + (int64_t)k * ld;
  for (int j = 0; j <= k; ++j) {
    double h = (j < k) ? ds.alpha[j] * an * tot[j] : an * an * t_u;
    const double* Lr = ds.Lm + (int64_t)j * ldl;
    for (int c = 0; c < j; ++c) h -= Lr[c] * Hc[c];
    Hc[j] = h;
  }
}

template <int TX, int TY>
int zchunk_for(const Stencil& st) {
  const int64_t tiles = ((st.nx + TX - 1) / TX) * ((st.ny + TY - 1) / TY);
  int64_t zc = tiles * st.nz / (148 * 8);   // ~8 waves of one block per SM
  if (zc > 128) zc = 128;
  if (zc < 8) zc = 8;
  if (zc > st.nz) zc = st.nz;
  return (int)zc;
}

template <int KIND, int TX, int TY, int KMAX>
void launch_t(FusedArgs a, cudaStream_t s) {
  using T = Tile<TX, TY>;
  const size_t smem = (size_t)(6 * T::HP + T::NI + (size_t)KMAX * T::NI) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fused_arnoldi_kernel<KIND, TX, TY, KMAX>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  a.zchunk = zchunk_for<TX, TY>(a.st);
  const int64_t tiles = ((a.st.nx + TX - 1) / TX) * ((a.st.ny + TY - 1) / TY) *
                        ((a.st.nz + a.zchunk - 1) / a.zchunk);
  fused_arnoldi_kernel<KIND, TX, TY, KMAX><<<(unsigned)tiles, T::THREADS, smem, s>>>(a);
}

template <int KIND, int TX, int TY>
void launch_k(const FusedArgs& a, cudaStream_t s) {
  if (a.k <= 8) launch_t<KIND, TX, TY, 8>(a, s);
  else if (a.k <= 16) launch_t<KIND, TX, TY, 16>(a, s);
  else launch_t<KIND, TX, TY, 32>(a, s);
}

template <int KIND>
void launch_kind(const FusedArgs& a, bool three_d, cudaStream_t s) {
  if (three_d) launch_k<KIND, 32, 8>(a, s);
  else launch_k<KIND, 256, 1>(a, s);
}

// 3-D view of the local grid for the fused pass: the march axis is the slowest one
Stencil march_view(const Stencil& st) {
  Stencil v = st;
  if (st.ndim == 1) {
    v.ny = 1;
    v.nz = 1;
    v.s[1] = v.s[2] = 0.0;
    v.a[1] = v.a[2] = 0.0;
  } else if (st.ndim == 2) {
    v.nz = st.ny;
    v.ny = 1;
    v.s[2] = st.s[1];
    v.a[2] = st.a[1];
    v.s[1] = 0.0;
    v.a[1] = 0.0;
  }
  return v;
}

}  // namespace

bool fused_supported(const Stencil& st, int k) {
  return st.kind != PSP_OP_DIA && k <= 32 && st.x_lo == nullptr && st.x_hi == nullptr;
}

void launch_fused(const Stencil& st0, Basis V, int k, int nA, const double* src, double* dstx,
                  double* dsty, double* slot_scale, int dst_slot, DevState ds, cudaStream_t s) {
  FusedArgs a;
  a.st = march_view(st0);
  a.V = V;
  a.k = k;
  a.nA = nA;
  a.src = src;
  a.dstx = dstx;
  a.dsty = dsty;
  a.slot_scale = slot_scale;
  a.dst_slot = dst_slot;
  a.zchunk = 1;
  a.ds = ds;
  const bool three_d = st0.ndim == 3;
  switch (st0.kind) {
    case PSP_OP_CONST_DIFF: launch_kind<PSP_OP_CONST_DIFF>(a, three_d, s); break;
    case PSP_OP_CELL_DIFF: launch_kind<PSP_OP_CELL_DIFF>(a, three_d, s); break;
    default: launch_kind<PSP_OP_CELL_ADVDIFF>(a, three_d, s); break;
  }
}

}  // namespace psp
