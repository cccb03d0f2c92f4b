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
// 8(2k+7) for separate matvec / dots / update passes.  Measured at 512^3 (tools/kstep.py):
// k <= 4 1.8 ms, k = 5..8 2.3-2.5, k = 9..12 2.9-3.2, k = 13..16 4.3-5.0 ms a pass; the split
// passes win from k = 17 (the two-threads-per-point tiles carry 1.6x halo work).
//
// Work layout: the compute threads of a block own a TX x TY tile of the (x, y) plane (3-D:
// 32 x 15, or 32 x 7 with two threads per point for k > 16; 2-D / 1-D: 256 x 1 or 224 x 1) and
// march a chunk of planes along the slowest axis.  Tiles overlap: threads on the tile edge
// compute u at their point (the stencil halo) but emit nothing, so no block ever waits for
// another (in x the tile starts two points before its interior: a TMA box's inner start must be
// 16-byte aligned).  One extra producer warp issues, per plane, a tensor-tile load
// (cp.async.bulk.tensor, 4-D map over the probe ring: x, y, plane, slot) for each of the k basis
// columns, for w~_k and for kappa into a ring of shared-memory stages (as many as fit: up to 12
// for narrow steps), completion on one `full` mbarrier per stage; out-of-grid boxes are
// zero-filled by the TMA unit, which is exactly the Dirichlet extension u = 0.  Per plane p the
// compute warps form u(p+1) from stage p+1 and publish it (with kappa) to a 4-plane ring, then
// w~(p) = A u(p) from u(p-1), u(p+1) in registers and the in-plane neighbours of plane p from
// the ring, and t_j = V_j(p)'w~(p).  For k <= 12 a thread's basis values of plane p+1 are kept
// in registers for those t_j, so stage p+1 goes back to the producer (an `empty` mbarrier
// arrival per warp) as soon as u(p+1) is formed: all stages but one are in flight.  There is no
// block-wide barrier in the plane loop: warps meet only on the u-ring mbarriers.
#include <cuda.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "givens.cuh"
#include "internal.h"

#ifndef PSP_FUSED_NSTMAX
#define PSP_FUSED_NSTMAX 12   // stage ring depth cap (narrow steps: many planes in flight)
#endif
#ifndef PSP_FUSED_UCH
#define PSP_FUSED_UCH 1       // independent FMA chains of the MGS update u (power of two)
#endif
#ifndef PSP_FUSED_SCH
#define PSP_FUSED_SCH 3       // stencil accumulators: 1 (one chain) or 3 (one per axis; 0-5 % faster)
#endif

namespace psp {
namespace {

struct FusedArgs {
  Stencil st;          // 3-D view (1-D / 2-D mapped to nx x 1 x nz)
  int k;               // step being finished; 0 = cycle-start pass (u = src, no update)
  int nA;
  int vs1, cap;        // V(:,j+1) = ring P_x slot (vs1 + j) % cap
  int src_slot;        // w~_k: ring P_y slot (k = 0: V_1 = ring P_x slot)
  int src_px;          // 1: src lives in the P_x ring; 2: src is a plain vector (map msrc)
  int jb;              // first basis column of this pass (split-column step: the columns [jb, k))
  int hyb;             // 1: split-column step -- src is u' (scale 1), sums go to ds.rpart
  const double* src_vec;  // src_px = 2
  double* dstx;        // u -> ring P_x slot of step k+1 (unused when k = 0)
  double* dsty;        // w~ -> ring P_y slot of step k+1
  double* slot_scale;  // per-slot probe scale
  int dst_slot;
  int zchunk;          // planes per tile along the march axis
  int zoff;            // multi-rank ghost-plane layout: plane p of a column is TMA plane p + zoff
  int lo_in, hi_in;    // the neighbour rank's planes exist below / above (ghost planes hold them)
  int64_t tiles_x, tiles_y, ntiles;
  DevState ds;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Transposing butterfly: v[0..7] per lane -> returns, in every lane l, the sum over the warp of
// v[l & 7] (9 double shuffles for 8 values).
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

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
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
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  }
}
// 4-D tensor tile (x, y, plane, slot) -> shared memory, completion on bar
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* map, int x, int y, int z, int sl, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(sl), "r"(su32(bar))
      : "memory");
}

template <int TX, int TY, int KMAX, int CS, int PP = 1>
struct FCfg {
  static constexpr int NT = TX * TY;
  static constexpr int NUB = 4;                              // u (and kappa) plane ring depth
  // RV: a plane's basis values are held in registers from its u to its t_j products, so its stage
  // is released as soon as u is formed (all but one stage in flight; the plane's kappa moves to
  // a kappa plane ring beside the u ring); wider thread column sets (KJ = 16) do not fit the
  // 128-register budget and keep the stage for the t_j and the stencil's kappa instead
  // (blocks of <= 288 threads have up to 224 registers a thread: room for 30 held values)
  static constexpr bool RV = KMAX / CS <= 12 || (KMAX / CS <= 16 && NT * CS / PP + 32 <= 384) ||
                             NT * CS / PP + 32 <= 288;
  static constexpr int NB = KMAX + 2;                        // boxes per stage: V_0..V_{KMAX-1}, w~, kappa
  static constexpr int STAGE = NB * NT;                      // doubles
  static constexpr int RING = (RV ? 2 : 1) * NUB * NT;       // u (+ kappa) plane rings, doubles
  static constexpr int NSTF = (int)((225 * 1024 - RING * 8 - 256) / (STAGE * 8 + 16));
  static constexpr int NST = NSTF > PSP_FUSED_NSTMAX ? PSP_FUSED_NSTMAX : NSTF;
  static_assert(NST >= 3, "a stage ring needs two resident planes and one in flight");
  static constexpr size_t SMEM = (size_t)NST * STAGE * 8 + (size_t)RING * 8 + 16 * NST + 8 * NUB + 128;
};

// Half-warp transposing butterfly (CS = 2): v[0..7] per lane -> lane l holds the sum over the
// 16 lanes of its half-warp of v[l & 7] (the halves own different basis columns).
__device__ __forceinline__ double butterfly8_half(double (&v)[8], int lane) {
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
  return r;
}

// CS = 2 (the widest steps): two threads per point, each owning half of the basis columns (the
// two halves of a warp hold the same 16 points), so a 32 x 8 tile -- the largest whose stage
// ring fits shared memory at k = 32 -- still runs 16 compute warps per SM.  The halves' partial
// MGS updates meet by one shuffle; each half keeps the dot products of its own columns.
//
// Warp roles: NT*CS compute threads plus one producer warp.  The producer issues the TMA boxes
// of plane after plane into the stage ring as soon as the compute warps release a stage (one
// `empty` mbarrier arrival per compute warp), so no compute warp carries the issue and there is
// no block-wide barrier in the plane loop: the in-plane u values the stencil needs are published
// through a 4-deep ring of shared-memory planes, each with an mbarrier the compute warps arrive
// on when they have written it (4 deep: a warp overwriting a plane buffer has already seen
// every warp's write of the plane two after the one last read from it).
template <int KIND, int TX, int TY, int KMAX, int CS, int PP>
__global__ void __launch_bounds__(TX * TY * CS / PP + 32, 1)
    fused_tma_kernel(const __grid_constant__ CUtensorMap mpx, const __grid_constant__ CUtensorMap mpy,
                     const __grid_constant__ CUtensorMap mkap, const __grid_constant__ CUtensorMap msrc,
                     FusedArgs a) {
  using Cfg = FCfg<TX, TY, KMAX, CS, PP>;
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr bool HASY = TY > 1;
  constexpr int NT = Cfg::NT, NST = Cfg::NST;      // NT points per tile
  constexpr int NC = NT * CS / PP, NWC = NC / 32;   // compute threads / warps (PP points a thread)
  constexpr int PSTR = NT / PP;                     // a thread's points: pt, pt + PSTR, ...
  constexpr int NTH = NC + 32, NW = NWC + 1;        // + the producer warp
  constexpr int NUB = Cfg::NUB;
  constexpr int KJ = KMAX / CS;                     // basis columns per thread
  constexpr bool REG = KJ <= 16;           // per-thread accumulators (else per-plane butterflies)
  constexpr int NCH = (KJ + 7) / 8;
  constexpr int NACC = REG ? KJ : NCH;
  constexpr bool RV = Cfg::RV;
  static_assert(CS == 1 || CS == 2, "column split 1 or 2");
  static_assert(PP == 1 || (PP == 2 && CS == 1 && NT % 64 == 0), "two points a thread: CS = 1, whole warps");
  static_assert(NC % 32 == 0, "whole compute warps");
  extern __shared__ __align__(128) double fsm[];
  // 128-byte aligned stage base by index arithmetic on the shared array (stays in .shared)
  double* stages = fsm + (((128u - (su32(fsm) & 127u)) & 127u) >> 3);
  double* Us = stages + NST * Cfg::STAGE;    // [NUB][NT] u planes
  double* Ks = Us + NUB * NT;                // [NUB][NT] kappa planes (RV)
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + NST * Cfg::STAGE + Cfg::RING);
  uint64_t* empty = full + NST;
  uint64_t* ubar = empty + NST;
  __shared__ double hs[KMAX];
  __shared__ int vslot[KMAX];
  __shared__ double tot[2 * KMAX + 2];
  __shared__ bool s_last;

  const Stencil& st = a.st;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool producer = warp == NWC;
  // this thread's point and column half (the producer warp aliases points 0..31: unused)
  const int half = (CS == 2) ? (lane >> 4) : 0;
  const int pt = producer ? lane : ((CS == 2) ? warp * 16 + (lane & 15) : t);
  const int j0 = half * KJ;
  const int k = a.k;
  const int kc = k - a.jb;                       // basis columns of this pass
  const int ld = a.nA + 1;
  if (t < KMAX) {
    hs[t] = (t < kc) ? a.ds.H[(int64_t)(k - 1) * ld + a.jb + t] * a.ds.alpha[a.jb + t] : 0.0;
    vslot[t] = (a.vs1 + a.jb + t) % a.cap;
  }
  // columns j >= k are never loaded: zero them once in every stage (coefficient 0, product 0)
  if (!producer && half == 0)
    for (int s = 0; s < NST; ++s)
      for (int j = kc; j < KMAX; ++j)
        for (int i = 0; i < PP; ++i) stages[(size_t)s * Cfg::STAGE + j * NT + pt + i * PSTR] = 0.0;
  if (t == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, NWC);
    }
    for (int q = 0; q < NUB; ++q) mbar_init(ubar + q, NWC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mpx)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mpy)) : "memory");
    if (cell) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mkap)) : "memory");
  }
  const double wsc = (k >= 1 && !a.hyb) ? a.ds.alpha[k - 1] : 1.0;
  __syncthreads();
  // narrow steps: the (negated) MGS coefficients in registers, not re-read from shared memory
  // every plane
  constexpr bool HREG = KJ <= 8;
  double hr[HREG ? KJ : 1];
#pragma unroll
  for (int j = 0; j < (HREG ? KJ : 1); ++j) hr[j] = HREG ? -hs[j0 + j] : 0.0;

  const int nload = (k == 0 ? 0 : kc) + 1 + (cell ? 1 : 0);
  const unsigned stage_bytes = (unsigned)(nload * NT * 8);

  double accl[NACC], acct[NACC];
#pragma unroll
  for (int c = 0; c < NACC; ++c) { accl[c] = 0.0; acct[c] = 0.0; }
  double nu = 0.0, tu = 0.0;

  if (producer) {
    // ---- producer: planes z0-1 .. z1 of every tile, in the order the compute warps take them ----
    uint32_t gs = 0;                             // running stage count (slot gs % NST)
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
      int64_t b = tile;
      const int64_t txi = b % a.tiles_x;
      b /= a.tiles_x;
      const int64_t tyi = b % a.tiles_y;
      const int64_t zci = b / a.tiles_y;
      const int x0 = (int)(txi * (TX - 4)) - 2, y0 = HASY ? (int)(tyi * (TY - 2)) - 1 : 0;
      const int64_t z0 = zci * a.zchunk;
      const int64_t z1 = (z0 + a.zchunk < st.nz) ? z0 + a.zchunk : st.nz;
      for (int64_t q = z0 - 1; q <= z1; ++q, ++gs) {
        const int si = (int)(gs % NST);
        // the slot's previous plane released by every compute warp (fresh barrier: passes)
        mbar_wait(empty + si, ((gs / NST) & 1u) ^ 1u);
        double* sb = stages + (size_t)si * Cfg::STAGE;
        const int zq = (int)q;                   // may be -1 or nz: zero-filled by the TMA unit
        if (lane == 0) mbar_expect_tx(full + si, stage_bytes);
        __syncwarp();
        for (int j = lane; j < nload; j += 32) {
          const int zt = zq + a.zoff;            // (the ghost planes of the multi-rank layout)
          if (j < (k > 0 ? kc : 0)) tma4(sb + j * NT, &mpx, x0, y0, zt, vslot[j], full + si);
          else if (j == (k > 0 ? kc : 0))
            tma4(sb + KMAX * NT, a.src_px == 2 ? &msrc : (a.src_px ? &mpx : &mpy), x0, y0, zt, a.src_slot, full + si);
          else tma4(sb + (KMAX + 1) * NT, &mkap, x0, y0, zt, 0, full + si);
        }
      }
    }
  } else {
    // ---- compute warps ----
    const double hsx = 0.5 * st.s[0], hsy = 0.5 * st.s[1], hsz = 0.5 * st.s[2];
    const int64_t plane = st.nx * st.ny;
    uint32_t gs = 0;                             // running stage count, as the producer's
    uint32_t us = 0;                             // running u-plane count (ring slot us % NUB)

    // products of this thread's columns with f (f = 0 for points that are not counted)
    auto add_products = [&](const double* vcol /* stage base; column j at j*NT */, int q, double f,
                            double (&acc)[NACC]) {
      if (REG) {
#pragma unroll
        for (int j = 0; j < KJ; ++j) acc[j] = fma(vcol[(j0 + j) * NT + q], f, acc[j]);
      } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c * 8 >= kc) break;                  // uniform
          double v8[8];
#pragma unroll
          for (int qq = 0; qq < 8; ++qq) v8[qq] = vcol[(j0 + c * 8 + qq) * NT + q] * f;
          acc[c] += (CS == 2) ? butterfly8_half(v8, lane) : butterfly8(v8, lane);
        }
      }
    };
    auto acquire = [&](uint32_t g) -> const double* {     // stage g's plane has landed
      const int si = (int)(g % NST);
      mbar_wait(full + si, (g / NST) & 1u);
      return stages + (size_t)si * Cfg::STAGE;
    };
    auto release = [&](uint32_t g) {                      // this warp is done with stage g
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + (g % NST))) : "memory");
    };
    auto publish_u = [&](uint32_t g, const double (&v)[PP], const double (&kv)[PP]) {  // u (+ kappa) of plane g
      if (half == 0) {
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          Us[(g % NUB) * NT + pt + i * PSTR] = v[i];
          if (RV && cell) Ks[(g % NUB) * NT + pt + i * PSTR] = kv[i];
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(ubar + (g % NUB))) : "memory");
    };
    auto await_u = [&](uint32_t g) -> const double* {    // every warp has published plane g
      mbar_wait(ubar + (g % NUB), (g / NUB) & 1u);
      return Us + (g % NUB) * NT;
    };

    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
      int64_t b = tile;
      const int64_t txi = b % a.tiles_x;
      b /= a.tiles_x;
      const int64_t tyi = b % a.tiles_y;
      const int64_t zci = b / a.tiles_y;
      // the box's inner start must be 16-byte aligned: x0 even, halo lanes 1 and TX-2
      const int x0 = (int)(txi * (TX - 4)) - 2, y0 = HASY ? (int)(tyi * (TY - 2)) - 1 : 0;
      const int64_t z0 = zci * a.zchunk;
      const int64_t z1 = (z0 + a.zchunk < st.nz) ? z0 + a.zchunk : st.nz;
      // this thread's points
      int ptv[PP];
      bool in_grid[PP], own[PP], emit[PP], nb_w[PP], nb_e[PP], nb_s[PP], nb_n[PP];
      int64_t col[PP];
#pragma unroll
      for (int i = 0; i < PP; ++i) {
        ptv[i] = pt + i * PSTR;
        const int lxi = ptv[i] % TX, lyi = ptv[i] / TX;
        const int64_t gx = x0 + lxi, gy = y0 + lyi;
        const bool interior = lxi >= 2 && lxi <= TX - 3 && (!HASY || (lyi >= 1 && lyi <= TY - 2));
        in_grid[i] = gx >= 0 && gx < st.nx && gy >= 0 && gy < st.ny;
        own[i] = interior && in_grid[i];
        emit[i] = own[i] && half == 0;           // stores and the u / w~ scalars: one thread per point
        col[i] = in_grid[i] ? gx + st.nx * gy : 0;
        nb_w[i] = gx > 0;
        nb_e[i] = gx + 1 < st.nx;
        nb_s[i] = gy > 0;
        nb_n[i] = gy + 1 < st.ny;
      }

      // u at point q of the staged plane (MGS update of step k, ICWY form)
      auto form_u = [&](const double* sb, int q) -> double {
        const double s0 = sb[KMAX * NT + q];
        if (k == 0) return s0;
        // UCH independent FMA chains (the k-long chain of one accumulator is the pass's critical
        // path: ncu "wait" stalls on the dependent DFMAs, r02_ncu/fused_k10)
        constexpr int UC = (KJ >= 2 * PSP_FUSED_UCH) ? PSP_FUSED_UCH : 1;
        double uu[UC];
        uu[0] = (half == 0) ? wsc * s0 : 0.0;
#pragma unroll
        for (int c = 1; c < UC; ++c) uu[c] = 0.0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) uu[j % UC] = fma(HREG ? hr[j] : -hs[j0 + j], sb[(j0 + j) * NT + q], uu[j % UC]);
#pragma unroll
        for (int w = 1; w < UC; w <<= 1)
#pragma unroll
          for (int c = 0; c + w < UC; c += 2 * w) uu[c] += uu[c + w];
        double u = uu[0];
        if (CS == 2) {                           // the halves' partial updates, same sum on both
          const double o = __shfl_xor_sync(0xffffffffu, u, 16);
          u = (half == 0) ? u + o : o + u;
        }
        return u;
      };
      // this thread's basis values of a staged plane -> registers (the plane's l_j products now,
      // its t_j products one plane later, after which the stage is long released)
      auto load_vr = [&](const double* sb, int q, double (&vr)[KJ]) {
#pragma unroll
        for (int j = 0; j < KJ; ++j) vr[j] = sb[(j0 + j) * NT + q];
      };
      auto add_products_r = [&](const double (&vr)[KJ], double f, double (&acc)[NACC]) {
        if (REG) {
#pragma unroll
          for (int j = 0; j < KJ; ++j) acc[j] = fma(vr[j], f, acc[j]);
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (c * 8 >= kc) break;              // uniform
            double v8[8];
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) v8[qq] = vr[c * 8 + qq] * f;
            acc[c] += (CS == 2) ? butterfly8_half(v8, lane) : butterfly8(v8, lane);
          }
        }
      };
      // prologue: u(z0-1) (stage released at once), u(z0) (+ l-products of plane z0)
      double vr[PP][KJ];
      double ub[PP], kb[PP], uc[PP], kc_[PP];
      double* ox[PP];
      double* oy[PP];
      const uint32_t gb = gs;                    // stage count of plane z0-1
      const double* sbm = acquire(gb);
#pragma unroll
      for (int i = 0; i < PP; ++i) {
        ub[i] = form_u(sbm, ptv[i]);
        kb[i] = cell ? sbm[(KMAX + 1) * NT + ptv[i]] : 0.0;
        if (!((z0 >= 1 || a.lo_in) && in_grid[i])) ub[i] = 0.0;
      }
      release(gb);
      const double* sbc = acquire(gb + 1);
#pragma unroll
      for (int i = 0; i < PP; ++i) {
        const int64_t g = col[i] + plane * z0;   // this point's index at plane z0
        ox[i] = a.dstx + g;
        oy[i] = a.dsty + g;
        uc[i] = form_u(sbc, ptv[i]);
        if (!in_grid[i]) uc[i] = 0.0;
        kc_[i] = cell ? sbc[(KMAX + 1) * NT + ptv[i]] : 0.0;
      }
      const uint32_t ub0 = us;                   // u-plane count of plane z0
      publish_u(ub0, uc, kc_);
#pragma unroll
      for (int i = 0; i < PP; ++i) {
        if (RV && k > 0) load_vr(sbc, ptv[i], vr[i]);
        if (emit[i] && k > 0) *ox[i] = uc[i];
        const double f = own[i] ? uc[i] : 0.0;
        if (half == 0) nu = fma(f, f, nu);
        if (k > 0) {
          if (RV) add_products_r(vr[i], f, accl);
          else add_products(sbc, ptv[i], f, accl);
        }
      }
      if (RV) release(gb + 1);

      for (int64_t p = z0; p < z1; ++p) {
        const uint32_t gp = gb + 1 + (uint32_t)(p - z0);   // stage of plane p
        const uint32_t up = ub0 + (uint32_t)(p - z0);      // u plane of p
        const int64_t pn = p + 1;
        // u(p+1) from stage p+1 (plane z1, the halo above the chunk, is staged too)
        const double* sn = acquire(gp + 1);
        double un[PP], kt[PP];
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          un[i] = form_u(sn, ptv[i]);
          if (!((pn < st.nz || a.hi_in) && in_grid[i])) un[i] = 0.0;
          kt[i] = cell ? sn[(KMAX + 1) * NT + ptv[i]] : 0.0;
        }
        if (pn < z1) publish_u(up + 1, un, kt);  // the stencil of plane p+1 needs them
        // w~ = A u at plane p (both halves compute it; the first one stores it)
        const double* Up = await_u(up);
        const double* Kp = RV ? Ks + (up % NUB) * NT : stages + (size_t)(gp % NST) * Cfg::STAGE + (KMAX + 1) * NT;
        double w[PP];
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          w[i] = 0.0;
          if (own[i]) {
            const int q = ptv[i];
            const double c0 = uc[i], kci = kc_[i];
            // SCH = 3: one accumulator per axis (three short chains), else one chain over the faces
            double acc3[3] = {0.0, 0.0, 0.0};
            constexpr int AY = PSP_FUSED_SCH >= 3 ? 1 : 0, AZ = PSP_FUSED_SCH >= 3 ? 2 : 0;
            // a neighbour outside the grid holds u = 0 (TMA zero fill), and its face takes
            // (s/2)(k_c + k_c) = s k_c exactly: only kappa needs the select
            auto face = [&](double& acc, double xn, double fn, bool nin, double s, double hsv) {
              const double kf = cell ? hsv * (kci + (nin ? fn : kci)) : s;
              acc = fma(kf, c0 - xn, acc);
            };
            const double xw = Up[q - 1], xe = Up[q + 1];
            face(acc3[0], xw, cell ? Kp[q - 1] : 0.0, nb_w[i], st.s[0], hsx);
            face(acc3[0], xe, cell ? Kp[q + 1] : 0.0, nb_e[i], st.s[0], hsx);
            if (KIND == PSP_OP_CELL_ADVDIFF) acc3[0] = fma(st.a[0], c0 - xw, acc3[0]);
            if (HASY) {
              const double xs_ = Up[q - TX], xn_ = Up[q + TX];
              face(acc3[AY], xs_, cell ? Kp[q - TX] : 0.0, nb_s[i], st.s[1], hsy);
              face(acc3[AY], xn_, cell ? Kp[q + TX] : 0.0, nb_n[i], st.s[1], hsy);
              if (KIND == PSP_OP_CELL_ADVDIFF) acc3[AY] = fma(st.a[1], c0 - xs_, acc3[AY]);
            }
            {
              // march-axis faces, also for a single-plane march axis (nz = 1): the Dirichlet
              // faces then hold u = 0 (ub / un are 0 off the grid), as in stencil.cu; the 1-D
              // view has s[2] = a[2] = 0, so the faces vanish there
              const bool inb = p > 0 || a.lo_in, int_ = p + 1 < st.nz || a.hi_in;
              face(acc3[AZ], ub[i], kb[i], inb, st.s[2], hsz);
              face(acc3[AZ], un[i], kt[i], int_, st.s[2], hsz);
              if (KIND == PSP_OP_CELL_ADVDIFF) acc3[AZ] = fma(st.a[2], c0 - ub[i], acc3[AZ]);
            }
            const double acc = PSP_FUSED_SCH >= 3 ? (acc3[0] + acc3[1]) + acc3[2] : acc3[0];
            w[i] = c0 + acc;
            if (half == 0) {
              *oy[i] = w[i];
              tu = fma(c0, w[i], tu);
            }
          }
        }
        // t_j = V_j(p)' w~(p); w = 0 off emitted points
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          if (k > 0) {
            if (RV) add_products_r(vr[i], w[i], acct);
            else add_products(stages + (size_t)(gp % NST) * Cfg::STAGE, ptv[i], w[i], acct);
          }
        }
        if (!RV) release(gp);                     // stage p done
        if (pn < z1) {
#pragma unroll
          for (int i = 0; i < PP; ++i) {
            if (RV && k > 0) load_vr(sn, ptv[i], vr[i]);   // V(p+1): its l_j now, its t_j next plane
            if (emit[i] && k > 0) ox[i][plane] = un[i];
            const double f = own[i] ? un[i] : 0.0;
            if (half == 0) nu = fma(f, f, nu);
            if (k > 0) {
              if (RV) add_products_r(vr[i], f, accl);
              else add_products(sn, ptv[i], f, accl);
            }
          }
        }
        if (RV || pn == z1) release(gp + 1);      // stage p+1 done (else: after its t_j)
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          ub[i] = uc[i]; uc[i] = un[i];
          kb[i] = kc_[i]; kc_[i] = kt[i];
          ox[i] += plane;
          oy[i] += plane;
        }
      }
      gs = gb + (uint32_t)(z1 - z0 + 2);          // planes z0-1 .. z1
      us = ub0 + (uint32_t)(z1 - z0);             // u planes z0 .. z1-1
    }
  }

  // reduce the accumulators across the points of the warp (value -> slot j0 + j)
  double outl[NCH], outt[NCH];
  if (REG) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      double v8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v8[q] = (c * 8 + q < NACC) ? accl[c * 8 + q] : 0.0;
      outl[c] = (CS == 2) ? butterfly8_half(v8, lane) : butterfly8(v8, lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) v8[q] = (c * 8 + q < NACC) ? acct[c * 8 + q] : 0.0;
      outt[c] = (CS == 2) ? butterfly8_half(v8, lane) : butterfly8(v8, lane);
    }
  } else {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      outl[c] = accl[c];
      outt[c] = acct[c];
    }
  }
  // ---- block reduction: [t_0..t_{k-1}, l_0..l_{k-1}, t_u, nu]; the stages are free now ----
  __syncthreads();
  double* accs = stages;                          // [NW][2 KMAX + 2]
  constexpr int AW = 2 * KMAX + 2;
  if ((lane & 15) < 8 && (CS == 2 || lane < 8)) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int j = j0 + c * 8 + (lane & 7);
      if (c * 8 + (lane & 7) < KJ) {
        accs[warp * AW + j] = outt[c];
        accs[warp * AW + KMAX + j] = outl[c];
      }
    }
  }
  nu = warp_sum(nu);
  tu = warp_sum(tu);
  if (lane == 0) {
    accs[warp * AW + 2 * KMAX] = tu;
    accs[warp * AW + 2 * KMAX + 1] = nu;
  }
  __syncthreads();
  const int nv = 2 * kc + 2;
  const int nb = gridDim.x;
  for (int v = t; v < nv; v += NTH) {
    const int src = (v < kc) ? v : (v < 2 * kc ? KMAX + v - kc : 2 * KMAX + (v - 2 * kc));
    double sum = 0.0;
    for (int w2 = 0; w2 < NW; ++w2) sum += accs[w2 * AW + src];
    a.ds.partials[(int64_t)v * nb + blockIdx.x] = sum;
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
  for (int v = warp; v < nv; v += NW) {          // totals in a fixed order (one warp per value)
    double sum = 0.0;
    for (int bb = lane; bb < nb; bb += 32) sum += ((volatile double*)a.ds.partials)[(int64_t)v * nb + bb];
    sum = warp_sum(sum);
    if (lane == 0) tot[v] = sum;
  }
  __syncthreads();
  if (a.hyb) {                                    // the dots pass that follows finishes the step
    for (int v = t; v < nv; v += NTH) a.ds.rpart[kHybOff + v] = tot[v];
    return;
  }
  if (a.ds.multi) {                               // every rank's totals are all-reduced first,
    for (int v = t; v < nv; v += NTH) a.ds.rpart[v] = tot[v];   // then EPI_FUSED (fused_tail)
    return;
  }
  if (t != 0) return;
  fused_tail(a.ds, k, a.nA, tot, a.slot_scale, a.dst_slot);
}

// ---- tensor maps (driver entry point fetched through the runtime: no -lcuda) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// launch_fused error codes: > 0 a CUresult of cuTensorMapEncodeTiled, else one of these
constexpr int kErrNoEncode = -1;   // the driver entry point cuTensorMapEncodeTiled is unavailable
constexpr int kErrLaunch = -2;     // cudaFuncSetAttribute / cudaLaunchKernelEx failed (cudaGetLastError)

// 4-D map (x, y, plane, slot) over nslots columns of n doubles at base; box TX x TY x 1 x 1
thread_local int g_map_err = 0;   // last cuTensorMapEncodeTiled result (diagnostics)
// ld: slot stride (doubles); nzx: planes per column (nz, or nz + 2 with the ghost planes)
bool make_map(CUtensorMap* m, const double* base, const Stencil& st, int nslots, int TX, int TY, int64_t ld,
              int64_t nzx) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) { g_map_err = -1; return false; }
  cuuint64_t dims[4] = {(cuuint64_t)st.nx, (cuuint64_t)st.ny, (cuuint64_t)nzx, (cuuint64_t)nslots};
  cuuint64_t strides[3] = {(cuuint64_t)st.nx * 8, (cuuint64_t)(st.nx * st.ny) * 8, (cuuint64_t)ld * 8};
  cuuint32_t box[4] = {(cuuint32_t)TX, (cuuint32_t)TY, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  g_map_err = (int)r;
  return r == CUDA_SUCCESS;
}

struct MapCache {
  const double* px = nullptr;
  const double* py = nullptr;
  const double* field = nullptr;
  int64_t nx = 0, ny = 0, nz = 0, ld = 0;
  int cap = 0, tx = 0, ty = 0, zoff = 0;
  const double* src = nullptr;
  CUtensorMap mpx, mpy, mk, ms;
  bool ok = false;
};

// ring_px / ring_py / field / src_vec: the column STARTS (the ghost plane when zoff = 1)
template <int KIND, int TX, int TY, int KMAX, int CS, int PP = 1>
int launch_t(FusedArgs a, const double* ring_px, const double* ring_py, const double* field, int64_t ld,
             cudaStream_t s) {
  using Cfg = FCfg<TX, TY, KMAX, CS, PP>;
  // per host thread and device: the maps encode this device's pointers, the attribute is a
  // property of this device's context
  thread_local MapCache mcs[kMaxDev];
  thread_local bool attr[kMaxDev] = {};
  const int dev = device_ordinal();
  MapCache& mc = mcs[dev];
  const Stencil& st = a.st;
  const int64_t nzx = st.nz + 2 * a.zoff;
  if (!mc.ok || mc.px != ring_px || mc.py != ring_py || mc.field != field || mc.nx != st.nx ||
      mc.ny != st.ny || mc.nz != st.nz || mc.cap != a.cap || mc.ld != ld || mc.zoff != a.zoff) {
    mc.ok = make_map(&mc.mpx, ring_px, st, a.cap, TX, TY, ld, nzx) && make_map(&mc.mpy, ring_py, st, a.cap, TX, TY, ld, nzx) &&
            (field == nullptr || make_map(&mc.mk, field, st, 1, TX, TY, ld, nzx));
    if (field == nullptr) mc.mk = mc.mpx;
    mc.px = ring_px; mc.py = ring_py; mc.field = field;
    mc.src = nullptr;
    mc.nx = st.nx; mc.ny = st.ny; mc.nz = st.nz; mc.cap = a.cap; mc.ld = ld; mc.zoff = a.zoff;
  }
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(fused_tma_kernel<KIND, TX, TY, KMAX, CS, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Cfg::SMEM) != cudaSuccess)
      return kErrLaunch;
    attr[dev] = true;
  }
  a.tiles_x = (st.nx + (TX - 4) - 1) / (TX - 4);
  a.tiles_y = TY > 1 ? (st.ny + (TY - 2) - 1) / (TY - 2) : st.ny;
  const int64_t txy = a.tiles_x * a.tiles_y;
  const int sms = device_sms();
  int64_t zc = txy * st.nz / (sms * 4);            // about 4 tiles per SM
  if (zc > 64) zc = 64;
  if (zc < 8) zc = 8;
  const char* zce = getenv("PSP_FUSED_ZC");      // tuning knobs (read per launch: cheap next to a pass)
  const int zc_env = zce ? atoi(zce) : 0;
  if (zc_env > 0) zc = zc_env;
  if (zc > st.nz) zc = st.nz;
  a.zchunk = (int)zc;
  a.ntiles = txy * ((st.nz + zc - 1) / zc);
  if (!mc.ok) return g_map_err ? g_map_err : kErrNoEncode;
  if (a.src_px == 2 && mc.src != a.src_vec) {      // plain-vector source (split-column step)
    if (!make_map(&mc.ms, a.src_vec, st, 1, TX, TY, ld, nzx)) return g_map_err ? g_map_err : kErrNoEncode;
    mc.src = a.src_vec;
  }
  if (a.src_px != 2 && mc.src == nullptr) mc.ms = mc.mpx;
  auto kern = fused_tma_kernel<KIND, TX, TY, KMAX, CS, PP>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(TX * TY * CS / PP + 32);    // compute warps + the TMA producer warp
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  int64_t grid = sms;                              // one resident block per SM (persistent)
  if (grid > a.ntiles) grid = a.ntiles;
  cfg.gridDim = dim3((unsigned)grid);
  if (cudaLaunchKernelEx(&cfg, kern, mc.mpx, mc.mpy, mc.mk, mc.ms, a) != cudaSuccess) return kErrLaunch;
  return 0;
}

template <int KIND>
int launch_kind(const FusedArgs& a, bool three_d, const double* rpx, const double* rpy, const double* fld, int64_t ld,
                cudaStream_t s) {
  const int kc = a.k - a.jb;                       // basis columns of the pass
  if (three_d) {
    // stage = (KMAX + 2) boxes: the narrowest instantiation that holds k columns keeps the most
    // planes in flight (measured at 512^3: k <= 4 1.9 vs 2.3 ms, k = 9..12 3.5-3.8 vs 3.8-4.1 ms).
    // 32 x 8 tiles for k <= 16 or 16 x 8 tiles for k > 16 were slower (more halo points per tile).
    // k <= 8: two points a thread on the tallest tiles whose stage ring still holds three
    // stages (32 x 30 at KMAX 4, 32 x 22 at KMAX 8): less halo work per point, same warps
    // (k = 2: 2.1 -> 1.97 ms, k = 5..8: 2.8-2.9 -> 2.6 ms at 512^3)
    // Odd widths in between (KMAX 6 / 10 / 14): a pass computes KMAX columns (the ones past kc
    // are zero), so a step of width kc runs at most one idle column instead of up to three
    const bool coarse = getenv("PSP_FUSED_COARSE") != nullptr;   // A/B knob (read per launch): KMAX 4/8/12/16 only
    if (kc <= 4) return launch_t<KIND, 32, 30, 4, 1, 2>(a, rpx, rpy, fld, ld, s);
    if (kc <= 6 && !coarse) return launch_t<KIND, 32, 22, 6, 1, 2>(a, rpx, rpy, fld, ld, s);
    if (kc <= 8) return launch_t<KIND, 32, 22, 8, 1, 2>(a, rpx, rpy, fld, ld, s);
    if (kc <= 10 && !coarse) return launch_t<KIND, 32, 15, 10, 1>(a, rpx, rpy, fld, ld, s);
    if (kc <= 12) return launch_t<KIND, 32, 15, 12, 1>(a, rpx, rpy, fld, ld, s);
    if (kc <= 14 && !coarse) return launch_t<KIND, 32, 14, 14, 1, 2>(a, rpx, rpy, fld, ld, s);
    // k = 13..16: 32 x 14 tiles with two points a thread (8 compute warps, up to 255 registers)
    // hold a thread's 16 basis values per point in registers, so a stage is released as soon as
    // u is formed; one thread per point on 32 x 15 tiles would keep two stages resident, on
    // 32 x 11 tiles (12 warps, 168 registers) carries more halo (cycle ~1.5 % slower); two
    // points a thread for k <= 12 was slower (2.0 -> 2.6 ms at k = 2)
    if (kc <= 16) return launch_t<KIND, 32, 14, 16, 1, 2>(a, rpx, rpy, fld, ld, s);
    {
      const char* we = getenv("PSP_FUSED_WIDE");   // A/B knob: one thread per point for k > 16
      const int wide = we ? atoi(we) : 0;
      if (wide == 1 && kc <= 30) return launch_t<KIND, 32, 8, 30, 1>(a, rpx, rpy, fld, ld, s);
      if (wide == 2) return launch_t<KIND, 32, 6, 32, 1>(a, rpx, rpy, fld, ld, s);
    }
    if (kc <= 24) return launch_t<KIND, 32, 7, 24, 2>(a, rpx, rpy, fld, ld, s);
    return launch_t<KIND, 32, 7, 32, 2>(a, rpx, rpy, fld, ld, s);
  }
  {
    // 2-D / 1-D rows: KMAX 4 / 12 between 8 and 16 as in 3-D (at most three idle columns)
    const bool coarse = getenv("PSP_FUSED_COARSE") != nullptr;
    if (kc <= 4 && !coarse) return launch_t<KIND, 256, 1, 4, 1>(a, rpx, rpy, fld, ld, s);
    if (kc <= 8) return launch_t<KIND, 256, 1, 8, 1>(a, rpx, rpy, fld, ld, s);
    if (kc <= 12 && !coarse) return launch_t<KIND, 256, 1, 12, 1>(a, rpx, rpy, fld, ld, s);
  }
  if (kc <= 16) return launch_t<KIND, 256, 1, 16, 1>(a, rpx, rpy, fld, ld, s);
  return launch_t<KIND, 224, 1, 32, 2>(a, rpx, rpy, fld, ld, s);
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

std::string fused_error(int code) {
  if (code == kErrNoEncode) return "cuTensorMapEncodeTiled is unavailable";
  if (code == kErrLaunch) return "launch failed: " + cuda_err_str(cudaGetLastError());
  return "tensor map encode failed (CUresult " + std::to_string(code) + ")";
}

bool fused_supported(const Stencil& st, int k) {
  // TMA maps need 16-byte row strides (nx even) and coordinates that fit int32
  return st.kind != PSP_OP_DIA && k <= 32 && st.x_lo == nullptr && st.x_hi == nullptr && st.nx % 2 == 0 &&
         st.nx * st.ny * st.nz < ((int64_t)1 << 31) && encode_fn() != nullptr;
}

int launch_fused(const Stencil& st0, const double* ring_px, const double* ring_py, int vs1, int cap, int k, int nA,
                  int src_slot, int src_px, double* dstx, double* dsty, double* slot_scale, int dst_slot,
                  DevState ds, cudaStream_t s, const FusedLayout& lay, int jb, const double* src_vec) {
  FusedArgs a;
  a.zoff = lay.zoff;
  a.lo_in = lay.lo_in;
  a.hi_in = lay.hi_in;
  a.jb = jb;
  a.hyb = src_vec != nullptr;
  a.src_vec = src_vec;
  if (src_vec != nullptr) {
    src_px = 2;
    src_slot = 0;
  }
  a.st = march_view(st0);
  a.k = k;
  a.nA = nA;
  a.vs1 = vs1;
  a.cap = cap;
  a.src_slot = src_slot;
  a.src_px = src_px;
  a.dstx = dstx;
  a.dsty = dsty;
  a.slot_scale = slot_scale;
  a.dst_slot = dst_slot;
  a.zchunk = 1;
  a.tiles_x = a.tiles_y = a.ntiles = 1;
  a.ds = ds;
  const bool three_d = st0.ndim == 3;
  switch (st0.kind) {
    case PSP_OP_CONST_DIFF: return launch_kind<PSP_OP_CONST_DIFF>(a, three_d, ring_px, ring_py, lay.field, lay.ld, s);
    case PSP_OP_CELL_DIFF: return launch_kind<PSP_OP_CELL_DIFF>(a, three_d, ring_px, ring_py, lay.field, lay.ld, s);
    default: return launch_kind<PSP_OP_CELL_ADVDIFF>(a, three_d, ring_px, ring_py, lay.field, lay.ld, s);
  }
}

}  // namespace psp
