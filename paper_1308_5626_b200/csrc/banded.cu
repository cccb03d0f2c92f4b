// banded.cu -- K4: the preconditioner solve N z = v (Alg.1 l.10 and l.42; "solved
// efficiently in O(n) FLOPs using Thomas algorithm"; d > 1 per P:161), by the
// unpivoted banded LU of N (Doolittle; for d = 1 the same operations as Thomas).
//
// Factorisation (a9, once per time step).  Doolittle's row recurrence is sequential: row i
// needs the U rows i-d..i-1.  It is split into chunks of kChunk rows, one thread each.  The
// default is one LU-writing pass in which every chunk starts kWarm rows early from the zero
// state, followed by a bitwise check of each chunk's start state against its left neighbour's
// end state; only on a mismatch does the exact chunked fixed point follow: pass p recomputes
// every chunk from the state its left neighbour produced in pass p-1, chunks 0..p-1 are then
// bitwise the sequential result, and the iteration stops at the first pass in which no chunk's
// outgoing state changed (at most #chunks+1 passes).  A warp's 32 chunks are staged by the warp
// together (cooperative cp.async copies of eight-row groups, factor_pass_kernel COOP).
//
// Solve (a2, every iteration).  Two sweeps, each a linear recurrence of order d:
//   forward  y_i = v_i - sum_{k=1..d} L(i,i-k) y_{i-k}
//   backward z_i = (y_i - sum_{k=1..d} U(i,i+k) z_{i+k}) / U(i,i)
// Each sweep reads the coefficients about once (wsweep_kernel): every warp walks a contiguous
// range of warp-tiles from a zero incoming state -- a lane runs its rows with d+1 simultaneous
// recurrences (zero state + the d unit states) for its affine map state_out = M state_in + t,
// a shuffle scan composes the lane maps -- and writes the zero-state rows and the range's map;
// one block scans the range maps into exact incoming states (wscan_kernel); one thread per range
// adds the homogeneous response to that state until it has decayed below 2^-60 of it
// (tile_fix_kernel), and a range whose response has not decayed is re-walked in full.
// Algorithmic bytes: forward 8(d+2), backward 8(d+3) per row.  The r01-r02 tile kernels
// (tile_map/scan/fix/apply: shared-memory tiles and a block scan) stay behind PSP_SOLVE_BLOCK.
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "internal.h"


namespace psp {
namespace {

#ifndef PSP_FACTOR_CHUNK
#define PSP_FACTOR_CHUNK 512
#endif
constexpr int kChunk = PSP_FACTOR_CHUNK;   // factor: rows per thread
constexpr int kWarm = 64;        // factor: warm-up rows before a chunk (first pass)
#ifndef PSP_FACTOR_PF
#define PSP_FACTOR_PF 3
#endif
#ifndef PSP_FACTOR_FASTRCP
#define PSP_FACTOR_FASTRCP 1   // factor: the pivot reciprocal by rcp.approx + Newton (recip_pivot)
#endif
#ifndef PSP_FACTOR_G
#define PSP_FACTOR_G 8     // factor (cooperative staging): rows a staged group (4 or 8)
#endif
#ifndef PSP_FACTOR_PFMAXD
#define PSP_FACTOR_PFMAXD 4
#endif
#ifndef PSP_FACTOR_TPB
#define PSP_FACTOR_TPB 64
#endif
// factor: prefetch ring depth (staged groups); d = 4 takes two (its nine bands a stage: three
// stages would leave one 64-thread block an SM; n = 2^26: 4.2 -> 2.9 ms with the ring)
template <int D>
constexpr int kPFd = D >= 4 ? 2 : PSP_FACTOR_PF;
// solve sweeps: 256-thread blocks (2 per SM) for d <= 2; 128-thread blocks for d >= 3, 4 per SM
// at d = 3 and 3 per SM at d = 4 (more independent tiles in flight; measured n = 2^26: d = 3
// 2.34 -> 2.04 ms, d = 4 4.25 -> 3.65 ms; d = 1 prefers 256)
#ifndef PSP_SOLVE_SR
#define PSP_SOLVE_SR 8
#endif
constexpr int SR = PSP_SOLVE_SR; // solve: rows per thread (the block scan of thread maps is per SR rows)
template <int D>
struct SW {
  static constexpr int TPB = D >= 3 ? 128 : 256;
  static constexpr int MINB = D >= 4 ? 3 : (D == 3 ? 4 : 2);   // d = 4: 3 blocks (168 registers) spill less
  static constexpr int TILE = TPB * SR;
};
constexpr int STPB = 128;        // solve: the smallest block (host-side sizing of per-tile arrays)
constexpr int STILE = STPB * SR; // solve: rows per tile
constexpr int SPAD = SR + 1;     // padded row stride in shared memory (bank conflicts)

// 1 / U(i,i) for the warp-range sweeps and their corrections: the hardware approximation and two
// Newton steps (within an ulp; unlike '/', no out-of-line special-case path -- a gated pivot is
// a normal number), PSP_WSWEEP_FASTRCP = 0: the IEEE division.  Measured n = 2^26: d = 1 0.63 ->
// 0.61 ms, d = 3 1.40 -> 1.34 ms, d = 4 2.21 -> 2.15 ms.
#ifndef PSP_WSWEEP_FASTRCP
#define PSP_WSWEEP_FASTRCP 1
#endif
__device__ __forceinline__ double recip_pivot(double u) {
  if (!PSP_WSWEEP_FASTRCP) return 1.0 / u;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  r = fma(r, fma(-u, r, 1.0), r);
  return fma(r, fma(-u, r, 1.0), r);
}

// ---------------------------------------------------------------------------------------
// Factorisation pass
// ---------------------------------------------------------------------------------------
// One pass over every chunk.  Rows are walked four at a time: a thread walks its own chunk, so a
// warp touches 32 chunks at once.  WRITE = 0: a state-only pass (the fixed point is iterated
// without storing LU; one WRITE pass follows convergence).
//
// COOP = 1 (d <= 3, 16-byte aligned bands, the default): the bands of the warp's 32 chunks are
// staged in groups of eight rows by the warp together -- lane j copies 16-byte piece (j & 3) of
// chunk 8q + (j >> 2), so one cp.async instruction covers eight 64-byte runs instead of 32
// scattered 16-byte pieces (ncu r02: the per-thread copies left the LSU throttled, mio/lg
// throttle and long-scoreboard stalls, 37 % DRAM throughput) -- and the LU rows of a staged group
// go back to HBM the same way from the stage they were computed in.  COOP = 0: each thread copies
// its own rows (groups of four; d = 4 without the shared-memory ring).
template <int D, bool WRITE, bool COOP>
__global__ void factor_pass_kernel(const double* __restrict__ bands, int64_t n, double* __restrict__ lu,
                                   const double* __restrict__ st_in, double* __restrict__ st_out,
                                   int first_pass, int* __restrict__ changed, int* __restrict__ bad,
                                   const double* __restrict__ prev, int has_prev, int has_next, int vec,
                                   int warm, double* __restrict__ st_start) {
  // has_prev / has_next (multi-rank): the global matrix continues before row 0 / after row n-1
  // of this block (rows of rank-1 / rank+1), so the band entries reaching there are real
  constexpr int W = D * (D + 1);  // last D rows of U: Uw[q][e] = U(r0-D+q, r0-D+q+e)
  constexpr int NB = 2 * D + 1;
  constexpr bool PFON = D <= PSP_FACTOR_PFMAXD;   // the cp.async ring (every d by default)
  static_assert(!COOP || PFON, "cooperative staging uses the prefetch ring");
  constexpr int G = COOP ? PSP_FACTOR_G : 4;   // rows a staged group (COOP 8: two walk steps of four rows)
  constexpr int NPC = G / 2;       // COOP: 16-byte pieces of a chunk's group in one band
  constexpr int CPI = 32 / NPC;    // COOP: chunks one warp-wide copy instruction covers
  static_assert(kWarm % 8 == 0, "warm-up rows: whole groups");
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!COOP && c >= nchunks) return;
  const bool valid = c < nchunks;  // COOP: lanes past the last chunk still copy for the others
  const int lane = threadIdx.x & 31;
  // chunk cc's rows [r0c, r1c) and walk start rsc (warm start: `warm` rows early from the zero state)
  auto geom = [&](int64_t cc, int64_t& r0c, int64_t& r1c, int64_t& rsc) {
    r0c = cc * kChunk;
    r1c = (r0c + kChunk < n) ? r0c + kChunk : n;
    rsc = (warm > 0 && first_pass && cc > 0) ? (r0c - warm > 0 ? r0c - warm : 0) : r0c;
  };
  int64_t r0, r1, rs;
  geom(valid ? c : 0, r0, r1, rs);
  double Uw[D][D + 1];
  // chunk 0 of rank r > 0 (after the first pass): the last-D-U-rows state of rank r-1
  const bool from_prev = (c == 0) && (prev != nullptr) && !first_pass;
  if (from_prev) {
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int e = 0; e <= D; ++e) Uw[q][e] = prev[q * (D + 1) + e];
  } else if (c == 0 || first_pass || !valid) {
    // matrix start (exact for chunk 0; the initial guess for the others)
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int e = 0; e <= D; ++e) Uw[q][e] = 0.0;
  } else {
    const double* s = st_in + (c - 1) * W;
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int e = 0; e <= D; ++e) Uw[q][e] = s[q * (D + 1) + e];
  }
  const bool at_start = !from_prev && ((c == 0) || first_pass);
  // first row of the walk's existing window rows: rows below lo do not exist
  const int64_t lo = at_start ? rs : (has_prev ? INT64_MIN / 2 : 0);
  double Ri[D];       // 1 / U(k,k) of the window rows (unused for rows that do not exist)
#pragma unroll
  for (int q = 0; q < D; ++q) Ri[q] = PSP_FACTOR_FASTRCP ? recip_pivot(Uw[q][0]) : 1.0 / Uw[q][0];
  int isbad = 0;
  // the bands of the next groups are prefetched into a PF-deep shared-memory ring by cp.async
  // (16-byte copies, no registers held): a walk is a serial recurrence, and without the prefetch
  // every group waits a full DRAM latency
  // [PF][NB][blockDim][GS]: a thread's G rows padded to GS doubles (COOP: 80-byte rows, so
  // the 16-byte accesses of eight consecutive threads fall in distinct banks)
  constexpr int GS = COOP ? G + 2 : G;
  extern __shared__ __align__(16) double pf[];
  auto pf_of = [&](int buf, int o, int t) -> double* {
    return pf + ((size_t)(buf * NB + o) * PSP_FACTOR_TPB + t) * GS;
  };
  // COOP: the NPC chunks this lane copies for (cl = CPI q + lane / NPC, piece lane % NPC): walk start,
  // rows of the walk, and the first live row, relative to the walk start
  int64_t qrs[COOP ? NPC : 1];
  int qlen[COOP ? NPC : 1], qoff[COOP ? NPC : 1];
  uint32_t qsa[COOP ? NPC : 1];
  if (COOP) {
    const int64_t wbase = c - lane;               // chunk of lane 0 of this warp
#pragma unroll
    for (int q = 0; q < NPC; ++q) {
      const int cl = CPI * q + lane / NPC;
      int64_t r0c, r1c, rsc;
      geom(wbase + cl, r0c, r1c, rsc);
      const bool ex = wbase + cl < nchunks;
      qrs[q] = rsc + 2 * (lane % NPC);
      qlen[q] = ex ? (int)(r1c - rsc) : 0;
      qoff[q] = (int)(r0c - rsc);
      qsa[q] = (uint32_t)__cvta_generic_to_shared(pf_of(0, 0, threadIdx.x - lane + cl) + 2 * (lane % NPC));
    }
  }
  constexpr uint32_t kStageB = (uint32_t)PSP_FACTOR_TPB * GS * 8;   // bytes a band of a stage
  auto prefetch = [&](int64_t sg, int buf) {      // group sg of the walk(s)
    if (!PFON) return;
    if (COOP) {
#pragma unroll
      for (int q = 0; q < NPC; ++q) {
        if (G * ((int)sg + 1) <= qlen[q]) {
          const double* g = bands + qrs[q] + (int64_t)G * sg;
#pragma unroll
          for (int o = 0; o < NB; ++o) {
            const uint32_t sa = qsa[q] + (uint32_t)(buf * NB + o) * kStageB;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g + (int64_t)o * n) : "memory");
          }
        }
      }
    } else {
      const int64_t i0 = rs + (int64_t)G * sg;
      if (vec && i0 + 4 <= r1) {
#pragma unroll
        for (int o = 0; o < NB; ++o) {
          const double* g = bands + (int64_t)o * n + i0;
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(pf_of(buf, o, threadIdx.x));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + 16), "l"(g + 2) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");   // (possibly empty: keeps the count)
  };
  // COOP: the LU rows of the warp's staged, live groups from the stage to HBM (coalesced)
  auto store_group = [&](int64_t sg, int buf) {
#pragma unroll
    for (int q = 0; q < NPC; ++q) {
      if (G * ((int)sg + 1) <= qlen[q] && G * (int)sg >= qoff[q]) {
        double* g = lu + qrs[q] + (int64_t)G * sg;
#pragma unroll
        for (int o = 0; o < NB; ++o) {
          double2 v;
          const uint32_t sa = qsa[q] + (uint32_t)(buf * NB + o) * kStageB;
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(sa));
          *reinterpret_cast<double2*>(g + (int64_t)o * n) = v;
        }
      }
    }
  };
  int itmax = valid ? (int)((r1 - rs + 3) / 4) : 0;   // walk steps of four rows
  if (COOP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) itmax = max(itmax, __shfl_xor_sync(0xffffffffu, itmax, o));
  }
#pragma unroll
  constexpr int kPF = kPFd<D>;
  for (int q = 0; q < kPF - 1; ++q) prefetch(q, q);
  int buf = 0;
  for (int it = 0; it < itmax; ++it) {
    const int h = COOP ? (it % (G / 4)) : 0;      // walk step within the staged group
    const int64_t sg = COOP ? (it / (G / 4)) : it; // staged group
    const int64_t i0 = rs + 4 * (int64_t)it;
    if (h == 0) {
      if (PFON) asm volatile("cp.async.wait_group %0;" ::"n"(kPF - 2) : "memory");   // group sg landed
      if (COOP) __syncwarp();                     // (copied by the other lanes)
      prefetch(sg + kPF - 1, buf == 0 ? kPF - 1 : buf - 1);   // into the slot read last group
    }
    if (valid && i0 < r1) {
      const bool live = i0 >= r0;                 // warm-up rows: state only
      if (warm > 0 && first_pass && c > 0 && i0 == r0) {
#pragma unroll
        for (int q = 0; q < D; ++q)
#pragma unroll
          for (int e = 0; e <= D; ++e) st_start[c * W + q * (D + 1) + e] = Uw[q][e];
      }
      const int nr = (r1 - i0) < 4 ? (int)(r1 - i0) : 4;
      // staged: COOP the whole group of eight (rows rs + 8 sg ..), else this step's four rows
      const bool staged = PFON && vec && (COOP ? (rs + (int64_t)G * sg + G <= r1) : (nr == 4));
      double bb[NB][4];
      if (staged) {
#pragma unroll
        for (int o = 0; o < NB; ++o) {
          const double* sp = pf_of(buf, o, threadIdx.x) + 4 * h;
          const double2 a = *reinterpret_cast<const double2*>(sp);
          const double2 b = *reinterpret_cast<const double2*>(sp + 2);
          bb[o][0] = a.x; bb[o][1] = a.y; bb[o][2] = b.x; bb[o][3] = b.y;
        }
      } else if (vec && nr == 4) {
#pragma unroll
        for (int o = 0; o < NB; ++o) {
          const double2 a = __ldg(reinterpret_cast<const double2*>(bands + (int64_t)o * n + i0));
          const double2 b = __ldg(reinterpret_cast<const double2*>(bands + (int64_t)o * n + i0 + 2));
          bb[o][0] = a.x; bb[o][1] = a.y; bb[o][2] = b.x; bb[o][3] = b.y;
        }
      } else {
#pragma unroll
        for (int o = 0; o < NB; ++o)
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) bb[o][rr] = (rr < nr) ? __ldg(bands + (int64_t)o * n + i0 + rr) : 0.0;
      }
      // results overwrite the consumed band values of their row (bb doubles as the output tile).
      // Steps whose rows all have a full window (no matrix / chunk start within D rows, no matrix
      // end within D rows) take the check-free copy of the row step.
      const bool full = (i0 - D >= lo) && (i0 + 3 + D < n || has_next);
      auto step = [&](auto chk) {
        constexpr bool C = decltype(chk)::value;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          if (rr >= nr) break;
          const int64_t i = i0 + rr;
          double Lr[D];       // L(i, i-D+q), q = 0..D-1
          double Ur[D + 1];   // U(i, i+e)
          // U(k, j) for window row k = i-D+q: Uw[q][j-k] when 0 <= j-k <= D (compile-time after
          // unrolling).  Rows before the matrix start (or before the walk start of a zero-state
          // walk) do not exist.
          auto row_exists = [&](int q) -> bool {
            if (!C) return true;
            const int64_t k = i - D + q;
            return (k >= 0 || has_prev) && !(at_start && k < rs);
          };
#pragma unroll
          for (int q = 0; q < D; ++q) {           // L(i,j), j = i-D+q  (ascending j)
            if (!row_exists(q)) { Lr[q] = 0.0; continue; }
            double sum = bb[q][rr];                 // N(i,j), band o = j-i+D = q
#pragma unroll
            for (int p = 0; p < q; ++p)           // U(k, j), k = i-D+p: window entry e = q - p
              if (row_exists(p)) sum -= Lr[p] * Uw[p][q - p];
            Lr[q] = sum * Ri[q];                  // / U(j,j), by its reciprocal
          }
#pragma unroll
          for (int e = 0; e <= D; ++e) {          // U(i,j), j = i+e
            if (C && i + e >= n && !has_next) { Ur[e] = 0.0; continue; }
            double sum = bb[D + e][rr];
#pragma unroll
            for (int p = 0; p < D; ++p)           // k = i-D+p in [j-D, i-1]: window entry D - p + e
              if (p >= e && row_exists(p)) sum -= Lr[p] * Uw[p][D - p + e];
            Ur[e] = sum;
          }
          if (live && !(fabs(Ur[0]) >= 1e-300)) isbad = 1;   // S:272 (also catches NaN)
#pragma unroll
          for (int q = 0; q < D; ++q) {
            if (live && !(fabs(Lr[q]) <= 1e100)) isbad = 1;  // S:293 growth / non-finite
            bb[q][rr] = Lr[q];
          }
#pragma unroll
          for (int e = 0; e <= D; ++e) {
            if (live && !(fabs(Ur[e]) <= 1e100)) isbad = 1;
            bb[D + e][rr] = Ur[e];
          }
          // shift the window (and the pivot reciprocals: one division per row)
#pragma unroll
          for (int q = 0; q < D - 1; ++q) {
#pragma unroll
            for (int e = 0; e <= D; ++e) Uw[q][e] = Uw[q + 1][e];
            Ri[q] = Ri[q + 1];
          }
#pragma unroll
          for (int e = 0; e <= D; ++e) Uw[D - 1][e] = Ur[e];
          Ri[D - 1] = PSP_FACTOR_FASTRCP ? recip_pivot(Ur[0]) : 1.0 / Ur[0];
        }
      };
      if (full) step(std::false_type{});
      else step(std::true_type{});
      if (WRITE && live) {
        if (COOP && staged) {                     // back into the stage: store_group writes it out
#pragma unroll
          for (int o = 0; o < NB; ++o) {
            double* sp = pf_of(buf, o, threadIdx.x) + 4 * h;
            *reinterpret_cast<double2*>(sp) = make_double2(bb[o][0], bb[o][1]);
            *reinterpret_cast<double2*>(sp + 2) = make_double2(bb[o][2], bb[o][3]);
          }
        } else if (vec && nr == 4) {
#pragma unroll
          for (int o = 0; o < NB; ++o) {
            *reinterpret_cast<double2*>(lu + (int64_t)o * n + i0) = make_double2(bb[o][0], bb[o][1]);
            *reinterpret_cast<double2*>(lu + (int64_t)o * n + i0 + 2) = make_double2(bb[o][2], bb[o][3]);
          }
        } else {
#pragma unroll
          for (int o = 0; o < NB; ++o)
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
              if (rr < nr) lu[(int64_t)o * n + i0 + rr] = bb[o][rr];
        }
      }
    }
    if (h == G / 4 - 1) {                         // end of the staged group
      if (COOP && WRITE) {
        __syncwarp();
        store_group(sg, buf);
        __syncwarp();                             // stage read before the next prefetch into it
      }
      buf = (buf + 1 == kPF) ? 0 : buf + 1;
    }
  }
  if (!valid) return;
  double* so = st_out + c * W;
  bool diff = first_pass != 0;
#pragma unroll
  for (int q = 0; q < D; ++q)
#pragma unroll
    for (int e = 0; e <= D; ++e) {
      const double v = Uw[q][e];
      if (!first_pass && __double_as_longlong(v) != __double_as_longlong(st_in[c * W + q * (D + 1) + e]))
        diff = true;
      so[q * (D + 1) + e] = v;
    }
  if (diff) atomicAdd(changed, 1);
  if (isbad) atomicOr(bad, 1);
}

// ---------------------------------------------------------------------------------------
// Solve sweeps with decoupled look-back
// ---------------------------------------------------------------------------------------
template <int D>
struct Map {
  double M[D][D];
  double t[D];
};

// c = a after b   (apply b first, then a):  M = Ma Mb, t = Ma tb + ta
template <int D>
__device__ __forceinline__ Map<D> compose(const Map<D>& a, const Map<D>& b) {
  Map<D> c;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double ti = a.t[i];
#pragma unroll
    for (int k = 0; k < D; ++k) ti = fma(a.M[i][k], b.t[k], ti);
    c.t[i] = ti;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s = fma(a.M[i][k], b.M[k][j], s);
      c.M[i][j] = s;
    }
  }
  return c;
}

template <int D>
__device__ __forceinline__ Map<D> shfl_up_map(const Map<D>& m, int off) {
  Map<D> r;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    r.t[i] = __shfl_up_sync(0xffffffffu, m.t[i], off);
#pragma unroll
    for (int j = 0; j < D; ++j) r.M[i][j] = __shfl_up_sync(0xffffffffu, m.M[i][j], off);
  }
  return r;
}

template <int D>
__device__ __forceinline__ Map<D> identity_map() {
  Map<D> m;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    m.t[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) m.M[i][j] = (i == j) ? 1.0 : 0.0;
  }
  return m;
}

template <int D>
__device__ __forceinline__ void apply(const Map<D>& m, const double (&s)[D], double (&o)[D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double v = m.t[i];
#pragma unroll
    for (int k = 0; k < D; ++k) v = fma(m.M[i][k], s[k], v);
    o[i] = v;
  }
}

// Descriptor layout per tile: [M (D*D) | t (D) | S (D)] doubles: the tile's affine map and
// the exact state entering it.
//
// A sweep is four launches, none with cross-block waits; block b owns a contiguous range of
// 2048-row tiles in processing order:
//   tile_map_kernel    walks its range from a zero incoming state: writes y0 (+ addend) and
//                      composes the range's affine map state_out = M state_in + t (per tile:
//                      zero-state run plus the d unit-state runs, block scan of thread maps);
//   tile_scan_kernel   one block composes the <= 1024 range maps: exact incoming state of every
//                      range (and the state after the last row, s_out);
//   tile_fix_kernel    one thread per range adds the homogeneous response to its exact incoming
//                      state, row by row, until it has decayed below 2^-60 of its start (under
//                      the dominance gate, tens to hundreds of rows);
//   tile_apply_kernel  re-walks, from the exact state, only the ranges whose response did not
//                      decay within kFixCap rows.
// So the coefficients and the right-hand side are read about once (8(d+2) forward, 8(d+3)
// backward per row, plus the short corrections), with no look-back chain: a single-pass
// chained scan over 2^16 tiles was latency-bound at ~1/4 of these rates.

// One recurrence step.  FWD: y = v - sum_k c[k] s[k]   (c[k] = L(i,i-k-1), s[k] = y_{i-k-1})
//                        BWD: z = (v - sum_k c[k] s[k]) / U(i,i) (c[k] = U(i,i+k+1), s[k] = z_{i+k+1}),
// evaluated with ui = 1 / U(i,i) formed once per row (the D unit-state runs of a tile map share
// it; one rounding more than a division, inside T2)
template <bool FWD, int D>
__device__ __forceinline__ double rec_step(double v, const double (&c)[D], const double (&s)[D],
                                           double ui) {
  double acc = v;
#pragma unroll
  for (int k = 0; k < D; ++k) acc -= c[k] * s[k];
  return FWD ? acc : acc * ui;
}

template <int D>
__device__ __forceinline__ void push_state(double (&s)[D], double y) {
#pragma unroll
  for (int k = D - 1; k > 0; --k) s[k] = s[k - 1];
  s[0] = y;
}

template <bool FWD, int D>
struct TileSmem {
  static constexpr int NA = 1 + D + (FWD ? 0 : 1);
  static constexpr size_t BYTES = (size_t)NA * SW<D>::TPB * SPAD * sizeof(double);
};

// stage the tile's rows (coalesced) into the per-thread padded layout: sv (rhs), sc[k]
// (recurrence coefficients), su0 (U(i,i), backward); padding rows are transparent
template <bool FWD, int D>
__device__ __forceinline__ void stage_tile(double* sv, const double* __restrict__ lu, int64_t n,
                                           const double* __restrict__ vin, double vsc, int64_t base) {
  double* sc0 = sv + SW<D>::TPB * SPAD;
  double* su0 = sv + (1 + D) * SW<D>::TPB * SPAD;
  constexpr int IT = SW<D>::TILE / SW<D>::TPB;              // rows per thread of the coalesced copy
  constexpr int NA = 1 + D + (FWD ? 0 : 1);
  // every load of a group of (up to) eight rows a thread is issued before its first shared-
  // memory store (one latency per group)
  constexpr int IG = IT <= 8 ? IT : (IT % 8 == 0 ? 8 : (IT % 6 == 0 ? 6 : 4));
  static_assert(IT % IG == 0, "row groups");
  const bool full = base + SW<D>::TILE <= n;
#pragma unroll
  for (int g0 = 0; g0 < IT; g0 += IG) {
    double r[IG][NA];
#pragma unroll
    for (int ig = 0; ig < IG; ++ig) {
      const int64_t i = base + threadIdx.x + (g0 + ig) * SW<D>::TPB;
      const bool in = full || i < n;
      r[ig][0] = (in && vin) ? __ldg(vin + i) : 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        // FWD: c[k] = L(i, i-k-1) = lu[(D-1-k) n + i];  BWD: c[k] = U(i, i+k+1) = lu[(D+1+k) n + i]
        const int o = FWD ? (D - 1 - k) : (D + 1 + k);
        r[ig][1 + k] = in ? __ldg(lu + (int64_t)o * n + i) : 0.0;
      }
      if (!FWD) r[ig][1 + D] = in ? __ldg(lu + (int64_t)D * n + i) : 1.0;
    }
#pragma unroll
    for (int ig = 0; ig < IG; ++ig) {
      const int q = threadIdx.x + (g0 + ig) * SW<D>::TPB;
      const int sidx = (q / SR) * SPAD + (q % SR);
      sv[sidx] = vsc * r[ig][0];
#pragma unroll
      for (int k = 0; k < D; ++k) sc0[k * SW<D>::TPB * SPAD + sidx] = r[ig][1 + k];
      if (!FWD) su0[sidx] = 1.0 / r[ig][1 + D];   // the reciprocal pivot (padding rows: 1)
    }
  }
}

// this thread's SR rows as an affine map (FWD ascending, BWD descending)
template <bool FWD, int D>
__device__ __forceinline__ Map<D> thread_map(const double* sv, int64_t base, int64_t n) {
  const double (*sc)[SW<D>::TPB * SPAD] = reinterpret_cast<const double (*)[SW<D>::TPB * SPAD]>(sv + SW<D>::TPB * SPAD);
  const double* su0 = sv + (1 + D) * SW<D>::TPB * SPAD;
  const int t = threadIdx.x;
  double sz[D];            // zero-state run
  double su[D][D];         // unit-state runs: su[q] starts at e_q
#pragma unroll
  for (int k = 0; k < D; ++k) {
    sz[k] = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) su[q][k] = (q == k) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int rr = 0; rr < SR; ++rr) {
    const int r = FWD ? rr : (SR - 1 - rr);
    if (base + (int64_t)t * SR + r >= n) continue;   // padding rows are transparent
    const int sidx = t * SPAD + r;
    double c[D];
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = sc[k][sidx];
    const double u0 = FWD ? 1.0 : su0[sidx];
    push_state<D>(sz, rec_step<FWD, D>(sv[sidx], c, sz, u0));
#pragma unroll
    for (int q = 0; q < D; ++q) push_state<D>(su[q], rec_step<FWD, D>(0.0, c, su[q], u0));
  }
  Map<D> my;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    my.t[i] = sz[i];
#pragma unroll
    for (int q = 0; q < D; ++q) my.M[i][q] = su[q][i];
  }
  return my;
}

// block scan of the thread maps in processing order (FWD thread 0 first, BWD thread SW<D>::TPB-1
// first): returns this thread's exclusive prefix; agg (valid in every thread) = the whole tile
template <bool FWD, int D>
__device__ __forceinline__ Map<D> block_prefix(const Map<D>& my, Map<D>* wtot, Map<D>& agg) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int NW = SW<D>::TPB / 32;
  Map<D> inc = my;  // inclusive prefix within the warp, in processing order
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Map<D> o;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      o.t[i] = FWD ? __shfl_up_sync(0xffffffffu, inc.t[i], off) : __shfl_down_sync(0xffffffffu, inc.t[i], off);
#pragma unroll
      for (int j = 0; j < D; ++j)
        o.M[i][j] = FWD ? __shfl_up_sync(0xffffffffu, inc.M[i][j], off) : __shfl_down_sync(0xffffffffu, inc.M[i][j], off);
    }
    const bool has = FWD ? (lane >= off) : (lane + off < 32);
    if (has) inc = compose<D>(inc, o);
  }
  Map<D> exw;  // exclusive-in-warp = inclusive of the previous lane (processing order)
#pragma unroll
  for (int i = 0; i < D; ++i) {
    exw.t[i] = FWD ? __shfl_up_sync(0xffffffffu, inc.t[i], 1) : __shfl_down_sync(0xffffffffu, inc.t[i], 1);
#pragma unroll
    for (int j = 0; j < D; ++j)
      exw.M[i][j] = FWD ? __shfl_up_sync(0xffffffffu, inc.M[i][j], 1) : __shfl_down_sync(0xffffffffu, inc.M[i][j], 1);
  }
  if (FWD ? (lane == 0) : (lane == 31)) exw = identity_map<D>();
  if (FWD ? (lane == 31) : (lane == 0)) wtot[warp] = inc;
  __syncthreads();
  Map<D> wpre = identity_map<D>();
  agg = identity_map<D>();
  if (FWD) {
    for (int w = 0; w < NW; ++w) {
      if (w == warp) wpre = agg;
      agg = compose<D>(wtot[w], agg);
    }
  } else {
    for (int w = NW - 1; w >= 0; --w) {
      if (w == warp) wpre = agg;
      agg = compose<D>(wtot[w], agg);
    }
  }
  __syncthreads();   // wtot may be reused
  return compose<D>(exw, wpre);   // warp prefix first, then the in-warp prefix
}

// Block b owns the contiguous range of tiles [b L, (b+1) L) in processing order (FWD:
// ascending tiles, BWD: descending).  tile_map_kernel composes its tiles' maps into the range
// map; tile_scan_kernel turns the range maps into exact incoming range states; tile_apply_kernel
// walks the range again from that state (each tile's map, recomputed, carries the state on).
template <bool FWD, int D>
__global__ void __launch_bounds__(SW<D>::TPB, SW<D>::MINB) tile_map_kernel(const double* __restrict__ lu, int64_t n,
                                                            const double* __restrict__ vin, const double* vscale,
                                                            const double* addend, double* out, int64_t L,
                                                            double* __restrict__ rmap) {
  // Walks its range from a ZERO incoming state: writes out = addend + y0 (the range's rows solved
  // as if the state entering the range were 0) and composes the range map (M, t).  The exact
  // solution differs from y0 only by the homogeneous response to the true incoming state,
  // which tile_fix_kernel adds (it decays geometrically under the dominance gate).
  extern __shared__ double smem_dyn[];
  __shared__ Map<D> wtot[SW<D>::TPB / 32];
  constexpr int DW = D * D + 2 * D;
  const int t = threadIdx.x;
  const int64_t ntiles = (n + SW<D>::TILE - 1) / SW<D>::TILE;
  const double vsc = vscale ? *vscale : 1.0;
  double* sv = smem_dyn;
  const double (*sc)[SW<D>::TPB * SPAD] = reinterpret_cast<const double (*)[SW<D>::TPB * SPAD]>(sv + SW<D>::TPB * SPAD);
  const double* su0 = sv + (1 + D) * SW<D>::TPB * SPAD;
  Map<D> range = identity_map<D>();
  double s0[D];
#pragma unroll
  for (int i = 0; i < D; ++i) s0[i] = 0.0;
  const int64_t p0 = (int64_t)blockIdx.x * L, p1 = (p0 + L < ntiles) ? p0 + L : ntiles;
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t tile = FWD ? p : ntiles - 1 - p;
    const int64_t base = tile * SW<D>::TILE;
    stage_tile<FWD, D>(sv, lu, n, vin, vsc, base);
    __syncthreads();
    const Map<D> my = thread_map<FWD, D>(sv, base, n);
    Map<D> agg;
    const Map<D> pre = block_prefix<FWD, D>(my, wtot, agg);
    range = compose<D>(agg, range);
    if (out != nullptr) {
      double st[D];
      apply<D>(pre, s0, st);
#pragma unroll
      for (int rr = 0; rr < SR; ++rr) {
        const int r = FWD ? rr : (SR - 1 - rr);
        if (base + (int64_t)t * SR + r >= n) continue;   // padding rows are transparent
        const int sidx = t * SPAD + r;
        double c[D];
#pragma unroll
        for (int k = 0; k < D; ++k) c[k] = sc[k][sidx];
        const double u0 = FWD ? 1.0 : su0[sidx];
        const double y = rec_step<FWD, D>(sv[sidx], c, st, u0);
        push_state<D>(st, y);
        sv[sidx] = y;
      }
      double s1[D];
      apply<D>(agg, s0, s1);
#pragma unroll
      for (int i = 0; i < D; ++i) s0[i] = s1[i];
      __syncthreads();
      for (int q = t; q < SW<D>::TILE; q += SW<D>::TPB) {
        const int64_t i = base + q;
        if (i < n) {
          const double y = sv[(q / SR) * SPAD + (q % SR)];
          out[i] = addend ? addend[i] + y : y;
        }
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    double* dd = rmap + blockIdx.x * DW;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      dd[D * D + i] = range.t[i];
#pragma unroll
      for (int j = 0; j < D; ++j) dd[i * D + j] = range.M[i][j];
    }
  }
}

// One thread per range: out += the homogeneous response to the range's exact incoming state,
// row by row from the range start, until it has decayed below 2^-60 of its initial size (the
// rows beyond are unchanged to working precision); a range whose response has not decayed
// within kFixCap rows is flagged for a full re-walk by tile_apply_kernel.
constexpr int64_t kFixCap = 16384;
template <bool FWD, int D>
__global__ void tile_fix_kernel(const double* __restrict__ lu, int64_t n, int64_t L, int nr, double* out,
                                const double* __restrict__ rmap, double* __restrict__ full, int64_t T) {
  // T: rows a tile (SW<D>::TILE for the tile kernels, WT for the warp-range kernels)
  constexpr int DW = D * D + 2 * D;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  full[r] = 0.0;
  double st[D], amax = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    st[i] = rmap[(int64_t)r * DW + D * D + D + i];
    amax = fmax(amax, fabs(st[i]));
  }
  if (!(amax > 0.0)) return;                       // zero incoming state: y0 is exact
  const double stop = amax * 0x1p-60;
  const int64_t ntiles = (n + T - 1) / T;
  const int64_t t0 = (int64_t)r * L, t1 = (t0 + L < ntiles) ? t0 + L : ntiles;
  // rows of the range in processing order
  const int64_t lo = (FWD ? t0 : ntiles - t1) * T;
  const int64_t hi = ((FWD ? t1 : ntiles - t0) * T < n) ? (FWD ? t1 : ntiles - t0) * T : n;
  const int64_t len = hi - lo;
  const int64_t cap = len < kFixCap ? len : kFixCap;
  int64_t q = 0;
  for (; q < cap; q += 8) {
    // the coefficients of the next 8 rows first (independent of the recurrence)
    double c8[8][D], u8[8], o8[8];
    int64_t idx[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t qq = q + e;
      idx[e] = FWD ? lo + qq : hi - 1 - qq;
      const bool ok = qq < cap;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int o = FWD ? (D - 1 - k) : (D + 1 + k);
        c8[e][k] = ok ? __ldg(lu + (int64_t)o * n + idx[e]) : 0.0;
      }
      u8[e] = (!FWD && ok) ? recip_pivot(__ldg(lu + (int64_t)D * n + idx[e])) : 1.0;   // reciprocal pivot
      o8[e] = ok ? out[idx[e]] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (q + e >= cap) break;
      const double y = rec_step<FWD, D>(0.0, c8[e], st, u8[e]);
      push_state<D>(st, y);
      out[idx[e]] = o8[e] + y;
    }
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) m = fmax(m, fabs(st[i]));
    if (m <= stop) return;                         // decayed: the rest of the range is exact
  }
  if (q < len) full[r] = 1.0;                      // not decayed within the cap: full re-walk
}

// one block: exact incoming state of every range (processing order), s_out after the last
constexpr int SCAN_T = 1024;
template <bool FWD, int D>
__global__ void __launch_bounds__(SCAN_T, 1) tile_scan_kernel(int nr, double* __restrict__ rmap,
                                                               const double* s_in0, double* s_out) {
  extern __shared__ double smem_dyn[];
  Map<D>* sm = reinterpret_cast<Map<D>*>(smem_dyn);   // [SCAN_T]
  constexpr int DW = D * D + 2 * D;
  const int t = threadIdx.x;
  Map<D> m = identity_map<D>();
  if (t < nr) {
    const double* dd = rmap + t * DW;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      m.t[i] = dd[D * D + i];
#pragma unroll
      for (int j = 0; j < D; ++j) m.M[i][j] = dd[i * D + j];
    }
  }
  sm[t] = m;
  __syncthreads();
  for (int off = 1; off < SCAN_T; off <<= 1) {      // inclusive (later ranges applied last)
    Map<D> o = identity_map<D>();
    if (t >= off) o = sm[t - off];
    __syncthreads();
    if (t >= off) sm[t] = compose<D>(sm[t], o);
    __syncthreads();
  }
  double s0[D], s[D];
#pragma unroll
  for (int i = 0; i < D; ++i) s0[i] = s_in0 ? s_in0[i] : 0.0;
  if (t > 0) apply<D>(sm[t - 1], s0, s);
  else
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = s0[i];
  if (t < nr)
#pragma unroll
    for (int i = 0; i < D; ++i) rmap[t * DW + D * D + D + i] = s[i];
  if (s_out && t == SCAN_T - 1) {
    double so[D];
    apply<D>(sm[SCAN_T - 1], s0, so);
#pragma unroll
    for (int i = 0; i < D; ++i) s_out[i] = so[i];
  }
}

template <bool FWD, int D>
__global__ void __launch_bounds__(SW<D>::TPB, SW<D>::MINB) tile_apply_kernel(const double* __restrict__ lu, int64_t n,
                                                              const double* __restrict__ vin, const double* vscale,
                                                              const double* addend, double* out, int64_t L,
                                                              const double* __restrict__ rmap,
                                                              const double* __restrict__ full) {
  extern __shared__ double smem_dyn[];
  __shared__ Map<D> wtot[SW<D>::TPB / 32];
  constexpr int DW = D * D + 2 * D;
  const int t = threadIdx.x;
  const int64_t ntiles = (n + SW<D>::TILE - 1) / SW<D>::TILE;
  const double vsc = vscale ? *vscale : 1.0;
  double* sv = smem_dyn;
  const double (*sc)[SW<D>::TPB * SPAD] = reinterpret_cast<const double (*)[SW<D>::TPB * SPAD]>(sv + SW<D>::TPB * SPAD);
  const double* su0 = sv + (1 + D) * SW<D>::TPB * SPAD;
  if (full != nullptr && full[blockIdx.x] == 0.0) return;   // tile_fix_kernel completed this range
  double s0[D];
#pragma unroll
  for (int i = 0; i < D; ++i) s0[i] = rmap[blockIdx.x * DW + D * D + D + i];
  const int64_t p0 = (int64_t)blockIdx.x * L, p1 = (p0 + L < ntiles) ? p0 + L : ntiles;
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t tile = FWD ? p : ntiles - 1 - p;
    const int64_t base = tile * SW<D>::TILE;
    stage_tile<FWD, D>(sv, lu, n, vin, vsc, base);
    __syncthreads();
    const Map<D> my = thread_map<FWD, D>(sv, base, n);
    Map<D> agg;
    const Map<D> pre = block_prefix<FWD, D>(my, wtot, agg);
    double st[D];
    apply<D>(pre, s0, st);
#pragma unroll
    for (int rr = 0; rr < SR; ++rr) {
      const int r = FWD ? rr : (SR - 1 - rr);
      if (base + (int64_t)t * SR + r >= n) continue;   // padding rows are transparent
      const int sidx = t * SPAD + r;
      double c[D];
#pragma unroll
      for (int k = 0; k < D; ++k) c[k] = sc[k][sidx];
      const double u0 = FWD ? 1.0 : su0[sidx];
      const double y = rec_step<FWD, D>(sv[sidx], c, st, u0);
      push_state<D>(st, y);
      sv[sidx] = y;
    }
    double s1[D];                                   // the state after this tile
    apply<D>(agg, s0, s1);
#pragma unroll
    for (int i = 0; i < D; ++i) s0[i] = s1[i];
    __syncthreads();
    for (int q = t; q < SW<D>::TILE; q += SW<D>::TPB) {
      const int64_t i = base + q;
      if (i < n) {
        const double y = sv[(q / SR) * SPAD + (q % SR)];
        out[i] = addend ? addend[i] + y : y;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// Warp-range sweeps (the default): the same decomposition as the tile kernels above with the
// warp as the unit.  Each warp owns a contiguous range of L warp-tiles (32 lanes x WSR rows) in
// processing order; a lane loads its WSR contiguous rows straight into registers (16-byte loads,
// whole sectors per warp), runs the zero-state and d unit-state recurrences over them, and a
// 5-level shuffle scan composes the lane maps.  No shared memory and no block barrier: the tile
// kernels spent ~10 warp instructions a row on staging, two block barriers and the serial
// cross-warp composition (ncu r02: tile_map issue-bound at 49 % issue-active, 21 % warps active,
// 32 % DRAM throughput); here a row costs ~3.  The lane's incoming state is the previous lane's
// inclusive state (one 3-double shuffle, not an exclusive map), the range map is composed only
// by the last lane in processing order (its inclusive map is the tile's), and the state carried
// to the next warp-tile is broadcast from that lane.
// ---------------------------------------------------------------------------------------
// rows a lane: 6 for d = 2, 3 (measured n = 2^26: d = 3 1.45 -> 1.40 ms, d = 2 0.89 -> 0.86 ms
// against 8; 4 is slower everywhere), 8 for d = 1 (0.63 vs 0.68 ms) and d = 4
template <int D>
struct WS {
#ifdef PSP_WSWEEP_SR
  static constexpr int SR = PSP_WSWEEP_SR;
#else
  static constexpr int SR = (D == 2 || D == 3) ? 6 : 8;
#endif
  static constexpr int T = 32 * SR;   // rows a warp-tile
};
constexpr int WWPB = 4;           // warps a block (independent ranges)
constexpr int NRMAX = 4096;       // ranges a sweep (scan capacity: 4 maps a scan thread)
#ifndef PSP_WSWEEP_RELOAD
#define PSP_WSWEEP_RELOAD 0       // 1: reload a lane's rows for the final walk instead of holding them
#endif
#ifndef PSP_WSWEEP_PF
#define PSP_WSWEEP_PF 1           // L2 bulk prefetch distance in warp-tiles (0: none)
#endif
#ifndef PSP_WSWEEP_BMINB
#define PSP_WSWEEP_BMINB 3        // blocks per SM asked of the d = 3 backward sweep (202 -> 166
#endif                            // registers, no spills: n = 2^26 1.34 -> 1.23 ms)
#ifndef PSP_WSWEEP_MINB
#define PSP_WSWEEP_MINB 1         // resident blocks per SM asked of the register allocator
#endif

template <bool FWD, int D>
__device__ __forceinline__ Map<D> shfl_scan_src(const Map<D>& m, int off) {
  Map<D> r;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    r.t[i] = FWD ? __shfl_up_sync(0xffffffffu, m.t[i], off) : __shfl_down_sync(0xffffffffu, m.t[i], off);
#pragma unroll
    for (int j = 0; j < D; ++j)
      r.M[i][j] = FWD ? __shfl_up_sync(0xffffffffu, m.M[i][j], off) : __shfl_down_sync(0xffffffffu, m.M[i][j], off);
  }
  return r;
}

// APPLY = false: walk every range from a zero incoming state, write out = addend + y0 (if out)
//                and the range map (M, t) into rmap.
// APPLY = true:  re-walk, from the exact incoming state in rmap, only the ranges flagged in full.
template <bool FWD, int D, bool APPLY>
__global__ void __launch_bounds__(32 * WWPB, (!FWD && D == 3) ? PSP_WSWEEP_BMINB : PSP_WSWEEP_MINB) wsweep_kernel(const double* __restrict__ lu, int64_t n,
                                                           const double* __restrict__ vin, const double* vscale,
                                                           const double* addend, double* out, int64_t L, int nr,
                                                           double* __restrict__ rmap,
                                                           const double* __restrict__ full, int vec) {
  constexpr int DW = D * D + 2 * D;
  constexpr int WSR = WS<D>::SR, WT = WS<D>::T;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * WWPB + (threadIdx.x >> 5);
  if (r >= nr) return;                               // warp-uniform
  if (APPLY && full[r] == 0.0) return;               // tile_fix_kernel completed this range
  constexpr int last = FWD ? 31 : 0;                 // last lane of a warp-tile in processing order
  const int64_t ntiles = (n + WT - 1) / WT;
  const double vsc = vscale ? *vscale : 1.0;
  double carried[D];
#pragma unroll
  for (int i = 0; i < D; ++i) carried[i] = APPLY ? rmap[(int64_t)r * DW + D * D + D + i] : 0.0;
  Map<D> range = identity_map<D>();                  // valid in lane `last`
  const int64_t p0 = (int64_t)r * L, p1 = (p0 + L < ntiles) ? p0 + L : ntiles;
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t tile = FWD ? p : ntiles - 1 - p;
    const int64_t rb = tile * WT + (int64_t)lane * WSR;   // this lane's first row
    const bool whole = rb + WSR <= n;
    if (PSP_WSWEEP_PF > 0 && vec && p + PSP_WSWEEP_PF < p1 && lane < 2 + D) {
      // the rows of the warp-tile PSP_WSWEEP_PF ahead into L2 (one bulk prefetch per array), so
      // its loads do not wait a full DRAM latency after the scans before it
      const int64_t nb0 = (FWD ? tile + PSP_WSWEEP_PF : tile - PSP_WSWEEP_PF) * WT;
      if (nb0 + WT <= n) {
        const double* a = lane == 0 ? vin
                        : lane <= D ? lu + (int64_t)(FWD ? (D - lane) : (D + lane)) * n
                                    : lu + (int64_t)D * n;
        if (a != nullptr && (FWD ? lane <= D : true))
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + nb0), "r"((unsigned)(WT * 8)) : "memory");
      }
    }
    double vv[WSR], cc[D][WSR], uu[WSR];
    auto load_rows = [&]() {
      if (vec && whole) {
#pragma unroll
        for (int q = 0; q < WSR; q += 2) {
          double2 a = vin ? __ldg(reinterpret_cast<const double2*>(vin + rb + q)) : make_double2(0.0, 0.0);
          vv[q] = vsc * a.x;
          vv[q + 1] = vsc * a.y;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            // FWD: c[k] = L(i, i-k-1) = lu[(D-1-k) n + i];  BWD: c[k] = U(i, i+k+1) = lu[(D+1+k) n + i]
            const int o = FWD ? (D - 1 - k) : (D + 1 + k);
            const double2 c2 = __ldg(reinterpret_cast<const double2*>(lu + (int64_t)o * n + rb + q));
            cc[k][q] = c2.x;
            cc[k][q + 1] = c2.y;
          }
          if (!FWD) {
            const double2 u2 = __ldg(reinterpret_cast<const double2*>(lu + (int64_t)D * n + rb + q));
            uu[q] = u2.x;
            uu[q + 1] = u2.y;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < WSR; ++q) {
          const int64_t i = rb + q;
          const bool in = i < n;
          vv[q] = (in && vin) ? vsc * __ldg(vin + i) : 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const int o = FWD ? (D - 1 - k) : (D + 1 + k);
            cc[k][q] = in ? __ldg(lu + (int64_t)o * n + i) : 0.0;
          }
          uu[q] = (!FWD && in) ? __ldg(lu + (int64_t)D * n + i) : 1.0;
        }
      }
      if (!FWD) {
#pragma unroll
        for (int q = 0; q < WSR; ++q) uu[q] = recip_pivot(uu[q]);   // once a row
      }
    };
    load_rows();
    // the lane's map: zero-state run + the D unit-state runs (padding rows >= n are skipped)
    double sz[D], su[D][D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      sz[k] = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q) su[q][k] = (q == k) ? 1.0 : 0.0;
    }
#pragma unroll
    for (int rr = 0; rr < WSR; ++rr) {
      const int q = FWD ? rr : (WSR - 1 - rr);
      if (rb + q >= n) continue;
      double c[D];
#pragma unroll
      for (int k = 0; k < D; ++k) c[k] = cc[k][q];
      const double u0 = FWD ? 1.0 : uu[q];
      push_state<D>(sz, rec_step<FWD, D>(vv[q], c, sz, u0));
#pragma unroll
      for (int s = 0; s < D; ++s) push_state<D>(su[s], rec_step<FWD, D>(0.0, c, su[s], u0));
    }
    Map<D> inc;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      inc.t[i] = sz[i];
#pragma unroll
      for (int s = 0; s < D; ++s) inc.M[i][s] = su[s][i];
    }
    // inclusive scan of the lane maps in processing order
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const Map<D> o = shfl_scan_src<FWD, D>(inc, off);
      const bool has = FWD ? (lane >= off) : (lane + off < 32);
      if (has) inc = compose<D>(inc, o);
    }
    double sinc[D], st[D];
    apply<D>(inc, carried, sinc);                    // the state after this lane's rows
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double prev = FWD ? __shfl_up_sync(0xffffffffu, sinc[i], 1) : __shfl_down_sync(0xffffffffu, sinc[i], 1);
      st[i] = (lane == (FWD ? 0 : 31)) ? carried[i] : prev;   // the state entering this lane
    }
    if (!APPLY && lane == last) range = compose<D>(inc, range);
#pragma unroll
    for (int i = 0; i < D; ++i) carried[i] = __shfl_sync(0xffffffffu, sinc[i], last);
    if (out != nullptr) {
      // RELOAD: the rows again (L1 / L2 hits), so that they are not live across the scan
      if (PSP_WSWEEP_RELOAD) load_rows();
      double y[WSR];
#pragma unroll
      for (int rr = 0; rr < WSR; ++rr) {
        const int q = FWD ? rr : (WSR - 1 - rr);
        if (rb + q >= n) { y[q] = 0.0; continue; }
        double c[D];
#pragma unroll
        for (int k = 0; k < D; ++k) c[k] = cc[k][q];
        y[q] = rec_step<FWD, D>(vv[q], c, st, FWD ? 1.0 : uu[q]);
        push_state<D>(st, y[q]);
      }
      if (vec && whole) {
#pragma unroll
        for (int q = 0; q < WSR; q += 2) {
          double2 w = make_double2(y[q], y[q + 1]);
          if (addend) {
            const double2 a = *reinterpret_cast<const double2*>(addend + rb + q);
            w.x += a.x;
            w.y += a.y;
          }
          *reinterpret_cast<double2*>(out + rb + q) = w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < WSR; ++q)
          if (rb + q < n) out[rb + q] = addend ? addend[rb + q] + y[q] : y[q];
      }
    }
  }
  if (!APPLY && lane == last) {
    double* dd = rmap + (int64_t)r * DW;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      dd[D * D + i] = range.t[i];
#pragma unroll
      for (int j = 0; j < D; ++j) dd[i * D + j] = range.M[i][j];
    }
  }
}

// one block: exact incoming state of up to NRMAX ranges (G consecutive ranges a thread: a local
// composition, the block scan of the thread aggregates, then the thread's ranges in order)
template <bool FWD, int D>
__global__ void __launch_bounds__(SCAN_T, 1) wscan_kernel(int nr, double* __restrict__ rmap,
                                                          const double* s_in0, double* s_out) {
  extern __shared__ double smem_dyn[];
  Map<D>* sm = reinterpret_cast<Map<D>*>(smem_dyn);   // [SCAN_T]
  constexpr int DW = D * D + 2 * D;
  const int t = threadIdx.x;
  const int G = (nr + SCAN_T - 1) / SCAN_T;
  const int j0 = t * G, j1 = (j0 + G < nr) ? j0 + G : nr;
  auto load = [&](int j) {
    Map<D> m;
    const double* dd = rmap + (int64_t)j * DW;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      m.t[i] = dd[D * D + i];
#pragma unroll
      for (int k = 0; k < D; ++k) m.M[i][k] = dd[i * D + k];
    }
    return m;
  };
  Map<D> agg = identity_map<D>();
  for (int j = j0; j < j1; ++j) agg = compose<D>(load(j), agg);
  sm[t] = agg;
  __syncthreads();
  for (int off = 1; off < SCAN_T; off <<= 1) {      // inclusive (later ranges applied last)
    Map<D> o = identity_map<D>();
    if (t >= off) o = sm[t - off];
    __syncthreads();
    if (t >= off) sm[t] = compose<D>(sm[t], o);
    __syncthreads();
  }
  double s0[D], s[D];
#pragma unroll
  for (int i = 0; i < D; ++i) s0[i] = s_in0 ? s_in0[i] : 0.0;
  if (t > 0) apply<D>(sm[t - 1], s0, s);
  else
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = s0[i];
  for (int j = j0; j < j1; ++j) {
    const Map<D> m = load(j);
#pragma unroll
    for (int i = 0; i < D; ++i) rmap[(int64_t)j * DW + D * D + D + i] = s[i];
    double s1[D];
    apply<D>(m, s, s1);
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = s1[i];
  }
  if (s_out && t == SCAN_T - 1) {
    double so[D];
    apply<D>(sm[SCAN_T - 1], s0, so);
#pragma unroll
    for (int i = 0; i < D; ++i) s_out[i] = so[i];
  }
}

// Warm-start check: chunk c's start state (from its warm-up rows) against chunk c-1's end state,
// bitwise; any difference sends the factorisation to the exact fixed-point passes.
__global__ void factor_verify_kernel(const double* __restrict__ st_start, const double* __restrict__ st_end,
                                     int64_t nchunks, int W, int* __restrict__ changed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (nchunks - 1) * W) return;
  const int64_t c = i / W + 1, e = i % W;
  if (__double_as_longlong(st_start[c * W + e]) != __double_as_longlong(st_end[(c - 1) * W + e]))
    atomicAdd(changed, 1);
}

template <int D>
void factor_launch(const double* bands, int64_t n, double* lu, const double* a, double* b,
                   int first, int* changed, int* bad, const double* prev, int has_prev, int has_next,
                   cudaStream_t s, bool write, int warm = 0, double* st_start = nullptr) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int tpb = PSP_FACTOR_TPB;
  const int vec = (n % 2 == 0) && (((uintptr_t)bands | (uintptr_t)lu) & 15) == 0;
  static const bool no_coop = getenv("PSP_FACTOR_NOCOOP") != nullptr;   // A/B: per-thread copies
  const bool coop = D <= PSP_FACTOR_PFMAXD && vec && !no_coop;
  const unsigned grid = (unsigned)((nchunks + tpb - 1) / tpb);
  constexpr int kPF = kPFd<D>;
  const size_t smem = D <= PSP_FACTOR_PFMAXD ? (size_t)kPF * (2 * D + 1) * tpb * (coop ? PSP_FACTOR_G + 2 : 4) * 8 : 0;
  thread_local bool attr[kMaxDev] = {};
  const int dev = device_ordinal();
  if (!attr[dev]) {
    const int s4 = D <= PSP_FACTOR_PFMAXD ? kPF * (2 * D + 1) * tpb * 4 * 8 : 0, s8 = s4 * (PSP_FACTOR_G + 2) / 4;
    cudaFuncSetAttribute(factor_pass_kernel<D, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4);
    cudaFuncSetAttribute(factor_pass_kernel<D, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4);
    if (D <= PSP_FACTOR_PFMAXD) {
      cudaFuncSetAttribute(factor_pass_kernel<D, true, (D <= PSP_FACTOR_PFMAXD)>, cudaFuncAttributeMaxDynamicSharedMemorySize, s8);
      cudaFuncSetAttribute(factor_pass_kernel<D, false, (D <= PSP_FACTOR_PFMAXD)>, cudaFuncAttributeMaxDynamicSharedMemorySize, s8);
    }
    attr[dev] = true;
  }
#define PSP_FACTOR_GO(WR, CO)                                                                      \
  factor_pass_kernel<D, WR, CO><<<grid, tpb, smem, s>>>(bands, n, lu, a, b, first, changed, bad, prev, \
                                                        has_prev, has_next, vec, warm, st_start)
  if (coop) {
    if (write) PSP_FACTOR_GO(true, (D <= PSP_FACTOR_PFMAXD));
    else PSP_FACTOR_GO(false, (D <= PSP_FACTOR_PFMAXD));
  } else {
    if (write) PSP_FACTOR_GO(true, false);
    else PSP_FACTOR_GO(false, false);
  }
#undef PSP_FACTOR_GO
}

// phase 0: the whole sweep; 1: map (zero-state rows written to out) + scan (s_out = the state after
// the last row from s_in0); 2: scan from s_in0 + fix + apply over the maps and rows phase 1 left
// (multi-rank: the incoming state is known only after the ranks' outgoing states are gathered)
template <bool FWD, int D>
void sweep_launch(const double* lu, int64_t n, const double* v, const double* vs, const double* add,
                  double* out, BandedScratch sc, cudaStream_t s, const double* s_in0, double* s_out, int phase) {
  const size_t smem = TileSmem<FWD, D>::BYTES;
  const size_t ssmem = (size_t)SCAN_T * sizeof(Map<D>);
  thread_local bool attr_set[kMaxDev] = {};
  thread_local int wblocks[kMaxDev] = {};            // resident warp-range blocks per SM
  const int dev = device_ordinal();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(tile_map_kernel<FWD, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tile_apply_kernel<FWD, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tile_scan_kernel<FWD, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
    cudaFuncSetAttribute(wscan_kernel<FWD, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wsweep_kernel<FWD, D, false>, 32 * WWPB, 0) !=
            cudaSuccess || per < 1)
      per = 1;
    wblocks[dev] = per;
    attr_set[dev] = true;
  }
  double* full = sc.states + (size_t)NRMAX * (D * D + 2 * D);   // per-range flag
  static const bool block_sweeps = getenv("PSP_SOLVE_BLOCK") != nullptr;   // A/B: the tile kernels
  if (!block_sweeps) {
    // one range per resident warp (one wave), at most NRMAX
    constexpr int WT = WS<D>::T;
    const int64_t ntiles = (n + WT - 1) / WT;
    int64_t nr = (int64_t)device_sms() * wblocks[dev] * WWPB;
    if (nr > NRMAX) nr = NRMAX;
    if (nr > ntiles) nr = ntiles;
    if (nr < 1) nr = 1;
    const int64_t L = (ntiles + nr - 1) / nr;
    nr = ntiles > 0 ? (ntiles + L - 1) / L : 0;
    const unsigned nb = (unsigned)((nr + WWPB - 1) / WWPB);
    const int vec = (n % 2 == 0) && ((((uintptr_t)lu) | ((uintptr_t)v) | ((uintptr_t)add) | ((uintptr_t)out)) & 15) == 0;
    if (ntiles > 0 && phase != 2)
      wsweep_kernel<FWD, D, false><<<nb, 32 * WWPB, 0, s>>>(lu, n, v, vs, add, out, L, (int)nr, sc.states,
                                                             nullptr, vec);
    wscan_kernel<FWD, D><<<1, SCAN_T, ssmem, s>>>((int)nr, sc.states, s_in0, s_out);
    if (out != nullptr && ntiles > 0 && phase != 1) {
      tile_fix_kernel<FWD, D><<<(unsigned)((nr + 63) / 64), 64, 0, s>>>(lu, n, L, (int)nr, out, sc.states, full, WT);
      wsweep_kernel<FWD, D, true><<<nb, 32 * WWPB, 0, s>>>(lu, n, v, vs, add, out, L, (int)nr, sc.states, full, vec);
    }
    return;
  }
  const int64_t ntiles = (n + SW<D>::TILE - 1) / SW<D>::TILE;
  // ranges: at most SCAN_T blocks (2 resident per SM), each a contiguous run of L tiles
  const int64_t nbmax = (int64_t)device_sms() * SW<D>::MINB * 3;
  int64_t nb = ntiles < nbmax ? ntiles : nbmax;
  if (nb > SCAN_T) nb = SCAN_T;
  if (nb < 1) nb = 1;
  const int64_t L = (ntiles + nb - 1) / nb;
  nb = (ntiles + L - 1) / L;
  if (ntiles > 0 && phase != 2)
    tile_map_kernel<FWD, D><<<(unsigned)nb, SW<D>::TPB, smem, s>>>(lu, n, v, vs, add, out, L, sc.states);
  tile_scan_kernel<FWD, D><<<1, SCAN_T, ssmem, s>>>(ntiles > 0 ? (int)nb : 0, sc.states, s_in0, s_out);
  if (out != nullptr && ntiles > 0 && phase != 1) {
    tile_fix_kernel<FWD, D><<<(unsigned)((nb + 63) / 64), 64, 0, s>>>(lu, n, L, (int)nb, out, sc.states, full,
                                                                      SW<D>::TILE);
    tile_apply_kernel<FWD, D><<<(unsigned)nb, SW<D>::TPB, smem, s>>>(lu, n, v, vs, add, out, L, sc.states, full);
  }
}

void sweep(bool fwd, int d, const double* lu, int64_t n, const double* v, const double* vs,
           const double* add, double* out, BandedScratch sc, cudaStream_t s, const double* s_in0,
           double* s_out, int phase = 0) {
#define PSP_SWEEP(DD)                                                                   \
  if (fwd) sweep_launch<true, DD>(lu, n, v, vs, add, out, sc, s, s_in0, s_out, phase); \
  else sweep_launch<false, DD>(lu, n, v, vs, add, out, sc, s, s_in0, s_out, phase);
  switch (d) {
    case 1: PSP_SWEEP(1) break;
    case 2: PSP_SWEEP(2) break;
    case 3: PSP_SWEEP(3) break;
    default: PSP_SWEEP(4) break;
  }
#undef PSP_SWEEP
}

// multi-rank helpers (one thread)
__global__ void flags_to_double_kernel(const int* f, double* out) {
  out[0] = (double)f[0];
  out[1] = (double)f[1];
}
__global__ void unit_vector_kernel(double* e, int d, int i) {
  for (int q = 0; q < d; ++q) e[q] = (q == i) ? 1.0 : 0.0;
}
__global__ void copy_col_kernel(const double* src, double* M, int d, int i) {
  for (int q = 0; q < d; ++q) M[q * d + i] = src[q];   // column i of the row-major d x d map
}
// incoming state of this rank: compose the affine maps s <- M_q s + t_q of the ranks before it
// (forward: q = 0..rank-1; backward: q = nranks-1..rank+1); identical arithmetic on every rank
__global__ void compose_states_kernel(const double* Mall, const double* tall, int d, int nranks,
                                      int rank, int fwd, double* sin) {
  double s[kMaxD] = {0.0, 0.0, 0.0, 0.0}, t2[kMaxD];
  if (fwd) {
    for (int q = 0; q < rank; ++q) {
      for (int i = 0; i < d; ++i) {
        double v = tall[q * d + i];
        for (int j = 0; j < d; ++j) v = fma(Mall[(q * d + i) * d + j], s[j], v);
        t2[i] = v;
      }
      for (int i = 0; i < d; ++i) s[i] = t2[i];
    }
  } else {
    for (int q = nranks - 1; q > rank; --q) {
      for (int i = 0; i < d; ++i) {
        double v = tall[q * d + i];
        for (int j = 0; j < d; ++j) v = fma(Mall[(q * d + i) * d + j], s[j], v);
        t2[i] = v;
      }
      for (int i = 0; i < d; ++i) s[i] = t2[i];
    }
  }
  for (int i = 0; i < d; ++i) sin[i] = s[i];
}

}  // namespace

// scratch: [ctl 4 x u64 | changed/bad 2 x int (16 B) | flags ntiles x u64 | desc ntiles x DW |
//           fixed-point states 2 x nchunks x D(D+1) | y n]
size_t banded_scratch_bytes(int64_t n, int d) {
  const int64_t ntiles = (n + STILE - 1) / STILE;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t DW = d * d + 2 * d;
  size_t b = 64 + 256;
  b += (size_t)ntiles * 8 + 256;
  b += (size_t)((ntiles > NRMAX ? ntiles : NRMAX) * DW + NRMAX) * 8 + 256;   // range maps + flags
  b += (size_t)2 * nchunks * d * (d + 1) * 8 + 256;
  b += (size_t)n * 8 + 256;
  return b;
}

static inline char* align256(char* p) { return (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255); }

BandedScratch banded_scratch(void* base, int64_t n, int d) {
  BandedScratch sc;
  const int64_t ntiles = (n + STILE - 1) / STILE;
  const int64_t DW = d * d + 2 * d;
  char* p = align256((char*)base);
  sc.tickets = (unsigned long long*)p;          // [0..3] ctl, [4..] flags
  sc.changed = (int*)(p + 32);                  // [0] changed, [1] bad
  p = align256(p + 64 + (size_t)ntiles * 8 + 64);
  sc.states = (double*)p;                       // range maps / states + flags (solve)
  p = align256(p + (size_t)((ntiles > NRMAX ? ntiles : NRMAX) * DW + NRMAX) * 8);
  sc.y = (double*)p;                            // intermediate vector, then factor states
  sc.desc_count = ntiles;
  return sc;
}

// The control words must be zero before the first use of a scratch (ctl epoch starts at 0).
static double* factor_states(BandedScratch sc, int64_t n) {
  return sc.y + ((n + 31) / 32) * 32;
}

// misc (multi-rank) layout, doubles: [prev W | dummy W | flags 2 | e d | col d | Mf p*d*d |
// Mb p*d*d | t d | tall p*d | sin d]
namespace {
struct Misc {
  double *prev, *dummy, *flags, *e, *col, *mine, *Mf, *Mb, *t, *tall, *sin;
  Misc(double* m, int d, int p) {
    const int W = d * (d + 1);
    prev = m;
    dummy = prev + W;
    flags = dummy + W;
    e = flags + 2;
    col = e + d;
    mine = col + d;
    Mf = mine + d * d;
    Mb = Mf + (size_t)p * d * d;
    t = Mb + (size_t)p * d * d;
    tall = t + d;
    sin = tall + (size_t)p * d;
  }
};
}  // namespace

size_t banded_misc_doubles(int d, int nranks) {
  return (size_t)2 * d * (d + 1) + 2 + 2 * d + d * d + (size_t)2 * nranks * d * d + d +
         (size_t)nranks * d + d;
}

int banded_factor(const double* bands, int64_t n, int d, double* lu, BandedScratch sc,
                  cudaStream_t s, int* passes, int64_t* launches, psp_comm* comm, double* misc) {
  const bool multi = comm && comm->nranks > 1;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int W = d * (d + 1);
  double* A = factor_states(sc, n);
  double* B = A + nchunks * W;
  Misc M(misc, d, multi ? comm->nranks : 1);
  int h[2] = {0, 0};
  double hd[2] = {0.0, 0.0};
  int p = 0;
  bool write = false;   // state-only passes until no chunk state changes, then one LU pass
  if (!multi && nchunks > 1) {
    // one LU-writing pass from warm-started chunk states (the solve's intermediate vector is
    // free during the factorisation and holds the start states), then the bitwise check; only
    // if some chunk's state had not converged do the exact fixed-point passes follow
    double* S0 = sc.y;
    cudaMemsetAsync(sc.changed, 0, 2 * sizeof(int), s);
    switch (d) {
      case 1: factor_launch<1>(bands, n, lu, A, B, 1, sc.changed, sc.changed + 1, nullptr, 0, 0, s, true, kWarm, S0); break;
      case 2: factor_launch<2>(bands, n, lu, A, B, 1, sc.changed, sc.changed + 1, nullptr, 0, 0, s, true, kWarm, S0); break;
      case 3: factor_launch<3>(bands, n, lu, A, B, 1, sc.changed, sc.changed + 1, nullptr, 0, 0, s, true, kWarm, S0); break;
      default: factor_launch<4>(bands, n, lu, A, B, 1, sc.changed, sc.changed + 1, nullptr, 0, 0, s, true, kWarm, S0); break;
    }
    cudaMemsetAsync(sc.changed, 0, sizeof(int), s);   // the pass counted every chunk as changed
    const int64_t nv = (nchunks - 1) * W;
    factor_verify_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, s>>>(S0, B, nchunks, W, sc.changed);
    if (launches) *launches += 2;
    p = 1;
    cudaMemcpyAsync(h, sc.changed, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double* tmp = A;
    A = B;
    B = tmp;
    if (h[0] == 0) {
      if (passes) *passes = p;
      return h[1] ? PSP_E_SINGULAR : PSP_OK;
    }
  }
  for (;;) {
    cudaMemsetAsync(sc.changed, 0, 2 * sizeof(int), s);
    const double* prev = (multi && comm->rank > 0 && p > 0) ? M.prev : nullptr;
    const int hp = (multi && comm->rank > 0) ? 1 : 0;
    const int hn = (multi && comm->rank < comm->nranks - 1) ? 1 : 0;
    switch (d) {
      case 1: factor_launch<1>(bands, n, lu, A, B, p == 0, sc.changed, sc.changed + 1, prev, hp, hn, s, write); break;
      case 2: factor_launch<2>(bands, n, lu, A, B, p == 0, sc.changed, sc.changed + 1, prev, hp, hn, s, write); break;
      case 3: factor_launch<3>(bands, n, lu, A, B, p == 0, sc.changed, sc.changed + 1, prev, hp, hn, s, write); break;
      default: factor_launch<4>(bands, n, lu, A, B, p == 0, sc.changed, sc.changed + 1, prev, hp, hn, s, write); break;
    }
    if (launches) *launches += 1;
    ++p;
    if (multi) {
      // the outgoing state of this rank's last chunk goes to rank+1 (its chunk 0 next pass)
      if (comm->sendrecv(M.dummy, M.prev, (size_t)W, B + (nchunks - 1) * W, M.dummy, (size_t)W, s)) return PSP_E_NCCL;
      flags_to_double_kernel<<<1, 1, 0, s>>>(sc.changed, M.flags);
      if (comm->allreduce(M.flags, 2, 0, s)) return PSP_E_NCCL;
      cudaMemcpyAsync(hd, M.flags, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      h[0] = (int)hd[0];
      h[1] = (int)hd[1];
    } else {
      cudaMemcpyAsync(h, sc.changed, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
    }
    double* tmp = A;
    A = B;
    B = tmp;
    if (write) break;                 // the LU pass from the converged states
    if (h[0] == 0 || p > nchunks * (multi ? comm->nranks : 1) + 1) write = true;
  }
  if (passes) *passes = p;
  if (h[1]) return PSP_E_SINGULAR;
  if (multi) {
    // this rank's homogeneous transfer maps (forward and backward), d unit-state sweeps each,
    // all-gathered so that every rank can compose the states entering it (banded_solve)
    for (int fwd = 1; fwd >= 0; --fwd) {
      for (int i = 0; i < d; ++i) {
        unit_vector_kernel<<<1, 1, 0, s>>>(M.e, d, i);
        sweep(fwd != 0, d, lu, n, nullptr, nullptr, nullptr, nullptr, sc, s, M.e, M.col);
        copy_col_kernel<<<1, 1, 0, s>>>(M.col, M.mine, d, i);
      }
      if (comm->allgather(M.mine, fwd ? M.Mf : M.Mb, (size_t)d * d, s)) return PSP_E_NCCL;
      if (launches) *launches += 3 * d;
    }
  }
  return PSP_OK;
}

// z = x0 + N^{-1}(vs v).  Multi-rank: each sweep is still ONE pass over the rows -- the zero-
// state pass writes its rows and yields this rank's outgoing state t_r; an all-gather of the t's;
// the state entering this rank composed from the ranks before it (maps from banded_factor); then
// only the range scan and the decaying homogeneous corrections from that state (tile_fix, and
// tile_apply for a range whose correction has not decayed).
int banded_solve(const double* lu, int64_t n, int d, const double* v, const double* vs,
                 const double* x0, double* z, BandedScratch sc, cudaStream_t s, int64_t* launches,
                 psp_comm* comm, double* misc) {
  if (!(comm && comm->nranks > 1)) {
    sweep(true, d, lu, n, v, vs, nullptr, sc.y, sc, s, nullptr, nullptr);
    sweep(false, d, lu, n, sc.y, nullptr, x0, z, sc, s, nullptr, nullptr);
    if (launches) *launches += 8;   // per sweep: map, scan, fix, apply
    return PSP_OK;
  }
  Misc M(misc, d, comm->nranks);
  for (int fwd = 1; fwd >= 0; --fwd) {
    const double* vin = fwd ? v : sc.y;
    const double* vsc = fwd ? vs : nullptr;
    const double* add = fwd ? nullptr : x0;
    double* out = fwd ? sc.y : z;
    sweep(fwd != 0, d, lu, n, vin, vsc, add, out, sc, s, nullptr, M.t, 1);
    if (comm->allgather(M.t, M.tall, (size_t)d, s)) return PSP_E_NCCL;
    compose_states_kernel<<<1, 1, 0, s>>>(fwd ? M.Mf : M.Mb, M.tall, d, comm->nranks, comm->rank, fwd,
                                          M.sin);
    sweep(fwd != 0, d, lu, n, vin, vsc, add, out, sc, s, M.sin, nullptr, 2);
  }
  if (launches) *launches += 12;   // per sweep: map + scan, compose, scan + fix + apply
  return PSP_OK;
}

}  // namespace psp
