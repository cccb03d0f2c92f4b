// stencil.cu -- K1: matrix-free y = A x = (I - dt L) x  (Eq.4; "replacing the
// matrix-vector product in the GMRES algorithm with residual computation").
//
// HBM-bound: algorithmic bytes per row = 8 (x) + 8 (field, CELL_* only) + 8 (y) [+ 8 when the
// probe copy P_x is written in the same pass].  One thread per grid point, blocks of 128
// threads along x; the +-x neighbours come from the same warp's lines, the +-y / +-z
// neighbours from L1/L2 (three planes of x and kappa are ~12 MB at 512^2, well inside the
// 126 MB L2), so DRAM sees each array once.
#include <stdlib.h>

#include "cg.cuh"
#include "internal.h"
#include "reduce.cuh"
#include "stencil_row.cuh"

#ifndef PSP_MARCH_MINB
#define PSP_MARCH_MINB 3   // resident blocks per SM of the vectorised march kernel
#endif

namespace psp {
namespace {

template <int KIND, int NDIM>
__global__ void __launch_bounds__(128) matvec_kernel(Stencil st, const double* __restrict__ x,
                                                     const double* xsp, double* __restrict__ y,
                                                     double* __restrict__ xcopy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= st.nx) return;
  const int64_t g = i + st.nx * (blockIdx.y + st.ny * (int64_t)blockIdx.z);
  const double xs = xsp ? *xsp : 1.0;
  double xc;
  const double ax = stencil_row<KIND, NDIM>(st, x, i, blockIdx.y, blockIdx.z, g, xc);
  // (the scale xs is linear: applied once to the result and to the probe copy)
  y[g] = xs * ax;
  if (xcopy != nullptr) xcopy[g] = xs * xc;
}

// ------------------------------------------------------------------------------------------
// 2.5-D marching kernel for 2-D / 3-D grids (the C2-C4 operators).  A block owns a BX x BY
// tile of the (x, y) plane and marches a chunk of planes along the slab axis (z in 3-D, y in
// 2-D, where the tile is BX x 1).  The slab-axis neighbours stay in registers (a queue of the
// planes below / at / above, prefetched two planes ahead), the in-plane neighbours come from a
// double-buffered shared-memory copy of the plane with its one-point halo ring, so DRAM sees
// x and the coefficient field once per chunk (+2 halo planes per chunk) and the kernel keeps
// 2 x 8 B loads per thread in flight for the next two planes.  Arithmetic per point is the
// same sequence of operations as matvec_kernel (bitwise-identical results).
// ------------------------------------------------------------------------------------------
struct MarchView {
  int64_t nx, ny, nz;        // tile plane nx x ny, march axis nz
  double s[3], a[3];         // axis 0 = x, 1 = in-plane y (3-D only), 2 = march axis
  const double* field;
  const double* x_lo;        // multi-rank halo planes along the march axis (NULL: Dirichlet)
  const double* x_hi;
  const double* f_lo;
  const double* f_hi;
  int zc;                    // planes per block
};

template <int KIND, int BX, int BY>
__global__ void __launch_bounds__(BX * BY, 4) march_matvec_kernel(MarchView v, const double* __restrict__ x,
                                                              const double* xsp, double* __restrict__ y,
                                                              double* __restrict__ xcopy) {
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr bool HASY = BY > 1;
  constexpr int SX = BX + 2, SY = HASY ? BY + 2 : 1;
  __shared__ double sx[2][SY][SX];
  __shared__ double sf[2][cell ? SY : 1][cell ? SX : 1];
  const double* __restrict__ f = v.field;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t i = (int64_t)blockIdx.x * BX + tx;
  const int64_t j = HASY ? (int64_t)blockIdx.y * BY + ty : 0;
  const int64_t z0 = (int64_t)blockIdx.z * v.zc;
  const int64_t z1 = (z0 + v.zc < v.nz) ? z0 + v.zc : v.nz;
  const bool in = i < v.nx && j < v.ny;
  const int64_t plane = v.nx * v.ny;
  const int64_t col = i + v.nx * j;          // in-plane index
  const int sy = HASY ? ty + 1 : 0;
  // halo duty: x halo for tx == 0 / BX-1, y halo for ty == 0 / BY-1
  const int hxdir = (tx == 0) ? -1 : (tx == BX - 1 ? 1 : 0);
  const int hydir = HASY ? ((ty == 0) ? -1 : (ty == BY - 1 ? 1 : 0)) : 0;
  const bool hx_in = hxdir != 0 && (i + hxdir) >= 0 && (i + hxdir) < v.nx && j < v.ny;
  const bool hy_in = hydir != 0 && (j + hydir) >= 0 && (j + hydir) < v.ny && i < v.nx;
  const int64_t hx_col = col + hxdir;
  const int64_t hy_col = col + hydir * v.nx;

  // march-axis value of x / field at plane p (halo planes beyond the local slab)
  auto ldx = [&](int64_t p) -> double {
    if (!in) return 0.0;
    if (p >= 0 && p < v.nz) return __ldg(x + col + plane * p);
    if (p < 0 && v.x_lo) return __ldg(v.x_lo + col);
    if (p >= v.nz && v.x_hi) return __ldg(v.x_hi + col);
    return 0.0;
  };
  auto ldf = [&](int64_t p) -> double {
    if (!cell || !in) return 0.0;
    if (p >= 0 && p < v.nz) return __ldg(f + col + plane * p);
    if (p < 0 && v.f_lo) return __ldg(v.f_lo + col);
    if (p >= v.nz && v.f_hi) return __ldg(v.f_hi + col);
    return 0.0;
  };
  const bool lo_in = v.x_lo != nullptr;      // a neighbour plane exists below local plane 0
  const bool hi_in = v.x_hi != nullptr;
  const double xs = xsp ? *xsp : 1.0;

  double xb = ldx(z0 - 1), xc = ldx(z0), xt = ldx(z0 + 1), xt2 = ldx(z0 + 2);
  double fb = ldf(z0 - 1), fc = ldf(z0), ft = ldf(z0 + 1), ft2 = ldf(z0 + 2);
  double hxv = 0.0, hxf = 0.0, hyv = 0.0, hyf = 0.0;   // halo of the current plane
  if (hx_in && z0 < v.nz) { hxv = __ldg(x + hx_col + plane * z0); if (cell) hxf = __ldg(f + hx_col + plane * z0); }
  if (hy_in && z0 < v.nz) { hyv = __ldg(x + hy_col + plane * z0); if (cell) hyf = __ldg(f + hy_col + plane * z0); }

  for (int64_t z = z0; z < z1; ++z) {
    const int b = (int)(z & 1);
    // prefetch: plane z+3 of the centre column, the halo of plane z+1
    const double xt3 = ldx(z + 3), ft3 = ldf(z + 3);
    double nhxv = 0.0, nhxf = 0.0, nhyv = 0.0, nhyf = 0.0;
    if (z + 1 < z1) {
      if (hx_in) { nhxv = __ldg(x + hx_col + plane * (z + 1)); if (cell) nhxf = __ldg(f + hx_col + plane * (z + 1)); }
      if (hy_in) { nhyv = __ldg(x + hy_col + plane * (z + 1)); if (cell) nhyf = __ldg(f + hy_col + plane * (z + 1)); }
    }
    // stage plane z
    sx[b][sy][tx + 1] = xc;
    if (cell) sf[b][sy][tx + 1] = fc;
    if (hxdir) {
      sx[b][sy][tx + 1 + hxdir] = hxv;
      if (cell) sf[b][sy][tx + 1 + hxdir] = hxf;
    }
    if (HASY && hydir) {
      sx[b][sy + hydir][tx + 1] = hyv;
      if (cell) sf[b][sy + hydir][tx + 1] = hyf;
    }
    __syncthreads();
    if (in) {
      double acc = 0.0;  // sum over faces of s_a * k_f * (x_c - x_nb) + upwind terms
      auto face = [&](double xn, double fn, bool nin, double s) {
        const double kf = cell ? (nin ? 0.5 * (fc + fn) : fc) : 1.0;
        acc = fma(s * kf, xc - xn, acc);
      };
      {
        const bool inw = i > 0, ine = i + 1 < v.nx;
        const double xw = inw ? sx[b][sy][tx] : 0.0, xe = ine ? sx[b][sy][tx + 2] : 0.0;
        face(xw, cell && inw ? sf[b][sy][tx] : 0.0, inw, v.s[0]);
        face(xe, cell && ine ? sf[b][sy][tx + 2] : 0.0, ine, v.s[0]);
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[0], xc - xw, acc);
      }
      if (HASY) {
        const bool ins = j > 0, inn = j + 1 < v.ny;
        const double xsn = ins ? sx[b][sy - 1][tx + 1] : 0.0, xnn = inn ? sx[b][sy + 1][tx + 1] : 0.0;
        face(xsn, cell && ins ? sf[b][sy - 1][tx + 1] : 0.0, ins, v.s[1]);
        face(xnn, cell && inn ? sf[b][sy + 1][tx + 1] : 0.0, inn, v.s[1]);
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[1], xc - xsn, acc);
      }
      {
        const bool inb = z > 0 || lo_in, int_ = z + 1 < v.nz || hi_in;
        face(xb, fb, inb, v.s[2]);
        face(xt, ft, int_, v.s[2]);
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[2], xc - xb, acc);
      }
      const int64_t g = col + plane * z;
      y[g] = xs * (xc + acc);
      if (xcopy != nullptr) xcopy[g] = xs * xc;
    }
    xb = xc; xc = xt; xt = xt2; xt2 = xt3;
    fb = fc; fc = ft; ft = ft2; ft2 = ft3;
    hxv = nhxv; hxf = nhxf; hyv = nhyv; hyf = nhyf;
  }
}

// Vectorised, barrier-free variant (the C2-C4 hot path).  Every thread owns two x-adjacent
// points of one (x, y) line and marches the slab axis: the slab-axis neighbours are a register
// queue prefetched three planes ahead (16-byte loads), the x neighbours come from the adjacent
// lanes by warp shuffles (one 8-byte load per tile row for lanes 0 / 31), the in-plane y
// neighbours are 16-byte loads of the lines j-1 / j+1, which the neighbouring warps of the block
// load as their own centre lines (L1 / L2 hits), so DRAM sees x and the coefficient field
// about once.  No shared memory and no barriers: warps run independently.  The domain
// boundary is folded into the data: a missing neighbour is x = 0 with the centre's
// coefficient, so every face is w = (s/2)(k_c + k_nb), acc += w (x_c - x_nb) -- for a boundary
// face (s/2)(2 k_c) = s k_c exactly, the value the scalar kernels use.  Needs nx even and
// 16-byte aligned vectors (checked at launch; otherwise march_matvec_kernel runs).
template <int KIND, int BY>
__global__ void __launch_bounds__(32 * BY, (BY > 1 ? PSP_MARCH_MINB : 16)) march3_kernel(MarchView v, const double* __restrict__ x,
                                                                    const double* xsp, double* __restrict__ y,
                                                                    double* __restrict__ xcopy) {
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr bool HASY = BY > 1;
  constexpr int TW = 64;
  const double* __restrict__ f = v.field;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int64_t i = (int64_t)blockIdx.x * TW + 2 * lane;    // first of this thread's two points
  const int64_t j = HASY ? (int64_t)blockIdx.y * BY + ty : 0;
  const int64_t z0 = (int64_t)blockIdx.z * v.zc;
  const int64_t z1 = (z0 + v.zc < v.nz) ? z0 + v.zc : v.nz;
  const bool in = i < v.nx && j < v.ny;                     // nx even: both points or none
  const int64_t plane = v.nx * v.ny;
  const int64_t col = in ? i + v.nx * j : 0;                 // outside: loads of point 0, no stores
  const bool has_w = i > 0, has_e = i + 2 < v.nx;
  const bool has_s = HASY && in && j > 0, has_n = HASY && in && j + 1 < v.ny;
  const bool lo_in = v.x_lo != nullptr, hi_in = v.x_hi != nullptr;
  const double xs = xsp ? *xsp : 1.0;
  const double hs0 = 0.5 * v.s[0], hs1 = 0.5 * v.s[1], hs2 = 0.5 * v.s[2];
  const double s0c = v.s[0], s1c = v.s[1], s2c = v.s[2];

  auto ld2 = [&](const double* a, const double* lo, const double* hi, int64_t p) -> double2 {
    if (p >= 0 && p < v.nz) return __ldg(reinterpret_cast<const double2*>(a + col + plane * p));
    if (p < 0 && lo) return __ldg(reinterpret_cast<const double2*>(lo + col));
    if (p >= v.nz && hi) return __ldg(reinterpret_cast<const double2*>(hi + col));
    return make_double2(0.0, 0.0);
  };
  const double2 zero2 = make_double2(0.0, 0.0);
  double2 xb = ld2(x, v.x_lo, v.x_hi, z0 - 1), xc = ld2(x, v.x_lo, v.x_hi, z0);
  double2 xt = ld2(x, v.x_lo, v.x_hi, z0 + 1), xt2 = ld2(x, v.x_lo, v.x_hi, z0 + 2);
  double2 fb = zero2, fc = zero2, ft = zero2, ft2 = zero2;
  if (cell) {
    fb = ld2(f, v.f_lo, v.f_hi, z0 - 1); fc = ld2(f, v.f_lo, v.f_hi, z0);
    ft = ld2(f, v.f_lo, v.f_hi, z0 + 1); ft2 = ld2(f, v.f_lo, v.f_hi, z0 + 2);
  }
  const double* px3 = x + col + plane * (z0 + 3);
  const double* pf3 = f + col + plane * (z0 + 3);
  const double* pxz = x + col + plane * z0;                  // plane z (in-plane neighbour loads)
  const double* pfz = f + col + plane * z0;
  double* py = y + col + plane * z0;
  double* pc = xcopy ? xcopy + col + plane * z0 : nullptr;

  for (int64_t z = z0; z < z1; ++z) {
    double2 xt3 = zero2, ft3 = zero2;
    if (z + 3 < v.nz) {
      xt3 = __ldg(reinterpret_cast<const double2*>(px3));
      if (cell) ft3 = __ldg(reinterpret_cast<const double2*>(pf3));
    } else if (z + 3 == v.nz) {
      xt3 = ld2(x, v.x_lo, v.x_hi, z + 3);
      if (cell) ft3 = ld2(f, v.f_lo, v.f_hi, z + 3);
    }
    // in-plane y neighbours (L1 / L2): missing -> x = 0, k = k_c
    double2 xsn = zero2, xnn = zero2, fsn = fc, fnn = fc;
    if (has_s) {
      xsn = __ldg(reinterpret_cast<const double2*>(pxz - v.nx));
      if (cell) fsn = __ldg(reinterpret_cast<const double2*>(pfz - v.nx));
    }
    if (has_n) {
      xnn = __ldg(reinterpret_cast<const double2*>(pxz + v.nx));
      if (cell) fnn = __ldg(reinterpret_cast<const double2*>(pfz + v.nx));
    }
    // x neighbours: the adjacent lanes' points; lanes 0 / 31 load across the tile edge
    double xw = __shfl_up_sync(0xffffffffu, xc.y, 1), xe = __shfl_down_sync(0xffffffffu, xc.x, 1);
    double fw = 0.0, fe = 0.0;
    if (cell) {
      fw = __shfl_up_sync(0xffffffffu, fc.y, 1);
      fe = __shfl_down_sync(0xffffffffu, fc.x, 1);
    }
    if (lane == 0 && in && has_w) { xw = __ldg(pxz - 1); if (cell) fw = __ldg(pfz - 1); }
    if (lane == 31 && in && has_e) { xe = __ldg(pxz + 2); if (cell) fe = __ldg(pfz + 2); }
    if (!has_w) { xw = 0.0; fw = fc.x; }
    if (!has_e) { xe = 0.0; fe = fc.y; }
    // slab-axis boundary (uniform per block)
    if (z == 0 && !lo_in) fb = fc;
    if (z + 1 == v.nz && !hi_in) ft = fc;
    auto point = [&](double c, double k, double xwv, double fwv, double xev, double fev, double xsv,
                     double fsv, double xnv, double fnv, double xbv, double fbv, double xtv, double ftv) {
      double acc = 0.0;
      if (cell) {
        acc = fma(hs0 * (k + fwv), c - xwv, acc);
        acc = fma(hs0 * (k + fev), c - xev, acc);
      } else {
        acc = fma(s0c, c - xwv, acc);
        acc = fma(s0c, c - xev, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[0], c - xwv, acc);
      if (HASY) {
        if (cell) {
          acc = fma(hs1 * (k + fsv), c - xsv, acc);
          acc = fma(hs1 * (k + fnv), c - xnv, acc);
        } else {
          acc = fma(s1c, c - xsv, acc);
          acc = fma(s1c, c - xnv, acc);
        }
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[1], c - xsv, acc);
      }
      if (cell) {
        acc = fma(hs2 * (k + fbv), c - xbv, acc);
        acc = fma(hs2 * (k + ftv), c - xtv, acc);
      } else {
        acc = fma(s2c, c - xbv, acc);
        acc = fma(s2c, c - xtv, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[2], c - xbv, acc);
      return xs * (c + acc);
    };
    if (in) {
      double2 out;
      out.x = point(xc.x, fc.x, xw, fw, xc.y, fc.y, xsn.x, fsn.x, xnn.x, fnn.x, xb.x, fb.x, xt.x, ft.x);
      out.y = point(xc.y, fc.y, xc.x, fc.x, xe, fe, xsn.y, fsn.y, xnn.y, fnn.y, xb.y, fb.y, xt.y, ft.y);
      *reinterpret_cast<double2*>(py) = out;
      if (pc) *reinterpret_cast<double2*>(pc) = make_double2(xs * xc.x, xs * xc.y);
    }
    px3 += plane; pf3 += plane; pxz += plane; pfz += plane; py += plane;
    if (pc) pc += plane;
    xb = xc; xc = xt; xt = xt2; xt2 = xt3;
    fb = fc; fc = ft; ft = ft2; ft2 = ft3;
  }
}

// Four x-adjacent points per thread (two 16-byte accesses per row and array): the per-point
// cost of loop control, address arithmetic and the y-neighbour loads halves against
// march3_kernel; z neighbours in a register queue prefetched two planes ahead.  Needs nx % 4 == 0
// and 16-byte aligned vectors.
template <int KIND, int BY, int MINB = 2>
__global__ void __launch_bounds__(32 * BY, MINB) march4_kernel(MarchView v, const double* __restrict__ x,
                                                           const double* xsp, double* __restrict__ y,
                                                           double* __restrict__ xcopy) {
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr bool HASY = BY > 1;
  constexpr int TW = 128;
  const double* __restrict__ f = v.field;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int64_t i = (int64_t)blockIdx.x * TW + 4 * lane;    // first of this thread's four points
  const int64_t j = HASY ? (int64_t)blockIdx.y * BY + ty : 0;
  const int64_t z0 = (int64_t)blockIdx.z * v.zc;
  const int64_t z1 = (z0 + v.zc < v.nz) ? z0 + v.zc : v.nz;
  const bool in = i < v.nx && j < v.ny;                     // nx % 4 == 0: all four or none
  const int64_t plane = v.nx * v.ny;
  const int64_t col = in ? i + v.nx * j : 0;
  const bool has_w = i > 0, has_e = i + 4 < v.nx;
  const bool has_s = HASY && in && j > 0, has_n = HASY && in && j + 1 < v.ny;
  const bool lo_in = v.x_lo != nullptr, hi_in = v.x_hi != nullptr;
  const double xs = xsp ? *xsp : 1.0;
  const double hs0 = 0.5 * v.s[0], hs1 = 0.5 * v.s[1], hs2 = 0.5 * v.s[2];
  const double s0c = v.s[0], s1c = v.s[1], s2c = v.s[2];
  struct Q4 { double a, b, c, d; };
  auto ld4 = [&](const double* base, int64_t off) -> Q4 {
    const double2 p = __ldg(reinterpret_cast<const double2*>(base + off));
    const double2 q = __ldg(reinterpret_cast<const double2*>(base + off + 2));
    return Q4{p.x, p.y, q.x, q.y};
  };
  auto plane4 = [&](const double* a, const double* lo, const double* hi, int64_t p) -> Q4 {
    if (p >= 0 && p < v.nz) return ld4(a, col + plane * p);
    if (p < 0 && lo) return ld4(lo, col);
    if (p >= v.nz && hi) return ld4(hi, col);
    return Q4{0.0, 0.0, 0.0, 0.0};
  };
  const Q4 zero4{0.0, 0.0, 0.0, 0.0};
  Q4 xb = plane4(x, v.x_lo, v.x_hi, z0 - 1), xc = plane4(x, v.x_lo, v.x_hi, z0), xt = plane4(x, v.x_lo, v.x_hi, z0 + 1);
  Q4 fb = zero4, fc = zero4, ft = zero4;
  if (cell) {
    fb = plane4(f, v.f_lo, v.f_hi, z0 - 1); fc = plane4(f, v.f_lo, v.f_hi, z0); ft = plane4(f, v.f_lo, v.f_hi, z0 + 1);
  }
  int64_t g = col + plane * z0;
  for (int64_t z = z0; z < z1; ++z) {
    // prefetch plane z+2
    Q4 xt2 = zero4, ft2 = zero4;
    if (z + 2 < v.nz) {
      xt2 = ld4(x, g + 2 * plane);
      if (cell) ft2 = ld4(f, g + 2 * plane);
    } else if (z + 2 == v.nz) {
      xt2 = plane4(x, v.x_lo, v.x_hi, z + 2);
      if (cell) ft2 = plane4(f, v.f_lo, v.f_hi, z + 2);
    }
    // in-plane y neighbours (L1 / L2): missing -> x = 0, k = k_c
    Q4 xsn = zero4, xnn = zero4, fsn = fc, fnn = fc;
    if (has_s) { xsn = ld4(x, g - v.nx); if (cell) fsn = ld4(f, g - v.nx); }
    if (has_n) { xnn = ld4(x, g + v.nx); if (cell) fnn = ld4(f, g + v.nx); }
    // x neighbours across threads: the adjacent lanes; lanes 0 / 31 load across the tile edge
    double xw = __shfl_up_sync(0xffffffffu, xc.d, 1), xe = __shfl_down_sync(0xffffffffu, xc.a, 1);
    double fw = 0.0, fe = 0.0;
    if (cell) {
      fw = __shfl_up_sync(0xffffffffu, fc.d, 1);
      fe = __shfl_down_sync(0xffffffffu, fc.a, 1);
    }
    if (lane == 0 && in && has_w) { xw = __ldg(x + g - 1); if (cell) fw = __ldg(f + g - 1); }
    if (lane == 31 && in && has_e) { xe = __ldg(x + g + 4); if (cell) fe = __ldg(f + g + 4); }
    if (!has_w) { xw = 0.0; fw = fc.a; }
    if (!has_e) { xe = 0.0; fe = fc.d; }
    if (z == 0 && !lo_in) fb = fc;
    if (z + 1 == v.nz && !hi_in) ft = fc;
    auto point = [&](double c, double k, double xwv, double fwv, double xev, double fev, double xsv,
                     double fsv, double xnv, double fnv, double xbv, double fbv, double xtv, double ftv) {
      double acc = 0.0;
      if (cell) {
        acc = fma(hs0 * (k + fwv), c - xwv, acc);
        acc = fma(hs0 * (k + fev), c - xev, acc);
      } else {
        acc = fma(s0c, c - xwv, acc);
        acc = fma(s0c, c - xev, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[0], c - xwv, acc);
      if (HASY) {
        if (cell) {
          acc = fma(hs1 * (k + fsv), c - xsv, acc);
          acc = fma(hs1 * (k + fnv), c - xnv, acc);
        } else {
          acc = fma(s1c, c - xsv, acc);
          acc = fma(s1c, c - xnv, acc);
        }
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[1], c - xsv, acc);
      }
      if (cell) {
        acc = fma(hs2 * (k + fbv), c - xbv, acc);
        acc = fma(hs2 * (k + ftv), c - xtv, acc);
      } else {
        acc = fma(s2c, c - xbv, acc);
        acc = fma(s2c, c - xtv, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[2], c - xbv, acc);
      return xs * (c + acc);
    };
    if (in) {
      const double o0 = point(xc.a, fc.a, xw, fw, xc.b, fc.b, xsn.a, fsn.a, xnn.a, fnn.a, xb.a, fb.a, xt.a, ft.a);
      const double o1 = point(xc.b, fc.b, xc.a, fc.a, xc.c, fc.c, xsn.b, fsn.b, xnn.b, fnn.b, xb.b, fb.b, xt.b, ft.b);
      const double o2 = point(xc.c, fc.c, xc.b, fc.b, xc.d, fc.d, xsn.c, fsn.c, xnn.c, fnn.c, xb.c, fb.c, xt.c, ft.c);
      const double o3 = point(xc.d, fc.d, xc.c, fc.c, xe, fe, xsn.d, fsn.d, xnn.d, fnn.d, xb.d, fb.d, xt.d, ft.d);
      *reinterpret_cast<double2*>(y + g) = make_double2(o0, o1);
      *reinterpret_cast<double2*>(y + g + 2) = make_double2(o2, o3);
      if (xcopy) {
        *reinterpret_cast<double2*>(xcopy + g) = make_double2(xs * xc.a, xs * xc.b);
        *reinterpret_cast<double2*>(xcopy + g + 2) = make_double2(xs * xc.c, xs * xc.d);
      }
    }
    g += plane;
    xb = xc; xc = xt; xt = xt2;
    fb = fc; fc = ft; ft = ft2;
  }
}

// f4 (PSP-CG, R27/R28): the direction pass p = z + beta p_old -> px, q = A p -> py (the probe
// (p, A p), recorded with scale 1/||p||) and p'q, p'p, in one pass over HBM: 8 (z) + 8 (p_old) +
// 8 (field) read, 16 written per row.  march4_kernel's layout (four x-adjacent points a thread,
// march-axis register queue, x neighbours by shuffles, y neighbours from the neighbouring lines),
// with every loaded value of p formed on the fly from z and p_old.  One rank (no halo planes).
template <int KIND, int BY>
__global__ void __launch_bounds__(32 * BY, 2) cg_dir4_kernel(MarchView v, const double* __restrict__ z,
                                                             const double* __restrict__ pold, double* __restrict__ pout,
                                                             double* __restrict__ q, int slot, DevState ds) {
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  constexpr bool HASY = BY > 1;
  constexpr int TW = 128;
  const double* __restrict__ f = v.field;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int64_t i = (int64_t)blockIdx.x * TW + 4 * lane;
  const int64_t j = HASY ? (int64_t)blockIdx.y * BY + ty : 0;
  const int64_t z0 = (int64_t)blockIdx.z * v.zc;
  const int64_t z1 = (z0 + v.zc < v.nz) ? z0 + v.zc : v.nz;
  const bool in = i < v.nx && j < v.ny;
  const int64_t plane = v.nx * v.ny;
  const int64_t col = in ? i + v.nx * j : 0;
  const bool has_w = i > 0, has_e = i + 4 < v.nx;
  const bool has_s = HASY && in && j > 0, has_n = HASY && in && j + 1 < v.ny;
  const double beta = pold ? ds.scal[SC_BETACG] : 0.0;
  const double hs0 = 0.5 * v.s[0], hs1 = 0.5 * v.s[1], hs2 = 0.5 * v.s[2];
  const double s0c = v.s[0], s1c = v.s[1], s2c = v.s[2];
  struct Q4 { double a, b, c, d; };
  auto ld4 = [&](const double* base, int64_t off) -> Q4 {
    const double2 p0 = __ldg(reinterpret_cast<const double2*>(base + off));
    const double2 p1 = __ldg(reinterpret_cast<const double2*>(base + off + 2));
    return Q4{p0.x, p0.y, p1.x, p1.y};
  };
  auto dir4 = [&](int64_t off) -> Q4 {            // p = z + beta p_old at four points
    Q4 r = ld4(z, off);
    if (pold) {
      const Q4 o = ld4(pold, off);
      r = Q4{fma(beta, o.a, r.a), fma(beta, o.b, r.b), fma(beta, o.c, r.c), fma(beta, o.d, r.d)};
    }
    return r;
  };
  auto dir1 = [&](int64_t off) -> double { return pold ? fma(beta, __ldg(pold + off), __ldg(z + off)) : __ldg(z + off); };
  const Q4 zero4{0.0, 0.0, 0.0, 0.0};
  auto plane4 = [&](const double* a, int64_t p) -> Q4 { return (p >= 0 && p < v.nz) ? ld4(a, col + plane * p) : zero4; };
  auto dplane4 = [&](int64_t p) -> Q4 { return (p >= 0 && p < v.nz) ? dir4(col + plane * p) : zero4; };
  Q4 xb = dplane4(z0 - 1), xc = dplane4(z0), xt = dplane4(z0 + 1);
  Q4 fb = zero4, fc = zero4, ft = zero4;
  if (cell) {
    fb = plane4(f, z0 - 1); fc = plane4(f, z0); ft = plane4(f, z0 + 1);
  }
  double pq = 0.0, pp = 0.0;
  int64_t g = col + plane * z0;
  for (int64_t zz = z0; zz < z1; ++zz) {
    Q4 xt2 = zero4, ft2 = zero4;
    if (zz + 2 < v.nz) {
      xt2 = dir4(g + 2 * plane);
      if (cell) ft2 = ld4(f, g + 2 * plane);
    }
    Q4 xsn = zero4, xnn = zero4, fsn = fc, fnn = fc;
    if (has_s) { xsn = dir4(g - v.nx); if (cell) fsn = ld4(f, g - v.nx); }
    if (has_n) { xnn = dir4(g + v.nx); if (cell) fnn = ld4(f, g + v.nx); }
    double xw = __shfl_up_sync(0xffffffffu, xc.d, 1), xe = __shfl_down_sync(0xffffffffu, xc.a, 1);
    double fw = 0.0, fe = 0.0;
    if (cell) {
      fw = __shfl_up_sync(0xffffffffu, fc.d, 1);
      fe = __shfl_down_sync(0xffffffffu, fc.a, 1);
    }
    if (lane == 0 && in && has_w) { xw = dir1(g - 1); if (cell) fw = __ldg(f + g - 1); }
    if (lane == 31 && in && has_e) { xe = dir1(g + 4); if (cell) fe = __ldg(f + g + 4); }
    if (!has_w) { xw = 0.0; fw = fc.a; }
    if (!has_e) { xe = 0.0; fe = fc.d; }
    if (zz == 0) fb = fc;
    if (zz + 1 == v.nz) ft = fc;
    auto point = [&](double c, double k, double xwv, double fwv, double xev, double fev, double xsv,
                     double fsv, double xnv, double fnv, double xbv, double fbv, double xtv, double ftv) {
      double acc = 0.0;
      if (cell) {
        acc = fma(hs0 * (k + fwv), c - xwv, acc);
        acc = fma(hs0 * (k + fev), c - xev, acc);
      } else {
        acc = fma(s0c, c - xwv, acc);
        acc = fma(s0c, c - xev, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[0], c - xwv, acc);
      if (HASY) {
        if (cell) {
          acc = fma(hs1 * (k + fsv), c - xsv, acc);
          acc = fma(hs1 * (k + fnv), c - xnv, acc);
        } else {
          acc = fma(s1c, c - xsv, acc);
          acc = fma(s1c, c - xnv, acc);
        }
        if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[1], c - xsv, acc);
      }
      if (cell) {
        acc = fma(hs2 * (k + fbv), c - xbv, acc);
        acc = fma(hs2 * (k + ftv), c - xtv, acc);
      } else {
        acc = fma(s2c, c - xbv, acc);
        acc = fma(s2c, c - xtv, acc);
      }
      if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(v.a[2], c - xbv, acc);
      return c + acc;
    };
    if (in) {
      const double o0 = point(xc.a, fc.a, xw, fw, xc.b, fc.b, xsn.a, fsn.a, xnn.a, fnn.a, xb.a, fb.a, xt.a, ft.a);
      const double o1 = point(xc.b, fc.b, xc.a, fc.a, xc.c, fc.c, xsn.b, fsn.b, xnn.b, fnn.b, xb.b, fb.b, xt.b, ft.b);
      const double o2 = point(xc.c, fc.c, xc.b, fc.b, xc.d, fc.d, xsn.c, fsn.c, xnn.c, fnn.c, xb.c, fb.c, xt.c, ft.c);
      const double o3 = point(xc.d, fc.d, xc.c, fc.c, xe, fe, xsn.d, fsn.d, xnn.d, fnn.d, xb.d, fb.d, xt.d, ft.d);
      *reinterpret_cast<double2*>(q + g) = make_double2(o0, o1);
      *reinterpret_cast<double2*>(q + g + 2) = make_double2(o2, o3);
      *reinterpret_cast<double2*>(pout + g) = make_double2(xc.a, xc.b);
      *reinterpret_cast<double2*>(pout + g + 2) = make_double2(xc.c, xc.d);
      pq = fma(xc.a, o0, pq); pq = fma(xc.b, o1, pq); pq = fma(xc.c, o2, pq); pq = fma(xc.d, o3, pq);
      pp = fma(xc.a, xc.a, pp); pp = fma(xc.b, xc.b, pp); pp = fma(xc.c, xc.c, pp); pp = fma(xc.d, xc.d, pp);
    }
    g += plane;
    xb = xc; xc = xt; xt = xt2;
    fb = fc; fc = ft; ft = ft2;
  }
  // deterministic grid reduction of (p'q, p'p) -> EPI_CG_DIR
  __shared__ double sm[BY * 2];
  double a[2] = {pq, pp};
  block_sum<2, BY>(a, sm);
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    ds.partials[bid] = a[0];
    ds.partials[nb + bid] = a[1];
  }
  if (finish_block(ds.tickets + TK_MAIN, nb)) {
    double t[2];
    t[0] = reduce_partials<BY>(ds.partials, 0, (int)nb, sm);
    t[1] = reduce_partials<BY>(ds.partials, 1, (int)nb, sm);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      if (ds.multi) { ds.rpart[0] = t[0]; ds.rpart[1] = t[1]; }
      else cg_epilogue(EPI_CG_DIR, ds, slot, 1, t);
    }
  }
}

__global__ void dia_matvec_kernel(int64_t n, int dA, const double* __restrict__ bands,
                                  const double* __restrict__ x, const double* xsp, double* __restrict__ y,
                                  double* __restrict__ xcopy) {
  const double xs = xsp ? *xsp : 1.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int o = 0; o <= 2 * dA; ++o) {
      int64_t jj = i + o - dA;
      if (jj < 0 || jj >= n) continue;
      s = fma(__ldg(bands + (int64_t)o * n + i), __ldg(x + jj), s);
    }
    y[i] = xs * s;
    if (xcopy != nullptr) xcopy[i] = xs * __ldg(x + i);
  }
}

inline int64_t planes_per_block(int64_t tiles, int64_t nz) {
  // about 8 resident waves of blocks, at least 16 planes per block (halo re-reads of 2 planes
  // per chunk <= 12.5%)
  int64_t zc = (tiles * nz) / ((int64_t)device_sms() * 8 * 8);
  if (zc < 16) zc = 16;
  if (zc > nz) zc = nz;
  if (zc < 1) zc = 1;
  return zc;
}

template <int KIND, int BX, int BY>
void launch_march(const MarchView& v0, const double* x, const double* xs, double* y, double* xcopy,
                  cudaStream_t s) {
  MarchView v = v0;
  const int64_t zc = planes_per_block(((v.nx + BX - 1) / BX) * ((v.ny + BY - 1) / BY), v.nz);
  v.zc = (int)zc;
  dim3 grid((unsigned)((v.nx + BX - 1) / BX), (unsigned)((v.ny + BY - 1) / BY),
            (unsigned)((v.nz + zc - 1) / zc));
  march_matvec_kernel<KIND, BX, BY><<<grid, dim3(BX, BY), 0, s>>>(v, x, xs, y, xcopy);
}

template <int KIND, int BY>
void launch_march4(const MarchView& v0, const double* x, const double* xs, double* y, double* xcopy,
                   cudaStream_t s) {
  MarchView v = v0;
  const int64_t zc = planes_per_block(((v.nx + 127) / 128) * ((v.ny + BY - 1) / BY), v.nz);
  v.zc = (int)zc;
  dim3 grid((unsigned)((v.nx + 127) / 128), (unsigned)((v.ny + BY - 1) / BY), (unsigned)((v.nz + zc - 1) / zc));
  // PSP_MARCH4_MINB=3: the 3-blocks-per-SM build of the kernel (85 registers; A/B knob)
  static const int minb = getenv("PSP_MARCH4_MINB") ? atoi(getenv("PSP_MARCH4_MINB")) : 2;
  if (minb >= 3) march4_kernel<KIND, BY, 3><<<grid, dim3(32, BY), 0, s>>>(v, x, xs, y, xcopy);
  else march4_kernel<KIND, BY><<<grid, dim3(32, BY), 0, s>>>(v, x, xs, y, xcopy);
}

template <int KIND, int BY>
void launch_march2(const MarchView& v0, const double* x, const double* xs, double* y, double* xcopy,
                   cudaStream_t s) {
  MarchView v = v0;
  const int64_t zc = planes_per_block(((v.nx + 63) / 64) * ((v.ny + BY - 1) / BY), v.nz);
  v.zc = (int)zc;
  dim3 grid((unsigned)((v.nx + 63) / 64), (unsigned)((v.ny + BY - 1) / BY), (unsigned)((v.nz + zc - 1) / zc));
  march3_kernel<KIND, BY><<<grid, dim3(32, BY), 0, s>>>(v, x, xs, y, xcopy);
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <int KIND>
void launch_kind(const Stencil& st, const double* x, const double* xs, double* y, double* xcopy,
                 cudaStream_t s) {
  if (st.ndim == 1) {
    dim3 grid((unsigned)((st.nx + 127) / 128), 1, 1);
    matvec_kernel<KIND, 1><<<grid, 128, 0, s>>>(st, x, xs, y, xcopy);
    return;
  }
  const bool vec_ok = (st.nx % 2 == 0) && aligned16(x) && aligned16(y) && aligned16(xcopy) &&
                      aligned16(st.field) && aligned16(st.x_lo) && aligned16(st.x_hi) &&
                      aligned16(st.f_lo) && aligned16(st.f_hi);
  MarchView v;
  v.field = st.field;
  v.x_lo = st.x_lo;
  v.x_hi = st.x_hi;
  v.f_lo = st.f_lo;
  v.f_hi = st.f_hi;
  v.zc = 1;
  v.s[0] = st.s[0];
  v.a[0] = st.a[0];
  if (st.ndim == 3) {
    v.nx = st.nx; v.ny = st.ny; v.nz = st.nz;
    v.s[1] = st.s[1]; v.a[1] = st.a[1];
    v.s[2] = st.s[2]; v.a[2] = st.a[2];
    if (vec_ok && v.nx % 4 == 0 && !getenv("PSP_MARCH3")) launch_march4<KIND, 8>(v, x, xs, y, xcopy, s);
    else if (vec_ok) launch_march2<KIND, 8>(v, x, xs, y, xcopy, s);
    else launch_march<KIND, 32, 8>(v, x, xs, y, xcopy, s);
  } else {
    v.nx = st.nx; v.ny = 1; v.nz = st.ny;
    v.s[1] = 0.0; v.a[1] = 0.0;
    v.s[2] = st.s[1]; v.a[2] = st.a[1];
    if (vec_ok) launch_march2<KIND, 1>(v, x, xs, y, xcopy, s);
    else launch_march<KIND, 256, 1>(v, x, xs, y, xcopy, s);
  }
}

}  // namespace

bool launch_cg_dir_fused(const Stencil& st, const double* z, const double* pold, double* px, double* py, int slot,
                         DevState ds, cudaStream_t s) {
  if (st.ndim != 3 || st.kind == PSP_OP_DIA || st.nx % 4 != 0 || st.x_lo || st.x_hi) return false;
  if (!aligned16(z) || !aligned16(pold) || !aligned16(px) || !aligned16(py) || !aligned16(st.field)) return false;
  MarchView v;
  v.field = st.field;
  v.x_lo = v.x_hi = v.f_lo = v.f_hi = nullptr;
  v.nx = st.nx; v.ny = st.ny; v.nz = st.nz;
  for (int a = 0; a < 3; ++a) { v.s[a] = st.s[a]; v.a[a] = st.a[a]; }
  constexpr int BY = 8;
  const int64_t zc = planes_per_block(((v.nx + 127) / 128) * ((v.ny + BY - 1) / BY), v.nz);
  v.zc = (int)zc;
  dim3 grid((unsigned)((v.nx + 127) / 128), (unsigned)((v.ny + BY - 1) / BY), (unsigned)((v.nz + zc - 1) / zc));
  const int64_t nb = (int64_t)grid.x * grid.y * grid.z;
  if (2 * nb > (int64_t)2 * kMaxRestart * 8 * device_sms()) return false;   // partials capacity
  switch (st.kind) {
    case PSP_OP_CONST_DIFF: cg_dir4_kernel<PSP_OP_CONST_DIFF, BY><<<grid, dim3(32, BY), 0, s>>>(v, z, pold, px, py, slot, ds); break;
    case PSP_OP_CELL_DIFF: cg_dir4_kernel<PSP_OP_CELL_DIFF, BY><<<grid, dim3(32, BY), 0, s>>>(v, z, pold, px, py, slot, ds); break;
    default: cg_dir4_kernel<PSP_OP_CELL_ADVDIFF, BY><<<grid, dim3(32, BY), 0, s>>>(v, z, pold, px, py, slot, ds); break;
  }
  return true;
}

void launch_matvec(const Stencil& st, const double* x, const double* xs, double* y, double* xcopy,
                   cudaStream_t s) {
  switch (st.kind) {
    case PSP_OP_CONST_DIFF: launch_kind<PSP_OP_CONST_DIFF>(st, x, xs, y, xcopy, s); break;
    case PSP_OP_CELL_DIFF: launch_kind<PSP_OP_CELL_DIFF>(st, x, xs, y, xcopy, s); break;
    case PSP_OP_CELL_ADVDIFF: launch_kind<PSP_OP_CELL_ADVDIFF>(st, x, xs, y, xcopy, s); break;
    default: {
      int blocks = (int)((st.n + 255) / 256);
      if (blocks > 16 * device_sms()) blocks = 16 * device_sms();
      if (blocks < 1) blocks = 1;
      dia_matvec_kernel<<<blocks, 256, 0, s>>>(st.n, st.dA, st.bands, x, xs, y, xcopy);
    }
  }
}

}  // namespace psp
