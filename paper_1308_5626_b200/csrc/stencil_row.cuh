// stencil_row.cuh -- one row of the matrix-free operator A = I - dt L (Eq.4; R24), for the
// row-parallel kernels (stencil.cu's scalar matvec, resident.cu's persistent solver).  The
// marching kernels of stencil.cu and the fused pass evaluate the same faces in the same order.
#pragma once
#include "internal.h"

namespace psp {

struct Nb {
  double x, f;
  bool in;
};

// neighbour of (i,j,k) along axis A, direction D (-1/+1).  Outside the local block: the slab
// halo plane if present (multi-rank), else the Dirichlet zero (R24).
// load policy of x: 0 read-only path (x not written in this launch), 1 L2 only (written by other
// blocks of this launch), 2 plain (written by this block: one-CTA launches)
template <int CG>
static __device__ __forceinline__ double ldx(const double* p) {
  if (CG == 1) return __ldcg(p);
  if (CG == 2) return *p;
  return __ldg(p);
}

template <int AXIS, int DIR, int CG = 0>
static __device__ __forceinline__ Nb neighbour(const Stencil& st, const double* __restrict__ x,
                                        const double* __restrict__ f, int64_t i, int64_t j,
                                        int64_t k, int64_t g, bool need_f) {
  Nb r{0.0, 0.0, false};
  int64_t c = (AXIS == 0) ? i : (AXIS == 1 ? j : k);
  int64_t ext = (AXIS == 0) ? st.nx : (AXIS == 1 ? st.ny : st.nz);
  int64_t stride = (AXIS == 0) ? 1 : (AXIS == 1 ? st.nx : st.nx * st.ny);
  int64_t cn = c + DIR;
  if (cn >= 0 && cn < ext) {
    r.x = ldx<CG>(x + g + DIR * stride);
    if (need_f) r.f = __ldg(f + g + DIR * stride);
    r.in = true;
    return r;
  }
  // leaving the local block along the slab axis: halo planes (the slowest axis of ndim)
  const bool slab_axis = (st.ndim == 3 && AXIS == 2) || (st.ndim == 2 && AXIS == 1) ||
                         (st.ndim == 1 && AXIS == 0);
  if (slab_axis) {
    const double* hx = (DIR < 0) ? st.x_lo : st.x_hi;
    const double* hf = (DIR < 0) ? st.f_lo : st.f_hi;
    if (hx != nullptr) {
      int64_t off = (st.ndim == 3) ? (i + st.nx * j) : (st.ndim == 2 ? i : 0);
      r.x = ldx<CG>(hx + off);
      if (need_f) r.f = __ldg(hf + off);
      r.in = true;
    }
  }
  return r;
}

// (A x)_g at grid point (i, j, k) of the local block, g = i + nx (j + ny k); xc <- x_g.
// A x = x - dt L x;  -dt L x = sum_faces s k_f (x_c - x_nb) + sum_a a_a (x_c - x_w).
// CG = true: x was written earlier in the same launch by other blocks (read through L2 only)
template <int KIND, int NDIM, int CG = 0>
static __device__ __forceinline__ double stencil_row(const Stencil& st, const double* __restrict__ x, int64_t i,
                                                    int64_t j, int64_t k, int64_t g, double& xc) {
  const double* __restrict__ f = st.field;
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  xc = ldx<CG>(x + g);
  const double fc = cell ? __ldg(f + g) : 0.0;
  double acc = 0.0;  // sum over faces of s_a * k_f * (x_c - x_nb) + upwind terms
  const double c0 = xc;
  auto face = [&](const Nb& nb, double s) {
    double kf = cell ? (nb.in ? 0.5 * (fc + nb.f) : fc) : 1.0;
    acc = fma(s * kf, c0 - nb.x, acc);
  };
  {
    Nb w = neighbour<0, -1, CG>(st, x, f, i, j, k, g, cell);
    Nb e = neighbour<0, +1, CG>(st, x, f, i, j, k, g, cell);
    face(w, st.s[0]);
    face(e, st.s[0]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[0], c0 - w.x, acc);
  }
  if (NDIM >= 2) {
    Nb sn = neighbour<1, -1, CG>(st, x, f, i, j, k, g, cell);
    Nb nn = neighbour<1, +1, CG>(st, x, f, i, j, k, g, cell);
    face(sn, st.s[1]);
    face(nn, st.s[1]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[1], c0 - sn.x, acc);
  }
  if (NDIM >= 3) {
    Nb b = neighbour<2, -1, CG>(st, x, f, i, j, k, g, cell);
    Nb t = neighbour<2, +1, CG>(st, x, f, i, j, k, g, cell);
    face(b, st.s[2]);
    face(t, st.s[2]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[2], c0 - b.x, acc);
  }
  return c0 + acc;
}

// (A x)_g of a DIA operator (PSP_OP_DIA; the paper's banded test matrices)
template <int CG = 0>
static __device__ __forceinline__ double dia_row(const Stencil& st, const double* __restrict__ x, int64_t g) {
  double s = 0.0;
  for (int o = 0; o <= 2 * st.dA; ++o) {
    const int64_t jj = g + o - st.dA;
    if (jj < 0 || jj >= st.n) continue;
    s = fma(__ldg(st.bands + (int64_t)o * st.n + g), ldx<CG>(x + jj), s);
  }
  return s;
}

}  // namespace psp
