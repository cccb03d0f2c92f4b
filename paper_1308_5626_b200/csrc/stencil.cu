// stencil.cu -- K1: matrix-free y = A x = (I - dt L) x  (Eq.4; "replacing the
// matrix-vector product in the GMRES algorithm with residual computation").
//
// HBM-bound: algorithmic bytes per row = 8 (x) + 8 (field, CELL_* only) + 8 (y) [+ 8 when the
// probe copy P_x is written in the same pass].  One thread per grid point, blocks of 128
// threads along x; the +-x neighbours come from the same warp's lines, the +-y / +-z
// neighbours from L1/L2 (three planes of x and kappa are ~12 MB at 512^2, well inside the
// 126 MB L2), so DRAM sees each array once.
#include "internal.h"

namespace psp {
namespace {

struct Nb {
  double x, f;
  bool in;
};

// neighbour of (i,j,k) along axis A, direction D (-1/+1).  Outside the local block: the slab
// halo plane if present (multi-rank), else the Dirichlet zero (R24).
template <int AXIS, int DIR>
__device__ __forceinline__ Nb neighbour(const Stencil& st, const double* __restrict__ x,
                                        const double* __restrict__ f, int64_t i, int64_t j,
                                        int64_t k, int64_t g, bool need_f) {
  Nb r{0.0, 0.0, false};
  int64_t c = (AXIS == 0) ? i : (AXIS == 1 ? j : k);
  int64_t ext = (AXIS == 0) ? st.nx : (AXIS == 1 ? st.ny : st.nz);
  int64_t stride = (AXIS == 0) ? 1 : (AXIS == 1 ? st.nx : st.nx * st.ny);
  int64_t cn = c + DIR;
  if (cn >= 0 && cn < ext) {
    r.x = __ldg(x + g + DIR * stride);
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
      r.x = __ldg(hx + off);
      if (need_f) r.f = __ldg(hf + off);
      r.in = true;
    }
  }
  return r;
}

template <int KIND, int NDIM>
__global__ void __launch_bounds__(128) matvec_kernel(Stencil st, const double* __restrict__ x,
                                                     const double* xsp, double* __restrict__ y,
                                                     double* __restrict__ xcopy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  const int64_t k = blockIdx.z;
  if (i >= st.nx) return;
  const int64_t g = i + st.nx * (j + st.ny * k);
  const double* __restrict__ f = st.field;
  constexpr bool cell = (KIND != PSP_OP_CONST_DIFF);
  const double xs = xsp ? *xsp : 1.0;
  const double xc = __ldg(x + g);
  const double fc = cell ? __ldg(f + g) : 0.0;
  double acc = 0.0;  // sum over faces of s_a * k_f * (x_c - x_nb) + upwind terms
  auto face = [&](const Nb& nb, double s) {
    double kf = cell ? (nb.in ? 0.5 * (fc + nb.f) : fc) : 1.0;
    acc = fma(s * kf, xc - nb.x, acc);
  };
  {
    Nb w = neighbour<0, -1>(st, x, f, i, j, k, g, cell);
    Nb e = neighbour<0, +1>(st, x, f, i, j, k, g, cell);
    face(w, st.s[0]);
    face(e, st.s[0]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[0], xc - w.x, acc);
  }
  if (NDIM >= 2) {
    Nb sn = neighbour<1, -1>(st, x, f, i, j, k, g, cell);
    Nb nn = neighbour<1, +1>(st, x, f, i, j, k, g, cell);
    face(sn, st.s[1]);
    face(nn, st.s[1]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[1], xc - sn.x, acc);
  }
  if (NDIM >= 3) {
    Nb b = neighbour<2, -1>(st, x, f, i, j, k, g, cell);
    Nb t = neighbour<2, +1>(st, x, f, i, j, k, g, cell);
    face(b, st.s[2]);
    face(t, st.s[2]);
    if (KIND == PSP_OP_CELL_ADVDIFF) acc = fma(st.a[2], xc - b.x, acc);
  }
  // A x = x - dt L x;  -dt L x = sum_faces s k_f (x_c - x_nb) + sum_a a_a (x_c - x_w)
  // (the scale xs is linear: applied once to the result and to the probe copy)
  y[g] = xs * (xc + acc);
  if (xcopy != nullptr) xcopy[g] = xs * xc;
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

template <int KIND>
void launch_kind(const Stencil& st, const double* x, const double* xs, double* y, double* xcopy,
                 cudaStream_t s) {
  dim3 block(128);
  dim3 grid((unsigned)((st.nx + 127) / 128), (unsigned)st.ny, (unsigned)st.nz);
  switch (st.ndim) {
    case 1: matvec_kernel<KIND, 1><<<grid, block, 0, s>>>(st, x, xs, y, xcopy); break;
    case 2: matvec_kernel<KIND, 2><<<grid, block, 0, s>>>(st, x, xs, y, xcopy); break;
    default: matvec_kernel<KIND, 3><<<grid, block, 0, s>>>(st, x, xs, y, xcopy); break;
  }
}

}  // namespace

void launch_matvec(const Stencil& st, const double* x, const double* xs, double* y, double* xcopy,
                   cudaStream_t s) {
  switch (st.kind) {
    case PSP_OP_CONST_DIFF: launch_kind<PSP_OP_CONST_DIFF>(st, x, xs, y, xcopy, s); break;
    case PSP_OP_CELL_DIFF: launch_kind<PSP_OP_CELL_DIFF>(st, x, xs, y, xcopy, s); break;
    case PSP_OP_CELL_ADVDIFF: launch_kind<PSP_OP_CELL_ADVDIFF>(st, x, xs, y, xcopy, s); break;
    default: {
      int blocks = (int)((st.n + 255) / 256);
      if (blocks > 148 * 16) blocks = 148 * 16;
      if (blocks < 1) blocks = 1;
      dia_matvec_kernel<<<blocks, 256, 0, s>>>(st.n, st.dA, st.bands, x, xs, y, xcopy);
    }
  }
}

}  // namespace psp
