// reduce.cuh -- deterministic grid reductions shared by the streaming kernels (krylov.cu, the CG
// passes of stencil.cu): every block writes one partial per value, the last block to finish
// (atomic ticket) sums the partials in a fixed order, so results are bitwise reproducible
// (S:437).  Device code only.
#pragma once
#include "internal.h"

namespace psp {

static __device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of NV values held per thread (NW warps); result valid in thread 0
template <int NV, int NW = kRedThreads / 32>
static __device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* NW*NV */) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x + blockDim.x * threadIdx.y) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) smem[warp * NV + q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += smem[w * NV + q];
      v[q] = s;
    }
  }
  __syncthreads();
}

// Publish this block's partials; returns true in every thread of the last of nb blocks to finish.
static __device__ bool finish_block(unsigned* ticket, unsigned nb) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == nb - 1);
    if (s_last) *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}
static __device__ bool finish_block(unsigned* ticket) { return finish_block(ticket, gridDim.x); }

// Last block: total of partials[v*nb + b] over b, fixed order.  Result valid in thread 0.
template <int NW = kRedThreads / 32>
static __device__ double reduce_partials(const double* partials, int v, int nb, double* smem) {
  double a[1] = {0.0};
  const int t = threadIdx.x + blockDim.x * threadIdx.y, nt = blockDim.x * blockDim.y;
  for (int b = t; b < nb; b += nt) a[0] += ((volatile const double*)partials)[(int64_t)v * nb + b];
  block_sum<1, NW>(a, smem);
  return a[0];
}

}  // namespace psp
