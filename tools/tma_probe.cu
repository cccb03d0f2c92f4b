// Minimal probe of the fused kernel's TMA usage (4-D tensor map, expect_tx, tile load, wait).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe_notile(const __grid_constant__ CUtensorMap m, double* out, int x0, int y0, int z0, int sl) {
  extern __shared__ __align__(128) double sm[];
  double* buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm) + 127) & ~uintptr_t(127));
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 32 * 16);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(MODE) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            su32(buf)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(x0), "r"(y0), "r"(z0), "r"(sl), "r"(su32(bar))
        : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(bar)), "r"(0u) : "memory");
  }
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) out[i] = buf[i];
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap m, double* out, int x0, int y0, int z0, int sl) {
  extern __shared__ __align__(128) double sm[];
  double* buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm) + 127) & ~uintptr_t(127));
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 32 * 16);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE >= 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32 * 16 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            su32(buf)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(x0), "r"(y0), "r"(z0), "r"(sl), "r"(su32(bar))
        : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(bar)), "r"(0u) : "memory");
  }
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = (variant >= 2 && variant != 10) ? 64 : 16, ny = (variant == 5) ? 8 : 16, nz = 16, ns = 3;
  const size_t n = (size_t)nx * ny * nz;
  double* h = (double*)malloc(n * ns * 8);
  for (size_t i = 0; i < n * ns; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, n * ns * 8);
  cudaMalloc(&o, 32 * 16 * 8);
  cudaMemcpy(d, h, n * ns * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn fn = (EncodeTiledFn)p;
  CUtensorMap m;
  cuuint64_t dims[4] = {nx, ny, nz, ns};
  cuuint64_t strides[3] = {nx * 8, nx * ny * 8, n * 8};
  cuuint32_t box[4] = {32, 16, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  const size_t smem = 32 * 16 * 8 + 256;
  for (int mode = 0; mode < 1; ++mode) {
    cudaMemset(o, 0, 32 * 16 * 8);
    if (variant == 0) probe<0><<<1, 128, smem>>>(m, o, -1, -1, 2, 1);
    else if (variant == 1) probe_notile<4096><<<1, 128, smem>>>(m, o, -1, -1, 2, 1);
    else if (variant == 2) probe<0><<<1, 128, smem>>>(m, o, 0, 0, 2, 1);
    else if (variant == 4) probe<0><<<1, 128, smem>>>(m, o, -1, -1, 2, 1);
    else if (variant == 6) probe<0><<<1, 128, smem>>>(m, o, -2, -1, 2, 1);
    else if (variant == 7) probe<0><<<1, 128, smem>>>(m, o, 1, 0, 2, 1);
    else if (variant == 8) probe<0><<<1, 128, smem>>>(m, o, -1, 0, 2, 1);
    else if (variant == 9) probe<0><<<1, 128, smem>>>(m, o, 2, 0, 2, 1);
    else if (variant == 10) probe<0><<<1, 128, smem>>>(m, o, -2, -1, 2, 1);
    else if (variant == 5) probe<0><<<1, 128, smem>>>(m, o, 40, 3, -1, 1);
    else probe_notile<4096><<<1, 128, smem>>>(m, o, 0, 0, 2, 1);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[32 * 16];
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("mode %d: %s  o[0]=%g o[33]=%g (expect %g)\n", mode, cudaGetErrorString(e), ho[0], ho[33],
           (double)(n * 1 + 2 * nx * ny + 0 * nx + 0));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
