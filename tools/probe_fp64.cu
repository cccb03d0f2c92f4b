// One-off probe: FP64 FMA throughput and FP64 streaming bandwidth on the box's B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0+a1+a2+a3+a4+a5+a6+a7;
  if (s == 12345.0) out[0] = s;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}
__global__ void triad(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ c, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) { double2 x=a[i], y=b[i]; c[i] = make_double2(x.x+2.0*y.x, x.y+2.0*y.y);} 
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sms %d cc %d.%d l2 %d MB smem/sm %zu regs/sm %d\n", p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize>>20, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  size_t freeb, totb; cudaMemGetInfo(&freeb, &totb); printf("mem free %.1f GiB total %.1f GiB\n", freeb/1073741824.0, totb/1073741824.0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2000;
  fma_loop<<<blocks, threads>>>(out, 10); cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); fma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("fp64 fma: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB per buffer
  double2 *a, *b, *c; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&c, n*16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n*16);
  for (int g : {148*4, 148*8, 148*16}) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<g, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid %d: %.1f GB/s\n", g, 2.0 * n * 16 / ms / 1e6);
    cudaEventRecord(e0); triad<<<g, 256>>>(a, b, c, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("triad grid %d: %.1f GB/s\n", g, 3.0 * n * 16 / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
