// Exploration micro-benchmark (not part of the product): variants of the ICWY update pass
// U = w - sum_j h_j V_j (+ ||U||^2) at n = 2^27, k = 16, to find what limits it.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TPB = 256;

template <int RPT, int JC, bool STORE>
__global__ void __launch_bounds__(TPB) upd(const double* __restrict__ V, long ldv, const double* __restrict__ w,
                                           double* __restrict__ U, const double* __restrict__ h, int k, long n,
                                           double* part) {
  constexpr int TILE = TPB * RPT;
  double acc = 0;
  long ntiles = (n + TILE - 1) / TILE;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    long r0 = tile * TILE + threadIdx.x;
    double u[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) u[i] = w[r0 + (long)TPB * i];
    for (int jb = 0; jb < k; jb += JC) {
      double v[JC][RPT];
#pragma unroll
      for (int c = 0; c < JC; ++c)
#pragma unroll
        for (int i = 0; i < RPT; ++i) v[c][i] = V[(long)(jb + c) * ldv + r0 + (long)TPB * i];
#pragma unroll
      for (int c = 0; c < JC; ++c)
#pragma unroll
        for (int i = 0; i < RPT; ++i) u[i] = fma(-h[jb + c], v[c][i], u[i]);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (STORE) U[r0 + (long)TPB * i] = u[i];
      acc = fma(u[i], u[i], acc);
    }
  }
  if (acc == 12345.0) part[0] = acc;
}

// row-per-thread, vectors innermost, double2 loads
__global__ void __launch_bounds__(TPB) upd_v2(const double2* __restrict__ V, long ldv2, const double2* __restrict__ w,
                                              double2* __restrict__ U, const double* __restrict__ h, int k, long n2,
                                              double* part) {
  double acc = 0;
  for (long r = blockIdx.x * (long)TPB + threadIdx.x; r < n2; r += (long)gridDim.x * TPB) {
    double2 u = w[r];
#pragma unroll 8
    for (int j = 0; j < k; ++j) {
      double2 v = V[(long)j * ldv2 + r];
      u.x = fma(-h[j], v.x, u.x);
      u.y = fma(-h[j], v.y, u.y);
    }
    U[r] = u;
    acc += u.x * u.x + u.y * u.y;
  }
  if (acc == 12345.0) part[0] = acc;
}

__global__ void dots(const double* __restrict__ V, long ldv, const double* __restrict__ w, int k, long n, double* part) {
  constexpr int RPT = 8, TILE = TPB * RPT, JC = 4;
  double tot = 0;
  long ntiles = (n + TILE - 1) / TILE;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    long r0 = tile * TILE + threadIdx.x;
    double wr[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) wr[i] = w[r0 + (long)TPB * i];
    for (int jb = 0; jb < k; jb += JC) {
      double a[JC] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < JC; ++c)
#pragma unroll
        for (int i = 0; i < RPT; ++i) a[c] = fma(V[(long)(jb + c) * ldv + r0 + (long)TPB * i], wr[i], a[c]);
      tot += a[0] + a[1] + a[2] + a[3];
    }
  }
  if (tot == 12345.0) part[0] = tot;
}

int main() {
  const long n = 1L << 27;
  const int k = 16;
  double *V, *w, *U, *h, *part;
  cudaMalloc(&V, sizeof(double) * n * (k + 1));
  cudaMalloc(&w, sizeof(double) * n);
  cudaMalloc(&U, sizeof(double) * n);
  cudaMalloc(&h, sizeof(double) * 64);
  cudaMalloc(&part, 64);
  cudaMemset(V, 0, sizeof(double) * n * (k + 1));
  cudaMemset(w, 0, sizeof(double) * n);
  cudaMemset(h, 0, 512);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes_upd = 8.0 * n * (k + 2), bytes_dots = 8.0 * n * (k + 1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %8.3f ms %8.1f GB/s  %s\n", name, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int g : {296, 592, 1184}) {
    char nm[128];
    snprintf(nm, 128, "upd RPT8 JC4 store grid%d", g);
    timeit(nm, bytes_upd, [&] { upd<8, 4, true><<<g, TPB>>>(V, n, w, U, h, k, n, part); });
    snprintf(nm, 128, "upd RPT8 JC4 nostore grid%d", g);
    timeit(nm, bytes_upd - 8.0 * n, [&] { upd<8, 4, false><<<g, TPB>>>(V, n, w, U, h, k, n, part); });
    snprintf(nm, 128, "upd RPT4 JC8 store grid%d", g);
    timeit(nm, bytes_upd, [&] { upd<4, 8, true><<<g, TPB>>>(V, n, w, U, h, k, n, part); });
    snprintf(nm, 128, "upd RPT2 JC16 store grid%d", g);
    timeit(nm, bytes_upd, [&] { upd<2, 16, true><<<g, TPB>>>(V, n, w, U, h, k, n, part); });
    snprintf(nm, 128, "upd_v2 double2 grid%d", g);
    timeit(nm, bytes_upd, [&] { upd_v2<<<g, TPB>>>((const double2*)V, n / 2, (const double2*)w, (double2*)U, h, k, n / 2, part); });
    snprintf(nm, 128, "dots RPT8 JC4 grid%d", g);
    timeit(nm, bytes_dots, [&] { dots<<<g, TPB>>>(V, n, w, k, n, part); });
  }
  return 0;
}
