// Latency / per-warp throughput probe for the FP64 ops of the series loops:
// dependent DADD / DFMA chains and chains of C independent DADDs in one warp.
// usage: fp64lat  -> prints cycles per op
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_dadd(double *out, long long *cyc, double y, int n) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; c++) x[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int c = 0; c < C; c++) x[c] = x[c] + y;
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; c++) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
__global__ void k_dfma(double *out, long long *cyc, double y, int n) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; c++) x[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int c = 0; c < C; c++) x[c] = fma(x[c], y, y);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; c++) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_lds(double *out, long long *cyc, int n) {
  __shared__ double2 tab[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = make_double2(0.0, (double)((i * 7 + 1) & 1023));
  __syncthreads();
  int j = threadIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    double2 v = tab[j];
    j = (int)v.y;
    acc += v.x;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + j;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double *out;
  long long *cyc, h;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
#define RUN(K, C, W)                                                                  \
  K<C><<<1, 32 * W>>>(out, cyc, 1.0000001, n);                                         \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                      \
  printf("%s chains=%d warps=%d: %.2f cycles per dependent step, %.3f cycles per warp-op\n", \
         #K, C, W, (double)h / n, (double)h / n / C / W * (W > 4 ? 4.0 / 4 : 1.0));
  RUN(k_dadd, 1, 1) RUN(k_dadd, 2, 1) RUN(k_dadd, 4, 1) RUN(k_dadd, 8, 1) RUN(k_dadd, 16, 1)
  RUN(k_dfma, 1, 1) RUN(k_dfma, 4, 1) RUN(k_dfma, 8, 1) RUN(k_dfma, 16, 1)
  RUN(k_dadd, 4, 4) RUN(k_dadd, 8, 4) RUN(k_dadd, 4, 8) RUN(k_dadd, 8, 8) RUN(k_dadd, 4, 16)
  k_lds<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("lds.128 dependent: %.2f cycles\n", (double)h / n);
  return 0;
}
