// fp64probe.cu — measurement tool (not product): FP64 roofline denominators.
//   probe_dfma_peak  : DFMA-bound kernel, 8 independent FMA chains per thread,
//                      grid = SMs x resident blocks; timed with CUDA events.
//   probe_unary      : `reps` calls of exp / log / div per thread, used under
//                      `ncu --metrics sm__sass_thread_inst_executed_op_d{fma,add,mul}_pred_on.sum`
//                      to freeze the FP64 op weight of one libdevice call
//                      (profiles/fp64_weights.json), which the Bessel/GMM
//                      algorithmic FLOP counts use.
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double b, double c) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
         a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5678) out[0] = s;  // keep live
}

__global__ void k_unary(int which, const double *x, double *out, int reps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = x[i], acc = 0.0;
  for (int r = 0; r < reps; r++) {
    double a = 1.5 + v + r * 1e-2;  // exp args in [-30, -1.5]: the series' range
    double y = which == 0 ? exp(-a) : which == 1 ? log(a) : 1.0 / a;
    acc += y;
  }
  out[i] = acc;
}

extern "C" {

// Returns achieved FP64 TFLOP/s (2 flops per DFMA) of a kernel lasting ~ms.
double probe_dfma_peak(int iters, float *ms_out) {
  int dev = 0, sms = 0, bps = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_dfma, 256, 0);
  double *out;
  cudaMalloc(&out, 8);
  dim3 grid(sms * bps), block(256);
  k_dfma<<<grid, block>>>(out, 16, 0.999999, 1e-7);  // warm up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_dfma<<<grid, block>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  if (ms_out) *ms_out = ms;
  double flops = 2.0 * 64.0 * iters * (double)grid.x * block.x;
  return flops / (ms * 1e-3) / 1e12;
}

int probe_unary(int which, int n_threads, int reps) {
  double *x, *y;
  cudaMalloc(&x, n_threads * 8);
  cudaMalloc(&y, n_threads * 8);
  cudaMemset(x, 0, n_threads * 8);
  k_unary<<<n_threads / 128, 128>>>(which, x, y, reps);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(x);
  cudaFree(y);
  return (int)e;
}
}
