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

// FP64 tensor-core throughput: independent mma.sync accumulators per warp.
__global__ void __launch_bounds__(256) k_dmma_m8n8k4(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; j++) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
  if (s == 1234.5678) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dmma_m16n8k16(double *out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; j++) b[j] = 1.0 - threadIdx.x * 1e-4 - j * 1e-5;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                     "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5678) out[0] = s;
}

// DMMA and DFMA issued together (each warp: `nm` m16n8k16 MMAs and 8 x `nf`
// DFMAs per iteration): do the FP64 tensor pipe and the FP64 FMA pipe add up?
__global__ void __launch_bounds__(256) k_mixed(double *out, int iters, int nm, int nf) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; j++) b[j] = 1.0 - threadIdx.x * 1e-4 - j * 1e-5;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
  double f0 = threadIdx.x * 1e-3, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5,
         f6 = f0 + 6, f7 = f0 + 7;
  const double fb = 0.999999, fc = 1e-7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (j < nm)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                     "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                       "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    for (int u = 0; u < nf; u++) {
      f0 = fma(f0, fb, fc); f1 = fma(f1, fb, fc); f2 = fma(f2, fb, fc); f3 = fma(f3, fb, fc);
      f4 = fma(f4, fb, fc); f5 = fma(f5, fb, fc); f6 = fma(f6, fb, fc); f7 = fma(f7, fb, fc);
    }
  }
  double s = f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
#pragma unroll
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5678) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dmma_m16n8k8(double *out, int iters) {
  double a[4], b[2];
#pragma unroll
  for (int j = 0; j < 4; j++) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 2; j++) b[j] = 1.0 - threadIdx.x * 1e-4 - j * 1e-5;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5678) out[0] = s;
}

// one warp: a dependent chain of m16n8k16 (which 1) / m16n8k8 (2) / m8n8k4 (0)
// MMAs on one accumulator; cycles per MMA into out[0]
__global__ void k_dmma_lat(double *out, int which, int n) {
  double a[8], b[4], c[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; j++) b[j] = 1.0 - threadIdx.x * 1e-4;
  const long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    if (which == 1)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                     "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    else if (which == 2)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    else
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / n;
  if (c[0] + c[1] + c[2] + c[3] == 1234.5678) out[1] = 1.0;
}

extern "C" {

double probe_dmma_latency(int which, int n) {
  double *out, h = 0;
  cudaMalloc(&out, 16);
  k_dmma_lat<<<1, 32>>>(out, which, n);
  k_dmma_lat<<<1, 32>>>(out, which, n);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  cudaFree(out);
  return h;
}

// TFLOP/s of k_mixed (DMMA 4096 flop each, DFMA 2 flop per lane)
double probe_mixed(int iters, int nm, int nf, float *ms_out) {
  int dev = 0, sms = 0, bps = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_mixed, 256, 0);
  double *out;
  cudaMalloc(&out, 8);
  dim3 grid(sms * bps), block(256);
  k_mixed<<<grid, block>>>(out, 16, nm, nf);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_mixed<<<grid, block>>>(out, iters, nm, nf);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  if (ms_out) *ms_out = ms;
  const double warps = (double)grid.x * (block.x / 32);
  const double flops = (double)iters * warps * (nm * 4096.0 + nf * 8.0 * 32 * 2);
  return flops / (ms * 1e-3) / 1e12;
}

// which: 0 = m8n8k4 (512 flop/mma), 1 = m16n8k16 (4096 flop/mma); TFLOP/s
double probe_dmma_peak(int which, int iters, float *ms_out) {
  int dev = 0, sms = 0, bps = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (which == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_dmma_m8n8k4, 256, 0);
  else if (which == 2)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_dmma_m16n8k8, 256, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_dmma_m16n8k16, 256, 0);
  double *out;
  cudaMalloc(&out, 8);
  dim3 grid(sms * bps), block(256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    if (which == 0) k_dmma_m8n8k4<<<grid, block>>>(out, iters);
    else if (which == 2) k_dmma_m16n8k8<<<grid, block>>>(out, iters);
    else k_dmma_m16n8k16<<<grid, block>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  if (ms_out) *ms_out = ms;
  const double per_mma = which == 0 ? 2.0 * 8 * 8 * 4 : (which == 2 ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16);
  const double mmas = (double)iters * (which == 0 ? 8 : 4) * grid.x * (block.x / 32);
  return mmas * per_mma / (ms * 1e-3) / 1e12;
}


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
