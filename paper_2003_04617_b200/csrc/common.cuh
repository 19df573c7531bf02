// common.cuh — shared device/host helpers for the revgpu kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/revgpu.h"

namespace rl {

// Programmatic dependent launch: a kernel launched with the
// ProgrammaticStreamSerialization attribute may start while its
// predecessor drains; it waits here (no-op for ordinary launches) before
// touching anything the predecessor writes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the next kernel of the chain to launch now (its own pdl_wait still
// waits for this grid to complete): used by short single-wave kernels so
// the next kernel's independent prologue overlaps them.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


constexpr unsigned FULL_MASK = 0xffffffffu;

// Host-computed natural-log table log(i), i in [0, LOGTAB_N), filled from the
// host C library (bit-identical to CPython's math.log, which the reference's
// s_log calls: values.py:365-372).  Integer logs are the whole transcendental
// cost of the series' integer divisions (`s /= k`, `s /= kn`).
constexpr int LOGTAB_N = 4096;

// Record a CUDA error for rl_last_error() and map it to RL_ERR_CUDA.
int cuda_status(cudaError_t e, const char *where);
int set_error(int code, const char *msg);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) / the occupancy query,
// cached per (function, device[, block, smem]): a host-buffer call or an
// un-graphed launch chain would otherwise pay them on every evaluation.
int smem_attr(const void *fn, size_t bytes, const char *what);
int occupancy(int *blocks_per_sm, const void *fn, int block, size_t smem, const char *what);

// Upload constant tables for the current device (idempotent, thread-safe).
int ensure_device_tables();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs of the current device (cached per device).
int sm_count();

// GMM: err! accumulated in the reference's order from err0, and (gradient)
// the primal-restoration residual and verdict (gmm.cu, k_gmm_restore)
struct GmmSeq {
  double err0;
  double *resid;     // device, 1 double (or null)
  int *code;         // device, 1 int32 (or null): RL_OK / RL_ERR_RESTORE
  int *verified;     // device, 1 int32 (or null): 1 = the parallel evaluation verified
  int force_serial;  // tests: take the sequential fallback
  int direction;     // objective only: +1 run, -1 uncall (~gmm)
};

// Block-wide sum of two counters and one atomicAdd per block.
template <int BLOCK>
__device__ __forceinline__ void block_add_counters(unsigned long long a, unsigned long long b,
                                                   unsigned long long *counters) {
  __shared__ unsigned long long red[2][BLOCK / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(FULL_MASK, a, o);
    b += __shfl_down_sync(FULL_MASK, b, o);
  }
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long sa = 0, sb = 0;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; w++) {
      sa += red[0][w];
      sb += red[1][w];
    }
    if (counters) {
      if (sa) atomicAdd(&counters[0], sa);
      if (sb) atomicAdd(&counters[1], sb);
    }
  }
}

}  // namespace rl
