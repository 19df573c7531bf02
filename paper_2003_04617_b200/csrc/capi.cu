// capi.cu — the extern "C" boundary (include/revgpu.h): status strings,
// error plumbing, per-device table upload, the device-pointer entry points
// and the host-buffer (`_host`) entry points that pipeline chunks of
// host->device copy, kernel and device->host copy over three streams.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace rl {

// kernels (besselj.cu, ba.cu, gmm.cu)
int besselj_tables_init();
int launch_besselj(int32_t nu, const double *z, int64_t n, double thr, double tol, double seed,
                   int64_t max_trips, int32_t invcheck, double *J, double *dJdz, uint8_t *fail,
                   unsigned long long *counters, cudaStream_t st);
int launch_ba(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams, const double *X,
              const double *w, const double *feats, const int32_t *obs, double tol,
              int32_t invcheck, double *err, double *J, double *Jfeat, uint8_t *fail,
              unsigned long long *counters, cudaStream_t st);
size_t gmm_workspace_bytes(int32_t d, int32_t K, int64_t N);
int launch_gmm(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
               const double *means, const double *icf, const double *x, double gamma, int32_t m,
               double cst, double tol, int32_t invcheck, int32_t add_param_terms, double *out,
               uint8_t *fail, unsigned long long *counters, void *ws, size_t ws_bytes,
               cudaStream_t st, int grad, const GmmSeq *seq);
int launch_seq_sum(const double *t, int64_t M, double e0, int64_t mark, int32_t force_serial,
                   double *out2, int32_t *verified, cudaStream_t st);
int launch_besselj_run(int32_t nu, const double *z, int64_t n, double thr, double tol,
                       int64_t max_trips, int32_t invcheck, int32_t direction,
                       const double *out_in, double *out, uint8_t *fail,
                       unsigned long long *counters, cudaStream_t st);
int launch_besselj_hess(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, double *d2Jdz2, uint8_t *fail,
                        unsigned long long *counters, cudaStream_t st);
int launch_ba_residuals(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                        const double *X, const double *w, const double *feats,
                        const int32_t *obs, double tol, int32_t invcheck, double *err,
                        uint8_t *fail, unsigned long long *counters, cudaStream_t st);
int launch_ba_csr(int32_t n_cams, int32_t n_pts, int64_t n_obs, int64_t obs_offset,
                  int64_t n_obs_total, const double *cams, const double *X, const double *w,
                  const double *feats, const int32_t *obs, double tol, int32_t invcheck,
                  double *err, int32_t *rows, int32_t *cols, double *vals, uint8_t *fail,
                  unsigned long long *counters, cudaStream_t st);

static thread_local char g_last_error[512];

int set_error(int code, const char *msg) {
  snprintf(g_last_error, sizeof g_last_error, "%s", msg);
  return code;
}

int cuda_status(cudaError_t e, const char *where) {
  if (e == cudaSuccess) return RL_OK;
  snprintf(g_last_error, sizeof g_last_error, "%s: %s (%s)", where, cudaGetErrorString(e),
           cudaGetErrorName(e));
  return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? RL_ERR_NO_DEVICE
                                                                     : RL_ERR_CUDA;
}

constexpr int MAX_DEV = 64;

int smem_attr(const void *fn, size_t bytes, const char *what) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t &have = done[{fn, dev}];
  if (have >= bytes) return RL_OK;
  const int rc = cuda_status(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), what);
  if (!rc) have = bytes;
  return rc;
}

int occupancy(int *blocks_per_sm, const void *fn, int block, size_t smem, const char *what) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, int, size_t>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(fn, dev, block, smem);
  const auto it = done.find(key);
  if (it != done.end()) {
    *blocks_per_sm = it->second;
    return RL_OK;
  }
  const int rc = cuda_status(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, block, smem), what);
  if (!rc) done[key] = *blocks_per_sm;
  return rc;
}

int ensure_device_tables() {
  static std::once_flag once[MAX_DEV];
  static int status[MAX_DEV];
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  if (dev < 0 || dev >= MAX_DEV) return set_error(RL_ERR_INVALID, "device ordinal out of range");
  std::call_once(once[dev], [dev] {
    cudaDeviceProp prop;
    int r = cuda_status(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (!r && prop.major != 10)
      r = set_error(RL_ERR_NO_DEVICE, "revgpu is built for sm_100a (B200); device is not cc 10.x");
    if (!r) r = besselj_tables_init();
    status[dev] = r;
  });
  return status[dev];
}

int sm_count() {
  static int cache[MAX_DEV];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAX_DEV) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline: chunk i's H2D, kernel and D2H are issued on stream
// i % NS; device buffers come from the stream-ordered pool allocator.
// ---------------------------------------------------------------------------
struct DevBuf {
  void *p = nullptr;
  cudaStream_t st = nullptr;
  int alloc(size_t bytes, cudaStream_t s) {
    st = s;
    return cuda_status(cudaMallocAsync(&p, bytes ? bytes : 1, s), "cudaMallocAsync");
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

struct Pipeline {
  // The three streams of the host-buffer entries are created once per
  // (host thread, device) and reused by every call: creating and destroying
  // streams per call cost more than a small GMM evaluation.
  static constexpr int NS = 3;
  cudaStream_t st[NS] = {nullptr, nullptr, nullptr};
  int dev_prev = -1;
  int init(int device) {
    cudaGetDevice(&dev_prev);
    if (device < 0 || device >= MAX_DEV) return set_error(RL_ERR_INVALID, "bad device ordinal");
    int rc = cuda_status(cudaSetDevice(device), "cudaSetDevice");
    if (rc) return rc;
    static thread_local cudaStream_t cache[MAX_DEV][NS];
    static thread_local bool made[MAX_DEV];
    if (!made[device]) {
      // keep freed stream-ordered allocations in the pool between calls (the
      // default threshold 0 returns them to the driver at every sync)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      for (auto &s : cache[device]) {
        rc = cuda_status(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
        if (rc) return rc;
      }
      made[device] = true;
    }
    for (int i = 0; i < NS; i++) st[i] = cache[device][i];
    return RL_OK;
  }
  // device scratch, cached per (host thread, device): a host-buffer call
  // carves its buffers out of it instead of allocating and freeing each one
  struct Arena {
    void *buf[MAX_DEV] = {};
    size_t have[MAX_DEV] = {};
    ~Arena() {                   // thread exit: give the device memory back
      for (int dv = 0; dv < MAX_DEV; dv++)
        if (buf[dv]) {
          cudaSetDevice(dv);
          cudaFree(buf[dv]);
        }
    }
  };
  static int arena(int device, size_t bytes, void **out) {
    static thread_local Arena a;
    if (bytes > a.have[device]) {
      if (a.buf[device]) cudaFree(a.buf[device]);
      a.buf[device] = nullptr;
      a.have[device] = 0;
      const int rc = cuda_status(cudaMalloc(&a.buf[device], bytes), "cudaMalloc arena");
      if (rc) return rc;
      a.have[device] = bytes;
    }
    *out = a.buf[device];
    return RL_OK;
  }
  // pinned host scratch, cached per host thread (a D2H copy into pageable
  // memory would block the host and serialise the chunk pipeline)
  static int pinned(size_t bytes, void **out) {
    static thread_local void *buf = nullptr;
    static thread_local size_t have = 0;
    if (bytes > have) {
      if (buf) cudaFreeHost(buf);
      buf = nullptr;
      have = 0;
      const int rc = cuda_status(cudaMallocHost(&buf, bytes), "cudaMallocHost");
      if (rc) return rc;
      have = bytes;
    }
    *out = buf;
    return RL_OK;
  }
  int finish() {
    int rc = RL_OK;
    for (auto &s : st)
      if (s) {
        int r = cuda_status(cudaStreamSynchronize(s), "pipeline sync");
        if (!rc) rc = r;
      }
    return rc;
  }
  ~Pipeline() {
    for (auto &s : st)
      if (s) cudaStreamSynchronize(s);
    if (dev_prev >= 0) cudaSetDevice(dev_prev);
  }
};

// Host-buffer pipeline of the per-element Bessel entries (run / uncall,
// Hessian): chunks of z (and out_in) go up, `nout` double arrays and the
// status bytes come down, over the three cached streams.  launch(s, m, dz,
// din, douts, dfail, counters, stream) runs the device entry on one chunk.
template <class Launch>
static int bessel_host_chunks(int64_t n, const double *z, const double *in2, int nout,
                              double *const outs[3], uint8_t *fail,
                              unsigned long long *n_failed, int32_t device, Launch launch) {
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  const int64_t CH = int64_t(1) << 22;
  const int64_t nch = (n + CH - 1) / CH;
  const int64_t bufn = std::min<int64_t>(CH, std::max<int64_t>(n, 1));
  DevBuf dz[Pipeline::NS], din[Pipeline::NS], dout[Pipeline::NS][3], dfl[Pipeline::NS], dc;
  if ((rc = dc.alloc(2 * 8 * Pipeline::NS, pl.st[0])) ||
      (rc = cuda_status(cudaMemsetAsync(dc.p, 0, 2 * 8 * Pipeline::NS, pl.st[0]), "memset")))
    return rc;
  for (int s = 0; s < Pipeline::NS && s < std::max<int64_t>(nch, 1); s++) {
    if ((rc = dz[s].alloc(bufn * 8, pl.st[s])) || (rc = din[s].alloc(in2 ? bufn * 8 : 8, pl.st[s])) ||
        (rc = dfl[s].alloc(bufn, pl.st[s])))
      return rc;
    for (int o = 0; o < nout; o++)
      if ((rc = dout[s][o].alloc(bufn * 8, pl.st[s]))) return rc;
  }
  if ((rc = pl.finish())) return rc;              // counters zeroed before any stream uses them
  auto *cnt = (unsigned long long *)dc.p;
  for (int64_t c = 0; c < nch; c++) {
    const int s = (int)(c % Pipeline::NS);
    const int64_t off = c * CH, m = std::min(CH, n - off);
    cudaStream_t st = pl.st[s];
    if ((rc = cuda_status(cudaMemcpyAsync(dz[s].p, z + off, m * 8, cudaMemcpyHostToDevice, st),
                          "H2D z")))
      return rc;
    if (in2 && (rc = cuda_status(cudaMemcpyAsync(din[s].p, in2 + off, m * 8,
                                                 cudaMemcpyHostToDevice, st), "H2D in")))
      return rc;
    double *douts[3] = {(double *)dout[s][0].p, (double *)dout[s][1].p, (double *)dout[s][2].p};
    if ((rc = launch(m, (const double *)dz[s].p, in2 ? (const double *)din[s].p : nullptr, douts,
                     (uint8_t *)dfl[s].p, cnt + 2 * s, st)))
      return rc;
    for (int o = 0; o < nout; o++)
      if ((rc = cuda_status(cudaMemcpyAsync(outs[o] + off, douts[o], m * 8,
                                            cudaMemcpyDeviceToHost, st), "D2H out")))
        return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(fail + off, dfl[s].p, m, cudaMemcpyDeviceToHost, st),
                          "D2H fail")))
      return rc;
  }
  if ((rc = pl.finish())) return rc;
  unsigned long long h[2 * Pipeline::NS];
  if ((rc = cuda_status(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost), "D2H counters")))
    return rc;
  unsigned long long nf = 0;
  for (int q = 0; q < Pipeline::NS; q++) nf += h[2 * q + 1];
  if (n_failed) *n_failed = nf;
  return RL_OK;
}

}  // namespace rl

using namespace rl;

extern "C" {

int rl_abi_version(void) { return RL_ABI_VERSION; }

const char *rl_strerror(int code) {
  switch (code) {
    case RL_OK: return "ok";
    case RL_ERR_POSTCONDITION: return "PostconditionMismatch";
    case RL_ERR_DIRTY_ANCILLA: return "DirtyAncilla";
    case RL_ERR_DOMAIN: return "RevDomainError";
    case RL_ERR_ITERATOR: return "LoopIteratorMutated";
    case RL_ERR_RESTORE: return "RevError";
    case RL_ERR_FUEL: return "FuelExhausted";
    case RL_ERR_KIND: return "KindError";
    case RL_ERR_INDEX: return "IndexOutOfBounds";
    case RL_ERR_OVERFLOW: return "OverflowError";
    case RL_ERR_INVALID: return "invalid argument";
    case RL_ERR_CUDA: return "CUDA error";
    case RL_ERR_NO_DEVICE: return "no usable sm_100 device";
    default: return "unknown status";
  }
}

const char *rl_last_error(void) { return g_last_error; }

int rl_besselj_grad_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, uint8_t *fail, unsigned long long *counters,
                        void *stream) {
  return launch_besselj(nu, z, n, thr, tol, seed, max_trips, invcheck, J, dJdz, fail, counters,
                        as_stream(stream));
}

// Per-chunk list of the nonzero status codes (index << 8 | code): almost every
// element succeeds, so the host-buffer entry downloads this list instead of
// one status byte per element.
__global__ void k_compact_fail(const uint8_t *__restrict__ f, int64_t m,
                               uint32_t *__restrict__ list, unsigned *__restrict__ count,
                               unsigned cap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t c = f[i];
    if (c) {
      const unsigned k = atomicAdd(count, 1u);
      if (k < cap) list[k] = ((uint32_t)i << 8) | c;
    }
  }
}

int rl_besselj_grad_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                             double seed, int64_t max_trips, int32_t invcheck, double *J,
                             double *dJdz, uint8_t *fail, unsigned long long *sum_trips,
                             unsigned long long *n_failed, int32_t device) {
  if (n < 0 || (n > 0 && (!z || !J || !dJdz || !fail)))
    return set_error(RL_ERR_INVALID, "rl_besselj_grad_f64_host: bad argument");
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
#ifndef BJ_HOST_CH_LOG2
#define BJ_HOST_CH_LOG2 22
#endif
  const int64_t CH = int64_t(1) << BJ_HOST_CH_LOG2;  // elements per chunk (4 Mi = 32 MiB of z)
  static_assert(BJ_HOST_CH_LOG2 <= 24, "chunk index must fit the 24-bit field of the fail list");
  constexpr unsigned CAP = 16384;                    // listed failures per chunk
  const int64_t nch = (n + CH - 1) / CH;
  const int64_t bufn = std::min<int64_t>(CH, std::max<int64_t>(n, 1));
  DevBuf dz[Pipeline::NS], dJ[Pipeline::NS], dg[Pipeline::NS], df, dl, dc;
  for (int s = 0; s < Pipeline::NS && s < std::max<int64_t>(nch, 1); s++) {
    if ((rc = dz[s].alloc(bufn * 8, pl.st[s])) || (rc = dJ[s].alloc(bufn * 8, pl.st[s])) ||
        (rc = dg[s].alloc(bufn * 8, pl.st[s])))
      return rc;
  }
  // status bytes stay on the device for the whole batch (the overflow path
  // reads them back); the lists and counts are per chunk
  const int64_t nl = std::max<int64_t>(nch, 1);
  if ((rc = df.alloc(std::max<int64_t>(n, 1), pl.st[0])) ||
      (rc = dl.alloc(nl * CAP * 4, pl.st[0])) ||
      (rc = dc.alloc(2 * sizeof(unsigned long long) * Pipeline::NS + nl * 4, pl.st[0])))
    return rc;
  auto *cnt = (unsigned long long *)dc.p;
  auto *fcount = (unsigned *)(cnt + 2 * Pipeline::NS);
  if ((rc = cuda_status(cudaMemsetAsync(dc.p, 0, 2 * 8 * Pipeline::NS + nl * 4, pl.st[0]),
                        "memset")))
    return rc;
  if ((rc = pl.finish())) return rc;  // counters zeroed before any stream uses them
  void *hp = nullptr;
  if ((rc = Pipeline::pinned((size_t)nl * (CAP + 1) * 4, &hp))) return rc;
  unsigned *hcount = (unsigned *)hp;
  uint32_t *hlist = hcount + nl;
  for (int64_t c = 0; c < nch; c++) {
    const int s = (int)(c % Pipeline::NS);
    const int64_t off = c * CH, m = std::min(CH, n - off);
    cudaStream_t st = pl.st[s];
    uint8_t *fc = (uint8_t *)df.p + off;
    uint32_t *lc = (uint32_t *)dl.p + c * CAP;
    if ((rc = cuda_status(cudaMemcpyAsync(dz[s].p, z + off, m * 8, cudaMemcpyHostToDevice, st),
                          "H2D z")))
      return rc;
    if ((rc = launch_besselj(nu, (double *)dz[s].p, m, thr, tol, seed, max_trips, invcheck,
                             (double *)dJ[s].p, (double *)dg[s].p, fc, cnt + 2 * s, st)))
      return rc;
    k_compact_fail<<<(unsigned)std::min<int64_t>((m + 255) / 256, 4 * sm_count()), 256, 0, st>>>(
        fc, m, lc, fcount + c, CAP);
    if ((rc = cuda_status(cudaGetLastError(), "k_compact_fail")) ||
        (rc = cuda_status(cudaMemcpyAsync(J + off, dJ[s].p, m * 8, cudaMemcpyDeviceToHost, st),
                          "D2H J")) ||
        (rc = cuda_status(cudaMemcpyAsync(dJdz + off, dg[s].p, m * 8, cudaMemcpyDeviceToHost, st),
                          "D2H dJdz")) ||
        (rc = cuda_status(cudaMemcpyAsync(&hcount[c], fcount + c, 4, cudaMemcpyDeviceToHost, st),
                          "D2H fail count")) ||
        (rc = cuda_status(cudaMemcpyAsync(&hlist[(size_t)c * CAP], lc, CAP * 4,
                                          cudaMemcpyDeviceToHost, st), "D2H fail list")))
      return rc;
  }
  memset(fail, 0, (size_t)n);  // the host thread is idle while the copies run
  if ((rc = pl.finish())) return rc;
  for (int64_t c = 0; c < nch; c++) {
    const int64_t off = c * CH, m = std::min(CH, n - off);
    if (hcount[c] > CAP) {       // more failures than the list holds: the whole chunk
      if ((rc = cuda_status(cudaMemcpy(fail + off, (uint8_t *)df.p + off, m,
                                       cudaMemcpyDeviceToHost), "D2H fail")))
        return rc;
      continue;
    }
    for (unsigned k = 0; k < hcount[c]; k++) {
      const uint32_t e = hlist[(size_t)c * CAP + k];
      fail[off + (e >> 8)] = (uint8_t)(e & 0xff);
    }
  }
  unsigned long long h[2 * Pipeline::NS];
  if ((rc = cuda_status(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost), "D2H counters")))
    return rc;
  unsigned long long tr = 0, nf = 0;
  for (int s = 0; s < Pipeline::NS; s++) {
    tr += h[2 * s];
    nf += h[2 * s + 1];
  }
  if (sum_trips) *sum_trips = tr;
  if (n_failed) *n_failed = nf;
  return RL_OK;
}

int rl_besselj_run_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                            int64_t max_trips, int32_t invcheck, int32_t direction,
                            const double *out_in, double *out, uint8_t *fail,
                            unsigned long long *n_failed, int32_t device) {
  if (n < 0 || (n > 0 && (!z || !out || !fail)) || (direction != 1 && direction != -1))
    return set_error(RL_ERR_INVALID, "rl_besselj_run_f64_host: bad argument");
  double *const outs[3] = {out, nullptr, nullptr};
  return bessel_host_chunks(
      n, z, out_in, 1, outs, fail, n_failed, device,
      [&](int64_t m, const double *dz, const double *din, double *const *douts, uint8_t *dfl,
          unsigned long long *cnt, cudaStream_t st) {
        return launch_besselj_run(nu, dz, m, thr, tol, max_trips, invcheck, direction, din,
                                  douts[0], dfl, cnt, st);
      });
}

int rl_besselj_hess_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                             double seed, int64_t max_trips, int32_t invcheck, double *J,
                             double *dJdz, double *d2Jdz2, uint8_t *fail,
                             unsigned long long *n_failed, int32_t device) {
  if (n < 0 || (n > 0 && (!z || !J || !dJdz || !d2Jdz2 || !fail)))
    return set_error(RL_ERR_INVALID, "rl_besselj_hess_f64_host: bad argument");
  double *const outs[3] = {J, dJdz, d2Jdz2};
  return bessel_host_chunks(
      n, z, nullptr, 3, outs, fail, n_failed, device,
      [&](int64_t m, const double *dz, const double *, double *const *douts, uint8_t *dfl,
          unsigned long long *cnt, cudaStream_t st) {
        return launch_besselj_hess(nu, dz, m, thr, tol, seed, max_trips, invcheck, douts[0],
                                   douts[1], douts[2], dfl, cnt, st);
      });
}

int rl_ba_residuals_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                             const double *X, const double *w, const double *feats,
                             const int32_t *obs, double tol, int32_t invcheck, double *err,
                             uint8_t *fail, unsigned long long *n_failed, int32_t device) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !err || !fail)))
    return set_error(RL_ERR_INVALID, "rl_ba_residuals_f64_host: bad argument");
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  cudaStream_t st = pl.st[0];
  const size_t sizes[8] = {(size_t)n_cams * 88, (size_t)n_pts * 24, (size_t)n_obs * 8,
                           (size_t)n_obs * 16, (size_t)n_obs * 8, (size_t)n_obs * 24,
                           (size_t)std::max<int64_t>(n_obs, 1), 16};
  size_t total = 0;
  for (size_t b : sizes) total += (b + 255) & ~size_t(255);
  void *base = nullptr;
  if ((rc = Pipeline::arena(device, total, &base))) return rc;
  char *q[8];
  size_t off = 0;
  for (int i = 0; i < 8; i++) {
    q[i] = (char *)base + off;
    off += (sizes[i] + 255) & ~size_t(255);
  }
  const void *src[5] = {cams, X, w, feats, obs};
  for (int i = 0; i < 5; i++)
    if (sizes[i] && (rc = cuda_status(cudaMemcpyAsync(q[i], src[i], sizes[i],
                                                      cudaMemcpyHostToDevice, st), "H2D")))
      return rc;
  if ((rc = cuda_status(cudaMemsetAsync(q[7], 0, 16, st), "memset")) ||
      (rc = launch_ba_residuals(n_cams, n_pts, n_obs, (double *)q[0], (double *)q[1],
                                (double *)q[2], (double *)q[3], (int32_t *)q[4], tol, invcheck,
                                (double *)q[5], (uint8_t *)q[6], (unsigned long long *)q[7], st)))
    return rc;
  unsigned long long h[2];
  if ((n_obs > 0 && ((rc = cuda_status(cudaMemcpyAsync(err, q[5], sizes[5], cudaMemcpyDeviceToHost,
                                                       st), "D2H err")) ||
                     (rc = cuda_status(cudaMemcpyAsync(fail, q[6], n_obs, cudaMemcpyDeviceToHost,
                                                       st), "D2H fail")))) ||
      (rc = cuda_status(cudaMemcpyAsync(h, q[7], 16, cudaMemcpyDeviceToHost, st), "D2H counters")))
    return rc;
  if ((rc = pl.finish())) return rc;
  if (n_failed) *n_failed = h[1];
  return RL_OK;
}

int rl_ba_jac_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                  const double *X, const double *w, const double *feats, const int32_t *obs,
                  double tol, int32_t invcheck, double *err, double *J, double *Jfeat,
                  uint8_t *fail, unsigned long long *counters, void *stream) {
  return launch_ba(n_cams, n_pts, n_obs, cams, X, w, feats, obs, tol, invcheck, err, J, Jfeat,
                   fail, counters, as_stream(stream));
}

int rl_ba_jac_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                       const double *X, const double *w, const double *feats,
                       const int32_t *obs, double tol, int32_t invcheck, double *err,
                       double *J, uint8_t *fail, unsigned long long *n_failed, int32_t device) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !J || !fail)))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_f64_host: bad argument");
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  // cameras and points are replicated once; observations stream in chunks
  DevBuf dcam, dX, dc;
  if ((rc = dcam.alloc((size_t)n_cams * 11 * 8, pl.st[0])) ||
      (rc = dX.alloc((size_t)n_pts * 3 * 8, pl.st[0])) ||
      (rc = dc.alloc(2 * 8 * Pipeline::NS, pl.st[0])))
    return rc;
  auto *cnt = (unsigned long long *)dc.p;
  if ((rc = cuda_status(cudaMemcpyAsync(dcam.p, cams, (size_t)n_cams * 88, cudaMemcpyHostToDevice,
                                        pl.st[0]), "H2D cams")) ||
      (rc = cuda_status(cudaMemcpyAsync(dX.p, X, (size_t)n_pts * 24, cudaMemcpyHostToDevice,
                                        pl.st[0]), "H2D X")) ||
      (rc = cuda_status(cudaMemsetAsync(cnt, 0, 2 * 8 * Pipeline::NS, pl.st[0]), "memset")))
    return rc;
  if ((rc = pl.finish())) return rc;
  const int64_t CH = int64_t(1) << 18;
  const int64_t nch = (n_obs + CH - 1) / CH;
  const int64_t bufn = std::min<int64_t>(CH, std::max<int64_t>(n_obs, 1));
  DevBuf dw[Pipeline::NS], df2[Pipeline::NS], dob[Pipeline::NS], dJ[Pipeline::NS],
      de[Pipeline::NS], dfl[Pipeline::NS];
  for (int s = 0; s < Pipeline::NS && s < std::max<int64_t>(nch, 1); s++) {
    if ((rc = dw[s].alloc(bufn * 8, pl.st[s])) || (rc = df2[s].alloc(bufn * 16, pl.st[s])) ||
        (rc = dob[s].alloc(bufn * 8, pl.st[s])) || (rc = dJ[s].alloc(bufn * 31 * 8, pl.st[s])) ||
        (rc = de[s].alloc(err ? bufn * 24 : 8, pl.st[s])) || (rc = dfl[s].alloc(bufn, pl.st[s])))
      return rc;
  }
  for (int64_t c = 0; c < nch; c++) {
    const int s = (int)(c % Pipeline::NS);
    const int64_t off = c * CH, m = std::min(CH, n_obs - off);
    cudaStream_t st = pl.st[s];
    if ((rc = cuda_status(cudaMemcpyAsync(dw[s].p, w + off, m * 8, cudaMemcpyHostToDevice, st),
                          "H2D w")) ||
        (rc = cuda_status(cudaMemcpyAsync(df2[s].p, feats + 2 * off, m * 16,
                                          cudaMemcpyHostToDevice, st), "H2D feats")) ||
        (rc = cuda_status(cudaMemcpyAsync(dob[s].p, obs + 2 * off, m * 8, cudaMemcpyHostToDevice,
                                          st), "H2D obs")))
      return rc;
    if ((rc = launch_ba(n_cams, n_pts, m, (double *)dcam.p, (double *)dX.p, (double *)dw[s].p,
                        (double *)df2[s].p, (int32_t *)dob[s].p, tol, invcheck,
                        err ? (double *)de[s].p : nullptr, (double *)dJ[s].p, nullptr,
                        (uint8_t *)dfl[s].p, cnt + 2 * s, st)))
      return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(J + 31 * off, dJ[s].p, m * 31 * 8,
                                          cudaMemcpyDeviceToHost, st), "D2H J")) ||
        (rc = cuda_status(cudaMemcpyAsync(fail + off, dfl[s].p, m, cudaMemcpyDeviceToHost, st),
                          "D2H fail")))
      return rc;
    if (err && (rc = cuda_status(cudaMemcpyAsync(err + 3 * off, de[s].p, m * 24,
                                                 cudaMemcpyDeviceToHost, st), "D2H err")))
      return rc;
  }
  if ((rc = pl.finish())) return rc;
  unsigned long long h[2 * Pipeline::NS];
  if ((rc = cuda_status(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost), "D2H counters")))
    return rc;
  unsigned long long nf = 0;
  for (int s = 0; s < Pipeline::NS; s++) nf += h[2 * s + 1];
  if (n_failed) *n_failed = nf;
  return RL_OK;
}

size_t rl_gmm_workspace_bytes(int32_t d, int32_t K, int64_t N) {
  return gmm_workspace_bytes(d, K, N);
}

int rl_gmm_grad_f64(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
                    const double *means, const double *icf, const double *x, double gamma,
                    int32_t m, double cst, double tol, int32_t invcheck,
                    int32_t add_param_terms, double *out, uint8_t *fail,
                    unsigned long long *counters, void *ws, size_t ws_bytes, void *stream) {
  return launch_gmm(d, K, N, N_total, alphas, means, icf, x, gamma, m, cst, tol, invcheck,
                    add_param_terms, out, fail, counters, ws, ws_bytes, as_stream(stream), 1,
                    nullptr);
}

int rl_gmm_gradient_f64(int32_t d, int32_t K, int64_t N, const double *alphas,
                        const double *means, const double *icf, const double *x, double gamma,
                        int32_t m, double cst, double err0, double tol, int32_t invcheck,
                        double *out, double *resid, int32_t *restore_code, uint8_t *fail,
                        unsigned long long *counters, void *ws, size_t ws_bytes, void *stream) {
  const GmmSeq seq{err0, resid, restore_code, nullptr, 0, 1};
  return launch_gmm(d, K, N, N, alphas, means, icf, x, gamma, m, cst, tol, invcheck, 1, out, fail,
                    counters, ws, ws_bytes, as_stream(stream), 1, &seq);
}

int rl_gmm_run_f64(int32_t d, int32_t K, int64_t N, const double *alphas, const double *means,
                   const double *icf, const double *x, double gamma, int32_t m, double cst,
                   double err0, double tol, int32_t invcheck, int32_t direction, double *err,
                   uint8_t *fail, unsigned long long *counters, void *ws, size_t ws_bytes,
                   void *stream) {
  if (direction != 1 && direction != -1)
    return set_error(RL_ERR_INVALID, "rl_gmm_run_f64: direction must be +1 or -1");
  const GmmSeq seq{err0, nullptr, nullptr, nullptr, 0, direction};
  return launch_gmm(d, K, N, N, alphas, means, icf, x, gamma, m, cst, tol, invcheck, 1, err, fail,
                    counters, ws, ws_bytes, as_stream(stream), 0, &seq);
}

int64_t rl_gmm_statement_count(int32_t d, int32_t K, int64_t N, int64_t U, int64_t A) {
  const int64_t dd = d, kk = K;
  return N * (6 * kk * dd * dd + 22 * kk * dd + 48 * kk + 13) + 4 * U + 3 * kk * dd * dd +
         9 * kk * dd + 28 * kk + 4 * A + 33;
}

int rl_seq_sum_f64(const double *t, int64_t M, double e0, int64_t mark, int32_t force_serial,
                   double *out2, int32_t *verified, void *stream) {
  return launch_seq_sum(t, M, e0, mark, force_serial, out2, verified, as_stream(stream));
}

int rl_gmm_objective_f64(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
                         const double *means, const double *icf, const double *x, double gamma,
                         int32_t m, double cst, double tol, int32_t invcheck,
                         int32_t add_param_terms, double *err, uint8_t *fail,
                         unsigned long long *counters, void *ws, size_t ws_bytes, void *stream) {
  return launch_gmm(d, K, N, N_total, alphas, means, icf, x, gamma, m, cst, tol, invcheck,
                    add_param_terms, err, fail, counters, ws, ws_bytes, as_stream(stream), 0,
                    nullptr);
}

int rl_besselj_run_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                       int64_t max_trips, int32_t invcheck, int32_t direction,
                       const double *out_in, double *out, uint8_t *fail,
                       unsigned long long *counters, void *stream) {
  return launch_besselj_run(nu, z, n, thr, tol, max_trips, invcheck, direction, out_in, out, fail,
                            counters, as_stream(stream));
}

int rl_besselj_hess_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, double *d2Jdz2, uint8_t *fail,
                        unsigned long long *counters, void *stream) {
  return launch_besselj_hess(nu, z, n, thr, tol, seed, max_trips, invcheck, J, dJdz, d2Jdz2,
                             fail, counters, as_stream(stream));
}

int rl_ba_residuals_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                        const double *X, const double *w, const double *feats,
                        const int32_t *obs, double tol, int32_t invcheck, double *err,
                        uint8_t *fail, unsigned long long *counters, void *stream) {
  return launch_ba_residuals(n_cams, n_pts, n_obs, cams, X, w, feats, obs, tol, invcheck, err,
                             fail, counters, as_stream(stream));
}

int rl_ba_jac_csr_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, int64_t obs_offset,
                      int64_t n_obs_total, const double *cams, const double *X, const double *w,
                      const double *feats, const int32_t *obs, double tol, int32_t invcheck,
                      double *err, int32_t *rows, int32_t *cols, double *vals, uint8_t *fail,
                      unsigned long long *counters, void *stream) {
  return launch_ba_csr(n_cams, n_pts, n_obs, obs_offset, n_obs_total, cams, X, w, feats, obs, tol,
                       invcheck, err, rows, cols, vals, fail, counters, as_stream(stream));
}

int rl_ba_jac_csr_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                           const double *X, const double *w, const double *feats,
                           const int32_t *obs, double tol, int32_t invcheck, int32_t *rows,
                           int32_t *cols, double *vals, uint8_t *fail,
                           unsigned long long *n_failed, int32_t device) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 || !vals || (cols && !rows) || (rows && !cols && n_obs > 0) ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !fail)))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_csr_f64_host: bad argument");
  if (31LL * n_obs > INT32_MAX || 11LL * n_cams + 3LL * n_pts + n_obs > INT32_MAX)
    return set_error(RL_ERR_INVALID,
                     "rl_ba_jac_csr_f64_host: nnz or ncols exceeds int32 (BASparseMat)");
  if (rows) rows[3 * n_obs] = (int32_t)(31 * n_obs);
  if (n_obs == 0) return RL_OK;
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  DevBuf dcam, dX, dc;
  if ((rc = dcam.alloc((size_t)n_cams * 11 * 8, pl.st[0])) ||
      (rc = dX.alloc((size_t)n_pts * 3 * 8, pl.st[0])) ||
      (rc = dc.alloc(2 * 8 * Pipeline::NS, pl.st[0])))
    return rc;
  auto *cnt = (unsigned long long *)dc.p;
  if ((rc = cuda_status(cudaMemcpyAsync(dcam.p, cams, (size_t)n_cams * 88, cudaMemcpyHostToDevice,
                                        pl.st[0]), "H2D cams")) ||
      (rc = cuda_status(cudaMemcpyAsync(dX.p, X, (size_t)n_pts * 24, cudaMemcpyHostToDevice,
                                        pl.st[0]), "H2D X")) ||
      (rc = cuda_status(cudaMemsetAsync(cnt, 0, 2 * 8 * Pipeline::NS, pl.st[0]), "memset")))
    return rc;
  if ((rc = pl.finish())) return rc;
  // each chunk is launched as a shard (obs_offset = chunk start, total = n_obs):
  // its local [reprojection | weight] parts land in the two halves of the
  // global arrays
  const int64_t CH = int64_t(1) << 18;
  const int64_t nch = (n_obs + CH - 1) / CH;
  const int64_t bufn = std::min<int64_t>(CH, n_obs);
  DevBuf dw[Pipeline::NS], df2[Pipeline::NS], dob[Pipeline::NS], dv[Pipeline::NS],
      dr[Pipeline::NS], dcl[Pipeline::NS], dfl[Pipeline::NS];
  for (int s = 0; s < Pipeline::NS && s < nch; s++) {
    if ((rc = dw[s].alloc(bufn * 8, pl.st[s])) || (rc = df2[s].alloc(bufn * 16, pl.st[s])) ||
        (rc = dob[s].alloc(bufn * 8, pl.st[s])) || (rc = dv[s].alloc(bufn * 31 * 8, pl.st[s])) ||
        (rc = dr[s].alloc(rows ? (bufn * 3 + 1) * 4 : 4, pl.st[s])) ||
        (rc = dcl[s].alloc(rows ? bufn * 31 * 4 : 4, pl.st[s])) ||
        (rc = dfl[s].alloc(bufn, pl.st[s])))
      return rc;
  }
  for (int64_t c = 0; c < nch; c++) {
    const int s = (int)(c % Pipeline::NS);
    const int64_t off = c * CH, m = std::min(CH, n_obs - off);
    cudaStream_t st = pl.st[s];
    if ((rc = cuda_status(cudaMemcpyAsync(dw[s].p, w + off, m * 8, cudaMemcpyHostToDevice, st),
                          "H2D w")) ||
        (rc = cuda_status(cudaMemcpyAsync(df2[s].p, feats + 2 * off, m * 16,
                                          cudaMemcpyHostToDevice, st), "H2D feats")) ||
        (rc = cuda_status(cudaMemcpyAsync(dob[s].p, obs + 2 * off, m * 8, cudaMemcpyHostToDevice,
                                          st), "H2D obs")))
      return rc;
    int32_t *r = rows ? (int32_t *)dr[s].p : nullptr, *cl = rows ? (int32_t *)dcl[s].p : nullptr;
    if ((rc = launch_ba_csr(n_cams, n_pts, m, off, n_obs, (double *)dcam.p, (double *)dX.p,
                            (double *)dw[s].p, (double *)df2[s].p, (int32_t *)dob[s].p, tol,
                            invcheck, nullptr, r, cl, (double *)dv[s].p, (uint8_t *)dfl[s].p,
                            cnt + 2 * s, st)))
      return rc;
    const double *v = (const double *)dv[s].p;
    if ((rc = cuda_status(cudaMemcpyAsync(vals + 30 * off, v, m * 30 * 8, cudaMemcpyDeviceToHost,
                                          st), "D2H vals")) ||
        (rc = cuda_status(cudaMemcpyAsync(vals + 30 * n_obs + off, v + 30 * m, m * 8,
                                          cudaMemcpyDeviceToHost, st), "D2H vals (w)")) ||
        (rc = cuda_status(cudaMemcpyAsync(fail + off, dfl[s].p, m, cudaMemcpyDeviceToHost, st),
                          "D2H fail")))
      return rc;
    if (rows &&
        ((rc = cuda_status(cudaMemcpyAsync(cols + 30 * off, cl, m * 30 * 4,
                                           cudaMemcpyDeviceToHost, st), "D2H cols")) ||
         (rc = cuda_status(cudaMemcpyAsync(cols + 30 * n_obs + off, cl + 30 * m, m * 4,
                                           cudaMemcpyDeviceToHost, st), "D2H cols (w)")) ||
         (rc = cuda_status(cudaMemcpyAsync(rows + 2 * off, r, m * 2 * 4, cudaMemcpyDeviceToHost,
                                           st), "D2H rows")) ||
         (rc = cuda_status(cudaMemcpyAsync(rows + 2 * n_obs + off, r + 2 * m, m * 4,
                                           cudaMemcpyDeviceToHost, st), "D2H rows (w)"))))
      return rc;
  }
  if ((rc = pl.finish())) return rc;
  unsigned long long h[2 * Pipeline::NS];
  if ((rc = cuda_status(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost), "D2H counters")))
    return rc;
  unsigned long long nf = 0;
  for (int s = 0; s < Pipeline::NS; s++) nf += h[2 * s + 1];
  if (n_failed) *n_failed = nf;
  return RL_OK;
}

// host-buffer GMM gradient; with `restore` the drop-in gradient() of
// rl_gmm_gradient_f64 (err! in the reference's order from err0, restoration
// verdict as the return code), else rl_gmm_grad_f64's
static int gmm_grad_host(int32_t d, int32_t K, int64_t N, int64_t N_total, int32_t add_param,
                         const double *alphas, const double *means, const double *icf,
                         const double *x, double gamma, int32_t m, double cst, double tol,
                         int32_t invcheck, double *out, unsigned long long *n_failed,
                         int32_t device, bool restore, double err0, double *resid) {
  if (d <= 0 || K <= 0 || N < 0 || N_total < N || !alphas || !means || !icf || (N > 0 && !x) ||
      !out)
    return set_error(RL_ERR_INVALID, "rl_gmm_grad_f64_host: bad argument");
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  cudaStream_t st = pl.st[0];
  const size_t P = (size_t)d * (d + 1) / 2;
  const size_t nout = 1 + K + (size_t)K * d + (size_t)K * P;
  const size_t wsb = gmm_workspace_bytes(d, K, N);
  // one cached device arena per (thread, device), carved 256-byte aligned
  // (the counters piece also holds the restoration residual and verdict)
  const size_t sizes[8] = {(size_t)K * 8, (size_t)K * d * 8, (size_t)K * P * 8,
                           (size_t)N * d * 8, nout * 8, (size_t)std::max<int64_t>(N, 1), wsb, 32};
  size_t total = 0;
  for (size_t b : sizes) total += (b + 255) & ~size_t(255);
  void *base = nullptr;
  if ((rc = Pipeline::arena(device, total, &base))) return rc;
  struct Piece { void *p; } da, dm, di, dx, dout, dfl, dws, dc;
  Piece *pieces[8] = {&da, &dm, &di, &dx, &dout, &dfl, &dws, &dc};
  size_t off = 0;
  for (int q = 0; q < 8; q++) {
    pieces[q]->p = (char *)base + off;
    off += (sizes[q] + 255) & ~size_t(255);
  }
  if ((rc = cuda_status(cudaMemcpyAsync(da.p, alphas, K * 8, cudaMemcpyHostToDevice, st), "H2D")) ||
      (rc = cuda_status(cudaMemcpyAsync(dm.p, means, (size_t)K * d * 8, cudaMemcpyHostToDevice, st),
                        "H2D")) ||
      (rc = cuda_status(cudaMemcpyAsync(di.p, icf, (size_t)K * P * 8, cudaMemcpyHostToDevice, st),
                        "H2D")) ||
      (rc = cuda_status(cudaMemcpyAsync(dx.p, x, (size_t)N * d * 8, cudaMemcpyHostToDevice, st),
                        "H2D")) ||
      (rc = cuda_status(cudaMemsetAsync(dc.p, 0, 32, st), "memset")))
    return rc;
  unsigned long long *dcnt = (unsigned long long *)dc.p;
  const GmmSeq seq{err0, (double *)(dcnt + 2), (int *)(dcnt + 3), nullptr, 0, 1};
  if ((rc = launch_gmm(d, K, N, N_total, (double *)da.p, (double *)dm.p, (double *)di.p,
                       (double *)dx.p, gamma, m, cst, tol, invcheck, add_param, (double *)dout.p,
                       (uint8_t *)dfl.p, dcnt, dws.p, wsb, st, 1, restore ? &seq : nullptr)))
    return rc;
  unsigned long long h[4];
  if ((rc = cuda_status(cudaMemcpyAsync(out, dout.p, nout * 8, cudaMemcpyDeviceToHost, st),
                        "D2H out")) ||
      (rc = cuda_status(cudaMemcpyAsync(h, dc.p, 32, cudaMemcpyDeviceToHost, st), "D2H counters")))
    return rc;
  if ((rc = pl.finish())) return rc;
  if (n_failed) *n_failed = h[1];
  if (!restore) return RL_OK;
  double r;
  int code;
  memcpy(&r, &h[2], 8);
  memcpy(&code, &h[3], 4);
  if (resid) *resid = r;
  return h[1] ? RL_OK : code;   // per-point errors take precedence (fail flags)
}

int rl_gmm_grad_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                         const double *means, const double *icf, const double *x, double gamma,
                         int32_t m, double cst, double tol, int32_t invcheck, double *out,
                         unsigned long long *n_failed, int32_t device) {
  return gmm_grad_host(d, K, N, N, 1, alphas, means, icf, x, gamma, m, cst, tol, invcheck, out,
                       n_failed, device, false, 0.0, nullptr);
}

int rl_gmm_grad_shard_f64_host(int32_t d, int32_t K, int64_t N, int64_t N_total,
                               const double *alphas, const double *means, const double *icf,
                               const double *x, double gamma, int32_t m, double cst, double tol,
                               int32_t invcheck, int32_t add_param_terms, double *out,
                               unsigned long long *n_failed, int32_t device) {
  return gmm_grad_host(d, K, N, N_total, add_param_terms ? 1 : 0, alphas, means, icf, x, gamma, m,
                       cst, tol, invcheck, out, n_failed, device, false, 0.0, nullptr);
}

int rl_gmm_gradient_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                             const double *means, const double *icf, const double *x,
                             double gamma, int32_t m, double cst, double err0, double tol,
                             int32_t invcheck, double *out, double *resid,
                             unsigned long long *n_failed, int32_t device) {
  return gmm_grad_host(d, K, N, N, 1, alphas, means, icf, x, gamma, m, cst, tol, invcheck, out,
                       n_failed, device, true, err0, resid);
}

int rl_gmm_run_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                        const double *means, const double *icf, const double *x, double gamma,
                        int32_t m, double cst, double err0, double tol, int32_t invcheck,
                        int32_t direction, double *err, unsigned long long *n_failed,
                        unsigned long long *argmax_steps, int32_t device) {
  if (d <= 0 || K <= 0 || N < 0 || !alphas || !means || !icf || (N > 0 && !x) || !err ||
      (direction != 1 && direction != -1))
    return set_error(RL_ERR_INVALID, "rl_gmm_run_f64_host: bad argument");
  Pipeline pl;
  int rc = pl.init(device);
  if (rc) return rc;
  cudaStream_t st = pl.st[0];
  const size_t P = (size_t)d * (d + 1) / 2;
  const size_t wsb = gmm_workspace_bytes(d, K, N);
  const size_t sizes[8] = {(size_t)K * 8, (size_t)K * d * 8, (size_t)K * P * 8,
                           (size_t)N * d * 8, 8, (size_t)std::max<int64_t>(N, 1), wsb, 16};
  size_t total = 0;
  for (size_t b : sizes) total += (b + 255) & ~size_t(255);
  void *base = nullptr;
  if ((rc = Pipeline::arena(device, total, &base))) return rc;
  char *q[8];
  size_t off = 0;
  for (int i = 0; i < 8; i++) {
    q[i] = (char *)base + off;
    off += (sizes[i] + 255) & ~size_t(255);
  }
  const void *src[4] = {alphas, means, icf, x};
  for (int i = 0; i < 4; i++)
    if (sizes[i] && (rc = cuda_status(cudaMemcpyAsync(q[i], src[i], sizes[i],
                                                      cudaMemcpyHostToDevice, st), "H2D")))
      return rc;
  if ((rc = cuda_status(cudaMemsetAsync(q[7], 0, 16, st), "memset"))) return rc;
  const GmmSeq seq{err0, nullptr, nullptr, nullptr, 0, direction};
  if ((rc = launch_gmm(d, K, N, N, (double *)q[0], (double *)q[1], (double *)q[2],
                       (double *)q[3], gamma, m, cst, tol, invcheck, 1, (double *)q[4],
                       (uint8_t *)q[5], (unsigned long long *)q[7], q[6], wsb, st, 0, &seq)))
    return rc;
  unsigned long long h[2];
  if ((rc = cuda_status(cudaMemcpyAsync(err, q[4], 8, cudaMemcpyDeviceToHost, st), "D2H err")) ||
      (rc = cuda_status(cudaMemcpyAsync(h, q[7], 16, cudaMemcpyDeviceToHost, st), "D2H counters")))
    return rc;
  if ((rc = pl.finish())) return rc;
  if (n_failed) *n_failed = h[1];
  if (argmax_steps) *argmax_steps = h[0];
  return RL_OK;
}

}  // extern "C"
