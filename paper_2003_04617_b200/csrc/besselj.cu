// besselj.cu — batched reversible gradient of J_nu(z) (programs/besselj.rnl).
//
// Replaces, for every element, reference `gradient(p, GradRequest("besselj",
// [0.0, nu, z]))` (autodiff.py:136-180), i.e. four interpreter sweeps over
// the series loop, with ONE fused pass per element held in registers:
//
//   sweep 1   forward routine R          (log-domain term s, alternating acc)
//             J = 0.0 + acc
//   sweep 4   ~R with the adjoint rules   (s walked back down to k = 0:
//                                          uncompute + cotangents, no tape)
//
// Sweeps 2 (forward ~R) and 3 (gradient-mode R) are elided: the reference
// re-executes bit-identical primal arithmetic in them (ancillas restart from
// their exact declared values, arguments are never written, and in sweep 3
// every accumulated cotangent is zero), so sweep 4 performs exactly the
// same checks sweep 2 would (this is the "dead uncompute" elision the paper
// allows).  All reversibility checks of the reference are
// evaluated on device, in the reference's order, into a per-element flag:
//   loop entry/iteration postconditions  interpreter.py:772-797
//   ancilla releases |v - decl| <= tol    interpreter.py:717-748, 365-395
//   domain/overflow of log/exp            values.py:343-372
//
// Arithmetic is the reference's operation sequence (this file is compiled
// with -fmad=false: no contraction, IEEE add/mul/div), so the only
// differences to the CPU oracle are the device exp()/log(z) (<= 1 ulp).
// Integer logs log(k), log(k + nu) come from a host-computed table.
//
// Scheduling (v1): one element per thread, grid-stride; the series loop of a
// warp runs to the warp's longest trip count, and the reverse loop is
// aligned on the same warp-uniform k so the log table is a broadcast read.
#include <math.h>

#include "common.cuh"

namespace rl {

__constant__ double c_logtab[LOGTAB_N];
constexpr double LN2 = 0.6931471805599453;  // == math.log(2) (host libm), bit for bit

__device__ __forceinline__ double logi(int i) {
  return i < LOGTAB_N ? c_logtab[i] : log((double)i);
}

__device__ __forceinline__ bool exp_overflowed(double t, double x) {
  return isinf(t) && isfinite(x);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_besselj_grad(
    int nu, const double *__restrict__ zin, long long n, double thr, double tol, double seed,
    long long max_trips, int chk, double *__restrict__ Jout, double *__restrict__ dzout,
    uint8_t *__restrict__ fail, unsigned long long *counters) {
  const int lane = threadIdx.x & 31;
  unsigned long long trips_sum = 0, nfail = 0;
  const long long stride = (long long)gridDim.x * BLOCK;
  for (long long base = (long long)blockIdx.x * BLOCK + (threadIdx.x & ~31); base < n;
       base += stride) {
    const long long i = base + lane;
    const bool valid = i < n;
    const double z = valid ? __ldg(zin + i) : 1.0;
    int code = 0;

    // ---------------- sweep 1: forward routine ----------------
    if (!(z > 0.0)) code = RL_ERR_DOMAIN;               // lz *= convert(z)
    const double logz = code ? 0.0 : log(z);
    double lz = 0.0 + logz;
    double halfz = 0.0 + lz;                             // halfz *= lz
    halfz = halfz - LN2;                                 // halfz /= 2
    double h2 = 0.0 + halfz;                             // halfz2 *= halfz (x2)
    h2 = h2 + halfz;
    double s = 0.0;
    for (int q = 1; q <= nu; q++) {                      // for i = 1:1:nu
      s = s + halfz;
      s = s - logi(q);
    }
    double t = exp(s);                                   // acc += convert(s)
    if (!code && exp_overflowed(t, s)) code = RL_ERR_OVERFLOW;
    double acc = 0.0 + t;
    int T = 0;
    bool go = valid && !code && (t > thr);               // while (s > thr, k != 0)
    int kk = 0;                                          // warp-uniform k
    while (__any_sync(FULL_MASK, go)) {
      kk++;
      if (go) {
        if (T >= max_trips) {
          code = RL_ERR_FUEL;
          go = false;
        } else {
          T++;
          const int kn = kk + nu;
          s = s + h2;                                    // s *= halfz2
          s = s - logi(kk);                              // s /= k
          if (kn <= 0) {                                 // s /= kn
            code = RL_ERR_DOMAIN;
            go = false;
          } else {
            s = s - logi(kn);
            t = exp(s);
            if (exp_overflowed(t, s)) {
              code = RL_ERR_OVERFLOW;
              go = false;
            } else {
              acc = (kk & 1) ? acc - t : acc + t;        // if (k % 2 == 0, ~)
              go = t > thr;
            }
          }
        }
      }
    }
    const double Jv = 0.0 + acc;                         // out! += acc
    const bool fwd_ok = valid && !code;

    // ---------------- sweep 4: ~routine with adjoints ----------------
    const double accg = 0.0 + (1.0 * seed) * 1.0;        // out! -= acc: acc.g += out.g
    double sg = 0.0, h2g = 0.0, hzg = 0.0, lzg = 0.0, zg = 0.0;
    if (fwd_ok && chk && t > thr) code = RL_ERR_POSTCONDITION;  // entry: post false
    const int Tmax = __reduce_max_sync(FULL_MASK, fwd_ok ? T : 0);
    for (int k = Tmax; k >= 1; k--) {                    // aligned: k warp-uniform
      if (fwd_ok && k <= T) {
        if (k & 1) {                                     // inverse if
          acc = acc + t;
          sg = sg + (-1.0 * accg) * t;
        } else {
          acc = acc - t;
          sg = sg + (1.0 * accg) * t;
        }
        const int kn = k + nu;
        s = s + logi(kn);                                // s *= kn
        s = s + logi(k);                                 // s *= k
        s = s - h2;                                      // s /= halfz2
        h2g = h2g + 1.0 * sg;
        t = exp(s);
        if (!code && exp_overflowed(t, s)) code = RL_ERR_OVERFLOW;
        if (!code && chk && !(t > thr)) code = RL_ERR_POSTCONDITION;
      }
    }
    if (fwd_ok) {
      acc = acc - t;                                     // acc -= convert(s)
      sg = sg + (1.0 * accg) * t;
      for (int q = nu; q >= 1; q--) {                    // for i = nu:-1:1
        s = s + logi(q);
        s = s - halfz;
        hzg = hzg + 1.0 * sg;
      }
      h2 = h2 - halfz;                                   // halfz2 /= halfz (x2)
      hzg = hzg + 1.0 * h2g;
      h2 = h2 - halfz;
      hzg = hzg + 1.0 * h2g;
      halfz = halfz + LN2;                               // halfz *= 2
      halfz = halfz - lz;                                // halfz /= lz
      lzg = lzg + 1.0 * hzg;
      lz = lz - logz;                                    // lz /= convert(z)
      zg = zg + (1.0 * lzg) / z;
      if (chk && !code) {                                // releases
        if (fabs(acc - 0.0) > tol || fabs(s - 0.0) > tol || fabs(h2 - 0.0) > tol ||
            fabs(halfz - 0.0) > tol || fabs(lz - 0.0) > tol)
          code = RL_ERR_DIRTY_ANCILLA;
      }
    }
    if (valid) {
      Jout[i] = fwd_ok ? Jv : __longlong_as_double(0x7ff8000000000000ULL);
      dzout[i] = fwd_ok ? zg : __longlong_as_double(0x7ff8000000000000ULL);
      fail[i] = (uint8_t)code;
      trips_sum += (unsigned long long)T;
      nfail += code != 0;
    }
  }
  block_add_counters<BLOCK>(trips_sum, nfail, counters);
}

static int upload_logtab() {
  static double tab[LOGTAB_N];
  tab[0] = -INFINITY;
  for (int i = 1; i < LOGTAB_N; i++) tab[i] = log((double)i);
  return cuda_status(cudaMemcpyToSymbol(c_logtab, tab, sizeof tab), "upload log table");
}

int besselj_tables_init() { return upload_logtab(); }

constexpr int BJ_BLOCK = 256;

int launch_besselj(int32_t nu, const double *z, int64_t n, double thr, double tol, double seed,
                   int64_t max_trips, int32_t invcheck, double *J, double *dJdz, uint8_t *fail,
                   unsigned long long *counters, cudaStream_t st) {
  if (n < 0 || (n > 0 && (!z || !J || !dJdz || !fail)) || max_trips < 0)
    return set_error(RL_ERR_INVALID, "rl_besselj_grad_f64: bad argument");
  int rc = ensure_device_tables();
  if (rc) return rc;
  if (n == 0) return RL_OK;
  int blocks_per_sm = 0;
  rc = cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                       &blocks_per_sm, k_besselj_grad<BJ_BLOCK>, BJ_BLOCK, 0),
                   "occupancy");
  if (rc) return rc;
  long long want = (n + BJ_BLOCK - 1) / BJ_BLOCK;
  long long cap = (long long)sm_count() * blocks_per_sm;
  int grid = (int)(want < cap ? want : cap);
  k_besselj_grad<BJ_BLOCK><<<grid, BJ_BLOCK, 0, st>>>(nu, z, n, thr, tol, seed, max_trips,
                                                      invcheck ? 1 : 0, J, dJdz, fail, counters);
  return cuda_status(cudaGetLastError(), "k_besselj_grad launch");
}

}  // namespace rl
