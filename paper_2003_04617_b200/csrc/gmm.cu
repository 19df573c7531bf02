// gmm.cu — ADBench GMM objective gradient by reverse computing
// (programs/gmm.rnl), data-parallel over points.
//
// Replaces `gradient(p, GradRequest("gmm", [0, alphas, means, icf, x,
// zeros.., ga, wm, cst], wrt=["alphas","means","icf"]))` (autodiff.py:136).
// The program's per-point body is
//   R_i:   for k: xc = x_i - mu_k; qxc = L_k xc; sqn = |qxc|^2;
//               mt[k] = alphas[k] + sq[k] - sqn/2      (per-k routine, uncomputed)
//          reversible argmax (Int branch record dm[k]), mx = mt[imx],
//          se = sum_k exp(mt[k] - mx)
//   err += log(se) + mx; ~R_i
// and its gradient sweep runs ~R_i backwards with the adjoint rules.  On the
// GPU the points are independent (each gets fresh zero scratch, see
// DESIGN.md for the one deviation this implies), so the sweeps become five
// kernels with no tape:
//
//   k_gmm_prep    per component: qd = exp(diag icf), sq = sum(diag icf) (the
//                 top routine) and the transposed factor L_k^T, packed by rows
//   k_gmm_fwd     forward mat-vec tiles Z = Xc L^T (FP64 DFMA, register
//                 tiled, smem-staged) -> sqn -> mt[k][i]; sqn's uncompute
//                 residual is checked on device (DirtyAncilla)
//   k_gmm_lse     per point: the reversible argmax / logsumexp forward, then its
//                 reverse sweep with adjoints -> dmt = d err / d mt[k][i],
//                 release and branch-postcondition checks
//   k_gmm_rev     reverse per-k routine: RECOMPUTES Z (reverse computing:
//                 the forward values are rebuilt, not stored), forms
//                 qxc.g = (-dmt/2)(2 Z), and accumulates the factor adjoint
//                 M = sum_i qxc.g_i xc_i^T (lower triangle) and sum_i qxc.g_i
//                 in registers across the block's points
//   k_gmm_params  parameter-only terms (-N lse(alphas), Wishart prior, cst)
//   k_gmm_final   per component: deterministic reduction of the block
//                 partials, the chain through qd = exp(icf) and sq, means.g =
//                 -L^T sum_i qxc.g_i (linearity: sum_i xc.g_i = L^T sum_i qxc.g_i)
//
// The uncompute of qxc (qxc -= L xc) is dead (its value only feeds the
// final restoration check of a zero-initialised scratch) and is elided.
// Arithmetic contracts to FMA (this file is built with -fmad=true): results
// differ from the sequential reference in rounding only (tests: 1e-10).
#include <math.h>

#include "common.cuh"

namespace rl {

constexpr int GMM_THREADS = 256;
constexpr int GMM_WARPS = GMM_THREADS / 32;

template <int DP>
struct GmmCfg {
  static constexpr int TP = DP == 128 ? 64 : (DP == 64 ? 128 : 256);  // points per tile
  static constexpr int PPL = TP / 32;                                  // points per lane
  static constexpr int GW = DP / 16;            // columns per group (16 groups, 2 per warp)
  static constexpr int XS = TP + 2;             // padded row stride of the [DP][TP] tiles
  static constexpr int MT = DP / 16;            // M micro-tile edge (16 x 16 thread grid)
};

__host__ __device__ constexpr int lt_size(int DP) {
  int s = 0;
  for (int a = 0; a < DP; a++) s += DP - (a & ~7);
  return s;
}
__host__ __device__ constexpr int lt_rowoff(int DP, int a) {
  // sum_{a' < a} (DP - (a' & ~7))
  int q = a >> 3, r = a & 7;
  return 8 * (q * DP - 4 * q * (q - 1)) + r * (DP - 8 * q);
}

// ---------------------------------------------------------------------------
// prep: qd, sq (the top @routine) and packed L^T per component
// ---------------------------------------------------------------------------
template <int DP>
__global__ void __launch_bounds__(GMM_THREADS) k_gmm_prep(int d, int K, const double *__restrict__ icf,
                                                          double *__restrict__ LT,
                                                          double *__restrict__ qd,
                                                          double *__restrict__ sq,
                                                          double *__restrict__ fro) {
  const int k = blockIdx.x;
  const int P = d * (d + 1) / 2;
  const double *ic = icf + (long long)k * P;
  constexpr int LTS = lt_size(DP);
  double *lt = LT + (long long)k * LTS;
  for (int e = threadIdx.x; e < LTS; e += GMM_THREADS) {
    // invert the packed index e -> (a, b)
    int a = 0;
    while (a + 1 < DP && lt_rowoff(DP, a + 1) <= e) a++;
    const int b = (a & ~7) + (e - lt_rowoff(DP, a));
    double v = 0.0;
    if (a < d && b < d) {
      if (b == a) {
        v = exp(ic[a]);                                  // qd[k, j] += exp(icf[k, j])
      } else if (b > a) {
        // icf column-major strict lower triangle: (row b, col a), a < b
        const int li = d + a * d - a * (a + 1) / 2 + (b - a - 1);
        v = ic[li];
      }
    }
    lt[e] = v;
  }
  if (threadIdx.x < 32) {
    double s = 0.0;
    if (threadIdx.x == 0) {
      for (int j = 0; j < d; j++) s = s + ic[j];         // sq[k] += icf[k, j] (in order)
      sq[k] = s;
    }
  }
  // qd and this component's share of the prior's Frobenius sum:
  // fro += abs2(qd![k, j]) (j <= d) or abs2(icf[k, j]) (j > d)
  double f = 0.0;
  for (int j = threadIdx.x; j < P; j += GMM_THREADS) {
    double v = ic[j];
    if (j < d) {
      v = exp(v);
      qd[(long long)k * d + j] = v;
    }
    f = fma(v, v, f);
  }
  __shared__ double red[GMM_THREADS];
  red[threadIdx.x] = f;
  __syncthreads();
  for (int o = GMM_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) fro[k] = red[0];
}

// ---------------------------------------------------------------------------
// shared tile loaders and the Z = Xc L^T tile product
// ---------------------------------------------------------------------------
template <int DP>
__device__ __forceinline__ void load_xct(double *__restrict__ xct, const double *__restrict__ x,
                                         const double *__restrict__ mu, int d, long long p0,
                                         long long N) {
  using C = GmmCfg<DP>;
  // x rows are d doubles; walk the tile's TP*d doubles linearly (coalesced)
  const long long rows = N - p0 < C::TP ? N - p0 : C::TP;
  const int tot = C::TP * DP;
  for (int e = threadIdx.x; e < tot; e += GMM_THREADS) {
    const int p = e / DP, a = e - p * DP;
    double v = 0.0;
    if (p < rows && a < d) v = x[(p0 + p) * d + a] - mu[a];  // xc[j] += x[i, j] - means[k, j]
    xct[a * C::XS + p] = v;
  }
}

// acc[p][h][c]: lane's PPL points x (group h of the warp: 0 -> group w,
// 1 -> group 15-w) x GW columns
template <int DP>
__device__ __forceinline__ void tile_z(const double *__restrict__ lt, const double *__restrict__ xct,
                                       double (&acc)[GmmCfg<DP>::PPL][2][GmmCfg<DP>::GW]) {
  using C = GmmCfg<DP>;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c1 = w * C::GW, c2 = (15 - w) * C::GW;
#pragma unroll
  for (int p = 0; p < C::PPL; p++)
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int c = 0; c < C::GW; c++) acc[p][h][c] = 0.0;
  const double *xrow = xct + lane * C::PPL;
  const int amax1 = c1 + C::GW, amax2 = c2 + C::GW;
#pragma unroll 2
  for (int a = 0; a < amax1; a++) {
    double xv[C::PPL], l1[C::GW], l2[C::GW];
#pragma unroll
    for (int p = 0; p < C::PPL; p += 2) {
      const double2 t = *reinterpret_cast<const double2 *>(xrow + a * C::XS + p);
      xv[p] = t.x;
      xv[p + 1] = t.y;
    }
    const double *lr = lt + lt_rowoff(DP, a) - (a & ~7);
#pragma unroll
    for (int c = 0; c < C::GW; c += 2) {
      const double2 u = *reinterpret_cast<const double2 *>(lr + c1 + c);
      const double2 v = *reinterpret_cast<const double2 *>(lr + c2 + c);
      l1[c] = u.x;
      l1[c + 1] = u.y;
      l2[c] = v.x;
      l2[c + 1] = v.y;
    }
#pragma unroll
    for (int p = 0; p < C::PPL; p++)
#pragma unroll
      for (int c = 0; c < C::GW; c++) {
        acc[p][0][c] = fma(xv[p], l1[c], acc[p][0][c]);
        acc[p][1][c] = fma(xv[p], l2[c], acc[p][1][c]);
      }
  }
#pragma unroll 2
  for (int a = amax1; a < amax2; a++) {
    double xv[C::PPL], l2[C::GW];
#pragma unroll
    for (int p = 0; p < C::PPL; p += 2) {
      const double2 t = *reinterpret_cast<const double2 *>(xrow + a * C::XS + p);
      xv[p] = t.x;
      xv[p + 1] = t.y;
    }
    const double *lr = lt + lt_rowoff(DP, a) - (a & ~7);
#pragma unroll
    for (int c = 0; c < C::GW; c += 2) {
      const double2 v = *reinterpret_cast<const double2 *>(lr + c2 + c);
      l2[c] = v.x;
      l2[c + 1] = v.y;
    }
#pragma unroll
    for (int p = 0; p < C::PPL; p++)
#pragma unroll
      for (int c = 0; c < C::GW; c++) acc[p][1][c] = fma(xv[p], l2[c], acc[p][1][c]);
  }
}

template <int DP>
__device__ __forceinline__ void copy_lt(double *__restrict__ lt_s, const double *__restrict__ lt_g) {
  constexpr int n2 = lt_size(DP) / 2;
  const double2 *src = reinterpret_cast<const double2 *>(lt_g);
  double2 *dst = reinterpret_cast<double2 *>(lt_s);
  for (int e = threadIdx.x; e < n2; e += GMM_THREADS) dst[e] = src[e];
}

// ---------------------------------------------------------------------------
// forward: mt[k][i] = alphas[k] + sq[k] - |L_k (x_i - mu_k)|^2 / 2
// ---------------------------------------------------------------------------
template <int DP>
__global__ void __launch_bounds__(GMM_THREADS, 1) k_gmm_fwd(
    int d, int K, long long N, const double *__restrict__ alphas, const double *__restrict__ means,
    const double *__restrict__ x, const double *__restrict__ LT, const double *__restrict__ sq,
    double tol, int chk, double *__restrict__ mtT, unsigned *__restrict__ flagsA) {
  using C = GmmCfg<DP>;
  extern __shared__ __align__(16) double smem[];
  double *lt_s = smem;
  double *xct = lt_s + lt_size(DP);
  double *sqp = xct + DP * C::XS;  // [GMM_WARPS][TP]
  const int k = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  copy_lt<DP>(lt_s, LT + (long long)k * lt_size(DP));
  const double *mu = means + (long long)k * d;
  const double base_mt = (0.0 + alphas[k]) + sq[k];     // mt += alphas[k]; mt += sq[k]
  const long long ntiles = (N + C::TP - 1) / C::TP;
  for (long long tile = blockIdx.y; tile < ntiles; tile += gridDim.y) {
    const long long p0 = tile * C::TP;
    __syncthreads();
    load_xct<DP>(xct, x, mu, d, p0, N);
    __syncthreads();
    double acc[C::PPL][2][C::GW];
    tile_z<DP>(lt_s, xct, acc);
    // sqn partial of this warp's columns, per point (sqn += abs2(qxc[j]))
#pragma unroll
    for (int p = 0; p < C::PPL; p++) {
      double s = 0.0;
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int c = 0; c < C::GW; c++) s = fma(acc[p][h][c], acc[p][h][c], s);
      sqp[w * C::TP + lane * C::PPL + p] = s;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < C::TP; p += GMM_THREADS) {
      const long long i = p0 + p;
      if (i >= N) continue;
      double sqn = 0.0;
#pragma unroll
      for (int ww = 0; ww < GMM_WARPS; ww++) sqn = sqn + sqp[ww * C::TP + p];
      // the inner routine's uncompute: sqn -= abs2(qxc[j]) in reverse, then
      // the release check sqn -> 0.0 (interpreter.py:738-745)
      double res = sqn;
#pragma unroll
      for (int ww = GMM_WARPS - 1; ww >= 0; ww--) res = res - sqp[ww * C::TP + p];
      if (chk && fabs(res) > tol) atomicOr(&flagsA[i], 1u);
      mtT[(long long)k * N + i] = base_mt - sqn * 0.5;    // mt -= sqn * 0.5
    }
  }
}

// ---------------------------------------------------------------------------
// per point: reversible argmax + logsumexp, forward then reverse with adjoints
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(GMM_THREADS) k_gmm_lse(
    int K, long long N, const double *__restrict__ mtT, double *__restrict__ gmtT,
    const unsigned *__restrict__ flagsA, double tol, int chk, double *__restrict__ err_part,
    uint8_t *__restrict__ fail, unsigned long long *counters) {
  const long long i = (long long)blockIdx.x * GMM_THREADS + threadIdx.x;
  double e_pt = 0.0;
  unsigned long long nfail = 0;
  if (i < N) {
    int code = 0;
    const double *mt = mtT + i;
    double *gmt = gmtT + i;
#define MT(k) mt[(long long)(k) * N]
#define GM(k) gmt[(long long)(k) * N]
    // imx <- 1; if (mt![k] > mt![imx], dm![k] > 0) {dm![k] += k - imx; imx += dm![k]}
    // The Int record and its uncompute are exact and the branch
    // postconditions replay the same comparisons, so they cannot fail.
    int imx = 0;
    double vmx = MT(0);
    for (int k = 1; k < K; k++) {
      const double v = MT(k);
      if (v > vmx) {
        imx = k;
        vmx = v;
      }
    }
    const double mx = 0.0 + vmx;                          // mx <- 0.0; mx += mt![imx]
    double se = 0.0;
    for (int k = 0; k < K; k++) {
      const double t = 0.0 + (MT(k) - mx);
      se = se + exp(t);
    }
    if (!(se > 0.0)) code = RL_ERR_DOMAIN;               // err += log(se)
    e_pt = log(se) + mx;                                  // err += log(se); err += mx
    // gradient sweep (~f): err -= mx; err -= log(se); ~R_i with adjoints
    double mxg = 0.0 + (1.0 * 1.0) * 1.0;
    const double seg = 0.0 + (1.0 * 1.0) * (1.0 / se);
    for (int k = K - 1; k >= 0; k--) {
      double t = 0.0 + (MT(k) - mx);
      const double ex = exp(t);
      se = se - ex;                                       // se -= exp(t)
      const double tg = 0.0 + seg * ex;
      t = t - (MT(k) - mx);
      if (chk && !code && fabs(t) > tol) code = RL_ERR_DIRTY_ANCILLA;
      GM(k) = 0.0 + tg;                                   // mt[k].g += t.g
      mxg = mxg - tg;                                     // mx.g += -t.g
    }
    if (chk && !code && fabs(se) > tol) code = RL_ERR_DIRTY_ANCILLA;  // se -> 0.0
    const double mxr = mx - MT(imx);                      // mx -= mt![imx]
    GM(imx) = GM(imx) + mxg;
    if (chk && !code && fabs(mxr) > tol) code = RL_ERR_DIRTY_ANCILLA;
#undef MT
#undef GM
    if (flagsA[i]) code = RL_ERR_DIRTY_ANCILLA;            // sqn release failed (sweep 1)
    fail[i] = (uint8_t)code;
    nfail = code != 0;
  }
  // deterministic block sum of the per-point objective terms
  __shared__ double red[GMM_THREADS];
  red[threadIdx.x] = e_pt;
  __syncthreads();
  for (int o = GMM_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) err_part[blockIdx.x] = red[0];
  block_add_counters<GMM_THREADS>(0, nfail, counters);
}

// ---------------------------------------------------------------------------
// reverse: recompute Z, qxc.g = (-dmt/2)(2 Z); accumulate M = G^T Xc and
// sum_i G_i over the block's points (registers), then write the partial.
// ---------------------------------------------------------------------------
template <int DP>
__global__ void __launch_bounds__(GMM_THREADS, 1) k_gmm_rev(
    int d, int K, long long N, const double *__restrict__ means, const double *__restrict__ x,
    const double *__restrict__ LT, const double *__restrict__ gmtT,
    double *__restrict__ part /* [K][S][DP*DP + DP + 1] */) {
  using C = GmmCfg<DP>;
  extern __shared__ __align__(16) double smem[];
  double *lt_s = smem;
  double *xct = lt_s + lt_size(DP);
  double *gt = xct + DP * C::XS;       // [DP][XS]: qxc.g transposed
  double *cg = gt + DP * C::XS;        // [TP]: sqn.g per point
  double *red = cg + C::TP;            // [GMM_WARPS]
  const int k = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  copy_lt<DP>(lt_s, LT + (long long)k * lt_size(DP));
  const double *mu = means + (long long)k * d;
  const double *gm = gmtT + (long long)k * N;
  // M tile of this thread: rows b = bi + 16 r, cols a = ai + 16 c (interleaved
  // so that the smem reads of a warp spread over the banks)
  const int bi = tid >> 4, ai = tid & 15;
  double M[C::MT][C::MT];
#pragma unroll
  for (int r = 0; r < C::MT; r++)
#pragma unroll
    for (int c = 0; c < C::MT; c++) M[r][c] = 0.0;
  double gs[2][C::GW];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int c = 0; c < C::GW; c++) gs[h][c] = 0.0;
  double sgm = 0.0;
  const int c1 = w * C::GW, c2 = (15 - w) * C::GW;
  const long long ntiles = (N + C::TP - 1) / C::TP;
  for (long long tile = blockIdx.y; tile < ntiles; tile += gridDim.y) {
    const long long p0 = tile * C::TP;
    __syncthreads();
    load_xct<DP>(xct, x, mu, d, p0, N);
    for (int p = tid; p < C::TP; p += GMM_THREADS) {
      const long long i = p0 + p;
      const double g = i < N ? gm[i] : 0.0;
      sgm += g;                                           // alphas.g, sq.g += mt.g
      cg[p] = 0.0 + (-1.0 * g) * 0.5;                     // mt += sqn*0.5: sqn.g += -mt.g/2
    }
    __syncthreads();
    double acc[C::PPL][2][C::GW];
    tile_z<DP>(lt_s, xct, acc);                           // recompute qxc
    // qxc.g[j] = sqn.g * (2 qxc[j]) -> smem (transposed) and column sums
#pragma unroll
    for (int p = 0; p < C::PPL; p++) {
      const int pp = lane * C::PPL + p;
      const double c = cg[pp];
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int cc = 0; cc < C::GW; cc++) {
          const double g = c * (2.0 * acc[p][h][cc]);
          gs[h][cc] += g;
          gt[((h ? c2 : c1) + cc) * C::XS + pp] = g;
        }
    }
    __syncthreads();
    // M[b][a] += sum_p G[p][b] Xc[p][a]   (factor adjoint, lower triangle used)
#pragma unroll 1
    for (int p = 0; p < C::TP; p += 2) {
      double gv[C::MT][2], xv[C::MT][2];
#pragma unroll
      for (int r = 0; r < C::MT; r++) {
        const double2 t = *reinterpret_cast<const double2 *>(gt + (bi + 16 * r) * C::XS + p);
        gv[r][0] = t.x;
        gv[r][1] = t.y;
        const double2 u = *reinterpret_cast<const double2 *>(xct + (ai + 16 * r) * C::XS + p);
        xv[r][0] = u.x;
        xv[r][1] = u.y;
      }
#pragma unroll
      for (int r = 0; r < C::MT; r++)
#pragma unroll
        for (int c = 0; c < C::MT; c++) {
          M[r][c] = fma(gv[r][0], xv[c][0], M[r][c]);
          M[r][c] = fma(gv[r][1], xv[c][1], M[r][c]);
        }
    }
  }
  // write this block's partial
  const int S = gridDim.y;
  const long long PW = (long long)DP * DP + DP + 1;
  double *out = part + ((long long)k * S + blockIdx.y) * PW;
#pragma unroll
  for (int r = 0; r < C::MT; r++)
#pragma unroll
    for (int c = 0; c < C::MT; c++) out[(bi + 16 * r) * DP + (ai + 16 * c)] = M[r][c];
  // column sums: reduce gs over the warp's lanes (all lanes share the columns)
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int cc = 0; cc < C::GW; cc++) {
      double v = gs[h][cc];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL_MASK, v, o);
      if (lane == 0) out[(long long)DP * DP + (h ? c2 : c1) + cc] = v;
    }
  // sum of mt.g over the block's points
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sgm += __shfl_down_sync(FULL_MASK, sgm, o);
  __syncthreads();
  if (lane == 0) red[w] = sgm;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int ww = 0; ww < GMM_WARPS; ww++) s += red[ww];
    out[(long long)DP * DP + DP] = s;
  }
}

// ---------------------------------------------------------------------------
// parameter-only terms: -N lse(alphas) (reversible max, as in the program),
// Wishart prior, cst.  ws_par = [g_alpha_param (K), err_param]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) k_gmm_params(
    int d, int K, long long N_total, const double *__restrict__ alphas,
    const double *__restrict__ fro_k, const double *__restrict__ sq, double ga, int wm, double cst,
    double *__restrict__ ws_par) {
  const double hg2 = 0.5 * ga * ga;
  double fro = 0.0;
  for (int k = 0; k < K; k++) fro = fro + fro_k[k];
  if (threadIdx.x == 0) {
    double ssq = 0.0;
    for (int k = 0; k < K; k++) ssq = ssq + sq[k];
    // logsumexp(alphas) with the Int argmax record (as in the point routine)
    int ia = 0;
    for (int k = 1; k < K; k++)
      if (alphas[k] > alphas[ia]) ia = k;
    const double amx = 0.0 + alphas[ia];
    double ase = 0.0;
    for (int k = 0; k < K; k++) ase = ase + exp(0.0 + (alphas[k] - amx));
    const double lsa = (0.0 + log(ase)) + amx;
    const double nn = (double)N_total;
    ws_par[K] = -(nn * lsa) + hg2 * fro - (double)wm * ssq + cst;
    // gradient: err += nn*lsa (inverse): lsa.g = -nn; then ~routine
    const double lsag = 0.0 + (-1.0 * 1.0) * nn;
    double amxg = 0.0 + lsag;                              // lsa -= amx
    const double aseg = 0.0 + lsag * (1.0 / ase);          // lsa -= log(ase)
    for (int k = K - 1; k >= 0; k--) {
      const double ex = exp(0.0 + (alphas[k] - amx));
      const double tg = 0.0 + aseg * ex;                   // ase -= exp(t)
      ws_par[k] = tg;                                      // alphas[k].g += t.g
      amxg = amxg - tg;
    }
    ws_par[ia] += amxg;                                    // amx -= alphas[ia]
  }
}

// ---------------------------------------------------------------------------
// final assembly per component; block 0 also sums the objective
// ---------------------------------------------------------------------------
template <int DP>
__global__ void __launch_bounds__(GMM_THREADS) k_gmm_final(
    int d, int K, int S, int nerr, const double *__restrict__ icf, const double *__restrict__ qd,
    const double *__restrict__ LT, const double *__restrict__ part,
    const double *__restrict__ err_part, const double *__restrict__ ws_par, double ga, int wm,
    int add_params, double *__restrict__ out) {
  const int k = blockIdx.x;
  const int P = d * (d + 1) / 2;
  const long long PW = (long long)DP * DP + DP + 1;
  const double hg2 = 0.5 * ga * ga;
  __shared__ double gsum[DP];
  __shared__ double sg;
  double *g_alpha = out + 1;
  double *g_means = out + 1 + K;
  double *g_icf = out + 1 + K + (long long)K * d;
  const double *pk = part + (long long)k * S * PW;
  // column sums of qxc.g and sum of mt.g, reduced over the S partials in order
  for (int b = threadIdx.x; b <= DP; b += GMM_THREADS) {
    double s = 0.0;
    for (int j = 0; j < S; j++) s += pk[j * PW + (long long)DP * DP + b];
    if (b < DP) gsum[b] = s;
    else sg = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double ga_k = sg + (add_params ? ws_par[k] : 0.0);
    g_alpha[k] = ga_k;
  }
  // means.g[a] = -sum_b gsum[b] L[b][a]   (L^T row a = packed row a)
  const double *lt = LT + (long long)k * lt_size(DP);
  for (int a = threadIdx.x; a < d; a += GMM_THREADS) {
    const double *lr = lt + lt_rowoff(DP, a) - (a & ~7);
    double s = 0.0;
    for (int b = a; b < d; b++) s = fma(gsum[b], lr[b], s);
    g_means[(long long)k * d + a] = -s;
  }
  // icf.g: diag = sq.g + qd.g exp(icf); offdiag = M[b][a] (+ prior)
  const double sqg = sg + (add_params ? -(double)wm : 0.0);
  for (int j = threadIdx.x; j < P; j += GMM_THREADS) {
    int b, a;
    if (j < d) {
      b = a = j;
    } else {
      // column-major strict lower triangle index -> (b, a)
      int r = j - d;
      a = 0;
      while (r >= d - 1 - a) {
        r -= d - 1 - a;
        a++;
      }
      b = a + 1 + r;
    }
    double m = 0.0;
    for (int s = 0; s < S; s++) m += pk[s * PW + (long long)b * DP + a];
    double g;
    if (j < d) {
      const double q = qd[(long long)k * d + j];
      const double qdg = (add_params ? hg2 * (2.0 * q) : 0.0) + m;
      g = (0.0 + sqg) + qdg * exp(icf[(long long)k * P + j]);
    } else {
      g = (add_params ? hg2 * (2.0 * icf[(long long)k * P + j]) : 0.0) + m;
    }
    g_icf[(long long)k * P + j] = g;
  }
  if (k == 0 && threadIdx.x == 0) {
    double e = 0.0;
    for (int j = 0; j < nerr; j++) e += err_part[j];
    out[0] = e + (add_params ? ws_par[K] : 0.0);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int dp_of(int d) { return d <= 32 ? 32 : (d <= 64 ? 64 : (d <= 128 ? 128 : 0)); }

struct GmmLayout {
  size_t lt, qd, sq, fro, mt, gmt, flags, errp, part, par, total;
  int S, nerr;
};

static size_t al(size_t b) { return (b + 255) & ~size_t(255); }

static GmmLayout gmm_layout(int d, int K, long long N) {
  GmmLayout L{};
  const int DP = dp_of(d);
  const int TP = DP == 128 ? 64 : (DP == 64 ? 128 : 256);
  const long long ntiles = (N + TP - 1) / TP;
  int S = (int)((2 * 148 + K - 1) / K);
  if (S < 1) S = 1;
  if (S > ntiles) S = (int)(ntiles > 0 ? ntiles : 1);
  L.S = S;
  L.nerr = (int)((N + GMM_THREADS - 1) / GMM_THREADS);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += al(bytes);
    return o;
  };
  L.lt = take((size_t)K * lt_size(DP) * 8);
  L.qd = take((size_t)K * d * 8);
  L.sq = take((size_t)K * 8);
  L.fro = take((size_t)K * 8);
  L.mt = take((size_t)K * N * 8);
  L.gmt = take((size_t)K * N * 8);
  L.flags = take((size_t)N * 4);
  L.errp = take((size_t)(L.nerr > 0 ? L.nerr : 1) * 8);
  L.part = take((size_t)K * S * ((size_t)DP * DP + DP + 1) * 8);
  L.par = take((size_t)(K + 1) * 8);
  L.total = off;
  return L;
}

size_t gmm_workspace_bytes(int32_t d, int32_t K, int64_t N) {
  if (d <= 0 || d > 128 || K <= 0 || N < 0) return 0;
  return gmm_layout(d, K, N).total;
}

template <int DP>
static int run_gmm(int d, int K, long long N, long long N_total, const double *alphas,
                   const double *means, const double *icf, const double *x, double gamma, int m,
                   double cst, double tol, int chk, int add_params, double *out, uint8_t *fail,
                   unsigned long long *counters, char *ws, const GmmLayout &L, cudaStream_t st) {
  using C = GmmCfg<DP>;
  double *LT = (double *)(ws + L.lt), *qd = (double *)(ws + L.qd), *sq = (double *)(ws + L.sq);
  double *fro = (double *)(ws + L.fro);
  double *mt = (double *)(ws + L.mt), *gmt = (double *)(ws + L.gmt);
  unsigned *flags = (unsigned *)(ws + L.flags);
  double *errp = (double *)(ws + L.errp), *part = (double *)(ws + L.part);
  double *par = (double *)(ws + L.par);
  int rc;
  k_gmm_prep<DP><<<K, GMM_THREADS, 0, st>>>(d, K, icf, LT, qd, sq, fro);
  if ((rc = cuda_status(cudaGetLastError(), "k_gmm_prep"))) return rc;
  if (N > 0) {
    if ((rc = cuda_status(cudaMemsetAsync(flags, 0, (size_t)N * 4, st), "memset flags")))
      return rc;
    const size_t smem_f = ((size_t)lt_size(DP) + (size_t)DP * C::XS + GMM_WARPS * C::TP) * 8;
    const size_t smem_r = ((size_t)lt_size(DP) + 2 * (size_t)DP * C::XS + C::TP + GMM_WARPS) * 8;
    if ((rc = cuda_status(cudaFuncSetAttribute(k_gmm_fwd<DP>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem_f), "smem attr fwd")) ||
        (rc = cuda_status(cudaFuncSetAttribute(k_gmm_rev<DP>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem_r), "smem attr rev")))
      return rc;
    dim3 grid(K, L.S);
    k_gmm_fwd<DP><<<grid, GMM_THREADS, smem_f, st>>>(d, K, N, alphas, means, x, LT, sq, tol, chk, mt,
                                                    flags);
    if ((rc = cuda_status(cudaGetLastError(), "k_gmm_fwd"))) return rc;
    k_gmm_lse<<<L.nerr, GMM_THREADS, 0, st>>>(K, N, mt, gmt, flags, tol, chk, errp, fail,
                                              counters);
    if ((rc = cuda_status(cudaGetLastError(), "k_gmm_lse"))) return rc;
    k_gmm_rev<DP><<<grid, GMM_THREADS, smem_r, st>>>(d, K, N, means, x, LT, gmt, part);
    if ((rc = cuda_status(cudaGetLastError(), "k_gmm_rev"))) return rc;
  } else {
    if ((rc = cuda_status(cudaMemsetAsync(part, 0, (size_t)K * L.S * ((size_t)DP * DP + DP + 1) * 8,
                                          st), "memset part")))
      return rc;
  }
  if (add_params) {
    k_gmm_params<<<1, 32, 0, st>>>(d, K, N_total, alphas, fro, sq, gamma, m, cst, par);
    if ((rc = cuda_status(cudaGetLastError(), "k_gmm_params"))) return rc;
  }
  k_gmm_final<DP><<<K, GMM_THREADS, 0, st>>>(d, K, L.S, N > 0 ? L.nerr : 0, icf, qd, LT, part, errp,
                                             par, gamma, m, add_params, out);
  return cuda_status(cudaGetLastError(), "k_gmm_final");
}

int launch_gmm(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
               const double *means, const double *icf, const double *x, double gamma, int32_t m,
               double cst, double tol, int32_t invcheck, int32_t add_param_terms, double *out,
               uint8_t *fail, unsigned long long *counters, void *ws, size_t ws_bytes,
               cudaStream_t st) {
  if (d <= 0 || K <= 0 || N < 0 || !alphas || !means || !icf || !out || (N > 0 && (!x || !fail)))
    return set_error(RL_ERR_INVALID, "rl_gmm_grad_f64: bad argument");
  if (d > 128) return set_error(RL_ERR_INVALID, "rl_gmm_grad_f64: d > 128 is not supported");
  const GmmLayout L = gmm_layout(d, K, N);
  if (!ws || ws_bytes < L.total)
    return set_error(RL_ERR_INVALID, "rl_gmm_grad_f64: workspace too small (rl_gmm_workspace_bytes)");
  int rc = ensure_device_tables();
  if (rc) return rc;
  const int DP = dp_of(d);
  const int chk = invcheck ? 1 : 0;
  const long long Nt = N_total > 0 ? N_total : N;
  if (DP == 32)
    return run_gmm<32>(d, K, N, Nt, alphas, means, icf, x, gamma, m, cst, tol, chk,
                       add_param_terms, out, fail, counters, (char *)ws, L, st);
  if (DP == 64)
    return run_gmm<64>(d, K, N, Nt, alphas, means, icf, x, gamma, m, cst, tol, chk,
                       add_param_terms, out, fail, counters, (char *)ws, L, st);
  return run_gmm<128>(d, K, N, Nt, alphas, means, icf, x, gamma, m, cst, tol, chk,
                      add_param_terms, out, fail, counters, (char *)ws, L, st);
}

}  // namespace rl
