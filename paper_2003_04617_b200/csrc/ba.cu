// ba.cu — ADBench bundle-adjustment Jacobian by reverse computing
// (programs/ba.rnl: ba_proj + rodrigues + ba_weight).
//
// Replaces, per observation, the reference's two seeded
// `gradient(p, GradRequest("ba_proj", ..., seeds=[e1!|e2!], wrt=[cam, X, w]))`
// calls plus `gradient(p, GradRequest("ba_weight", [0.0, w]))`
// (autodiff.py:136-180) with ONE thread that runs
//
//   sweep 1  the routine R of ba_proj forward (rodrigues inlined), e = w * d
//   sweep 4  ~R with the adjoint rules for BOTH seeds at once: the primal
//            uncompute is seed-independent, so the two gradient passes of
//            the reference share it and carry two cotangent lanes (a = e1!,
//            b = e2!).  Each lane's accumulation order is the reference's,
//            so lane a / lane b equal the two separate passes bit for bit.
//
// Sweeps 2 and 3 are elided (bit-identical primal recomputation, zero
// cotangents; see besselj.cu).  rodrigues' own uncompute, which the
// reference runs inside sweep 1's call (and again inside the uncall of
// sweep 4), is executed once, in sweep 4; its release checks are reported
// with sweep-1 priority so the first failing check is the reference's.
// Compiled with -fmad=false: every add/mul/div/sqrt is the reference's IEEE
// operation; sin/cos are the only (<= 1-2 ulp) differences to the oracle.
//
// Memory: gathers cams[c] (88 B) and X[p] (24 B) through the read-only path
// (cameras and points are re-read by many observations and stay in L2),
// streams obs/w/feats coalesced, and stages the 31-double Jacobian rows of a
// block in shared memory so that the dominant stream — 248 B of J per
// observation — is written with coalesced 16-byte stores.
#include <math.h>

#include "common.cuh"

namespace rl {

struct G2 {
  double a, b;
};

// g += (sign * gy) * p for both lanes (numerics.py:419-486); compiled out in
// the residual-only (run) instantiation
#define GACC(g, sg, p)                  \
  do {                                  \
    if (GRAD) {                         \
      const double _p = (p);            \
      (g).a = (g).a + (sg).a * _p;      \
      (g).b = (g).b + (sg).b * _p;      \
    }                                   \
  } while (0)

__device__ __forceinline__ G2 neg(G2 g) { return G2{-g.a, -g.b}; }
__device__ __forceinline__ G2 zero2() { return G2{0.0, 0.0}; }

#ifndef BA_MINB
#define BA_MINB 10         // blocks per SM: up to 204 registers, no spills
#endif
#ifndef BA_BLOCK_SZ
#define BA_BLOCK_SZ 32     // one warp per block (measured best: tools/build_variants.sh sweep)
#endif
constexpr int BA_BLOCK = BA_BLOCK_SZ;
constexpr int BA_ROW = 31;
constexpr int BA_STAGE = 17;       // staged inputs per observation: cam 11, X 3, w, feat 2
constexpr int BA_SMEM = (BA_ROW + BA_STAGE) * BA_BLOCK * 8;   // dynamic smem per block
constexpr int BA_SMEM_CSR = BA_SMEM + (31 + 3) * BA_BLOCK * 4;  // + int32 cols / row pointers

// GRAD: the Jacobian (sweeps 1 + 4 with two cotangent lanes).  !GRAD: run
// of ba_proj / ba_weight on zero outputs — the residuals [e1, e2, 1 - w^2]
// with every check of the primal sweeps (the objective-only kernel).
//
// CSR: write the Jacobian as this shard's part of ADBench's BASparseMat
// (see BaCsr) instead of dense (p, 31) rows.
struct BaCsr {
  int32_t *rows;   // [2 p_l + p_l + 1] global row pointers (nullptr: values only)
  int32_t *cols;   // [31 p_l] global column indices   (nullptr: values only)
  double *vals;    // [31 p_l]
  long long off;   // global index of this shard's first observation
  long long P;     // global number of observations
  int col_pt;      // 11 n: first point column
  int col_w;       // 11 n + 3 m: first weight column
};

template <bool WANT_ERR, bool WANT_FEAT, bool GRAD = true, bool CSR = false>
__global__ void __launch_bounds__(BA_BLOCK, BA_MINB) k_ba_jac(
    int n_cams, int n_pts, long long n_obs, const double *__restrict__ cams,
    const double *__restrict__ Xs, const double *__restrict__ ws,
    const double *__restrict__ feats, const int2 *__restrict__ obs, double tol, int chk,
    double *__restrict__ err_out, double *__restrict__ J_out, double *__restrict__ Jf_out,
    uint8_t *__restrict__ fail, unsigned long long *counters, BaCsr csr) {
  // dynamic smem: the J row tile (31 doubles per observation), then the
  // per-thread input stage (17 doubles per observation, [17][BA_BLOCK])
  extern __shared__ __align__(16) double ba_dyn[];
  double *tile = ba_dyn;
  double *stage = ba_dyn + BA_BLOCK * BA_ROW;
  unsigned long long nfail = 0;
  const long long stride = (long long)gridDim.x * BA_BLOCK;
  const int tid = threadIdx.x;
  // Software pipeline: each thread gathers the camera row, point, weight and
  // feature of its NEXT observation (one block-stride ahead) into its own
  // stage slots with cp.async while it computes the current one, and holds
  // the observation index two strides ahead in a register.  The stage is
  // private per thread (no block barrier); the next gather is issued only
  // after every staged value of the current observation has been consumed.
  const unsigned st_s = (unsigned)__cvta_generic_to_shared(stage) + 8u * tid;
  auto cp8 = [&](int slot, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(st_s + 8u * BA_BLOCK * slot),
                 "l"(src) : "memory");
  };
  auto gather = [&](long long i, int2 o) {
    if (i < n_obs) {
      if (o.x >= 0 && o.x < n_cams && o.y >= 0 && o.y < n_pts) {
        const double *cp = cams + 11 * (long long)o.x;
#pragma unroll
        for (int j = 0; j < 11; j++) cp8(j, cp + j);
        const double *xp = Xs + 3 * (long long)o.y;
        cp8(11, xp);
        cp8(12, xp + 1);
        cp8(13, xp + 2);
      }
      cp8(14, ws + i);
      cp8(15, feats + 2 * i);
      cp8(16, feats + 2 * i + 1);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto sget = [&](int slot) { return stage[BA_BLOCK * slot + tid]; };
  const long long blk_first = (long long)blockIdx.x * BA_BLOCK;
  int2 o_cur = blk_first + tid < n_obs ? __ldg(obs + blk_first + tid) : make_int2(0, 0);
  gather(blk_first + tid, o_cur);
  int2 o_nxt = blk_first + stride + tid < n_obs ? __ldg(obs + blk_first + stride + tid)
                                                : make_int2(0, 0);
  for (long long blk0 = blk_first; blk0 < n_obs; blk0 += stride) {
    const long long i = blk0 + tid;
    const bool valid = i < n_obs;
    double row[BA_ROW];
    int code_final = 0;
    asm volatile("cp.async.wait_all;" ::: "memory");
    const int2 o = o_cur;
    const long long i_next = i + stride;
    auto prefetch_next = [&]() {
      gather(i_next, o_nxt);
      o_cur = o_nxt;
      o_nxt = i_next + stride < n_obs ? __ldg(obs + i_next + stride) : make_int2(0, 0);
    };
    const bool in_range = o.x >= 0 && o.x < n_cams && o.y >= 0 && o.y < n_pts;
    if (valid) {
      if (!in_range) {
        code_final = RL_ERR_INDEX;
        prefetch_next();
#pragma unroll
        for (int j = 0; j < BA_ROW; j++) row[j] = __longlong_as_double(0x7ff8000000000000ULL);
      } else {
        double c[11];
#pragma unroll
        for (int j = 0; j < 11; j++) c[j] = sget(j);
        const double X0 = sget(11), X1 = sget(12), X2 = sget(13);
        const double w = sget(14);
        const double f1 = sget(15), f2 = sget(16);
        int code1 = 0, code_rod = 0, code4 = 0;

        // ------------------------- sweep 1 -------------------------
        double x1 = 0.0 + (X0 - c[3]);
        double x2 = 0.0 + (X1 - c[4]);
        double x3 = 0.0 + (X2 - c[5]);
        double sqt = 0.0 + c[0] * c[0];
        sqt = sqt + c[1] * c[1];
        sqt = sqt + c[2] * c[2];
        double r1 = 0.0, r2 = 0.0, r3 = 0.0;
        const bool took = sqt != 0.0;
        // rodrigues' routine values (recomputed bit-identically in sweep 4)
        double th = 0, ct = 0, st = 0, ti = 0, w1 = 0, w2 = 0, w3 = 0, cc1 = 0, cc2 = 0, cc3 = 0,
               dt = 0, omc = 0, tmp = 0;
        // sqrt(sqt), sin/cos(th) and 1/th are evaluated once: the reference
        // re-evaluates them in its uncompute with the same arguments, i.e.
        // bit-identical values, so sweep 4 reuses them
        double sq_t = 0, s_th = 0, c_th = 0, inv_th = 0;
        if (took) {
          sq_t = sqrt(sqt);
          th = 0.0 + sq_t;
          sincos(th, &s_th, &c_th);
          inv_th = 1.0 / th;
          ct = 0.0 + c_th;
          st = 0.0 + s_th;
          ti = 0.0 + inv_th;
          w1 = 0.0 + c[0] * ti;
          w2 = 0.0 + c[1] * ti;
          w3 = 0.0 + c[2] * ti;
          cc1 = 0.0 + w2 * x3;
          cc1 = cc1 - w3 * x2;
          cc2 = 0.0 + w3 * x1;
          cc2 = cc2 - w1 * x3;
          cc3 = 0.0 + w1 * x2;
          cc3 = cc3 - w2 * x1;
          dt = 0.0 + w1 * x1;
          dt = dt + w2 * x2;
          dt = dt + w3 * x3;
          omc = 0.0 + (1.0 - ct);
          tmp = 0.0 + dt * omc;
          r1 = r1 + x1 * ct;
          r2 = r2 + x2 * ct;
          r3 = r3 + x3 * ct;
          r1 = r1 + cc1 * st;
          r2 = r2 + cc2 * st;
          r3 = r3 + cc3 * st;
          r1 = r1 + w1 * tmp;
          r2 = r2 + w2 * tmp;
          r3 = r3 + w3 * tmp;
        } else {
          r1 = r1 + x1;
          r2 = r2 + x2;
          r3 = r3 + x3;
          r1 = r1 + c[1] * x3;
          r1 = r1 - c[2] * x2;
          r2 = r2 + c[2] * x1;
          r2 = r2 - c[0] * x3;
          r3 = r3 + c[0] * x2;
          r3 = r3 - c[1] * x1;
        }
        if (r3 == 0.0) code1 = RL_ERR_DOMAIN;   // p1 += r1 / r3 (values.s_div)
        double p1 = 0.0 + r1 / r3;
        double p2 = 0.0 + r2 / r3;
        double rsq = 0.0 + p1 * p1;
        rsq = rsq + p2 * p2;
        double rsq2 = 0.0 + rsq * rsq;
        double lf = 1.0;
        lf = lf + c[9] * rsq;
        lf = lf + c[10] * rsq2;
        double q1 = 0.0 + p1 * lf;
        double q2 = 0.0 + p2 * lf;
        double d1 = 0.0 + q1 * c[6];
        double d2 = 0.0 + q2 * c[6];
        d1 = d1 + c[7];
        d2 = d2 + c[8];
        d1 = d1 - f1;
        d2 = d2 - f2;
        const double e1 = 0.0 + w * d1;
        const double e2 = 0.0 + w * d2;
        prefetch_next();                  // every staged input has been consumed

        // ---------------- sweep 3's middle: e2! -= w*d2; e1! -= w*d1 ----------------
        const G2 ge1{1.0, 0.0}, ge2{0.0, 1.0};
        G2 gw = zero2(), gd1 = zero2(), gd2 = zero2();
        GACC(gw, ge2, d2);
        GACC(gd2, ge2, w);
        GACC(gw, ge1, d1);
        GACC(gd1, ge1, w);

        // ------------------------- sweep 4 -------------------------
        G2 gc[11];
#pragma unroll
        for (int j = 0; j < 11; j++) gc[j] = zero2();
        G2 gX0 = zero2(), gX1 = zero2(), gX2 = zero2(), gf1 = zero2(), gf2 = zero2();
        G2 gq1 = zero2(), gq2 = zero2(), glf = zero2(), grsq = zero2(), grsq2 = zero2();
        G2 gp1 = zero2(), gp2 = zero2(), gr1 = zero2(), gr2 = zero2(), gr3 = zero2();
        G2 gx1 = zero2(), gx2 = zero2(), gx3 = zero2(), gsqt = zero2();
        d2 = d2 + f2;
        GACC(gf2, neg(gd2), 1.0);
        d1 = d1 + f1;
        GACC(gf1, neg(gd1), 1.0);
        d2 = d2 - c[8];
        GACC(gc[8], gd2, 1.0);
        d1 = d1 - c[7];
        GACC(gc[7], gd1, 1.0);
        d2 = d2 - q2 * c[6];
        GACC(gq2, gd2, c[6]);
        GACC(gc[6], gd2, q2);
        d1 = d1 - q1 * c[6];
        GACC(gq1, gd1, c[6]);
        GACC(gc[6], gd1, q1);
        if (chk && !code4 && (fabs(d2) > tol || fabs(d1) > tol)) code4 = RL_ERR_DIRTY_ANCILLA;
        q2 = q2 - p2 * lf;
        GACC(gp2, gq2, lf);
        GACC(glf, gq2, p2);
        q1 = q1 - p1 * lf;
        GACC(gp1, gq1, lf);
        GACC(glf, gq1, p1);
        if (chk && !code4 && (fabs(q2) > tol || fabs(q1) > tol)) code4 = RL_ERR_DIRTY_ANCILLA;
        lf = lf - c[10] * rsq2;
        GACC(gc[10], glf, rsq2);
        GACC(grsq2, glf, c[10]);
        lf = lf - c[9] * rsq;
        GACC(gc[9], glf, rsq);
        GACC(grsq, glf, c[9]);
        if (chk && !code4 && fabs(lf - 1.0) > tol) code4 = RL_ERR_DIRTY_ANCILLA;
        rsq2 = rsq2 - rsq * rsq;
        GACC(grsq, grsq2, 2.0 * rsq);
        if (chk && !code4 && fabs(rsq2) > tol) code4 = RL_ERR_DIRTY_ANCILLA;
        rsq = rsq - p2 * p2;
        GACC(gp2, grsq, 2.0 * p2);
        rsq = rsq - p1 * p1;
        GACC(gp1, grsq, 2.0 * p1);
        if (chk && !code4 && fabs(rsq) > tol) code4 = RL_ERR_DIRTY_ANCILLA;
        {
          p2 = p2 - r2 / r3;
          const double pa = 1.0 / r3, pb = r2 / (r3 * r3);
          GACC(gr2, gp2, pa);
          GACC(gr3, gp2, -pb);
          p1 = p1 - r1 / r3;
          const double pa1 = 1.0 / r3, pb1 = r1 / (r3 * r3);
          GACC(gr1, gp1, pa1);
          GACC(gr3, gp1, -pb1);
        }
        if (chk && !code4 && (fabs(p2) > tol || fabs(p1) > tol)) code4 = RL_ERR_DIRTY_ANCILLA;
        if (took) {
          // ~rodrigues: routine recomputed (values above are bit-identical),
          // inverted middle, then its uncompute with the adjoints
          G2 gw1 = zero2(), gw2 = zero2(), gw3 = zero2(), gtmp = zero2(), gcc1 = zero2(),
             gcc2 = zero2(), gcc3 = zero2(), gst = zero2(), gct = zero2(), gdt = zero2(),
             gomc = zero2(), gti = zero2(), gth = zero2();
          r3 = r3 - w3 * tmp;
          GACC(gw3, gr3, tmp);
          GACC(gtmp, gr3, w3);
          r2 = r2 - w2 * tmp;
          GACC(gw2, gr2, tmp);
          GACC(gtmp, gr2, w2);
          r1 = r1 - w1 * tmp;
          GACC(gw1, gr1, tmp);
          GACC(gtmp, gr1, w1);
          r3 = r3 - cc3 * st;
          GACC(gcc3, gr3, st);
          GACC(gst, gr3, cc3);
          r2 = r2 - cc2 * st;
          GACC(gcc2, gr2, st);
          GACC(gst, gr2, cc2);
          r1 = r1 - cc1 * st;
          GACC(gcc1, gr1, st);
          GACC(gst, gr1, cc1);
          r3 = r3 - x3 * ct;
          GACC(gx3, gr3, ct);
          GACC(gct, gr3, x3);
          r2 = r2 - x2 * ct;
          GACC(gx2, gr2, ct);
          GACC(gct, gr2, x2);
          r1 = r1 - x1 * ct;
          GACC(gx1, gr1, ct);
          GACC(gct, gr1, x1);
          // rodrigues' ~@routine
          tmp = tmp - dt * omc;
          GACC(gdt, gtmp, omc);
          GACC(gomc, gtmp, dt);
          if (chk && !code_rod && fabs(tmp) > tol) code_rod = RL_ERR_DIRTY_ANCILLA;
          omc = omc - (1.0 - ct);
          GACC(gct, gomc, -1.0);
          if (chk && !code_rod && fabs(omc) > tol) code_rod = RL_ERR_DIRTY_ANCILLA;
          dt = dt - w3 * x3;
          GACC(gw3, gdt, x3);
          GACC(gx3, gdt, w3);
          dt = dt - w2 * x2;
          GACC(gw2, gdt, x2);
          GACC(gx2, gdt, w2);
          dt = dt - w1 * x1;
          GACC(gw1, gdt, x1);
          GACC(gx1, gdt, w1);
          if (chk && !code_rod && fabs(dt) > tol) code_rod = RL_ERR_DIRTY_ANCILLA;
          cc3 = cc3 + w2 * x1;
          GACC(gw2, neg(gcc3), x1);
          GACC(gx1, neg(gcc3), w2);
          cc3 = cc3 - w1 * x2;
          GACC(gw1, gcc3, x2);
          GACC(gx2, gcc3, w1);
          cc2 = cc2 + w1 * x3;
          GACC(gw1, neg(gcc2), x3);
          GACC(gx3, neg(gcc2), w1);
          cc2 = cc2 - w3 * x1;
          GACC(gw3, gcc2, x1);
          GACC(gx1, gcc2, w3);
          cc1 = cc1 + w3 * x2;
          GACC(gw3, neg(gcc1), x2);
          GACC(gx2, neg(gcc1), w3);
          cc1 = cc1 - w2 * x3;
          GACC(gw2, gcc1, x3);
          GACC(gx3, gcc1, w2);
          if (chk && !code_rod && (fabs(cc3) > tol || fabs(cc2) > tol || fabs(cc1) > tol))
            code_rod = RL_ERR_DIRTY_ANCILLA;
          w3 = w3 - c[2] * ti;
          GACC(gc[2], gw3, ti);
          GACC(gti, gw3, c[2]);
          w2 = w2 - c[1] * ti;
          GACC(gc[1], gw2, ti);
          GACC(gti, gw2, c[1]);
          w1 = w1 - c[0] * ti;
          GACC(gc[0], gw1, ti);
          GACC(gti, gw1, c[0]);
          if (chk && !code_rod && (fabs(w3) > tol || fabs(w2) > tol || fabs(w1) > tol))
            code_rod = RL_ERR_DIRTY_ANCILLA;
          ti = ti - inv_th;
          GACC(gth, gti, -(1.0 / (th * th)));
          st = st - s_th;
          GACC(gth, gst, c_th);
          ct = ct - c_th;
          GACC(gth, gct, -s_th);
          if (chk && !code_rod && (fabs(ti) > tol || fabs(st) > tol || fabs(ct) > tol))
            code_rod = RL_ERR_DIRTY_ANCILLA;
          th = th - sq_t;
          GACC(gsqt, gth, 0.5 / sq_t);
          if (chk && !code_rod && fabs(th) > tol) code_rod = RL_ERR_DIRTY_ANCILLA;
        } else {
          r3 = r3 + c[1] * x1;
          GACC(gc[1], neg(gr3), x1);
          GACC(gx1, neg(gr3), c[1]);
          r3 = r3 - c[0] * x2;
          GACC(gc[0], gr3, x2);
          GACC(gx2, gr3, c[0]);
          r2 = r2 + c[0] * x3;
          GACC(gc[0], neg(gr2), x3);
          GACC(gx3, neg(gr2), c[0]);
          r2 = r2 - c[2] * x1;
          GACC(gc[2], gr2, x1);
          GACC(gx1, gr2, c[2]);
          r1 = r1 + c[2] * x2;
          GACC(gc[2], neg(gr1), x2);
          GACC(gx2, neg(gr1), c[2]);
          r1 = r1 - c[1] * x3;
          GACC(gc[1], gr1, x3);
          GACC(gx3, gr1, c[1]);
          r3 = r3 - x3;
          GACC(gx3, gr3, 1.0);
          r2 = r2 - x2;
          GACC(gx2, gr2, 1.0);
          r1 = r1 - x1;
          GACC(gx1, gr1, 1.0);
        }
        if (chk && !code4 && (fabs(r3) > tol || fabs(r2) > tol || fabs(r1) > tol))
          code4 = RL_ERR_DIRTY_ANCILLA;
        sqt = sqt - c[2] * c[2];
        GACC(gc[2], gsqt, 2.0 * c[2]);
        sqt = sqt - c[1] * c[1];
        GACC(gc[1], gsqt, 2.0 * c[1]);
        sqt = sqt - c[0] * c[0];
        GACC(gc[0], gsqt, 2.0 * c[0]);
        if (chk && !code4 && fabs(sqt) > tol) code4 = RL_ERR_DIRTY_ANCILLA;
        x3 = x3 - (X2 - c[5]);
        GACC(gX2, gx3, 1.0);
        GACC(gc[5], gx3, -1.0);
        x2 = x2 - (X1 - c[4]);
        GACC(gX1, gx2, 1.0);
        GACC(gc[4], gx2, -1.0);
        x1 = x1 - (X0 - c[3]);
        GACC(gX0, gx1, 1.0);
        GACC(gc[3], gx1, -1.0);
        if (chk && !code4 && (fabs(x3) > tol || fabs(x2) > tol || fabs(x1) > tol))
          code4 = RL_ERR_DIRTY_ANCILLA;
        // primal restoration: e1!, e2! back to 0 (exact here: e - w*d with
        // the same bits); ba_weight pass
        double ew = 0.0 + 1.0;
        ew = ew - w * w;
        const double EW = ew;
        ew = ew + w * w;
        const double gww = 0.0 + (-1.0 * 1.0) * (2.0 * w);
        ew = ew - 1.0;
        if (!code4 && !(fabs(ew - 0.0) <= tol)) code4 = RL_ERR_RESTORE;
        code_final = code_rod ? code_rod : (code1 ? code1 : code4);

#pragma unroll
        for (int j = 0; j < 11; j++) {
          row[j] = gc[j].a;
          row[15 + j] = gc[j].b;
        }
        row[11] = gX0.a;
        row[12] = gX1.a;
        row[13] = gX2.a;
        row[14] = gw.a;
        row[26] = gX0.b;
        row[27] = gX1.b;
        row[28] = gX2.b;
        row[29] = gw.b;
        row[30] = gww;
        if (WANT_ERR) {
          err_out[3 * i] = e1;
          err_out[3 * i + 1] = e2;
          err_out[3 * i + 2] = EW;
        }
        if (WANT_FEAT && GRAD) {
          Jf_out[4 * i] = gf1.a;
          Jf_out[4 * i + 1] = gf2.a;
          Jf_out[4 * i + 2] = gf1.b;
          Jf_out[4 * i + 3] = gf2.b;
        }
      }
      fail[i] = (uint8_t)code_final;
      nfail += code_final != 0;
    } else {
      prefetch_next();
    }
    if (!GRAD) continue;
    // stage the block's rows and write them out: one TMA bulk store of the
    // whole tile (the block's rows are one contiguous run of J), issued by
    // one thread and overlapping the next observation's compute; otherwise
    // (CSR, a partial block, misaligned J) coalesced 16-byte stores
    if (tid == 0)                          // previous bulk stores have read the tile
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    const long long rows = n_obs - blk0 < BA_BLOCK ? n_obs - blk0 : BA_BLOCK;
    if (CSR) {
      // ADBench BASparseMat::insert_reproj_err_block order: per observation two
      // rows of 15 (cam 11 | point 3 | weight 1), then all weight rows
      // (insert_w_err_block) after the 2P reprojection rows.  The block's
      // values, column indices and row pointers are staged in shared memory
      // in their CSR order (each piece one contiguous run of the output) and
      // leave as bulk stores where the run is 16-byte aligned and sized.
      double *vA = tile, *vW = tile + BA_BLOCK * 30;
      int32_t *cA = reinterpret_cast<int32_t *>(tile + BA_BLOCK * BA_ROW + BA_BLOCK * BA_STAGE);
      int32_t *cW = cA + BA_BLOCK * 30, *rA = cW + BA_BLOCK, *rW = rA + 2 * BA_BLOCK;
      if (valid) {
        const long long g = csr.off + i;                   // global observation
#pragma unroll
        for (int j = 0; j < 30; j++) vA[tid * 30 + j] = row[j];
        vW[tid] = row[30];
        if (csr.cols) {
          const int cc = in_range ? 11 * o.x : -1, cp = in_range ? csr.col_pt + 3 * o.y : -1;
          const int cw = csr.col_w + (int)g;
#pragma unroll
          for (int h = 0; h < 2; h++) {
#pragma unroll
            for (int j = 0; j < 11; j++) cA[tid * 30 + 15 * h + j] = cc < 0 ? -1 : cc + j;
#pragma unroll
            for (int j = 0; j < 3; j++) cA[tid * 30 + 15 * h + 11 + j] = cp < 0 ? -1 : cp + j;
            cA[tid * 30 + 15 * h + 14] = cw;
          }
          cW[tid] = cw;
          rA[2 * tid] = (int32_t)(30 * g);
          rA[2 * tid + 1] = (int32_t)(30 * g + 15);
          rW[tid] = (int32_t)(30 * csr.P + g);
          if (i == n_obs - 1) csr.rows[3 * n_obs] = (int32_t)(30 * csr.P + g + 1);
        }
      }
      __syncthreads();
      const int nr = (int)rows;
      auto put = [&](void *dst, const void *src, int bytes, int esz) {
        // bulk store when 16-byte aligned and sized, else a cooperative copy
        if (((reinterpret_cast<uintptr_t>(dst) | (unsigned)bytes) & 15) == 0) {
          if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes) : "memory");
          }
        } else if (esz == 8) {
          for (int k = tid; k < bytes / 8; k += BA_BLOCK)
            static_cast<double *>(dst)[k] = static_cast<const double *>(src)[k];
        } else {
          for (int k = tid; k < bytes / 4; k += BA_BLOCK)
            static_cast<int32_t *>(dst)[k] = static_cast<const int32_t *>(src)[k];
        }
      };
      put(csr.vals + blk0 * 30, vA, nr * 240, 8);
      put(csr.vals + n_obs * 30 + blk0, vW, nr * 8, 8);
      if (csr.cols) {
        put(csr.cols + blk0 * 30, cA, nr * 120, 4);
        put(csr.cols + n_obs * 30 + blk0, cW, nr * 4, 4);
        put(csr.rows + 2 * blk0, rA, nr * 8, 4);
        put(csr.rows + 2 * n_obs + blk0, rW, nr * 4, 4);
      }
      if (tid == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      continue;
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < BA_ROW; j++) tile[threadIdx.x * BA_ROW + j] = row[j];
    }
    __syncthreads();
    const int nd = (int)rows * BA_ROW;
    double *dst = J_out + blk0 * BA_ROW;
    if (rows == BA_BLOCK && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"((unsigned)__cvta_generic_to_shared(tile)), "r"(nd * 8) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      const int nv = nd >> 1;
      double2 *d2p = reinterpret_cast<double2 *>(dst);
      const double2 *s2p = reinterpret_cast<const double2 *>(tile);
      for (int k = threadIdx.x; k < nv; k += BA_BLOCK) d2p[k] = s2p[k];
      if ((nd & 1) && threadIdx.x == 0) dst[nd - 1] = tile[nd - 1];
    } else {
      for (int k = threadIdx.x; k < nd; k += BA_BLOCK) dst[k] = tile[k];
    }
  }
  if (GRAD && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  block_add_counters<BA_BLOCK>(0, nfail, counters);
}

int launch_ba(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams, const double *X,
              const double *w, const double *feats, const int32_t *obs, double tol,
              int32_t invcheck, double *err, double *J, double *Jfeat, uint8_t *fail,
              unsigned long long *counters, cudaStream_t st) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !J || !fail)))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_f64: bad argument");
  if ((reinterpret_cast<uintptr_t>(feats) & 15) || (reinterpret_cast<uintptr_t>(obs) & 7))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_f64: feats must be 16-byte and obs 8-byte aligned");
  int rc = ensure_device_tables();
  if (rc) return rc;
  if (n_obs == 0) return RL_OK;
  auto kern = err ? (Jfeat ? k_ba_jac<true, true> : k_ba_jac<true, false>)
                  : (Jfeat ? k_ba_jac<false, true> : k_ba_jac<false, false>);
  int bps = 0;
  rc = smem_attr((const void *)kern, BA_SMEM, "smem attr");
  if (rc) return rc;
  rc = occupancy(&bps, (const void *)kern, BA_BLOCK, BA_SMEM,
                   "occupancy");
  if (rc) return rc;
  long long want = (n_obs + BA_BLOCK - 1) / BA_BLOCK;
  long long cap = (long long)sm_count() * (bps > 0 ? bps : 1);
  int grid = (int)(want < cap ? want : cap);
  kern<<<grid, BA_BLOCK, BA_SMEM, st>>>(n_cams, n_pts, n_obs, cams, X, w, feats,
                                  reinterpret_cast<const int2 *>(obs), tol, invcheck ? 1 : 0, err,
                                  J, Jfeat, fail, counters, BaCsr{});
  return cuda_status(cudaGetLastError(), "k_ba_jac launch");
}

int launch_ba_residuals(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                        const double *X, const double *w, const double *feats,
                        const int32_t *obs, double tol, int32_t invcheck, double *err,
                        uint8_t *fail, unsigned long long *counters, cudaStream_t st) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !err || !fail)))
    return set_error(RL_ERR_INVALID, "rl_ba_residuals_f64: bad argument");
  if ((reinterpret_cast<uintptr_t>(feats) & 15) || (reinterpret_cast<uintptr_t>(obs) & 7))
    return set_error(RL_ERR_INVALID, "rl_ba_residuals_f64: feats must be 16-byte and obs 8-byte aligned");
  int rc = ensure_device_tables();
  if (rc) return rc;
  if (n_obs == 0) return RL_OK;
  auto kern = k_ba_jac<true, false, false>;
  int bps = 0;
  rc = smem_attr((const void *)kern, BA_SMEM, "smem attr");
  if (rc) return rc;
  rc = occupancy(&bps, (const void *)kern, BA_BLOCK, BA_SMEM,
                   "occupancy");
  if (rc) return rc;
  long long want = (n_obs + BA_BLOCK - 1) / BA_BLOCK;
  long long cap = (long long)sm_count() * (bps > 0 ? bps : 1);
  int grid = (int)(want < cap ? want : cap);
  kern<<<grid, BA_BLOCK, BA_SMEM, st>>>(n_cams, n_pts, n_obs, cams, X, w, feats,
                                  reinterpret_cast<const int2 *>(obs), tol, invcheck ? 1 : 0, err,
                                  nullptr, nullptr, fail, counters, BaCsr{});
  return cuda_status(cudaGetLastError(), "k_ba_jac (residuals) launch");
}

int launch_ba_csr(int32_t n_cams, int32_t n_pts, int64_t n_obs, int64_t obs_offset,
                  int64_t n_obs_total, const double *cams, const double *X, const double *w,
                  const double *feats, const int32_t *obs, double tol, int32_t invcheck,
                  double *err, int32_t *rows, int32_t *cols, double *vals, uint8_t *fail,
                  unsigned long long *counters, cudaStream_t st) {
  if (n_obs < 0 || n_cams < 0 || n_pts < 0 || obs_offset < 0 || n_obs_total < obs_offset + n_obs ||
      (n_obs > 0 && (!cams || !X || !w || !feats || !obs || !vals || !fail)) ||
      (cols && !rows) || (rows && !cols && n_obs > 0))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_csr_f64: bad argument");
  // BASparseMat holds int row pointers / column indices
  const long long ncols = 11LL * n_cams + 3LL * n_pts + n_obs_total;
  if (31LL * n_obs_total > INT32_MAX || ncols > INT32_MAX)
    return set_error(RL_ERR_INVALID, "rl_ba_jac_csr_f64: nnz or ncols exceeds int32 (BASparseMat)");
  if ((reinterpret_cast<uintptr_t>(feats) & 15) || (reinterpret_cast<uintptr_t>(obs) & 7))
    return set_error(RL_ERR_INVALID, "rl_ba_jac_csr_f64: feats must be 16-byte and obs 8-byte aligned");
  int rc = ensure_device_tables();
  if (rc) return rc;
  if (n_obs == 0) {
    if (rows) {
      const int32_t end = (int32_t)(30 * n_obs_total + obs_offset);
      return cuda_status(cudaMemcpyAsync(rows, &end, sizeof end, cudaMemcpyHostToDevice, st),
                         "rows terminator");
    }
    return RL_OK;
  }
  auto kern = err ? k_ba_jac<true, false, true, true> : k_ba_jac<false, false, true, true>;
  int bps = 0;
  rc = smem_attr((const void *)kern, BA_SMEM_CSR, "smem attr");
  if (rc) return rc;
  rc = occupancy(&bps, (const void *)kern, BA_BLOCK, BA_SMEM_CSR,
                   "occupancy");
  if (rc) return rc;
  long long want = (n_obs + BA_BLOCK - 1) / BA_BLOCK;
  long long cap = (long long)sm_count() * (bps > 0 ? bps : 1);
  int grid = (int)(want < cap ? want : cap);
  BaCsr csr{rows, cols, vals, obs_offset, n_obs_total, 11 * n_cams, 11 * n_cams + 3 * n_pts};
  kern<<<grid, BA_BLOCK, BA_SMEM_CSR, st>>>(n_cams, n_pts, n_obs, cams, X, w, feats,
                                  reinterpret_cast<const int2 *>(obs), tol, invcheck ? 1 : 0, err,
                                  nullptr, nullptr, fail, counters, csr);
  return cuda_status(cudaGetLastError(), "k_ba_jac (csr) launch");
}

}  // namespace rl
