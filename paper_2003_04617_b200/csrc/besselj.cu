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
// same checks sweep 2 would (the "dead uncompute" elision the paper allows,
// PAPER.md:650-651).  All reversibility checks of the reference are
// evaluated on device, in the reference's order, into a per-element flag:
//   loop entry/iteration postconditions  interpreter.py:772-797
//   ancilla releases |v - decl| <= tol    interpreter.py:717-748, 365-395
//   domain/overflow of log/exp            values.py:343-372
//
// Arithmetic is the reference's operation sequence (this file is compiled
// with -fmad=false: no contraction, IEEE add/mul/div).  Integer logs
// log(k), log(k + nu) come from a host libm table (bit-identical to the
// reference); exp is fexp.cuh (0.5 ulp + O(2^-60), bit-identical to the
// host libm in 99.92% of calls (tests/test_fexp.py), <= 1 ulp otherwise); log(z) and the final
// division are libdevice (<= 1 ulp / correctly rounded).
//
// Scheduling.  The series trip count T(z) is non-decreasing in z (every
// term grows with z), and a warp runs as long as its longest lane.  Each
// block therefore takes a chunk of C = BLOCK*M elements, counting-sorts it
// in shared memory by a z bucket (one smem atomic + scan per element), and
// each 32-lane round processes 32 neighbours in z order: lanes then have
// (nearly) equal trip counts and the loops run converged, with a
// warp-uniform k (the log table is a broadcast constant-cache read).  Warp
// w takes rounds w, w + W, ... so every warp gets the same mix of small
// and large z.  Results go back to the original order through shared
// memory and leave with coalesced stores.
#include <math.h>

#include "common.cuh"
#include "fexp.cuh"

namespace rl {

#ifdef BJ_PHASES   // timing-only builds: cycles per phase, summed over warps (tools)
__device__ unsigned long long g_bj_phase[16];
__shared__ long long s_bj_t[32];
#define BJ_MARK(ph)                                                              \
  do {                                                                           \
    __syncwarp();                                                                \
    const long long now_ = clock64();                                            \
    if ((threadIdx.x & 31) == 0) {                                               \
      atomicAdd(&g_bj_phase[ph], (unsigned long long)(now_ - s_bj_t[threadIdx.x >> 5])); \
      s_bj_t[threadIdx.x >> 5] = now_;                                           \
    }                                                                            \
  } while (0)
#else
#define BJ_MARK(ph) (void)0
#endif

__constant__ double c_logtab[LOGTAB_N];
constexpr double LN2 = 0.6931471805599453;  // == math.log(2) (host libm), bit for bit
#ifndef BJ_EXPN
#define BJ_EXPN 1024       // exp table size: 64 (degree-6 polynomial) or 1024 (degree 4)
#endif
#if BJ_EXPN == 1024
__device__ Exp2Tab g_exp2tab[1024] = RL_EXP2_TABLE_INIT_1024;
__constant__ ExpConsts1024 c_expk = RL_EXP_CONSTS_1024_INIT;
#elif BJ_EXPN == 256
__device__ Exp2Tab g_exp2tab[256] = RL_EXP2_TABLE_INIT_256;
__constant__ ExpConsts256 c_expk = RL_EXP_CONSTS_256_INIT;
#else
__device__ Exp2Tab g_exp2tab[64] = RL_EXP2_TABLE_INIT;
__constant__ ExpConsts c_expk = RL_EXP_CONSTS_INIT;
#endif
#ifndef BJ_REVU
#define BJ_REVU 2          // reverse-sweep trips per loop iteration (2 or 4; measured equal)
#endif

#ifndef BJ_SPEC
#define BJ_SPEC 2          // speculative trips per warp vote (2: fewer live registers -> 3 CTAs/SM, measured best)
#endif
#ifndef BJ_PAIR
#define BJ_PAIR 0          // 1: two z-neighbours per lane in the gradient / run kernels
#endif
#ifndef BJ_MINB
#if BJ_PAIR
#define BJ_MINB 2          // two elements per lane: up to 128 registers
#else
#define BJ_MINB 3          // __launch_bounds__ min blocks per SM (80 registers, no spills)
#endif
#endif
#ifndef BJ_HESS_PAIRS
#define BJ_HESS_PAIRS 1    // Hessian kernel: unpredicated trip pairs while every lane is live
#endif
#ifndef BJ_M
#define BJ_M 5             // chunk = BJ_M elements per thread (z-sorted per chunk; 3 CTAs/SM fit)
#endif
constexpr int BJ_BLOCK = 256;
constexpr int BJ_C = BJ_BLOCK * BJ_M;  // elements per chunk
constexpr int BJ_NB = 256;              // z buckets
constexpr int BJ_WARPS = BJ_BLOCK / 32;
// dynamic smem per block: prefetch buffer + sorted z + J + dz (doubles),
// original index (u16) and status (u8) per chunk element
constexpr int BJ_SMEM = BJ_C * (4 * 8 + 2 + 1);

// 2^(i/N) table, copied to shared memory per block (lane-varying index).
// The 256-entry form is replicated 8x with entry (i, c) at 16-byte slot
// 8 i + c and lane l reading copy c = l & 7: the 8 lanes of a quarter-warp
// then always hit 8 different bank groups (conflict-free 16-byte loads).
#if BJ_EXPN == 256
constexpr int BJ_EXPREP = 8;
#else
constexpr int BJ_EXPREP = 1;
#endif
__shared__ __align__(16) Exp2Tab s_exp2tab[BJ_EXPN * BJ_EXPREP];   // 16-byte loads
// (log k, log(k + nu)) for k < BJ_KP: one broadcast 16-byte shared load per
// series trip (k is warp-uniform) instead of two indexed constant loads
#ifndef BJ_KP
#define BJ_KP 512          // shared (log k, log(k + nu)) pairs (k beyond: the constant table)
#endif
__shared__ double2 s_logpair[BJ_KP];

__device__ __forceinline__ double logi(int i) {
  return i < LOGTAB_N ? c_logtab[i] : log((double)i);
}

// (log k, log(k + nu)); TAB: k < BJ_KP (shared-memory pair table)
template <bool TAB>
__device__ __forceinline__ double2 logpair(int k, int nu) {
  return TAB ? s_logpair[k] : make_double2(logi(k), logi(k + nu));
}

struct ExpR {
  double t;
  int code;
};

// exp with the reference's overflow semantics (math.exp raises
// OverflowError for a finite argument whose result overflows)
__device__ __forceinline__ ExpR rexp_slow(double x) {
  ExpR r;
  r.t = exp(x);
  r.code = (isinf(r.t) && isfinite(x)) ? RL_ERR_OVERFLOW : 0;
  return r;
}

// Two exp flavours.  FAST: table exp only, no range test: every argument of
// an element that passes the up-front safety bound (besselj_element) lies in
// (-700, 700).  Elements that fail the bound — only z in the hundreds, z
// below ~1e-140, or extreme nu / thr — are recomputed by the CAREFUL
// flavour, which tests every argument, takes libdevice's exp outside
// (-708, 708) and reports the reference's OverflowError.
template <bool CAREFUL>
__device__ __forceinline__ ExpR rexp(double x) {
  ExpR r;
#if BJ_EXPN == 256
  const unsigned lanebase =
      (unsigned)__cvta_generic_to_shared(s_exp2tab) + ((threadIdx.x & 7u) << 4);
#endif
  if (CAREFUL && (__double2hiint(x) & 0x7fffffff) >= 0x40862000) return rexp_slow(x);
#if BJ_EXPN == 1024
  // entry address = base + (i << 4): one IMAD from the masked index (the
  // compiler's own form is shift, mask, add)
  r.t = fexp1024(x,
                 [](int i) {
                   double2 v;
                   asm("{\n\t.reg .u32 a;\n\tmad.lo.u32 a, %2, 16, %3;\n\t"
                       "ld.shared.v2.f64 {%0, %1}, [a];\n\t}"
                       : "=d"(v.x), "=d"(v.y)
                       : "r"(i), "r"((unsigned)__cvta_generic_to_shared(s_exp2tab)));
                   return v;
                 },
                 c_expk);
#elif BJ_EXPN == 256
  r.t = fexp256(x,
                [lanebase](int i) {
                  double2 v;
                  asm("{\n\t.reg .u32 a;\n\tmad.lo.u32 a, %2, 128, %3;\n\t"
                      "ld.shared.v2.f64 {%0, %1}, [a];\n\t}"
                      : "=d"(v.x), "=d"(v.y)
                      : "r"(i), "r"(lanebase));
                  return v;
                },
                c_expk);
#else
  r.t = fexp_core(x, s_exp2tab, c_expk);
#endif
  r.code = 0;
  return r;
}

__device__ __forceinline__ int zbucket(double z) {
  if (!(z > 0.0)) return 0;
  return z < 21.0 ? (int)(z * 12.0) : BJ_NB - 1;
}

struct BJOut {
  double J, dz;
  int code, T;
  bool bad;
};

// One forward series trip at (warp-uniform) k; ODD = 1 / 0 when k is known
// to be odd / even (static sign of the alternating series), -1 otherwise.
// PRED: only lanes with `act` advance.
template <bool CAREFUL, bool TAB, bool PRED, int ODD>
__device__ __forceinline__ void fwd_trip(int k, int nu, double h2, double thr, bool &act,
                                         double &s, double &t, double &acc, int &T, int &code) {
  const double2 L = logpair<TAB>(k, nu);
  double sn = s + h2;                                    // s *= halfz2
  sn = sn - L.x;                                         // s /= k
  sn = sn - L.y;                                         // s /= kn
  const ExpR e = rexp<CAREFUL>(sn);
  // if (k % 2 == 0, ~): even k adds, odd k subtracts
  const bool odd = ODD == 1 || (ODD < 0 && (k & 1));
  const double an = odd ? acc - e.t : acc + e.t;
  if (!PRED || act) {
    s = sn;
    t = e.t;
    acc = an;
    T = k;
    if (CAREFUL) code = e.code;
    act = (!CAREFUL || !e.code) && e.t > thr;
  }
}

// One reverse trip at (warp-uniform) k for lanes with k <= T (PRED) or
// all lanes (the caller guarantees every live lane has k <= T).  With
// !GRAD (run / uncall / objective only) the cotangents are not carried.
// Unpredicated FAST trips do not touch `code`: they AND their postcondition
// into `ok` (one predicated compare), which the caller turns into the
// reference's PostconditionMismatch after the loop — the same first-failure
// result, since no other check can fire in between.
template <bool CAREFUL, bool TAB, bool PRED, int ODD, bool GRAD = true, bool UNIT = false>
__device__ __forceinline__ void rev_trip(int k, int nu, double h2, double thr, double paccg,
                                         double naccg, int chk, bool live, int T, double &acc,
                                         double &sg, double &s, double &h2g, double &t,
                                         int &code, bool &ok) {
  const double2 L = logpair<TAB>(k, nu);
  const double l2 = L.y, l1 = L.x;
  // inverse if: odd k: acc += convert(s) (sign -1); even: acc -= convert(s)
  const bool odd = ODD == 1 || (ODD < 0 && (k & 1));
  const double an = odd ? acc + t : acc - t;
  // UNIT (acc.g == 1.0 exactly): (+-1.0) * t == +-t, so sg +- t is the same sum
  const double sgn = !GRAD ? 0.0 : UNIT ? (odd ? sg - t : sg + t) : sg + (odd ? naccg : paccg) * t;
  double sn = s + l2;                                    // s *= kn
  sn = sn + l1;                                          // s *= k
  sn = sn - h2;                                          // s /= halfz2
  const double h2gn = GRAD ? h2g + sgn : 0.0;              // h2g += 1.0 * sg (x*1.0 == x exactly)
  const ExpR e = rexp<CAREFUL>(sn);
  if (!PRED || k <= T) {
    acc = an;
    sg = sgn;
    s = sn;
    h2g = h2gn;
    t = e.t;
    if (!CAREFUL && !PRED) {
      ok = ok && e.t > thr;
    } else {
      const int c = (CAREFUL && e.code) ? e.code
                                        : ((chk && !(e.t > thr)) ? RL_ERR_POSTCONDITION : 0);
      if (live && !code) code = c;
    }
  }
}

// One element; all 32 lanes of the warp call it together (`valid` false for
// padding lanes), because the loops are warp-synchronous: the trip index k
// is warp-uniform.  Lanes are z-sorted, so their trip counts (nearly)
// agree: the loops run unpredicated while every live lane is active and
// fall back to predicated trips only for the tail.
// ktab (uniform) = last k of the shared log-pair table; kfuel = the fuel
// cap on trips; sfloor = log(thr) - 2 log(kfuel + |nu| + 1) (host).
//
// Safety bound of the FAST flavour (no per-exp range test).  Every exp
// argument whose result is kept is a series log-term s_k: s_0 (tested), and
// s_k = s_{k-1} + h2 - log k - log(k + nu) where trip k only runs after
// exp(s_{k-1}) > thr, so s_k > log(thr) + h2 - 2 log(k + |nu|) >= h2 + sfloor;
// from above s_k <= log I_nu(z) <= z.  The reverse sweep walks the same s
// values back (to rounding).  So z < 700, |s_0| < 700 and h2 + sfloor > -700
// keep every argument inside (-700, 700); other elements (and thr <= 0 or
// NaN) are flagged `bad` and recomputed CAREFUL.  Speculative trips past a
// lane's end are discarded, so their arguments need no bound.
template <bool CAREFUL, bool GRAD>
__device__ __forceinline__ BJOut besselj_element(double z, bool valid, int nu, double thr,
                                                 double tol, double seed, int ktab, int kfuel,
                                                 int chk, double sfloor) {
  int code = 0;
  // ---------------- sweep 1: forward routine ----------------
  if (valid && !(z > 0.0)) code = RL_ERR_DOMAIN;        // lz *= convert(z)
  if (kfuel < 0 && valid && !code) code = RL_ERR_FUEL;   // the prologue alone exceeds max_steps
  const double logz = (valid && !code) ? log(z) : 0.0;
  double halfz = 0.0 + (0.0 + logz);                     // lz = 0 + log z; halfz *= lz
  halfz = halfz - LN2;                                   // halfz /= 2
  double h2 = 0.0 + halfz;                               // halfz2 *= halfz (x2)
  h2 = h2 + halfz;
  double s = 0.0;
  for (int q = 1; q <= nu; q++) {                        // for i = 1:1:nu
    s = s + halfz;
    s = s - (q < BJ_KP ? s_logpair[q].x : logi(q));
  }
  asm volatile("" : "+d"(h2));  // keep h2 live: no per-trip rematerialisation
  double t, acc;
  {
    const ExpR e = rexp<CAREFUL>(s);                     // acc += convert(s)
    t = e.t;
    if (!code) code = e.code;
    acc = 0.0 + t;
  }
  const bool bad = !CAREFUL && valid && !code &&
                   !(z < 700.0 && s > -700.0 && s < 700.0 && h2 + sfloor > -700.0);
  int T = 0;
  bool act = valid && !code && (t > thr);                // while (s > thr, k != 0)
  const bool dead = !valid || code;                      // state irrelevant from here
  const int code0 = code;
  int k = 0;
  if (nu < 0 && __any_sync(FULL_MASK, act)) {            // first trip: s /= kn, kn <= 0
    if (act) code = kfuel > 0 ? RL_ERR_DOMAIN : RL_ERR_FUEL;
    act = false;
  }
  const int kend = ktab < kfuel ? ktab : kfuel;
  if (!CAREFUL) BJ_MARK(6);                               // prologue
  // main phase: every non-dead lane still active -> no predication.  Two
  // trips (odd k+1, even k+2) are computed speculatively per warp vote: the
  // term s of trip k+2 does not depend on exp() of trip k+1, so the two exp
  // chains overlap; a lane whose loop ended at k+1 keeps its trip-(k+1)
  // state and discards trip k+2.
  if (!CAREFUL && __all_sync(FULL_MASK, act || dead) && __any_sync(FULL_MASK, act)) {
#if BJ_SPEC == 4
    while (k + 4 <= kend) {                              // k even: trips odd, even, odd, even
      const double2 L1 = s_logpair[k + 1], L2 = s_logpair[k + 2];
      const double2 L3 = s_logpair[k + 3], L4 = s_logpair[k + 4];
      double s1 = s + h2;
      s1 = s1 - L1.x;
      s1 = s1 - L1.y;
      double s2 = s1 + h2;
      s2 = s2 - L2.x;
      s2 = s2 - L2.y;
      double s3 = s2 + h2;
      s3 = s3 - L3.x;
      s3 = s3 - L3.y;
      double s4 = s3 + h2;
      s4 = s4 - L4.x;
      s4 = s4 - L4.y;
      const double t1 = rexp<CAREFUL>(s1).t;
      const double t2 = rexp<CAREFUL>(s2).t;
      const double t3 = rexp<CAREFUL>(s3).t;
      const double t4 = rexp<CAREFUL>(s4).t;
      const double a1 = acc - t1;
      const double a2 = a1 + t2;
      const double a3 = a2 - t3;
      const double a4 = a3 + t4;
      const bool act1 = t1 > thr, act2 = t2 > thr, act3 = t3 > thr, act4 = t4 > thr;
      if (__all_sync(FULL_MASK, (act1 && act2 && act3 && act4) || dead)) {
        s = s4;
        t = t4;
        acc = a4;
        k += 4;
        T = k;
        continue;
      }
      if (!act1) {
        s = s1; t = t1; acc = a1; T = k + 1; act = false;
      } else if (!act2) {
        s = s2; t = t2; acc = a2; T = k + 2; act = false;
      } else if (!act3) {
        s = s3; t = t3; acc = a3; T = k + 3; act = false;
      } else {
        s = s4; t = t4; acc = a4; T = k + 4; act = act4;
      }
      k += 4;
      break;
    }
#else
    while (k + 2 <= kend) {
      const double2 L1 = s_logpair[k + 1], L2 = s_logpair[k + 2];
      double s1 = s + h2;                                // trip k+1 (odd)
      s1 = s1 - L1.x;
      s1 = s1 - L1.y;
      double s2 = s1 + h2;                               // trip k+2 (even)
      s2 = s2 - L2.x;
      s2 = s2 - L2.y;
      const double t1 = rexp<CAREFUL>(s1).t;
      const double t2 = rexp<CAREFUL>(s2).t;
      const double a1 = acc - t1;                        // odd k subtracts
      const double a2 = a1 + t2;                         // even k adds
      const bool act1 = t1 > thr, act2 = t2 > thr;
      if (__all_sync(FULL_MASK, (act1 && act2) || dead)) {
        s = s2;
        t = t2;
        acc = a2;
        k += 2;
        T = k;
        continue;
      }
      if (act1) {
        s = s2;
        t = t2;
        acc = a2;
        T = k + 2;
        act = act2;
      } else {
        s = s1;
        t = t1;
        acc = a1;
        T = k + 1;
        act = false;
      }
      k += 2;
      break;
    }
#endif
    if (dead) {                                          // undo the unpredicated trips
      act = false;
      T = 0;
      code = code0;
    }
  }
  // tail: predicated
  while (k < kend && __any_sync(FULL_MASK, act)) {
    k++;
    fwd_trip<CAREFUL, true, true, -1>(k, nu, h2, thr, act, s, t, acc, T, code);
  }
  while (k < kfuel && __any_sync(FULL_MASK, act)) {      // beyond the table (huge nu / T)
    k++;
    fwd_trip<CAREFUL, false, true, -1>(k, nu, h2, thr, act, s, t, acc, T, code);
  }
  if (act) code = RL_ERR_FUEL;                           // still running at the fuel cap
  if (!CAREFUL) BJ_MARK(7);                               // forward loops
  BJOut o;
  o.J = 0.0 + acc;                                       // out! += acc
  o.T = T;
  const bool fwd_ok = valid && !code;

  // ---------------- sweep 4: ~routine with adjoints ----------------
  const double accg = 0.0 + (1.0 * seed) * 1.0;          // out! -= acc: acc.g += out.g
  const double paccg = 1.0 * accg, naccg = -1.0 * accg;
  double sg = 0.0, h2g = 0.0;
  bool ok = true;                                        // postconditions of unpredicated trips
  if (fwd_ok && chk && t > thr) code = RL_ERR_POSTCONDITION;  // entry: post false
  const int Tmax = __reduce_max_sync(FULL_MASK, fwd_ok ? T : 0);
  const unsigned Tmin = __reduce_min_sync(FULL_MASK, fwd_ok ? (unsigned)T : 0x7fffffffu);
  int kr = Tmax;
  for (; kr > ktab; kr--)                                // beyond the table
    rev_trip<CAREFUL, false, true, -1, GRAD>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok,
                                       fwd_ok ? T : 0, acc, sg, s, h2g, t, code, ok);
  for (; kr > (int)Tmin; kr--)                           // tail: predicated
    rev_trip<CAREFUL, true, true, -1, GRAD>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok,
                                      fwd_ok ? T : 0, acc, sg, s, h2g, t, code, ok);
  // the reverse loop is counted (no votes): pairs already overlap the exp chains
  if (kr >= 1 && !(kr & 1)) {                            // align: pairs start at odd k
    rev_trip<CAREFUL, true, false, 0, GRAD>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg, s,
                                      h2g, t, code, ok);
    kr--;
  }
#if BJ_REVU == 4
  for (; kr >= 4; kr -= 4) {                             // main, 4 trips: the exp chains overlap
    rev_trip<CAREFUL, true, false, 1, GRAD>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg, s,
                                      h2g, t, code, ok);
    rev_trip<CAREFUL, true, false, 0, GRAD>(kr - 1, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg,
                                      s, h2g, t, code, ok);
    rev_trip<CAREFUL, true, false, 1, GRAD>(kr - 2, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg,
                                      s, h2g, t, code, ok);
    rev_trip<CAREFUL, true, false, 0, GRAD>(kr - 3, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg,
                                      s, h2g, t, code, ok);
  }
#endif
  if (accg == 1.0) {                                     // the default seed (uniform branch)
    for (; kr >= 2; kr -= 2) {                           // main: every live lane active
      rev_trip<CAREFUL, true, false, 1, GRAD, true>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok, T,
                                                    acc, sg, s, h2g, t, code, ok);
      rev_trip<CAREFUL, true, false, 0, GRAD, true>(kr - 1, nu, h2, thr, paccg, naccg, chk, fwd_ok,
                                                    T, acc, sg, s, h2g, t, code, ok);
    }
  }
  for (; kr >= 2; kr -= 2) {                             // main: every live lane active
    rev_trip<CAREFUL, true, false, 1, GRAD>(kr, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg, s,
                                      h2g, t, code, ok);
    rev_trip<CAREFUL, true, false, 0, GRAD>(kr - 1, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg,
                                      s, h2g, t, code, ok);
  }
  if (kr == 1)
    rev_trip<CAREFUL, true, false, 1, GRAD>(1, nu, h2, thr, paccg, naccg, chk, fwd_ok, T, acc, sg, s,
                                      h2g, t, code, ok);
  if (!CAREFUL && chk && fwd_ok && !ok && !code) code = RL_ERR_POSTCONDITION;
  if (!CAREFUL) BJ_MARK(8);                               // reverse loops
  double zg = 0.0;
  if (fwd_ok) {
    acc = acc - t;                                       // acc -= convert(s)
    if (GRAD) sg = sg + (1.0 * accg) * t;
    double hzg = 0.0;
    for (int q = nu; q >= 1; q--) {                      // for i = nu:-1:1
      s = s + (q < BJ_KP ? s_logpair[q].x : logi(q));
      s = s - halfz;
      hzg = hzg + 1.0 * sg;
    }
    h2 = h2 - halfz;                                     // halfz2 /= halfz (x2)
    hzg = hzg + 1.0 * h2g;
    h2 = h2 - halfz;
    hzg = hzg + 1.0 * h2g;
    double lz = 0.0 + logz;
    halfz = halfz + LN2;                                 // halfz *= 2
    halfz = halfz - lz;                                  // halfz /= lz
    const double lzg = 0.0 + 1.0 * hzg;
    lz = lz - logz;                                      // lz /= convert(z)
    if (GRAD) zg = zg + (1.0 * lzg) / z;
    if (chk && !code) {                                  // releases
      if (fabs(acc - 0.0) > tol || fabs(s - 0.0) > tol || fabs(h2 - 0.0) > tol ||
          fabs(halfz - 0.0) > tol || fabs(lz - 0.0) > tol)
        code = RL_ERR_DIRTY_ANCILLA;
    }
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ULL);
  if (!fwd_ok) o.J = qnan;
  o.dz = fwd_ok ? zg : qnan;
  o.code = code;
  o.bad = valid && bad;
  if (!CAREFUL) BJ_MARK(9);                               // epilogue
  return o;
}


// ---------------------------------------------------------------------------
// Forward-over-reverse Hessian (autodiff.hessian, autodiff.py:216-257): the
// gradient sweeps over Dual numbers (values.py:258-340), z carrying the unit
// tangent, so dz.g's tangent is d2J/dz2.  Every Dual operation is the
// reference's: add/sub componentwise, (p, t) * f = (p f, t f + p 0.0), the
// quotient rule of Dual.__truediv__, s_exp = (e^p, t e^p), s_log = (log p,
// t / p); floats enter as (f, 0.0) (bit-identical to _as_dual: the same two
// tangent products, IEEE + and * commute).  Sweeps 3 / 4 use the gradient-
// mode forms (log_x +- contrib, delta = (sign gy) * s_exp(log_x)); the primal
// halves are the gradient kernel's arithmetic, so J and dJ/dz are bit-equal
// to rl_besselj_grad_f64's.  Per-lane loops (lanes are z-sorted, so their
// trip counts agree); not the speculative structure of the gradient path.
// ---------------------------------------------------------------------------
struct Dl {
  double p, t;
};
__device__ __forceinline__ Dl dadd(Dl a, Dl b) { return Dl{a.p + b.p, a.t + b.t}; }
__device__ __forceinline__ Dl dsub(Dl a, Dl b) { return Dl{a.p - b.p, a.t - b.t}; }
__device__ __forceinline__ Dl dmul(Dl a, Dl b) { return Dl{a.p * b.p, a.t * b.p + a.p * b.t}; }
__device__ __forceinline__ Dl ddiv(Dl a, Dl b) {
  const double q = a.p / b.p;
  return Dl{q, (a.t - q * b.t) / b.p};
}
__device__ __forceinline__ Dl dflt(double f) { return Dl{f, 0.0}; }
template <bool CAREFUL>
__device__ __forceinline__ Dl dexp(Dl a, int &code) {
  const ExpR e = rexp<CAREFUL>(a.p);
  if (CAREFUL && e.code && !code) code = e.code;
  return Dl{e.t, a.t * e.t};
}
__device__ __forceinline__ double2 logpair_any(int k, int nu) {
  return k < BJ_KP ? s_logpair[k] : make_double2(logi(k), logi(k + nu));
}

struct BJHOut {
  double J, dz, d2;
  int code, T;
  bool bad;
};

template <bool CAREFUL>
__device__ __forceinline__ BJHOut besselj_hess_element(double z, bool valid, int nu, double thr,
                                                       double tol, double seed, int kfuel,
                                                       int chk, double sfloor) {
  int code = 0;
  // ---------------- sweep 3 (= sweep 1 primal): R over Duals ----------------
  if (valid && !(z > 0.0)) code = RL_ERR_DOMAIN;        // lz *= convert(z)
  if (kfuel < 0 && valid && !code) code = RL_ERR_FUEL;   // the prologue alone exceeds max_steps
  const bool zok = valid && !code;
  const Dl Z{z, 1.0};
  const Dl clz{zok ? log(z) : 0.0, zok ? 1.0 / z : 0.0};   // s_log(Dual(z, 1))
  Dl lz = dadd(dflt(0.0), clz);
  Dl halfz = dadd(dflt(0.0), lz);                         // halfz *= lz
  halfz = dsub(halfz, dflt(LN2));                         // halfz /= 2
  Dl h2 = dadd(dflt(0.0), halfz);                         // halfz2 *= halfz (x2)
  h2 = dadd(h2, halfz);
  Dl s = dflt(0.0);
  for (int q = 1; q <= nu; q++) {                         // for i = 1:1:nu
    s = dadd(s, halfz);
    s = dsub(s, dflt(logi(q)));
  }
  Dl e = dexp<CAREFUL>(s, code);                          // acc += convert(s)
  Dl acc = dadd(dflt(0.0), e);
  const bool bad = !CAREFUL && zok &&
                   !(z < 700.0 && s.p > -700.0 && s.p < 700.0 && h2.p + sfloor > -700.0);
  bool act = valid && !code && e.p > thr;                 // while (s > thr, k != 0)
  if (nu < 0 && act) {                                    // first trip: s /= kn, kn <= 0
    code = kfuel > 0 ? RL_ERR_DOMAIN : RL_ERR_FUEL;
    act = false;
  }
  int k = 0;
#if BJ_HESS_PAIRS
  // FAST main phase, as in besselj_element: while every live lane is still
  // active the trips run in unpredicated pairs with one vote per pair (the
  // pair's second log-domain term does not depend on the first's exp); the
  // predicated loop below finishes the tail.  Same Dual operations in the
  // same order per lane; dead lanes are restored afterwards.
  if (!CAREFUL) {
    const bool dead = !valid || code;
    const int kend = (BJ_KP - 1) < kfuel ? (BJ_KP - 1) : kfuel;
    if (__all_sync(FULL_MASK, act || dead) && __any_sync(FULL_MASK, act)) {
      while (k + 2 <= kend) {
        const double2 L1 = s_logpair[k + 1], L2 = s_logpair[k + 2];
        Dl s1 = dadd(s, h2);
        s1 = dsub(s1, dflt(L1.x));
        s1 = dsub(s1, dflt(L1.y));
        Dl s2 = dadd(s1, h2);
        s2 = dsub(s2, dflt(L2.x));
        s2 = dsub(s2, dflt(L2.y));
        int cf = 0;
        const Dl e1 = dexp<false>(s1, cf), e2 = dexp<false>(s2, cf);
        const bool odd1 = (k + 1) & 1;
        const Dl a1 = odd1 ? dsub(acc, e1) : dadd(acc, e1);
        const Dl a2 = odd1 ? dadd(a1, e2) : dsub(a1, e2);
        const bool act1 = e1.p > thr, act2 = e2.p > thr;
        if (__all_sync(FULL_MASK, (act1 && act2) || dead)) {
          s = s2;
          e = e2;
          acc = a2;
          k += 2;
          continue;
        }
        if (act1) {
          s = s2;
          e = e2;
          acc = a2;
          k += 2;
          act = act2;
        } else {
          s = s1;
          e = e1;
          acc = a1;
          k += 1;
          act = false;
        }
        break;
      }
      if (dead) {
        act = false;
        k = 0;
      }
    }
  }
#endif
  while (__any_sync(FULL_MASK, act)) {
    if (act) {
      if (k >= kfuel) {
        code = RL_ERR_FUEL;
        act = false;
      } else {
        k++;
        const double2 L = logpair_any(k, nu);
        s = dadd(s, h2);                                  // s *= halfz2
        s = dsub(s, dflt(L.x));                           // s /= k
        s = dsub(s, dflt(L.y));                           // s /= kn
        e = dexp<CAREFUL>(s, code);
        acc = (k & 1) ? dsub(acc, e) : dadd(acc, e);      // if (k % 2 == 0, ~)
        act = !code && e.p > thr;
      }
    }
  }
  const int T = k;
  BJHOut o;
  o.J = 0.0 + acc.p;                                      // out! += acc
  o.T = T;
  const bool fwd_ok = valid && !code;
  // ---------------- sweep 4: ~R with the adjoint rules over Duals ----------------
  const double gacc = (1.0 * seed) * 1.0;                 // out! -= acc: acc.g += out.g
  Dl gs = dflt(0.0), gh2 = dflt(0.0);
  if (fwd_ok && chk && e.p > thr) code = RL_ERR_POSTCONDITION;  // entry: post false
  int kr = fwd_ok ? T : 0;
  auto rtrip = [&](int kk) {                              // one reverse trip at kk (kr = kk)
    if (kk & 1) {                                         // acc += convert(s): sign -1
      acc = dadd(acc, e);
      gs = dadd(gs, dmul(dflt(-1.0 * gacc), e));
    } else {                                              // acc -= convert(s): sign +1
      acc = dsub(acc, e);
      gs = dadd(gs, dmul(dflt(1.0 * gacc), e));
    }
    const double2 L = logpair_any(kk, nu);
    s = dadd(s, dflt(L.y));                               // s *= kn
    s = dadd(s, dflt(L.x));                               // s *= k
    s = dsub(s, h2);                                      // s /= halfz2
    gh2 = dadd(gh2, dmul(dflt(1.0), gs));
    int c = 0;
    e = dexp<CAREFUL>(s, c);
    if (!code) code = c ? c : ((chk && !(e.p > thr)) ? RL_ERR_POSTCONDITION : 0);
  };
#if BJ_HESS_PAIRS
  if (!CAREFUL) {
    // predicated until every live lane is down to the warp's smallest trip
    // count, then the rest unpredicated for all lanes (dead lanes compute
    // values that are never stored)
    const unsigned tmin = __reduce_min_sync(FULL_MASK, fwd_ok ? (unsigned)T : 0x7fffffffu);
    if (tmin != 0x7fffffffu) {
      while (__any_sync(FULL_MASK, kr > (int)tmin))
        if (kr > (int)tmin) rtrip(kr--);
      int kk = (int)tmin;
      for (; kk >= 2; kk -= 2) {
        rtrip(kk);
        rtrip(kk - 1);
      }
      if (kk == 1) rtrip(1);
      kr = 0;
    }
  }
#endif
  while (__any_sync(FULL_MASK, kr >= 1)) {
    if (kr >= 1) rtrip(kr--);
  }
  Dl gz = dflt(0.0);
  if (fwd_ok) {
    acc = dsub(acc, e);                                   // acc -= convert(s)
    gs = dadd(gs, dmul(dflt(1.0 * gacc), e));
    Dl gh = dflt(0.0);
    for (int q = nu; q >= 1; q--) {                       // for i = nu:-1:1
      s = dadd(s, dflt(logi(q)));
      s = dsub(s, halfz);
      gh = dadd(gh, dmul(dflt(1.0), gs));
    }
    h2 = dsub(h2, halfz);                                 // halfz2 /= halfz (x2)
    gh = dadd(gh, dmul(dflt(1.0), gh2));
    h2 = dsub(h2, halfz);
    gh = dadd(gh, dmul(dflt(1.0), gh2));
    halfz = dadd(halfz, dflt(LN2));                       // halfz *= 2
    halfz = dsub(halfz, lz);                              // halfz /= lz
    const Dl glz = dadd(dflt(0.0), dmul(dflt(1.0), gh));
    lz = dsub(lz, clz);                                   // lz /= convert(z)
    gz = dadd(gz, ddiv(dmul(dflt(1.0), glz), Z));
    if (chk && !code) {                                   // releases
      if (fabs(acc.p - 0.0) > tol || fabs(s.p - 0.0) > tol || fabs(h2.p - 0.0) > tol ||
          fabs(halfz.p - 0.0) > tol || fabs(lz.p - 0.0) > tol)
        code = RL_ERR_DIRTY_ANCILLA;
    }
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ULL);
  if (!fwd_ok) o.J = qnan;
  o.dz = fwd_ok ? gz.p : qnan;
  o.d2 = fwd_ok ? gz.t : qnan;
  o.code = code;
  o.bad = valid && bad;
  if (!CAREFUL) BJ_MARK(9);                               // epilogue
  return o;
}

// MODE 1: gradient (sweeps 1 + 4, Jout = J, dzout = dJ/dz).  MODE 0: run /
// uncall of besselj (Jout = out_in + sign * J with every check of the two
// primal sweeps; dzout unused): the objective-only ("-O") kernel.  MODE 2:
// the Hessian (Dual sweeps; d2out = d2J/dz2).
// ---------------------------------------------------------------------------
// Two elements per lane (BJ_PAIR): besselj_element<false, GRAD>'s
// per-element operation sequence (bit-identical results) over two
// z-neighbours, interleaved so each warp carries two independent dependency
// chains; the warp votes and the trip bounds cover both.  Elements failing
// the FAST bound are recomputed by the single-element CAREFUL path.
// ---------------------------------------------------------------------------
struct BJS {
  double z, logz, halfz, h2, s, t, acc, sg, h2g, J;
  int code, code0, T;
  bool valid, act, dead, bad, fwd_ok, ok;
};

__device__ __forceinline__ void bjp_prologue(BJS &e, int nu, double thr, int kfuel, double sfloor) {
  e.code = 0;
  if (e.valid && !(e.z > 0.0)) e.code = RL_ERR_DOMAIN;       // lz *= convert(z)
  if (kfuel < 0 && e.valid && !e.code) e.code = RL_ERR_FUEL;
  e.logz = (e.valid && !e.code) ? log(e.z) : 0.0;
  double halfz = 0.0 + (0.0 + e.logz);                      // lz = 0 + log z; halfz *= lz
  halfz = halfz - LN2;                                       // halfz /= 2
  double h2 = 0.0 + halfz;                                   // halfz2 *= halfz (x2)
  h2 = h2 + halfz;
  double s = 0.0;
  for (int q = 1; q <= nu; q++) {                            // for i = 1:1:nu
    s = s + halfz;
    s = s - (q < BJ_KP ? s_logpair[q].x : logi(q));
  }
  e.halfz = halfz;
  e.h2 = h2;
  e.s = s;
  e.t = rexp<false>(s).t;                                    // acc += convert(s)
  e.acc = 0.0 + e.t;
  e.bad = e.valid && !e.code &&
          !(e.z < 700.0 && s > -700.0 && s < 700.0 && h2 + sfloor > -700.0);
  e.T = 0;
  e.act = e.valid && !e.code && (e.t > thr);                 // while (s > thr, k != 0)
  e.dead = !e.valid || e.code;
  e.code0 = e.code;
}

// one speculative pair of forward trips (odd k + 1, even k + 2) of one element
struct BJSpec {
  double s1, s2, t1, t2, a1, a2;
  bool act1, act2;
};
__device__ __forceinline__ BJSpec bjp_spec(const BJS &e, double2 L1, double2 L2, double thr) {
  BJSpec p;
  p.s1 = e.s + e.h2;                                         // trip k+1 (odd)
  p.s1 = p.s1 - L1.x;
  p.s1 = p.s1 - L1.y;
  p.s2 = p.s1 + e.h2;                                        // trip k+2 (even)
  p.s2 = p.s2 - L2.x;
  p.s2 = p.s2 - L2.y;
  p.t1 = rexp<false>(p.s1).t;
  p.t2 = rexp<false>(p.s2).t;
  p.a1 = e.acc - p.t1;                                       // odd k subtracts
  p.a2 = p.a1 + p.t2;                                        // even k adds
  p.act1 = p.t1 > thr;
  p.act2 = p.t2 > thr;
  return p;
}

template <bool GRAD>
__device__ __forceinline__ BJOut bjp_epilogue(BJS &e, int nu, double tol, double accg, int chk) {
  double zg = 0.0;
  if (e.fwd_ok) {
    double acc = e.acc - e.t;                                // acc -= convert(s)
    double sg = e.sg;
    if (GRAD) sg = sg + (1.0 * accg) * e.t;
    double s = e.s, hzg = 0.0;
    for (int q = nu; q >= 1; q--) {                          // for i = nu:-1:1
      s = s + (q < BJ_KP ? s_logpair[q].x : logi(q));
      s = s - e.halfz;
      hzg = hzg + 1.0 * sg;
    }
    double h2 = e.h2 - e.halfz;                              // halfz2 /= halfz (x2)
    hzg = hzg + 1.0 * e.h2g;
    h2 = h2 - e.halfz;
    hzg = hzg + 1.0 * e.h2g;
    double lz = 0.0 + e.logz;
    double halfz = e.halfz + LN2;                            // halfz *= 2
    halfz = halfz - lz;                                      // halfz /= lz
    const double lzg = 0.0 + 1.0 * hzg;
    lz = lz - e.logz;                                        // lz /= convert(z)
    if (GRAD) zg = zg + (1.0 * lzg) / e.z;
    if (chk && !e.code) {                                    // releases
      if (fabs(acc - 0.0) > tol || fabs(s - 0.0) > tol || fabs(h2 - 0.0) > tol ||
          fabs(halfz - 0.0) > tol || fabs(lz - 0.0) > tol)
        e.code = RL_ERR_DIRTY_ANCILLA;
    }
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ULL);
  BJOut o;
  o.J = e.fwd_ok ? e.J : qnan;
  o.dz = e.fwd_ok ? zg : qnan;
  o.T = e.T;
  o.code = e.code;
  o.bad = e.valid && e.bad;
  return o;
}

template <bool GRAD>
__device__ __forceinline__ void besselj_pair(BJS &A, BJS &B, int nu, double thr, double tol,
                                             double seed, int ktab, int kfuel, int chk,
                                             double sfloor, BJOut &oa, BJOut &ob) {
  // ---------------- sweep 1: forward routine ----------------
  bjp_prologue(A, nu, thr, kfuel, sfloor);
  bjp_prologue(B, nu, thr, kfuel, sfloor);
  int k = 0;
  if (nu < 0 && __any_sync(FULL_MASK, A.act || B.act)) {     // first trip: s /= kn, kn <= 0
    if (A.act) A.code = kfuel > 0 ? RL_ERR_DOMAIN : RL_ERR_FUEL;
    if (B.act) B.code = kfuel > 0 ? RL_ERR_DOMAIN : RL_ERR_FUEL;
    A.act = B.act = false;
  }
  const int kend = ktab < kfuel ? ktab : kfuel;
  if (__all_sync(FULL_MASK, (A.act || A.dead) && (B.act || B.dead)) &&
      __any_sync(FULL_MASK, A.act || B.act)) {
    while (k + 2 <= kend) {
      const double2 L1 = s_logpair[k + 1], L2 = s_logpair[k + 2];
      const BJSpec pa = bjp_spec(A, L1, L2, thr), pb = bjp_spec(B, L1, L2, thr);
      if (__all_sync(FULL_MASK, ((pa.act1 && pa.act2) || A.dead) &&
                                    ((pb.act1 && pb.act2) || B.dead))) {
        A.s = pa.s2; A.t = pa.t2; A.acc = pa.a2;
        B.s = pb.s2; B.t = pb.t2; B.acc = pb.a2;
        k += 2;
        A.T = k;
        B.T = k;
        continue;
      }
      auto commit = [&](BJS &e, const BJSpec &p) {
        if (p.act1) {
          e.s = p.s2; e.t = p.t2; e.acc = p.a2; e.T = k + 2; e.act = p.act2;
        } else {
          e.s = p.s1; e.t = p.t1; e.acc = p.a1; e.T = k + 1; e.act = false;
        }
      };
      commit(A, pa);
      commit(B, pb);
      k += 2;
      break;
    }
    if (A.dead) { A.act = false; A.T = 0; A.code = A.code0; }   // undo the unpredicated trips
    if (B.dead) { B.act = false; B.T = 0; B.code = B.code0; }
  }
  // tail: predicated
  while (k < kend && __any_sync(FULL_MASK, A.act || B.act)) {
    k++;
    fwd_trip<false, true, true, -1>(k, nu, A.h2, thr, A.act, A.s, A.t, A.acc, A.T, A.code);
    fwd_trip<false, true, true, -1>(k, nu, B.h2, thr, B.act, B.s, B.t, B.acc, B.T, B.code);
  }
  while (k < kfuel && __any_sync(FULL_MASK, A.act || B.act)) {   // beyond the table
    k++;
    fwd_trip<false, false, true, -1>(k, nu, A.h2, thr, A.act, A.s, A.t, A.acc, A.T, A.code);
    fwd_trip<false, false, true, -1>(k, nu, B.h2, thr, B.act, B.s, B.t, B.acc, B.T, B.code);
  }
  if (A.act) A.code = RL_ERR_FUEL;                           // still running at the fuel cap
  if (B.act) B.code = RL_ERR_FUEL;
  A.J = 0.0 + A.acc;                                         // out! += acc
  B.J = 0.0 + B.acc;
  A.fwd_ok = A.valid && !A.code;
  B.fwd_ok = B.valid && !B.code;

  // ---------------- sweep 4: ~routine with adjoints ----------------
  const double accg = 0.0 + (1.0 * seed) * 1.0;              // out! -= acc: acc.g += out.g
  const double paccg = 1.0 * accg, naccg = -1.0 * accg;
  A.sg = A.h2g = B.sg = B.h2g = 0.0;
  A.ok = B.ok = true;
  if (A.fwd_ok && chk && A.t > thr) A.code = RL_ERR_POSTCONDITION;   // entry: post false
  if (B.fwd_ok && chk && B.t > thr) B.code = RL_ERR_POSTCONDITION;
  const int TA = A.fwd_ok ? A.T : 0, TB = B.fwd_ok ? B.T : 0;
  const int Tmax = __reduce_max_sync(FULL_MASK, TA > TB ? TA : TB);
  const unsigned Tmin = __reduce_min_sync(
      FULL_MASK, (unsigned)min(A.fwd_ok ? A.T : 0x7fffffff, B.fwd_ok ? B.T : 0x7fffffff));
  int kr = Tmax;
#define BJP_REV(CAR, TAB, PRED, ODD, UNIT, KK)                                               \
  do {                                                                                       \
    rev_trip<CAR, TAB, PRED, ODD, GRAD, UNIT>(KK, nu, A.h2, thr, paccg, naccg, chk, A.fwd_ok, \
                                              PRED ? TA : A.T, A.acc, A.sg, A.s, A.h2g, A.t,  \
                                              A.code, A.ok);                                 \
    rev_trip<CAR, TAB, PRED, ODD, GRAD, UNIT>(KK, nu, B.h2, thr, paccg, naccg, chk, B.fwd_ok, \
                                              PRED ? TB : B.T, B.acc, B.sg, B.s, B.h2g, B.t,  \
                                              B.code, B.ok);                                 \
  } while (0)
  for (; kr > ktab; kr--) BJP_REV(false, false, true, -1, false, kr);   // beyond the table
  for (; kr > (int)Tmin; kr--) BJP_REV(false, true, true, -1, false, kr);   // tail: predicated
  if (kr >= 1 && !(kr & 1)) {                                // align: pairs start at odd k
    BJP_REV(false, true, false, 0, false, kr);
    kr--;
  }
  if (accg == 1.0) {                                         // the default seed (uniform branch)
    for (; kr >= 2; kr -= 2) {
      BJP_REV(false, true, false, 1, true, kr);
      BJP_REV(false, true, false, 0, true, kr - 1);
    }
  }
  for (; kr >= 2; kr -= 2) {
    BJP_REV(false, true, false, 1, false, kr);
    BJP_REV(false, true, false, 0, false, kr - 1);
  }
  if (kr == 1) BJP_REV(false, true, false, 1, false, 1);
#undef BJP_REV
  if (chk && A.fwd_ok && !A.ok && !A.code) A.code = RL_ERR_POSTCONDITION;
  if (chk && B.fwd_ok && !B.ok && !B.code) B.code = RL_ERR_POSTCONDITION;
  oa = bjp_epilogue<GRAD>(A, nu, tol, accg, chk);
  ob = bjp_epilogue<GRAD>(B, nu, tol, accg, chk);
}

constexpr int BJ_RUN = 0, BJ_GRAD = 1, BJ_HESS = 2;

template <int MODE>
__global__ void __launch_bounds__(BJ_BLOCK, MODE == 2 ? 2 : BJ_MINB) k_besselj(
    int nu, const double *__restrict__ zin, long long n, double thr, double tol, double seed,
    long long max_trips, int chk, const double *__restrict__ out_in, double sign,
    double *__restrict__ Jout, double *__restrict__ dzout, uint8_t *__restrict__ fail,
    unsigned long long *counters, double sfloor, double *__restrict__ d2out) {
  constexpr bool GRAD = MODE >= BJ_GRAD;
  const int ktab = BJ_KP - 1;
  // trip cap: -1 = the prologue alone exceeds the reference's max_steps
  const int kfuel = (int)(max_trips < 0 ? -1 : (max_trips < (1LL << 30) ? max_trips : (1LL << 30)));
  __shared__ int s_hist[BJ_NB];
  __shared__ int s_wsum[BJ_WARPS];
  __shared__ int s_round;
  extern __shared__ __align__(16) double bj_dyn[];     // BJ_SMEM bytes
  double *s_zin = bj_dyn;                              // cp.async target: next chunk's z
  double *s_z = s_zin + BJ_C;
  double *s_J = s_z + BJ_C;
  double *s_dz = s_J + BJ_C;
  double *s_d2 = s_dz + BJ_C;                          // MODE 2 only
  uint16_t *s_idx = reinterpret_cast<uint16_t *>(s_d2 + (MODE == BJ_HESS ? BJ_C : 0));
  uint8_t *s_fail = reinterpret_cast<uint8_t *>(s_idx + BJ_C);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < BJ_EXPN * BJ_EXPREP; i += BJ_BLOCK) s_exp2tab[i] = g_exp2tab[i / BJ_EXPREP];
  for (int k = tid; k < BJ_KP; k += BJ_BLOCK)
    s_logpair[k] = make_double2(logi(k), k + nu >= 0 ? logi(k + nu) : __longlong_as_double(0x7ff8000000000000ULL));
  unsigned long long trips_sum = 0, nfail = 0;
  // z chunks are prefetched into shared memory with cp.async one chunk
  // ahead, so the DRAM latency of the next chunk hides behind this one's
  // series work
  const unsigned zin_s = (unsigned)__cvta_generic_to_shared(s_zin);
  auto prefetch = [&](long long b) {
    if (b >= n) return;
    const int c = (int)(n - b < BJ_C ? n - b : BJ_C);
#pragma unroll
    for (int m = 0; m < BJ_M; m++) {
      const int e = m * BJ_BLOCK + tid;
      if (e < c)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(zin_s + 8u * e),
                     "l"(zin + b + e) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch((long long)blockIdx.x * BJ_C);

  for (long long base = (long long)blockIdx.x * BJ_C; base < n;
       base += (long long)gridDim.x * BJ_C) {
    const int cnt = (int)(n - base < BJ_C ? n - base : BJ_C);
#ifdef BJ_PHASES
    if ((threadIdx.x & 31) == 0) s_bj_t[threadIdx.x >> 5] = clock64();
#endif
    // 1. bucket histogram (rank within bucket from the atomic)
    for (int b = tid; b < BJ_NB; b += BJ_BLOCK) s_hist[b] = 0;
    if (tid == 0) s_round = 0;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double zr[BJ_M];
    int key[BJ_M], rnk[BJ_M];
#pragma unroll
    for (int m = 0; m < BJ_M; m++) {
      const int e = m * BJ_BLOCK + tid;
      if (e < cnt) {
        zr[m] = s_zin[e];                              // each thread reads what it copied
        key[m] = zbucket(zr[m]);
        rnk[m] = atomicAdd(&s_hist[key[m]], 1);
      }
    }
    __syncthreads();
    prefetch(base + (long long)gridDim.x * BJ_C);
    BJ_MARK(0);
    // 2. exclusive scan of the 256 buckets (one per thread)
    {
      const int v = s_hist[tid];
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      __syncthreads();
      int off = 0;
#pragma unroll
      for (int w = 0; w < BJ_WARPS; w++) off += w < warp ? s_wsum[w] : 0;
      __syncthreads();
      s_hist[tid] = off + x - v;
    }
    __syncthreads();
    BJ_MARK(1);
    // 3. scatter into z order
#pragma unroll
    for (int m = 0; m < BJ_M; m++) {
      const int e = m * BJ_BLOCK + tid;
      if (e < cnt) {
        const int pos = s_hist[key[m]] + rnk[m];
        s_z[pos] = zr[m];
        s_idx[pos] = (uint16_t)e;
      }
    }
    __syncthreads();
    BJ_MARK(2);
    // 4. rounds of 32 z-neighbours, handed out dynamically from the largest z
    //    down (longest first), so the block's warps reach the barrier together
    //    (the next round's ticket is drawn one round ahead, off the
    //    critical path)
    constexpr int RW = (BJ_PAIR && MODE != BJ_HESS) ? 64 : 32;  // elements per warp round
    const int nrounds = (cnt + RW - 1) / RW;
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(&s_round, 1);
#pragma unroll 1
    for (;;) {
      const int got = __shfl_sync(FULL_MASK, ticket, 0);
      if (got >= nrounds) break;
      if (lane == 0) ticket = atomicAdd(&s_round, 1);
      const int r = nrounds - 1 - got;
#if BJ_PAIR
      if (MODE != BJ_HESS) {
        BJS A, B;
        const int pa = r * 64 + 2 * lane, pb = pa + 1;
        A.valid = pa < cnt;
        B.valid = pb < cnt;
        if (!__any_sync(FULL_MASK, A.valid)) continue;
        A.z = A.valid ? s_z[pa] : 1.0;
        B.z = B.valid ? s_z[pb] : 1.0;
        BJOut oa, ob;
        besselj_pair<GRAD>(A, B, nu, thr, tol, seed, ktab, kfuel, chk, sfloor, oa, ob);
        if (__any_sync(FULL_MASK, oa.bad || ob.bad)) {          // |exp arg| >= 708 somewhere
          const BJOut ca =
              besselj_element<true, GRAD>(A.z, oa.bad, nu, thr, tol, seed, ktab, kfuel, chk, sfloor);
          if (oa.bad) oa = ca;
          const BJOut cb =
              besselj_element<true, GRAD>(B.z, ob.bad, nu, thr, tol, seed, ktab, kfuel, chk, sfloor);
          if (ob.bad) ob = cb;
        }
        auto put = [&](int pos, bool valid, const BJOut &o) {
          if (!valid) return;
          const int oi = s_idx[pos];
          s_J[oi] = o.J;
          s_dz[oi] = o.dz;
          s_fail[oi] = (uint8_t)o.code;
          if (!o.code) trips_sum += (unsigned long long)o.T;   // trips of the elements that succeed
          nfail += o.code != 0;
        };
        put(pa, A.valid, oa);
        put(pb, B.valid, ob);
        continue;
      }
#endif
      const int pos = r * 32 + lane;
      const bool valid = pos < cnt;
      if (__any_sync(FULL_MASK, valid)) {
        const double z = valid ? s_z[pos] : 1.0;
        if (MODE == BJ_HESS) {
          BJHOut o = besselj_hess_element<false>(z, valid, nu, thr, tol, seed, kfuel, chk, sfloor);
          if (__any_sync(FULL_MASK, o.bad)) {
            const BJHOut c = besselj_hess_element<true>(z, o.bad, nu, thr, tol, seed, kfuel, chk,
                                                        sfloor);
            if (o.bad) o = c;
          }
          if (valid) {
            const int oi = s_idx[pos];
            s_J[oi] = o.J;
            s_dz[oi] = o.dz;
            s_d2[oi] = o.d2;
            s_fail[oi] = (uint8_t)o.code;
            if (!o.code) trips_sum += (unsigned long long)o.T;   // trips of the elements that succeed
            nfail += o.code != 0;
          }
          continue;
        }
        BJOut o = besselj_element<false, GRAD>(z, valid, nu, thr, tol, seed, ktab, kfuel, chk,
                                               sfloor);
        if (__any_sync(FULL_MASK, o.bad)) {              // |exp arg| >= 708 somewhere
          const BJOut c =
              besselj_element<true, GRAD>(z, o.bad, nu, thr, tol, seed, ktab, kfuel, chk, sfloor);
          if (o.bad) o = c;
        }
        if (valid) {
          const int oi = s_idx[pos];
          s_J[oi] = o.J;
          s_dz[oi] = o.dz;
          s_fail[oi] = (uint8_t)o.code;
          if (!o.code) trips_sum += (unsigned long long)o.T;     // trips of the elements that succeed
          nfail += o.code != 0;
        }
      }
    }
    BJ_MARK(3);
    __syncthreads();
    BJ_MARK(4);
    // 5. coalesced stores in the original order (TMA bulk stores of s_J /
    //    s_dz / s_fail measured no faster: the kernel is throughput-bound, the
    //    warps' store time moved to the next chunk's wait)
#pragma unroll
    for (int m = 0; m < BJ_M; m++) {
      const int e = m * BJ_BLOCK + tid;
      if (e < cnt) {
        if (GRAD) {
          __stcs(Jout + base + e, s_J[e]);
          __stcs(dzout + base + e, s_dz[e]);
          if (MODE == BJ_HESS) __stcs(d2out + base + e, s_d2[e]);
        } else {
          // out! += acc (run) / out! -= acc (uncall): one IEEE add, like the reference
          const double o0 = out_in ? __ldcs(out_in + base + e) : 0.0;
          __stcs(Jout + base + e, sign > 0 ? o0 + s_J[e] : o0 - s_J[e]);
        }
        fail[base + e] = s_fail[e];
      }
    }
    __syncthreads();
    BJ_MARK(5);
  }
  block_add_counters<BJ_BLOCK>(trips_sum, nfail, counters);
}

#ifdef BJ_PHASES
extern "C" int rl_debug_bj_phases(unsigned long long *out16) {  // timing-only builds
  cudaMemcpyFromSymbol(out16, g_bj_phase, 16 * sizeof(unsigned long long));
  static const unsigned long long zero[16] = {0};
  return (int)cudaMemcpyToSymbol(g_bj_phase, zero, sizeof zero);
}
#endif

static int upload_logtab() {
  static double tab[LOGTAB_N];
  tab[0] = -INFINITY;
  for (int i = 1; i < LOGTAB_N; i++) tab[i] = log((double)i);
  return cuda_status(cudaMemcpyToSymbol(c_logtab, tab, sizeof tab), "upload log table");
}

int besselj_tables_init() { return upload_logtab(); }

template <int MODE>
static int launch_besselj_t(int32_t nu, const double *z, int64_t n, double thr, double tol,
                            double seed, int64_t max_trips, int32_t invcheck,
                            const double *out_in, double sign, double *J, double *dJdz,
                            double *d2, uint8_t *fail, unsigned long long *counters,
                            cudaStream_t st) {
  int rc = ensure_device_tables();
  if (rc) return rc;
  if (n == 0) return RL_OK;
  const int smem = BJ_SMEM + (MODE == BJ_HESS ? BJ_C * 8 : 0);
  int blocks_per_sm = 0;
  rc = smem_attr((const void *)k_besselj<MODE>, smem, "smem attr");
  if (rc) return rc;
  rc = occupancy(&blocks_per_sm, (const void *)k_besselj<MODE>, BJ_BLOCK, smem, "occupancy");
  if (rc) return rc;
  const long long want = (n + BJ_C - 1) / BJ_C;
  const long long cap = (long long)sm_count() * (blocks_per_sm > 0 ? blocks_per_sm : 1);
  const int grid = (int)(want < cap ? want : cap);
  // FAST-flavour safety bound (besselj_element): log(thr) - 2 log(kfuel + |nu| + 1)
  const double kfuel = (double)(max_trips < 0 ? 0 : (max_trips < (1LL << 30) ? max_trips : (1LL << 30)));
  const double sfloor = log(thr) - 2.0 * log(kfuel + fabs((double)nu) + 1.0);
  k_besselj<MODE><<<grid, BJ_BLOCK, smem, st>>>(nu, z, n, thr, tol, seed, max_trips,
                                                invcheck ? 1 : 0, out_in, sign, J, dJdz, fail,
                                                counters, sfloor, d2);
  return cuda_status(cudaGetLastError(), "k_besselj launch");
}

int launch_besselj(int32_t nu, const double *z, int64_t n, double thr, double tol, double seed,
                   int64_t max_trips, int32_t invcheck, double *J, double *dJdz, uint8_t *fail,
                   unsigned long long *counters, cudaStream_t st) {
  if (n < 0 || (n > 0 && (!z || !J || !dJdz || !fail)) || max_trips < -1)
    return set_error(RL_ERR_INVALID, "rl_besselj_grad_f64: bad argument");
  return launch_besselj_t<BJ_GRAD>(nu, z, n, thr, tol, seed, max_trips, invcheck, nullptr, 1.0,
                                   J, dJdz, nullptr, fail, counters, st);
}

int launch_besselj_hess(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, double *d2Jdz2, uint8_t *fail,
                        unsigned long long *counters, cudaStream_t st) {
  if (n < 0 || (n > 0 && (!z || !J || !dJdz || !d2Jdz2 || !fail)) || max_trips < -1)
    return set_error(RL_ERR_INVALID, "rl_besselj_hess_f64: bad argument");
  return launch_besselj_t<BJ_HESS>(nu, z, n, thr, tol, seed, max_trips, invcheck, nullptr, 1.0,
                                   J, dJdz, d2Jdz2, fail, counters, st);
}

int launch_besselj_run(int32_t nu, const double *z, int64_t n, double thr, double tol,
                       int64_t max_trips, int32_t invcheck, int32_t direction,
                       const double *out_in, double *out, uint8_t *fail,
                       unsigned long long *counters, cudaStream_t st) {
  if (n < 0 || (n > 0 && (!z || !out || !fail)) || max_trips < -1 ||
      (direction != 1 && direction != -1))
    return set_error(RL_ERR_INVALID, "rl_besselj_run_f64: bad argument");
  return launch_besselj_t<BJ_RUN>(nu, z, n, thr, tol, 0.0, max_trips, invcheck, out_in,
                                  (double)direction, out, nullptr, nullptr, fail, counters, st);
}

}  // namespace rl
