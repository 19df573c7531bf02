// seqsum.cuh — the reference's left-to-right binary64 accumulation
//     e_{j+1} = fl(e_j + t_j),  j = 0 .. M-1,  e_0 given
// evaluated EXACTLY (bit for bit the sequential result) by one CTA.
//
// The reference accumulates `err! += term` one statement at a time
// (interpreter.py:912-937, `_plus_minus_plain` numerics.py:296-339), and its
// primal-restoration check (autodiff.py:169-172) compares err! after the
// gradient sweep with its entry value: the residual is exactly the rounding
// of that sequential chain.  A dependent DADD chain of 4N+8 terms costs
// ~8 cycles a term on one thread (0.16 ms at N = 10^4), so the chain is
// parallelised instead, without changing a single rounding:
//
//  * while e_j and e_{j+1} stay in one binade [2^p, 2^(p+1)) of one sign,
//    e_j is a multiple of u = 2^(p-52) and fl(e_j + t_j) = e_j + rint(t_j/u) u
//    (no tie), so a run of such steps is one exact integer sum R and the run
//    moves e by the exact double R u;
//  * an approximate prefix S_j (block scan in binary64; |S_j - e_j| <= Delta,
//    a bound on both roundings) predicts each step's binade; a step whose
//    prediction is ambiguous (S within Delta of a power of two or of zero), a
//    tie, or a binade change becomes a single-term "breakpoint";
//  * each thread's run of terms compresses to a few chain values (exact run
//    shifts R u and breakpoint terms t_j); one thread folds the short chain
//    with true DADDs (e = fl(e + v)), giving every run's start value; a run
//    with more than SEQ_PER values (many binade changes, e.g. the first run
//    of a growing sum) is folded term by term instead;
//  * VERIFICATION: every thread re-walks its run with true DADDs from that
//    start and must land bit-exactly on the next run's start.  By induction
//    from e_0 every start is then the true sequential value — whatever the
//    predictions were.  Any mismatch (a wrong prediction, chain overflow)
//    falls back to the plain sequential loop, so the result is always the
//    sequential one; the fast path only decides how quickly it is reached.
#pragma once

#include <stdint.h>

namespace rl {

constexpr int SEQ_THREADS = 512;
constexpr int SEQ_PER = 8;        // chain values of one run (more: folded term by term)
constexpr int SEQ_CH = 16;        // terms per thread per staged chunk

struct SeqSmem {
  double chain[SEQ_THREADS * SEQ_PER];
  double pre[SEQ_THREADS * SEQ_PER + 1];
  double stage[2][SEQ_THREADS][SEQ_CH + 1];  // warp-transposed term chunks, double-buffered
  int off[SEQ_THREADS + 1];
  int mk_pos[SEQ_THREADS];        // chain slot of each term-by-term run, in order
  int mk_run[SEQ_THREADS];
  double wsum[SEQ_THREADS / 32];
  int wcnt[SEQ_THREADS / 32];
  int flag;
};

__device__ __forceinline__ double seq_pow2(int k) {  // 2^k, k in [-1022, 1023]
  return __longlong_as_double((long long)(k + 1023) << 52);
}

// binade p of s (|s| in [2^p, 2^(p+1))) when it is certain under an error
// of delta, else INT_MIN
__device__ __forceinline__ int seq_binade(double s, double delta) {
  const double a = fabs(s);
  const int p = (int)((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
  if (!(a > delta) || p < -960 || p > 1000) return -0x7fffffff;
  if (!(a - seq_pow2(p) > delta) || !(seq_pow2(p + 1) - a > delta)) return -0x7fffffff;
  return p;
}

// exclusive block scan of one double per thread (approximate), returns the
// thread's exclusive prefix; *total = block total
__device__ __forceinline__ double seq_scan_d(double v, double *total, SeqSmem &sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    double s = lane < SEQ_THREADS / 32 ? sm.wsum[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < SEQ_THREADS / 32) sm.wsum[lane] = s;
  }
  __syncthreads();
  const double base = w ? sm.wsum[w - 1] : 0.0;
  *total = sm.wsum[SEQ_THREADS / 32 - 1];
  __syncthreads();
  return base + x - v;
}

__device__ __forceinline__ int seq_scan_i(int v, int *total, SeqSmem &sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.wcnt[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < SEQ_THREADS / 32 ? sm.wcnt[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < SEQ_THREADS / 32) sm.wcnt[lane] = s;
  }
  __syncthreads();
  const int base = w ? sm.wcnt[w - 1] : 0;
  *total = sm.wcnt[SEQ_THREADS / 32 - 1];
  __syncthreads();
  return base + x - v;
}

__device__ __forceinline__ void seq_cp8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void seq_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void seq_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Calls f(j, t[j]) for j = lo .. lo + len - 1 of the calling thread's run, in
// order.  Each thread's run is contiguous, so direct loads would touch 32
// cache lines per warp instruction; instead the warp copies SEQ_CH-term
// chunks of all 32 runs (two runs' chunks per instruction, coalesced) into
// shared memory with cp.async, transposed, one chunk ahead of the one being
// consumed.  All threads of the warp must call it (uniform trip count over
// the block's longest run); a thread with nothing to walk passes len = 0.
template <class F>
__device__ __forceinline__ void seq_walk(const double *__restrict__ t, long long lo, int len,
                                         int maxlen, SeqSmem &sm, F &&f) {
  const int lane = threadIdx.x & 31, wbase = threadIdx.x & ~31;
  const int half = lane >> 4, i = lane & 15;
  if (!__any_sync(0xffffffffu, len > 0)) return;  // warp-uniform
  auto issue = [&](int c, int b) {
#pragma unroll
    for (int q2 = 0; q2 < 32; q2 += 2) {
      const int q = q2 + half;
      const long long lo_q = __shfl_sync(0xffffffffu, lo, q);
      const int len_q = __shfl_sync(0xffffffffu, len, q);
      if (c + i < len_q) seq_cp8(&sm.stage[b][wbase + q][i], t + lo_q + c + i);
    }
    seq_commit();
  };
  issue(0, 0);
  int b = 0;
  for (int c = 0; c < maxlen; c += SEQ_CH, b ^= 1) {
    if (c + SEQ_CH < maxlen) {
      issue(c + SEQ_CH, b ^ 1);
      seq_wait<1>();
    } else {
      seq_wait<0>();
    }
    __syncwarp();
    const int n = min(SEQ_CH, len - c);
#pragma unroll
    for (int k = 0; k < SEQ_CH; k++)
      if (k < n) f(lo + c + k, sm.stage[b][threadIdx.x][k]);
    __syncwarp();
  }
}

// rint(q) for |q| < 2^51 by the 1.5 * 2^52 shifter (round half to even)
__device__ __forceinline__ double seq_rint(double q) {
  return __dsub_rn(__dadd_rn(q, 0x1.8p52), 0x1.8p52);
}

// The whole CTA (SEQ_THREADS threads) evaluates the chain over the device
// array t[0, M).  Thread 0 returns e_mark = e_{mark} (the value before term
// `mark`, mark in [0, M]) and e_final = e_M; the return value is 1 when the
// parallel path verified, 0 when the sequential fallback ran (or was forced).
__device__ int seq_sum_block(const double *__restrict__ t, long long M, double e0, long long mark,
                             int force_serial, SeqSmem &sm, double *e_mark, double *e_final,
                             double *diag = nullptr) {
  const int r = threadIdx.x;
  const long long lo = M * r / SEQ_THREADS, hi = M * (r + 1) / SEQ_THREADS;
  const int len = (int)(hi - lo), maxlen = (int)((M + SEQ_THREADS - 1) / SEQ_THREADS);
#ifdef SEQ_DIAG   // phase timestamps (tools/seq_probe.py with a SEQ_DIAG build)
#define SEQ_TICK(n)                                          \
  do {                                                       \
    __syncthreads();                                         \
    if (diag && r == 0) diag[n] = (double)clock64();         \
  } while (0)
#else
#define SEQ_TICK(n) (void)diag
#endif
  SEQ_TICK(0);
  if (r == 0) sm.flag = force_serial;
  // walk 1: run sums (approximate) and the magnitude bound
  double s = 0.0, sa = 0.0;
  seq_walk(t, lo, len, maxlen, sm, [&](long long, double x) {
    s = s + x;
    sa = sa + fabs(x);
  });
  SEQ_TICK(1);
  double tot;
  const double S0 = e0 + seq_scan_d(s, &tot, sm);
  double atot;
  (void)seq_scan_d(sa, &atot, sm);
  // |S_j - e_j| <= (M + 64) 2^-52 (|e0| + sum |t|): the sequential chain's
  // rounding plus the scan's (generous; only speed depends on it)
  const double delta = ((double)M + 64.0) * 0x1p-51 * (fabs(e0) + atot);
  SEQ_TICK(2);
  // walk 2: compress the run into chain values.  A step is "simple" when
  // its approximate pre- and post-values lie in the tracked binade
  // [2^p + delta, 2^(p+1) - delta] of the tracked sign and t/u is no tie and
  // below 2^51; simple steps accumulate R = sum rint(t/u) (an integer below
  // 2^53 in magnitude: exact in binary64); any other step is a breakpoint
  // (emitted as its own term) after which the binade is re-derived.
  double *slot = sm.pre + r * SEQ_PER;      // staging (pre is rebuilt after)
  int cnt = 0;
  bool over = false;
  int p1 = -0x7fffffff;                      // binade/shift of the run's single piece
  double R1 = 0.0;
  {
    double S = S0;
    int p = seq_binade(S, delta);
    double blo = 0.0, bhi = -1.0, sc = 1.0;
    bool pos = S > 0.0;
    auto track = [&](double v) {
      p = seq_binade(v, delta);
      pos = v > 0.0;
      if (p != -0x7fffffff) {
        blo = seq_pow2(p) + delta;
        bhi = seq_pow2(p + 1) - delta;
        sc = seq_pow2(52 - p);
      } else {
        blo = 0.0;
        bhi = -1.0;                          // nothing is inside
      }
    };
    track(S);
    double R = 0.0;
    bool act = false;
    int pact = 0;
    auto emit = [&](double v) {
      if (cnt < SEQ_PER) slot[cnt] = v;
      else over = true;
      cnt++;
    };
    seq_walk(t, lo, len, maxlen, sm, [&](long long, double x) {
      const double S1 = S + x;
      const double a1 = fabs(S1);
      const double q = x * sc;
      const double rq = seq_rint(q);
      const bool simple = a1 > blo && a1 < bhi && ((S1 > 0.0) == pos) && fabs(q) < 0x1p51 &&
                          fabs(q - rq) != 0.5;
      if (simple) {
        R = act ? R + rq : rq;
        if (!act) pact = p;
        act = true;
      } else {
        if (act) {
          emit(R * seq_pow2(pact - 52));
          p1 = pact;
          R1 = R;
          act = false;
        }
        emit(x);
        p1 = -0x7fffffff;
        track(S1);
      }
      S = S1;
    });
    if (act) {
      emit(R * seq_pow2(pact - 52));
      p1 = pact;
      R1 = R;
    }
  }
  SEQ_TICK(3);
  // A warp whose 32 runs are each one exact shift in one common binade
  // moves e by the exact sum of their shifts: it enters the chain as ONE
  // value, and its runs' starts are the warp's start plus exact prefix
  // shifts (walk 3 verifies them like every other start).
  const int lane = r & 31;
  const bool single = cnt == 1 && !over && p1 != -0x7fffffff;
  const int pw = __shfl_sync(0xffffffffu, p1, 0);
  const bool uni = __all_sync(0xffffffffu, single && p1 == pw);
  double Rx = 0.0;                           // exclusive prefix of R1 within the warp
  if (uni) {
    double x = R1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;                 // integers below 2^53: exact
    }
    Rx = x - R1;
    const double tw = __shfl_sync(0xffffffffu, x, 31);
    cnt = lane == 0 ? 1 : 0;
    if (lane == 0) slot[0] = tw * seq_pow2(pw - 52);
  }
  if (over) cnt = 1;                          // one placeholder slot: folded term by term
  int ntot, nmk;
  const int off = seq_scan_i(cnt, &ntot, sm);
  const int mki = seq_scan_i(over ? 1 : 0, &nmk, sm);
  if (!over)
    for (int i = 0; i < cnt; i++) sm.chain[off + i] = slot[i];
  else {
    sm.mk_pos[mki] = off;
    sm.mk_run[mki] = r;
  }
  sm.off[r] = uni ? __shfl_sync(0xffffffffu, off, 0) : off;
  if (r == 0) sm.off[SEQ_THREADS] = ntot;
  SEQ_TICK(4);
  __syncthreads();
  // the chain, one thread, true DADDs
  if (r == 0 && !sm.flag) {
    double e = e0;
    int k = 0;
    for (int i = 0; i <= nmk; i++) {
      const int end = i < nmk ? sm.mk_pos[i] : ntot;
      for (; k + 8 <= end; k += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = sm.chain[k + q];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          sm.pre[k + q] = e;
          e = e + v[q];
        }
      }
      for (; k < end; k++) {
        sm.pre[k] = e;
        e = e + sm.chain[k];
      }
      if (i < nmk) {                            // a run folded term by term
        sm.pre[k] = e;
        const int rr = sm.mk_run[i];
        const long long a = M * rr / SEQ_THREADS, b = M * (rr + 1) / SEQ_THREADS;
        long long j = a;
        for (; j + 4 <= b; j += 4) {
          const double t0 = t[j], t1 = t[j + 1], t2 = t[j + 2], t3 = t[j + 3];
          e = e + t0;
          e = e + t1;
          e = e + t2;
          e = e + t3;
        }
        for (; j < b; j++) e = e + t[j];
        k++;
      }
    }
    sm.pre[ntot] = e;
  }
  __syncthreads();
  // run starts: the chain value at the run's slot, plus (uniform warps) the
  // exact prefix shift within the warp
  {
    double st = sm.pre[sm.off[r]];
    if (uni) st = st + Rx * seq_pow2(pw - 52);
    sm.chain[r] = st;                           // (the chain values are consumed)
  }
  __syncthreads();
  SEQ_TICK(5);
  // walk 3: verify every run from its start with true DADDs
  bool ok = true;
  if (!sm.flag) {
    double e = sm.chain[r];
    double em = 0.0;
    bool has_mark = false;
    seq_walk(t, lo, len, maxlen, sm, [&](long long j, double x) {
      if (j == mark) {
        em = e;
        has_mark = true;
      }
      e = e + x;
    });
    if (has_mark) *e_mark = em;                 // the owning thread (shared result slot)
    if (mark == M && r == SEQ_THREADS - 1) *e_mark = e;
    if (r == SEQ_THREADS - 1) *e_final = e;
    else ok = __double_as_longlong(e) == __double_as_longlong(sm.chain[r + 1]);
  }
  if (!ok) sm.flag = 1;
  SEQ_TICK(6);
  if (diag && r == 0) diag[8] = nmk + 1000.0 * ntot;
  __syncthreads();
  if (!sm.flag) return 1;
  if (r == 0) {                               // sequential fallback
    double e = e0;
    for (long long j = 0; j < M; j++) {
      if (j == mark) *e_mark = e;
      e = e + t[j];
    }
    if (mark == M) *e_mark = e;
    *e_final = e;
  }
  __syncthreads();
  return 0;
}

}  // namespace rl
