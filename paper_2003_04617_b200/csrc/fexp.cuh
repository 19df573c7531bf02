// fexp.cuh — table-driven binary64 exp for the series kernels.
//
// e^x = 2^m * 2^(i/64) * e^r,  x = (64 m + i) ln2/64 + r,  |r| <= ln2/128.
// 2^(i/64) is stored as a hi + lo pair (exact to ~106 bits, generated with
// mpmath); e^r - 1 is its degree-6 Taylor polynomial (truncation 3e-20).
// Result = T_hi + fma(T_hi, p, T_lo): one final rounding, so the error is
// 0.5 ulp + O(2^-60) — correctly rounded except within ~1e-3 ulp of a
// rounding boundary (the host libm exp CPython calls, which the oracle
// reproduces, is correctly rounded in practice; tests/test_fexp.py
// measures the agreement).  12 FP64 instructions (21 flops) and one 16-byte
// table read, against ~18.5 instructions (31.5 flops, profiles/
// fp64_weights.json) for libdevice exp.  Arguments outside (-708, 708)
// (subnormal results, overflow) take libdevice's exp.
//
// Host-compilable (tests/test_fexp.py builds it with g++ and compares bit
// patterns against glibc on 10^7 arguments).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "exp2tab_1024.inc"
#include "exp2tab_256.inc"

#ifdef __CUDACC__
#define RL_HD __host__ __device__ __forceinline__
#define RL_HDM __host__ __device__ __forceinline__
#else
#define RL_HD static inline
#define RL_HDM inline
struct double2 {
  double x, y;
};
#endif

namespace rl {

struct alignas(16) Exp2Tab {
  double hi, lo;
};

#define RL_EXP2_TABLE_INIT { \
    {0x1.0000000000000p+0, 0x0.0p+0}, \
    {0x1.02c9a3e778061p+0, -0x1.19083535b085dp-56}, \
    {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55}, \
    {0x1.0874518759bc8p+0, 0x1.186be4bb284ffp-57}, \
    {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54}, \
    {0x1.0e3ec32d3d1a2p+0, 0x1.03a1727c57b53p-59}, \
    {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54}, \
    {0x1.1429aaea92de0p+0, -0x1.32fbf9af1369ep-54}, \
    {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55}, \
    {0x1.1a35beb6fcb75p+0, 0x1.e5b4c7b4968e4p-55}, \
    {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54}, \
    {0x1.2063b88628cd6p+0, 0x1.dc775814a8495p-55}, \
    {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54}, \
    {0x1.26b4565e27cddp+0, 0x1.2bd339940e9d9p-55}, \
    {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55}, \
    {0x1.2d285a6e4030bp+0, 0x1.0024754db41d5p-54}, \
    {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55}, \
    {0x1.33c08b26416ffp+0, 0x1.32721843659a6p-54}, \
    {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54}, \
    {0x1.3a7db34e59ff7p+0, -0x1.5e436d661f5e3p-56}, \
    {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55}, \
    {0x1.4160a21f72e2ap+0, -0x1.ef3691c309278p-58}, \
    {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59}, \
    {0x1.486a2b5c13cd0p+0, 0x1.3c1a3b69062f0p-56}, \
    {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56}, \
    {0x1.4f9b2769d2ca7p+0, -0x1.4b309d25957e3p-54}, \
    {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55}, \
    {0x1.56f4736b527dap+0, 0x1.9bb2c011d93adp-54}, \
    {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54}, \
    {0x1.5e76f15ad2148p+0, 0x1.ba6f93080e65ep-54}, \
    {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54}, \
    {0x1.6623882552225p+0, -0x1.bb60987591c34p-54}, \
    {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54}, \
    {0x1.6dfb23c651a2fp+0, -0x1.bbe3a683c88abp-57}, \
    {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55}, \
    {0x1.75feb564267c9p+0, -0x1.0245957316dd3p-54}, \
    {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55}, \
    {0x1.7e2f336cf4e62p+0, 0x1.05d02ba15797ep-56}, \
    {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54}, \
    {0x1.868d99b4492edp+0, -0x1.fc6f89bd4f6bap-54}, \
    {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54}, \
    {0x1.8f1ae99157736p+0, 0x1.5cc13a2e3976cp-55}, \
    {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57}, \
    {0x1.97d829fde4e50p+0, -0x1.d185b7c1b85d1p-54}, \
    {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56}, \
    {0x1.a0c667b5de565p+0, -0x1.359495d1cd533p-54}, \
    {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54}, \
    {0x1.a9e6b5579fdbfp+0, 0x1.0fac90ef7fd31p-54}, \
    {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54}, \
    {0x1.b33a2b84f15fbp+0, -0x1.2805e3084d708p-57}, \
    {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56}, \
    {0x1.bcc1e904bc1d2p+0, 0x1.23dd07a2d9e84p-55}, \
    {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55}, \
    {0x1.c67f12e57d14bp+0, 0x1.2884dff483cadp-54}, \
    {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56}, \
    {0x1.d072d4a07897cp+0, -0x1.cbc3743797a9cp-54}, \
    {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55}, \
    {0x1.da9e603db3285p+0, 0x1.c2300696db532p-54}, \
    {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54}, \
    {0x1.e502ee78b3ff6p+0, 0x1.39e8980a9cc8fp-55}, \
    {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54}, \
    {0x1.efa1bee615a27p+0, 0x1.dc7f486a4b6b0p-54}, \
    {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54}, \
    {0x1.fa7c1819e90d8p+0, 0x1.74853f3a5931ep-55}, \
  }

constexpr double EXP_INV_LN2_64 = 0x1.71547652b82fep+6;
constexpr double EXP_LN2_64_HI = 0x1.62e42fefa3000p-7;
constexpr double EXP_LN2_64_LO = 0x1.3de6af278ece6p-48;
constexpr double EXP_SHIFT = 0x1.8p52;

// Constants as a struct so that device code can keep them in __constant__
// memory (they become DFMA constant-bank operands instead of immediates
// that need two uniform moves each).
struct ExpConsts {
  double inv_ln2_64, ln2_64_hi_neg, ln2_64_lo_neg, shift, c6, c5, c4, c3, c2;
};
#define RL_EXP_CONSTS_INIT \
  {rl::EXP_INV_LN2_64, -rl::EXP_LN2_64_HI, -rl::EXP_LN2_64_LO, rl::EXP_SHIFT, 1.0 / 720.0, 1.0 / 120.0, \
   1.0 / 24.0, 1.0 / 6.0, 0.5}

// `tab` must point to shared memory in device code.
RL_HD double fexp_core(double x, const Exp2Tab *tab, const ExpConsts &K) {
  // x in (-708, 708): the caller guarantees the range
  const double t = fma(x, K.inv_ln2_64, K.shift);
  int64_t tb;
  memcpy(&tb, &t, 8);
  const int j = (int)(int32_t)(uint32_t)tb;          // round(x * 64 / ln2)
  const double jd = t - K.shift;
  double r = fma(jd, K.ln2_64_hi_neg, x);
  r = fma(jd, K.ln2_64_lo_neg, r);
  double q = fma(K.c6, r, K.c5);
  q = fma(q, r, K.c4);
  q = fma(q, r, K.c3);
  q = fma(q, r, K.c2);
  const double r2 = r * r;
  const double p = fma(q, r2, r);                    // e^r - 1
#if defined(__CUDA_ARCH__)
  // 32-bit shared-window address: one LDS.128, no generic-address setup
  double ehi, elo;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];"
      : "=d"(ehi), "=d"(elo)
      : "r"((unsigned)__cvta_generic_to_shared(tab) + (unsigned)((j & 63) << 4)));
  const Exp2Tab e{ehi, elo};
#else
  const Exp2Tab e = tab[j & 63];
#endif
  double res = e.hi + fma(e.hi, p, e.lo);
  // scale by 2^(j >> 6): integer add into the exponent field
  int64_t rb;
  memcpy(&rb, &res, 8);
  rb += (int64_t)(j >> 6) * ((int64_t)1 << 52);
  memcpy(&res, &rb, 8);
  return res;
}

// ---------------------------------------------------------------------------
// 1024-entry variant: e^x = 2^m * 2^(i/1024) * e^r, |r| <= ln2/2048, so the
// degree-4 Taylor polynomial suffices (truncation 4e-20 relative): 10 FP64
// instructions and a 3-shorter dependency chain than the 64-entry form, for
// a 16 KB shared-memory table (exp2tab_1024.inc, tools/gen_exp_table.py).
// Error: 0.5 ulp + O(2^-64).
//
// Device form: the table must be a __shared__ array (its address is then an
// immediate of the LDS), and the 2^m scale is one integer add into the high
// word (SHF + LEA) instead of a 64-bit add.
struct ExpConsts1024 {
  double inv_ln2_n, ln2_n_hi_neg, ln2_n_lo_neg, shift, c4, c3, c2;
};
#define RL_EXP_CONSTS_1024_INIT \
  {RL_EXP_INV_LN2_1024, -RL_EXP_LN2_1024_HI, -RL_EXP_LN2_1024_LO, rl::EXP_SHIFT, 1.0 / 24.0, \
   1.0 / 6.0, 0.5}

// `tab(i)` returns entry i as a double2 {hi, lo}: device code passes an
// accessor of a static __shared__ array, so the load is one LDS with an
// immediate base (a generic pointer would cost a runtime base add).
template <class TabFn>
RL_HD double fexp1024(double x, TabFn tab, const ExpConsts1024 &K) {
  const double t = fma(x, K.inv_ln2_n, K.shift);
  int64_t tb;
  memcpy(&tb, &t, 8);
  const int j = (int)(int32_t)(uint32_t)tb;          // round(x * 1024 / ln2)
  const double jd = t - K.shift;
  double r = fma(jd, K.ln2_n_hi_neg, x);
  r = fma(jd, K.ln2_n_lo_neg, r);
  double q = fma(K.c4, r, K.c3);
  q = fma(q, r, K.c2);
  const double r2 = r * r;
  const double p = fma(q, r2, r);                    // e^r - 1
  const auto e = tab(j & 1023);
  const double res = e.x + fma(e.x, p, e.y);
  // scale by 2^m, m = j >> 10: integer add into the exponent field
#if defined(__CUDA_ARCH__)
  int hi;
  asm("{\n\t.reg .s32 m;\n\tshr.s32 m, %1, 10;\n\tmad.lo.s32 %0, m, 1048576, %2;\n\t}"
      : "=r"(hi)
      : "r"(j), "r"(__double2hiint(res)));
  return __hiloint2double(hi, __double2loint(res));
#else
  int64_t rb;
  memcpy(&rb, &res, 8);
  rb += (int64_t)(j >> 10) * ((int64_t)1 << 52);
  double out;
  memcpy(&out, &rb, 8);
  return out;
#endif
}

// 256-entry variant: |r| <= ln2/512, degree-5 polynomial (truncation 1e-20
// relative), 11 FP64 instructions.  The kernel stores the table replicated
// per lane-in-quarter-warp so that its 16-byte loads are bank-conflict free.
struct ExpConsts256 {
  double inv_ln2_n, ln2_n_hi_neg, ln2_n_lo_neg, shift, c5, c4, c3, c2;
};
#define RL_EXP_CONSTS_256_INIT \
  {RL_EXP_INV_LN2_256, -RL_EXP_LN2_256_HI, -RL_EXP_LN2_256_LO, rl::EXP_SHIFT, 1.0 / 120.0, \
   1.0 / 24.0, 1.0 / 6.0, 0.5}

template <class TabFn>
RL_HD double fexp256(double x, TabFn tab, const ExpConsts256 &K) {
  const double t = fma(x, K.inv_ln2_n, K.shift);
  int64_t tb;
  memcpy(&tb, &t, 8);
  const int j = (int)(int32_t)(uint32_t)tb;          // round(x * 256 / ln2)
  const double jd = t - K.shift;
  double r = fma(jd, K.ln2_n_hi_neg, x);
  r = fma(jd, K.ln2_n_lo_neg, r);
  double q = fma(K.c5, r, K.c4);
  q = fma(q, r, K.c3);
  q = fma(q, r, K.c2);
  const double r2 = r * r;
  const double p = fma(q, r2, r);                    // e^r - 1
  const auto e = tab(j & 255);
  const double res = e.x + fma(e.x, p, e.y);
#if defined(__CUDA_ARCH__)
  int hi;
  asm("{\n\t.reg .s32 m;\n\tshr.s32 m, %1, 8;\n\tmad.lo.s32 %0, m, 1048576, %2;\n\t}"
      : "=r"(hi)
      : "r"(j), "r"(__double2hiint(res)));
  return __hiloint2double(hi, __double2loint(res));
#else
  int64_t rb;
  memcpy(&rb, &res, 8);
  rb += (int64_t)(j >> 8) * ((int64_t)1 << 52);
  double out;
  memcpy(&out, &rb, 8);
  return out;
#endif
}

struct Exp2TabFn {
  const Exp2Tab *tab;
  RL_HDM double2 operator()(int i) const {
    double2 v;
    v.x = tab[i].hi;
    v.y = tab[i].lo;
    return v;
  }
};

RL_HD double fexp1024_core(double x, const Exp2Tab *tab, const ExpConsts1024 &K) {
  return fexp1024(x, Exp2TabFn{tab}, K);
}

RL_HD double fexp256_core(double x, const Exp2Tab *tab, const ExpConsts256 &K) {
  return fexp256(x, Exp2TabFn{tab}, K);
}

}  // namespace rl
