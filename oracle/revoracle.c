/*
 * revoracle.c — CPU ORACLE (test infrastructure; never shipped, never timed
 * as the product).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.
 *
 * A statement-by-statement restatement, in plain C, of what the reference
 * interpreter executes for `revlang.gradient(program, GradRequest(...))`
 * (autodiff.py:136-180) over the three benchmark programs in
 * paper_2003_04617_b200/programs/ (besselj, ba, gmm .rnl).  The pipeline is reproduced in full
 * — all four sweeps, with every reversibility check:
 *
 *   sweep 1  forward  R            (interpreter.py:424 run_function)
 *            out! += acc
 *   sweep 2  forward  R^-1         (uncompute, ancilla-release checks)
 *   sweep 3  gradient R            (~f in gradient_mode: GVar cells,
 *            out! -= acc            autodiff.py:162-167; reverser.py:86-163)
 *   sweep 4  gradient R^-1         (adjoint rules numerics.py:435-505)
 *   final    primal-restoration check values_close(.., tol) autodiff.py:169-172
 *
 * Arithmetic follows the reference operation by operation so that results
 * are bit-identical to CPython's (same libm; compile with
 * -ffp-contract=off, no fast-math):
 *   y += f(a)      t = f(a); y = y + t          numerics.py:296-339
 *   ULog y *= a    y.log_x = y.log_x + contrib  numerics.py:342-368
 *   adjoint        a.g = a.g + (sign*y.g)*p     numerics.py:419-486
 *                  sign = +1 when the executed (inverted) op is -=.
 *   ULog *= / /=   a.g += sign*y.g (ULog arg) or sign*y.g / a (float arg)
 *                                                numerics.py:489-505
 *   convert(ULog)  a.g += sign*y.g*exp(log_x)    numerics.py:447-456
 *   compare on ULog uses exp(log_x)              interpreter.py:_compare, values.py:114
 *   ancilla release |v - decl| <= tol (NaN passes), Int exact
 *                                                interpreter.py:365-395
 * For besselj and ba, gradient-mode forward sweeps only target fresh
 * ancillas whose cotangents are zero, so their adjoint accumulations add
 * (+/-)0 and are omitted; gmm's scratch arguments are handled in full.
 *
 * Error codes are include/revgpu.h's RL_ERR_*; the first failing check
 * stops the call exactly where the reference would raise.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/revgpu.h"

/* Python's math.exp raises OverflowError when a finite argument overflows. */
static int py_exp(double x, double *out) {
  double r = exp(x);
  if (isinf(r) && isfinite(x)) return RL_ERR_OVERFLOW;
  *out = r;
  return RL_OK;
}

/* values.s_log: RevDomainError unless x > 0 (values.py:365-372). */
#define PY_LOG(x, out)                              \
  do {                                              \
    double _x = (x);                                \
    if (!(_x > 0)) return RL_ERR_DOMAIN;            \
    (out) = log(_x);                                \
  } while (0)

#define TRY(e)                  \
  do {                          \
    int _rc = (e);              \
    if (_rc != RL_OK) return _rc; \
  } while (0)

/* ancilla release check (interpreter.py:738-745, _ancilla_residual :365-395) */
#define RELEASE_F(v, decl, tol)                            \
  do {                                                     \
    if (chk && fabs((v) - (decl)) > (tol)) return RL_ERR_DIRTY_ANCILLA; \
  } while (0)
#define RELEASE_I(v, decl)                                 \
  do {                                                     \
    if (chk && (v) != (decl)) return RL_ERR_DIRTY_ANCILLA; \
  } while (0)

/* =========================================================================
 * Bessel J_nu (programs/besselj.rnl)
 * ========================================================================= */

typedef struct {
  long k, kn;
  double lz, halfz, halfz2, s, acc; /* ULog cells hold log_x */
} bj_state;

typedef struct {
  double lz, halfz, halfz2, s, acc, z; /* cotangents (ULog ones in log space) */
} bj_grad;

/* The @routine block, forward (sweeps 1 and 3). */
static int bj_routine(bj_state *st, long nu, double z, double thr, long max_trips, int chk,
                      long *trips) {
  double t, lg;
  st->k = 0;
  st->kn = 0;
  st->lz = st->halfz = st->halfz2 = st->s = log(1.0); /* ulog(1.0) */
  st->acc = 0.0;
  PY_LOG(z, lg); /* lz *= convert(z) */
  st->lz = st->lz + lg;
  st->halfz = st->halfz + st->lz;         /* halfz *= lz */
  st->halfz = st->halfz - log(2.0);       /* halfz /= 2 */
  st->halfz2 = st->halfz2 + st->halfz;    /* halfz2 *= halfz (x2) */
  st->halfz2 = st->halfz2 + st->halfz;
  for (long i = 1; i <= nu; i++) {        /* for i = 1:1:nu */
    st->s = st->s + st->halfz;            /*   s *= halfz */
    st->s = st->s - log((double)i);       /*   s /= i */
  }
  TRY(py_exp(st->s, &t));                 /* acc += convert(s) */
  st->acc = st->acc + t;
  /* while (s > thr, k != 0)  interpreter.py:772-797 */
  if (chk && st->k != 0) return RL_ERR_POSTCONDITION;
  long T = 0;
  for (;;) {
    TRY(py_exp(st->s, &t));
    if (!(t > thr)) break;
    if (T >= max_trips) return RL_ERR_FUEL;
    T++;
    st->k += 1;
    st->kn += st->k;
    st->kn += nu;
    st->s = st->s + st->halfz2;           /* s *= halfz2 */
    st->s = st->s - log((double)st->k);   /* s /= k */
    PY_LOG((double)st->kn, lg);           /* s /= kn */
    st->s = st->s - lg;
    st->kn -= nu;
    st->kn -= st->k;
    TRY(py_exp(st->s, &t));
    if (st->k % 2 == 0) st->acc = st->acc + t; /* if (k % 2 == 0, ~) */
    else st->acc = st->acc - t;
    if (chk && !(st->k != 0)) return RL_ERR_POSTCONDITION;
  }
  *trips = T;
  return RL_OK;
}

/* ~@routine: the inverted block (sweep 2 when g == NULL, sweep 4 with the
 * adjoint rules when g != NULL). */
static int bj_unroutine(bj_state *st, bj_grad *g, long nu, double z, double thr, double tol,
                        int chk) {
  double t, lg;
  /* inverse while: While(pre = k != 0, post = s > thr)  reverser.py:110 */
  if (chk) {
    TRY(py_exp(st->s, &t));
    if (t > thr) return RL_ERR_POSTCONDITION;
  }
  while (st->k != 0) {
    /* inverse if: even k: acc -= convert(s) (sign +1); odd: acc += (sign -1) */
    TRY(py_exp(st->s, &t));
    if (st->k % 2 == 0) {
      st->acc = st->acc - t;
      if (g) g->s = g->s + (1.0 * g->acc) * t;
    } else {
      st->acc = st->acc + t;
      if (g) g->s = g->s + (-1.0 * g->acc) * t;
    }
    st->kn += st->k;
    st->kn += nu;
    PY_LOG((double)st->kn, lg);           /* s *= kn */
    st->s = st->s + lg;
    st->s = st->s + log((double)st->k);   /* s *= k */
    st->s = st->s - st->halfz2;           /* s /= halfz2 */
    if (g) g->halfz2 = g->halfz2 + 1.0 * g->s;
    st->kn -= nu;
    st->kn -= st->k;
    st->k -= 1;
    if (chk) {
      TRY(py_exp(st->s, &t));
      if (!(t > thr)) return RL_ERR_POSTCONDITION;
    }
  }
  TRY(py_exp(st->s, &t));                 /* acc -= convert(s) */
  st->acc = st->acc - t;
  if (g) g->s = g->s + (1.0 * g->acc) * t;
  for (long i = nu; i >= 1; i--) {        /* for i = nu:-1:1 */
    st->s = st->s + log((double)i);       /*   s *= i */
    st->s = st->s - st->halfz;            /*   s /= halfz */
    if (g) g->halfz = g->halfz + 1.0 * g->s;
  }
  st->halfz2 = st->halfz2 - st->halfz;    /* halfz2 /= halfz (x2) */
  if (g) g->halfz = g->halfz + 1.0 * g->halfz2;
  st->halfz2 = st->halfz2 - st->halfz;
  if (g) g->halfz = g->halfz + 1.0 * g->halfz2;
  st->halfz = st->halfz + log(2.0);       /* halfz *= 2 */
  st->halfz = st->halfz - st->lz;         /* halfz /= lz */
  if (g) g->lz = g->lz + 1.0 * g->halfz;
  PY_LOG(z, lg);                          /* lz /= convert(z) */
  st->lz = st->lz - lg;
  if (g) g->z = g->z + (1.0 * g->lz) / z;
  /* releases, reverse allocation order */
  RELEASE_F(st->acc, 0.0, tol);
  RELEASE_F(st->s, log(1.0), tol);
  RELEASE_F(st->halfz2, log(1.0), tol);
  RELEASE_F(st->halfz, log(1.0), tol);
  RELEASE_F(st->lz, log(1.0), tol);
  RELEASE_I(st->kn, 0);
  RELEASE_I(st->k, 0);
  return RL_OK;
}

int orc_besselj_grad(int nu, double z, double thr, double tol, double seed, long max_trips,
                     int invcheck, double *J, double *dJdz, long *trips) {
  bj_state st, st3;
  bj_grad g;
  long T = 0, T3 = 0;
  int chk = invcheck != 0;
  *J = NAN;
  *dJdz = NAN;
  *trips = 0;
  /* sweep 1 + out! += acc + sweep 2 */
  TRY(bj_routine(&st, nu, z, thr, max_trips, chk, &T));
  double out = 0.0;
  out = out + st.acc;
  const double J1 = out;
  TRY(bj_unroutine(&st, NULL, nu, z, thr, tol, chk));
  /* sweep 3: ~f recomputes the routine on GVar cells, then out! -= acc */
  memset(&g, 0, sizeof g);
  TRY(bj_routine(&st3, nu, z, thr, max_trips, chk, &T3));
  out = out - st3.acc;
  g.acc = g.acc + (1.0 * seed) * 1.0;
  /* sweep 4 */
  TRY(bj_unroutine(&st3, &g, nu, z, thr, tol, chk));
  /* primal restoration (autodiff.py:169-172): out! back to 0.0, z untouched */
  if (!(fabs(out - 0.0) <= tol)) return RL_ERR_RESTORE;
  *J = J1;
  *dJdz = g.z;
  *trips = T;
  return RL_OK;
}

/* -------------------------------------------------------------------------
 * Forward-over-reverse Hessian (autodiff.hessian, autodiff.py:216-257): the
 * gradient sweeps run over Dual numbers (values.py:258-340) with z carrying
 * the unit tangent.  Floats are represented as Dual(f, 0.0): for + - * /
 * this is bit-identical to the reference's _as_dual promotion (the two
 * tangent products are the same terms, IEEE + and * commute).  Sweeps 3 and
 * 4 follow _mul_div_adjoint (log_x + contrib / log_x - contrib) and
 * _plus_minus_adjoint (delta = (sign * gy) * s_exp(log_x)); sweep 3's
 * accumulations add exact zeros and are omitted like in the gradient.
 * ------------------------------------------------------------------------- */
typedef struct {
  double p, t;
} dual;

static dual d_add(dual a, dual b) { return (dual){a.p + b.p, a.t + b.t}; }
static dual d_sub(dual a, dual b) { return (dual){a.p - b.p, a.t - b.t}; }
static dual d_f(double f) { return (dual){f, 0.0}; }
static dual d_mul(dual a, dual b) { return (dual){a.p * b.p, a.t * b.p + a.p * b.t}; }
static dual d_div(dual a, dual b) {
  const double q = a.p / b.p;
  return (dual){q, (a.t - q * b.t) / b.p};
}
static int d_exp(dual a, dual *out) { /* s_exp: Dual(r, t r) */
  double r;
  TRY(py_exp(a.p, &r));
  *out = (dual){r, a.t * r};
  return RL_OK;
}
static int d_log(dual a, dual *out) { /* s_log: Dual(log p, t / p) */
  double l;
  PY_LOG(a.p, l);
  *out = (dual){l, a.t / a.p};
  return RL_OK;
}

int orc_besselj_hess(int nu, double z, double thr, double tol, double seed, long max_trips,
                     int invcheck, double *J, double *dJdz, double *d2Jdz2, long *trips) {
  int chk = invcheck != 0;
  double Jp, dz;
  long T;
  *d2Jdz2 = NAN;
  /* sweeps 1 and 2 (primal; the Dual run's primal is this) and every check */
  TRY(orc_besselj_grad(nu, z, thr, tol, seed, max_trips, invcheck, &Jp, &dz, &T));
  /* sweep 3: R in gradient mode over Duals */
  const dual Z = {z, 1.0};
  dual lz = d_f(0.0), halfz = d_f(0.0), halfz2 = d_f(0.0), s = d_f(0.0), acc = d_f(0.0), c, e;
  long k = 0, kn = 0;
  TRY(d_log(Z, &c)); /* lz *= convert(z) */
  lz = d_add(lz, c);
  halfz = d_add(halfz, lz);                   /* halfz *= lz */
  halfz = d_sub(halfz, d_f(log(2.0)));        /* halfz /= 2 */
  halfz2 = d_add(halfz2, halfz);              /* halfz2 *= halfz (x2) */
  halfz2 = d_add(halfz2, halfz);
  for (long i = 1; i <= nu; i++) {
    s = d_add(s, halfz);                      /* s *= halfz */
    s = d_sub(s, d_f(log((double)i)));        /* s /= i */
  }
  TRY(d_exp(s, &e));                          /* acc += convert(s) */
  acc = d_add(acc, e);
  for (;;) {
    TRY(d_exp(s, &e));
    if (!(e.p > thr)) break;
    k += 1;
    kn += k;
    kn += nu;
    s = d_add(s, halfz2);                     /* s *= halfz2 */
    s = d_sub(s, d_f(log((double)k)));        /* s /= k */
    s = d_sub(s, d_f(log((double)kn)));       /* s /= kn */
    kn -= nu;
    kn -= k;
    TRY(d_exp(s, &e));
    acc = (k % 2 == 0) ? d_add(acc, e) : d_sub(acc, e);
  }
  /* out! -= acc: acc.g += (1.0 * out.g) * 1.0 (a float) */
  const dual gacc = d_f((1.0 * seed) * 1.0);
  dual gs = d_f(0.0), gh2 = d_f(0.0), gh = d_f(0.0), glz = d_f(0.0), gz = d_f(0.0);
  /* sweep 4: ~R with the adjoint rules over Duals */
  while (k != 0) {
    TRY(d_exp(s, &e));
    if (k % 2 == 0) { /* acc -= convert(s): sign +1 */
      acc = d_sub(acc, e);
      gs = d_add(gs, d_mul(d_f(1.0 * gacc.p), e));
    } else {          /* acc += convert(s): sign -1 */
      acc = d_add(acc, e);
      gs = d_add(gs, d_mul(d_f(-1.0 * gacc.p), e));
    }
    kn += k;
    kn += nu;
    s = d_add(s, d_f(log((double)kn)));       /* s *= kn */
    s = d_add(s, d_f(log((double)k)));        /* s *= k */
    s = d_sub(s, halfz2);                     /* s /= halfz2 */
    gh2 = d_add(gh2, d_mul(d_f(1.0), gs));
    kn -= nu;
    kn -= k;
    k -= 1;
  }
  TRY(d_exp(s, &e));                          /* acc -= convert(s) */
  acc = d_sub(acc, e);
  gs = d_add(gs, d_mul(d_f(1.0 * gacc.p), e));
  for (long i = nu; i >= 1; i--) {
    s = d_add(s, d_f(log((double)i)));        /* s *= i */
    s = d_sub(s, halfz);                      /* s /= halfz */
    gh = d_add(gh, d_mul(d_f(1.0), gs));
  }
  halfz2 = d_sub(halfz2, halfz);              /* halfz2 /= halfz (x2) */
  gh = d_add(gh, d_mul(d_f(1.0), gh2));
  halfz2 = d_sub(halfz2, halfz);
  gh = d_add(gh, d_mul(d_f(1.0), gh2));
  halfz = d_add(halfz, d_f(log(2.0)));        /* halfz *= 2 */
  halfz = d_sub(halfz, lz);                   /* halfz /= lz */
  glz = d_add(glz, d_mul(d_f(1.0), gh));
  TRY(d_log(Z, &c));                          /* lz /= convert(z) */
  lz = d_sub(lz, c);
  gz = d_add(gz, d_div(d_mul(d_f(1.0), glz), Z));
  (void)chk;
  (void)tol;
  if (J) *J = Jp;
  if (dJdz) *dJdz = gz.p;
  *d2Jdz2 = gz.t;
  if (trips) *trips = T;
  return RL_OK;
}

long orc_besselj_hess_batch(int nu, const double *z, long n, double thr, double tol,
                            double seed, long max_trips, int invcheck, double *J, double *dJdz,
                            double *d2Jdz2, uint8_t *fail) {
  long total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (long i = 0; i < n; i++) {
    long T = 0;
    int rc = orc_besselj_hess(nu, z[i], thr, tol, seed, max_trips, invcheck, &J[i], &dJdz[i],
                              &d2Jdz2[i], &T);
    fail[i] = (uint8_t)rc;
    total += T;
  }
  return total;
}

/* batch helper for the CPU baseline (OpenMP over independent elements) */
long orc_besselj_grad_batch(int nu, const double *z, long n, double thr, double tol,
                            double seed, long max_trips, int invcheck, double *J,
                            double *dJdz, uint8_t *fail) {
  long total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (long i = 0; i < n; i++) {
    long T = 0;
    int rc = orc_besselj_grad(nu, z[i], thr, tol, seed, max_trips, invcheck, &J[i], &dJdz[i], &T);
    fail[i] = (uint8_t)rc;
    total += T;
  }
  return total;
}

/* =========================================================================
 * Bundle adjustment (programs/ba.rnl): ba_proj, rodrigues, ba_weight
 * cam index c[0..10] == cam[1..11]
 * ========================================================================= */

typedef struct {
  double x1, x2, x3, sqt, r1, r2, r3, p1, p2, rsq, rsq2, lf, q1, q2, d1, d2;
  int took; /* branch sqt != 0.0 */
} ba_state;

typedef struct {
  double th, ct, st, ti, w1, w2, w3, c1, c2, c3, dt, omc, tmp;
} rod_state;

typedef struct {
  double cam[11], X[3], w, f1, f2, e1, e2;
  double x1, x2, x3, sqt, r1, r2, r3, p1, p2, rsq, rsq2, lf, q1, q2, d1, d2;
} ba_grad;

static int py_div(double a, double b, double *out) { /* values.s_div */
  if (b == 0) return RL_ERR_DOMAIN;
  *out = a / b;
  return RL_OK;
}

static int py_sqrt(double x, double *out) {
  if (x < 0) return RL_ERR_DOMAIN;
  *out = sqrt(x);
  return RL_OK;
}

/* rodrigues' @routine block, forward */
static int rod_routine(rod_state *s, const double *c, double x1, double x2, double x3,
                       double sqt) {
  double t;
  s->th = 0.0;
  TRY(py_sqrt(sqt, &t));
  s->th = s->th + t;
  s->ct = 0.0;
  s->st = 0.0;
  s->ti = 0.0;
  s->ct = s->ct + cos(s->th);
  s->st = s->st + sin(s->th);
  TRY(py_div(1.0, s->th, &t));
  s->ti = s->ti + t;
  s->w1 = 0.0;
  s->w2 = 0.0;
  s->w3 = 0.0;
  s->w1 = s->w1 + c[0] * s->ti;
  s->w2 = s->w2 + c[1] * s->ti;
  s->w3 = s->w3 + c[2] * s->ti;
  s->c1 = 0.0;
  s->c2 = 0.0;
  s->c3 = 0.0;
  s->c1 = s->c1 + s->w2 * x3;
  s->c1 = s->c1 - s->w3 * x2;
  s->c2 = s->c2 + s->w3 * x1;
  s->c2 = s->c2 - s->w1 * x3;
  s->c3 = s->c3 + s->w1 * x2;
  s->c3 = s->c3 - s->w2 * x1;
  s->dt = 0.0;
  s->dt = s->dt + s->w1 * x1;
  s->dt = s->dt + s->w2 * x2;
  s->dt = s->dt + s->w3 * x3;
  s->omc = 0.0;
  s->omc = s->omc + (1.0 - s->ct);
  s->tmp = 0.0;
  s->tmp = s->tmp + s->dt * s->omc;
  return RL_OK;
}

/* rodrigues' ~@routine; adjoints into g when non-NULL */
static int rod_unroutine(rod_state *s, const double *c, double x1, double x2, double x3,
                         double sqt, ba_grad *g, double tol, int chk, double *gth_out,
                         double *gti_io, double gw[3], double gc[3], double *gdt_io,
                         double *gomc_io, double *gtmp_io, double *gct_io, double *gst_io) {
  double t;
  double gtmp = g ? *gtmp_io : 0, gomc = g ? *gomc_io : 0, gdt = g ? *gdt_io : 0;
  double gct = g ? *gct_io : 0, gst = g ? *gst_io : 0, gti = g ? *gti_io : 0, gth = 0;
  double gw1 = g ? gw[0] : 0, gw2 = g ? gw[1] : 0, gw3 = g ? gw[2] : 0;
  double gc1 = g ? gc[0] : 0, gc2 = g ? gc[1] : 0, gc3 = g ? gc[2] : 0;
  /* tmp -= dt * omc */
  s->tmp = s->tmp - s->dt * s->omc;
  if (g) {
    gdt = gdt + (1.0 * gtmp) * s->omc;
    gomc = gomc + (1.0 * gtmp) * s->dt;
  }
  RELEASE_F(s->tmp, 0.0, tol);
  /* omc -= 1.0 - ct */
  s->omc = s->omc - (1.0 - s->ct);
  if (g) gct = gct + (1.0 * gomc) * -1.0;
  RELEASE_F(s->omc, 0.0, tol);
  /* dt -= w3*x3; w2*x2; w1*x1 */
  s->dt = s->dt - s->w3 * x3;
  if (g) { gw3 = gw3 + (1.0 * gdt) * x3; g->x3 = g->x3 + (1.0 * gdt) * s->w3; }
  s->dt = s->dt - s->w2 * x2;
  if (g) { gw2 = gw2 + (1.0 * gdt) * x2; g->x2 = g->x2 + (1.0 * gdt) * s->w2; }
  s->dt = s->dt - s->w1 * x1;
  if (g) { gw1 = gw1 + (1.0 * gdt) * x1; g->x1 = g->x1 + (1.0 * gdt) * s->w1; }
  RELEASE_F(s->dt, 0.0, tol);
  /* c3 += w2*x1 (inverse of -=, sign -1); c3 -= w1*x2 */
  s->c3 = s->c3 + s->w2 * x1;
  if (g) { gw2 = gw2 + (-1.0 * gc3) * x1; g->x1 = g->x1 + (-1.0 * gc3) * s->w2; }
  s->c3 = s->c3 - s->w1 * x2;
  if (g) { gw1 = gw1 + (1.0 * gc3) * x2; g->x2 = g->x2 + (1.0 * gc3) * s->w1; }
  s->c2 = s->c2 + s->w1 * x3;
  if (g) { gw1 = gw1 + (-1.0 * gc2) * x3; g->x3 = g->x3 + (-1.0 * gc2) * s->w1; }
  s->c2 = s->c2 - s->w3 * x1;
  if (g) { gw3 = gw3 + (1.0 * gc2) * x1; g->x1 = g->x1 + (1.0 * gc2) * s->w3; }
  s->c1 = s->c1 + s->w3 * x2;
  if (g) { gw3 = gw3 + (-1.0 * gc1) * x2; g->x2 = g->x2 + (-1.0 * gc1) * s->w3; }
  s->c1 = s->c1 - s->w2 * x3;
  if (g) { gw2 = gw2 + (1.0 * gc1) * x3; g->x3 = g->x3 + (1.0 * gc1) * s->w2; }
  RELEASE_F(s->c3, 0.0, tol);
  RELEASE_F(s->c2, 0.0, tol);
  RELEASE_F(s->c1, 0.0, tol);
  /* w3 -= cam[3]*ti; w2; w1 */
  s->w3 = s->w3 - c[2] * s->ti;
  if (g) { g->cam[2] = g->cam[2] + (1.0 * gw3) * s->ti; gti = gti + (1.0 * gw3) * c[2]; }
  s->w2 = s->w2 - c[1] * s->ti;
  if (g) { g->cam[1] = g->cam[1] + (1.0 * gw2) * s->ti; gti = gti + (1.0 * gw2) * c[1]; }
  s->w1 = s->w1 - c[0] * s->ti;
  if (g) { g->cam[0] = g->cam[0] + (1.0 * gw1) * s->ti; gti = gti + (1.0 * gw1) * c[0]; }
  RELEASE_F(s->w3, 0.0, tol);
  RELEASE_F(s->w2, 0.0, tol);
  RELEASE_F(s->w1, 0.0, tol);
  /* ti -= 1.0 / th; st -= sin(th); ct -= cos(th) */
  TRY(py_div(1.0, s->th, &t));
  s->ti = s->ti - t;
  if (g) {
    double p;
    TRY(py_div(1.0, s->th * s->th, &p));
    gth = gth + (1.0 * gti) * -p;
  }
  s->st = s->st - sin(s->th);
  if (g) gth = gth + (1.0 * gst) * cos(s->th);
  s->ct = s->ct - cos(s->th);
  if (g) gth = gth + (1.0 * gct) * -sin(s->th);
  RELEASE_F(s->ti, 0.0, tol);
  RELEASE_F(s->st, 0.0, tol);
  RELEASE_F(s->ct, 0.0, tol);
  /* th -= sqrt(sqt) */
  TRY(py_sqrt(sqt, &t));
  s->th = s->th - t;
  if (g) {
    double p;
    TRY(py_div(0.5, sqrt(sqt), &p));
    g->sqt = g->sqt + (1.0 * gth) * p;
  }
  RELEASE_F(s->th, 0.0, tol);
  if (gth_out) *gth_out = gth;
  return RL_OK;
}

/* rodrigues(r1!, r2!, r3!, cam, x1, x2, x3, sqt), forward (sweeps 1, 3) and its
 * uncall (sweeps 2, 4) */
static int rod_call(ba_state *m, const double *c, double tol, int chk) {
  rod_state s;
  TRY(rod_routine(&s, c, m->x1, m->x2, m->x3, m->sqt));
  m->r1 = m->r1 + m->x1 * s.ct;
  m->r2 = m->r2 + m->x2 * s.ct;
  m->r3 = m->r3 + m->x3 * s.ct;
  m->r1 = m->r1 + s.c1 * s.st;
  m->r2 = m->r2 + s.c2 * s.st;
  m->r3 = m->r3 + s.c3 * s.st;
  m->r1 = m->r1 + s.w1 * s.tmp;
  m->r2 = m->r2 + s.w2 * s.tmp;
  m->r3 = m->r3 + s.w3 * s.tmp;
  TRY(rod_unroutine(&s, c, m->x1, m->x2, m->x3, m->sqt, NULL, tol, chk, NULL, NULL, NULL, NULL,
                    NULL, NULL, NULL, NULL, NULL));
  return RL_OK;
}

static int rod_uncall(ba_state *m, const double *c, ba_grad *g, double tol, int chk) {
  rod_state s;
  /* ~rodrigues = @routine R; inverted middle; ~@routine */
  TRY(rod_routine(&s, c, m->x1, m->x2, m->x3, m->sqt));
  double gtmp = 0, gst = 0, gct = 0, gomc = 0, gdt = 0, gti = 0;
  double gw[3] = {0, 0, 0}, gc[3] = {0, 0, 0};
  m->r3 = m->r3 - s.w3 * s.tmp;
  if (g) { gw[2] = gw[2] + (1.0 * g->r3) * s.tmp; gtmp = gtmp + (1.0 * g->r3) * s.w3; }
  m->r2 = m->r2 - s.w2 * s.tmp;
  if (g) { gw[1] = gw[1] + (1.0 * g->r2) * s.tmp; gtmp = gtmp + (1.0 * g->r2) * s.w2; }
  m->r1 = m->r1 - s.w1 * s.tmp;
  if (g) { gw[0] = gw[0] + (1.0 * g->r1) * s.tmp; gtmp = gtmp + (1.0 * g->r1) * s.w1; }
  m->r3 = m->r3 - s.c3 * s.st;
  if (g) { gc[2] = gc[2] + (1.0 * g->r3) * s.st; gst = gst + (1.0 * g->r3) * s.c3; }
  m->r2 = m->r2 - s.c2 * s.st;
  if (g) { gc[1] = gc[1] + (1.0 * g->r2) * s.st; gst = gst + (1.0 * g->r2) * s.c2; }
  m->r1 = m->r1 - s.c1 * s.st;
  if (g) { gc[0] = gc[0] + (1.0 * g->r1) * s.st; gst = gst + (1.0 * g->r1) * s.c1; }
  m->r3 = m->r3 - m->x3 * s.ct;
  if (g) { g->x3 = g->x3 + (1.0 * g->r3) * s.ct; gct = gct + (1.0 * g->r3) * m->x3; }
  m->r2 = m->r2 - m->x2 * s.ct;
  if (g) { g->x2 = g->x2 + (1.0 * g->r2) * s.ct; gct = gct + (1.0 * g->r2) * m->x2; }
  m->r1 = m->r1 - m->x1 * s.ct;
  if (g) { g->x1 = g->x1 + (1.0 * g->r1) * s.ct; gct = gct + (1.0 * g->r1) * m->x1; }
  TRY(rod_unroutine(&s, c, m->x1, m->x2, m->x3, m->sqt, g, tol, chk, NULL, &gti, gw, gc, &gdt,
                    &gomc, &gtmp, &gct, &gst));
  return RL_OK;
}

/* ba_proj's @routine block, forward */
static int ba_routine(ba_state *m, const double *c, const double *X, double f1, double f2,
                      double tol, int chk) {
  double t;
  m->x1 = 0.0;
  m->x2 = 0.0;
  m->x3 = 0.0;
  m->x1 = m->x1 + (X[0] - c[3]);
  m->x2 = m->x2 + (X[1] - c[4]);
  m->x3 = m->x3 + (X[2] - c[5]);
  m->sqt = 0.0;
  m->sqt = m->sqt + c[0] * c[0];
  m->sqt = m->sqt + c[1] * c[1];
  m->sqt = m->sqt + c[2] * c[2];
  m->r1 = 0.0;
  m->r2 = 0.0;
  m->r3 = 0.0;
  m->took = m->sqt != 0.0;
  if (m->took) {
    TRY(rod_call(m, c, tol, chk));
  } else {
    m->r1 = m->r1 + m->x1;
    m->r2 = m->r2 + m->x2;
    m->r3 = m->r3 + m->x3;
    m->r1 = m->r1 + c[1] * m->x3;
    m->r1 = m->r1 - c[2] * m->x2;
    m->r2 = m->r2 + c[2] * m->x1;
    m->r2 = m->r2 - c[0] * m->x3;
    m->r3 = m->r3 + c[0] * m->x2;
    m->r3 = m->r3 - c[1] * m->x1;
  }
  if (chk && (m->sqt != 0.0) != m->took) return RL_ERR_POSTCONDITION;
  m->p1 = 0.0;
  m->p2 = 0.0;
  TRY(py_div(m->r1, m->r3, &t));
  m->p1 = m->p1 + t;
  TRY(py_div(m->r2, m->r3, &t));
  m->p2 = m->p2 + t;
  m->rsq = 0.0;
  m->rsq = m->rsq + m->p1 * m->p1;
  m->rsq = m->rsq + m->p2 * m->p2;
  m->rsq2 = 0.0;
  m->rsq2 = m->rsq2 + m->rsq * m->rsq;
  m->lf = 1.0;
  m->lf = m->lf + c[9] * m->rsq;
  m->lf = m->lf + c[10] * m->rsq2;
  m->q1 = 0.0;
  m->q2 = 0.0;
  m->q1 = m->q1 + m->p1 * m->lf;
  m->q2 = m->q2 + m->p2 * m->lf;
  m->d1 = 0.0;
  m->d2 = 0.0;
  m->d1 = m->d1 + m->q1 * c[6];
  m->d2 = m->d2 + m->q2 * c[6];
  m->d1 = m->d1 + c[7];
  m->d2 = m->d2 + c[8];
  m->d1 = m->d1 - f1;
  m->d2 = m->d2 - f2;
  return RL_OK;
}

/* ba_proj's ~@routine; adjoint rules when g != NULL */
static int ba_unroutine(ba_state *m, const double *c, const double *X, double f1, double f2,
                        ba_grad *g, double tol, int chk) {
  double t;
  (void)X;
  m->d2 = m->d2 + f2;                       /* d2 += f2  (inverse of -=: sign -1) */
  if (g) g->f2 = g->f2 + (-1.0 * g->d2) * 1.0;
  m->d1 = m->d1 + f1;
  if (g) g->f1 = g->f1 + (-1.0 * g->d1) * 1.0;
  m->d2 = m->d2 - c[8];
  if (g) g->cam[8] = g->cam[8] + (1.0 * g->d2) * 1.0;
  m->d1 = m->d1 - c[7];
  if (g) g->cam[7] = g->cam[7] + (1.0 * g->d1) * 1.0;
  m->d2 = m->d2 - m->q2 * c[6];
  if (g) { g->q2 = g->q2 + (1.0 * g->d2) * c[6]; g->cam[6] = g->cam[6] + (1.0 * g->d2) * m->q2; }
  m->d1 = m->d1 - m->q1 * c[6];
  if (g) { g->q1 = g->q1 + (1.0 * g->d1) * c[6]; g->cam[6] = g->cam[6] + (1.0 * g->d1) * m->q1; }
  RELEASE_F(m->d2, 0.0, tol);
  RELEASE_F(m->d1, 0.0, tol);
  m->q2 = m->q2 - m->p2 * m->lf;
  if (g) { g->p2 = g->p2 + (1.0 * g->q2) * m->lf; g->lf = g->lf + (1.0 * g->q2) * m->p2; }
  m->q1 = m->q1 - m->p1 * m->lf;
  if (g) { g->p1 = g->p1 + (1.0 * g->q1) * m->lf; g->lf = g->lf + (1.0 * g->q1) * m->p1; }
  RELEASE_F(m->q2, 0.0, tol);
  RELEASE_F(m->q1, 0.0, tol);
  m->lf = m->lf - c[10] * m->rsq2;
  if (g) { g->cam[10] = g->cam[10] + (1.0 * g->lf) * m->rsq2; g->rsq2 = g->rsq2 + (1.0 * g->lf) * c[10]; }
  m->lf = m->lf - c[9] * m->rsq;
  if (g) { g->cam[9] = g->cam[9] + (1.0 * g->lf) * m->rsq; g->rsq = g->rsq + (1.0 * g->lf) * c[9]; }
  RELEASE_F(m->lf, 1.0, tol);
  m->rsq2 = m->rsq2 - m->rsq * m->rsq;
  if (g) g->rsq = g->rsq + (1.0 * g->rsq2) * (2.0 * m->rsq);
  RELEASE_F(m->rsq2, 0.0, tol);
  m->rsq = m->rsq - m->p2 * m->p2;
  if (g) g->p2 = g->p2 + (1.0 * g->rsq) * (2.0 * m->p2);
  m->rsq = m->rsq - m->p1 * m->p1;
  if (g) g->p1 = g->p1 + (1.0 * g->rsq) * (2.0 * m->p1);
  RELEASE_F(m->rsq, 0.0, tol);
  TRY(py_div(m->r2, m->r3, &t));            /* p2 -= r2 / r3 */
  m->p2 = m->p2 - t;
  if (g) {
    double pa, pb;
    TRY(py_div(1.0, m->r3, &pa));
    TRY(py_div(m->r2, m->r3 * m->r3, &pb));
    g->r2 = g->r2 + (1.0 * g->p2) * pa;
    g->r3 = g->r3 + (1.0 * g->p2) * -pb;
  }
  TRY(py_div(m->r1, m->r3, &t));            /* p1 -= r1 / r3 */
  m->p1 = m->p1 - t;
  if (g) {
    double pa, pb;
    TRY(py_div(1.0, m->r3, &pa));
    TRY(py_div(m->r1, m->r3 * m->r3, &pb));
    g->r1 = g->r1 + (1.0 * g->p1) * pa;
    g->r3 = g->r3 + (1.0 * g->p1) * -pb;
  }
  RELEASE_F(m->p2, 0.0, tol);
  RELEASE_F(m->p1, 0.0, tol);
  /* inverse if (sqt != 0.0, ~) */
  int took = m->sqt != 0.0;
  if (took) {
    TRY(rod_uncall(m, c, g, tol, chk));
  } else {
    m->r3 = m->r3 + c[1] * m->x1;
    if (g) { g->cam[1] = g->cam[1] + (-1.0 * g->r3) * m->x1; g->x1 = g->x1 + (-1.0 * g->r3) * c[1]; }
    m->r3 = m->r3 - c[0] * m->x2;
    if (g) { g->cam[0] = g->cam[0] + (1.0 * g->r3) * m->x2; g->x2 = g->x2 + (1.0 * g->r3) * c[0]; }
    m->r2 = m->r2 + c[0] * m->x3;
    if (g) { g->cam[0] = g->cam[0] + (-1.0 * g->r2) * m->x3; g->x3 = g->x3 + (-1.0 * g->r2) * c[0]; }
    m->r2 = m->r2 - c[2] * m->x1;
    if (g) { g->cam[2] = g->cam[2] + (1.0 * g->r2) * m->x1; g->x1 = g->x1 + (1.0 * g->r2) * c[2]; }
    m->r1 = m->r1 + c[2] * m->x2;
    if (g) { g->cam[2] = g->cam[2] + (-1.0 * g->r1) * m->x2; g->x2 = g->x2 + (-1.0 * g->r1) * c[2]; }
    m->r1 = m->r1 - c[1] * m->x3;
    if (g) { g->cam[1] = g->cam[1] + (1.0 * g->r1) * m->x3; g->x3 = g->x3 + (1.0 * g->r1) * c[1]; }
    m->r3 = m->r3 - m->x3;
    if (g) g->x3 = g->x3 + (1.0 * g->r3) * 1.0;
    m->r2 = m->r2 - m->x2;
    if (g) g->x2 = g->x2 + (1.0 * g->r2) * 1.0;
    m->r1 = m->r1 - m->x1;
    if (g) g->x1 = g->x1 + (1.0 * g->r1) * 1.0;
  }
  if (chk && (m->sqt != 0.0) != took) return RL_ERR_POSTCONDITION;
  RELEASE_F(m->r3, 0.0, tol);
  RELEASE_F(m->r2, 0.0, tol);
  RELEASE_F(m->r1, 0.0, tol);
  m->sqt = m->sqt - c[2] * c[2];
  if (g) g->cam[2] = g->cam[2] + (1.0 * g->sqt) * (2.0 * c[2]);
  m->sqt = m->sqt - c[1] * c[1];
  if (g) g->cam[1] = g->cam[1] + (1.0 * g->sqt) * (2.0 * c[1]);
  m->sqt = m->sqt - c[0] * c[0];
  if (g) g->cam[0] = g->cam[0] + (1.0 * g->sqt) * (2.0 * c[0]);
  RELEASE_F(m->sqt, 0.0, tol);
  m->x3 = m->x3 - (X[2] - c[5]);
  if (g) { g->X[2] = g->X[2] + (1.0 * g->x3) * 1.0; g->cam[5] = g->cam[5] + (1.0 * g->x3) * -1.0; }
  m->x2 = m->x2 - (X[1] - c[4]);
  if (g) { g->X[1] = g->X[1] + (1.0 * g->x2) * 1.0; g->cam[4] = g->cam[4] + (1.0 * g->x2) * -1.0; }
  m->x1 = m->x1 - (X[0] - c[3]);
  if (g) { g->X[0] = g->X[0] + (1.0 * g->x1) * 1.0; g->cam[3] = g->cam[3] + (1.0 * g->x1) * -1.0; }
  RELEASE_F(m->x3, 0.0, tol);
  RELEASE_F(m->x2, 0.0, tol);
  RELEASE_F(m->x1, 0.0, tol);
  return RL_OK;
}

/* One gradient() call of ba_proj with seed on e1! (row 0) or e2! (row 1). */
static int ba_gradient_pass(const double *c, const double *X, double w, double f1, double f2,
                            int row, double tol, int chk, double e[2], double Jrow[15]) {
  ba_state m;
  ba_grad g;
  double e1 = 0.0, e2 = 0.0;
  /* sweeps 1, 2 */
  TRY(ba_routine(&m, c, X, f1, f2, tol, chk));
  e1 = e1 + w * m.d1;
  e2 = e2 + w * m.d2;
  const double E1 = e1, E2 = e2;
  TRY(ba_unroutine(&m, c, X, f1, f2, NULL, tol, chk));
  /* sweep 3: ~ba_proj = R; e2! -= w*d2; e1! -= w*d1; R^-1 */
  memset(&g, 0, sizeof g);
  if (row == 0) g.e1 = 1.0; else g.e2 = 1.0;
  TRY(ba_routine(&m, c, X, f1, f2, tol, chk));
  e2 = e2 - w * m.d2;
  g.w = g.w + (1.0 * g.e2) * m.d2;
  g.d2 = g.d2 + (1.0 * g.e2) * w;
  e1 = e1 - w * m.d1;
  g.w = g.w + (1.0 * g.e1) * m.d1;
  g.d1 = g.d1 + (1.0 * g.e1) * w;
  /* sweep 4 */
  TRY(ba_unroutine(&m, c, X, f1, f2, &g, tol, chk));
  if (!(fabs(e1 - 0.0) <= tol) || !(fabs(e2 - 0.0) <= tol)) return RL_ERR_RESTORE;
  e[0] = E1;
  e[1] = E2;
  memcpy(Jrow, g.cam, 11 * sizeof(double));
  memcpy(Jrow + 11, g.X, 3 * sizeof(double));
  Jrow[14] = g.w;
  return RL_OK;
}

/* gradient of ba_weight(e!, w): e! += 1.0; e! -= abs2(w) */
static int ba_weight_pass(double w, double tol, double *ew, double *dw) {
  double e = 0.0, gw = 0.0, ge = 1.0;
  e = e + 1.0;
  e = e - w * w;
  const double E = e;
  /* ~ba_weight: e! += abs2(w) (sign -1); e! -= 1.0 */
  e = e + w * w;
  gw = gw + (-1.0 * ge) * (2.0 * w);
  e = e - 1.0;
  if (!(fabs(e - 0.0) <= tol)) return RL_ERR_RESTORE;
  *ew = E;
  *dw = gw;
  return RL_OK;
}

/* One observation: 2 seeded passes + the weight residual.
 * J[31] = [row e1 (15), row e2 (15), d(1-w^2)/dw]; err[3] = e1, e2, 1-w^2 */
int orc_ba_obs(const double *cam, const double *X, double w, double f1, double f2, double tol,
               int invcheck, double *err, double *J) {
  int chk = invcheck != 0;
  double e[2];
  for (int i = 0; i < 31; i++) J[i] = NAN;
  TRY(ba_gradient_pass(cam, X, w, f1, f2, 0, tol, chk, e, J));
  TRY(ba_gradient_pass(cam, X, w, f1, f2, 1, tol, chk, e, J + 15));
  double ew;
  TRY(ba_weight_pass(w, tol, &ew, &J[30]));
  if (err) {
    err[0] = e[0];
    err[1] = e[1];
    err[2] = ew;
  }
  return RL_OK;
}

long orc_ba_jac_batch(int n_cams, int n_pts, long n_obs, const double *cams, const double *X,
                      const double *w, const double *feats, const int32_t *obs, double tol,
                      int invcheck, double *err, double *J, uint8_t *fail) {
  long nfail = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : nfail)
  for (long i = 0; i < n_obs; i++) {
    int c = obs[2 * i], p = obs[2 * i + 1];
    int rc;
    if (c < 0 || c >= n_cams || p < 0 || p >= n_pts) {
      rc = RL_ERR_INDEX;
      for (int j = 0; j < 31; j++) J[31 * i + j] = NAN;
    } else {
      rc = orc_ba_obs(cams + 11 * (long)c, X + 3 * (long)p, w[i], feats[2 * i],
                      feats[2 * i + 1], tol, invcheck, err ? err + 3 * i : NULL, J + 31 * i);
    }
    fail[i] = (uint8_t)rc;
    nfail += rc != RL_OK;
  }
  return nfail;
}

/* =========================================================================
 * GMM (programs/gmm.rnl)
 *
 * Unlike the two programs above, gmm's scratch ARGUMENTS (qd!, sq!, xc!,
 * qxc!, mt!, dm!) are GVar cells whose cotangents persist across points in
 * gradient mode, so gradient-mode forward statements on them are NOT
 * no-ops: every statement below applies its adjoint rule whenever
 * `c->gm` is set, in both directions (sign -1 for an executed +=, +1 for
 * an executed -=; numerics.py:444).  Values also carry round-off residue
 * from point to point exactly as in the sequential reference.
 * Arrays are 0-based here; the program's 1-based index i maps to i-1.
 * ========================================================================= */

typedef struct {
  int d, K, N, P, wm, gm, chk;
  int fresh; /* 1: scratch zeroed per (point, component) — the device's semantics */
  double tol, ga;
  const double *x, *alphas, *means, *icf;
  double *qd, *sq, *xc, *qxc, *mt; /* Float scratch values */
  long *dmi;                          /* Int scratch: argmax steps */
  double err, cst;
  /* cotangents (gm) */
  double *g_alphas, *g_means, *g_icf, *g_x, *g_qd, *g_sq, *g_xc, *g_qxc, *g_mt;
  double g_err, g_cst;
} gmm_ctx;

#define GM(c) ((c)->gm)
/* a.g += (sign * y.g) * p */
#define ADJ(c, ag, sgy, p)            \
  do {                                \
    if (GM(c)) (ag) = (ag) + (sgy) * (p); \
  } while (0)

/* @routine of the whole function: qd = exp(diag icf), sq = sum(diag icf) */
static int gmm_top(gmm_ctx *c, int inverse) {
  const int d = c->d, K = c->K, P = c->P;
  double e;
  if (!inverse) {
    for (int k = 0; k < K; k++)
      for (int j = 0; j < d; j++) {
        TRY(py_exp(c->icf[k * P + j], &e));
        c->qd[k * d + j] = c->qd[k * d + j] + e;
        ADJ(c, c->g_icf[k * P + j], -1.0 * c->g_qd[k * d + j], e);
        c->sq[k] = c->sq[k] + c->icf[k * P + j];
        ADJ(c, c->g_icf[k * P + j], -1.0 * c->g_sq[k], 1.0);
      }
  } else {
    for (int k = K - 1; k >= 0; k--)
      for (int j = d - 1; j >= 0; j--) {
        c->sq[k] = c->sq[k] - c->icf[k * P + j];
        ADJ(c, c->g_icf[k * P + j], 1.0 * c->g_sq[k], 1.0);
        TRY(py_exp(c->icf[k * P + j], &e));
        c->qd[k * d + j] = c->qd[k * d + j] - e;
        ADJ(c, c->g_icf[k * P + j], 1.0 * c->g_qd[k * d + j], e);
      }
  }
  return RL_OK;
}

/* inner @routine for point i, component k: xc = x_i - mu_k, qxc = L_k xc,
 * sqn = |qxc|^2.  Forward (inverse == 0) or inverted. */
static int gmm_ik(gmm_ctx *c, int i, int k, int inverse, double *sqn, double *g_sqn) {
  const int chk = c->chk;
  const int d = c->d, P = c->P;
  const double *xi = c->x + (long)i * d, *mk = c->means + k * d, *Lk = c->icf + k * P;
  double *gxi = GM(c) ? c->g_x + (long)i * d : NULL;
  double *gmk = GM(c) ? c->g_means + k * d : NULL, *gLk = GM(c) ? c->g_icf + k * P : NULL;
  double *gqdk = GM(c) ? c->g_qd + k * d : NULL;
  const double *qdk = c->qd + k * d;
  if (!inverse) {
    *sqn = 0.0;
    *g_sqn = 0.0;
    for (int j = 0; j < d; j++) {
      c->xc[j] = c->xc[j] + (xi[j] - mk[j]);
      ADJ(c, gxi[j], -1.0 * c->g_xc[j], 1.0);
      ADJ(c, gmk[j], -1.0 * c->g_xc[j], -1.0);
      c->qxc[j] = c->qxc[j] + qdk[j] * c->xc[j];
      ADJ(c, gqdk[j], -1.0 * c->g_qxc[j], c->xc[j]);
      ADJ(c, c->g_xc[j], -1.0 * c->g_qxc[j], qdk[j]);
    }
    int li = d; /* 1-based packed index; icf[k, li] == Lk[li - 1] */
    for (int a = 0; a < d; a++)
      for (int b = a + 1; b < d; b++) {
        li += 1; /* INC(li) */
        c->qxc[b] = c->qxc[b] + Lk[li - 1] * c->xc[a];
        ADJ(c, gLk[li - 1], -1.0 * c->g_qxc[b], c->xc[a]);
        ADJ(c, c->g_xc[a], -1.0 * c->g_qxc[b], Lk[li - 1]);
      }
    RELEASE_I(li, P);
    for (int j = 0; j < d; j++) {
      *sqn = *sqn + c->qxc[j] * c->qxc[j];
      ADJ(c, c->g_qxc[j], -1.0 * *g_sqn, 2.0 * c->qxc[j]);
    }
  } else {
    for (int j = d - 1; j >= 0; j--) {
      *sqn = *sqn - c->qxc[j] * c->qxc[j];
      ADJ(c, c->g_qxc[j], 1.0 * *g_sqn, 2.0 * c->qxc[j]);
    }
    int li = P;
    for (int a = d - 1; a >= 0; a--)
      for (int b = d - 1; b >= a + 1; b--) {
        c->qxc[b] = c->qxc[b] - Lk[li - 1] * c->xc[a];
        ADJ(c, gLk[li - 1], 1.0 * c->g_qxc[b], c->xc[a]);
        ADJ(c, c->g_xc[a], 1.0 * c->g_qxc[b], Lk[li - 1]);
        li -= 1; /* DEC(li) */
      }
    RELEASE_I(li, d);
    for (int j = d - 1; j >= 0; j--) {
      c->qxc[j] = c->qxc[j] - qdk[j] * c->xc[j];
      ADJ(c, gqdk[j], 1.0 * c->g_qxc[j], c->xc[j]);
      ADJ(c, c->g_xc[j], 1.0 * c->g_qxc[j], qdk[j]);
      c->xc[j] = c->xc[j] - (xi[j] - mk[j]);
      ADJ(c, gxi[j], 1.0 * c->g_xc[j], 1.0);
      ADJ(c, gmk[j], 1.0 * c->g_xc[j], -1.0);
    }
    RELEASE_F(*sqn, 0.0, c->tol);
  }
  return RL_OK;
}

/* for-k body: @routine ik; mt += alphas; mt += sq; mt -= sqn*0.5; ~@routine
 * (mirror == 1: the inverted body, whose middle is mt += sqn*0.5; mt -= sq;
 * mt -= alphas) */
static int gmm_k_body(gmm_ctx *c, int i, int k, int mirror) {
  double sqn, g_sqn;
  if (c->fresh) /* NOT the reference: the device's per-(point, component) scratch */
    for (int j = 0; j < c->d; j++) {
      c->xc[j] = 0.0;
      c->qxc[j] = 0.0;
      if (GM(c)) {
        c->g_xc[j] = 0.0;
        c->g_qxc[j] = 0.0;
      }
    }
  TRY(gmm_ik(c, i, k, 0, &sqn, &g_sqn));
  double *mt = &c->mt[k];
  double *gmt = GM(c) ? &c->g_mt[k] : NULL;
  if (!mirror) {
    *mt = *mt + c->alphas[k];
    ADJ(c, c->g_alphas[k], -1.0 * *gmt, 1.0);
    *mt = *mt + c->sq[k];
    ADJ(c, c->g_sq[k], -1.0 * *gmt, 1.0);
    *mt = *mt - sqn * 0.5;
    ADJ(c, g_sqn, 1.0 * *gmt, 0.5);
  } else {
    *mt = *mt + sqn * 0.5;
    ADJ(c, g_sqn, -1.0 * *gmt, 0.5);
    *mt = *mt - c->sq[k];
    ADJ(c, c->g_sq[k], 1.0 * *gmt, 1.0);
    *mt = *mt - c->alphas[k];
    ADJ(c, c->g_alphas[k], 1.0 * *gmt, 1.0);
  }
  TRY(gmm_ik(c, i, k, 1, &sqn, &g_sqn));
  return RL_OK;
}

/* reversible logsumexp over v[0..K) (the point routine's tail and the
 * alphas routine share it): argmax record in the Int scratch dmi
 * (imx <- 1; if (v[k] > v[imx], dm![k] > 0) {dm![k] += k - imx; imx += dm![k]}),
 * mx <- 0.0; mx += v[imx]; se = sum exp(v - mx).  gv: cotangent array of v
 * (the argmax record is Int: no cotangents).  imx is 0-based here; the
 * recorded steps k - imx are the same in both bases. */
static int gmm_lse_fwd(gmm_ctx *c, const double *v, double *gv, int *imx, double *mx,
                       double *gmx, double *se, double *gse) {
  const int chk = c->chk;
  const int K = c->K;
  double e;
  *imx = 0;
  for (int k = 1; k < K; k++) {
    int took = v[k] > v[*imx];
    if (took) {
      c->dmi[k] = c->dmi[k] + (k - *imx);
      *imx = *imx + (int)c->dmi[k];
    }
    if (chk && (c->dmi[k] > 0) != took) return RL_ERR_POSTCONDITION;
  }
  *mx = 0.0;
  *gmx = 0.0;
  *mx = *mx + v[*imx];
  ADJ(c, gv[*imx], -1.0 * *gmx, 1.0);
  *se = 0.0;
  *gse = 0.0;
  for (int k = 0; k < K; k++) {
    double t = 0.0, gt = 0.0;
    t = t + (v[k] - *mx);
    ADJ(c, gv[k], -1.0 * gt, 1.0);
    ADJ(c, *gmx, -1.0 * gt, -1.0);
    TRY(py_exp(t, &e));
    *se = *se + e;
    ADJ(c, gt, -1.0 * *gse, e);
    t = t - (v[k] - *mx);
    ADJ(c, gv[k], 1.0 * gt, 1.0);
    ADJ(c, *gmx, 1.0 * gt, -1.0);
    RELEASE_F(t, 0.0, c->tol);
  }
  return RL_OK;
}

static int gmm_lse_inv(gmm_ctx *c, const double *v, double *gv, int *imx, double *mx,
                       double *gmx, double *se, double *gse) {
  const int chk = c->chk;
  const int K = c->K;
  double e;
  for (int k = K - 1; k >= 0; k--) {
    double t = 0.0, gt = 0.0;
    t = t + (v[k] - *mx);
    ADJ(c, gv[k], -1.0 * gt, 1.0);
    ADJ(c, *gmx, -1.0 * gt, -1.0);
    TRY(py_exp(t, &e));
    *se = *se - e;
    ADJ(c, gt, 1.0 * *gse, e);
    t = t - (v[k] - *mx);
    ADJ(c, gv[k], 1.0 * gt, 1.0);
    ADJ(c, *gmx, 1.0 * gt, -1.0);
    RELEASE_F(t, 0.0, c->tol);
  }
  RELEASE_F(*se, 0.0, c->tol);
  *mx = *mx - v[*imx];                 /* mx -= v[imx] */
  ADJ(c, gv[*imx], 1.0 * *gmx, 1.0);
  RELEASE_F(*mx, 0.0, c->tol);
  for (int k = K - 1; k >= 1; k--) {
    int took = c->dmi[k] > 0;          /* inverted If: pre/post swapped (reverser.py:106-108) */
    if (took) {
      *imx = *imx - (int)c->dmi[k];
      c->dmi[k] = c->dmi[k] - (k - *imx);
    }
    if (chk && (v[k] > v[*imx]) != took) return RL_ERR_POSTCONDITION;
  }
  RELEASE_I(*imx, 0);                  /* imx -> 1 */
  return RL_OK;
}

/* for-i body: @routine R_i; err += log(se); err += mx; ~@routine
 * (mirror: err -= mx; err -= log(se)) */
static int gmm_point(gmm_ctx *c, int i, int mirror) {
  const int K = c->K;
  double mx, gmx, se, gse, l, p;
  int imx;
  double *gmt = GM(c) ? c->g_mt : NULL;
  if (c->fresh) /* NOT the reference: the device's per-point scratch */
    for (int k = 0; k < K; k++) {
      c->mt[k] = 0.0;
      if (GM(c)) c->g_mt[k] = 0.0;
    }
  for (int k = 0; k < K; k++) TRY(gmm_k_body(c, i, k, 0));
  TRY(gmm_lse_fwd(c, c->mt, gmt, &imx, &mx, &gmx, &se, &gse));
  PY_LOG(se, l);
  if (!mirror) {
    c->err = c->err + l;
    if (GM(c)) { TRY(py_div(1.0, se, &p)); ADJ(c, gse, -1.0 * c->g_err, p); }
    c->err = c->err + mx;
    ADJ(c, gmx, -1.0 * c->g_err, 1.0);
  } else {
    c->err = c->err - mx;
    ADJ(c, gmx, 1.0 * c->g_err, 1.0);
    c->err = c->err - l;
    if (GM(c)) { TRY(py_div(1.0, se, &p)); ADJ(c, gse, 1.0 * c->g_err, p); }
  }
  TRY(gmm_lse_inv(c, c->mt, gmt, &imx, &mx, &gmx, &se, &gse));
  for (int k = K - 1; k >= 0; k--) TRY(gmm_k_body(c, i, k, 1));
  return RL_OK;
}

/* @routine amx/ase/lsa/nn; err -= nn*lsa (mirror: +=); ~@routine */
static int gmm_alpha_lse(gmm_ctx *c, int mirror) {
  const int chk = c->chk;
  double amx, gamx, ase, gase, lsa = 0.0, glsa = 0.0, l, p;
  int ia;
  double *ga = GM(c) ? c->g_alphas : NULL;
  TRY(gmm_lse_fwd(c, c->alphas, ga, &ia, &amx, &gamx, &ase, &gase));
  PY_LOG(ase, l);
  lsa = lsa + l;
  if (GM(c)) { TRY(py_div(1.0, ase, &p)); ADJ(c, gase, -1.0 * glsa, p); }
  lsa = lsa + amx;
  ADJ(c, gamx, -1.0 * glsa, 1.0);
  const long nn = c->N;
  if (!mirror) {
    c->err = c->err - (double)nn * lsa;
    ADJ(c, glsa, 1.0 * c->g_err, (double)nn);
  } else {
    c->err = c->err + (double)nn * lsa;
    ADJ(c, glsa, -1.0 * c->g_err, (double)nn);
  }
  /* inverse: nn -> N; lsa -= amx; lsa -= log(ase); lsa -> 0 */
  lsa = lsa - amx;
  ADJ(c, gamx, 1.0 * glsa, 1.0);
  PY_LOG(ase, l);
  lsa = lsa - l;
  if (GM(c)) { TRY(py_div(1.0, ase, &p)); ADJ(c, gase, 1.0 * glsa, p); }
  RELEASE_F(lsa, 0.0, c->tol);
  TRY(gmm_lse_inv(c, c->alphas, ga, &ia, &amx, &gamx, &ase, &gase));
  return RL_OK;
}

/* @routine hg2/fro/ssq; err += hg2*fro; err -= wm*ssq; ~@routine
 * (mirror: err += wm*ssq; err -= hg2*fro) */
static int gmm_prior(gmm_ctx *c, int mirror) {
  const int chk = c->chk;
  const int d = c->d, K = c->K, P = c->P;
  double hg2 = 0.5 * c->ga * c->ga, ghg2 = 0.0, fro = 0.0, gfro = 0.0, ssq = 0.0, gssq = 0.0;
  for (int k = 0; k < K; k++)
    for (int j = 0; j < P; j++) {
      if (j < d) {
        double q = c->qd[k * d + j];
        fro = fro + q * q;
        ADJ(c, c->g_qd[k * d + j], -1.0 * gfro, 2.0 * q);
      } else {
        double q = c->icf[k * P + j];
        fro = fro + q * q;
        ADJ(c, c->g_icf[k * P + j], -1.0 * gfro, 2.0 * q);
      }
    }
  for (int k = 0; k < K; k++) {
    ssq = ssq + c->sq[k];
    ADJ(c, c->g_sq[k], -1.0 * gssq, 1.0);
  }
  const double wm = (double)c->wm;
  if (!mirror) {
    c->err = c->err + hg2 * fro;
    ADJ(c, ghg2, -1.0 * c->g_err, fro);
    ADJ(c, gfro, -1.0 * c->g_err, hg2);
    c->err = c->err - wm * ssq;
    ADJ(c, gssq, 1.0 * c->g_err, wm);
  } else {
    c->err = c->err + wm * ssq;
    ADJ(c, gssq, -1.0 * c->g_err, wm);
    c->err = c->err - hg2 * fro;
    ADJ(c, ghg2, 1.0 * c->g_err, fro);
    ADJ(c, gfro, 1.0 * c->g_err, hg2);
  }
  for (int k = K - 1; k >= 0; k--) {
    ssq = ssq - c->sq[k];
    ADJ(c, c->g_sq[k], 1.0 * gssq, 1.0);
  }
  RELEASE_F(ssq, 0.0, c->tol);
  for (int k = K - 1; k >= 0; k--)
    for (int j = P - 1; j >= 0; j--) {
      if (j < d) {
        double q = c->qd[k * d + j];
        fro = fro - q * q;
        ADJ(c, c->g_qd[k * d + j], 1.0 * gfro, 2.0 * q);
      } else {
        double q = c->icf[k * P + j];
        fro = fro - q * q;
        ADJ(c, c->g_icf[k * P + j], 1.0 * gfro, 2.0 * q);
      }
    }
  RELEASE_F(fro, 0.0, c->tol);
  RELEASE_F(hg2, 0.5 * c->ga * c->ga, c->tol);
  (void)ghg2;
  return RL_OK;
}

/* the whole function body, forward (f) or inverted (~f) */
static int gmm_body(gmm_ctx *c, int inverted) {
  TRY(gmm_top(c, 0));
  if (!inverted) {
    for (int i = 0; i < c->N; i++) TRY(gmm_point(c, i, 0));
    TRY(gmm_alpha_lse(c, 0));
    TRY(gmm_prior(c, 0));
    c->err = c->err + c->cst;
    ADJ(c, c->g_cst, -1.0 * c->g_err, 1.0);
  } else {
    c->err = c->err - c->cst;
    ADJ(c, c->g_cst, 1.0 * c->g_err, 1.0);
    TRY(gmm_prior(c, 1));
    TRY(gmm_alpha_lse(c, 1));
    for (int i = c->N - 1; i >= 0; i--) TRY(gmm_point(c, i, 1));
  }
  TRY(gmm_top(c, 1));
  return RL_OK;
}

static int all_close_zero(const double *v, long n, double tol) {
  for (long i = 0; i < n; i++)
    if (!(fabs(v[i] - 0.0) <= tol)) return 0;
  return 1;
}

/* gradient(p, GradRequest("gmm", [0.0, alphas, means, icf, x, zeros..., ga, wm, cst],
 *          wrt=["alphas","means","icf"])).  Outputs: *err and the three
 * cotangent arrays (caller-allocated, K, K*d, K*P).  Sequential by
 * construction (scratch is shared across points). */
int orc_gmm_grad_ex(int d, int K, int N, const double *alphas, const double *means,
                    const double *icf, const double *x, double ga, int wm, double cst,
                    double err0, double tol, int invcheck, int fresh, double *err_out,
                    double *resid_out, double *g_alphas, double *g_means, double *g_icf);

int orc_gmm_grad(int d, int K, int N, const double *alphas, const double *means,
                 const double *icf, const double *x, double ga, int wm, double cst, double tol,
                 int invcheck, double *err_out, double *g_alphas, double *g_means,
                 double *g_icf) {
  double resid;
  return orc_gmm_grad_ex(d, K, N, alphas, means, icf, x, ga, wm, cst, 0.0, tol, invcheck, 0,
                         err_out, &resid, g_alphas, g_means, g_icf);
}

/* As orc_gmm_grad with err! = err0 on entry (args[0]); also returns err!
 * after the gradient sweep (*resid_out, the value autodiff.py:169-172
 * compares with err0) whether or not the restoration check passes.
 * fresh = 1 is NOT the reference: the scratch arguments are zeroed per
 * (point, component) as on the device (DESIGN §2 deviation 1), which pins
 * the device's restoration verdict; fresh = 0 is the reference. */
int orc_gmm_grad_ex(int d, int K, int N, const double *alphas, const double *means,
                    const double *icf, const double *x, double ga, int wm, double cst,
                    double err0, double tol, int invcheck, int fresh, double *err_out,
                    double *resid_out, double *g_alphas, double *g_means, double *g_icf) {
  const int P = d * (d + 1) / 2;
  gmm_ctx c;
  memset(&c, 0, sizeof c);
  c.d = d; c.K = K; c.N = N; c.P = P; c.wm = wm; c.chk = invcheck != 0; c.tol = tol;
  c.ga = ga; c.cst = cst; c.x = x; c.alphas = alphas; c.means = means; c.icf = icf;
  c.fresh = fresh != 0;
  const long nscr = (long)K * d + K + d + d + K;
  double *scr = calloc(2 * nscr + (long)N * d, sizeof(double));
  long *dmi = calloc(K, sizeof(long));
  if (!scr || !dmi) {
    free(scr);
    free(dmi);
    return RL_ERR_INVALID;
  }
  c.qd = scr; c.sq = c.qd + K * d; c.xc = c.sq + K; c.qxc = c.xc + d; c.mt = c.qxc + d;
  c.dmi = dmi;
  double *gscr = scr + nscr;
  int rc;
  /* sweeps 1-2: f */
  c.err = err0;
  rc = gmm_body(&c, 0);
  if (rc != RL_OK) goto done;
  const double E = c.err;
  *err_out = E;
  /* sweeps 3-4: ~f in gradient mode, err!.g = 1 (default seed) */
  c.gm = 1;
  memset(g_alphas, 0, K * sizeof(double));
  memset(g_means, 0, (long)K * d * sizeof(double));
  memset(g_icf, 0, (long)K * P * sizeof(double));
  c.g_alphas = g_alphas; c.g_means = g_means; c.g_icf = g_icf;
  c.g_qd = gscr; c.g_sq = c.g_qd + K * d; c.g_xc = c.g_sq + K; c.g_qxc = c.g_xc + d;
  c.g_mt = c.g_qxc + d; c.g_x = gscr + nscr;
  c.g_err = 1.0;
  rc = gmm_body(&c, 1);
  if (rc != RL_OK) goto done;
  /* primal restoration (autodiff.py:169-172): err! back to err0, scratch
   * back to zero */
  *resid_out = c.err;
  if (!(fabs(c.err - err0) <= tol) || !all_close_zero(scr, nscr, tol)) {
    rc = RL_ERR_RESTORE;
    goto done;
  }
  for (int k = 0; k < K; k++)
    if (dmi[k] != 0) {
      rc = RL_ERR_RESTORE;
      goto done;
    }
done:
  free(scr);
  free(dmi);
  return rc;
}
