/*
 * revgpu.h — C ABI of the B200-native reversible-AD gradient kernels.
 *
 * The reference (`revlang`, /root/reference/pkg/src/revlang) is a pure-Python
 * interpreter with no FFI; its hot path is `autodiff.gradient`
 * (autodiff.py:136-180): run f forward, wrap outputs in GVar cells, seed,
 * run the mechanically inverted ~f in gradient mode (numerics.py:435-505
 * adjoint rules), check the primal restoration.  Each entry point below
 * replaces that call for one registered program, batched over independent
 * inputs, as ONE fused forward + reverse-sweep kernel with no tape.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the function name ends in
 *     `_host`; buffers are caller-owned, C-contiguous, row-major.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous; they do not synchronise unless noted.
 *   - Return value: RL_OK, a positive revlang error class (only from the
 *     `_host` calls and argument validation), or a negative usage/CUDA error.
 *   - Per-element reversibility failures are reported in `fail[i]` (one of
 *     the positive codes; 0 = ok), never by aborting the batch: a kernel
 *     cannot throw.  `counters` (device, uint64) accumulate
 *     [0] = total loop trips / work units, [1] = number of failed elements.
 *   - No global mutable state: the library is re-entrant across streams
 *     and host threads.
 */
#ifndef REVGPU_H
#define REVGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RL_ABI_VERSION 1

/* Status / per-element failure codes.  Positive codes name the revlang
 * exception class the reference interpreter raises for the same input
 * (revlang/errors.py). */
enum rl_status {
  RL_OK = 0,
  RL_ERR_POSTCONDITION = 1, /* PostconditionMismatch  errors.py:64; interpreter.py:764-792 */
  RL_ERR_DIRTY_ANCILLA = 2, /* DirtyAncilla           errors.py:68; interpreter.py:738-745 */
  RL_ERR_DOMAIN = 3,        /* RevDomainError         errors.py:87; values.py:343-431      */
  RL_ERR_ITERATOR = 4,      /* LoopIteratorMutated    errors.py:75; interpreter.py:863-884 */
  RL_ERR_RESTORE = 5,       /* RevError "backward pass failed to restore" autodiff.py:169-172 */
  RL_ERR_FUEL = 6,          /* FuelExhausted          errors.py:95; interpreter.py:461-466 */
  RL_ERR_KIND = 7,          /* KindError              errors.py:111                        */
  RL_ERR_INDEX = 8,         /* IndexOutOfBounds       errors.py:103; values.py:172-183     */
  RL_ERR_OVERFLOW = 9,      /* Python OverflowError from math.exp (values.py:362)          */
  RL_ERR_ALIAS = 10,        /* AliasedArguments (generated kernels) interpreter.py:624-658 */
  RL_ERR_ASSERT = 11,       /* AssertFailed @safe assert (generated kernels)               */
  RL_ERR_INVALID = -1,      /* bad argument: null pointer, negative size, bad shape        */
  RL_ERR_CUDA = -2,         /* CUDA runtime error (see rl_last_error())                    */
  RL_ERR_NO_DEVICE = -3     /* no sm_100 device visible                                     */
};

int rl_abi_version(void);
const char *rl_strerror(int code);
/* Message of the last negative status on the calling host thread. */
const char *rl_last_error(void);

/* ------------------------------------------------------------------------
 * Bessel J_nu(z) power series (programs/besselj.rnl).
 * Replaces: gradient(p, GradRequest("besselj", [0.0, nu, z[i]])) for every i
 *   (autodiff.py:136; default seed out!.g = 1.0, autodiff.py:99-110).
 * Outputs: J[i] = primal out!, dJdz[i] = z.g for out!.g = seed, fail[i].
 * thr: the loop threshold literal of the program (1e-16); tol: the
 * ExecOptions.float_tolerance (interpreter.py:39, 1e-9); max_trips: fuel cap
 * on series terms: FuelExhausted for an element needing more trips, -1 for
 * every element that passes the z > 0 check.  The reference's fuel
 * (ExecOptions.max_steps, statement executions per sweep, interpreter.py:
 * 461-466) maps exactly: besselj runs 31 + 6 nu + 22 T statements in each
 * sweep, so max_trips = (max_steps - 31 - 6 max(nu, 0)) div 22 (floor,
 * at least -1); invcheck: ExecOptions.invcheck.
 * counters[0] += sum of the series trips of the elements that succeed (the
 * oracle's definition), counters[1] += failed elements.
 * ---------------------------------------------------------------------- */
int rl_besselj_grad_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, uint8_t *fail, unsigned long long *counters,
                        void *stream);

/* Same computation from HOST buffers (pageable or pinned): chunked
 * host->device copies, kernels and device->host copies pipelined on the
 * library's own streams on `device`.  Synchronous.  Writes sum_trips /
 * n_failed if non-NULL.  This is the entry a reference-side FFI binds. */
int rl_besselj_grad_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                             double seed, int64_t max_trips, int32_t invcheck, double *J,
                             double *dJdz, uint8_t *fail, unsigned long long *sum_trips,
                             unsigned long long *n_failed, int32_t device);

/* ------------------------------------------------------------------------
 * ADBench bundle adjustment Jacobian (programs/ba.rnl).
 * Replaces, per observation i with (c, p) = obs[i]:
 *   gradient(p, GradRequest("ba_proj", [0,0,cams[c],X[p],w[i],feats[i]],
 *            seeds=[("e1!",(),1)] / [("e2!",(),1)], wrt=["cam","X","w"]))
 *   and gradient(p, GradRequest("ba_weight", [0.0, w[i]])).
 * cams: n_cams x 11, X: n_pts x 3, w: n_obs, feats: n_obs x 2,
 * obs: n_obs x 2 int32 (camera index, point index; 0-based).
 * J: n_obs x 31 = [de1/d(cam,X,w) (15), de2/d(cam,X,w) (15), d(1-w^2)/dw].
 * err (optional, may be NULL): n_obs x 3 = [e1, e2, 1 - w^2].
 * Jfeat (optional, may be NULL): n_obs x 4 = [de1/df1, de1/df2, de2/df1,
 * de2/df2], the feature columns of the reference's full jacobian().
 * Out-of-range indices set fail[i] = RL_ERR_INDEX (values.py:172-183).
 * ---------------------------------------------------------------------- */
int rl_ba_jac_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                  const double *X, const double *w, const double *feats, const int32_t *obs,
                  double tol, int32_t invcheck, double *err, double *J, double *Jfeat,
                  uint8_t *fail, unsigned long long *counters, void *stream);

int rl_ba_jac_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                       const double *X, const double *w, const double *feats,
                       const int32_t *obs, double tol, int32_t invcheck, double *err,
                       double *J, uint8_t *fail, unsigned long long *n_failed, int32_t device);

/* ------------------------------------------------------------------------
 * ADBench GMM objective gradient (programs/gmm.rnl).
 * Replaces: gradient(p, GradRequest("gmm", [0.0, alphas, means, icf, x,
 *   zeros..., gamma, m, cst], wrt=["alphas","means","icf"])).
 * alphas: K, means: K x d, icf: K x d(d+1)/2 (d log-diagonal entries, then the
 * strict lower triangle column by column), x: N x d (this call's points).
 * out (device, 1 + K + K*d + K*d(d+1)/2 doubles, OVERWRITTEN):
 *   [err, g_alphas, g_means, g_icf].  With add_param_terms = 0 only the
 *   per-point terms of this shard are produced (for a sum-allreduce across
 *   ranks); with 1 the parameter-only terms (-N_total*lse(alphas), Wishart
 *   prior, cst) are added too.  fail: N per-point flags.
 * counters[0] += the argmax record steps taken over the points (the number
 * of times a later component beats the running max: the data-dependent part
 * of the reference's statement count, see rl_gmm_statement_count),
 * counters[1] += failed points.
 * ws: device workspace of rl_gmm_workspace_bytes() bytes.
 * d <= 128 (the kernels' widest tile): d > 128 is RL_ERR_INVALID and
 * rl_gmm_workspace_bytes returns 0; the Python drop-in sends such calls to
 * the generic compiler's kernel (codegen.py).
 * ---------------------------------------------------------------------- */
size_t rl_gmm_workspace_bytes(int32_t d, int32_t K, int64_t N);
int rl_gmm_grad_f64(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
                    const double *means, const double *icf, const double *x, double gamma,
                    int32_t m, double cst, double tol, int32_t invcheck,
                    int32_t add_param_terms, double *out, uint8_t *fail,
                    unsigned long long *counters, void *ws, size_t ws_bytes, void *stream);

int rl_gmm_grad_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                         const double *means, const double *icf, const double *x, double gamma,
                         int32_t m, double cst, double tol, int32_t invcheck, double *out,
                         unsigned long long *n_failed, int32_t device);

/* rl_gmm_grad_f64's shard form over host buffers: this rank's N of N_total
 * points, add_param_terms on exactly one rank; the caller sum-allreduces out
 * across ranks (the multi-GPU drop-in, bench.py's N>1 e2e). */
int rl_gmm_grad_shard_f64_host(int32_t d, int32_t K, int64_t N, int64_t N_total,
                               const double *alphas, const double *means, const double *icf,
                               const double *x, double gamma, int32_t m, double cst, double tol,
                               int32_t invcheck, int32_t add_param_terms, double *out,
                               unsigned long long *n_failed, int32_t device);

/* ------------------------------------------------------------------------
 * The reference's fuel for gmm (ExecOptions.max_steps counts statement
 * executions per interpreter, interpreter.py:461-466): one sweep of
 * programs/gmm.rnl (the run, and the gradient's uncall alike) executes
 *   N (6 K d^2 + 22 K d + 48 K + 13) + 4 U + 3 K d^2 + 9 K d + 28 K + 4 A + 33
 * statements, U = the points' argmax record steps (counters[0] of the GMM
 * entries), A = those of the alphas' logsumexp (measured on the reference,
 * pinned by tests/golden/gmm_fuel.npz).  FuelExhausted iff it exceeds
 * max_steps.  Host-only arithmetic.
 * ---------------------------------------------------------------------- */
int64_t rl_gmm_statement_count(int32_t d, int32_t K, int64_t N, int64_t U, int64_t A);

/* ------------------------------------------------------------------------
 * The whole gradient() call of gmm on one device, in the reference's order:
 * replaces gradient(p, GradRequest("gmm", [err0, alphas, means, icf, x,
 *   zeros..., gamma, m, cst], wrt=["alphas","means","icf"])) (autodiff.py:
 * 136-180) including its primal-restoration check (autodiff.py:169-172).
 * out[0] = err! after the forward run, accumulated from err0 term by term in
 * the program's order (bit-exactly the sequential binary64 chain over the
 * device's per-point terms; see rl_seq_sum_f64); out[1..] = the cotangents
 * as rl_gmm_grad_f64.  resid (device, 1 double, may be NULL) = err! after
 * the gradient sweep; restore_code (device, int32, may be NULL) =
 * RL_ERR_RESTORE when |resid - err0| > tol (values_close, values.py:562-589;
 * unconditional in the reference: independent of invcheck), else RL_OK.
 * Per-point errors still go to fail / counters and take precedence (the
 * reference raises them before the restoration check).  d <= 128.
 * Workspace: rl_gmm_workspace_bytes(d, K, N).
 *
 * rl_gmm_run_f64 replaces run(p, "gmm", [err0, ...]) (direction +1,
 * interpreter.py:1021) or uncall(...) (direction -1, :1026): err[0] = err!
 * after the forward (inverse) program, accumulated from err0 in its order.
 * rl_gmm_gradient_f64_host: host buffers; returns RL_ERR_RESTORE (outputs
 * written, *resid set) when the restoration check fails.
 * ---------------------------------------------------------------------- */
int rl_gmm_gradient_f64(int32_t d, int32_t K, int64_t N, const double *alphas,
                        const double *means, const double *icf, const double *x, double gamma,
                        int32_t m, double cst, double err0, double tol, int32_t invcheck,
                        double *out, double *resid, int32_t *restore_code, uint8_t *fail,
                        unsigned long long *counters, void *ws, size_t ws_bytes, void *stream);
int rl_gmm_run_f64(int32_t d, int32_t K, int64_t N, const double *alphas, const double *means,
                   const double *icf, const double *x, double gamma, int32_t m, double cst,
                   double err0, double tol, int32_t invcheck, int32_t direction, double *err,
                   uint8_t *fail, unsigned long long *counters, void *ws, size_t ws_bytes,
                   void *stream);
int rl_gmm_gradient_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                             const double *means, const double *icf, const double *x,
                             double gamma, int32_t m, double cst, double err0, double tol,
                             int32_t invcheck, double *out, double *resid,
                             unsigned long long *n_failed, int32_t device);

/* ------------------------------------------------------------------------
 * Sequential binary64 accumulation e_{j+1} = fl(e_j + t_j), j < M, from e0
 * (the reference's `acc += term` statement chain, numerics.py:296-339),
 * evaluated in parallel by one CTA and verified bit-exact against the
 * sequential definition (falls back to it when the verification fails).
 * out2 (device, 2 doubles) = [e_mark, e_M]; verified (device int32, may be
 * NULL) = 1 when the parallel path verified.  force_serial = 1 runs the
 * sequential loop (tests).  t: device, M doubles.
 * ---------------------------------------------------------------------- */
int rl_seq_sum_f64(const double *t, int64_t M, double e0, int64_t mark, int32_t force_serial,
                   double *out2, int32_t *verified, void *stream);

/* ------------------------------------------------------------------------
 * run / uncall / objective-only ("-O") entries: the primal sweeps of the same
 * programs with every reversibility check, no cotangents.
 *
 * rl_besselj_run_f64 replaces run(p, "besselj", [out_in[i], nu, z[i]])
 * (direction +1, interpreter.py:1021) or uncall(...) (direction -1,
 * interpreter.py:1026): out[i] = out_in[i] +/- J_nu(z[i]); out_in may be NULL
 * (zeros).  rl_ba_residuals_f64: run of ba_proj and ba_weight on zero
 * outputs, err = n_obs x 3 [e1, e2, 1 - w^2].  rl_gmm_objective_f64: run of
 * gmm, err[0] = the objective (per-point terms of this shard, plus the
 * parameter terms when add_param_terms); same workspace as the gradient.
 * ---------------------------------------------------------------------- */
int rl_besselj_run_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                       int64_t max_trips, int32_t invcheck, int32_t direction,
                       const double *out_in, double *out, uint8_t *fail,
                       unsigned long long *counters, void *stream);
int rl_ba_residuals_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                        const double *X, const double *w, const double *feats,
                        const int32_t *obs, double tol, int32_t invcheck, double *err,
                        uint8_t *fail, unsigned long long *counters, void *stream);
int rl_gmm_objective_f64(int32_t d, int32_t K, int64_t N, int64_t N_total, const double *alphas,
                         const double *means, const double *icf, const double *x, double gamma,
                         int32_t m, double cst, double tol, int32_t invcheck,
                         int32_t add_param_terms, double *err, uint8_t *fail,
                         unsigned long long *counters, void *ws, size_t ws_bytes, void *stream);

/* Host-buffer forms of the entries above (pinned or pageable host memory;
 * chunked over three streams for Bessel; n_failed = failed elements /
 * points; gmm: argmax_steps = counters[0] for rl_gmm_statement_count). */
int rl_besselj_run_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                            int64_t max_trips, int32_t invcheck, int32_t direction,
                            const double *out_in, double *out, uint8_t *fail,
                            unsigned long long *n_failed, int32_t device);
int rl_ba_residuals_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                             const double *X, const double *w, const double *feats,
                             const int32_t *obs, double tol, int32_t invcheck, double *err,
                             uint8_t *fail, unsigned long long *n_failed, int32_t device);
int rl_gmm_run_f64_host(int32_t d, int32_t K, int64_t N, const double *alphas,
                        const double *means, const double *icf, const double *x, double gamma,
                        int32_t m, double cst, double err0, double tol, int32_t invcheck,
                        int32_t direction, double *err, unsigned long long *n_failed,
                        unsigned long long *argmax_steps, int32_t device);

/* ----------------------------------------------------------------------
 * Batched forward-over-reverse Hessian of besselj:
 * replaces reference autodiff.hessian(p, "besselj", [0.0, nu, z[i]])
 * (autodiff.py:216-257) for every z[i]: the gradient sweeps run over Dual
 * numbers with z carrying the unit tangent, so H[z, z] = d2Jdz2[i]; the
 * other entries of the reference's 2x2 matrix (leaves out!, z) are 0.  J,
 * dJdz, fail and counters are bit-identical to rl_besselj_grad_f64's.
 * ---------------------------------------------------------------------- */
int rl_besselj_hess_f64(int32_t nu, const double *z, int64_t n, double thr, double tol,
                        double seed, int64_t max_trips, int32_t invcheck, double *J,
                        double *dJdz, double *d2Jdz2, uint8_t *fail,
                        unsigned long long *counters, void *stream);
int rl_besselj_hess_f64_host(int32_t nu, const double *z, int64_t n, double thr, double tol,
                             double seed, int64_t max_trips, int32_t invcheck, double *J,
                             double *dJdz, double *d2Jdz2, uint8_t *fail,
                             unsigned long long *n_failed, int32_t device);

/* ----------------------------------------------------------------------
 * BA Jacobian in ADBench's sparse layout (BASparseMat, CSR with int row
 * pointers and column indices).  Same values as
 * rl_ba_jac_f64 (the reference's two seeded gradient(p, GradRequest(
 * "ba_proj", ...)) calls + gradient of ba_weight, autodiff.py:136-180),
 * stored as ADBench's insert_reproj_err_block / insert_w_err_block build
 * it: nrows = 3P, ncols = 11 n_cams + 3 n_pts + P, nnz = 31P;
 *   rows 2i, 2i+1 (i < P): 15 entries each — cols 11c..11c+10 (camera c),
 *     11 n_cams + 3p .. +2 (point p), 11 n_cams + 3 n_pts + i (weight i);
 *   row 2P + i: one entry, col 11 n_cams + 3 n_pts + i, value -2 w_i.
 * A call may produce one shard of the observations: obs_offset is the
 * global index of obs[0] and n_obs_total = P.  The shard's arrays are its
 * two pieces of the global arrays, concatenated:
 *   vals/cols [31 n_obs]   = global [30 off, 30 (off+n_obs)) ++ [30P + off, 30P + off + n_obs)
 *   rows [3 n_obs + 1]     = global rows [2 off, 2 (off+n_obs)) ++ [2P + off, 2P + off + n_obs]
 * (with obs_offset = 0 and n_obs_total = n_obs these are exactly the
 * BASparseMat arrays).  rows and cols are both NULL (values only: the
 * pattern depends on obs alone) or both non-NULL.  Errors: RL_ERR_INVALID
 * when 31P or ncols does not fit int32; per-observation codes in fail[] as
 * for rl_ba_jac_f64.  The _host variant takes whole-problem host arrays.
 * ---------------------------------------------------------------------- */
int rl_ba_jac_csr_f64(int32_t n_cams, int32_t n_pts, int64_t n_obs, int64_t obs_offset,
                      int64_t n_obs_total, const double *cams, const double *X, const double *w,
                      const double *feats, const int32_t *obs, double tol, int32_t invcheck,
                      double *err, int32_t *rows, int32_t *cols, double *vals, uint8_t *fail,
                      unsigned long long *counters, void *stream);
int rl_ba_jac_csr_f64_host(int32_t n_cams, int32_t n_pts, int64_t n_obs, const double *cams,
                           const double *X, const double *w, const double *feats,
                           const int32_t *obs, double tol, int32_t invcheck, int32_t *rows,
                           int32_t *cols, double *vals, uint8_t *fail,
                           unsigned long long *n_failed, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* REVGPU_H */
