/*
 * tf.h -- C ABI of the B200 (sm_100a) dGN evaluation hot path of Tensor Fox
 * (F. Bottega Diniz, "Tensor decompositions and algorithms, with applications
 * to tensor learning", arxiv 2110.05997; PAPER.md line numbers below).
 *
 * Library: paper_2110_05997_b200/libtf.so. Plain C types only.
 *
 * Conventions (all arrays IEEE fp64):
 *   T      dense I x J x K tensor, first index fastest: T[i + ldT*(j + J*k)]
 *          with ldT >= I (Alg. Unfolding: the innermost loop
 *          runs over i_1). Frontal slice T[:,:,k] is a contiguous column-major
 *          block.
 *   w      packed parameters [vec A; vec B; vec C], A (I x R), B (J x R),
 *          C (K_total x R) column-major, n = R*(I+J+K_total).
 *          grad, v, y, rhs, x use the same layout.
 *   grams  [A^T A | B^T B | C^T C], each R x R column-major.
 *   pi     [Pi^(1) | Pi^(2) | Pi^(3) | Pi^(1,2) | Pi^(1,3) | Pi^(2,3)], R x R each
 *          (for L = 3, Pi^(l',l'') = pi^(l) of the third mode).
 *
 * K-sharding (data parallel over frontal slices): a call may hold only slices
 * k_begin .. k_begin+K-1 of a tensor with K_total slices (T points at slice
 * k_begin); w always holds the full C (K_total rows).
 *
 * Ownership: every pointer argument is caller-owned memory. Device pointers
 * (all arguments of the non-_host calls) must be on the ctx's device; the
 * library never frees or retains them beyond the call. The ctx owns its
 * workspace (partial-sum buffers, TMA descriptors, CG vectors), grows it on
 * demand and frees it in tf_ctx_destroy; steady-state calls allocate nothing.
 *
 * Asynchrony: calls are enqueued on the ctx stream and return before the GPU
 * finishes (except tf_cg_solve's host outputs and the _host variants, which
 * synchronize the stream). Outputs are valid after the stream is synchronized.
 *
 * Errors: every call returns a tf_status; nothing is thrown or exits across
 * the ABI. TF_ERR_ARG: null pointer, a dimension < 1, ldT < I, or
 * k_begin + K > K_total. TF_ERR_ALIGN: T not 8-byte aligned. TF_ERR_UNSUPPORTED:
 * R above TF_MAX_R. TF_ERR_CUDA: a launch or runtime error (detail in
 * tf_last_error). TF_ERR_NONFINITE: CG met a non-finite alpha/beta (iteration
 * index in tf_last_error). TF_ERR_ALLOC: workspace allocation failed.
 */
#ifndef TF_H_
#define TF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_MAX_R 128

typedef enum {
  TF_OK = 0,
  TF_ERR_ARG = 1,
  TF_ERR_ALIGN = 2,
  TF_ERR_UNSUPPORTED = 3,
  TF_ERR_CUDA = 4,
  TF_ERR_NONFINITE = 5,
  TF_ERR_ALLOC = 6
} tf_status;

typedef struct tf_ctx tf_ctx;

/* I, J: full mode sizes; K: local number of frontal slices; R: CPD rank;
 * ldT: leading dimension of T (>= I, 0 means I); K_total: slices of the whole
 * tensor (0 means K); k_begin: global index of the first local slice. */
typedef struct {
  int64_t I, J, K, R, ldT, K_total, k_begin;
} tf_dims;

/* Create a context bound to CUDA device `device`, enqueueing on `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream). */
tf_status tf_ctx_create(tf_ctx **out, int device, void *cuda_stream);
tf_status tf_ctx_destroy(tf_ctx *ctx);
/* Re-target the ctx to another stream of the same device. */
tf_status tf_ctx_set_stream(tf_ctx *ctx, void *cuda_stream);
const char *tf_status_str(tf_status s);
/* Detail of the last error on this ctx (offending argument, CG iteration, CUDA message). */
const char *tf_last_error(const tf_ctx *ctx);
int tf_version(void);

/* a1: pi^(l) = W^(l)^T W^(l) for the three modes. grams: 3*R*R doubles. */
tf_status tf_grams(tf_ctx *ctx, tf_dims d, const double *w, double *grams);

/* a7: Hadamard chains from the Grams. pi: 6*R*R doubles. */
tf_status tf_hadamard(tf_ctx *ctx, int64_t R, const double *grams, double *pi);

/* a2-a6: one evaluation on the local slices.
 *   f    (1 double)  F = 1/2 ||T - [[A,B,C]]||^2 over the local slices
 *   grad (n doubles) grad F = J_f^T f = W Pi - T_(l)(.W).
 *        With K < K_total, the dF/dA and dF/dB blocks and f are partial sums over
 *        the local slices and dF/dC holds rows k_begin..k_begin+K-1 (other rows 0):
 *        an elementwise SUM over shards of [grad | f] gives the global result.
 *   grams (nullable, 3*R*R) the Grams of the full factors at w, exactly what tf_grams returns, also
 *        for a K-shard (C^T C over all K_total rows); the evaluation forms most of them anyway.
 * The three MTTKRPs are fused in one pass over T: by default the guarded Pi form (grad = W Pi - M,
 * f by the Gram expansion, rerun in the residual form on the device when cancellation would cost
 * accuracy; reading R31), or the residual form (tf_ctx_set_eval_form). */
tf_status tf_cpd_eval(tf_ctx *ctx, tf_dims d, const double *T, const double *w, double *f, double *grad,
                      double *grams);

/* Same as tf_cpd_eval with HOST inputs/outputs (pageable or pinned). T is streamed
 * to the device in slabs of frontal slices overlapped with the fused kernel, so
 * T need not fit in device memory. Synchronizes the ctx stream before returning. */
tf_status tf_cpd_eval_host(tf_ctx *ctx, tf_dims d, const double *T_host, const double *w_host, double *f_host,
                           double *grad_host);

/* a8: y = (J_f^T J_f + lambda I) v by Thm Hv, from the Grams
 * at w (grams as produced by tf_grams) and w itself (Thm Hv's off-diagonal blocks
 * need the factors). v, y: n doubles (y must not alias v). */
tf_status tf_gn_matvec(tf_ctx *ctx, tf_dims d, const double *grams, const double *w, const double *v,
                       double lambda, double *y);

/* a9: Alg. CG-dGN: solve (J^T J + lambda I) x = rhs with
 * x0 = 0, at most maxiter iterations, stopping when ||r||^2 < tol (tol = 0: run
 * exactly maxiter; rhs = 0 returns x = 0 after zero iterations, reading R33). jacobi != 0 preconditions with M = diag(J^T J) + lambda I as
 * M^{-1/2} (.) M^{-1/2} and returns x in
 * w-coordinates (x = M^{-1/2} x_hat). The iteration runs on the device with no
 * host round trip; iters_done and res2 (host pointers, nullable) receive the
 * number of iterations run and the final ||r||^2 after a stream synchronize.
 * x: n doubles (device). Returns TF_ERR_NONFINITE if alpha or beta became
 * non-finite (x then holds the last finite iterate). */
tf_status tf_cg_solve(tf_ctx *ctx, tf_dims d, const double *grams, const double *w, const double *rhs,
                      double lambda, int maxiter, double tol, int jacobi, double *x, int *iters_done,
                      double *res2);

/* NEXT #1 -- Tensor Fox's own damping ("Diagonal regularization"): the CG system
 * is (J^T J + mu D) x = rhs with D = diag(gamma_l^(r) I_{I_l}) and
 *   G = max_r' max{ ||Y_r'|| ||Z_r'||, ||X_r'|| ||Z_r'||, ||X_r'|| ||Y_r'|| },
 *   gamma_X^(r) = ||Y_r|| ||Z_r|| G,  gamma_Y^(r) = ||X_r|| ||Z_r|| G,  gamma_Z^(r) = ||X_r|| ||Y_r|| G
 * (X, Y, Z = A, B, C), which makes every row of J^T J + D dominate its off-diagonal entries. */

/* gamma (3*R doubles, device) = [gamma_X | gamma_Y | gamma_Z] from the Grams (||W_r||^2 = pi^(l)_rr). */
tf_status tf_reg_gamma(tf_ctx *ctx, int64_t R, const double *grams, double *gamma);

/* y = (J^T J + mu D) v, D = diag over (mode, r) of damp (3*R doubles, device; NULL = identity, i.e.
 * tf_gn_matvec). Same layouts and rules as tf_gn_matvec. */
tf_status tf_gn_matvec_damped(tf_ctx *ctx, tf_dims d, const double *grams, const double *w, const double *v, double mu,
                              const double *damp, double *y);

/* Alg. CG-dGN on (J^T J + mu D) x = rhs; with jacobi != 0 the preconditioner is
 * M = diag(J^T J) + mu diag(D). damp NULL = identity (tf_cg_solve). */
tf_status tf_cg_solve_damped(tf_ctx *ctx, tf_dims d, const double *grams, const double *w, const double *rhs,
                             double mu, const double *damp, int maxiter, double tol, int jacobi, double *x,
                             int *iters_done, double *res2);

/* NEXT #2 -- the damped Gauss-Newton outer loop of Tensor Fox around the hot path,
 * run by the library on the device (one host synchronisation per dGN iteration). Iteration k:
 *   x = CG-dGN on (J^T J + mu D) x = -grad F(w) with cg_iters[k-1] iterations, CG tolerance tol
 *       (D = Tensor Fox's gamma if use_gamma else I; Jacobi M = diag(J^T J) + mu diag(D) if jacobi);
 *   w += x; norm balancing if balance; F, grad at the new w (fused evaluation);
 *   gain ratio g = (F_old - F_new) / (-<grad_old, x> - 1/2 x^T J^T J x);
 *   g < 0.25 -> mu *= 3, g > 0.75 -> mu /= 3; stopping conditions 1-7.
 * mu^(0) = mu0 if > 0 else mean |T| (tau = 1). cg_iters (host) holds the random CG budgets
 * drawn by the caller from [1 + ceil(k^0.4), 2 + ceil(k^0.9)]. */
typedef struct {
  int maxiter;          /* dGN iterations (paper default 200) */
  double tol;           /* every stopping tolerance and the CG tolerance (paper default 1e-6) */
  double mu0;           /* initial damping; <= 0 selects mean |T| */
  int use_gamma;        /* 1: damping mu*D with Tensor Fox's gamma; 0: mu*I */
  int jacobi;           /* 1: Jacobi-preconditioned CG */
  int balance;          /* 1: norm-balance the factors after every step */
  const int *cg_iters;  /* host, >= maxiter entries */
} tf_dgn_params;

typedef struct {
  int iters;            /* dGN iterations done */
  int reason;           /* 0 maxiter; 1..7 stopping condition of PAPER.md:2756-2773; 8 non-finite */
  double f;             /* F at the returned w */
  double rel_err;       /* ||T - [[A,B,C]]|| / ||T|| */
  double mu;            /* damping after the last update */
} tf_dgn_result;

/* Runs the dGN loop from w (device, n doubles, overwritten with the result). Requires the whole tensor
 * (K == K_total). hist (host, nullable): 5 doubles per iteration [F, rel_err, mu used, g, ||x||]. */
tf_status tf_cpd_dgn(tf_ctx *ctx, tf_dims d, const double *T, double *w, const tf_dgn_params *prm,
                     tf_dgn_result *res, double *hist);

/* ---------------------------------------------------------------------------------------------------
 * NEXT #3 -- compression before the path (Tensor Fox section "Compression"): the
 * truncated MLSVD of T (Alg. MLSVD; Thm MLSVD 1296-1301) with each mode's SVD taken
 * through the unfolding Gram T_(l) T_(l)^T (Remark MLSVD-SVD 4446-4448, Lemma svd-transpose 4434-4436)
 * and truncated to P_l = min(I_l, R) singular values, the rank choice of Alg. Compression
 * (2566-2583), the MLSVD-energy initialisation (2600-2605) and the uncompression W~ = U W (2857-2868).
 * All pointers are device memory unless stated; matrices are column-major with the leading dimension
 * equal to their row count; these calls need the whole tensor (K == K_total, k_begin == 0).
 * Readings: R23 singular-vector signs -- the largest-magnitude entry of every column of U_l
 * is positive; R25 energy initialisation -- the R entries of largest |s| (ties: storage order), the
 * coefficient on mode 1. */

/* G_l = T_(l) T_(l)^T for l = 1, 2, 3 (I x I, J x J, K x K, symmetric, full storage); any output may be
 * NULL to skip that mode. Entry (p, q) is the inner product of the mode-l hyperslices i_l = p and q
 * (PAPER.md:1293). */
tf_status tf_unfolding_grams(tf_ctx *ctx, tf_dims d, const double *T, double *G1, double *G2, double *G3);

/* Top-P eigenpairs of a symmetric positive semidefinite n x n matrix G (the unfolding Gram) by subspace
 * iteration from the n x P start block Omega (seeded N(0,1), drawn by the caller: the randomized range
 * finder of PAPER.md:1424 / rand_svd) with Householder orthonormalisation and a Rayleigh-Ritz step
 * (Jacobi) per iteration, until every Ritz residual ||G u_j - lam_j u_j|| <= max(tol, 16 sqrt(n) 2^-53)
 * |lam_1| (or it stagnates at the fp64 floor, or maxiter). Outputs: U (n x P, orthonormal, R23 signs),
 * lam (P, sorted by |lam| decreasing); iters (host, nullable) = iterations done. 1 <= P <= min(n, 128). */
tf_status tf_sym_eig_top(tf_ctx *ctx, int64_t n, const double *G, int64_t P, const double *Omega, int maxiter,
                         double tol, double *U, double *lam, int *iters);

/* S = (U1^T, U2^T, U3^T) . T, the multilinear product of the MLSVD core, computed as
 * three DMMA GEMMs over chunks of frontal slices (mode 1, then mode 2 per slice, then mode 3). U1 (I x P1),
 * U2 (J x P2), U3 (K x P3); S (P1 x P2 x P3, first index fastest). P_l <= 128. */
tf_status tf_multilinear_core(tf_ctx *ctx, tf_dims d, const double *T, const double *U1, int64_t P1,
                              const double *U2, int64_t P2, const double *U3, int64_t P3, double *S);

/* Alg. Compression with d.R as the target CPD rank. Omega: start blocks [I x P1 | J x P2 | K x P3]
 * (P_l = min(I_l, R)). Outputs: U = [U1 | U2 | U3] in the same layout (all P_l columns; the first R~_l
 * are U~_l), sigma = [sigma^(1) | sigma^(2) | sigma^(3)] (P_l each, decreasing), S = the truncated core
 * S~ (R~1 x R~2 x R~3, first index fastest; capacity P1*P2*P3), ranks (host, 3) = (R~1, R~2, R~3):
 * for each mode the first i with sum_{r>i} sigma_r^2 / sum_{r<=P_l} sigma_r^2 < mlsvd_tol / 3.
 * eig_iters (host, nullable, 3). Synchronizes the stream (the ranks size the core). */
tf_status tf_compress(tf_ctx *ctx, tf_dims d, const double *T, const double *Omega, double mlsvd_tol,
                      int eig_maxiter, double eig_tol, double *U, double *sigma, double *S, int64_t *ranks,
                      int *eig_iters);

/* Alg. ST-MLSVD, the sequentially truncated variant Tensor Fox can switch to (1439):
 * mode 1's SVD from T_(1) T_(1)^T, then X1 = U~1^T T_(1); mode 2's from the Gram of X1's mode-2 unfolding,
 * X2 = X1 x_2 U~2^T; mode 3's from X2's, S = X2 x_3 U~3^T. Each step's rank follows Alg. Compression's rule
 * on that step's singular values (reading R32). Same arguments and layouts as tf_compress (sigma holds each
 * step's singular values; U_l all P_l columns). Cheaper than tf_compress: after mode 1 every pass reads the
 * R~1 x J x K intermediate instead of T. */
tf_status tf_compress_st(tf_ctx *ctx, tf_dims d, const double *T, const double *Omega, double mlsvd_tol,
                         int eig_maxiter, double eig_tol, double *U, double *sigma, double *S, int64_t *ranks,
                         int *eig_iters);

/* K-sharded Alg. ST-MLSVD: this rank holds slices k_begin .. k_begin+K-1 (d.K local, d.K_total global). The
 * mode-1 and mode-2 Grams are sums over slices and are summed over the ranks through the all-reduce hook
 * (tf_allreduce_fn: the contract described at tf_cpd_dgn_sharded); mode 3 needs every slice of X2 = T x1 U~1^T x2 U~2^T,
 * which each rank writes into its columns of a zeroed R~1 R~2 x K_total buffer completed by the same hook.
 * Outputs as tf_compress_st, identical on every rank (U3 has K_total rows). xbuf (device, caller-owned) must
 * hold max(I^2, J^2, P1 P2 K_total) doubles. */
typedef int (*tf_allreduce_fn)(double *buf, int64_t count, void *user);
tf_status tf_compress_st_sharded(tf_ctx *ctx, tf_dims d, const double *T_local, const double *Omega,
                                 double mlsvd_tol, int eig_maxiter, double eig_tol, double *U, double *sigma,
                                 double *S, int64_t *ranks, int *eig_iters, tf_allreduce_fn allreduce, void *user,
                                 double *xbuf);

/* MLSVD-energy initialisation on the core S (R1 x R2 x R3): w = [vec W1; vec W2; vec W3] (R*(R1+R2+R3))
 * with W1[:, r] = s_j e_{j1}, W2[:, r] = e_{j2}, W3[:, r] = e_{j3} for the R entries j of largest |s|. */
tf_status tf_energy_init(tf_ctx *ctx, int64_t R1, int64_t R2, int64_t R3, const double *S, int64_t R, double *w);

/* Uncompression of one mode: out (n x R) = U (n x Rl) . W (Rl x R). */
tf_status tf_uncompress(tf_ctx *ctx, int64_t n, int64_t Rl, const double *U, const double *W, int64_t R,
                        double *out);

/* The whole Tensor Fox flow (flow chart "Compression -> Initialization -> dGN ->
 * Uncompression"): tf_compress of T to the R~1 x R~2 x R~3 core; the starting point on the core from the
 * MLSVD-energy initialisation (init = 1) or from w0_core (init = 0: rows 0..R~_l-1 of each block of
 * [W1 (P1 x R) | W2 (P2 x R) | W3 (P3 x R)], e.g. N(0,1) entries drawn by the caller);
 * tf_cpd_dgn on the core; uncompression W~_l = U~_l W_l; and the output form with unit columns and
 * lambda_r = prod_l ||W~_l[:, r]||. W (device, R*(I+J+K), w layout) gets the unit
 * factors, lambda (device, R) the weights. res->rel_err is ||T - sum_r lambda_r w_r^(1) (x) w_r^(2) (x)
 * w_r^(3)|| / ||T|| on the ORIGINAL tensor, from one fused evaluation. hist (host, nullable): the dGN
 * history on the core (5 doubles per iteration, as tf_cpd_dgn). Synchronizes the stream. */
typedef struct {
  double mlsvd_tol;       /* Alg. Compression tolerance */
  int eig_maxiter;        /* subspace-iteration cap per mode */
  int init;               /* 1: MLSVD-energy initialisation; 0: w0_core */
  tf_dgn_params dgn;      /* the dGN loop on the core */
  int sequential;         /* 1: compress by Alg. ST-MLSVD (tf_compress_st) instead of the classic MLSVD */
} tf_cpd_params;

typedef struct {
  int64_t ranks[3];       /* R~1, R~2, R~3 */
  int eig_iters[3];
  tf_dgn_result dgn;      /* on the core */
  double rel_err;         /* on the original tensor */
} tf_cpd_result;

tf_status tf_cpd(tf_ctx *ctx, tf_dims d, const double *T, const double *Omega, const double *w0_core,
                 const tf_cpd_params *prm, double *W, double *lambda, tf_cpd_result *res, double *hist);

/* The flow on a K-sharded tensor (T_local = slices k_begin .. k_begin+K-1): compression by
 * tf_compress_st_sharded (always ST-MLSVD), then the dGN on the core, the uncompression and the unit-column
 * form replicated on every rank; the final fit sums the ranks' partial F and ||T||^2 through the hook.
 * xbuf as for tf_compress_st_sharded (>= 3 doubles in any case). */
tf_status tf_cpd_sharded(tf_ctx *ctx, tf_dims d, const double *T_local, const double *Omega, const double *w0_core,
                         const tf_cpd_params *prm, double *W, double *lambda, tf_cpd_result *res, double *hist,
                         tf_allreduce_fn allreduce, void *user, double *xbuf);

/* ---------------------------------------------------------------------------------------------------
 * NEXT #4 -- CP-ALS (Alg. ALS), the second workload on the slice-streaming MTTKRP. */

/* M = T_(mode) (W^(L) ⊙ ... ⊙ W^(mode+1) ⊙ W^(mode-1) ⊙ ... ⊙ W^(1)) (Thm unfolding-formula2's order,
 * PAPER.md:1282-1285): I_mode x R, column-major. Runs as DMMA GEMMs over chunks of the materialised
 * Khatri-Rao product (<= 512 MB each). K-sharded calls: modes 1 and 2 give the partial sum over the local
 * slices, mode 3 the local rows k_begin .. k_begin+K-1 (M is K x R). */
tf_status tf_mttkrp(tf_ctx *ctx, tf_dims d, const double *T, const double *w, int mode, double *M);

/* `sweeps` sweeps of Alg. ALS from w (device, updated in place): for l = 1, 2, 3 in turn,
 * W^(l) = T_(l) (⊙ others) ((* others' Grams))^dagger (Thm special-products 11-12), the
 * pseudo-inverse taken from the Jacobi eigen-decomposition with numpy's cut-off (eigenvalues below
 * 1e-15 x the largest are dropped; reading R30). f_hist (host, nullable, 3*sweeps): F after every update,
 * from one fused evaluation each (extra passes over T). Needs the whole tensor (K == K_total). */
tf_status tf_als(tf_ctx *ctx, tf_dims d, const double *T, double *w, int sweeps, double *f_hist);

/* How tf_cpd_eval forms F and grad F (both give the same values to fp64 accuracy; reading R31):
 *   0 (default, auto): form 2 when the evaluation is large enough to amortise its extra launches
 *     (6*I*J*K*R >= 5e9 flops), else form 1;
 *   2 guarded Pi form at any size: one pass over T computes the three MTTKRPs T_(l)(.W) (two DMMA slice
 *     contractions, 4*I*J*K*R flops; PAPER.md:2641 grad = W Pi - T_(l)(.W)) and F = 1/2||T||^2 - <A, M1> +
 *     1/2 sum(piA * piB * piC); when cancellation makes that unsafe (2F < 1e-3 ||T||^2 or
 *     ||grad|| < 1e-3 ||W Pi||, i.e. near an exact fit or a stationary point) the residual form is rerun
 *     on the device automatically;
 *   1 residual form always: E_k = T_k - A diag(c_k) B^T in registers, F = 1/2 sum E^2, grad = J^T f
 *     (three contractions, 6*I*J*K*R flops). The environment variable TF_EVAL_FORM=residual selects 1
 *     for new contexts. */
tf_status tf_ctx_set_eval_form(tf_ctx *ctx, int form);
/* Synchronizes and reports whether the last evaluation on this ctx ran the guarded Pi form and fell back
 * to the residual form (1), ran it without falling back (0), or did not run the Pi form at all (-1: no
 * evaluation yet, or the last one was a residual-form evaluation). */
tf_status tf_ctx_eval_fallback(tf_ctx *ctx, int *fell_back);
/* Which load path the last tf_cpd_eval on this ctx ran (the library may fall back instead
 * of failing on alignment, but must say which path it ran): *tma = 1 when the frontal-slice tiles were
 * staged by TMA (cp.async.bulk.tensor; T 16-byte aligned and ldT even), 0 when T is not 16-byte aligned or
 * ldT is odd and the kernel loaded the tiles with cooperative 8-byte loads, -1 before the first evaluation.
 * Both paths compute the same values. */
tf_status tf_ctx_eval_path(tf_ctx *ctx, int *tma);

/* Test/diagnostic knob for the persistent CG and GN-matvec kernel (rows a8/a9): nblocks > 0 launches the
 * grid kernel with min(nblocks, #SMs) blocks (and never the single-CTA kernel for small systems), so that
 * every block processes several work items at small sizes, as it does at c5 on the full grid; 0 (default)
 * restores the normal choice (all SMs; one CTA for n <= 4096). Same arithmetic and the same results to
 * rounding; TF_ERR_ARG if nblocks < 0. */
tf_status tf_ctx_set_cg_grid(tf_ctx *ctx, int nblocks);

/* K-sharded dGN loop: every rank holds slices k_begin .. k_begin+K-1 of T (d.K local,
 * d.K_total global) and the full w; each evaluation's partial [grad | F] and the tensor sums are summed over
 * the ranks through the caller's all-reduce hook, everything else (Grams, gamma, CG, balancing, damping,
 * stopping) runs replicated, so every rank returns the same w. The hook is called from the host thread
 * after the library synchronized its stream, with `buf` = xbuf (device, caller-owned, >= n + 1 doubles,
 * n = R(I+J+K_total)) holding `count` doubles; it must replace them with their elementwise SUM over the
 * ranks (e.g. an NCCL all-reduce of the tensor that owns xbuf) before returning 0 (nonzero -> TF_ERR_CUDA). */
tf_status tf_cpd_dgn_sharded(tf_ctx *ctx, tf_dims d, const double *T_local, double *w, const tf_dgn_params *prm,
                             tf_dgn_result *res, double *hist, tf_allreduce_fn allreduce, void *user, double *xbuf);

/* Instrumentation (bench.py): when enabled, the fused evaluation kernel is
 * bracketed by CUDA events on the ctx stream; tf_ctx_kernel_stats synchronizes
 * and returns the summed device time (ms) and count of the fused-kernel launches
 * since the last reset, plus the total number of kernels this ctx launched. */
tf_status tf_ctx_set_timing(tf_ctx *ctx, int enable);
tf_status tf_ctx_kernel_stats(tf_ctx *ctx, double *eval_kernel_ms, int64_t *eval_kernel_launches,
                              int64_t *total_launches, int reset);

#ifdef __cplusplus
}
#endif

#endif /* TF_H_ */
