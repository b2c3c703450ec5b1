// Internal declarations shared by the C-ABI host code and the kernels.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tfk {

struct EvalArgs {
  const double* A;  // I x R column-major
  const double* B;  // J x R
  const double* C;  // K_total x R
  int64_t I, J, K, R, ldT, Ktot, kbeg;
  int nTi, nTj, kSplit, nCta;
  int64_t kChunk, Ipad, Jpad;
  int64_t unitsPerCta;   // stream-K: (tile, slice) units per CTA of the persistent grid
  int streamK;           // 1: stream-K segments (kSplit = partial slots per tile); 0: one k-chunk per CTA
  int tma4;              // 1: interior i-tiles load through the 4-D map (no over-read of the 4 padding rows)
  int decouple;          // 1: Pi-form pass with the two warp groups decoupled (mbarrier hand-offs, no per-slice
                         //    block barrier; used by the instantiations that support it, ignored elsewhere)
  int skewNs;            // decoupled pass: head start of warp group 0 over group 1 at each segment start
  double* gAp;  // [nTj*kSplit][Ipad][RP]
  double* gBp;  // [nTi*kSplit][Jpad][RP]
  double* gCp;  // [nTi*nTj][K][RP]
  double* fp;   // [nCta]
  const int* run_if;   // nullable: the kernel runs only if *run_if != 0 (guarded fallback)
};

// Pi-form evaluation (PAPER.md:2641 grad = W Pi - T_(l)(.W); f by the Gram expansion), guarded:
//   launch_eval(..., recon = false) writes the three MTTKRPs of T and sum t^2 into the partials;
//   launch_eval_finalize_pi forms grad = W Pi - M and per-block partials of <A, M1>, ||grad||^2, ||W Pi||^2;
//   launch_eval_pi_guard sums them, writes f and *flag = 1 when cancellation makes the expansion unsafe
//   (2f < 1e-3 ||T||^2 or ||grad|| < 1e-3 ||W Pi||), in which case the residual form is rerun (run_if = flag).
cudaError_t launch_eval_finalize_pi(const EvalArgs& p, int RP, double* grad, double* part, int nblk,
                                    cudaStream_t st);
cudaError_t launch_eval_pi_guard(const EvalArgs& p, const double* grams, const double* part, int nblk, double* f,
                                 int* flag, cudaStream_t st, bool check_grad = true);
int eval_pi_blocks(int nsm);

// map[0]: the 3-D TMA view of T, map[1]: the 4-D view of its whole i-tiles (used when p.tma4)
cudaError_t launch_eval(const CUtensorMap* map, const double* T, const EvalArgs& p, int NT, bool tma, int BT,
                        cudaStream_t st, bool recon = true);
cudaError_t launch_eval_finalize(const EvalArgs& p, int RP, double* f, double* grad, int nsm, cudaStream_t st);
size_t eval_smem_bytes(int NT, int BT);
int eval_ctas_per_sm(int NT, bool recon);   // resident CTAs per SM of the 64-wide tile kernel

// ---- small kernels (k_small.cu)
struct Modes {
  const double* W[3];
  int64_t n[3];
  int64_t off[3];  // offsets of the modes in a packed vector
  int64_t R;
};

// grams[l] = W_l^T W_l (3 R x R, column-major); Gpart: gram_partial_slots(m) * 3 R^2 doubles of scratch
cudaError_t launch_grams_ws(const Modes& m, double* Gpart, double* grams, cudaStream_t st);
int gram_partial_slots(const Modes& m);
int cg_partial_slots(const Modes& m);
cudaError_t launch_jacobi_scale(const Modes& m, const double* pi, double lambda, const double* damp, double* dscale,
                                cudaStream_t st);
cudaError_t launch_reg_gamma(int64_t R, const double* grams, double* gamma, cudaStream_t st);

struct MatvecWs {
  double* G;       // Gram partials of the persistent kernel
  double* S;       // 3 R x R : sum_{l' != l} Pi^(l,l') * G_l'
  double* pi;      // 6 R x R
  double* dscale;  // 3R : Jacobi scale per (mode, r)
  double* partial; // per-block partial sums
  int nblk_dot;
};
// pi = [Pi1 | Pi2 | Pi3 | Pi12 | Pi13 | Pi23]
cudaError_t launch_hadamard(int64_t R, const double* grams, double* pi, cudaStream_t st);

struct CgState {
  double rr;      // ||r||^2 (current)
  double alpha, beta, pz;
  double rr0;
  int iters;
  int done;       // 1 once ||r||^2 < tol or non-finite
  int nonfinite;  // iteration index (1-based) at which alpha/beta became non-finite, else 0
  unsigned int counter;
  unsigned int counter2;
};

// Persistent cooperative CG (mode 0) or single GN matvec y = (J^T J + lambda I) v into x (mode 1).
// part: 2 * nsm doubles; G: 3 R^2; st_dev receives iters / final ||r||^2 / non-finite iteration.
cudaError_t launch_cg_persistent(const Modes& m, const double* pi, const double* dscale, const double* damp,
                                 double lambda, double tol,
                                 int maxiter, const double* rhs, const double* v, double* x, double* r, double* p,
                                 double* z, double* G, double* S, double* part, CgState* st_dev, int mode, int grid,
                                 bool allow_small, cudaStream_t st);
size_t cg_gram_partial_doubles(int64_t R);
// Row-owned persistent CG (k_cg_rows.cu): used by launch_cg_persistent when cg_rows_fits()
bool cg_rows_fits(const Modes& m, int grid, size_t gram_partial_doubles);
cudaError_t launch_cg_rows(const Modes& m, const double* pi, const double* dscale, const double* damp, double lambda,
                           double tol, int maxiter, const double* rhs, const double* v, double* x, double* G,
                           double* S, double* part, CgState* st_dev, int mode, int grid, cudaStream_t st);

// dGN outer-loop helpers (k_small.cu)
cudaError_t launch_dots(int64_t n, const double* g, const double* x, const double* y, double* partial, double* out,
                        cudaStream_t st);   // out = {g.x, x.y, x.x, max|g|}; partial: red_blocks()*4
cudaError_t launch_tsums(int64_t I, int64_t J, int64_t K, int64_t ldT, const double* T, double* partial, double* out,
                         cudaStream_t st);  // out = {sum|t|, sum t^2}; partial: red_blocks()*2
cudaError_t launch_axpy_inplace(int64_t n, const double* x, double* w, const CgState* gate, cudaStream_t st);
cudaError_t launch_scale_copy(int64_t n, double alpha, const double* x, double* y, cudaStream_t st);
cudaError_t launch_balance(const Modes& m, const double* grams, double* w, const CgState* gate, cudaStream_t st);
int red_blocks();

// y += x (n doubles), used by the host-streamed evaluation
cudaError_t launch_axpy1(int64_t n, const double* x, double* y, cudaStream_t st);

// ---- compression stage (NEXT #3): generic DMMA GEMM (k_gemm.cu) and eigen/QR kernels (k_eig.cu)
struct GemmOperand {
  const double* ptr;
  int64_t ld;       // X[p, k] = ptr[k + ld*p] (kc) or ptr[p + ld*k] (!kc)
  int64_t bstride;  // batch stride (0: the same operand for every batch)
  bool kc;
};
// C[m, n] = alpha * sum_b sum_k A_b[m, k] B_b[n, k] + beta * C
struct GemmArgs {
  GemmOperand a, b;
  int64_t M, N, Kd, batch;
  bool sum_batch;      // batches summed into one C, else one C per batch (cstride apart)
  bool sym;            // A == B: only tiles tn >= tm, mirrored
  int64_t out_batches; // sum_batch ? 1 : batch
  double* C;
  int64_t ldc, cstride;
  double alpha, beta;
  int BM, BN;
  int64_t ntm, ntn;
  int ksplit;
  int64_t steps_per_split;
  double* part;        // [items][ksplit][BM*BN] when ksplit > 1
};
cudaError_t launch_gemm(const CUtensorMap* ma, const CUtensorMap* mb, const GemmArgs& g, int64_t items, bool tma,
                        cudaStream_t st);
size_t gemm_smem_bytes(int BM, int BN, bool akc, bool bkc);
constexpr int kGemmBK = 32;

// Householder QR of Z (n x P, ld) -> Q with orthonormal columns spanning Z (Z is overwritten)
cudaError_t launch_house_qr(int64_t n, int P, double* Z, int64_t ldz, double* Q, int64_t ldq, cudaStream_t st);
// W[:, j] = Z[:, j] / ||Z[:, j]||; *fail = 1 on a zero column
cudaError_t launch_col_normalize(int64_t n, int P, const double* Z, int64_t ldz, double* W, int64_t ldw, int* fail,
                                 cudaStream_t st);
// B = L L^T (P x P) and Linv = L^{-1}; *fail = 1 when a pivot is below 1e-8
cudaError_t launch_chol_inv(int P, const double* B, double* Linv, int* fail, cudaStream_t st);
// symmetric eigen-decomposition of (H + H^T)/2 (P x P) by parallel cyclic Jacobi in one CTA:
// theta sorted by |theta| decreasing, V (P x P, ld P) the matching eigenvectors; Vtmp: P*P scratch
cudaError_t launch_jacobi_eig(int P, const double* H, int64_t ldh, double* Vtmp, double* V, double* theta,
                              cudaStream_t st, int max_sweeps = 60);
// res[j] = || ZV[:, j] - theta_j U[:, j] ||_2
cudaError_t launch_eig_residual(int64_t n, int P, const double* ZV, const double* U, int64_t ld, const double* theta,
                                double* res, cudaStream_t st);
// reading R23: make the largest-magnitude entry of every column positive (first on ties)
cudaError_t launch_sign_fix(int64_t n, int P, double* U, int64_t ld, cudaStream_t st);
// sigma = sqrt(|lam|)
cudaError_t launch_sqrt_abs(int64_t n, const double* lam, double* sigma, cudaStream_t st);
// Alg. Compression rank choice for one mode: first i with sum_{r>i} s_r^2 / sum s_r^2 < tol3 (s = sigma)
cudaError_t launch_trunc_rank(int P, const double* sigma, double tol3, int64_t* rank, cudaStream_t st);
// copy rows 0..Rt_l-1 of each P_l x R block of w0 = [W1 | W2 | W3] into the packed core point w
cudaError_t launch_truncate_rows(const int64_t* P, const int64_t* Rt, int64_t R, const double* w0, double* w,
                                 cudaStream_t st);
// unit columns and lambda_r = prod_l ||W_l[:, r]|| (one block per r); zero columns are left as they are
cudaError_t launch_normalize_cpd(const int64_t* n, int64_t R, double* w, double* lambda, cudaStream_t st);
// MLSVD-energy initialisation: the R entries of largest |s| of S (P1 x P2 x P3) -> packed w (core dims)
cudaError_t launch_energy_init(int64_t P1, int64_t P2, int64_t P3, const double* S, int64_t R, double* w,
                               cudaStream_t st);

// ---- CP-ALS (NEXT #4, k_als.cu)
cudaError_t launch_khatri_rao(int64_t nx, const double* X, int64_t x0, int64_t xn, int64_t ny, const double* Y,
                              int64_t R, double* KR, cudaStream_t st);
cudaError_t launch_pinv_from_eig(int R, const double* Q, const double* theta, double* out, cudaStream_t st);

}  // namespace tfk
