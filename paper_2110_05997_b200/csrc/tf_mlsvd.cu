// C-ABI of the compression stage (NEXT #3, include/tf.h): argument checks, GEMM planning (tile shape,
// split-K, TMA descriptors) and the orchestration of the truncated MLSVD. Every arithmetic step runs in
// the kernels of k_gemm.cu and k_eig.cu; the host only decides sizes, convergence and control flow.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "tf_ctx.h"

using namespace tfk;
using namespace tfh;

namespace tfh {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool op_tma_ok(const GemmOperand& x) {
  return aligned16(x.ptr) && (x.ld % 2 == 0) && (x.bstride % 2 == 0) && x.ld < (1LL << 36);
}

// TMA descriptor of one operand in its [p, k] view (see k_gemm.cu): box = one BP x 32 stage tile
// plus the 4-double pad that gives the conflict-free shared-memory pitch.
bool make_map(CUtensorMap* map, const GemmOperand& x, int64_t np, int64_t nk, int64_t nbat, int BP) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[3], gstride[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  if (x.kc) {
    gdim[0] = (cuuint64_t)nk;
    gdim[1] = (cuuint64_t)np;
    box[0] = kGemmBK + 4;
    box[1] = (cuuint32_t)BP;
  } else {
    gdim[0] = (cuuint64_t)np;
    gdim[1] = (cuuint64_t)nk;
    box[0] = (cuuint32_t)(BP + 4);
    box[1] = kGemmBK;
  }
  gdim[2] = (cuuint64_t)nbat;
  box[2] = 1;
  gstride[0] = (cuuint64_t)x.ld * 8;
  gstride[1] = x.bstride ? (cuuint64_t)x.bstride * 8 : (cuuint64_t)x.ld * 8 * (cuuint64_t)gdim[1];
  if (gdim[0] >= (1ULL << 31) || gdim[1] >= (1ULL << 31) || gdim[2] >= (1ULL << 31)) return false;
  if (gstride[1] >= (1ULL << 40) || gstride[1] % 16) return false;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x.ptr), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

GemmOperand opnd(const double* p, int64_t ld, bool kc, int64_t bstride) {
  GemmOperand o;
  o.ptr = p;
  o.ld = ld;
  o.kc = kc;
  o.bstride = bstride;
  return o;
}

// Plan and launch C = alpha * sum A B^T (+ beta C) (k_gemm.cu). Split-K minimises
// waves * (k-steps per split + overhead) over the SMs, bounded by the partial-buffer size.
tf_status gemm_run(tf_ctx* c, GemmArgs g) {
  if (g.M <= 0 || g.N <= 0) return TF_OK;
  // tile: 128 or 64 rows; 128, 112, 96 or 64 columns (the narrower widths cut the padding of N = R
  // around 100 on the 128-row tile)
  g.BM = g.M > 64 ? 128 : 64;
  g.BN = g.N > 112 ? 128 : g.N > 96 ? 112 : g.N > 64 ? 96 : g.N > 32 ? 64 : 32;
  if (g.BM == 64 && (g.BN == 112 || g.BN == 96)) g.BN = 128;
  if (g.BM == 64 && g.BN == 32) g.BN = 64;
  if (g.sym) {
    // symmetric Grams: the square tile with the least padded area over the upper triangle
    static const int force = [] {
      const char* e = getenv("TF_GEMM_SYM_TILE");
      return e ? atoi(e) : 0;
    }();
    if (force == 64 || force == 128) {
      g.BM = force;
    } else {
      // 64-wide tiles: half the padding and a finer upper triangle; measured on c5's 1200^2 Grams at 30.3 TF/s
      // (82% of the DMMA peak) against 27.3 TF/s with 128-wide tiles
      g.BM = 64;
    }
    g.BN = g.BM;
  }
  g.ntm = (g.M + g.BM - 1) / g.BM;
  g.ntn = (g.N + g.BN - 1) / g.BN;
  const int64_t tiles = g.sym ? g.ntm * (g.ntm + 1) / 2 : g.ntm * g.ntn;
  g.out_batches = g.sum_batch ? 1 : g.batch;
  const int64_t items = tiles * g.out_batches;
  const int64_t nks = (g.Kd + kGemmBK - 1) / kGemmBK;
  const int64_t total = (g.sum_batch ? g.batch : 1) * nks;
  if (total == 0) return set_err(c, TF_ERR_ARG, "gemm with an empty inner dimension");
  const double overhead = 4.0;
  const int64_t tile_bytes = (int64_t)g.BM * g.BN * 8;
  const int64_t part_cap = (int64_t)1 << 30;   // partial-sum buffer bound
  int best = 1;
  double best_cost = 1e300;
  for (int64_t ks = 1; ks <= std::min<int64_t>(total, 2048); ++ks) {
    if (ks > 1 && items * ks * tile_bytes > part_cap) break;
    const int64_t per = (total + ks - 1) / ks;
    if ((total + per - 1) / per != ks) continue;
    const int64_t waves = (items * ks + c->nsm - 1) / c->nsm;
    const double cost = (double)waves * ((double)per + overhead);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = (int)ks;
    }
  }
  g.ksplit = best;
  g.steps_per_split = (total + best - 1) / best;
  g.part = nullptr;
  if (g.ksplit > 1) {
    tf_status s = ensure(c, c->gemmPart, (size_t)items * g.ksplit * tile_bytes);
    if (s) return s;
    g.part = (double*)c->gemmPart.p;
  }
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  bool tma = op_tma_ok(g.a) && op_tma_ok(g.b);
  if (tma) {
    tma = make_map(&ma, g.a, g.M, g.Kd, g.a.bstride ? g.batch : 1, g.BM) &&
          make_map(&mb, g.b, g.N, g.Kd, g.b.bstride ? g.batch : 1, g.BN);
  }
  TF_CUDA(c, launch_gemm(&ma, &mb, g, items, tma, c->stream));
  c->total_launches += g.ksplit > 1 ? 2 : 1;
  return TF_OK;
}

GemmArgs gemm_args(GemmOperand a, GemmOperand b, int64_t M, int64_t N, int64_t Kd, double* C, int64_t ldc) {
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.a = a;
  g.b = b;
  g.M = M;
  g.N = N;
  g.Kd = Kd;
  g.batch = 1;
  g.sum_batch = true;
  g.C = C;
  g.ldc = ldc;
  g.alpha = 1.0;
  g.beta = 0.0;
  return g;
}

}  // namespace tfh

namespace {

tf_status check_whole(tf_ctx* c, tf_dims& d) {
  if (!c) return TF_ERR_ARG;
  if (d.ldT == 0) d.ldT = d.I;
  if (d.K_total == 0) d.K_total = d.K;
  if (d.I < 1 || d.J < 1 || d.K < 1) return set_err(c, TF_ERR_ARG, "dimensions must be >= 1");
  if (d.ldT < d.I) return set_err(c, TF_ERR_ARG, "ldT < I");
  if (d.K != d.K_total || d.k_begin != 0)
    return set_err(c, TF_ERR_UNSUPPORTED, "the compression stage needs the whole tensor (K == K_total)");
  if (d.I > (1LL << 31) - 1 || d.J > (1LL << 31) - 1 || d.K > (1LL << 31) - 1)
    return set_err(c, TF_ERR_UNSUPPORTED, "mode size >= 2^31");
  return TF_OK;
}

// ---- unfolding Grams
tf_status grams_mode(tf_ctx* c, const tf_dims& d, const double* T, int mode, double* G) {
  const int64_t I = d.I, J = d.J, K = d.K, ld = d.ldT;
  GemmArgs g;
  if (mode == 1) {          // T_(1) = I x JK, column c = (j, k) at T + ldT*c
    GemmOperand a = opnd(T, ld, false);
    g = gemm_args(a, a, I, I, J * K, G, I);
  } else if (mode == 2) {   // sum_k T_k^T T_k: A_k[j, i] = T[i + ldT j + ldT J k]
    GemmOperand a = opnd(T, ld, true, ld * J);
    g = gemm_args(a, a, J, J, I, G, J);
    g.batch = K;
  } else if (ld == I) {     // T_(3) rows are whole frontal slices: A[k, e] = T[e + IJ k]
    GemmOperand a = opnd(T, I * J, true);
    g = gemm_args(a, a, K, K, I * J, G, K);
  } else {                  // padded slices: sum over j of A_j[k, i] = T[i + ldT j + ldT J k]
    GemmOperand a = opnd(T, ld * J, true, ld);
    g = gemm_args(a, a, K, K, I, G, K);
    g.batch = J;
  }
  g.sym = true;
  return gemm_run(c, g);
}

int64_t even(int64_t x) { return x + (x & 1); }

// ---- subspace iteration for the top-P eigenpairs of G (n x n)
tf_status eig_top_impl(tf_ctx* c, int64_t n, const double* G, int P, const double* Omega, int maxiter, double tol,
                       double* U, double* lam, int* iters_out) {
  const int64_t ldw = even(n);
  tf_status s;
  if ((s = ensure(c, c->eigQ, (size_t)ldw * P * 8))) return s;
  if ((s = ensure(c, c->eigZ, (size_t)ldw * P * 8))) return s;
  if ((s = ensure(c, c->eigU, (size_t)ldw * P * 8))) return s;
  if ((s = ensure(c, c->eigRes, (size_t)ldw * P * 8))) return s;   // ZV
  if ((s = ensure(c, c->eigH, (size_t)P * P * 8))) return s;
  if ((s = ensure(c, c->eigV, (size_t)2 * P * P * 8))) return s;
  if ((s = ensure(c, c->eigScal, (size_t)2 * P * 8 + 64))) return s;
  if ((s = ensure(c, c->eigB, (size_t)2 * P * P * 8))) return s;
  double* Q = (double*)c->eigQ.p;
  double* Z = (double*)c->eigZ.p;
  double* Uw = (double*)c->eigU.p;
  double* ZV = (double*)c->eigRes.p;
  double* H = (double*)c->eigH.p;
  double* V = (double*)c->eigV.p;
  double* Vt = V + (size_t)P * P;
  double* theta = (double*)c->eigScal.p;
  double* res = theta + P;
  int* fail = reinterpret_cast<int*>(res + P);
  double* Bm = (double*)c->eigB.p;
  double* Linv = Bm + (size_t)P * P;
  // Q = orth(X): column-scaled CholeskyQR2 (X's columns are nearly orthogonal after the Ritz rotation, so
  // its Gram is ~I; a few GEMMs and one small Cholesky per pass), Householder QR when Cholesky reports a
  // numerically dependent block (exact low rank). X is preserved by CholeskyQR2; W, tmp are scratch.
  auto orth = [&](double* X, double* W, double* tmp) -> tf_status {
    int hfail = 0;
    tf_status st;
    TF_CUDA(c, cudaMemsetAsync(fail, 0, sizeof(int), c->stream));
    TF_CUDA(c, launch_col_normalize(n, P, X, ldw, W, ldw, fail, c->stream));
    double* src = W;
    for (int pass = 0; pass < 2; ++pass) {
      if ((st = gemm_run(c, gemm_args(opnd(src, ldw, true), opnd(src, ldw, true), P, P, n, Bm, P)))) return st;
      TF_CUDA(c, launch_chol_inv(P, Bm, Linv, fail, c->stream));
      if ((st = gemm_run(c, gemm_args(opnd(src, ldw, false), opnd(Linv, P, false), n, P, P, pass ? Q : tmp, ldw))))
        return st;
      src = tmp;
    }
    c->total_launches += 4;
    TF_CUDA(c, cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
    if (hfail) {
      TF_CUDA(c, launch_house_qr(n, P, X, ldw, Q, ldw, c->stream));
      c->total_launches += 1;
    }
    return TF_OK;
  };
  TF_CUDA(c, cudaMemcpy2DAsync(Z, ldw * 8, Omega, n * 8, n * 8, P, cudaMemcpyDeviceToDevice, c->stream));
  if ((s = orth(Z, ZV, Uw))) return s;
  const double u = std::ldexp(1.0, -53);
  const double tol_eff = std::max(tol, 16.0 * std::sqrt((double)n) * u);
  double host[2 * TF_MAX_R + 2];
  double prev = INFINITY;
  int it = 0;
  for (it = 1; it <= maxiter; ++it) {
    // Z = G Q ; H = Q^T Z ; (theta, V) = eig(H) ; U = Q V ; ZV = Z V
    if ((s = gemm_run(c, gemm_args(opnd(G, n, false), opnd(Q, ldw, true), n, P, n, Z, ldw)))) return s;
    if ((s = gemm_run(c, gemm_args(opnd(Q, ldw, true), opnd(Z, ldw, true), P, P, n, H, P)))) return s;
    // the first two Rayleigh-Ritz steps act on a still-rotating subspace: a few Jacobi sweeps give a rotation
    // good enough for the orthonormalisation; the converged iterations run Jacobi to the end
    const bool early = it <= 2 && it < maxiter;
    TF_CUDA(c, launch_jacobi_eig(P, H, P, Vt, V, theta, c->stream, early ? 4 : 60));
    if ((s = gemm_run(c, gemm_args(opnd(Q, ldw, false), opnd(V, P, true), n, P, P, Uw, ldw)))) return s;
    if ((s = gemm_run(c, gemm_args(opnd(Z, ldw, false), opnd(V, P, true), n, P, P, ZV, ldw)))) return s;
    TF_CUDA(c, launch_eig_residual(n, P, ZV, Uw, ldw, theta, res, c->stream));
    c->total_launches += 2;
    TF_CUDA(c, cudaMemcpyAsync(host, theta, (size_t)2 * P * 8, cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
    double maxres = 0.0;
    for (int j = 0; j < P; ++j) maxres = std::max(maxres, host[P + j]);
    const double scale = std::fabs(host[0]);
    if (!std::isfinite(maxres) || !std::isfinite(scale))
      return set_err(c, TF_ERR_NONFINITE, "non-finite Ritz values in the subspace iteration");
    const bool conv = !early && (maxres <= tol_eff * scale || scale == 0.0);
    const bool stall = it >= 4 && maxres > 0.5 * prev && maxres <= 1e3 * tol_eff * scale;
    if (conv || stall || it == maxiter) break;
    prev = maxres;
    // orthonormalise the Ritz-rotated block ZV ~ U Theta for the next iteration
    if ((s = orth(ZV, Z, Uw))) return s;
  }
  if (it > maxiter) it = maxiter;
  TF_CUDA(c, launch_sign_fix(n, P, Uw, ldw, c->stream));
  TF_CUDA(c, cudaMemcpy2DAsync(U, n * 8, Uw, ldw * 8, n * 8, P, cudaMemcpyDeviceToDevice, c->stream));
  TF_CUDA(c, cudaMemcpyAsync(lam, theta, (size_t)P * 8, cudaMemcpyDeviceToDevice, c->stream));
  c->total_launches += 2;
  if (iters_out) *iters_out = it;
  return TF_OK;
}

// ---- S = (U1^T, U2^T, U3^T) . T over chunks of frontal slices
tf_status core_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* U1, int64_t P1, const double* U2,
                    int64_t P2, const double* U3, int64_t P3, double* S) {
  const int64_t I = d.I, J = d.J, K = d.K, ld = d.ldT;
  const int64_t P1e = even(P1);
  const int64_t budget = (int64_t)1 << 30;
  int64_t kc = std::max<int64_t>(2, budget / std::max<int64_t>(1, P1e * J * 8));
  kc -= kc & 1;
  kc = std::min<int64_t>(kc, K);
  tf_status s;
  if ((s = ensure(c, c->mlX, (size_t)P1e * J * kc * 8))) return s;
  if ((s = ensure(c, c->mlY, (size_t)P1 * P2 * kc * 8))) return s;
  double* X = (double*)c->mlX.p;
  double* Y = (double*)c->mlY.p;
  for (int64_t k0 = 0; k0 < K; k0 += kc) {
    const int64_t kn = std::min<int64_t>(kc, K - k0);
    // X[a, (j, k)] = sum_i U1[i, a] T[i, j, k0 + k]     (mode-1 product, inner dimension I)
    GemmArgs g1 = gemm_args(opnd(U1, I, true), opnd(T + k0 * ld * J, ld, true), P1, J * kn, I, X, P1e);
    if ((s = gemm_run(c, g1))) return s;
    // Y_k[a, b] = sum_j X[a, j, k] U2[j, b]              (mode-2 product per slice)
    GemmArgs g2 = gemm_args(opnd(X, P1e, false, P1e * J), opnd(U2, J, true), P1, P2, J, Y, P1);
    g2.batch = kn;
    g2.sum_batch = false;
    g2.cstride = P1 * P2;
    if ((s = gemm_run(c, g2))) return s;
    // S[(a, b), c] (+)= sum_k Y[(a, b), k] U3[k0 + k, c] (mode-3 product)
    GemmArgs g3 = gemm_args(opnd(Y, P1 * P2, false), opnd(U3 + k0, K, true), P1 * P2, P3, kn, S, P1 * P2);
    g3.beta = k0 == 0 ? 0.0 : 1.0;
    if ((s = gemm_run(c, g3))) return s;
  }
  return TF_OK;
}

}  // namespace

extern "C" {

tf_status tf_unfolding_grams(tf_ctx* c, tf_dims d, const double* T, double* G1, double* G2, double* G3) {
  tf_status s = check_whole(c, d);
  if (s) return s;
  if (!T) return set_err(c, TF_ERR_ARG, "null T");
  if (reinterpret_cast<uintptr_t>(T) & 7) return set_err(c, TF_ERR_ALIGN, "T not 8-byte aligned");
  cudaSetDevice(c->device);
  if (G1 && (s = grams_mode(c, d, T, 1, G1))) return s;
  if (G2 && (s = grams_mode(c, d, T, 2, G2))) return s;
  if (G3 && (s = grams_mode(c, d, T, 3, G3))) return s;
  return TF_OK;
}

tf_status tf_sym_eig_top(tf_ctx* c, int64_t n, const double* G, int64_t P, const double* Omega, int maxiter,
                         double tol, double* U, double* lam, int* iters) {
  if (!c) return TF_ERR_ARG;
  if (n < 1 || P < 1 || P > n || !G || !Omega || !U || !lam || maxiter < 1)
    return set_err(c, TF_ERR_ARG, "tf_sym_eig_top: bad argument");
  if (P > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "P > TF_MAX_R");
  cudaSetDevice(c->device);
  return eig_top_impl(c, n, G, (int)P, Omega, maxiter, tol, U, lam, iters);
}

tf_status tf_multilinear_core(tf_ctx* c, tf_dims d, const double* T, const double* U1, int64_t P1,
                              const double* U2, int64_t P2, const double* U3, int64_t P3, double* S) {
  tf_status s = check_whole(c, d);
  if (s) return s;
  if (!T || !U1 || !U2 || !U3 || !S) return set_err(c, TF_ERR_ARG, "null pointer");
  if (P1 < 1 || P2 < 1 || P3 < 1 || P1 > d.I || P2 > d.J || P3 > d.K)
    return set_err(c, TF_ERR_ARG, "core ranks must satisfy 1 <= P_l <= I_l");
  if (P1 > TF_MAX_R || P2 > TF_MAX_R || P3 > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "P_l > TF_MAX_R");
  cudaSetDevice(c->device);
  return core_impl(c, d, T, U1, P1, U2, P2, U3, P3, S);
}

tf_status tf_compress(tf_ctx* c, tf_dims d, const double* T, const double* Omega, double mlsvd_tol, int eig_maxiter,
                      double eig_tol, double* U, double* sigma, double* S, int64_t* ranks, int* eig_iters) {
  tf_status s = check_whole(c, d);
  if (s) return s;
  if (!T || !Omega || !U || !sigma || !S || !ranks) return set_err(c, TF_ERR_ARG, "null pointer");
  if (d.R < 1) return set_err(c, TF_ERR_ARG, "R < 1");
  if (!(mlsvd_tol > 0.0)) return set_err(c, TF_ERR_ARG, "mlsvd_tol must be > 0");
  if (eig_maxiter < 1) return set_err(c, TF_ERR_ARG, "eig_maxiter < 1");
  cudaSetDevice(c->device);
  const int64_t dims[3] = {d.I, d.J, d.K};
  int64_t P[3], off[3], soff[3];
  int64_t o = 0, so = 0;
  for (int l = 0; l < 3; ++l) {
    P[l] = std::min<int64_t>(dims[l], d.R);
    if (P[l] > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "min(I_l, R) > TF_MAX_R");
    off[l] = o;
    soff[l] = so;
    o += dims[l] * P[l];
    so += P[l];
  }
  const int64_t nmax = std::max(dims[0], std::max(dims[1], dims[2]));
  if ((s = ensure(c, c->mlG, (size_t)nmax * nmax * 8))) return s;
  if ((s = ensure(c, c->mlLam, (size_t)TF_MAX_R * 8))) return s;
  if ((s = ensure(c, c->mlRanks, 3 * sizeof(int64_t)))) return s;
  double* G = (double*)c->mlG.p;
  double* lam = (double*)c->mlLam.p;
  int64_t* rk = (int64_t*)c->mlRanks.p;
  for (int l = 0; l < 3; ++l) {
    if ((s = grams_mode(c, d, T, l + 1, G))) return s;
    int it = 0;
    if ((s = eig_top_impl(c, dims[l], G, (int)P[l], Omega + off[l], eig_maxiter, eig_tol, U + off[l], lam, &it)))
      return s;
    if (eig_iters) eig_iters[l] = it;
    TF_CUDA(c, launch_sqrt_abs(P[l], lam, sigma + soff[l], c->stream));
    TF_CUDA(c, launch_trunc_rank((int)P[l], sigma + soff[l], mlsvd_tol / 3.0, rk + l, c->stream));
    c->total_launches += 2;
  }
  TF_CUDA(c, cudaMemcpyAsync(ranks, rk, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  return core_impl(c, d, T, U + off[0], ranks[0], U + off[1], ranks[1], U + off[2], ranks[2], S);
}

}  // extern "C"

namespace {

// Exchange of a device buffer through the caller's all-reduce hook (K-sharded calls): src -> xbuf, SUM over
// the ranks, xbuf -> src. No-op without a hook.
tf_status exchange(tf_ctx* c, tf_allreduce_fn xfn, void* xuser, double* xbuf, double* src, int64_t cnt) {
  if (!xfn) return TF_OK;
  TF_CUDA(c, cudaMemcpyAsync(xbuf, src, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  if (xfn(xbuf, cnt, xuser) != 0) return set_err(c, TF_ERR_CUDA, "the all-reduce hook reported a failure");
  TF_CUDA(c, cudaMemcpyAsync(src, xbuf, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
  return TF_OK;
}

// Alg. ST-MLSVD on the local slices d.k_begin .. d.k_begin + d.K - 1 of a K_total-slice tensor. Modes 1 and 2
// only need sums over slices (their Grams are all-reduced); mode 3 needs every slice of X2 = T x1 U~1^T x2 U~2^T,
// which each rank writes into its columns of a zeroed R~1 R~2 x K_total buffer that the all-reduce completes.
// Everything after that (G3, U3, the core) is computed identically on every rank.
tf_status compress_st_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* Omega, double mlsvd_tol,
                           int eig_maxiter, double eig_tol, double* U, double* sigma, double* S, int64_t* ranks,
                           int* eig_iters, tf_allreduce_fn xfn, void* xuser, double* xbuf) {
  tf_status s;
  const int64_t I = d.I, J = d.J, Kl = d.K, Kt = d.K_total, kb = d.k_begin, ld = d.ldT;
  const int64_t dims[3] = {I, J, Kt};
  int64_t P[3], off[3], soff[3];
  int64_t o = 0, so = 0;
  for (int l = 0; l < 3; ++l) {
    P[l] = std::min<int64_t>(dims[l], d.R);
    if (P[l] > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "min(I_l, R) > TF_MAX_R");
    off[l] = o;
    soff[l] = so;
    o += dims[l] * P[l];
    so += P[l];
  }
  const int64_t nmax = std::max(I, std::max(J, Kt));
  if ((s = ensure(c, c->mlG, (size_t)nmax * nmax * 8))) return s;
  if ((s = ensure(c, c->mlLam, (size_t)TF_MAX_R * 8))) return s;
  if ((s = ensure(c, c->mlRanks, 3 * sizeof(int64_t)))) return s;
  double* G = (double*)c->mlG.p;
  double* lam = (double*)c->mlLam.p;
  int64_t* rk = (int64_t*)c->mlRanks.p;
  // one mode: eigenpairs of the Gram in G, sigma, the Alg. Compression rank (synchronizes for it)
  auto mode_step = [&](int l) -> tf_status {
    tf_status st;
    int it = 0;
    if ((st = eig_top_impl(c, dims[l], G, (int)P[l], Omega + off[l], eig_maxiter, eig_tol, U + off[l], lam, &it)))
      return st;
    if (eig_iters) eig_iters[l] = it;
    TF_CUDA(c, launch_sqrt_abs(P[l], lam, sigma + soff[l], c->stream));
    TF_CUDA(c, launch_trunc_rank((int)P[l], sigma + soff[l], mlsvd_tol / 3.0, rk + l, c->stream));
    TF_CUDA(c, cudaMemcpyAsync(ranks + l, rk + l, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
    c->total_launches += 2;
    return TF_OK;
  };
  // step 1: T_(1) T_(1)^T (summed over the ranks' slices), U1, then X1 = U~1^T T_(1)  (r1 x J x K local)
  if ((s = grams_mode(c, d, T, 1, G))) return s;
  if ((s = exchange(c, xfn, xuser, xbuf, G, I * I))) return s;
  if ((s = mode_step(0))) return s;
  const int64_t r1 = ranks[0], r1e = even(r1);
  if ((s = ensure(c, c->mlX, (size_t)r1e * J * Kl * 8))) return s;
  double* X1 = (double*)c->mlX.p;
  if ((s = gemm_run(c, gemm_args(opnd(U + off[0], I, true), opnd(T, ld, true), r1, J * Kl, I, X1, r1e)))) return s;
  // step 2: Gram of the mode-2 unfolding of X1 (sum over slices of X1_k^T X1_k), U2, X2_k = X1_k U~2
  {
    GemmOperand a = opnd(X1, r1e, true, r1e * J);
    GemmArgs g = gemm_args(a, a, J, J, r1, G, J);
    g.batch = Kl;
    g.sym = true;
    if ((s = gemm_run(c, g))) return s;
  }
  if ((s = exchange(c, xfn, xuser, xbuf, G, J * J))) return s;
  if ((s = mode_step(1))) return s;
  const int64_t r2 = ranks[1];
  if ((s = ensure(c, c->mlY, (size_t)r1 * r2 * Kt * 8))) return s;
  double* X2 = (double*)c->mlY.p;   // r1 r2 x K_total; this rank's columns kb .. kb + Kl - 1
  if (xfn) TF_CUDA(c, cudaMemsetAsync(X2, 0, (size_t)r1 * r2 * Kt * 8, c->stream));
  {
    GemmArgs g = gemm_args(opnd(X1, r1e, false, r1e * J), opnd(U + off[1], J, true), r1, r2, J, X2 + kb * r1 * r2,
                           r1);
    g.batch = Kl;
    g.sum_batch = false;
    g.cstride = r1 * r2;
    if ((s = gemm_run(c, g))) return s;
  }
  if ((s = exchange(c, xfn, xuser, xbuf, X2, r1 * r2 * Kt))) return s;
  // step 3: Gram of X2 as (r1 r2) x K_total, U3, S = X2 x_3 U~3^T
  {
    GemmOperand a = opnd(X2, r1 * r2, true);
    GemmArgs g = gemm_args(a, a, Kt, Kt, r1 * r2, G, Kt);
    g.sym = true;
    if ((s = gemm_run(c, g))) return s;
  }
  if ((s = mode_step(2))) return s;
  const int64_t r3 = ranks[2];
  return gemm_run(c, gemm_args(opnd(X2, r1 * r2, false), opnd(U + off[2], Kt, true), r1 * r2, r3, Kt, S, r1 * r2));
}

tf_status check_compress_args(tf_ctx* c, const tf_dims& d, const double* T, const double* Omega, double mlsvd_tol,
                              int eig_maxiter, double* U, double* sigma, double* S, int64_t* ranks) {
  if (!T || !Omega || !U || !sigma || !S || !ranks) return set_err(c, TF_ERR_ARG, "null pointer");
  if (d.R < 1) return set_err(c, TF_ERR_ARG, "R < 1");
  if (!(mlsvd_tol > 0.0)) return set_err(c, TF_ERR_ARG, "mlsvd_tol must be > 0");
  if (eig_maxiter < 1) return set_err(c, TF_ERR_ARG, "eig_maxiter < 1");
  return TF_OK;
}

tf_status check_shard(tf_ctx* c, tf_dims& d) {
  if (!c) return TF_ERR_ARG;
  if (d.ldT == 0) d.ldT = d.I;
  if (d.K_total == 0) d.K_total = d.K + d.k_begin;
  if (d.I < 1 || d.J < 1 || d.K < 1) return set_err(c, TF_ERR_ARG, "dimensions must be >= 1");
  if (d.ldT < d.I) return set_err(c, TF_ERR_ARG, "ldT < I");
  if (d.k_begin < 0 || d.k_begin + d.K > d.K_total) return set_err(c, TF_ERR_ARG, "k_begin + K > K_total");
  if (d.I > (1LL << 31) - 1 || d.J > (1LL << 31) - 1 || d.K_total > (1LL << 31) - 1)
    return set_err(c, TF_ERR_UNSUPPORTED, "mode size >= 2^31");
  return TF_OK;
}

}  // namespace

extern "C" {

tf_status tf_compress_st(tf_ctx* c, tf_dims d, const double* T, const double* Omega, double mlsvd_tol,
                         int eig_maxiter, double eig_tol, double* U, double* sigma, double* S, int64_t* ranks,
                         int* eig_iters) {
  tf_status s = check_whole(c, d);
  if (s) return s;
  if ((s = check_compress_args(c, d, T, Omega, mlsvd_tol, eig_maxiter, U, sigma, S, ranks))) return s;
  cudaSetDevice(c->device);
  return compress_st_impl(c, d, T, Omega, mlsvd_tol, eig_maxiter, eig_tol, U, sigma, S, ranks, eig_iters, nullptr,
                          nullptr, nullptr);
}

tf_status tf_compress_st_sharded(tf_ctx* c, tf_dims d, const double* T_local, const double* Omega, double mlsvd_tol,
                                 int eig_maxiter, double eig_tol, double* U, double* sigma, double* S, int64_t* ranks,
                                 int* eig_iters, tf_allreduce_fn allreduce, void* user, double* xbuf) {
  tf_status s = check_shard(c, d);
  if (s) return s;
  if ((s = check_compress_args(c, d, T_local, Omega, mlsvd_tol, eig_maxiter, U, sigma, S, ranks))) return s;
  if (!allreduce || !xbuf) return set_err(c, TF_ERR_ARG, "null all-reduce hook or exchange buffer");
  cudaSetDevice(c->device);
  return compress_st_impl(c, d, T_local, Omega, mlsvd_tol, eig_maxiter, eig_tol, U, sigma, S, ranks, eig_iters,
                          allreduce, user, xbuf);
}

tf_status tf_energy_init(tf_ctx* c, int64_t R1, int64_t R2, int64_t R3, const double* S, int64_t R, double* w) {
  if (!c) return TF_ERR_ARG;
  if (R1 < 1 || R2 < 1 || R3 < 1 || R < 1 || !S || !w) return set_err(c, TF_ERR_ARG, "tf_energy_init: bad argument");
  if (R > R1 * R2 * R3) return set_err(c, TF_ERR_ARG, "R exceeds the number of core entries");
  cudaSetDevice(c->device);
  TF_CUDA(c, launch_energy_init(R1, R2, R3, S, R, w, c->stream));
  c->total_launches += 1;
  return TF_OK;
}

tf_status tf_uncompress(tf_ctx* c, int64_t n, int64_t Rl, const double* U, const double* W, int64_t R, double* out) {
  if (!c) return TF_ERR_ARG;
  if (n < 1 || Rl < 1 || R < 1 || !U || !W || !out) return set_err(c, TF_ERR_ARG, "tf_uncompress: bad argument");
  cudaSetDevice(c->device);
  return gemm_run(c, gemm_args(opnd(U, n, false), opnd(W, Rl, true), n, R, Rl, out, n));
}

}  // extern "C"

namespace {

// The whole flow on the local slices of a K_total-slice tensor; with an exchange hook the compression is the
// K-sharded ST-MLSVD and the final fit sums the ranks' partial F and ||T||^2; the dGN on the core and the
// uncompression run replicated (every rank holds the full core and U).
tf_status cpd_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* Omega, const double* w0_core,
                   const tf_cpd_params* prm, double* W, double* lambda, tf_cpd_result* res, double* hist,
                   tf_allreduce_fn xfn, void* xuser, double* xbuf) {
  tf_status s;
  const int64_t R = d.R;
  const int64_t dims[3] = {d.I, d.J, d.K_total};
  int64_t P[3];
  int64_t nU = 0;
  for (int l = 0; l < 3; ++l) {
    P[l] = std::min<int64_t>(dims[l], R);
    nU += dims[l] * P[l];
  }
  const int64_t n = R * (d.I + d.J + d.K_total);
  if ((s = ensure(c, c->cpdU, (size_t)nU * 8))) return s;
  if ((s = ensure(c, c->cpdSig, (size_t)(P[0] + P[1] + P[2]) * 8))) return s;
  if ((s = ensure(c, c->cpdS, (size_t)P[0] * P[1] * P[2] * 8))) return s;
  if ((s = ensure(c, c->cpdW, (size_t)R * (P[0] + P[1] + P[2]) * 8))) return s;
  if ((s = ensure(c, c->cpdGrad, (size_t)n * 8))) return s;
  if ((s = ensure(c, c->cpdScal, (size_t)red_blocks() * 2 * 8 + 64))) return s;
  double* U = (double*)c->cpdU.p;
  double* S = (double*)c->cpdS.p;
  double* wc = (double*)c->cpdW.p;
  // 1. compression
  int64_t rk[3];
  if (xfn || prm->sequential)
    s = compress_st_impl(c, d, T, Omega, prm->mlsvd_tol, prm->eig_maxiter, 0.0, U, (double*)c->cpdSig.p, S, rk,
                         res->eig_iters, xfn, xuser, xbuf);
  else
    s = tf_compress(c, d, T, Omega, prm->mlsvd_tol, prm->eig_maxiter, 0.0, U, (double*)c->cpdSig.p, S, rk,
                    res->eig_iters);
  if (s) return s;
  for (int l = 0; l < 3; ++l) res->ranks[l] = rk[l];
  // 2. initialisation on the core
  if (prm->init) {
    if (R > rk[0] * rk[1] * rk[2]) return set_err(c, TF_ERR_ARG, "R exceeds the entries of the truncated core");
    TF_CUDA(c, launch_energy_init(rk[0], rk[1], rk[2], S, R, wc, c->stream));
  } else {
    TF_CUDA(c, launch_truncate_rows(P, rk, R, w0_core, wc, c->stream));
  }
  c->total_launches += 1;
  // 3. dGN on the core
  tf_dims dc;
  memset(&dc, 0, sizeof(dc));
  dc.I = rk[0];
  dc.J = rk[1];
  dc.K = rk[2];
  dc.R = R;
  if ((s = tf_cpd_dgn(c, dc, S, wc, &prm->dgn, &res->dgn, hist))) return s;
  // 4. uncompression W~_l = U~_l W_l (U~_l = the first R~_l columns of U_l)
  int64_t uoff = 0, woff = 0, ooff = 0;
  for (int l = 0; l < 3; ++l) {
    if ((s = gemm_run(c, gemm_args(opnd(U + uoff, dims[l], false), opnd(wc + woff, rk[l], true), dims[l], R, rk[l],
                                   W + ooff, dims[l]))))
      return s;
    uoff += dims[l] * P[l];
    woff += rk[l] * R;
    ooff += dims[l] * R;
  }
  // 5. relative error on the original tensor. W = (U1, U2, U3) W_core with orthonormal U, so
  //    <T, [[W]]> = <S, [[W_core]]> and ||[[W]]|| = ||[[W_core]]||, hence
  //    ||T - [[W]]||^2 = (||T||^2 - ||S||^2) + ||S - [[W_core]]||^2 = (||T||^2 - ||S||^2) + 2 F_core:
  //    one streaming pass for ||T||^2 instead of an evaluation. The difference cancels when the fit is
  //    close (2F < 1e-3 ||T||^2, the guard of reading R31): then one F-only evaluation of the local slices
  //    (summed over the ranks) gives F directly.
  double* scal = (double*)c->cpdScal.p;
  double* part = scal + 8;
  TF_CUDA(c, launch_tsums(d.I, d.J, d.K, d.ldT, T, part, scal, c->stream));
  TF_CUDA(c, launch_tsums(rk[0], rk[1] * rk[2], 1, rk[0], S, part, scal + 4, c->stream));   // ||S||^2 (replicated)
  c->total_launches += 2;
  if ((s = exchange(c, xfn, xuser, xbuf, scal, 2))) return s;
  double h[6];
  TF_CUDA(c, cudaMemcpyAsync(h, scal, 6 * 8, cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  const double normT2 = h[1], normS2 = h[5];
  double Ff = 0.5 * (normT2 - normS2) + res->dgn.f;
  if (!(std::isfinite(Ff) && 2.0 * Ff >= 1e-3 * normT2)) {
    if ((s = eval_f_only(c, d, T, W, scal + 2, (double*)c->cpdGrad.p))) return s;
    if ((s = exchange(c, xfn, xuser, xbuf, scal + 2, 1))) return s;
    TF_CUDA(c, cudaMemcpyAsync(&Ff, scal + 2, 8, cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  TF_CUDA(c, launch_normalize_cpd(dims, R, W, lambda, c->stream));
  c->total_launches += 1;
  res->rel_err = normT2 > 0.0 ? std::sqrt(2.0 * std::max(Ff, 0.0) / normT2) : 0.0;
  return TF_OK;
}

tf_status check_cpd_args(tf_ctx* c, const tf_dims& d, const double* T, const double* Omega, const double* w0_core,
                         const tf_cpd_params* prm, double* W, double* lambda, tf_cpd_result* res) {
  if (!T || !Omega || !prm || !W || !lambda || !res) return set_err(c, TF_ERR_ARG, "null pointer");
  if (!prm->init && !w0_core) return set_err(c, TF_ERR_ARG, "init = 0 needs w0_core");
  if (d.R < 1 || d.R > TF_MAX_R) return set_err(c, d.R < 1 ? TF_ERR_ARG : TF_ERR_UNSUPPORTED, "bad R");
  if (!(prm->mlsvd_tol > 0.0) || prm->eig_maxiter < 1) return set_err(c, TF_ERR_ARG, "bad compression parameters");
  return TF_OK;
}

}  // namespace

extern "C" {

tf_status tf_cpd(tf_ctx* c, tf_dims d, const double* T, const double* Omega, const double* w0_core,
                 const tf_cpd_params* prm, double* W, double* lambda, tf_cpd_result* res, double* hist) {
  tf_status s = check_whole(c, d);
  if (s) return s;
  if ((s = check_cpd_args(c, d, T, Omega, w0_core, prm, W, lambda, res))) return s;
  cudaSetDevice(c->device);
  return cpd_impl(c, d, T, Omega, w0_core, prm, W, lambda, res, hist, nullptr, nullptr, nullptr);
}

tf_status tf_cpd_sharded(tf_ctx* c, tf_dims d, const double* T_local, const double* Omega, const double* w0_core,
                         const tf_cpd_params* prm, double* W, double* lambda, tf_cpd_result* res, double* hist,
                         tf_allreduce_fn allreduce, void* user, double* xbuf) {
  tf_status s = check_shard(c, d);
  if (s) return s;
  if ((s = check_cpd_args(c, d, T_local, Omega, w0_core, prm, W, lambda, res))) return s;
  if (!allreduce || !xbuf) return set_err(c, TF_ERR_ARG, "null all-reduce hook or exchange buffer");
  cudaSetDevice(c->device);
  return cpd_impl(c, d, T_local, Omega, w0_core, prm, W, lambda, res, hist, allreduce, user, xbuf);
}

}  // extern "C"
