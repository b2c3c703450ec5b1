// C-ABI of the CP-ALS sweep (NEXT #4, include/tf.h): single-mode MTTKRPs as chunked DMMA GEMMs over
// materialised Khatri–Rao chunks, and Alg. ALS's factor updates W^(l) = M^(l) V_l^dagger.
// Host code only plans and orders the launches; the arithmetic runs in k_gemm.cu, k_als.cu, k_eig.cu,
// k_small.cu.
#include <cmath>
#include <cstring>
#include <string>

#include "tf_ctx.h"

using namespace tfk;
using namespace tfh;

namespace {

constexpr int64_t kKrBudget = (int64_t)512 << 20;   // bytes of one Khatri–Rao chunk

tf_status mttkrp_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* w, int mode, double* M) {
  const int64_t I = d.I, J = d.J, K = d.K, R = d.R, ld = d.ldT, Kt = d.K_total, kb = d.k_begin;
  const double* A = w;
  const double* B = w + I * R;
  const double* C = w + (I + J) * R;
  tf_status s;
  if (mode == 1 || mode == 2) {
    const int64_t rowsPerSlice = mode == 1 ? J : I;
    int64_t kc = std::max<int64_t>(2, kKrBudget / (rowsPerSlice * R * 8));
    kc -= kc & 1;
    kc = std::min<int64_t>(kc, K);
    if ((s = ensure(c, c->alsKR, (size_t)rowsPerSlice * kc * R * 8))) return s;
    double* KR = (double*)c->alsKR.p;
    for (int64_t k0 = 0; k0 < K; k0 += kc) {
      const int64_t kn = std::min<int64_t>(kc, K - k0);
      const double* Tk = T + k0 * ld * J;
      GemmArgs g;
      if (mode == 1) {   // M1 += T_(1)[:, (j, k) in chunk] (C ⊙ B)[chunk rows]
        TF_CUDA(c, launch_khatri_rao(Kt, C, kb + k0, kn, J, B, R, KR, c->stream));
        g = gemm_args(opnd(Tk, ld, false), opnd(KR, J * kn, true), I, R, J * kn, M, I);
      } else {           // M2 += sum_k T_k^T (A diag(c_k)) = T_(2)[:, (i, k) in chunk] (C ⊙ A)[chunk rows]
        TF_CUDA(c, launch_khatri_rao(Kt, C, kb + k0, kn, I, A, R, KR, c->stream));
        g = gemm_args(opnd(Tk, ld, true, ld * J), opnd(KR, I * kn, true, I), J, R, I, M, J);
        g.batch = kn;
      }
      g.beta = k0 == 0 ? 0.0 : 1.0;
      c->total_launches += 1;
      if ((s = gemm_run(c, g))) return s;
    }
    return TF_OK;
  }
  // mode 3: M3[k, r] = sum_(i, j) T[i, j, k] (B ⊙ A)[(i, j), r], chunked over j
  int64_t jc = std::max<int64_t>(2, kKrBudget / (I * R * 8));
  jc -= jc & 1;
  jc = std::min<int64_t>(jc, J);
  if ((s = ensure(c, c->alsKR, (size_t)I * jc * R * 8))) return s;
  double* KR = (double*)c->alsKR.p;
  for (int64_t j0 = 0; j0 < J; j0 += jc) {
    const int64_t jn = std::min<int64_t>(jc, J - j0);
    TF_CUDA(c, launch_khatri_rao(J, B, j0, jn, I, A, R, KR, c->stream));
    GemmArgs g;
    if (ld == I) {
      g = gemm_args(opnd(T + I * j0, I * J, true), opnd(KR, I * jn, true), K, R, I * jn, M, K);
    } else {
      g = gemm_args(opnd(T + ld * j0, ld * J, true, ld), opnd(KR, I * jn, true, I), K, R, I, M, K);
      g.batch = jn;
    }
    g.beta = j0 == 0 ? 0.0 : 1.0;
    c->total_launches += 1;
    if ((s = gemm_run(c, g))) return s;
  }
  return TF_OK;
}

tf_status check(tf_ctx* c, tf_dims& d) {
  if (!c) return TF_ERR_ARG;
  if (d.ldT == 0) d.ldT = d.I;
  if (d.K_total == 0) d.K_total = d.K + d.k_begin;
  if (d.I < 1 || d.J < 1 || d.K < 1 || d.R < 1) return set_err(c, TF_ERR_ARG, "dimensions must be >= 1");
  if (d.ldT < d.I) return set_err(c, TF_ERR_ARG, "ldT < I");
  if (d.k_begin < 0 || d.k_begin + d.K > d.K_total) return set_err(c, TF_ERR_ARG, "k_begin + K > K_total");
  if (d.R > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "R > TF_MAX_R");
  return TF_OK;
}

}  // namespace

extern "C" {

tf_status tf_mttkrp(tf_ctx* c, tf_dims d, const double* T, const double* w, int mode, double* M) {
  tf_status s = check(c, d);
  if (s) return s;
  if (!T || !w || !M) return set_err(c, TF_ERR_ARG, "null pointer");
  if (mode < 1 || mode > 3) return set_err(c, TF_ERR_ARG, "mode must be 1, 2 or 3");
  if (reinterpret_cast<uintptr_t>(T) & 7) return set_err(c, TF_ERR_ALIGN, "T not 8-byte aligned");
  cudaSetDevice(c->device);
  return mttkrp_impl(c, d, T, w, mode, M);
}

tf_status tf_als(tf_ctx* c, tf_dims d, const double* T, double* w, int sweeps, double* f_hist) {
  tf_status s = check(c, d);
  if (s) return s;
  if (!T || !w) return set_err(c, TF_ERR_ARG, "null pointer");
  if (sweeps < 0) return set_err(c, TF_ERR_ARG, "sweeps < 0");
  if (d.K != d.K_total || d.k_begin != 0)
    return set_err(c, TF_ERR_UNSUPPORTED, "tf_als needs the whole tensor on one device (K == K_total)");
  cudaSetDevice(c->device);
  const int64_t I = d.I, J = d.J, K = d.K, R = d.R, RR = R * R;
  const int64_t dims[3] = {I, J, K};
  const int64_t off[3] = {0, I * R, (I + J) * R};
  const int64_t nmax = std::max(I, std::max(J, K));
  if ((s = ensure(c, c->alsM, (size_t)nmax * R * 8))) return s;
  if ((s = ensure(c, c->alsSmall, (size_t)(3 * RR + 6 * RR + 3 * RR + R + 8) * 8))) return s;
  const int nf = f_hist ? 3 * sweeps : 0;
  if ((s = ensure(c, c->alsF, (size_t)(nf + 1) * 8))) return s;
  if (f_hist && (s = ensure(c, c->cpdGrad, (size_t)R * (I + J + K) * 8))) return s;
  double* M = (double*)c->alsM.p;
  double* grams = (double*)c->alsSmall.p;
  double* pi = grams + 3 * RR;
  double* V = pi + 6 * RR;
  double* Vt = V + RR;
  double* Vp = Vt + RR;
  double* theta = Vp + RR;
  double* fdev = (double*)c->alsF.p;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int l = 0; l < 3; ++l) {
      // M = T_(l) (⊙ of the other factors) with the newest factors (Alg. ALS order 1, 2, 3)
      if ((s = mttkrp_impl(c, d, T, w, l + 1, M))) return s;
      // V_l = Hadamard product of the other Grams (= Pi^(l)), its pseudo-inverse, W_l = M V_l^dagger
      if ((s = tf_grams(c, d, w, grams))) return s;
      if ((s = tf_hadamard(c, R, grams, pi))) return s;
      TF_CUDA(c, launch_jacobi_eig((int)R, pi + l * RR, R, Vt, V, theta, c->stream));
      TF_CUDA(c, launch_pinv_from_eig((int)R, V, theta, Vp, c->stream));
      c->total_launches += 2;
      if ((s = gemm_run(c, gemm_args(opnd(M, dims[l], false), opnd(Vp, R, true), dims[l], R, R, w + off[l],
                                     dims[l]))))
        return s;
      if (f_hist && (s = tf_cpd_eval(c, d, T, w, fdev + 3 * sw + l, (double*)c->cpdGrad.p, nullptr))) return s;
    }
  }
  if (f_hist && nf) {
    TF_CUDA(c, cudaMemcpyAsync(f_hist, fdev, (size_t)nf * 8, cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  return TF_OK;
}

}  // extern "C"
