// Small dense kernels of the compression stage (NEXT #3): the pieces of the truncated SVD of each
// unfolding through its Gram (Remark MLSVD-SVD; Lemma svd-transpose 4434-4436)
// that are not GEMMs — Householder orthonormalisation of the subspace-iteration block, the
// Rayleigh–Ritz eigenproblem (parallel cyclic Jacobi in one CTA), Ritz residuals and the sign
// convention of reading R23 — plus the rank choice of Alg. Compression and the
// MLSVD-energy initialisation. All reductions run in a fixed order.
#include <cfloat>
#include <cstdio>

#include "tf_device.cuh"
#include "../../include/tf.h"
#include "tf_internal.h"

namespace tfk {

namespace {

constexpr int kQrThreads = 1024;

// fixed-order block sum (every thread gets the result); red: >= 33 doubles of shared memory
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    red[32] = s;
  }
  __syncthreads();
  return red[32];
}

}  // namespace

// Householder QR, one CTA: Z = Q R with Q = H_0 ... H_{P-1} [I; 0]. A zero column gives H_j = I, so Q
// keeps orthonormal columns even when Z is rank deficient (exact low multilinear rank).
__global__ void __launch_bounds__(kQrThreads) k_house_qr(int64_t n, int P, double* __restrict__ Z, int64_t ldz,
                                                         double* __restrict__ Q, int64_t ldq) {
  __shared__ double red[33];
  __shared__ double beta[TF_MAX_R];
  __shared__ double dots[TF_MAX_R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < P; ++j) {
    double* x = Z + (int64_t)j * ldz;
    double s = 0.0;
    for (int64_t i = j + tid; i < n; i += kQrThreads) s += x[i] * x[i];
    const double nrm2 = block_sum(s, red);
    if (tid == 0) {
      const double x0 = j < n ? x[j] : 0.0;
      double b = 0.0;
      if (nrm2 > 0.0) {
        const double nrm = sqrt(nrm2);
        const double alpha = x0 >= 0.0 ? -nrm : nrm;
        const double v0 = x0 - alpha;
        const double vtv = (nrm2 - x0 * x0) + v0 * v0;
        if (vtv > 0.0) {
          b = 2.0 / vtv;
          x[j] = v0;
        }
      }
      beta[j] = b;
    }
    __syncthreads();
    const double bj = beta[j];
    if (bj != 0.0) {
      for (int c = j + 1 + warp; c < P; c += kQrThreads / 32) {
        const double* y = Z + (int64_t)c * ldz;
        double d = 0.0;
        for (int64_t i = j + lane; i < n; i += 32) d += x[i] * y[i];
        d = warp_sum(d);
        if (lane == 0) dots[c] = bj * d;
      }
      __syncthreads();
      const int64_t rows = n - j;
      const int64_t cols = P - j - 1;
      for (int64_t e = tid; e < rows * cols; e += kQrThreads) {
        const int64_t i = j + e % rows;
        const int c = j + 1 + (int)(e / rows);
        Z[i + (int64_t)c * ldz] -= dots[c] * x[i];
      }
    }
    __syncthreads();
  }
  // Q = H_0 (H_1 (... (H_{P-1} [I; 0])))
  for (int64_t e = tid; e < n * P; e += kQrThreads) {
    const int64_t i = e % n;
    const int c = (int)(e / n);
    Q[i + (int64_t)c * ldq] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = P - 1; j >= 0; --j) {
    const double bj = beta[j];
    if (bj == 0.0) continue;   // uniform across the block
    const double* v = Z + (int64_t)j * ldz;   // v_j = [1 .. at j: v0, below: x_i]
    for (int c = j + warp; c < P; c += kQrThreads / 32) {
      const double* y = Q + (int64_t)c * ldq;
      double d = 0.0;
      for (int64_t i = j + lane; i < n; i += 32) d += v[i] * y[i];
      d = warp_sum(d);
      if (lane == 0) dots[c] = bj * d;
    }
    __syncthreads();
    const int64_t rows = n - j;
    const int64_t cols = P - j;
    for (int64_t e = tid; e < rows * cols; e += kQrThreads) {
      const int64_t i = j + e % rows;
      const int c = j + (int)(e / rows);
      Q[i + (int64_t)c * ldq] -= dots[c] * v[i];
    }
    __syncthreads();
  }
}

// Parallel cyclic Jacobi (round-robin pairing, Golub–Van Loan sym.schur2 rotations) on the symmetric
// part of H, one CTA, H in shared memory; Vtmp accumulates the rotations; the output is sorted by
// |theta| decreasing (the ordering of Lemma svd-transpose) with ties kept in index order.
#ifdef TF_JACOBI_STATS
__device__ int g_jac_sweeps[64];
__device__ int g_jac_calls;
#endif
__global__ void __launch_bounds__(1024) k_jacobi_eig(int P, const double* __restrict__ H, int64_t ldh,
                                                     double* __restrict__ Vt, double* __restrict__ V,
                                                     double* __restrict__ theta, int vsm, int max_sweeps) {
  extern __shared__ double hs[];
  const int Pp = P + (P & 1);
  const int half = Pp / 2;
  const int LH = Pp + 1;                    // odd pitch: a row of H (stride LH) touches every bank
  double* cs = hs + (size_t)LH * Pp;        // [half][2]
  int* pr = reinterpret_cast<int*>(cs + 2 * half);   // [half][2]
  // the rotation accumulator lives in shared memory when it fits (P <= 112), else in global memory
  double* Vw = vsm ? reinterpret_cast<double*>(pr + 2 * half + 2) : Vt;
  __shared__ int rotated;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < Pp * Pp; e += nt) {
    const int r = e % Pp, c = e / Pp;
    double v = 0.0;
    if (r < P && c < P) v = 0.5 * (H[r + (int64_t)c * ldh] + H[c + (int64_t)r * ldh]);
    hs[r + LH * c] = v;
  }
  for (int e = tid; e < P * P; e += nt) Vw[e] = (e % P == e / P) ? 1.0 : 0.0;
  __shared__ double hmax_s;
  if (tid == 0) {
    double hm = 0.0;
    for (int i = 0; i < P; ++i) hm = fmax(hm, fabs(hs[i + LH * i]));
    hmax_s = hm;
  }
  __syncthreads();
  // rotations below DBL_EPSILON * 1e-3 * max|h_ii| cannot move an eigenvalue by more than ~1e-38 |H| or a
  // vector by more than ~1e-19 |H| / gap: skipping them stops the sweeps that would only chase rounding noise
  // among the (near-)zero eigenvalues of a rank-deficient Gram
  const double abs_floor = DBL_EPSILON * 1e-3 * hmax_s;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int step = 0; step < Pp - 1; ++step) {
      for (int k = tid; k < half; k += nt) {
        auto idx = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + step) % (Pp - 1); };
        int p = idx(k), q = idx(Pp - 1 - k);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < P) {
          const double apq = hs[p + LH * q];
          const double app = hs[p + LH * p], aqq = hs[q + LH * q];
          if (fabs(apq) > abs_floor && fabs(apq) > DBL_EPSILON * 0.5 * sqrt(fabs(app)) * sqrt(fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150) t = 0.5 / tau;
            else t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            rotated = 1;
          }
        }
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
        pr[2 * k] = p;
        pr[2 * k + 1] = q;
      }
      __syncthreads();
      // thread (lane-column x0 = tid % 128, pair group kg = tid / 128): no integer division in the loops
      const int x0 = tid & 127, kg = tid >> 7, ng = nt >> 7;
      // rows p, q  <-  J^T (rows)
      for (int x = x0; x < Pp; x += 128) {
        for (int k = kg; k < half; k += ng) {
          const double c = cs[2 * k], s = cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = pr[2 * k], q = pr[2 * k + 1];
          const double hp = hs[p + LH * x], hq = hs[q + LH * x];
          hs[p + LH * x] = c * hp - s * hq;
          hs[q + LH * x] = s * hp + c * hq;
        }
      }
      __syncthreads();
      // columns p, q  <-  (cols) J, and V <- V J; the rotated pair's own off-diagonal entries are set to 0
      for (int x = x0; x < Pp; x += 128) {
        for (int k = kg; k < half; k += ng) {
          const double c = cs[2 * k], s = cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = pr[2 * k], q = pr[2 * k + 1];
          const double hp = hs[x + LH * p], hq = hs[x + LH * q];
          hs[x + LH * p] = x == q ? 0.0 : c * hp - s * hq;
          hs[x + LH * q] = x == p ? 0.0 : s * hp + c * hq;
          if (x < P) {
            const double vp = Vw[x + (int64_t)P * p], vq = Vw[x + (int64_t)P * q];
            Vw[x + (int64_t)P * p] = c * vp - s * vq;
            Vw[x + (int64_t)P * q] = s * vp + c * vq;
          }
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
#ifdef TF_JACOBI_STATS
    if (tid == 0) g_jac_sweeps[min(g_jac_calls, 63)] = sweep + 1;
#endif
    if (!any) break;
  }
#ifdef TF_JACOBI_STATS
  if (tid == 0) g_jac_calls++;
#endif
  // sort by |theta| decreasing, ties in index order: rank_i = #{j : |t_j| > |t_i| or (== and j < i)}
  for (int i = tid; i < P; i += nt) {
    const double ti = fabs(hs[i + LH * i]);
    int rank = 0;
    for (int j = 0; j < P; ++j) {
      const double tj = fabs(hs[j + LH * j]);
      rank += (tj > ti) || (tj == ti && j < i);
    }
    theta[rank] = hs[i + LH * i];
    for (int r = 0; r < P; ++r) V[r + (int64_t)P * rank] = Vw[r + (int64_t)P * i];
  }
}

// res[j] = || ZV[:, j] - theta_j U[:, j] ||, one block per column
__global__ void k_eig_residual(int64_t n, const double* __restrict__ ZV, const double* __restrict__ U, int64_t ld,
                               const double* __restrict__ theta, double* __restrict__ res) {
  __shared__ double red[33];
  const int j = blockIdx.x;
  const double t = theta[j];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = ZV[i + ld * j] - t * U[i + ld * j];
    s += d * d;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) res[j] = sqrt(s);
}

// reading R23: the entry of largest magnitude of each column is made positive (first index on ties)
__global__ void k_sign_fix(int64_t n, double* __restrict__ U, int64_t ld) {
  __shared__ double bv[32];
  __shared__ long long bi[32];
  __shared__ double flip;
  double* u = U + ld * blockIdx.x;
  double best = -1.0;
  long long bidx = -1;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(u[i]);
    if (a > best) {   // strictly greater keeps the first index within a thread's strided run
      best = a;
      bidx = i;
    }
  }
  // warp argmax, ties -> smaller index
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi >= 0 && (bidx < 0 || oi < bidx))) {
      best = ob;
      bidx = oi;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -1.0;
    long long bx = -1;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      if (bv[w] > b || (bv[w] == b && bi[w] >= 0 && (bx < 0 || bi[w] < bx))) {
        b = bv[w];
        bx = bi[w];
      }
    flip = (bx >= 0 && u[bx] < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  if (flip < 0.0)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) u[i] = -u[i];
}

__global__ void k_sqrt_abs(int64_t n, const double* __restrict__ lam, double* __restrict__ sigma) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) sigma[i] = sqrt(fabs(lam[i]));
}

// Alg. Compression for one mode (single thread; P <= TF_MAX_R)
__global__ void k_trunc_rank(int P, const double* __restrict__ sigma, double tol3, int64_t* __restrict__ rank) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0.0;
  for (int r = 0; r < P; ++r) total += sigma[r] * sigma[r];
  int64_t chosen = P;
  for (int i = 1; i <= P; ++i) {
    double tail = 0.0;
    for (int r = i; r < P; ++r) tail += sigma[r] * sigma[r];
    const double rel = total > 0.0 ? tail / total : 0.0;
    if (rel < tol3) {
      chosen = i;
      break;
    }
  }
  *rank = chosen;
}

// MLSVD-energy initialisation (one CTA): the entries in the order (|s| decreasing, storage index
// increasing) — round r takes the first entry after the previous pick in that order — then
// W1[:, r] = s e_a, W2[:, r] = e_b, W3[:, r] = e_c.
__global__ void __launch_bounds__(1024) k_energy_init(int64_t P1, int64_t P2, int64_t P3,
                                                      const double* __restrict__ S, int64_t R,
                                                      double* __restrict__ w) {
  __shared__ double bv[32];
  __shared__ long long bi[32];
  __shared__ double prev_a;
  __shared__ long long prev_i;
  const int64_t N = P1 * P2 * P3;
  const int64_t n = R * (P1 + P2 + P3);
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) w[e] = 0.0;
  if (threadIdx.x == 0) {
    prev_a = INFINITY;
    prev_i = -1;
  }
  __syncthreads();
  for (int64_t r = 0; r < R; ++r) {
    const double pa = prev_a;
    const long long pi = prev_i;
    double best = -1.0;
    long long bidx = -1;
    for (int64_t e = threadIdx.x; e < N; e += blockDim.x) {
      const double a = fabs(S[e]);
      const bool after = (a < pa) || (a == pa && e > pi);
      if (after && a > best) {
        best = a;
        bidx = e;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi >= 0 && (bidx < 0 || oi < bidx))) {
        best = ob;
        bidx = oi;
      }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
      bv[warp] = best;
      bi[warp] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      long long bx = -1;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
        if (bv[q] > b || (bv[q] == b && bi[q] >= 0 && (bx < 0 || bi[q] < bx))) {
          b = bv[q];
          bx = bi[q];
        }
      if (bx >= 0) {
        const int64_t a = bx % P1, bb = (bx / P1) % P2, c = bx / (P1 * P2);
        w[a + P1 * r] = S[bx];
        w[R * P1 + bb + P2 * r] = 1.0;
        w[R * (P1 + P2) + c + P3 * r] = 1.0;
        prev_a = b;
        prev_i = bx;
      }
    }
    __syncthreads();
  }
}

// Column normalisation W[:, j] = Z[:, j] / ||Z[:, j]|| (one block per column); flags a zero column.
__global__ void k_col_normalize(int64_t n, const double* __restrict__ Z, int64_t ldz, double* __restrict__ W,
                                int64_t ldw, int* __restrict__ fail) {
  __shared__ double red[33];
  const int j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double z = Z[i + ldz * j];
    s += z * z;
  }
  s = block_sum(s, red);
  if (!(s > 0.0) || !isfinite(s)) {
    if (threadIdx.x == 0) atomicExch(fail, 1);
    return;
  }
  const double inv = 1.0 / sqrt(s);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) W[i + ldw * j] = Z[i + ldz * j] * inv;
}

// Cholesky B = L L^T of the symmetric part of B (P x P, one CTA, right-looking, B in shared memory) and
// Linv = L^{-1} by forward substitution (one column per thread). A pivot below 1e-8 (B comes from
// column-normalised vectors, so its diagonal is ~1) flags the block as numerically dependent.
__global__ void __launch_bounds__(1024) k_chol_inv(int P, const double* __restrict__ B, double* __restrict__ Linv,
                                                   int* __restrict__ fail) {
  extern __shared__ double bs[];   // P x P, column-major; the lower triangle becomes L
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < P * P; e += nt) {
    const int r = e % P, c = e / P;
    bs[e] = 0.5 * (B[r + (int64_t)P * c] + B[c + (int64_t)P * r]);
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < P; ++j) {
    if (tid == 0) {
      const double d = bs[j + P * j];
      if (!(d > 1e-8)) bad = 1;
      bs[j + P * j] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    const double ljj = bs[j + P * j];
    for (int i = j + 1 + tid; i < P; i += nt) bs[i + P * j] /= ljj;
    __syncthreads();
    const int m = P - j - 1;
    for (int e = tid; e < m * m; e += nt) {
      const int i = j + 1 + e % m, k = j + 1 + e / m;
      if (i >= k) bs[i + P * k] -= bs[i + P * j] * bs[k + P * j];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) atomicExch(fail, 1);
    return;
  }
  for (int c = tid; c < P; c += nt) {
    for (int i = 0; i < c; ++i) Linv[i + (int64_t)P * c] = 0.0;
    Linv[c + (int64_t)P * c] = 1.0 / bs[c + P * c];
    for (int i = c + 1; i < P; ++i) {
      double acc = 0.0;
      for (int k = c; k < i; ++k) acc += bs[i + P * k] * Linv[k + (int64_t)P * c];
      Linv[i + (int64_t)P * c] = -acc / bs[i + P * i];
    }
  }
}

cudaError_t launch_col_normalize(int64_t n, int P, const double* Z, int64_t ldz, double* W, int64_t ldw, int* fail,
                                 cudaStream_t st) {
  k_col_normalize<<<P, 256, 0, st>>>(n, Z, ldz, W, ldw, fail);
  return cudaGetLastError();
}

cudaError_t launch_chol_inv(int P, const double* B, double* Linv, int* fail, cudaStream_t st) {
  const size_t smem = (size_t)P * P * 8;
  cudaError_t e = cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_chol_inv<<<1, 1024, smem, st>>>(P, B, Linv, fail);
  return cudaGetLastError();
}

__global__ void k_truncate_rows(int64_t P1, int64_t P2, int64_t P3, int64_t R1, int64_t R2, int64_t R3, int64_t R,
                                const double* __restrict__ w0, double* __restrict__ w) {
  const int64_t n = R * (R1 + R2 + R3);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t src;
    if (e < R * R1) {
      src = (e % R1) + P1 * (e / R1);
    } else if (e < R * (R1 + R2)) {
      const int64_t x = e - R * R1;
      src = R * P1 + (x % R2) + P2 * (x / R2);
    } else {
      const int64_t x = e - R * (R1 + R2);
      src = R * (P1 + P2) + (x % R3) + P3 * (x / R3);
    }
    w[e] = w0[src];
  }
}

__global__ void k_normalize_cpd(int64_t n1, int64_t n2, int64_t n3, int64_t R, double* __restrict__ w,
                                double* __restrict__ lambda) {
  __shared__ double red[33];
  const int64_t r = blockIdx.x;
  const int64_t ns[3] = {n1, n2, n3};
  const int64_t off[3] = {0, R * n1, R * (n1 + n2)};
  double lam = 1.0;
  for (int l = 0; l < 3; ++l) {
    double* col = w + off[l] + ns[l] * r;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < ns[l]; i += blockDim.x) s += col[i] * col[i];
    s = block_sum(s, red);
    const double nrm = sqrt(s);
    lam *= nrm;
    if (nrm > 0.0) {
      const double inv = 1.0 / nrm;
      for (int64_t i = threadIdx.x; i < ns[l]; i += blockDim.x) col[i] *= inv;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) lambda[r] = lam;
}

cudaError_t launch_truncate_rows(const int64_t* P, const int64_t* Rt, int64_t R, const double* w0, double* w,
                                 cudaStream_t st) {
  k_truncate_rows<<<64, 256, 0, st>>>(P[0], P[1], P[2], Rt[0], Rt[1], Rt[2], R, w0, w);
  return cudaGetLastError();
}

cudaError_t launch_normalize_cpd(const int64_t* n, int64_t R, double* w, double* lambda, cudaStream_t st) {
  k_normalize_cpd<<<(unsigned)R, 256, 0, st>>>(n[0], n[1], n[2], R, w, lambda);
  return cudaGetLastError();
}

cudaError_t launch_house_qr(int64_t n, int P, double* Z, int64_t ldz, double* Q, int64_t ldq, cudaStream_t st) {
  k_house_qr<<<1, kQrThreads, 0, st>>>(n, P, Z, ldz, Q, ldq);
  return cudaGetLastError();
}

cudaError_t launch_jacobi_eig(int P, const double* H, int64_t ldh, double* Vtmp, double* V, double* theta,
                              cudaStream_t st, int max_sweeps) {
  const int Pp = P + (P & 1);
  size_t smem = (size_t)(Pp + 1) * Pp * 8 + (size_t)Pp * 8 + (size_t)Pp * 4 + 16;
  const int vsm = smem + (size_t)P * P * 8 <= 220 * 1024;
  if (vsm) smem += (size_t)P * P * 8;
  cudaError_t e = cudaFuncSetAttribute(k_jacobi_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_jacobi_eig<<<1, 1024, smem, st>>>(P, H, ldh, Vtmp, V, theta, vsm, max_sweeps);
  return cudaGetLastError();
}

#ifdef TF_JACOBI_STATS
}  // namespace tfk
extern "C" void tf_jacobi_stats_dump() {
  int h[64], n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, tfk::g_jac_calls, sizeof(int));
  cudaMemcpyFromSymbol(h, tfk::g_jac_sweeps, sizeof(h));
  printf("jacobi calls %d, sweeps:", n);
  for (int i = 0; i < n && i < 64; ++i) printf(" %d", h[i]);
  printf("\n");
}
namespace tfk {
#endif
cudaError_t launch_eig_residual(int64_t n, int P, const double* ZV, const double* U, int64_t ld, const double* theta,
                                double* res, cudaStream_t st) {
  k_eig_residual<<<P, 256, 0, st>>>(n, ZV, U, ld, theta, res);
  return cudaGetLastError();
}

cudaError_t launch_sign_fix(int64_t n, int P, double* U, int64_t ld, cudaStream_t st) {
  k_sign_fix<<<P, 256, 0, st>>>(n, U, ld);
  return cudaGetLastError();
}

cudaError_t launch_sqrt_abs(int64_t n, const double* lam, double* sigma, cudaStream_t st) {
  k_sqrt_abs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, lam, sigma);
  return cudaGetLastError();
}

cudaError_t launch_trunc_rank(int P, const double* sigma, double tol3, int64_t* rank, cudaStream_t st) {
  k_trunc_rank<<<1, 32, 0, st>>>(P, sigma, tol3, rank);
  return cudaGetLastError();
}

cudaError_t launch_energy_init(int64_t P1, int64_t P2, int64_t P3, const double* S, int64_t R, double* w,
                               cudaStream_t st) {
  k_energy_init<<<1, 1024, 0, st>>>(P1, P2, P3, S, R, w);
  return cudaGetLastError();
}

}  // namespace tfk
