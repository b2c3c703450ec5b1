// Small kernels of the hot path: Grams (a1), Hadamard chains (a7), the Jacobi scaling of the CG
// (a9 preconditioner) and the slab accumulation of the host-streamed evaluation. The GN matvec and
// CG themselves are the persistent cooperative kernel of k_cg.cu. Every reduction runs in a fixed
// order, so results are bitwise reproducible run to run.
#include "tf_internal.h"
#include "tf_device.cuh"

namespace tfk {

constexpr int kGT = 32;   // Gram tile (r, s)
constexpr int kGA = 32;   // rows per smem chunk

// Gpart[z][l][r + R*s] = sum_{a in chunk z} V_l[a, r] * W_l[a, s],   V = D o v (or W when v == nullptr)
// grid: x = 3 * ntile * ntile, y = ksplit
__global__ void k_gram_partial(Modes m, const double* __restrict__ v, const double* __restrict__ dscale,
                               int ntile, int64_t rows_per_split, double* __restrict__ Gpart) {
  __shared__ double sV[kGA][kGT + 1];
  __shared__ double sW[kGA][kGT + 1];
  const int R = (int)m.R;
  const int l = blockIdx.x / (ntile * ntile);
  const int tt = blockIdx.x % (ntile * ntile);
  const int r0 = (tt % ntile) * kGT, s0 = (tt / ntile) * kGT;
  const int64_t n = m.n[l];
  const double* W = m.W[l];
  const double* V = v ? v + m.off[l] : W;
  const int64_t a_begin = blockIdx.y * rows_per_split;
  const int64_t a_end = min(n, a_begin + rows_per_split);
  const int tid = threadIdx.x;
  const int tr = tid & 15, ts = tid >> 4;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t a0 = a_begin; a0 < a_end; a0 += kGA) {
    for (int idx = tid; idx < kGA * kGT; idx += blockDim.x) {
      const int a = idx % kGA, c = idx / kGA;
      const int64_t ga = a0 + a;
      const int r = r0 + c, s = s0 + c;
      double vv = 0.0, ww = 0.0;
      if (ga < a_end) {
        if (r < R) {
          vv = V[ga + n * r];
          if (v && dscale) vv *= dscale[l * R + r];
        }
        if (s < R) ww = W[ga + n * s];
      }
      sV[a][c] = vv;
      sW[a][c] = ww;
    }
    __syncthreads();
#pragma unroll 8
    for (int a = 0; a < kGA; ++a) {
      const double v0 = sV[a][tr], v1 = sV[a][tr + 16];
      const double w0 = sW[a][ts], w1 = sW[a][ts + 16];
      acc[0][0] = fma(v0, w0, acc[0][0]);
      acc[0][1] = fma(v0, w1, acc[0][1]);
      acc[1][0] = fma(v1, w0, acc[1][0]);
      acc[1][1] = fma(v1, w1, acc[1][1]);
    }
    __syncthreads();
  }
  double* out = Gpart + ((int64_t)blockIdx.y * 3 + l) * R * R;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = r0 + tr + 16 * i, s = s0 + ts + 16 * j;
      if (r < R && s < R) out[r + (int64_t)R * s] = acc[i][j];
    }
}

// G[l] = sum_z Gpart[z][l] (fixed order). If pi != nullptr also
// S_l = sum_{l' != l} Pi^(l,l') * G_l'  with Pi^(1,2) = pi[3], Pi^(1,3) = pi[4], Pi^(2,3) = pi[5].
__global__ void k_gram_final(int64_t R, int ksplit, const double* __restrict__ Gpart, const double* __restrict__ pi,
                             double* __restrict__ G, double* __restrict__ S) {
  const int64_t RR = R * R;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < RR; q += (int64_t)gridDim.x * blockDim.x) {
    double g[3] = {0.0, 0.0, 0.0};
    for (int z = 0; z < ksplit; ++z)
#pragma unroll
      for (int l = 0; l < 3; ++l) g[l] += Gpart[((int64_t)z * 3 + l) * RR + q];
#pragma unroll
    for (int l = 0; l < 3; ++l) G[l * RR + q] = g[l];
    if (pi) {
      const double p12 = pi[3 * RR + q], p13 = pi[4 * RR + q], p23 = pi[5 * RR + q];
      S[0 * RR + q] = p12 * g[1] + p13 * g[2];
      S[1 * RR + q] = p12 * g[0] + p23 * g[2];
      S[2 * RR + q] = p13 * g[0] + p23 * g[1];
    }
  }
}

__global__ void k_hadamard(int64_t R, const double* __restrict__ g, double* __restrict__ pi) {
  const int64_t RR = R * R;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < RR; q += (int64_t)gridDim.x * blockDim.x) {
    const double a = g[q], b = g[RR + q], c = g[2 * RR + q];
    pi[q] = b * c;            // Pi^(1) = pi_B * pi_C
    pi[RR + q] = a * c;       // Pi^(2) = pi_A * pi_C
    pi[2 * RR + q] = a * b;   // Pi^(3) = pi_A * pi_B
    pi[3 * RR + q] = c;       // Pi^(1,2)
    pi[4 * RR + q] = b;       // Pi^(1,3)
    pi[5 * RR + q] = a;       // Pi^(2,3)
  }
}

__global__ void k_jacobi_scale(int64_t R, const double* __restrict__ pi, double lambda, const double* __restrict__ damp,
                               double* __restrict__ d) {
  const int64_t RR = R * R;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < 3 * R; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = q / R, r = q % R;
    // M_(l,a,r) = Pi^(l)_rr + lambda * D_(l,r)   (D = I when damp == nullptr)
    d[q] = 1.0 / sqrt(pi[l * RR + r + R * r] + lambda * (damp ? damp[q] : 1.0));
  }
}

// Tensor Fox's diagonal regularizer from the Grams: ||W_r|| = sqrt(pi^(l)_rr),
// G = max_r max{||Y_r|| ||Z_r||, ||X_r|| ||Z_r||, ||X_r|| ||Y_r||}, gamma_X^(r) = ||Y_r|| ||Z_r|| G, ...
// One block; the max is order-independent, so the result is deterministic.
__global__ void k_reg_gamma(int64_t R, const double* __restrict__ grams, double* __restrict__ gamma) {
  __shared__ double red[32];
  const int64_t RR = R * R;
  double m = 0.0;
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
    const double x = sqrt(grams[r + R * r]), y = sqrt(grams[RR + r + R * r]), z = sqrt(grams[2 * RR + r + R * r]);
    m = fmax(m, fmax(y * z, fmax(x * z, x * y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  double G = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) G = fmax(G, red[i]);
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
    const double x = sqrt(grams[r + R * r]), y = sqrt(grams[RR + r + R * r]), z = sqrt(grams[2 * RR + r + R * r]);
    gamma[r] = y * z * G;
    gamma[R + r] = x * z * G;
    gamma[2 * R + r] = x * y * G;
  }
}

__global__ void k_axpy1(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    y[q] += x[q];
}

// ---------------------------------------------------------------------------------------------- host side
static int gram_ksplit(const Modes& m, int64_t* rows_per_split) {
  const int ntile = (int)((m.R + kGT - 1) / kGT);
  const int64_t nmax = std::max(m.n[0], std::max(m.n[1], m.n[2]));
  const int base = 3 * ntile * ntile;
  int ks = (int)std::max<int64_t>(1, std::min<int64_t>((296 + base - 1) / base, (nmax + 255) / 256));
  int64_t rps = (nmax + ks - 1) / ks;
  rps = ((rps + kGA - 1) / kGA) * kGA;
  *rows_per_split = rps;
  return (int)((nmax + rps - 1) / rps);
}

int gram_partial_slots(const Modes& m) {
  int64_t rps;
  return gram_ksplit(m, &rps);
}

static cudaError_t gram_common(const Modes& m, const double* v, const double* dscale, const double* pi,
                               double* Gpart, double* G, double* S, cudaStream_t st) {
  int64_t rps;
  const int ks = gram_ksplit(m, &rps);
  const int ntile = (int)((m.R + kGT - 1) / kGT);
  dim3 grid(3 * ntile * ntile, ks);
  k_gram_partial<<<grid, 256, 0, st>>>(m, v, dscale, ntile, rps, Gpart);
  const int64_t RR = m.R * m.R;
  k_gram_final<<<(int)std::min<int64_t>((RR + 255) / 256, 1024), 256, 0, st>>>(m.R, ks, Gpart, pi, G, S);
  return cudaGetLastError();
}

cudaError_t launch_grams_ws(const Modes& m, double* Gpart, double* grams, cudaStream_t st) {
  return gram_common(m, nullptr, nullptr, nullptr, Gpart, grams, nullptr, st);
}

cudaError_t launch_hadamard(int64_t R, const double* grams, double* pi, cudaStream_t st) {
  const int64_t RR = R * R;
  k_hadamard<<<(int)std::min<int64_t>((RR + 255) / 256, 1024), 256, 0, st>>>(R, grams, pi);
  return cudaGetLastError();
}

cudaError_t launch_jacobi_scale(const Modes& m, const double* pi, double lambda, const double* damp, double* dscale,
                                cudaStream_t st) {
  k_jacobi_scale<<<(int)((3 * m.R + 255) / 256), 256, 0, st>>>(m.R, pi, lambda, damp, dscale);
  return cudaGetLastError();
}

cudaError_t launch_reg_gamma(int64_t R, const double* grams, double* gamma, cudaStream_t st) {
  k_reg_gamma<<<1, 256, 0, st>>>(R, grams, gamma);
  return cudaGetLastError();
}

static int vec_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 592)); }

int cg_partial_slots(const Modes& m) {
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  return vec_blocks(n);
}

cudaError_t launch_axpy1(int64_t n, const double* x, double* y, cudaStream_t st) {
  k_axpy1<<<vec_blocks(n), 256, 0, st>>>(n, x, y);
  return cudaGetLastError();
}

}  // namespace tfk

namespace tfk {

// ---------------------------------------------------------------------------------- dGN outer-loop helpers
// Fixed-order reductions: per-block partials, then one block sums them in order (deterministic).
constexpr int kRedBlocks = 296;

// partial[b][0..3] = { sum g*x, sum x*y, sum x*x, max |g| } over this block's grid-stride share
__global__ void k_dots_partial(int64_t n, const double* __restrict__ g, const double* __restrict__ x,
                               const double* __restrict__ y, double* __restrict__ partial) {
  __shared__ double red[4][8];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double xv = x[q], gv = g[q];
    s0 = fma(gv, xv, s0);
    s1 = fma(xv, y[q], s1);
    s2 = fma(xv, xv, s2);
    m = fmax(m, fabs(gv));
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = s0;
    red[1][w] = s1;
    red[2][w] = s2;
    red[3][w] = m;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
      v = threadIdx.x == 3 ? fmax(v, red[3][i]) : v + red[threadIdx.x][i];
    partial[blockIdx.x * 4 + threadIdx.x] = v;
  }
}

// partial[b][0..1] = { sum |t|, sum t^2 } over the I x J x K tensor with leading dimension ldT
// sum |t| and sum t^2 over the tensor (one streaming pass). Dense storage (ldT = I, 16-byte aligned) is read as
// a flat array of double2 with 8 independent loads in flight per thread; a padded leading dimension walks the
// rows. Each thread's sums follow a fixed order (deterministic).
__global__ void __launch_bounds__(256) k_tsums_partial(int64_t I, int64_t JK, int64_t ldT,
                                                       const double* __restrict__ T, double* __restrict__ partial) {
  __shared__ double red[2][8];
  constexpr int U = 8;
  double sa[U], s2[U];
#pragma unroll
  for (int u = 0; u < U; ++u) sa[u] = s2[u] = 0.0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  if (ldT == I && (reinterpret_cast<uintptr_t>(T) & 15) == 0) {
    const int64_t N = I * JK, N2 = N / 2;
    const double2* T2 = reinterpret_cast<const double2*>(T);
    int64_t q = tid;
    for (; q + (U - 1) * stride < N2; q += U * stride) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(T2 + q + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sa[u] += fabs(v[u].x) + fabs(v[u].y);
        s2[u] = fma(v[u].y, v[u].y, fma(v[u].x, v[u].x, s2[u]));
      }
    }
    for (; q < N2; q += stride) {
      const double2 v = __ldg(T2 + q);
      sa[0] += fabs(v.x) + fabs(v.y);
      s2[0] = fma(v.y, v.y, fma(v.x, v.x, s2[0]));
    }
    if ((N & 1) && tid == 0) {
      const double t = T[N - 1];
      sa[1] += fabs(t);
      s2[1] = fma(t, t, s2[1]);
    }
  } else {
    for (int64_t jk = blockIdx.x; jk < JK; jk += gridDim.x)
      for (int64_t i = threadIdx.x; i < I; i += blockDim.x) {
        const double t = T[i + ldT * jk];
        sa[0] += fabs(t);
        s2[0] = fma(t, t, s2[0]);
      }
  }
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a += sa[u];
    b += s2[u];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = a;
    red[1][w] = b;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double v = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) v += red[threadIdx.x][i];
    partial[blockIdx.x * 2 + threadIdx.x] = v;
  }
}

// out[c] = ordered combination over blocks of partial[b][c] (c < ncomp <= 4; component max_comp is a max):
// every thread folds a fixed strided subset of the blocks, then the warps and the block combine in a fixed
// order (deterministic; independent loads instead of one serial chain of L2 round trips)
__global__ void __launch_bounds__(256) k_partial_final(int nblk, int ncomp, int max_comp,
                                                       const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double red[4][8];
  for (int c = 0; c < ncomp; ++c) {
    const bool mx = c == max_comp;
    double v = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
      const double p = partial[b * ncomp + c];
      v = mx ? fmax(v, p) : v + p;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = mx ? fmax(v, u) : v + u;
    }
    if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < ncomp) {
    const bool mx = (int)threadIdx.x == max_comp;
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = mx ? fmax(v, red[threadIdx.x][w]) : v + red[threadIdx.x][w];
    out[threadIdx.x] = v;
  }
}

// gate (nullable): the CG state of the step; a CG that met a non-finite alpha/beta leaves w untouched (the dGN
// loop then stops with reason 8 at w^(k-1), as the oracle does)
__global__ void k_axpy_inplace(int64_t n, const double* __restrict__ x, double* __restrict__ w, const CgState* gate) {
  if (gate && gate->nonfinite) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    w[q] += x[q];
}

// Norm balancing: column r of every mode gets the norm (prod_l ||w_r^(l)||)^(1/3); column
// norms from the Grams' diagonals. Columns of a rank-one term with a zero factor are left unchanged.
__global__ void k_balance(Modes m, const double* __restrict__ grams, double* __restrict__ w, const CgState* gate) {
  if (gate && gate->nonfinite) return;
  const int64_t R = m.R, RR = R * R;
  const int64_t n = R * (m.n[0] + m.n[1] + m.n[2]);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int l = q >= m.off[2] ? 2 : (q >= m.off[1] ? 1 : 0);
    const int64_t r = (q - m.off[l]) / m.n[l];
    const double n0 = sqrt(grams[r + R * r]), n1 = sqrt(grams[RR + r + R * r]), n2 = sqrt(grams[2 * RR + r + R * r]);
    const double prod = n0 * n1 * n2;
    if (prod == 0.0) continue;
    const double nl = l == 0 ? n0 : (l == 1 ? n1 : n2);
    w[q] *= cbrt(prod) / nl;
  }
}

cudaError_t launch_dots(int64_t n, const double* g, const double* x, const double* y, double* partial, double* out,
                        cudaStream_t st) {
  k_dots_partial<<<kRedBlocks, 256, 0, st>>>(n, g, x, y, partial);
  k_partial_final<<<1, 256, 0, st>>>(kRedBlocks, 4, 3, partial, out);
  return cudaGetLastError();
}

cudaError_t launch_tsums(int64_t I, int64_t J, int64_t K, int64_t ldT, const double* T, double* partial, double* out,
                         cudaStream_t st) {
  k_tsums_partial<<<kRedBlocks, 256, 0, st>>>(I, J * K, ldT, T, partial);
  k_partial_final<<<1, 256, 0, st>>>(kRedBlocks, 2, -1, partial, out);
  return cudaGetLastError();
}

__global__ void k_scale_copy(int64_t n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    y[q] = alpha * x[q];
}

cudaError_t launch_scale_copy(int64_t n, double alpha, const double* x, double* y, cudaStream_t st) {
  k_scale_copy<<<vec_blocks(n), 256, 0, st>>>(n, alpha, x, y);
  return cudaGetLastError();
}

cudaError_t launch_axpy_inplace(int64_t n, const double* x, double* w, const CgState* gate, cudaStream_t st) {
  k_axpy_inplace<<<vec_blocks(n), 256, 0, st>>>(n, x, w, gate);
  return cudaGetLastError();
}

cudaError_t launch_balance(const Modes& m, const double* grams, double* w, const CgState* gate, cudaStream_t st) {
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  k_balance<<<vec_blocks(n), 256, 0, st>>>(m, grams, w, gate);
  return cudaGetLastError();
}

int red_blocks() { return kRedBlocks; }

}  // namespace tfk
