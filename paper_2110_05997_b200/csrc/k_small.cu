// Small kernels of the hot path: Grams (a1), Hadamard chains (a7), the Gauss-Newton matvec by
// Thm Hv (a8) and the device-resident CG of Alg. CG-dGN (a9). All O(R^2 * sum I) work; every
// reduction runs in a fixed order (block partials + last-block ordered sum), so results are
// bitwise reproducible run to run.
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

__global__ void k_jacobi_scale(int64_t R, const double* __restrict__ pi, double lambda, double* __restrict__ d) {
  const int64_t RR = R * R;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < 3 * R; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = q / R, r = q % R;
    d[q] = 1.0 / sqrt(pi[l * RR + r + R * r] + lambda);  // M_(l,a,r) = Pi^(l)_rr + lambda
  }
}

// Ordered last-block reduction helper: partial[blockIdx] = v (block sum); returns true in the last
// block to finish, which then sees every partial.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;  // valid in thread 0
}

__device__ __forceinline__ bool last_block_arrive(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ double ordered_sum(const double* partial, int n, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += partial[i];
  return block_sum(v, red);
}

constexpr int kMR = 64;   // apply tile rows
constexpr int kMS = 32;   // apply tile cols
constexpr int kMK = 16;   // inner chunk

struct ApplyTiles {
  int tiles_r[3];
  int tiles_s;
  int total;
};

__host__ __device__ inline ApplyTiles apply_tiles(const Modes& m) {
  ApplyTiles t;
  t.tiles_s = (int)((m.R + kMS - 1) / kMS);
  t.total = 0;
  for (int l = 0; l < 3; ++l) {
    t.tiles_r[l] = (int)((m.n[l] + kMR - 1) / kMR);
    t.total += t.tiles_r[l] * t.tiles_s;
  }
  return t;
}

// y = D (V Pi^(l) + W S_l + lambda V) for every mode l, V = D v (Thm Hv; three-step
// Jacobi product). If dot_partial != nullptr, also partial sums of <v, y> per block and,
// in the last block, alpha = rr / <p, z> into the CG state.
__global__ void __launch_bounds__(256) k_matvec_apply(Modes m, const double* __restrict__ v, double lambda,
                                                      const double* __restrict__ pi, const double* __restrict__ S,
                                                      const double* __restrict__ dscale, double* __restrict__ y,
                                                      double* __restrict__ dot_partial, CgState* cg) {
  __shared__ double sX[kMK][kMR + 1];
  __shared__ double sM[kMK][kMS + 1];
  __shared__ double red[8];
  if (cg && cg->done) return;
  const ApplyTiles at = apply_tiles(m);
  int b = blockIdx.x, l = 0;
  while (b >= at.tiles_r[l] * at.tiles_s) {
    b -= at.tiles_r[l] * at.tiles_s;
    ++l;
  }
  const int R = (int)m.R;
  const int64_t RR = (int64_t)R * R;
  const int64_t n = m.n[l];
  const int64_t a0 = (int64_t)(b % at.tiles_r[l]) * kMR;
  const int s0 = (b / at.tiles_r[l]) * kMS;
  const double* W = m.W[l];
  const double* Vv = v + m.off[l];
  const double* P = pi + l * RR;   // Pi^(l)
  const double* Sl = S + l * RR;
  const double* D = dscale ? dscale + l * R : nullptr;
  const int tid = threadIdx.x, ta = tid & 15, ts = tid >> 4;
  double acc[4][2] = {};
  for (int pass = 0; pass < 2; ++pass) {
    const double* X = pass == 0 ? Vv : W;
    const double* M = pass == 0 ? P : Sl;
    for (int r0 = 0; r0 < R; r0 += kMK) {
      for (int idx = tid; idx < kMK * kMR; idx += blockDim.x) {
        const int a = idx % kMR, c = idx / kMR;
        const int64_t ga = a0 + a;
        const int r = r0 + c;
        double xv = 0.0;
        if (ga < n && r < R) {
          xv = X[ga + n * r];
          if (pass == 0 && D) xv *= D[r];
        }
        sX[c][a] = xv;
      }
      for (int idx = tid; idx < kMK * kMS; idx += blockDim.x) {
        const int c = idx % kMK, s = idx / kMK;
        const int r = r0 + c;
        sM[c][s] = (r < R && s0 + s < R) ? M[r + (int64_t)R * (s0 + s)] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < kMK; ++c) {
        double xa[4], ms[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) xa[i] = sX[c][ta + 16 * i];
#pragma unroll
        for (int j = 0; j < 2; ++j) ms[j] = sM[c][ts + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) acc[i][j] = fma(xa[i], ms[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  double dsum = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t ga = a0 + ta + 16 * i;
      const int s = s0 + ts + 16 * j;
      if (ga < n && s < R) {
        const double vin = Vv[ga + n * s];
        const double ds = D ? D[s] : 1.0;
        const double yv = (acc[i][j] + lambda * vin * ds) * ds;
        y[m.off[l] + ga + n * s] = yv;
        dsum = fma(vin, yv, dsum);
      }
    }
  if (dot_partial) {
    const double t = block_sum(dsum, red);
    if (threadIdx.x == 0) dot_partial[blockIdx.x] = t;
    if (last_block_arrive(&cg->counter)) {
      const double pz = ordered_sum(dot_partial, gridDim.x, red);
      if (threadIdx.x == 0) {
        cg->counter = 0;
        cg->pz = pz;
        const double alpha = cg->rr / pz;
        cg->alpha = alpha;
        if (!isfinite(alpha)) {
          cg->nonfinite = cg->iters + 1;
          cg->done = 1;
        }
      }
    }
  }
}

// x += alpha p; r -= alpha z; partial ||r||^2; last block: beta, rr, iters, done.
__global__ void k_cg_update(int64_t n, double tol, double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ z, double* __restrict__ partial,
                            CgState* cg) {
  __shared__ double red[8];
  if (cg->done) return;
  const double alpha = cg->alpha;
  double s = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    x[q] = fma(alpha, p[q], x[q]);
    const double rn = fma(-alpha, z[q], r[q]);
    r[q] = rn;
    s = fma(rn, rn, s);
  }
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block_arrive(&cg->counter2)) {
    const double rr_new = ordered_sum(partial, gridDim.x, red);
    if (threadIdx.x == 0) {
      cg->counter2 = 0;
      const double beta = rr_new / cg->rr;
      cg->beta = beta;
      cg->rr = rr_new;
      cg->iters += 1;
      if (!isfinite(beta)) {
        cg->nonfinite = cg->iters;
        cg->done = 1;
      } else if (rr_new < tol) {
        cg->done = 1;
      }
    }
  }
}

__global__ void k_cg_direction(int64_t n, const double* __restrict__ r, double* __restrict__ p, const CgState* cg) {
  if (cg->done) return;
  const double beta = cg->beta;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    p[q] = fma(beta, p[q], r[q]);
}

// x = 0; r = D rhs; p = r; rr = ||r||^2
__global__ void k_cg_init(int64_t n, Modes m, const double* __restrict__ rhs, const double* __restrict__ dscale,
                          double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                          double* __restrict__ partial, CgState* cg) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double d = 1.0;
    if (dscale) {
      const int l = q >= m.off[2] ? 2 : (q >= m.off[1] ? 1 : 0);
      const int64_t rr = (q - m.off[l]) / m.n[l];
      d = dscale[l * m.R + rr];
    }
    const double v = rhs[q] * d;
    x[q] = 0.0;
    r[q] = v;
    p[q] = v;
    s = fma(v, v, s);
  }
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block_arrive(&cg->counter)) {
    const double rr = ordered_sum(partial, gridDim.x, red);
    if (threadIdx.x == 0) {
      cg->counter = 0;
      cg->rr = rr;
      cg->rr0 = rr;
      cg->alpha = cg->beta = cg->pz = 0.0;
      cg->iters = 0;
      cg->done = 0;
      cg->nonfinite = 0;
    }
  }
}

__global__ void k_cg_finish(int64_t n, Modes m, const double* __restrict__ dscale, double* __restrict__ x) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int l = q >= m.off[2] ? 2 : (q >= m.off[1] ? 1 : 0);
    const int64_t rr = (q - m.off[l]) / m.n[l];
    x[q] *= dscale[l * m.R + rr];
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

cudaError_t launch_jacobi_scale(const Modes& m, const double* pi, double lambda, double* dscale, cudaStream_t st) {
  k_jacobi_scale<<<(int)((3 * m.R + 255) / 256), 256, 0, st>>>(m.R, pi, lambda, dscale);
  return cudaGetLastError();
}

int matvec_blocks(const Modes& m) { return apply_tiles(m).total; }

// ws.partial must hold gram_partial_slots(m)*3*R*R doubles at ws.partial (Gram split-K partials) and
// ws.nblk_dot doubles after that for dot partials.
cudaError_t launch_matvec_core(const Modes& m, const double* v, double lambda, const MatvecWs& ws, bool jacobi,
                               double* y, double* dot_partial, CgState* cg, cudaStream_t st) {
  cudaError_t e = gram_common(m, v, jacobi ? ws.dscale : nullptr, ws.pi, ws.partial, ws.G, ws.S, st);
  if (e != cudaSuccess) return e;
  const int nb = matvec_blocks(m);
  k_matvec_apply<<<nb, 256, 0, st>>>(m, v, lambda, ws.pi, ws.S, jacobi ? ws.dscale : nullptr, y, dot_partial, cg);
  return cudaGetLastError();
}

cudaError_t launch_matvec(const Modes& m, const double* v, double lambda, const MatvecWs& ws, bool jacobi, double* y,
                          cudaStream_t st) {
  return launch_matvec_core(m, v, lambda, ws, jacobi, y, nullptr, nullptr, st);
}

static int vec_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 592)); }

int cg_partial_slots(const Modes& m) {
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  return std::max(vec_blocks(n), matvec_blocks(m));
}

cudaError_t launch_cg_init(int64_t n, const double* rhs, const double* dscale, const Modes& m, double* x, double* r,
                           double* p, double* partial, int nblk, CgState* cg, cudaStream_t st) {
  (void)nblk;
  k_cg_init<<<vec_blocks(n), 256, 0, st>>>(n, m, rhs, dscale, x, r, p, partial, cg);
  return cudaGetLastError();
}

// One CG iteration: z = B p (grams of V = D p, S, apply + <p,z> + alpha), update, new direction.
cudaError_t launch_cg_iteration(const Modes& m, double lambda, const MatvecWs& ws, bool jacobi, double tol, double* x,
                                double* r, double* p, double* z, CgState* cg, cudaStream_t st) {
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  double* dotp = ws.partial + (int64_t)gram_partial_slots(m) * 3 * m.R * m.R;
  cudaError_t e = launch_matvec_core(m, p, lambda, ws, jacobi, z, dotp, cg, st);
  if (e != cudaSuccess) return e;
  k_cg_update<<<vec_blocks(n), 256, 0, st>>>(n, tol, x, r, p, z, dotp, cg);
  k_cg_direction<<<vec_blocks(n), 256, 0, st>>>(n, r, p, cg);
  return cudaGetLastError();
}

cudaError_t launch_cg_finish(int64_t n, const Modes& m, const double* dscale, bool jacobi, double* x, cudaStream_t st) {
  if (!jacobi) return cudaSuccess;
  k_cg_finish<<<vec_blocks(n), 256, 0, st>>>(n, m, dscale, x);
  return cudaGetLastError();
}

cudaError_t launch_axpy1(int64_t n, const double* x, double* y, cudaStream_t st) {
  k_axpy1<<<vec_blocks(n), 256, 0, st>>>(n, x, y);
  return cudaGetLastError();
}

}  // namespace tfk
