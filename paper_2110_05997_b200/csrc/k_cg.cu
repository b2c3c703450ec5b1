// Persistent cooperative kernels for the Gauss-Newton matvec (Thm Hv, row a8) and Alg. CG-dGN (row a9).
//
// One launch runs the whole CG: every block stays resident (cooperative launch, one block per SM) and
// the iteration is three grid-wide stages separated by grid barriers:
//   G  (Gram)  G_l = V_l^T W_l,  V = D (r + beta p)           3 R x R outputs, DMMA, fixed-order
//   Y  (apply) p <- r + beta p;  z = D (V Pi^(l) + W S_l + lambda V) with S_l = sum_{l'!=l} Pi^(l,l') * G_l'
//              (Thm Hv; three-step Jacobi product PAPER.md:2690-2695); partial <p, z>
//   U  (update) alpha = ||r||^2 / <p,z>; x += alpha p; r -= alpha z; partial ||r||^2  -> beta next stage
// All scalars are recomputed by every block from per-block partials summed in a fixed order, so the
// whole solve is deterministic and needs no host round trip.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "tf_internal.h"
#include "tf_device.cuh"

namespace cg = cooperative_groups;

namespace tfk {

unsigned long long* cg_debug_tstamp();
constexpr int kCgThreads = 256;
constexpr int kGramZ = 64;   // max row splits of one mode's Gram (full-width partials)

struct CgArgs {
  Modes m;
  const double* pi;       // 6 R x R
  const double* dscale;   // 3R or nullptr: Jacobi scaling M^{-1/2} per (mode, r)
  const double* damp;     // 3R or nullptr: damping matrix D per (mode, r) (the paper's gamma; nullptr = I)
  double lambda, tol;
  int maxiter;
  const double* rhs;      // CG right-hand side (w-coordinates)
  const double* v;        // matvec input (matvec mode)
  double* x;              // CG solution / matvec output y
  double *r, *p, *z;      // CG vectors; p holds 2n doubles: the current and the next direction
  double* G;              // kGramZ x 3 x R x R Gram partials
  double* S;              // 3 x R x R
  double* part;           // 2 * gridDim partials
  CgState* st;
  int mode;               // 0 = CG, 1 = single matvec y = (J^T J + lambda I) v
  unsigned long long* tstamp;   // optional: block-0 globaltimer at each stage boundary (profiling)
};

__device__ __forceinline__ void stamp(const CgArgs& A, int slot) {
  if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && slot < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.tstamp[slot] = t;
  }
}

__device__ __forceinline__ int mode_of(const Modes& m, int64_t q) { return q >= m.off[2] ? 2 : (q >= m.off[1] ? 1 : 0); }

// V element (a, r) of mode l: D_l[r] * (r_vec + beta * p)   (CG)   or   v   (matvec)
struct VSrc {
  const double* a;     // r vector or v
  const double* b;     // p (CG) or nullptr
  double beta;
  const double* D;     // dscale or nullptr
  __device__ __forceinline__ double raw(int64_t q) const { return b ? fma(beta, b[q], a[q]) : a[q]; }
};

// ---- stage G: G_l[r + R s] = sum_a V_l[a, r] W_l[a, s]. Items (mode l, row split z): every item computes
// the FULL R x R partial of its rows, so each row of V (= D (r + beta p)) and W is read once per
// iteration (32 x 32 output tiles re-read every column block 4x: the stage was bound by L2 -> SM traffic).
// The item's rows are staged by cp.async in chunks of kGRows as [column][row] (pitch 4 mod 16: conflict-free
// fragments); warp w owns the r-tiles mi = w, w + 8 (all 8-column tiles ni), so per k-step it loads <= 2 A
// and NT B fragments for <= 2 NT DMMAs. The Z partials per mode are summed in stage S in a fixed order.
#ifndef TF_GRAM_DIV
#define TF_GRAM_DIV 3
#endif
constexpr int kGRows = 32, kGLd = kGRows + 4;
__device__ __forceinline__ int gram_splits(const Modes& m) {
  (void)m;
  return max(1, min(kGramZ, (int)gridDim.x / TF_GRAM_DIV));
}
__host__ __device__ constexpr size_t gram_smem_doubles(int R4) { return (size_t)3 * R4 * kGLd; }

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
// 16-byte copy with zero fill beyond src_bytes (0, 8 or 16)
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <int NT>
__device__ void stage_gram(const CgArgs& A, const VSrc& V, double* smem) {
  const Modes& m = A.m;
  const int R = (int)m.R;
  const int R4 = 4 * ((R + 3) / 4);
  const int Z = gram_splits(m);
  const int items = 3 * Z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const bool hasP = V.b != nullptr;
  double* sR = smem;                 // [R4][kGLd]
  double* sP = sR + R4 * kGLd;
  double* sW = sP + R4 * kGLd;
  constexpr int MT = (NT + 7) / 8;   // r-tiles per warp (<= 2)
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int z = item % Z, l = item / Z;
    const int64_t n = m.n[l];
    const double* W = m.W[l];
    const int64_t off = m.off[l];
    const double* D = V.D ? V.D + l * R : nullptr;
    const int64_t rps = ((n + 4 * Z - 1) / (4 * Z)) * 4;          // rows per split
    const int64_t zb = z * rps, ze = min(n, zb + rps);
    double dr[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int r = 8 * (warp + 8 * i) + g;
      dr[i] = (D && r < R) ? D[r] : 1.0;
    }
    double acc[MT][NT][2] = {};
    const bool pair16 = ((n | off | zb) & 1) == 0 &&
                        ((reinterpret_cast<uintptr_t>(V.a) | reinterpret_cast<uintptr_t>(W) |
                          reinterpret_cast<uintptr_t>(hasP ? V.b : V.a)) & 15) == 0;
    for (int64_t c0 = zb; c0 < ze; c0 += kGRows) {
      __syncthreads();   // the previous chunk (or item) is consumed
      if (pair16) {   // 16-byte row pairs (every column start aligned)
        for (int idx = threadIdx.x; idx < (kGRows / 2) * R4; idx += blockDim.x) {
          const int a = 2 * (idx % (kGRows / 2)), col = idx / (kGRows / 2);
          int64_t rem = ze - (c0 + a);
          rem = rem < 0 ? 0 : (rem > 2 ? 2 : rem);
          const int valid = col < R ? (int)rem : 0;
          const int64_t ix = valid ? c0 + a + n * col : 0;
          cp_async16(&sR[col * kGLd + a], V.a + off + ix, 8 * valid);
          if (hasP) cp_async16(&sP[col * kGLd + a], V.b + off + ix, 8 * valid);
          cp_async16(&sW[col * kGLd + a], W + ix, 8 * valid);
        }
      } else {
        for (int idx = threadIdx.x; idx < kGRows * R4; idx += blockDim.x) {
          const int a = idx % kGRows, col = idx / kGRows;
          const bool ok = col < R && c0 + a < ze;
          const int64_t ix = ok ? c0 + a + n * col : 0;
          cp_async8(&sR[col * kGLd + a], V.a + off + ix, ok);
          if (hasP) cp_async8(&sP[col * kGLd + a], V.b + off + ix, ok);
          cp_async8(&sW[col * kGLd + a], W + ix, ok);
        }
      }
      cp_async_wait_all();
      __syncthreads();
#pragma unroll 2
      for (int ks = 0; ks < kGRows / 4; ++ks) {
        const int a = 4 * ks + q;
        double fa[MT], fb[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int o = (8 * (warp + 8 * i) + g) * kGLd + a;
          fa[i] = (warp + 8 * i < NT) ? dr[i] * (hasP ? fma(V.beta, sP[o], sR[o]) : sR[o]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) fb[j] = sW[(8 * j + g) * kGLd + a];
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (warp + 8 * i < NT) {
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma(acc[i][j], fa[i], fb[j]);
          }
      }
    }
    // partial (z, l): element (r = 8 mi + g, c = 8 j + 2q + e)
    double* Gz = A.G + ((int64_t)z * 3 + l) * R * R;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int r = 8 * (warp + 8 * i) + g;
      if (warp + 8 * i >= NT || r >= R) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          if (c < R) Gz[r + (int64_t)R * c] = acc[i][j][e];
        }
    }
  }
}

// ---- stage S: G_l = sum_z Gpart[z][l] (fixed order) and S_l = sum_{l' != l} Pi^(l,l') * G_l'. Four lanes
// share one entry: lane t of the group sums the splits z = t, t + 4, ... of the three modes, and the four
// partial sums are combined by a fixed butterfly.
__device__ void stage_s(const CgArgs& A) {
  const int64_t R = A.m.R, RR = R * R;
  const int Z = gram_splits(A.m);
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int sub = (int)(gt & 3);
  for (int64_t base = gt >> 2; base < ((RR + 7) / 8) * 8; base += nthr >> 2) {
    const int64_t qi = base;
    double gsum[3] = {0.0, 0.0, 0.0};
    if (qi < RR) {
      const double* gp = A.G + qi;
      int z = sub;
      for (; z + 12 < Z; z += 16) {   // four splits per step: 12 loads in flight, added in z order
        double v[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int l = 0; l < 3; ++l) v[u][l] = gp[((int64_t)(z + 4 * u) * 3 + l) * RR];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int l = 0; l < 3; ++l) gsum[l] += v[u][l];
      }
      for (; z < Z; z += 4)
#pragma unroll
        for (int l = 0; l < 3; ++l) gsum[l] += gp[((int64_t)z * 3 + l) * RR];
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      gsum[l] += __shfl_xor_sync(0xffffffffu, gsum[l], 1);
      gsum[l] += __shfl_xor_sync(0xffffffffu, gsum[l], 2);
    }
    if (sub == 0 && qi < RR) {
      const double p12 = A.pi[3 * RR + qi], p13 = A.pi[4 * RR + qi], p23 = A.pi[5 * RR + qi];
      A.S[qi] = p12 * gsum[1] + p13 * gsum[2];
      A.S[RR + qi] = p12 * gsum[0] + p23 * gsum[2];
      A.S[2 * RR + qi] = p13 * gsum[0] + p23 * gsum[1];
    }
  }
}

// ---- stage Y: for rows of mode l: y = D (V Pi^(l) + W S_l + lambda V) with V = D (r + beta p).
// items (l, YR-row chunk, column half h). The operands of the whole 2R contraction are staged once into
// shared memory with cp.async (8-byte LDGSTS, zero-fill for padding, all copies of a thread in flight at
// once): sXr/sXp/sW = rows of r, p, W (YR x R4), sM = [Pi^(l) ; S_l] columns of the half (2R4 x 8*NTH).
// Warp w: m-tile w % (YR/8), n-tiles w / (YR/8) + (8*8/YR) j. If write_p != nullptr the raw V values (the
// new CG direction) are written after a block barrier. Returns the block's partial sum of raw(V) . y.
template <int NT>
__host__ __device__ constexpr int apply_rows() { return NT > 13 ? 16 : 32; }

template <int NT>
__host__ __device__ constexpr size_t apply_smem_doubles(int R4) {
  return (size_t)3 * R4 * (apply_rows<NT>() + 8) + (size_t)(8 * ((NT + 1) / 2)) * (2 * R4 + 16);
}

template <int NT>
__device__ double stage_apply(const CgArgs& A, const VSrc& V, double* y, double* write_p, double* smem) {
  constexpr int YR = apply_rows<NT>();       // rows per item (32, or 16 for R > 104)
  constexpr int MT = YR / 8;                 // m-tiles per item
  constexpr int WG = 8 / MT;                 // warps sharing one m-tile
  constexpr int NTH = (NT + 1) / 2;          // n-tiles per column half
  constexpr int NTW = (NTH + WG - 1) / WG;   // n-tiles per warp
  const Modes& m = A.m;
  const int R = (int)m.R;
  const int64_t RR = (int64_t)R * R;
  const int R4 = 4 * ((R + 3) / 4);
  constexpr int LDX = YR + 8;                // [r][row] staging, 8 mod 16 doubles: conflict-free copies
                                             // (consecutive rows) and A fragments (lane (g,q) -> 8q + g)
  double* sXr = smem;                        // [R4][LDX]
  double* sXp = sXr + R4 * LDX;
  double* sW = sXp + R4 * LDX;
  // [Pi; S] columns of the half, transposed: sMT[c][k] (k < R4: Pi, R4 + k: S) with a pitch of 4 mod 16
  // doubles: contiguous (16-byte) copies of Pi's columns, conflict-free B fragments (lane (g,q) -> 4g + q)
  const int LDMT = 2 * R4 + ((4 - 2 * R4) % 16 + 16) % 16;
  double* sMT = sW + R4 * LDX;                // [8 NTH][LDMT]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int mt = warp % MT, tw = warp / MT;
  const int nh = NT > 1 ? 2 : 1;
  int items = 0, chunks[3];
  for (int l = 0; l < 3; ++l) {
    chunks[l] = (int)((m.n[l] + YR - 1) / YR) * nh;
    items += chunks[l];
  }
  const double bet = V.b ? V.beta : 0.0;
  double dsum = 0.0;
  int nit = 0;
  // contiguous item ranges per block, items ordered (mode, column half, row chunk): a block's consecutive
  // items share [Pi; S] columns, which are then staged once
  const int per = (items + (int)gridDim.x - 1) / (int)gridDim.x;
  const int it_end = min(items, ((int)blockIdx.x + 1) * per);
  int staged_l = -1, staged_h = -1;
  for (int item = (int)blockIdx.x * per; item < it_end; ++item, ++nit) {
    stamp(A, 40 + 4 * nit);
    int l = 0, c = item;
    while (c >= chunks[l]) {
      c -= chunks[l];
      ++l;
    }
    const int nck = chunks[l] / nh;
    const int h = c / nck;
    const int64_t a0 = (int64_t)(c % nck) * YR;
    const int64_t n = m.n[l];
    const int64_t off = m.off[l];
    const double* W = m.W[l];
    const double* P = A.pi + l * RR;
    const double* Sl = A.S + l * RR;
    const double* D = V.D ? V.D + l * R : nullptr;
    const int t0 = h * NTH;
    const int s_lo = 8 * t0;
    const double* va = V.a + off;
    const double* vb = V.b ? V.b + off : V.a + off;
    __syncthreads();   // previous item consumed the staging buffers
    // 16-byte copies of row pairs when every column start is 16-byte aligned (n and the offsets even)
    const bool pair16 = ((n | off | a0) & 1) == 0 && ((reinterpret_cast<uintptr_t>(V.a) | reinterpret_cast<uintptr_t>(W) |
                                                      reinterpret_cast<uintptr_t>(V.b ? V.b : V.a)) & 15) == 0;
    if (pair16) {
      for (int idx = threadIdx.x; idx < (YR / 2) * R4; idx += blockDim.x) {
        const int a = 2 * (idx % (YR / 2)), kk = idx / (YR / 2);
        int64_t rem = n - (a0 + a);
        rem = rem < 0 ? 0 : (rem > 2 ? 2 : rem);
        const int valid = kk < R ? (int)rem : 0;   // rows of the pair in range
        const int64_t ix = valid ? a0 + a + n * kk : 0;
        cp_async16(&sXr[kk * LDX + a], va + ix, 8 * valid);
        cp_async16(&sXp[kk * LDX + a], vb + ix, V.b != nullptr ? 8 * valid : 0);
        cp_async16(&sW[kk * LDX + a], W + ix, 8 * valid);
      }
    } else {
      for (int idx = threadIdx.x; idx < YR * R4; idx += blockDim.x) {
        const int a = idx % YR, kk = idx / YR;
        const bool ok = kk < R && a0 + a < n;
        const int64_t ix = ok ? a0 + a + n * kk : 0;
        cp_async8(&sXr[kk * LDX + a], va + ix, ok);
        cp_async8(&sXp[kk * LDX + a], vb + ix, ok && V.b != nullptr);
        cp_async8(&sW[kk * LDX + a], W + ix, ok);
      }
    }
    // [Pi; S] columns of the half (restaged only when the mode or half changes): 16-byte k-pairs when R is even
    const bool restage = l != staged_l || h != staged_h;
    staged_l = l;
    staged_h = h;
    if (restage) {
      const bool kpair = (R & 1) == 0 && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Sl)) & 15) == 0;
      if (kpair) {
        for (int idx = threadIdx.x; idx < (R4 / 2) * 8 * NTH; idx += blockDim.x) {
          const int kk = 2 * (idx % (R4 / 2)), cc = idx / (R4 / 2);
          const int valid = (s_lo + cc < R) ? (kk + 1 < R ? 16 : (kk < R ? 8 : 0)) : 0;
          const int64_t ix = valid ? kk + (int64_t)R * (s_lo + cc) : 0;
          cp_async16(&sMT[cc * LDMT + kk], P + ix, valid);
          cp_async16(&sMT[cc * LDMT + R4 + kk], Sl + ix, valid);
        }
      } else {
        for (int idx = threadIdx.x; idx < R4 * 8 * NTH; idx += blockDim.x) {
          const int kk = idx % R4, cc = idx / R4;
          const bool ok = kk < R && s_lo + cc < R;
          const int64_t ix = ok ? kk + (int64_t)R * (s_lo + cc) : 0;
          cp_async8(&sMT[cc * LDMT + kk], P + ix, ok);
          cp_async8(&sMT[cc * LDMT + R4 + kk], Sl + ix, ok);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
    stamp(A, 41 + 4 * nit);
    double acc[NTW][2] = {};
    const int row = 8 * mt + g;
    // V Pi^(l): A fragment = D_r (r + beta p)
#pragma unroll 4
    for (int ks = 0; ks < R4 / 4; ++ks) {
      const int r = 4 * ks + q;
      const double dr = D ? D[min(r, R - 1)] : 1.0;
      const double fa = dr * fma(bet, sXp[r * LDX + row], sXr[r * LDX + row]);
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        const int tl = tw + WG * j;
        if (tl < NTH && t0 + tl < NT) dmma(acc[j], fa, sMT[(8 * tl + g) * LDMT + r]);
      }
    }
    // W S_l
#pragma unroll 4
    for (int ks = 0; ks < R4 / 4; ++ks) {
      const int r = 4 * ks + q;
      const double fa = sW[r * LDX + row];
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        const int tl = tw + WG * j;
        if (tl < NTH && t0 + tl < NT) dmma(acc[j], fa, sMT[(8 * tl + g) * LDMT + R4 + r]);
      }
    }
    stamp(A, 42 + 4 * nit);
    // epilogue: row a = a0 + 8 mt + g, cols s = 8 (t0 + tl) + 2q + e
    const int64_t arow = a0 + row;
    const bool rok = arow < n;
    double pnew[NTW][2];
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int tl = tw + WG * j;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        pnew[j][e] = 0.0;
        const int sc = 8 * (t0 + tl) + 2 * q + e;
        if (tl < NTH && rok && sc < R) {
          const double pr = fma(bet, sXp[sc * LDX + row], sXr[sc * LDX + row]);
          const double ds = D ? D[sc] : 1.0;
          const double lam = A.damp ? A.lambda * A.damp[l * R + sc] : A.lambda;
          const double yv = ds * fma(lam, ds * pr, acc[j][e]);
          y[off + arow + n * sc] = yv;
          dsum = fma(pr, yv, dsum);
          pnew[j][e] = pr;
        }
      }
    }
    if (write_p) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        const int tl = tw + WG * j;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int sc = 8 * (t0 + tl) + 2 * q + e;
          if (tl < NTH && rok && sc < R) write_p[off + arow + n * sc] = pnew[j][e];
        }
      }
    }
  }
  return dsum;
}

__device__ __forceinline__ double block_reduce(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kCgThreads / 32; ++i) t += red[i];
  __syncthreads();
  return t;   // every thread gets the same value
}

// every block sums the per-block partials in the same fixed order
__device__ __forceinline__ double grid_total(const double* part, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x) v += part[i];
  return block_reduce(v, red);
}

template <int NT>
__global__ void __launch_bounds__(kCgThreads, 1) k_cg_persistent(CgArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double cg_smem[];
  double* red = cg_smem;
  const Modes& m = A.m;
  const int R = (int)m.R;
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  const int64_t tid_g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double* part0 = A.part;
  double* part1 = A.part + gridDim.x;

  if (A.mode == 1) {   // single matvec: y = (J^T J + lambda I) v
    VSrc V{A.v, nullptr, 0.0, nullptr};
    stage_gram<NT>(A, V, cg_smem);
    grid.sync();
    stage_s(A);
    grid.sync();
    stage_apply<NT>(A, V, A.x, nullptr, cg_smem);
    return;
  }

  // init: x = 0, r = D rhs, p = 0 (so p_new = r + 0 * p = r), rr = ||r||^2
  double s = 0.0;
  for (int64_t qi = tid_g; qi < n; qi += stride) {
    double d = 1.0;
    if (A.dscale) {
      const int l = mode_of(m, qi);
      d = A.dscale[l * R + (qi - m.off[l]) / m.n[l]];
    }
    const double v = A.rhs[qi] * d;
    A.x[qi] = 0.0;
    A.r[qi] = v;
    A.p[qi] = 0.0;
    s = fma(v, v, s);
  }
  s = block_reduce(s, red);
  if (threadIdx.x == 0) part1[blockIdx.x] = s;
  grid.sync();
  double rr = grid_total(part1, red);
  double beta = 0.0;
  int iters = 0, nonfinite = 0;
  // The apply stage writes the new direction into the other half of p: blocks that still stage rows of the
  // current direction (the other column half of the same rows) never see a partially updated vector.
  double* pc = A.p;
  double* pn = A.p + n;
  // reading R33: rhs = 0 is solved by x = 0 (the printed loop would compute alpha = 0 / 0)
  const int maxit = rr == 0.0 ? 0 : A.maxiter;
  for (int it = 1; it <= maxit; ++it) {
    VSrc V{A.r, pc, beta, A.dscale};
    const int sb = 8 * (it - 1);
    stamp(A, sb + 0);
    stage_gram<NT>(A, V, cg_smem);
    stamp(A, sb + 1);
    grid.sync();
    stamp(A, sb + 2);
    stage_s(A);
    grid.sync();
    stamp(A, sb + 3);
    // z = B p_new, pn <- p_new, partial <p_new, z>
    const double pz_part = stage_apply<NT>(A, V, A.z, pn, cg_smem);
    stamp(A, sb + 4);
    const double pzb = block_reduce(pz_part, red);
    if (threadIdx.x == 0) part0[blockIdx.x] = pzb;
    grid.sync();
    const double pz = grid_total(part0, red);
    const double alpha = rr / pz;
    if (!isfinite(alpha)) {
      nonfinite = it;
      break;
    }
    stamp(A, sb + 5);
    double s2 = 0.0;
    for (int64_t q0 = tid_g; q0 < n; q0 += 4 * stride) {
      double xp[4], xx[4], xz[4], xr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t qi = min(q0 + u * stride, n - 1);
        xp[u] = pn[qi];
        xx[u] = A.x[qi];
        xz[u] = A.z[qi];
        xr[u] = A.r[qi];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t qi = q0 + u * stride;
        if (qi < n) {
          A.x[qi] = fma(alpha, xp[u], xx[u]);
          const double rn = fma(-alpha, xz[u], xr[u]);
          A.r[qi] = rn;
          s2 = fma(rn, rn, s2);
        }
      }
    }
    s2 = block_reduce(s2, red);
    if (threadIdx.x == 0) part1[blockIdx.x] = s2;
    grid.sync();
    stamp(A, sb + 6);
    const double rr_new = grid_total(part1, red);
    beta = rr_new / rr;
    rr = rr_new;
    iters = it;
    double* const tswap = pc;
    pc = pn;
    pn = tswap;
    if (!isfinite(beta)) {
      nonfinite = it;
      break;
    }
    if (rr_new < A.tol) break;
  }
  // x in w-coordinates: x = D x_hat
  if (A.dscale) {
    for (int64_t qi = tid_g; qi < n; qi += stride) {
      const int l = mode_of(m, qi);
      A.x[qi] *= A.dscale[l * R + (qi - m.off[l]) / m.n[l]];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.st->rr = rr;
    A.st->iters = iters;
    A.st->nonfinite = nonfinite;
    A.st->done = 1;
  }
}

// ---- small systems: the whole CG (or one matvec) in ONE CTA with every vector in shared memory. For
// n = R (I + J + K) up to a few thousand the persistent grid kernel sits on a ~14 us per-iteration latency
// floor (its stages talk through global memory and grid barriers); here a stage is a block barrier. Same
// algorithm and formulas (Gram G_l = V_l^T W_l of V = D (r + beta p), S_l = sum Pi^(l,l') * G_l', Thm-Hv apply
// z = D (V Pi^(l) + W S_l + lambda V), the CG recurrences), plain FP64 FMAs in a fixed per-thread order.
constexpr int kCgSmallThreads = 1024;
__host__ __device__ constexpr size_t cg_small_smem_doubles(int64_t n, int64_t R) {
  return (size_t)6 * n + (size_t)12 * R * R + 64;
}

__device__ __forceinline__ double small_block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kCgSmallThreads, 1) k_cg_small(CgArgs A) {
  extern __shared__ __align__(16) double sm[];
  const Modes& m = A.m;
  const int R = (int)m.R;
  const int64_t RR = (int64_t)R * R;
  const int64_t n = m.R * (m.n[0] + m.n[1] + m.n[2]);
  const int tid = threadIdx.x, nt = blockDim.x;
  double* sx = sm;
  double* sr = sx + n;
  double* sp = sr + n;          // current direction (raw)
  double* sq = sp + n;          // new direction (raw) = r + beta p
  double* sz = sq + n;
  double* sW = sz + n;
  double* sPi = sW + n;         // 6 R^2
  double* sG = sPi + 6 * RR;    // 3 R^2
  double* sS = sG + 3 * RR;     // 3 R^2
  double* red = sS + 3 * RR;    // 64
  auto dsc = [&](int64_t qi) -> double {   // Jacobi scale of element qi (1 without)
    if (!A.dscale) return 1.0;
    const int l = mode_of(m, qi);
    return A.dscale[l * R + (qi - m.off[l]) / m.n[l]];
  };
  for (int64_t qi = tid; qi < n; qi += nt) {
    const int l = mode_of(m, qi);
    sW[qi] = m.W[l][qi - m.off[l]];
  }
  for (int64_t e = tid; e < 6 * RR; e += nt) sPi[e] = A.pi[e];
  // z = D (V Pi + W S + lambda V) for V = D * sq (sq raw); returns this thread's share of <sq, z>
  auto matvec = [&](bool scaled) -> double {
    // Gram G_l[r + R s] = sum_a V[a, r] W[a, s]
    for (int64_t e = tid; e < 3 * RR; e += nt) {
      const int l = (int)(e / RR);
      const int64_t rs = e % RR, r = rs % R, c = rs / R, nl = m.n[l], off = m.off[l];
      const double dr = (scaled && A.dscale) ? A.dscale[l * R + r] : 1.0;
      double acc = 0.0;
      for (int64_t a = 0; a < nl; ++a) acc = fma(sq[off + a + nl * r], sW[off + a + nl * c], acc);
      sG[e] = dr * acc;
    }
    __syncthreads();
    for (int64_t qi = tid; qi < RR; qi += nt) {
      const double p12 = sPi[3 * RR + qi], p13 = sPi[4 * RR + qi], p23 = sPi[5 * RR + qi];
      const double g0 = sG[qi], g1 = sG[RR + qi], g2 = sG[2 * RR + qi];
      sS[qi] = p12 * g1 + p13 * g2;
      sS[RR + qi] = p12 * g0 + p23 * g2;
      sS[2 * RR + qi] = p13 * g0 + p23 * g1;
    }
    __syncthreads();
    double dsum = 0.0;
    for (int64_t qi = tid; qi < n; qi += nt) {
      const int l = mode_of(m, qi);
      const int64_t nl = m.n[l], off = m.off[l], loc = qi - off, a = loc % nl, sc = loc / nl;
      const double* P = sPi + l * RR;
      const double* S = sS + l * RR;
      const double* D = (scaled && A.dscale) ? A.dscale + l * R : nullptr;
      double acc = 0.0;
      for (int r = 0; r < R; ++r) {
        const double vr = sq[off + a + nl * r] * (D ? D[r] : 1.0);
        acc = fma(vr, P[r + (int64_t)R * sc], acc);
      }
      for (int r = 0; r < R; ++r) acc = fma(sW[off + a + nl * r], S[r + (int64_t)R * sc], acc);
      const double pr = sq[qi];
      const double ds = D ? D[sc] : 1.0;
      const double lam = A.damp ? A.lambda * A.damp[l * R + sc] : A.lambda;
      const double yv = ds * fma(lam, ds * pr, acc);
      sz[qi] = yv;
      dsum = fma(pr, yv, dsum);
    }
    __syncthreads();
    return dsum;
  };
  if (A.mode == 1) {   // single matvec y = (J^T J + lambda I) v
    for (int64_t qi = tid; qi < n; qi += nt) sq[qi] = A.v[qi];
    __syncthreads();
    matvec(false);
    for (int64_t qi = tid; qi < n; qi += nt) A.x[qi] = sz[qi];
    return;
  }
  double s0 = 0.0;
  for (int64_t qi = tid; qi < n; qi += nt) {
    const double v = A.rhs[qi] * dsc(qi);
    sx[qi] = 0.0;
    sr[qi] = v;
    sp[qi] = 0.0;
    s0 = fma(v, v, s0);
  }
  double rr = small_block_sum(s0, red);
  double beta = 0.0;
  int iters = 0, nonfinite = 0;
  const int maxit = rr == 0.0 ? 0 : A.maxiter;   // reading R33
  for (int it = 1; it <= maxit; ++it) {
    for (int64_t qi = tid; qi < n; qi += nt) sq[qi] = fma(beta, sp[qi], sr[qi]);
    __syncthreads();
    const double pz = small_block_sum(matvec(true), red);
    const double alpha = rr / pz;
    if (!isfinite(alpha)) {
      nonfinite = it;
      break;
    }
    double s2 = 0.0;
    for (int64_t qi = tid; qi < n; qi += nt) {
      sx[qi] = fma(alpha, sq[qi], sx[qi]);
      const double rn = fma(-alpha, sz[qi], sr[qi]);
      sr[qi] = rn;
      sp[qi] = sq[qi];
      s2 = fma(rn, rn, s2);
    }
    const double rr_new = small_block_sum(s2, red);
    beta = rr_new / rr;
    rr = rr_new;
    iters = it;
    if (!isfinite(beta)) {
      nonfinite = it;
      break;
    }
    if (rr_new < A.tol) break;
  }
  for (int64_t qi = tid; qi < n; qi += nt) A.x[qi] = sx[qi] * dsc(qi);
  if (tid == 0) {
    A.st->rr = rr;
    A.st->iters = iters;
    A.st->nonfinite = nonfinite;
    A.st->done = 1;
  }
}

template <int NT>
static cudaError_t launch_persistent_nt(const CgArgs& a, int nsm, cudaStream_t st) {
  auto kern = k_cg_persistent<NT>;
  const int R4 = (int)(4 * ((a.m.R + 3) / 4));
  const size_t smem = 8 * std::max<size_t>(std::max<size_t>(1024, gram_smem_doubles(R4)), apply_smem_doubles<NT>(R4));
  cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ea != cudaSuccess) return ea;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCgThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  dim3 grid(nsm), block(kCgThreads);
  CgArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)kern, grid, block, params, smem, st);
}

cudaError_t launch_cg_persistent(const Modes& m, const double* pi, const double* dscale, const double* damp,
                                 double lambda, double tol,
                                 int maxiter, const double* rhs, const double* v, double* x, double* r, double* p,
                                 double* z, double* G, double* S, double* part, CgState* st_dev, int mode, int nsm,
                                 bool allow_small, cudaStream_t st) {
  CgArgs a;
  a.S = S;
  a.tstamp = cg_debug_tstamp();
  a.m = m;
  a.pi = pi;
  a.dscale = dscale;
  a.damp = damp;
  a.lambda = lambda;
  a.tol = tol;
  a.maxiter = maxiter;
  a.rhs = rhs;
  a.v = v;
  a.x = x;
  a.r = r;
  a.p = p;
  a.z = z;
  a.G = G;
  a.part = part;
  a.st = st_dev;
  a.mode = mode;
  const int64_t ntot = m.R * (m.n[0] + m.n[1] + m.n[2]);
  const size_t small_smem = 8 * cg_small_smem_doubles(ntot, m.R);
  if (allow_small && ntot <= 4096 && small_smem <= 200 * 1024 && !cg_debug_tstamp()) {   // one CTA, vectors in shared memory
    cudaError_t ea = cudaFuncSetAttribute(k_cg_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_smem);
    if (ea != cudaSuccess) return ea;
    k_cg_small<<<1, kCgSmallThreads, small_smem, st>>>(a);
    return cudaGetLastError();
  }
  // the row-owned kernel (k_cg_rows.cu) whenever every block's rows, vectors and operand ring fit in shared
  // memory; TF_CG_KERNEL=grid selects this kernel instead (development comparisons)
  const char* kenv = getenv("TF_CG_KERNEL");   // read per call: the parity tests switch it
  const bool force_grid = kenv && kenv[0] == 'g';
  if (!force_grid && cg_rows_fits(m, nsm, cg_gram_partial_doubles(m.R)))
    return launch_cg_rows(m, pi, dscale, damp, lambda, tol, maxiter, rhs, v, x, G, S, part, st_dev, mode, nsm, st);
  const int NT = (int)((m.R + 7) / 8);
  switch (NT) {
#define TF_CASE(k) \
  case k:          \
    return launch_persistent_nt<k>(a, nsm, st);
    TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
    TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

size_t cg_gram_partial_doubles(int64_t R) { return (size_t)kGramZ * 3 * R * R; }

// Development aid: if TF_CG_TSTAMP is set, block 0 of the persistent CG records %globaltimer at the stage
// boundaries of the first iterations into a device buffer, printed by tf_cg_debug_dump().
static unsigned long long* g_tstamp = nullptr;
unsigned long long* cg_debug_tstamp() {
  static bool init = false;
  if (!init) {
    init = true;
    if (getenv("TF_CG_TSTAMP")) cudaMalloc(&g_tstamp, 64 * sizeof(unsigned long long));
  }
  return g_tstamp;
}

}  // namespace tfk

extern "C" void tf_cg_debug_dump(void) {
  if (!tfk::g_tstamp) return;
  unsigned long long h[64];
  cudaDeviceSynchronize();
  cudaMemcpy(h, tfk::g_tstamp, sizeof(h), cudaMemcpyDeviceToHost);
  // slots 8 (it - 1) + 0..7; row-owned kernel: start, Gram done, barrier, S done, barrier, apply done,
  // <p,z> barrier, ||r||^2 barrier (the grid kernel's slots: start, gram, sync, S+sync, apply, sync+alpha, update)
  for (int it = 0; it < 3; ++it) {
    const unsigned long long* b = h + 8 * it;
    printf("iter %d:", it + 1);
    for (int k = 1; k < 8; ++k) printf(" %.2f", (b[k] - b[k - 1]) * 1e-3);
    printf(" us; next start %.2f\n", (b[8] - b[7]) * 1e-3);
  }
  if (h[59] > h[56] && h[56])
    printf("prologue: operands %.2f us, W -> tensor memory %.2f us, rhs + first barrier %.2f us; first iteration "
           "starts %.2f us after it\n", (h[57] - h[56]) * 1e-3, (h[58] - h[57]) * 1e-3, (h[59] - h[58]) * 1e-3,
           (h[0] - h[59]) * 1e-3);
}
