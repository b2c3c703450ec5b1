// Row-owned persistent CG (rows a8/a9: Thm Hv; Alg. CG-dGN).
//
// One cooperative launch runs the whole CG. Block b owns a contiguous range of <= 8*mtb rows of ONE mode l
// (blocks per mode in proportion to the mode sizes). For the whole solve it keeps the rows of W_l in tensor memory
// (tcgen05.st once, as the DMMA fragments of both contractions); in shared memory the rows of the search direction
// p ([column][row], pitch 8 mtb + 4 = 4 or 12 mod 16: conflict-free DMMA fragments in both contractions), the
// constant Pi~_l = D_l Pi^(l) D_l and, per iteration, S~_l ([column][k], pitch R8 + 4); every thread keeps its
// entries of r in registers (the positions of its output tiles of the apply) and its entries of x in tensor
// memory (in global memory when a thread owns two m-tiles). No other vector travels through global memory inside
// the loop: per iteration the global traffic is the Gram partial of each block (R^2 doubles) and the reduced S~.
// Four grid-wide steps per iteration:
//   G  p <- r + beta p (registers -> shared); Gram partial P_b = p_rows^T W_rows (DMMA, inner dim = rows),
//      stored transposed (16-byte stores of a lane's two adjacent columns)
//   S  G_l = D_l sum_b P_b (fixed order, one lane per mode and entry, the loads in flight while the first half
//      of p Pi~ runs) and S~_l = (sum_{l' != l} Pi^(l,l') * G_l') D_l                 (Thm Hv's S_l, scaled)
//   Y  z = p Pi~_l + W S~_l + lambda_c D_c^2 p: the Thm-Hv apply with the Jacobi scaling folded into the
//      operands (z = D (V Pi + W S + lambda V), V = p D); the second half of p Pi~ runs
//      from shared memory while all of S~_l is staged by cp.async; W's fragments come from tensor memory;
//      z stays in registers; partial <p, z>
//   U  alpha = ||r||^2 / <p, z>; r -= alpha z (registers); x += alpha p (tensor memory); partial ||r||^2 -> beta
// Scalars are recomputed by every block from the per-block partials in the same fixed order (deterministic,
// no host round trip). Mode 1 (single matvec y = (J^T J + lambda D) v) runs G, S and Y once.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "tf_internal.h"
#include "tf_device.cuh"

namespace cg = cooperative_groups;

namespace tfk {

unsigned long long* cg_debug_tstamp();

constexpr int kRThreads = 256;
constexpr int kRMaxMT = 6;        // m-tiles (8 rows) per block at most
constexpr int kSBatch = 32;       // Gram partials loaded at once per lane in stage S
constexpr int kRedSlots = 64;

struct RowsArgs {
  Modes m;
  const double* pi;       // 6 R^2 Hadamard chains [Pi1 | Pi2 | Pi3 | Pi12 | Pi13 | Pi23]
  const double* dscale;   // 3R or nullptr: Jacobi M^{-1/2} per (mode, r)
  const double* damp;     // 3R or nullptr: damping matrix D per (mode, r) (nullptr = I)
  double lambda, tol;
  int maxiter;
  const double* rhs;      // CG right-hand side (w-coordinates)
  const double* v;        // matvec input
  double* x;              // CG solution / matvec output
  double* G;              // nblk x R^2 Gram partials
  double* S;              // 3 R^2: S~_l
  double* part;           // 2 x nblk scalar partials
  unsigned int* bar;      // grid-barrier arrival counter (zeroed before the launch)
  CgState* st;
  int mode;               // 0 CG, 1 single matvec
  int bstart[4];          // first block of each mode; bstart[3] = number of blocks
  int mtb;                // row capacity per block = 8 mtb
  int xtmem;              // 1: x lives in tensor memory (the columns fit), else in global memory
  unsigned long long* tstamp;
};

__host__ __device__ constexpr int rows_ldr(int mtb) { return 8 * mtb + 4; }
__host__ __device__ constexpr int rows_ldpi(int NT) { return 8 * NT + 4; }
__host__ __device__ constexpr size_t rows_smem_doubles(int NT, int mtb) {
  // p rows [R8][LDR], Pi~ and S~ [R8][LDPI] (S~ doubles as the staging buffer of the W rows in the prologue),
  // D, lambda D^2, reduction scratch; W itself lives in tensor memory
  return (size_t)(8 * NT) * rows_ldr(mtb) + (size_t)(8 * NT) * rows_ldpi(NT) +
         (size_t)(8 * NT) * (rows_ldpi(NT) > rows_ldr(mtb) ? rows_ldpi(NT) : rows_ldr(mtb)) + (size_t)2 * (8 * NT) +
         kRedSlots;
}
// tensor-memory columns per lane quadrant: the Gram's B fragments W[4s+q][8j+g] (2 mtb k-steps x NT doubles) and the
// apply's A fragments W[8 mt + g][4s+q] (MG m-tiles x R8/4 k-steps), 2 columns per double
__host__ __device__ constexpr int rows_tmem_cols(int NT, int mtb, int MG) { return 2 * (2 * mtb * NT + MG * 2 * NT); }
// x in tensor memory as well: 2 MG NH doubles per thread, one region per column half
__host__ __device__ constexpr int rows_tmem_x_cols(int NT, int MG) { return 8 * MG * ((NT + 1) / 2); }

__device__ __forceinline__ void rstamp(const RowsArgs& A, int slot) {
  if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && slot < 48) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.tstamp[slot] = t;
  }
}

// Grid-wide barrier of the cooperative launch: every block's thread 0 adds one arrival with release semantics
// (after a block barrier, so the block's earlier writes are ordered before it) and spins with acquire loads until
// all blocks of this phase have arrived; the counter only grows (phase e waits for e * nblk arrivals).
__device__ __forceinline__ void rows_grid_sync(unsigned int* bar, unsigned int& phase, int nblk) {
  __syncthreads();
  ++phase;
  if (threadIdx.x == 0) {
    const unsigned int target = phase * (unsigned int)nblk;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// prologue stamps (slots 56..59: entry, operands staged, W parked in tensor memory, first barrier passed)
__device__ __forceinline__ void pstamp(const RowsArgs& A, int k) {
  if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.tstamp[56 + k] = t;
  }
}

__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa16(double* dst, const double* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
// a global load issued where it stands (volatile: not sunk to its first use, so that its latency overlaps the
// work placed between the load and the use)
__device__ __forceinline__ double ld_early(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// the same total in every block: warp 0 sums the per-block partials (fixed lane order + fixed butterfly)
__device__ __forceinline__ double rows_grid_total(const double* part, int nblk, double* red) {
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nblk; i += 32) v += part[i];
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double t = red[0];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double rows_block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[1 + (threadIdx.x >> 5)] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kRThreads / 32; ++i) t += red[1 + i];
  __syncthreads();
  return t;
}

// One k-step of the apply for a warp's tiles: m-tile wsub (and wsub + 4 when MGT = 2 and it exists) times the NJ
// column tiles J0 .. J0 + NJ - 1. A fragments from [k][row] rows (pitch ldr), B from [column][k] operands (pitch
// ldb). Every DMMA of the common path is unconditional (no per-instruction predicate, no warp re-convergence).
template <int NJ, int J0, int MGT, int NH>
__device__ __forceinline__ void apply_kstep(double (&acc)[MGT][NH][2], const double* arows, int ldr, const double* bops,
                                            int ldb, int ka, int kb, int wsub, int g, bool second) {
  double fa0 = arows[ka * ldr + 8 * wsub + g];
  double fb[NJ > 0 ? NJ : 1];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) fb[jj] = bops[(8 * (J0 + jj) + g) * ldb + kb];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) dmma(acc[0][jj], fa0, fb[jj]);
  if (MGT > 1 && second) {
    const double fa1 = arows[ka * ldr + 8 * (wsub + 4) + g];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) dmma(acc[MGT - 1][jj], fa1, fb[jj]);
  }
}

// The same with the A fragments given (tensor memory).
template <int NJ, int J0, int MGT, int NH>
__device__ __forceinline__ void apply_kstep_v(double (&acc)[MGT][NH][2], double fa0, double fa1, const double* bops,
                                              int ldb, int kb, int g, bool second) {
  double fb[NJ > 0 ? NJ : 1];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) fb[jj] = bops[(8 * (J0 + jj) + g) * ldb + kb];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) dmma(acc[0][jj], fa0, fb[jj]);
  if (MGT > 1 && second) {
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) dmma(acc[MGT - 1][jj], fa1, fb[jj]);
  }
}

// All of S~_l (R x R column-major) into sS[c][k] (pitch ldpi), zero for k, c >= R; cp.async, one commit group.
__device__ __forceinline__ void stage_S(const double* src, int R, int R8, int ldpi, double* sS, bool pair) {
  if (pair) {
    for (int idx = threadIdx.x; idx < R8 * (R8 / 2); idx += kRThreads) {
      const int c = idx / (R8 / 2), k = 2 * (idx % (R8 / 2));
      const int valid = c < R ? (k + 1 < R ? 16 : (k < R ? 8 : 0)) : 0;
      cpa16(sS + c * ldpi + k, valid ? src + k + (int64_t)R * c : src, valid);
    }
  } else {
    for (int idx = threadIdx.x; idx < R8 * R8; idx += kRThreads) {
      const int c = idx / R8, k = idx % R8;
      const bool ok = c < R && k < R;
      cpa8(sS + c * ldpi + k, ok ? src + k + (int64_t)R * c : src, ok);
    }
  }
  cpa_commit();
}

template <int NT, int MGT>
__global__ void __launch_bounds__(kRThreads, 1) k_cg_rows(RowsArgs A) {
  unsigned int bar_phase = 0;
  extern __shared__ __align__(16) double rsm[];
  constexpr int R8 = 8 * NT;
  constexpr int NH = (NT + 1) / 2;                       // apply n-tiles per warp (column half)
  constexpr int MG = MGT;                                // apply m-tiles per warp at most (s, s + 4)
  constexpr int GBASE = (NT / 4) * 4;                   // Gram i-tiles handled as full rows of tiles
  constexpr int GLO = ((NT - GBASE) * NT + 7) / 8;       // leftover Gram tiles per warp at most
  constexpr int LDPI = rows_ldpi(NT);
  const Modes& m = A.m;
  const int R = (int)m.R;
  const int64_t RR = (int64_t)R * R;
  const int nblk = A.bstart[3];
  const int LDR = rows_ldr(A.mtb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;

  // ---- this block's rows
  const int b = blockIdx.x;
  int l = 0;
  while (l < 2 && b >= A.bstart[l + 1]) ++l;
  const int bi = b - A.bstart[l], nbl = A.bstart[l + 1] - A.bstart[l];
  const int64_t nl = m.n[l], off = m.off[l];
  const int64_t a0 = nl * bi / nbl, a1 = nl * (bi + 1) / nbl;
  const int nr = (int)(a1 - a0);
  const int MTb = (nr + 7) / 8;
  const double* Dl = A.dscale ? A.dscale + l * R : nullptr;

  double* sP = rsm;
  double* sPi = sP + R8 * LDR;
  double* sS = sPi + R8 * LDPI;            // S~ [c][k]; in the prologue the staging buffer of the W rows
  double* sW = sS;
  double* sD = sS + R8 * max(LDPI, LDR);   // D_c (Jacobi scale of this mode; 1 without)
  double* sLD = sD + R8;                   // lambda_c D_c^2 (lambda_c = lambda damp_c)
  double* red = sLD + R8;
  __shared__ uint32_t tmem_base_s;

  // apply tiles of this warp: sub-partition s = warp % 4 owns m-tiles s and s + 4 (every SMSP the same share
  // of the critical 8-row tiles), the two warps of a sub-partition split the NT column tiles in halves (NH, NT - NH);
  // all bounds are warp-uniform. The thread owns the entries (row 8 mt + g, column 8 j + 2 q + e) of r, x and z.
  const int wsub = warp & 3, whalf = warp >> 2;
#define TF_TILES(BODY)                                       \
  _Pragma("unroll") for (int mi = 0; mi < MG; ++mi)          \
  _Pragma("unroll") for (int jj = 0; jj < NH; ++jj) {        \
    const int mt = wsub + 4 * mi, j = whalf * NH + jj;       \
    if (mt < MTb && j < NT) { BODY }                         \
  }

  // ---- prologue (every copy in flight at once): W rows, p = 0 (or v), Pi^(l), D; then Pi~ = D Pi^(l) D in place;
  // r = D rhs in registers, x = 0
  pstamp(A, 0);
  const double* Wl = m.W[l];
  for (int idx = threadIdx.x; idx < R8 * LDR; idx += kRThreads) {
    const int c = idx / LDR, a = idx % LDR;
    const bool ok = c < R && a < nr;
    const int64_t gi = ok ? a0 + a + nl * c : 0;
    cpa8(sW + idx, Wl + gi, ok);
    cpa8(sP + idx, (A.mode == 1 ? A.v : Wl) + (A.mode == 1 ? off : 0) + gi, ok && A.mode == 1);
  }
  {
    const double* P = A.pi + (int64_t)l * RR;
    for (int idx = threadIdx.x; idx < R8 * LDPI; idx += kRThreads) {
      const int c = idx / LDPI, k = idx % LDPI;
      const bool ok = c < R && k < R;
      cpa8(sPi + idx, P + (ok ? k + (int64_t)R * c : 0), ok);
    }
  }
  for (int c = threadIdx.x; c < R8; c += kRThreads) cpa8(sD + c, Dl ? Dl + min(c, R - 1) : Wl, Dl != nullptr && c < R);
  cpa_commit();
  cpa_wait<0>();
  __syncthreads();
  for (int c = threadIdx.x; c < R8; c += kRThreads) {
    if (!Dl) sD[c] = c < R ? 1.0 : 0.0;
    const double lam = c < R ? (A.damp ? A.lambda * A.damp[l * R + c] : A.lambda) : 0.0;
    sLD[c] = lam * sD[c] * sD[c];
  }
  if (Dl) {
    for (int idx = threadIdx.x; idx < R8 * LDPI; idx += kRThreads) {
      const int c = idx / LDPI, k = idx % LDPI;
      if (c < R8 && k < R8) sPi[idx] *= sD[k] * sD[c];
    }
  }
  // W in tensor memory (512 columns; a warp touches its lane quadrant warp % 4): per lane, the Gram's B fragments
  // W[4s + q][8j + g] at columns 2 (s NT + j) and, after them, the apply's A fragments W[8 (wsub + 4 mi) + g][4s + q]
  // at 2 (KG NT + mi R8/4 + s) — both are the same for the two warps of a quadrant, so warps 0-3 write them once
  pstamp(A, 1);
  const int KG = 2 * A.mtb;                // Gram k-steps at most (rows padded to 8 mtb)
  if (warp == 0) tmem_alloc(&tmem_base_s, 512);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t ta = tmem_base_s + ((uint32_t)(32 * wsub) << 16);
  const uint32_t taA = ta + 2 * KG * NT;
  // when the columns fit, this thread's entries of x (2 MG NH doubles) live in tensor memory too, after the A
  // fragments, one region per column half (the two warps of a quadrant own different entries)
  const bool kXT = A.xtmem != 0;
  const uint32_t taX = taA + 2 * MG * (R8 / 4) + whalf * 4 * MG * NH;
  if (warp < 4) {
#pragma unroll 1
    for (int s = 0; s < KG; ++s) {
#pragma unroll
      for (int j0 = 0; j0 < NT; j0 += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (j0 + u < NT) ? sW[(8 * (j0 + u) + g) * LDR + 4 * s + q] : 0.0;
        if (j0 + 4 <= NT) tmem_st4(ta + 2 * (s * NT + j0), v);
        else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u < NT) tmem_st1(ta + 2 * (s * NT + j0 + u), v[u]);
        }
      }
    }
#pragma unroll 1
    for (int mi = 0; mi < MG; ++mi) {
      const int mt = wsub + 4 * mi;
#pragma unroll 1
      for (int s = 0; s < R8 / 4; s += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = (mt < A.mtb && s + u < R8 / 4) ? sW[(4 * (s + u) + q) * LDR + 8 * mt + g] : 0.0;
        if (s + 4 <= R8 / 4) tmem_st4(taA + 2 * (mi * (R8 / 4) + s), v);
        else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (s + u < R8 / 4) tmem_st1(taA + 2 * (mi * (R8 / 4) + s + u), v[u]);
        }
      }
    }
    tmem_wait_st();
  }
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  pstamp(A, 2);
  double rreg[MG][NH][2];
  double s0 = 0.0;
#pragma unroll
  for (int mi = 0; mi < MG; ++mi)
#pragma unroll
    for (int jj = 0; jj < NH; ++jj) rreg[mi][jj][0] = rreg[mi][jj][1] = 0.0;
  if (A.mode == 0) {
    TF_TILES({
      const int row = 8 * mt + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * q + e;
        if (row < nr && c < R) {
          const double rv = A.rhs[off + a0 + row + nl * c] * sD[c];
          rreg[mi][jj][e] = rv;
          s0 = fma(rv, rv, s0);
        }
      }
    })
    // x = 0 (after the loads of rhs: no load waits behind a store)
    if (kXT) {
      double z0[2 * MG * NH];
#pragma unroll
      for (int i = 0; i < 2 * MG * NH; ++i) z0[i] = 0.0;
      tmem_st_doubles<2 * MG * NH>(taX, z0);
      tmem_wait_st();
    } else {
      TF_TILES({
        const int row = 8 * mt + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          if (row < nr && c < R) A.x[off + a0 + row + nl * c] = 0.0;
        }
      })
    }
  }
  double* part0 = A.part;
  double* part1 = A.part + nblk;
  double rr = 0.0;
  if (A.mode == 0) {
    s0 = rows_block_sum(s0, red);
    if (threadIdx.x == 0) part1[b] = s0;
    rows_grid_sync(A.bar, bar_phase, nblk);
    rr = rows_grid_total(part1, nblk, red);
    pstamp(A, 3);
  } else {
    __syncthreads();
  }

  const double* Sl = A.S + (int64_t)l * RR;
  const bool pairS = (R & 1) == 0 && (reinterpret_cast<uintptr_t>(Sl) & 15) == 0;
  double beta = 0.0;
  int iters = 0, nonfinite = 0;
  const int maxit = A.mode == 1 ? 1 : (rr == 0.0 ? 0 : A.maxiter);   // reading R33
  double acc[MG][NH][2];

  for (int it = 1; it <= maxit; ++it) {
    const int sb = 8 * (it - 1);
    rstamp(A, sb + 0);
    // ---- G: p <- r + beta p at this thread's positions; Gram partial of the raw p rows
    if (A.mode == 0) {
      TF_TILES({
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int o = (8 * j + 2 * q + e) * LDR + 8 * mt + g;
          sP[o] = fma(beta, sP[o], rreg[mi][jj][e]);
        }
      })
      __syncthreads();
    }
    {
      // warp w: i-tiles w and w + 8 of the GBASE full rows of tiles, one row of NT tiles at a time (B fragments
      // reloaded per row: 1.08 shared loads per DMMA), then its share of the leftover tiles (i >= GBASE)
      const int ks = (nr + 3) / 4;
      double* Gp = A.G + (int64_t)b * RR;
#pragma unroll 1
      for (int ii = 0; ii < 2; ++ii) {
        const int i = warp + 8 * ii;
        if (i >= GBASE) break;
        double gf[NT][2];
#pragma unroll
        for (int j = 0; j < NT; ++j) gf[j][0] = gf[j][1] = 0.0;
        for (int s = 0; s < ks; ++s) {
          const int a = 4 * s + q;
          const double fa = sP[(8 * i + g) * LDR + a];
          double fb[NT];
          tmem_ld_doubles<NT>(ta + 2 * s * NT, fb);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(gf[j], fa, fb[j]);
        }
        // the partial is stored transposed (entry (r, c) at c + R r): a lane's two columns are adjacent
        const int r = 8 * i + g;
        if (r < R) {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int c = 8 * j + 2 * q;
            double* dst = Gp + c + (int64_t)R * r;
            if (c + 1 < R && (R & 1) == 0) *reinterpret_cast<double2*>(dst) = make_double2(gf[j][0], gf[j][1]);
            else {
              if (c < R) dst[0] = gf[j][0];
              if (c + 1 < R) dst[1] = gf[j][1];
            }
          }
        }
      }
      // leftover tiles (i >= GBASE): tile warp + 8u; the bound is warp-uniform, so it is a branch around an
      // unpredicated k-loop
#pragma unroll 1
      for (int u = 0; u < GLO; ++u) {
        const int t = warp + 8 * u;
        if (t >= (NT - GBASE) * NT) break;
        const int i = GBASE + t / NT, j = t % NT;
        double gl[2] = {0.0, 0.0};
        for (int s = 0; s < ks; ++s) {
          double fb;
          tmem_ld_d1(ta + 2 * (s * NT + j), &fb);
          tmem_wait_ld();
          dmma(gl, sP[(8 * i + g) * LDR + 4 * s + q], fb);
        }
        const int r = 8 * i + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          if (r < R && c < R) Gp[c + (int64_t)R * r] = gl[e];
        }
      }
    }
    // p Pi~ does not depend on S: a third of it runs while this block's partial stores drain (before the grid
    // barrier), a third while stage S's loads are in flight and the rest while S~ is staged
#pragma unroll
    for (int mi = 0; mi < MG; ++mi)
#pragma unroll
      for (int jj = 0; jj < NH; ++jj) acc[mi][jj][0] = acc[mi][jj][1] = 0.0;
    const bool second = MG > 1 && wsub + 4 < MTb;
    auto pi_steps = [&](int s0, int s1) {
#pragma unroll 4
      for (int s = s0; s < s1; ++s) {
        if (whalf == 0) apply_kstep<NH, 0, MG, NH>(acc, sP, LDR, sPi, LDPI, 4 * s + q, 4 * s + q, wsub, g, second);
        else apply_kstep<NT - NH, NH, MG, NH>(acc, sP, LDR, sPi, LDPI, 4 * s + q, 4 * s + q, wsub, g, second);
      }
    };
    constexpr int KS0 = (R8 / 4) / 3, KS1 = 2 * (R8 / 4) / 3;
    pi_steps(0, KS0);
    rstamp(A, sb + 1);
    rows_grid_sync(A.bar, bar_phase, nblk);
    rstamp(A, sb + 2);
    // ---- S: one lane per (entry, mode) issues the loads of that mode's partials (block order, all in flight),
    // the DMMAs of p Pi~ run while they are in flight, then the lane sums them in block order; the three lanes
    // of an entry exchange their sums and each writes its mode's S~
    {
      const int gw = blockIdx.x * (kRThreads / 32) + warp, nw = nblk * (kRThreads / 32);
      const int ll = lane % 3;
      bool first = true;
      for (int64_t eb = (int64_t)gw * 10; first || eb < RR; eb += (int64_t)nw * 10) {
        const int64_t e = eb + lane / 3;
        const bool act = lane < 30 && e < RR;
        const int be = A.bstart[ll + 1];
        const double* gp = A.G + (act ? e : 0);
        int bb = A.bstart[ll];
        double v[kSBatch];
#pragma unroll
        for (int u = 0; u < kSBatch; ++u) {
          const bool ok = act && bb + u < be;
          v[u] = ok ? gp[(int64_t)(bb + u) * RR] : 0.0;
        }
        const int r = act ? (int)(e / R) : 0, c = act ? (int)(e % R) : 0;   // partials are stored transposed
        const double* D = A.dscale;
        double d0 = 1.0, d1 = 1.0, d2 = 1.0, dc = 1.0, p12 = 0.0, p13 = 0.0, p23 = 0.0;
        if (act) {
          if (D) {
            d0 = D[r];
            d1 = D[R + r];
            d2 = D[2 * R + r];
            dc = D[ll * R + c];
          }
          const int64_t rc = r + (int64_t)R * c;
          p12 = A.pi[3 * RR + rc];
          p13 = A.pi[4 * RR + rc];
          p23 = A.pi[5 * RR + rc];
        }
        if (first) pi_steps(KS0, KS1);   // the loads above are in flight meanwhile
        first = false;
        double gsum = 0.0;
#pragma unroll
        for (int u = 0; u < kSBatch; ++u) gsum += v[u];
        for (bb += kSBatch; bb < be; bb += kSBatch) {   // modes with more than kSBatch blocks
#pragma unroll
          for (int u = 0; u < kSBatch; ++u) v[u] = (act && bb + u < be) ? gp[(int64_t)(bb + u) * RR] : 0.0;
#pragma unroll
          for (int u = 0; u < kSBatch; ++u) gsum += v[u];
        }
        const int base = 3 * (lane / 3);
        const double x0 = __shfl_sync(0xffffffffu, gsum, min(base, 31));
        const double x1 = __shfl_sync(0xffffffffu, gsum, min(base + 1, 31));
        const double x2 = __shfl_sync(0xffffffffu, gsum, min(base + 2, 31));
        if (act) {
          const double g0 = x0 * d0, g1 = x1 * d1, g2 = x2 * d2;
          double sv;
          if (ll == 0) sv = p12 * g1 + p13 * g2;
          else if (ll == 1) sv = p12 * g0 + p23 * g2;
          else sv = p13 * g0 + p23 * g1;
          A.S[(int64_t)ll * RR + r + (int64_t)R * c] = sv * dc;
        }
      }
    }
    rstamp(A, sb + 3);
    rows_grid_sync(A.bar, bar_phase, nblk);
    rstamp(A, sb + 4);
    // ---- Y: all of S~_l is staged while the second half of p Pi~ runs, then W S~ with W from tensor memory
    stage_S(Sl, R, R8, LDPI, sS, pairS);
    pi_steps(KS1, R8 / 4);
    cpa_wait<0>();
    __syncthreads();
#pragma unroll 1
    for (int hk = 0; hk < 2; ++hk) {   // the R8/4 = 2 NT k-steps in two batches of NT A fragments
      double wa[MG][NT];
      tmem_ld_doubles<NT>(taA + 2 * hk * NT, wa[0]);
      if (MG > 1 && second) tmem_ld_doubles<NT>(taA + 2 * (R8 / 4 + hk * NT), wa[MG - 1]);
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < NT; ++u) {
        const int kb = 4 * (hk * NT + u) + q;
        const double fa1 = MG > 1 ? wa[MG - 1][u] : 0.0;
        if (whalf == 0) apply_kstep_v<NH, 0, MG, NH>(acc, wa[0][u], fa1, sS, LDPI, kb, g, second);
        else apply_kstep_v<NT - NH, NH, MG, NH>(acc, wa[0][u], fa1, sS, LDPI, kb, g, second);
      }
    }
    rstamp(A, sb + 5);
    // epilogue: z (registers) and <p, z>; matvec mode writes y
    double pz = 0.0;
    TF_TILES({
      const int row = 8 * mt + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * q + e;
        if (row < nr && c < R) {
          const double pv = sP[c * LDR + row];
          const double z = fma(sLD[c], pv, acc[mi][jj][e]);
          acc[mi][jj][e] = z;
          if (A.mode == 1) A.x[off + a0 + row + nl * c] = z;
          else pz = fma(pv, z, pz);
        }
      }
    })
    if (A.mode == 1) break;
    pz = rows_block_sum(pz, red);
    if (threadIdx.x == 0) part0[b] = pz;
    rows_grid_sync(A.bar, bar_phase, nblk);
    rstamp(A, sb + 6);
    const double alpha = rr / rows_grid_total(part0, nblk, red);
    if (!isfinite(alpha)) {
      nonfinite = it;
      break;
    }
    // ---- U: r -= alpha z, x += alpha p at this thread's positions; ||r||^2 (x: all loads first, then stores)
    double s2 = 0.0;
    if (kXT) {   // x in tensor memory: load, update, store back
      double xt[2 * MG * NH];
      tmem_ld_doubles<2 * MG * NH>(taX, xt);
      tmem_wait_ld();
      TF_TILES({
        const int row = 8 * mt + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          if (row < nr && c < R) {
            xt[2 * (mi * NH + jj) + e] = fma(alpha, sP[c * LDR + row], xt[2 * (mi * NH + jj) + e]);
            const double rn = fma(-alpha, acc[mi][jj][e], rreg[mi][jj][e]);
            rreg[mi][jj][e] = rn;
            s2 = fma(rn, rn, s2);
          }
        }
      })
      tmem_st_doubles<2 * MG * NH>(taX, xt);
      tmem_wait_st();
    } else {
      double xv[MG][NH][2];
      TF_TILES({
        const int row = 8 * mt + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          xv[mi][jj][e] = (row < nr && c < R) ? A.x[off + a0 + row + nl * c] : 0.0;
        }
      })
      TF_TILES({
        const int row = 8 * mt + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * q + e;
          if (row < nr && c < R) {
            A.x[off + a0 + row + nl * c] = fma(alpha, sP[c * LDR + row], xv[mi][jj][e]);
            const double rn = fma(-alpha, acc[mi][jj][e], rreg[mi][jj][e]);
            rreg[mi][jj][e] = rn;
            s2 = fma(rn, rn, s2);
          }
        }
      })
    }
    s2 = rows_block_sum(s2, red);
    if (threadIdx.x == 0) part1[b] = s2;
    rows_grid_sync(A.bar, bar_phase, nblk);
    rstamp(A, sb + 7);
    const double rr_new = rows_grid_total(part1, nblk, red);
    beta = rr_new / rr;
    rr = rr_new;
    iters = it;
    if (!isfinite(beta)) {
      nonfinite = it;
      break;
    }
    if (rr_new < A.tol) break;
  }
  cpa_wait<0>();
  if (kXT && A.mode == 0) {   // x in w-coordinates: x = D x_hat, from tensor memory
    double xt[2 * MG * NH];
    tmem_ld_doubles<2 * MG * NH>(taX, xt);
    tmem_wait_ld();
    TF_TILES({
      const int row = 8 * mt + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * q + e;
        if (row < nr && c < R) A.x[off + a0 + row + nl * c] = xt[2 * (mi * NH + jj) + e] * sD[c];
      }
    })
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base_s, 512);
  if (A.mode == 1) return;
  // x in w-coordinates: x = D x_hat
  if (!kXT && Dl) {
    TF_TILES({
      const int row = 8 * mt + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * q + e;
        if (row < nr && c < R) A.x[off + a0 + row + nl * c] *= sD[c];
      }
    })
  }
#undef TF_TILES
  if (b == 0 && threadIdx.x == 0) {
    A.st->rr = rr;
    A.st->iters = iters;
    A.st->nonfinite = nonfinite;
    A.st->done = 1;
  }
}

// Blocks per mode: start from one each and give every further block to the mode with the most rows per block;
// returns the m-tile capacity needed (0 if a mode has no rows).
static int rows_plan(const Modes& m, int grid, int bstart[4]) {
  int nb[3] = {1, 1, 1};
  for (int l = 0; l < 3; ++l)
    if (m.n[l] < 1) return 0;
  // add blocks only while some block owns more than 24 rows (measured: c2/c3 run 13/15 us per iteration instead
  // of 17 us on the full grid, c4/c5 are unchanged): fewer blocks mean fewer Gram partials to reduce in stage S
  static const int target = [] {
    const char* e = getenv("TF_CG_ROWS_TARGET");
    return e ? atoi(e) : 24;
  }();
  for (int k = 3; k < grid; ++k) {
    int best = -1;
    int64_t most = 0;
    for (int l = 0; l < 3; ++l) {
      if (nb[l] >= m.n[l]) continue;
      const int64_t rows = (m.n[l] + nb[l] - 1) / nb[l];
      if (rows > most && rows > target) {
        most = rows;
        best = l;
      }
    }
    if (best < 0) break;
    nb[best] += 1;
  }
  bstart[0] = 0;
  int64_t rmax = 0;
  for (int l = 0; l < 3; ++l) {
    bstart[l + 1] = bstart[l] + nb[l];
    rmax = std::max<int64_t>(rmax, (m.n[l] + nb[l] - 1) / nb[l]);
  }
  // capacity of at least 4 m-tiles: sub-partition s always computes m-tile s (zero rows when beyond the block)
  return std::max(4, (int)((rmax + 7) / 8));
}

template <int NT>
static cudaError_t launch_rows_nt(RowsArgs& a, cudaStream_t st) {
  auto kern = a.mtb > 4 ? k_cg_rows<NT, 2> : k_cg_rows<NT, 1>;
  // at least 120 KB of shared memory: one block per SM, since every block allocates all 512 tensor-memory columns
  // (a second block on the SM would wait in tcgen05.alloc while the first waits for it at a grid barrier)
  const size_t smem = std::max<size_t>(8 * rows_smem_doubles(NT, a.mtb), 120 * 1024);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  void* params[] = {&a};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(a.bstart[3]), dim3(kRThreads), params, smem, st);
}

// Plans the row-owned kernel for these modes on `grid` blocks; returns false (nothing launched) when a block
// would own more than 8 kRMaxMT rows, shared memory does not fit, or the scratch buffers are too small.
bool cg_rows_fits(const Modes& m, int grid, size_t gram_partial_doubles) {
  if (grid < 3) return false;   // one block per mode at least (a smaller cap goes to the grid kernel)
  int bs[4];
  const int mtb = rows_plan(m, grid, bs);
  const int NT = (int)((m.R + 7) / 8);
  if (mtb < 1 || mtb > kRMaxMT || NT > 16) return false;
  if (8 * rows_smem_doubles(NT, mtb) > 227 * 1024) return false;
  if (rows_tmem_cols(NT, mtb, mtb > 4 ? 2 : 1) > 512) return false;
  return (size_t)bs[3] * m.R * m.R <= gram_partial_doubles;
}

cudaError_t launch_cg_rows(const Modes& m, const double* pi, const double* dscale, const double* damp, double lambda,
                           double tol, int maxiter, const double* rhs, const double* v, double* x, double* G,
                           double* S, double* part, CgState* st_dev, int mode, int grid, cudaStream_t st) {
  RowsArgs a;
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
  a.S = S;
  a.part = part;
  // the last 16 doubles of the partial-sum workspace hold the grid-barrier counter
  a.bar = reinterpret_cast<unsigned int*>(part + 2 * (size_t)grid);
  cudaError_t ez = cudaMemsetAsync(a.bar, 0, 8, st);
  if (ez != cudaSuccess) return ez;
  a.st = st_dev;
  a.mode = mode;
  a.tstamp = cg_debug_tstamp();
  a.mtb = rows_plan(m, grid, a.bstart);
  {
    const int NTh = (int)((m.R + 7) / 8), MGh = a.mtb > 4 ? 2 : 1;
    a.xtmem = rows_tmem_cols(NTh, a.mtb, MGh) + rows_tmem_x_cols(NTh, MGh) <= 512 ? 1 : 0;
  }
  a.G = G;
  const int NT = (int)((m.R + 7) / 8);
  switch (NT) {
#define TF_CASE(k) \
  case k:          \
    return launch_rows_nt<k>(a, st);
    TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
    TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace tfk
