// Generic FP64 tensor-core GEMM for the compression stage (NEXT #3): the unfolding Grams
// T_(l) T_(l)^T (Remark MLSVD-SVD), the subspace-iteration products G·Q, the
// multilinear products of the core S = (U1^T, U2^T, U3^T)·T and the
// uncompression U·W.
//
//   C[m, n] (+)= alpha * sum_b sum_k  A_b[m, k] * B_b[n, k]      (+ beta * C)
//
// Each operand X is addressed in a [p, k] view: X[p, k] = ptr[k + ld*p] (k contiguous, "kc") or
// ptr[p + ld*k] (p contiguous), plus a batch stride. Batches are either summed into one C (the
// unfolding Gram of mode 2, Σ_k T_k^T T_k) or produce one C each.
//
// Kernel: BM x BN output tile per CTA (128x{128,112,96,64,32}, 64x128 or 64x64), 8 warps, warp tile
// 32 x (BN/WN) built from 8x8 DMMA fragments (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4); k-steps of
// BK = 32 staged through a 3-deep shared-memory ring by TMA (cp.async.bulk.tensor, complete_tx on an
// mbarrier; out-of-bounds boxes are zero-filled, which handles every ragged edge), or by 8-byte
// cp.async with zero-fill when an operand is not 16-byte aligned. Shared-memory pitches are ≡ 4
// (mod 16) doubles so that every fragment load is bank-conflict free (two wavefronts per warp).
// Split-K over the (batch, k-step) space writes per-split partial tiles that k_gemm_reduce sums in
// a fixed order (deterministic). `sym` computes only the tiles on and above the diagonal of a
// symmetric product (A == B) and mirrors them.
#include "tf_device.cuh"
#include "tf_internal.h"

namespace tfk {

namespace {

constexpr int GBK = 32;          // k-step
constexpr int GSTAGES = 3;
constexpr int GTHREADS = 256;

__host__ __device__ constexpr int op_tile_doubles(int BP, bool kc) {
  return kc ? BP * (GBK + 4) : GBK * (BP + 4);
}

template <int BM, int BN>
struct GemmCfg {
  static constexpr int WM = BM / 32;        // warps along m
  static constexpr int WN = 8 / WM;         // warps along n
  static constexpr int WTN = BN / WN;       // warp tile width
  static constexpr int FM = 4;              // 8-row fragments per warp (32 rows)
  static constexpr int FN = WTN / 8;        // 8-col fragments per warp
  static_assert(WM * WN == 8 && FN >= 1, "bad tile");
};

__device__ __forceinline__ void cp_async8z(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// fragment element X[p][k] of a staged tile
template <int BP, bool KC>
__device__ __forceinline__ double frag(const double* s, int p, int k) {
  return KC ? s[p * (GBK + 4) + k] : s[k * (BP + 4) + p];
}

// cp.async fallback: stage X[p0 .. p0+BP) x [k0 .. k0+GBK) of batch b
template <int BP, bool KC>
__device__ __forceinline__ void stage_generic(double* s, const GemmOperand& X, int64_t np, int64_t nk, int64_t p0,
                                              int64_t k0, int64_t b) {
  const double* base = X.ptr + (X.bstride ? b * X.bstride : 0);
  for (int e = threadIdx.x; e < BP * GBK; e += GTHREADS) {
    int pp, kk;
    if (KC) {
      pp = e / GBK;
      kk = e % GBK;
    } else {
      kk = e / BP;
      pp = e % BP;
    }
    const int64_t p = p0 + pp, k = k0 + kk;
    const bool ok = p < np && k < nk;
    const double* src = ok ? (KC ? base + k + X.ld * p : base + p + X.ld * k) : X.ptr;
    cp_async8z(KC ? &s[pp * (GBK + 4) + kk] : &s[kk * (BP + 4) + pp], src, ok);
  }
}

template <int BP, bool KC>
__device__ __forceinline__ void stage_tma(double* s, const CUtensorMap* map, int64_t p0, int64_t k0, int64_t b,
                                          uint64_t* bar) {
  if (KC)
    tma_load_3d(s, map, (int)k0, (int)p0, (int)b, bar);
  else
    tma_load_3d(s, map, (int)p0, (int)k0, (int)b, bar);
}

}  // namespace

template <int BM, int BN, bool AKC, bool BKC, bool TMA>
__global__ void __launch_bounds__(GTHREADS, 1)
    k_gemm_dmma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, GemmArgs g) {
  using Cf = GemmCfg<BM, BN>;
  constexpr int SA = op_tile_doubles(BM, AKC), SB = op_tile_doubles(BN, BKC);
  extern __shared__ __align__(128) double gsm[];
  double* sA = gsm;
  double* sB = gsm + GSTAGES * SA;
  __shared__ __align__(8) uint64_t full[GSTAGES];

  // ---- decode the work item: (tile, output batch, split)
  int64_t item = blockIdx.x;
  const int split = (int)(item % g.ksplit);
  item /= g.ksplit;
  const int64_t ob = item % g.out_batches;   // output batch (0 when batches are summed)
  const int64_t tile = item / g.out_batches;
  int64_t tm, tn;
  if (g.sym) {   // upper-triangular tile enumeration: row tm holds tiles tn = tm .. ntn-1
    int64_t t = tile;
    tm = 0;
    while (t >= g.ntn - tm) {
      t -= g.ntn - tm;
      ++tm;
    }
    tn = tm + t;
  } else {
    tm = tile % g.ntm;
    tn = tile / g.ntm;
  }
  const int64_t m0 = tm * BM, n0 = tn * BN;

  // k-step range of this split over the (batch, k-step) space
  const int64_t nks = (g.Kd + GBK - 1) / GBK;
  const int64_t kb = g.sum_batch ? g.batch : 1;
  const int64_t total = kb * nks;
  const int64_t s_beg = (int64_t)split * g.steps_per_split;
  const int64_t s_end = s_beg + g.steps_per_split < total ? s_beg + g.steps_per_split : total;
  const int64_t nsteps = s_end > s_beg ? s_end - s_beg : 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, qq = lane & 3;
  const int wm = warp % Cf::WM, wn = warp / Cf::WM;

  if (TMA && threadIdx.x == 0) {
    prefetch_tmap(&mapA);
    prefetch_tmap(&mapB);
    for (int s = 0; s < GSTAGES; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto issue = [&](int64_t step, int slot) {
    const int64_t st = s_beg + step;
    const int64_t b = g.sum_batch ? st / nks : ob;
    const int64_t k0 = (st % nks) * GBK;
    if (TMA) {
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();   // generic reads of this slot (previous round) before the async write
        mbar_arrive_expect_tx(&full[slot], (uint32_t)((SA + SB) * 8));
        stage_tma<BM, AKC>(sA + slot * SA, &mapA, m0, k0, g.a.bstride ? b : 0, &full[slot]);
        stage_tma<BN, BKC>(sB + slot * SB, &mapB, n0, k0, g.b.bstride ? b : 0, &full[slot]);
      }
    } else {
      stage_generic<BM, AKC>(sA + slot * SA, g.a, g.M, g.Kd, m0, k0, b);
      stage_generic<BN, BKC>(sB + slot * SB, g.b, g.N, g.Kd, n0, k0, b);
      cp_async_commit();
    }
  };

  double acc[Cf::FM][Cf::FN][2];
#pragma unroll
  for (int i = 0; i < Cf::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cf::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nsteps) issue(s, s);
    else if (!TMA) cp_async_commit();
  }

  const int am = wm * 32 + gq;
  const int bn = wn * Cf::WTN + gq;
  for (int64_t step = 0; step < nsteps; ++step) {
    const int slot = (int)(step % GSTAGES);
    // keep GSTAGES-1 loads in flight: issue step + GSTAGES - 1 into the slot freed last iteration
    if (step + GSTAGES - 1 < nsteps) issue(step + GSTAGES - 1, (int)((step + GSTAGES - 1) % GSTAGES));
    else if (!TMA) cp_async_commit();
    if (TMA) {
      mbar_wait(&full[slot], (uint32_t)((step / GSTAGES) & 1));
    } else {
      cp_async_wait<GSTAGES - 1>();
      __syncthreads();
    }
    const double* a = sA + slot * SA;
    const double* b = sB + slot * SB;
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[Cf::FM], fb[Cf::FN];
#pragma unroll
      for (int i = 0; i < Cf::FM; ++i) fa[i] = frag<BM, AKC>(a, am + 8 * i, kk + qq);
#pragma unroll
      for (int j = 0; j < Cf::FN; ++j) fb[j] = frag<BN, BKC>(b, bn + 8 * j, kk + qq);
#pragma unroll
      for (int i = 0; i < Cf::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cf::FN; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    __syncthreads();   // every warp is done with `slot` before it is refilled
  }

  // ---- epilogue
  if (g.ksplit == 1) {
    double* C = g.C + ob * g.cstride;
#pragma unroll
    for (int i = 0; i < Cf::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cf::FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t m = m0 + am + 8 * i;
          const int64_t n = n0 + wn * Cf::WTN + 8 * j + 2 * qq + e;
          if (m < g.M && n < g.N) {
            double v = g.alpha * acc[i][j][e];
            if (g.beta != 0.0) v += g.beta * C[m + g.ldc * n];
            C[m + g.ldc * n] = v;
            if (g.sym && tm != tn) C[n + g.ldc * m] = v;
          }
        }
  } else {
    // partial tile in fragment order: part[((item * ksplit) + split) * BM*BN + ...]
    double* P = g.part + (((int64_t)item * g.ksplit) + split) * (int64_t)(BM * BN);
#pragma unroll
    for (int i = 0; i < Cf::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cf::FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = am + 8 * i;
          const int c = wn * Cf::WTN + 8 * j + 2 * qq + e;
          P[r + BM * c] = acc[i][j][e];
        }
  }
}

// Fixed-order sum of the split partials: one thread per output element of a tile item.
template <int BM, int BN>
__global__ void k_gemm_reduce(GemmArgs g) {
  const int64_t item = blockIdx.y;   // (tile, out batch)
  const int64_t ob = item % g.out_batches;
  const int64_t tile = item / g.out_batches;
  int64_t tm, tn;
  if (g.sym) {
    int64_t t = tile;
    tm = 0;
    while (t >= g.ntn - tm) {
      t -= g.ntn - tm;
      ++tm;
    }
    tn = tm + t;
  } else {
    tm = tile % g.ntm;
    tn = tile / g.ntm;
  }
  double* C = g.C + ob * g.cstride;
  const double* P = g.part + item * g.ksplit * (int64_t)(BM * BN);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < BM * BN; e += gridDim.x * blockDim.x) {
    const int r = e % BM, c = e / BM;
    const int64_t m = tm * BM + r, n = tn * BN + c;
    if (m >= g.M || n >= g.N) continue;
    double s = 0.0;
    for (int sp = 0; sp < g.ksplit; ++sp) s += P[(int64_t)sp * BM * BN + e];
    double v = g.alpha * s;
    if (g.beta != 0.0) v += g.beta * C[m + g.ldc * n];
    C[m + g.ldc * n] = v;
    if (g.sym && tm != tn) C[n + g.ldc * m] = v;
  }
}

size_t gemm_smem_bytes(int BM, int BN, bool akc, bool bkc) {
  return (size_t)GSTAGES * (op_tile_doubles(BM, akc) + op_tile_doubles(BN, bkc)) * 8;
}

template <int BM, int BN, bool AKC, bool BKC, bool TMA>
static cudaError_t launch_t(const CUtensorMap* ma, const CUtensorMap* mb, const GemmArgs& g, int64_t items,
                            cudaStream_t st) {
  auto kern = k_gemm_dmma<BM, BN, AKC, BKC, TMA>;
  const size_t smem = gemm_smem_bytes(BM, BN, AKC, BKC);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(items * g.ksplit), GTHREADS, smem, st>>>(*ma, *mb, g);
  e = cudaGetLastError();
  if (e != cudaSuccess || g.ksplit == 1) return e;
  dim3 rg(BM * BN / 256 > 16 ? 16 : BM * BN / 256, (unsigned)items);
  k_gemm_reduce<BM, BN><<<rg, 256, 0, st>>>(g);
  return cudaGetLastError();
}

template <int BM, int BN, bool TMA>
static cudaError_t launch_kc(const CUtensorMap* ma, const CUtensorMap* mb, const GemmArgs& g, int64_t items,
                             cudaStream_t st) {
  if (g.a.kc) {
    if (g.b.kc) return launch_t<BM, BN, true, true, TMA>(ma, mb, g, items, st);
    return launch_t<BM, BN, true, false, TMA>(ma, mb, g, items, st);
  }
  if (g.b.kc) return launch_t<BM, BN, false, true, TMA>(ma, mb, g, items, st);
  return launch_t<BM, BN, false, false, TMA>(ma, mb, g, items, st);
}

template <int BM, int BN>
static cudaError_t launch_tma(const CUtensorMap* ma, const CUtensorMap* mb, const GemmArgs& g, int64_t items,
                              bool tma, cudaStream_t st) {
  return tma ? launch_kc<BM, BN, true>(ma, mb, g, items, st) : launch_kc<BM, BN, false>(ma, mb, g, items, st);
}

cudaError_t launch_gemm(const CUtensorMap* ma, const CUtensorMap* mb, const GemmArgs& g, int64_t items, bool tma,
                        cudaStream_t st) {
  if (g.BM == 128 && g.BN == 128) return launch_tma<128, 128>(ma, mb, g, items, tma, st);
  if (g.BM == 128 && g.BN == 112) return launch_tma<128, 112>(ma, mb, g, items, tma, st);
  if (g.BM == 128 && g.BN == 96) return launch_tma<128, 96>(ma, mb, g, items, tma, st);
  if (g.BM == 128 && g.BN == 64) return launch_tma<128, 64>(ma, mb, g, items, tma, st);
  if (g.BM == 128 && g.BN == 32) return launch_tma<128, 32>(ma, mb, g, items, tma, st);
  if (g.BM == 64 && g.BN == 128) return launch_tma<64, 128>(ma, mb, g, items, tma, st);
  return launch_tma<64, 64>(ma, mb, g, items, tma, st);
}

}  // namespace tfk
