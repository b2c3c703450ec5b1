// Fused one-pass evaluation of F and grad F for the dGN hot path.
//
// For each frontal slice k (slice formula X_k = A diag(c_k) B^T) and each
// 64x64 tile (i-tile, j-tile) of it, one CTA does, with FP64 tensor-core MMA (DMMA.8x8x4):
//   phase 1  E   = T_k - A diag(c_k) B^T          residual, inner dim R
//            f  += sum E^2                         objective
//   phase 2  P   = E B                             (I-tile x R), inner dim 64 (j)
//            accA += P diag(c_k)                   -> dF/dA = -sum_k E_k B diag(c_k)
//            gCp[k] = sum_i A o P                  -> dF/dC[k,:] = -sum_ij E_ij A_i: B_j:
//   phase 3  accB^T += (A diag(c_k))^T E           -> dF/dB = -sum_k E_k^T A diag(c_k), inner dim 64 (i)
// i.e. grad F = J_f^T f (Lemma gradF; Lemma partialf 1855-1863) with all three
// MTTKRPs T_(l)(.W) (Kolda) fused on one read of T. T tiles are staged through
// shared memory by TMA (cp.async.bulk.tensor, double-buffered, mbarrier completion); E lives in
// registers (phase 1) and in the same shared buffer that held T_k (phases 2-3): never in HBM.
// A CTA owns one (i-tile, j-tile) and a contiguous range of slices; accA/accB stay in registers
// over the range and are written once as partials; k_eval_finalize reduces all partials in a
// fixed order (deterministic, bitwise reproducible).
#include <cstdio>

#include "tf_internal.h"
#include "tf_device.cuh"

namespace tfk {

#ifndef TF_P3_UNROLL
#define TF_P3_UNROLL 4
#endif
constexpr int kP3Unroll = TF_P3_UNROLL;   // Pi-form phase-3 k-loop unroll (development knob)
#ifndef TF_TMEM_A
#define TF_TMEM_A 1   // 1: phase-3 A fragments in tensor memory; 2: phase-2 B fragments instead; 0: neither
#endif
#ifndef TF_C_ASYNC
#define TF_C_ASYNC 1     // the c_k ring is filled by cp.async two slices ahead (no load latency on the slice path)
#endif
#ifndef TF_P2_SOUTER
#define TF_P2_SOUTER 1   // Pi-form phase 2 with the k-steps outer (NT independent accumulators per warp)
#endif
#ifndef TF_PI_PRE_MAXNT
#define TF_PI_PRE_MAXNT 0   // Pi pass: prescaled -A diag(c_k) rebuilt per slice up to this NT, else unscaled A in TMEM
#endif
#ifndef TF_P2_UNROLL
#define TF_P2_UNROLL 8   // Pi-form phase-2 k-step loop unroll from TF_P2_UNROLL_MINNT r-tiles on (else full)
#endif
#ifndef TF_P2_UNROLL_MINNT
// measured (tools/gpu_r02unr.sh): unroll 8 instead of 16 is 1.1% faster at NT = 13 (c5), 0.25% at NT = 15, 0.9%
// slower at NT = 9; c4's NT = 7 1.1% slower (a smaller body helps once the fully unrolled slice exceeds ~15 KB)
#define TF_P2_UNROLL_MINNT 13
#endif
#ifndef TF_P3_UNROLL_T
#define TF_P3_UNROLL_T 16   // Pi-form phase-3 (tensor-memory) k-step loop unroll (development knob; even)
#endif
template <int NT>
__host__ __device__ constexpr int p2_unroll() { return NT >= TF_P2_UNROLL_MINNT ? TF_P2_UNROLL : 16; }
template <int NT>
__host__ __device__ constexpr int p3_unroll() { return TF_P3_UNROLL_T; }
#ifndef TF_TMEM_PIPE
#define TF_TMEM_PIPE 1   // phase-3 tensor-memory loads one k-step ahead (c4 -1.7%, c5 -0.2%)
#endif

// Tile geometry: a CTA owns a BT x BT tile (BT = 64: 8 warps, 1 CTA/SM; BT = 32: 4 warps, 2 CTAs/SM).
template <int BT>
struct EvalTile {
  static constexpr int BI = BT, BJ = BT;
  static constexpr int LDE = BT + 4;             // smem leading dim of a T/E tile [j][i]; 4 mod 16 -> conflict-free
  static constexpr int NW = BT / 8;              // warps: one 8-row i-tile (phase 2) / 8-col j-tile (phase 3) each
  static constexpr int THREADS = NW * 32;
  static constexpr int WC = NW / 2;              // phase-1 warp grid 2 x WC
  static constexpr int MF = BT / 16;             // phase-1 m-fragments per warp (rows BT/2)
  static constexpr int NF = 2;                   // phase-1 n-fragments per warp (cols 16)
  static constexpr int TILE_BYTES = LDE * BJ * 8;   // one TMA box LDE x BJ doubles
};

template <int NT, int BT>
struct EvalSmem {
  using G = EvalTile<BT>;
  static constexpr int RP = 8 * NT;          // padded rank
  static constexpr int LDF = 8 * NT + 4;     // factor tile leading dim (4 mod 16 in doubles)
  static constexpr size_t off_te = 0;                                     // 2 x [BJ][LDE] doubles
  static constexpr size_t off_a = off_te + 2 * (size_t)G::TILE_BYTES;     // [BI][LDF]
  static constexpr size_t off_b = off_a + (size_t)G::BI * LDF * 8;        // [BJ][LDF]
  static constexpr size_t off_c = off_b + (size_t)G::BJ * LDF * 8;        // 4 x [RP]  (ring of c_k rows)
  // Per-warp dF/dC rows: lane quarter q of the butterfly holds t in [q NV/4, (q+1) NV/4) and stores at
  // 8t + g + q GCP, so each quarter's run starts 4 doubles further round the banks (conflict-free STS).
  static constexpr int NV = ((NT + 3) / 4) * 4;
  static constexpr int GCP = ((4 - 2 * NV) % 16 + 16) % 16;   // 2 NV + GCP = 4 mod 16
  static constexpr int GCS = RP + 3 * GCP;                     // row stride of the dF/dC partials
  static constexpr size_t off_gc = off_c + 4 * (size_t)RP * 8;            // 2 x [NW][GCS] (per-warp dF/dC partials)
  static constexpr size_t off_red = off_gc + 2 * G::NW * (size_t)GCS * 8; // [NW]
  // 12 mbarriers: full[2], p3done, aready; the decoupled Pi pass adds empty[2], gcf[2], gce[2], mid[2]
  static constexpr size_t off_bar = off_red + G::NW * 8;
  static constexpr size_t bytes = off_bar + 12 * 8;
  static_assert(bytes <= 232448, "exceeds the 227 KB per-CTA shared memory of sm_100a");
};

// Butterfly sum over the 4 lanes that share g = lane/4 (lane bits 0..1) of N values per lane;
// afterwards lane (g, q) holds N/4 sums: value j is index base(q) + j with
// base(q) = (q>>1&1)*N/2 + (q&1)*N/4. N must be a multiple of 4.
template <int N>
__device__ __forceinline__ void butterfly4(double (&v)[N], int q) {
  constexpr int H1 = N / 2, H2 = N / 4;
  const bool b1 = (q >> 1) & 1, b0 = q & 1;
#pragma unroll
  for (int j = 0; j < H1; ++j) {
    const double send = b1 ? v[j] : v[H1 + j];
    const double keep = b1 ? v[H1 + j] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int j = 0; j < H2; ++j) {
    const double send = b0 ? v[j] : v[H2 + j];
    const double keep = b0 ? v[H2 + j] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// one arrival on the mbarrier once every cp.async this thread issued so far has landed (not counted in advance:
// the barrier's expected count includes it)
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// block barrier 1 among the 128 threads of warp group 1 (warps 4-7)
__device__ __forceinline__ void group1_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Schedule of one CTA over its slices (one block-wide barrier per slice; the sAc hand-off uses two
// 8-warp mbarriers whose waits sit after independent work, so they normally cost nothing):
//   wait full[b] (T_k), wait aready (sAc_k)   | phase 1_k: E = T + sAc B^T, f
//   __syncthreads (S2_k)                        | E complete; buffers of slice k-1 free -> TMA T_{k+1},
//                                               | reduce sGC of slice k-1, prefetch c_{k+2}
//   phase 3_k (reads sAc_k) ; arrive p3done     |
//   phase 2_k, first half of the r-tiles        |
//   wait p3done ; rebuild sAc_{k+1} ; arrive aready
//   phase 2_k, second half ; dF/dC butterfly -> sGC[k%2]
#ifdef TF_EVAL_PROFILE
// Development timeline: CTA 0, lane 0 of every warp records clock64 at 8 points of its first 16 slices.
__device__ unsigned long long g_eval_tl[16 * 16 * 8];
__device__ unsigned long long g_eval_cta[4096 * 4];   // per CTA: globaltimer at start, loop start, loop end, end
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TLC(pt)                                                                   \
  do {                                                                            \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_eval_cta[blockIdx.x * 4 + (pt)] = gtimer(); \
  } while (0)
#define TL(kk, pt)                                                                                          \
  do {                                                                                                      \
    if (blockIdx.x == 0 && lane == 0 && (kk) < 16) g_eval_tl[((kk) * 16 + warp) * 8 + (pt)] = clock64(); \
  } while (0)
#else
#define TL(kk, pt) \
  do {             \
  } while (0)
#define TLC(pt) \
  do {          \
  } while (0)
#endif

// RECON = false is the Pi-form pass (the three MTTKRPs of T itself): phase 1 is skipped,
// phases 2-3 run on T_k, and the per-CTA scalar is sum t^2 (for the Gram expansion of f).
// two co-resident CTAs of the 64-wide tile where R is small enough (<= 128 registers; measured: c3's Pi pass 0.49
// vs 0.56 ms with one CTA per SM, the second CTA hides the per-slice barrier and reduction latency)
template <int NT, bool RECON>
constexpr int eval_min_blocks(int BT) {
  return (BT == 32 || NT <= 2 || (!RECON && NT <= 3)) ? 2 : 1;
}
template <int NT, bool kTMA, int BT, bool RECON>
__global__ void __launch_bounds__(EvalTile<BT>::THREADS, eval_min_blocks<NT, RECON>(BT))
    k_eval_fused(const __grid_constant__ CUtensorMap tmapT, const __grid_constant__ CUtensorMap tmapT4,
                 const double* __restrict__ T, EvalArgs p) {
  if (p.run_if && *p.run_if == 0) return;   // guarded fallback not needed (uniform across the grid)
  using S = EvalSmem<NT, BT>;
  using Gm = EvalTile<BT>;
  // phase 3 with the prescaled tile -A diag(c_k) (rebuilt per slice, needed by phase 1 of the residual form)
  // or, in the Pi pass, with unscaled A (in tensor memory) and the per-slice scaling on the product (measured: c4/c5
  // 6%/2.5% faster; at small R, with the stream-K grid and A in tensor memory, too: 500^3 R = 16/24/32 -5%/-2%/-8%,
  // R = 8 equal; round 1's prescaled path was 9% faster at c3 when A came from shared memory)
  constexpr bool kPre = RECON || NT <= TF_PI_PRE_MAXNT;
  // Pi pass with the unscaled A: phase 3's A fragments are the same for every slice and every warp, so they
  // are parked once in tensor memory (16 k-steps x NT4 doubles per lane = 512 columns) and read with
  // tcgen05.ld instead of 13 shared-memory loads per k-step
  constexpr bool kTmemA = !kPre && TF_TMEM_A == 1;
  constexpr bool kTmemB = (RECON && NT > 4) || (!kPre && TF_TMEM_A == 2);   // residual form: B of phase 2 in TMEM
  // Pi form with R > 32 (measured: c5 -0.8%, c4 -1.4%; for R <= 32 the prescaled path with its hand-off inside
  // phase 2 stays, s-outer there was 0.4% slower at c3)
  constexpr bool kP2SOuter = TF_P2_SOUTER && !RECON && !kPre && !kTmemB;
  constexpr int NT4 = 4 * ((NT + 3) / 4);
  constexpr int kP2U = p2_unroll<NT>(), kP3U = p3_unroll<NT>();
  // tensor-memory columns: 16 k-steps x NT4 (phase-3 A) or NT x 16 (phase-2 B) doubles per lane, 2 columns each,
  // rounded up to a power of two (small R leaves room for a co-resident CTA's allocation)
  constexpr int kTmemNeed = kTmemB ? 32 * NT : 32 * NT4;
  constexpr int kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  // sAc pitch: with the fragments in TMEM the only per-slice reads of sAc are dF/dC's rows 8w + 2q + e, which a
  // pitch = 2 (mod 8) doubles makes conflict-free (2 * pitch = 4 mod 16); otherwise the fragment pitch LDF
  constexpr int LDA = kTmemA ? 8 * NT + 2 : S::LDF;
  constexpr int kBI = Gm::BI, kBJ = Gm::BJ, kLDE = Gm::LDE, NW = Gm::NW, kThreads = Gm::THREADS;
  constexpr int MF = Gm::MF, NF = Gm::NF;
  constexpr int kTileBytes = Gm::TILE_BYTES;
  constexpr int RP = S::RP;
  constexpr int LDF = S::LDF;
  constexpr int NV = ((NT + 3) / 4) * 4;   // dF/dC values per lane, padded for the butterfly
  constexpr int NT1 = (NT + 1) / 2;        // r-tiles of phase 2 before the sAc hand-off
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  double* sTE = reinterpret_cast<double*>(smem + S::off_te);
  double* sAc = reinterpret_cast<double*>(smem + S::off_a);   // -A diag(c_k)
  double* sB = reinterpret_cast<double*>(smem + S::off_b);    // B (unscaled)
  double* sC = reinterpret_cast<double*>(smem + S::off_c);    // c_k at sC[(k%4)*RP]
  double* sGC = reinterpret_cast<double*>(smem + S::off_gc);
  double* sRed = reinterpret_cast<double*>(smem + S::off_red);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::off_bar);
  uint64_t* full = bar;          // [2] TMA completion per T/E buffer
  uint64_t* p3done = bar + 2;    // all 8 warps finished reading sAc_k (phase 3)
  uint64_t* aready = bar + 3;    // all 8 warps wrote their rows of sAc_{k+1}
  // Decoupled Pi pass (kDec): no block barrier per slice. Warp group 0 (warps 0-3) runs ahead of group 1 (warps
  // 4-7, one of each per sub-partition), so that one warp's slice epilogue (scaling, butterfly, dF/dC rows) and
  // barrier waits overlap the other's DMMA stream instead of idling the pipe on every sub-partition at once.
  //   full[b]  T_k (TMA) and c_k (cp.async, 32 lanes of warp 4) landed in buffer / slot b = k % 2 (33 arrivals)
  //   empty[b] all 8 warps are done with buffer b; warp 4 then issues slice k + 2 into it
  //   gcf[x]   group 0 wrote its dF/dC rows of slice k into sGC[x = k % 2]; group 1 reduces them with its own
  //   gce[x]   group 1 finished reducing sGC[x]; group 0 may overwrite it (slice k + 2)
  uint64_t* empty = bar + 4;
  uint64_t* gcf = bar + 6;
  uint64_t* gce = bar + 8;
  //   mid[x]   group 1 finished phase 3 of slice k (x = k % 2): group 0 starts slice k + 1 only then, so that it
  //            leads by at most about half a slice (the TMA of slice k + 2, issued when slice k is done everywhere,
  //            keeps half a slice of lead; unthrottled, group 0 ran up to the TMA and waited on it every slice)
  uint64_t* mid = bar + 10;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int bid = blockIdx.x;
  constexpr bool kDecOK = kTMA && !RECON && !kPre && kTmemA && kP2SOuter && TF_TMEM_PIPE && BT == 64;
  const bool dec = kDecOK && p.decouple;
  auto init_bars = [&]() {
    mbar_init(&full[0], dec ? 33 : 1);
    mbar_init(&full[1], dec ? 33 : 1);
    mbar_init(p3done, NW);
    mbar_init(aready, NW);
    if (dec) {
      for (int x = 0; x < 2; ++x) {
        mbar_init(&empty[x], NW);
        mbar_init(&gcf[x], 4);
        mbar_init(&gce[x], 4);
        mbar_init(&mid[x], 4);
      }
    }
    fence_barrier_init();
  };
  const int ks1 = (int)((p.R + 3) / 4);    // phase-1 k-steps actually needed (R padded to 4, not 8)

  // ---- once per CTA: barriers, tensor memory
  TLC(0);
  if (tid == 0) {
    if (kTMA) {
      prefetch_tmap(&tmapT);
      if (p.tma4) prefetch_tmap(&tmapT4);
    }
    init_bars();
  }
  // the decoupled pass fills only rows < R of the c slots (cp.async): the padding rows stay zero from here
  if (dec)
    for (int x = tid; x < 4 * RP; x += kThreads) sC[x] = 0.0;
  uint32_t ta = 0;
  if constexpr (kTmemA || kTmemB) {
    if (warp == 0) tmem_alloc(&tmem_base_s, kTmemCols);
  }
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  if constexpr (kTmemA || kTmemB) ta = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16);
  double fsum0 = 0.0, fsum1 = 0.0;

  // ---- the CTA's segments. Stream-K (p.streamK): the (tile, slice) units in tile-major order are cut into
  // equal runs of p.unitsPerCta, one per CTA of a persistent grid (no partial last wave); a run covers the tail
  // of one tile, whole tiles and the head of another, each a segment with its own partial slot (sidx < nseg
  // <= p.kSplit). Otherwise one segment per CTA: tile bid % tiles, k-chunk bid / tiles.
  const int64_t tiles = (int64_t)p.nTi * p.nTj;
  int64_t u = p.streamK ? (int64_t)bid * p.unitsPerCta : 0;
  const int64_t uend = p.streamK ? min(tiles * p.K, u + p.unitsPerCta) : 1;
  for (bool firstSeg = true; u < uend; firstSeg = false) {
  int64_t tile, kA, kB;
  int sidx, nseg;
  if (p.streamK) {
    tile = u / p.K;
    kA = u - tile * p.K;
    kB = min(p.K, kA + (uend - u));
    const int64_t c0 = (tile * p.K) / p.unitsPerCta, c1 = (tile * p.K + p.K - 1) / p.unitsPerCta;
    sidx = (int)(bid - c0);
    nseg = (int)(c1 - c0 + 1);
    u += kB - kA;
  } else {
    tile = bid % tiles;
    const int kc = (int)(bid / tiles);
    kA = (int64_t)kc * p.kChunk;
    kB = min(p.K, kA + p.kChunk);
    sidx = kc;
    nseg = p.kSplit;
    u = 1;
  }
  const int it = (int)(tile % p.nTi), jt = (int)(tile / p.nTi);
  const int64_t i0 = (int64_t)it * kBI, j0 = (int64_t)jt * kBJ;
  const int nk = (int)max((int64_t)0, kB - kA);
  if (!firstSeg) {   // every barrier of the previous segment has completed all its phases: start afresh
    if (tid == 0) {
      for (int b = 0; b < (dec ? 12 : 4); ++b) mbar_inval(&bar[b]);
      init_bars();
    }
    __syncthreads();
  }

  auto load_c = [&](int64_t kloc, int slot) {
    if (tid < RP) sC[slot * RP + tid] = (tid < p.R) ? p.C[(p.kbeg + kloc) + p.Ktot * tid] : 0.0;
  };
  // in-loop refill of the ring: asynchronous; waited for (wait_group 0) just before the next slice barrier, a
  // whole slice after the issue. Rows R..RP-1 of every slot stay zero from the prologue fill.
  auto load_c_async = [&](int64_t kloc, int slot) {
    if (tid < p.R) cp_async8_ca(&sC[slot * RP + tid], &p.C[(p.kbeg + kloc) + p.Ktot * tid]);
    cp_async_commit();
  };
  // TMA box of BT + 4 rows (the smem row pitch; bank-conflict-free fragments) by BT columns. Interior i-tiles
  // go through the 4-D view (i mod BT, i / BT, j, k) whose first extent is BT, so the 4 padding rows are out of
  // bounds there (zero fill, never fetched: otherwise each 512-byte row read drags in the next tile's first
  // sector, which the stream-K grid no longer reads at the same time — 19.0 instead of 13.9 GB at c5); the last,
  // partial i-tile uses the 3-D map (its padding rows are past I anyway).
  auto load_tile_tma = [&](double* dst, int64_t kloc, uint64_t* fb) {
    if (p.tma4 && i0 + kBI <= p.I) tma_load_4d(dst, &tmapT4, 0, it, (int)j0, (int)kloc, fb);
    else tma_load_3d(dst, &tmapT, (int)i0, (int)j0, (int)kloc, fb);
  };
  auto load_tile_plain = [&](int64_t kloc, double* dst) {
    for (int idx = tid; idx < kBI * kBJ; idx += kThreads) {
      const int j = idx / kBI, i = idx % kBI;
      const int64_t gi = i0 + i, gj = j0 + j;
      dst[j * kLDE + i] = (gi < p.I && gj < p.J) ? T[gi + p.ldT * (gj + p.J * kloc)] : 0.0;
    }
  };

  // decoupled pass: warp 4 issues slice kloc into buffer / c slot buf (TMA of T_k by lane 0, c_k by cp.async)
  auto issue_dec = [&](int64_t kloc, int buf) {
    if (lane == 0) {
      fence_proxy_async_smem();   // generic-proxy reads of the buffer (previous slice) before the async write
      mbar_arrive_expect_tx(&full[buf], kTileBytes);
      load_tile_tma(sTE + buf * (kLDE * kBJ), kloc, &full[buf]);
    }
    for (int r = lane; r < p.R; r += 32) cp_async8_ca(&sC[buf * RP + r], &p.C[(p.kbeg + kloc) + p.Ktot * r]);
    cp_async_mbar_arrive_noinc(&full[buf]);
  };
  // ---- segment prologue
  if (dec) {
    if (warp == 4)
      for (int u = 0; u < 2 && u < nk; ++u) issue_dec(kA + u, u);
  } else if (kTMA && tid == 0) {
    fence_proxy_async_smem();   // generic-proxy use of the tile buffers by the previous segment
    for (int u = 0; u < 2 && u < nk; ++u) {
      mbar_arrive_expect_tx(&full[u], kTileBytes);
      load_tile_tma(sTE + u * (kLDE * kBJ), kA + u, &full[u]);
    }
  }
  if (!kTMA && nk > 0) load_tile_plain(kA, sTE);
  // Factor tiles, coalesced along the contiguous (row) index of the column-major factors and batched so
  // that 8 loads per thread are in flight: B -> sB (unscaled, kept), A -> sAc (unscaled, staging only).
  {
    constexpr int kLoadBatch = 8;
    for (int base = tid; base < kBJ * LDF; base += kLoadBatch * kThreads) {
      double v[kLoadBatch];
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = base + u * kThreads;
        const int j = idx % kBJ, r = idx / kBJ;
        const int64_t gj = j0 + j;
        const bool ok = idx < kBJ * LDF && gj < p.J && r < p.R;
        v[u] = ok ? p.B[gj + p.J * r] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = base + u * kThreads;
        if (idx < kBJ * LDF) sB[(idx % kBJ) * LDF + idx / kBJ] = v[u];
      }
    }
    for (int base = tid; base < kBI * LDA; base += kLoadBatch * kThreads) {
      double v[kLoadBatch];
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = base + u * kThreads;
        const int i = idx % kBI, r = idx / kBI;
        const int64_t gi = i0 + i;
        const bool ok = idx < kBI * LDA && gi < p.I && r < p.R;
        v[u] = ok ? p.A[gi + p.I * r] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = base + u * kThreads;
        if (idx < kBI * LDA) sAc[(idx % kBI) * LDA + idx / kBI] = v[u];
      }
    }
  }
  __syncthreads();
  // Unscaled A, distributed over the CTA: thread (warp, g, q) owns A[8*warp + 2q + e][8t + g] (its
  // phase-2 P^T fragment positions); used for dF/dC and to rebuild sAc = -A diag(c_k) each slice.
  // Read from the staged tile; the first rebuild overwrites exactly these positions (same thread).
  // (the Pi form keeps sAc = A unscaled for the whole CTA: phase 3 scales its per-slice product instead, so
  // neither Areg nor the per-slice rebuild and its hand-off exist there)
  double Areg[NT][2];
  if constexpr (kPre) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) Areg[t][e] = sAc[(8 * warp + 2 * q + e) * LDA + 8 * t + g];
  }
  if constexpr (kTmemB) {   // phase-2 B fragments B[4s + q][8t + g], per lane: t-major, 16 k-steps per t
    if (warp < 4) {
#pragma unroll 1
      for (int t = 0; t < NT; ++t) {
#pragma unroll
        for (int s0 = 0; s0 < kBJ / 4; s0 += 4) {
          double v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = sB[(4 * (s0 + j) + q) * LDF + 8 * t + g];
          tmem_st4(ta + 2 * (t * 16 + s0), v);
        }
      }
      tmem_wait_st();
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
  }
  if constexpr (kTmemA) {
    if (warp < 4) {   // one warp per lane quadrant writes the fragments A[4s + q][8t + g] of every (s, t)
#pragma unroll 1
      for (int s2 = 0; s2 < kBI / 4; ++s2) {
#pragma unroll
        for (int t0 = 0; t0 < NT4; t0 += 4) {
          double v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = (t0 + j < NT) ? sAc[(4 * s2 + q) * LDA + 8 * (t0 + j) + g] : 0.0;
          tmem_st4(ta + 2 * (s2 * NT4 + t0), v);
        }
      }
      tmem_wait_st();
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
  }
  auto rebuild_sAc = [&](const double* c) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double cr = -c[8 * t + g];
      sAc[(8 * warp + 2 * q) * LDA + 8 * t + g] = Areg[t][0] * cr;
      sAc[(8 * warp + 2 * q + 1) * LDA + 8 * t + g] = Areg[t][1] * cr;
    }
  };
  if (nk > 0 && !dec) {
    for (int u = 0; u < 4; ++u) load_c(kA + min(u, nk - 1), u);   // all four slots: sets the zero padding rows
    __syncthreads();
    if constexpr (kPre) rebuild_sAc(sC);
  }
  __syncthreads();

  double accA[NT][2], accB[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) accA[t][0] = accA[t][1] = accB[t][0] = accB[t][1] = 0.0;

  const int wi = warp & 1, wj = warp >> 1;   // phase-1 warp tile: rows (BT/2)*wi.., cols 16*wj..

  TLC(1);
  if constexpr (kDecOK) {
    if (dec) {
      const int grp = warp >> 2;
      if (grp == 1 && p.skewNs > 0) {   // group 0's head start (re-established at every segment start)
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
          __nanosleep(256);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (t - t0 < (unsigned long long)p.skewNs);
      }
      for (int kk = 0; kk < nk; ++kk) {
        const int b = kk & 1;
        const uint32_t use = (uint32_t)(kk >> 1);   // how many times buffer / slot b was used before
        const int64_t k = kA + kk;
        const double* sT = sTE + b * (kLDE * kBJ);
        const double* sc = sC + b * RP;
        if (grp == 0 && kk > 0 && p.decouple == 1) mbar_wait(&mid[b ^ 1], ((kk - 1) >> 1) & 1);
        mbar_wait(&full[b], use & 1);
        // ---- phase 3: Q = A^T T_k (A fragments from tensor memory), accB^T -= diag(c_k) Q
        {
          double Qt[NT][2];
#pragma unroll
          for (int t = 0; t < NT; ++t) Qt[t][0] = Qt[t][1] = 0.0;
          const double* pe = sT + (8 * warp + g) * kLDE + q;
          double af[2][NT];
          tmem_ld_doubles<NT>(ta, af[0]);
          tmem_wait_ld();
#pragma unroll
          for (int s = 0; s < kBI / 4; ++s) {
            if (s + 1 < kBI / 4) tmem_ld_doubles<NT>(ta + 2 * (s + 1) * NT4, af[(s + 1) & 1]);
            const double bb = pe[4 * s];
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma(Qt[t], af[s & 1][t], bb);
            if (s + 1 < kBI / 4) tmem_wait_ld();
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double cr = -sc[8 * t + g];
            accB[t][0] = fma(cr, Qt[t][0], accB[t][0]);
            accB[t][1] = fma(cr, Qt[t][1], accB[t][1]);
          }
        }
        if (grp == 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&mid[b]);
        }
        // ---- phase 2: P = T_k B (k-steps outer, NT accumulators), accA += P diag(c_k), dF/dC rows
        double Pt[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) Pt[t][0] = Pt[t][1] = 0.0;
#pragma unroll
        for (int s = 0; s < kBJ / 4; ++s) {
          const double e = sT[(4 * s + q) * kLDE + 8 * warp + g];
          if (s & 1) fsum1 = fma(e, e, fsum1);
          else fsum0 = fma(e, e, fsum0);
          const double* pbs = sB + (4 * s + q) * LDF + g;
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma(Pt[t], pbs[8 * t], e);
        }
        double gcv[NV];
#pragma unroll
        for (int j = NT; j < NV; ++j) gcv[j] = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double cr = sc[8 * t + g];
          const double P0 = Pt[t][0], P1 = Pt[t][1];
          accA[t][0] = fma(cr, P0, accA[t][0]);
          accA[t][1] = fma(cr, P1, accA[t][1]);
          const double* pa = sAc + (8 * warp + 2 * q) * LDA + 8 * t + g;
          gcv[t] = fma(pa[0], P0, pa[LDA] * P1);
        }
        butterfly4<NV>(gcv, q);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);   // this warp's last reads of buffer b and c slot b are done
        if (grp == 0 && kk >= 2) mbar_wait(&gce[b], (use - 1) & 1);   // group 1 reduced slice k - 2 from sGC[b]
        {
          const int base = ((q >> 1) & 1) * (NV / 2) + (q & 1) * (NV / 4);
          double* gdst = sGC + b * NW * S::GCS + warp * S::GCS + q * S::GCP;
#pragma unroll
          for (int j = 0; j < NV / 4; ++j) {
            const int t = base + j;
            if (t < NT) gdst[8 * t + g] = gcv[j];
          }
        }
        if (grp == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&gcf[b]);
        } else {
          group1_sync();                   // group 1's rows of slice k are in sGC[b]
          mbar_wait(&gcf[b], use & 1);     // and group 0's
          const int t1 = tid - 128;
          if (t1 < RP) {
            const double* gsrc = sGC + b * NW * S::GCS + t1 + ((t1 >> 3) / (NV / 4)) * S::GCP;
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += gsrc[w * S::GCS];
            p.gCp[((int64_t)(it * p.nTj + jt) * p.K + k) * RP + t1] = v;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&gce[b]);
          if (warp == 4 && kk + 2 < nk) {
            mbar_wait(&empty[b], use & 1);   // every warp is done with slice k
            issue_dec(k + 2, b);
          }
        }
      }
    }
  }
  for (int kk = 0; kk < (dec ? 0 : nk); ++kk) {
    const int b = kk & 1;
    const int64_t k = kA + kk;
    double* sT = sTE + b * (kLDE * kBJ);
    const double* sc = sC + (kk & 3) * RP;
    TL(kk, 0);
    if (kTMA) mbar_wait(&full[b], (kk >> 1) & 1);
    if (kPre && kk > 0) mbar_wait(aready, (kk - 1) & 1);
    TL(kk, 1);

    // ---- phase 1: E = T + (-A diag(c)) B^T on a (BT/2) x 16 warp tile (MF x 2 fragments)
    if (RECON) {
      double E[MF][NF][2];
#pragma unroll
      for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            E[m][n][e] = sT[(16 * wj + 8 * n + 2 * q + e) * kLDE + (kBI / 2) * wi + 8 * m + g];
      const double* pa = sAc + ((kBI / 2) * wi + g) * LDA + q;
      const double* pb = sB + (16 * wj + g) * LDF + q;
#pragma unroll
      for (int s = 0; s < RP / 4; ++s) {
        if (s < ks1) {
          double a[MF], bb[NF];
#pragma unroll
          for (int m = 0; m < MF; ++m) a[m] = pa[8 * m * LDF + 4 * s];
#pragma unroll
          for (int n = 0; n < NF; ++n) bb[n] = pb[8 * n * LDF + 4 * s];
#pragma unroll
          for (int m = 0; m < MF; ++m)
#pragma unroll
            for (int n = 0; n < NF; ++n) dmma(E[m][n], a[m], bb[n]);
        }
      }
#pragma unroll
      for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n) {
          fsum0 = fma(E[m][n][0], E[m][n][0], fsum0);
          fsum1 = fma(E[m][n][1], E[m][n][1], fsum1);
#pragma unroll
          for (int e = 0; e < 2; ++e)
            sT[(16 * wj + 8 * n + 2 * q + e) * kLDE + (kBI / 2) * wi + 8 * m + g] = E[m][n][e];
        }
    }
    TL(kk, 2);
    if (TF_C_ASYNC) cp_async_wait0();   // c_{k+1} (issued in slice k-1) has landed
    __syncthreads();  // S2_k: E_k complete; every warp is past phases 2/3 of slice k-1
    TL(kk, 3);

    if (kk + 1 < nk) {
      if (kTMA) {
        if (kk >= 1 && tid == 0) {   // slices 0 and 1 were issued in the prologue
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[b ^ 1], kTileBytes);
          load_tile_tma(sTE + (b ^ 1) * (kLDE * kBJ), k + 1, &full[b ^ 1]);
        }
      }
    }
    if (kk > 0 && tid < RP) {
      const double* gsrc = sGC + ((kk - 1) & 1) * NW * S::GCS + tid + ((tid >> 3) / (NV / 4)) * S::GCP;
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += gsrc[w * S::GCS];
      p.gCp[((int64_t)(it * p.nTj + jt) * p.K + (k - 1)) * RP + tid] = v;
    }
    if (kk + 2 < nk) {
      if (TF_C_ASYNC) load_c_async(k + 2, (kk + 2) & 3);
      else load_c(k + 2, (kk + 2) & 3);
    }

    // ---- phase 3: accB^T += (-A diag c)^T E for j-cols 8*warp.., all R (prescaled sAc: no DMUL)
    if constexpr (kPre) {
      const double* pe = sT + (8 * warp + g) * kLDE + q;
      const double* pa = sAc + q * LDA + g;
#pragma unroll 4
      for (int s = 0; s < kBI / 4; ++s) {
        const double bb = pe[4 * s];
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(accB[t], pa[4 * s * LDF + 8 * t], bb);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(p3done);
    } else {
      // Pi form: Q = A^T T_k (unscaled A, fresh per slice), then accB^T -= diag(c_k) Q (one DFMA per entry)
      double Qt[NT][2];
#pragma unroll
      for (int t = 0; t < NT; ++t) Qt[t][0] = Qt[t][1] = 0.0;
      const double* pe = sT + (8 * warp + g) * kLDE + q;
      const double* pa = sAc + q * LDA + g;
      if constexpr (kTmemA) {
#if TF_TMEM_PIPE
        // the fragments of k-step s+1 are loaded before the DMMAs of step s issue; the wait for them sits
        // after those DMMAs (fully unrolled: both fragment buffers are static registers)
        double af[2][NT];
        tmem_ld_doubles<NT>(ta, af[0]);
        tmem_wait_ld();
#pragma unroll kP3U
        for (int s = 0; s < kBI / 4; ++s) {
          if (s + 1 < kBI / 4) tmem_ld_doubles<NT>(ta + 2 * (s + 1) * NT4, af[(s + 1) & 1]);
          const double bb = pe[4 * s];
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma(Qt[t], af[s & 1][t], bb);
          if (s + 1 < kBI / 4) tmem_wait_ld();
        }
#else
#pragma unroll 2
        for (int s = 0; s < kBI / 4; ++s) {
          double af[NT];
          tmem_ld_doubles<NT>(ta + 2 * s * NT4, af);
          const double bb = pe[4 * s];
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma(Qt[t], af[t], bb);
        }
#endif
      } else {
#pragma unroll kP3Unroll
        for (int s = 0; s < kBI / 4; ++s) {
          const double bb = pe[4 * s];
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma(Qt[t], pa[4 * s * LDF + 8 * t], bb);
        }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double cr = -sc[8 * t + g];   // accB[t][e] is (r = 8t+g, j = 8w+2q+e)
        accB[t][0] = fma(cr, Qt[t][0], accB[t][0]);
        accB[t][1] = fma(cr, Qt[t][1], accB[t][1]);
      }
    }
    TL(kk, 4);

    // ---- phase 2: P^T_t = B_t^T E^T for i-cols 8*warp.. (t outer, E fragments in registers);
    //      accA^T += diag(c) P^T; dF/dC partial = sum_i A o P; the sAc hand-off sits between the halves
    if constexpr (kP2SOuter) {
      // Pi form (no sAc hand-off inside phase 2): k-steps outer and the NT r-tiles inner, so every warp keeps NT
      // independent DMMA accumulators in flight (like phase 3) instead of two chains per r-tile
      double Pt[NT][2];
#pragma unroll
      for (int t = 0; t < NT; ++t) Pt[t][0] = Pt[t][1] = 0.0;
#pragma unroll kP2U
      for (int s = 0; s < kBJ / 4; ++s) {
        const double e = sT[(4 * s + q) * kLDE + 8 * warp + g];
        if (s & 1) fsum1 = fma(e, e, fsum1);   // sum t^2 of this slice tile (rows 8w.., all 64 columns)
        else fsum0 = fma(e, e, fsum0);
        const double* pbs = sB + (4 * s + q) * LDF + g;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(Pt[t], pbs[8 * t], e);
      }
      double gcv[NV];
#pragma unroll
      for (int j = NT; j < NV; ++j) gcv[j] = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double cr = sc[8 * t + g];
        const double P0 = Pt[t][0], P1 = Pt[t][1];   // P[i = 8w+2q+e][r = 8t+g]
        accA[t][0] = fma(cr, P0, accA[t][0]);
        accA[t][1] = fma(cr, P1, accA[t][1]);
        const double* pa = sAc + (8 * warp + 2 * q) * LDA + 8 * t + g;
        gcv[t] = fma(pa[0], P0, pa[LDA] * P1);
      }
      TL(kk, 7);
      butterfly4<NV>(gcv, q);
      const int base = ((q >> 1) & 1) * (NV / 2) + (q & 1) * (NV / 4);
      double* gdst = sGC + (kk & 1) * NW * S::GCS + warp * S::GCS + q * S::GCP;
#pragma unroll
      for (int j = 0; j < NV / 4; ++j) {
        const int t = base + j;
        if (t < NT) gdst[8 * t + g] = gcv[j];
      }
    } else {
      double ea[kBJ / 4];
#pragma unroll
      for (int s = 0; s < kBJ / 4; ++s) ea[s] = sT[(4 * s + q) * kLDE + 8 * warp + g];
      if (!RECON) {   // sum t^2 of this slice tile: warp w's fragments cover rows 8w.., all 64 columns
#pragma unroll
        for (int s = 0; s < kBJ / 4; s += 2) {
          fsum0 = fma(ea[s], ea[s], fsum0);
          fsum1 = fma(ea[s + 1], ea[s + 1], fsum1);
        }
      }
      double gcv[NV];
#pragma unroll
      for (int j = NT; j < NV; ++j) gcv[j] = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (kPre && t == NT1 && kk + 1 < nk) {
          TL(kk, 5);
          mbar_wait(p3done, kk & 1);          // every warp is done reading sAc_k
          TL(kk, 6);
          rebuild_sAc(sC + ((kk + 1) & 3) * RP);
          __syncwarp();
          if (lane == 0) mbar_arrive(aready);
        }
        double p0[2] = {0.0, 0.0}, p1[2] = {0.0, 0.0};
        const double* pbt = sB + q * LDF + 8 * t + g;
        if constexpr (kTmemB) {
          double bf[16];
          tmem_ld_d16(ta + 32 * t, bf);
          tmem_wait_ld();
#pragma unroll
          for (int s = 0; s < kBJ / 4; s += 2) {
            dmma(p0, bf[s], ea[s]);
            dmma(p1, bf[s + 1], ea[s + 1]);
          }
        } else {
#pragma unroll
          for (int s = 0; s < kBJ / 4; s += 2) {
            dmma(p0, pbt[(4 * s) * LDF], ea[s]);
            dmma(p1, pbt[(4 * s + 4) * LDF], ea[s + 1]);
          }
        }
        const double cr = sc[8 * t + g];
        const double P0 = p0[0] + p1[0], P1 = p0[1] + p1[1];   // P[i = 8w+2q+e][r = 8t+g]
        accA[t][0] = fma(cr, P0, accA[t][0]);
        accA[t][1] = fma(cr, P1, accA[t][1]);
        if constexpr (kPre) {
          gcv[t] = fma(Areg[t][0], P0, Areg[t][1] * P1);
        } else {
          const double* pa = sAc + (8 * warp + 2 * q) * LDA + 8 * t + g;
          gcv[t] = fma(pa[0], P0, pa[LDA] * P1);
        }
      }
      if (kPre && NT1 >= NT && kk + 1 < nk) {   // NT == 1: hand-off after the only tile
        mbar_wait(p3done, kk & 1);
        rebuild_sAc(sC + ((kk + 1) & 3) * RP);
        __syncwarp();
        if (lane == 0) mbar_arrive(aready);
      }
      TL(kk, 7);
      butterfly4<NV>(gcv, q);
      const int base = ((q >> 1) & 1) * (NV / 2) + (q & 1) * (NV / 4);
      double* gdst = sGC + (kk & 1) * NW * S::GCS + warp * S::GCS + q * S::GCP;
#pragma unroll
      for (int j = 0; j < NV / 4; ++j) {
        const int t = base + j;
        if (t < NT) gdst[8 * t + g] = gcv[j];
      }
    }
    if (!kTMA && kk + 1 < nk) {
      __syncthreads();   // no TMA: everyone is done with buffer b^1 (slice k-1) and with the c ring
      load_tile_plain(k + 1, sTE + (b ^ 1) * (kLDE * kBJ));
      __syncthreads();
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  if (nk > 0 && tid < RP && !dec) {
    const double* gsrc = sGC + ((nk - 1) & 1) * NW * S::GCS + tid + ((tid >> 3) / (NV / 4)) * S::GCP;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += gsrc[w * S::GCS];
    p.gCp[((int64_t)(it * p.nTj + jt) * p.K + (kB - 1)) * RP + tid] = v;
  }

  // ---- epilogue: partials (accA: +sum E B diag c; accB: -sum (A diag c)^T E, i.e. dF/dB directly)
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t i = i0 + 8 * warp + 2 * q + e;
      p.gAp[((int64_t)(jt * p.kSplit + sidx) * p.Ipad + i) * RP + 8 * t + g] = accA[t][e];
      if (sidx == nseg - 1)   // the tile's last segment zeroes the slots no segment of this tile uses
        for (int s2 = nseg; s2 < p.kSplit; ++s2) p.gAp[((int64_t)(jt * p.kSplit + s2) * p.Ipad + i) * RP + 8 * t + g] = 0.0;
    }
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = j0 + 8 * warp + 2 * q + e;
      p.gBp[((int64_t)(it * p.kSplit + sidx) * p.Jpad + j) * RP + 8 * t + g] = accB[t][e];
      if (sidx == nseg - 1)
        for (int s2 = nseg; s2 < p.kSplit; ++s2) p.gBp[((int64_t)(it * p.kSplit + s2) * p.Jpad + j) * RP + 8 * t + g] = 0.0;
    }
  }   // segments
  TLC(2);
  if constexpr (kTmemA || kTmemB) {
    if (warp == 0) tmem_dealloc(tmem_base_s, kTmemCols);
  }
  double fsum = warp_sum(fsum0 + fsum1);
  if (lane == 0) sRed[warp] = fsum;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += sRed[w];
    p.fp[bid] = v;
  }
  TLC(3);
}

// Fixed-order reduction of all partials into the packed gradient and f (row a6). Threads run along r
// (contiguous in the partial buffers) so the partial reads coalesce; the packed gradient writes are strided
// but small. grad blocks: dF/dA = -sum accA, dF/dB = +sum accB (accB already holds -(A diag c)^T E),
// dF/dC = -sum gC partials (rows outside the local slices are written 0).
// Ordered sum of n partials x[s * stride] with 8 loads in flight (fixed left-to-right order of the partial
// sums within each of the 8 lanes, then lanes combined in order: deterministic for given n).
__device__ __forceinline__ double ordered_sum8(const double* __restrict__ x, int64_t n, int64_t stride) {
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t s = 0;
  for (; s + 8 <= n; s += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += x[(s + u) * stride];
  }
  for (int u = 0; s < n; ++s, ++u) acc[u] += x[s * stride];
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

__global__ void k_eval_finalize(EvalArgs p, int RP, double* __restrict__ f, double* __restrict__ grad) {
  if (p.run_if && *p.run_if == 0) return;
  const int64_t R = p.R;
  const int64_t nA = p.I * R, nB = p.J * R, nC = p.Ktot * R;
  const int64_t total = nA + nB + nC;
  const int64_t nPA = (int64_t)p.nTj * p.kSplit, nPB = (int64_t)p.nTi * p.kSplit, nPC = (int64_t)p.nTi * p.nTj;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < nA) {
      const int64_t i = idx / R, r = idx % R;
      grad[i + p.I * r] = -ordered_sum8(p.gAp + i * RP + r, nPA, p.Ipad * RP);
    } else if (idx < nA + nB) {
      const int64_t qq = idx - nA, j = qq / R, r = qq % R;
      grad[nA + j + p.J * r] = ordered_sum8(p.gBp + j * RP + r, nPB, p.Jpad * RP);
    } else {
      const int64_t qq = idx - nA - nB, kg = qq / R, r = qq % R;
      const int64_t k = kg - p.kbeg;
      double v = 0.0;
      if (k >= 0 && k < p.K) v = -ordered_sum8(p.gCp + k * RP + r, nPC, p.K * RP);
      grad[nA + nB + kg + p.Ktot * r] = v;
    }
  }
  if (blockIdx.x == 0) {
    __shared__ double red[32];
    double v = 0.0;
    for (int64_t s = threadIdx.x; s < p.nCta; s += blockDim.x) v += p.fp[s];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      *f = 0.5 * t;
    }
  }
}

// Pi-form reduction: the MTTKRP partials of the RECON = false pass (accA = +M1, accB = -M2, gC = +M3) become
// grad = W Pi - M (Kolda's theorem). On entry grad already holds W Pi (three small DMMA
// GEMMs with Pi^(l) = Hadamard product of the other Grams, the C Gram over the local slices); rows of dF/dC
// outside the local slices are written 0. part[blk] = {<A, M1>, ||grad||^2, ||W Pi||^2} per block.
constexpr int kPiThreads = 256;
__global__ void __launch_bounds__(kPiThreads) k_eval_finalize_pi(EvalArgs p, int RP, double* __restrict__ grad,
                                                                 double* __restrict__ part) {
  const int64_t R = p.R;
  const int64_t nA = p.I * R, nB = p.J * R, nC = p.Ktot * R;
  const int64_t total = nA + nB + nC;
  const int64_t nPA = (int64_t)p.nTj * p.kSplit, nPB = (int64_t)p.nTi * p.kSplit, nPC = (int64_t)p.nTi * p.nTj;
  double ip = 0.0, g2 = 0.0, w2 = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double m = 0.0;
    int64_t out;
    bool live = true;
    if (idx < nA) {
      const int64_t i = idx / R, r = idx % R;
      m = ordered_sum8(p.gAp + i * RP + r, nPA, p.Ipad * RP);
      out = i + p.I * r;
      ip = fma(p.A[out], m, ip);
    } else if (idx < nA + nB) {
      const int64_t qq = idx - nA, j = qq / R, r = qq % R;
      m = -ordered_sum8(p.gBp + j * RP + r, nPB, p.Jpad * RP);
      out = nA + j + p.J * r;
    } else {
      const int64_t qq = idx - nA - nB, kg = qq / R, r = qq % R;
      const int64_t k = kg - p.kbeg;
      out = nA + nB + kg + p.Ktot * r;
      if (k >= 0 && k < p.K) m = ordered_sum8(p.gCp + k * RP + r, nPC, p.K * RP);
      else live = false;
    }
    const double wp = live ? grad[out] : 0.0;
    const double gval = wp - m;
    grad[out] = gval;
    g2 = fma(gval, gval, g2);
    w2 = fma(wp, wp, w2);
  }
  __shared__ double red[3][kPiThreads / 32];
  ip = warp_sum(ip);
  g2 = warp_sum(g2);
  w2 = warp_sum(w2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = ip;
    red[1][threadIdx.x >> 5] = g2;
    red[2][threadIdx.x >> 5] = w2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < kPiThreads / 32; ++w) v += red[threadIdx.x][w];
    part[blockIdx.x * 3 + threadIdx.x] = v;
  }
}

// f = 1/2 ||T||^2 - <A, M1> + 1/2 1^T (piA * piB * piC) 1 and the cancellation guard (one block; every sum in
// a fixed order: strided per-thread partials, then warps, then thread 0 over the warps).
__global__ void __launch_bounds__(1024) k_eval_pi_guard(EvalArgs p, const double* __restrict__ grams,
                                                       const double* __restrict__ part, int nblk,
                                                       double* __restrict__ f, int* __restrict__ flag,
                                                       int check_grad) {
  __shared__ double red[5][32];
  const int64_t R = p.R, RR = R * R;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // t2, x2, ip, g2, w2
  for (int64_t s = threadIdx.x; s < p.nCta; s += blockDim.x) v[0] += p.fp[s];
#pragma unroll 4
  for (int64_t e = threadIdx.x; e < RR; e += blockDim.x) v[1] += grams[e] * grams[RR + e] * grams[2 * RR + e];
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    v[2] += part[3 * b];
    v[3] += part[3 * b + 1];
    v[4] += part[3 * b + 2];
  }
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const double x = warp_sum(v[u]);
    if ((threadIdx.x & 31) == 0) red[u][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int u = 0; u < 5; ++u)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t[u] += red[u][w];
    const double fv = (0.5 * t[0] - t[2]) + 0.5 * t[1];
    *f = fv;
    const bool safe = (2.0 * fv >= 1e-3 * t[0]) && (!check_grad || t[3] >= 1e-6 * t[4]) && isfinite(fv);
    *flag = safe ? 0 : 1;
  }
}

int eval_pi_blocks(int nsm) { return 2 * nsm; }

cudaError_t launch_eval_finalize_pi(const EvalArgs& p, int RP, double* grad, double* part, int nblk,
                                    cudaStream_t st) {
  k_eval_finalize_pi<<<nblk, kPiThreads, 0, st>>>(p, RP, grad, part);
  return cudaGetLastError();
}

cudaError_t launch_eval_pi_guard(const EvalArgs& p, const double* grams, const double* part, int nblk, double* f,
                                 int* flag, cudaStream_t st, bool check_grad) {
  k_eval_pi_guard<<<1, 1024, 0, st>>>(p, grams, part, nblk, f, flag, check_grad ? 1 : 0);
  return cudaGetLastError();
}

template <int NT, int BT, bool RECON>
static cudaError_t launch_eval_ntr(const CUtensorMap* map, const double* T, const EvalArgs& p, bool tma,
                                   cudaStream_t st) {
  const size_t smem = EvalSmem<NT, BT>::bytes;
  constexpr int threads = EvalTile<BT>::THREADS;
  if (tma) {
    auto kern = k_eval_fused<NT, true, BT, RECON>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<p.nCta, threads, smem, st>>>(map[0], map[1], T, p);
  } else {
    auto kern = k_eval_fused<NT, false, BT, RECON>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<p.nCta, threads, smem, st>>>(map[0], map[1], T, p);
  }
  return cudaGetLastError();
}

template <int NT, int BT>
static cudaError_t launch_eval_nt(const CUtensorMap* map, const double* T, const EvalArgs& p, bool tma,
                                  cudaStream_t st, bool recon) {
  if (BT == 64 && !recon) return launch_eval_ntr<NT, 64, false>(map, T, p, tma, st);
  return launch_eval_ntr<NT, BT, true>(map, T, p, tma, st);
}

cudaError_t launch_eval(const CUtensorMap* map, const double* T, const EvalArgs& p, int NT, bool tma, int BT,
                        cudaStream_t st, bool recon) {
  if (BT == 32) {
    if (!recon) return cudaErrorInvalidValue;   // the Pi-form pass exists for the 64-wide tile only
    switch (NT) {
#define TF_CASE(n) \
  case n:          \
    return launch_eval_nt<n, 32>(map, T, p, tma, st, true);
      TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
      TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
      default:
        return cudaErrorInvalidValue;
    }
  }
  switch (NT) {
#define TF_CASE(n) \
  case n:          \
    return launch_eval_nt<n, 64>(map, T, p, tma, st, recon);
    TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
    TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_eval_finalize(const EvalArgs& p, int RP, double* f, double* grad, int nsm, cudaStream_t st) {
  const int64_t total = (p.I + p.J + p.Ktot) * p.R;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 4LL * nsm);
  if (blocks < 1) blocks = 1;
  k_eval_finalize<<<blocks, 256, 0, st>>>(p, RP, f, grad);
  return cudaGetLastError();
}

// Resident CTAs per SM of the evaluation kernel actually launched (small R leaves room for 2-3 CTAs of the
// 64-wide tile; the k-chunk planner sizes the grid with it).
template <int NT>
static int eval_occ_nt(bool recon) {
  const size_t smem = EvalSmem<NT, 64>::bytes;
  int n = 0;
  cudaError_t e;
  if (recon) {
    e = cudaFuncSetAttribute(k_eval_fused<NT, true, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_eval_fused<NT, true, 64, true>,
                                                        EvalTile<64>::THREADS, smem);
  } else {
    e = cudaFuncSetAttribute(k_eval_fused<NT, true, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_eval_fused<NT, true, 64, false>,
                                                        EvalTile<64>::THREADS, smem);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return n < 1 ? 1 : n;
}

int eval_ctas_per_sm(int NT, bool recon) {
  static int cache[2][17] = {};
  if (NT < 1 || NT > 16) return 1;
  int& v = cache[recon ? 1 : 0][NT];
  if (v) return v;
  switch (NT) {
#define TF_CASE(n) \
  case n:          \
    v = eval_occ_nt<n>(recon); \
    break;
    TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
    TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
  }
  return v;
}

size_t eval_smem_bytes(int NT, int BT) {
  switch (NT) {
#define TF_CASE(n) \
  case n:          \
    return BT == 32 ? EvalSmem<n, 32>::bytes : EvalSmem<n, 64>::bytes;
    TF_CASE(1) TF_CASE(2) TF_CASE(3) TF_CASE(4) TF_CASE(5) TF_CASE(6) TF_CASE(7) TF_CASE(8)
    TF_CASE(9) TF_CASE(10) TF_CASE(11) TF_CASE(12) TF_CASE(13) TF_CASE(14) TF_CASE(15) TF_CASE(16)
#undef TF_CASE
    default:
      return 0;
  }
}

}  // namespace tfk

#ifdef TF_EVAL_PROFILE
extern "C" void tf_eval_cta_dump(int ncta) {
  static unsigned long long h[4096 * 4];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, tfk::g_eval_cta, sizeof(h));
  unsigned long long t0 = ~0ull, t1 = 0;
  double pro = 0, loop = 0, epi = 0;
  int n = ncta < 4096 ? ncta : 4096;
  for (int b = 0; b < n; ++b) {
    t0 = h[b * 4] < t0 ? h[b * 4] : t0;
    t1 = h[b * 4 + 3] > t1 ? h[b * 4 + 3] : t1;
    pro += (h[b * 4 + 1] - h[b * 4]) * 1e-3;
    loop += (h[b * 4 + 2] - h[b * 4 + 1]) * 1e-3;
    epi += (h[b * 4 + 3] - h[b * 4 + 2]) * 1e-3;
  }
  printf("CTAs %d: span %.1f us; per CTA avg prologue %.2f us, loop %.2f us, epilogue %.2f us\n", n, (t1 - t0) * 1e-3,
         pro / n, loop / n, epi / n);
  // per-SM style view: sum of CTA lifetimes vs span x concurrency
  double life = 0;
  for (int b = 0; b < n; ++b) life += (h[b * 4 + 3] - h[b * 4]) * 1e-3;
  printf("sum of CTA lifetimes %.1f us = %.3f x (span x 148)\n", life, life / ((t1 - t0) * 1e-3 * 148));
}

extern "C" void tf_eval_timeline_dump(void) {
  unsigned long long h[16 * 16 * 8];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, tfk::g_eval_tl, sizeof(h));
  const char* names[8] = {"top", "waits", "ph1 end", "S2", "ph3 end", "ph2 half", "p3done", "ph2 end"};
  for (int kk = 2; kk < 6; ++kk) {
    printf("slice %d (cycles from warp0 top):\n", kk);
    const unsigned long long t0 = h[(kk * 16 + 0) * 8 + 0];
    for (int w = 0; w < 8; ++w) {
      printf("  w%d:", w);
      for (int pt = 0; pt < 8; ++pt) printf(" %s=%lld", names[pt], (long long)(h[(kk * 16 + w) * 8 + pt] - t0));
      printf("\n");
    }
  }
}
#endif
