// Probe of the sm_100a int8 tensor-core path (tcgen05.mma kind::i8, int32 accumulators in TMEM) that an
// Ozaki-split evaluation would run on: (1) exactness against a host integer GEMM for K-major and MN-major
// A operands in the SWIZZLE_NONE canonical layouts, N = 96 + 8 (R = 100 padded to 104); (2) the
// sustained int8 MMA rate with operands resident in shared memory (148 CTAs, one issuing thread each).
// Development tool, not part of libtf.so.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8probe i8probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));          \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SWIZZLE_NONE shared-memory matrix descriptor (version 1 for sm_100)
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// instruction descriptor: s8 x s8 -> s32
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_mn, int b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(dst)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t t, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(t), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

constexpr int M = 128, N = 104, KD = 64;   // one CTA tile; K = 64 = two K=32 MMAs

// K-major canonical (16-byte units): ((8,n),2):((1,SBO),LBO) -> byte(row, k) = (k/16) LBO + (row/8) SBO + (row%8) 16 + k%16
__device__ __forceinline__ int kmaj(int row, int k, int rows) { return (k / 16) * (rows / 8) * 128 + (row / 8) * 128 + (row % 8) * 16 + (k % 16); }
// MN-major canonical: ((1,n),(8,k)):((X,SBO),(1,LBO)) -> byte(m, k) = (m/16) SBO + (k/8) LBO + (k%8) 16 + m%16
__device__ __forceinline__ int mnmaj(int m, int k, int kdim) { return (m / 16) * (kdim / 8) * 128 + (k / 8) * 128 + (k % 8) * 16 + (m % 16); }

__global__ void k_check(const int8_t* A, const int8_t* B, int32_t* D, int a_mn) {
  __shared__ __align__(1024) int8_t sA[M * KD];
  __shared__ __align__(1024) int8_t sB[N * KD];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * KD; i += blockDim.x) {
    const int m = i / KD, k = i % KD;   // A row-major [m][k]
    sA[a_mn ? mnmaj(m, k, KD) : kmaj(m, k, M)] = A[i];
  }
  for (int i = tid; i < N * KD; i += blockDim.x) {
    const int n = i / KD, k = i % KD;   // B as [n][k]
    sB[kmaj(n, k, N)] = B[i];
  }
  if (tid == 0) mbar_init(&bar, 1);
  if (warp == 0) tmem_alloc(&tbase, 128);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (tid == 0) {
    for (int s = 0; s < KD / 32; ++s) {
      uint64_t da;
      if (a_mn) da = sdesc(sA + s * 4 * 128, /*LBO k-group*/ 128, /*SBO m-group*/ (KD / 8) * 128);
      else da = sdesc(sA + s * 2 * (M / 8) * 128, /*LBO k-chunk*/ (M / 8) * 128, /*SBO*/ 128);
      const uint64_t db0 = sdesc(sB + s * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      const uint64_t db1 = sdesc(sB + s * 2 * (N / 8) * 128 + 96 / 8 * 128, (N / 8) * 128, 128);
      mma_i8(t0, da, db0, idesc_i8(M, 96, a_mn, 0), s > 0);
      mma_i8(t0 + 96, da, db1, idesc_i8(M, 8, a_mn, 0), s > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    int32_t r[8];
    tmem_ld8(t0 + ((uint32_t)(32 * warp) << 16) + c, r);
    for (int j = 0; j < 8; ++j) D[(32 * warp + (tid & 31)) * N + c + j] = r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(t0, 128);
}

// throughput: every CTA issues `iters` x (K/32) MMAs of M=128 x N x K=32 on resident operands
template <int NN>
__global__ void k_rate(int iters, int a_mn, unsigned long long* cyc) {
  extern __shared__ __align__(1024) int8_t sm[];
  int8_t* sA = sm;                 // 128 x 256 K
  int8_t* sB = sm + M * 256;       // NN x 256 K
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + NN) * 256; i += blockDim.x) sm[i] = (int8_t)((i * 7) & 63);
  if (tid == 0) mbar_init(&bar, 1);
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  unsigned long long c0 = clock64();
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, NN, a_mn, 0);
    for (int it = 0; it < iters; ++it)
      for (int s = 0; s < 8; ++s) {
        const uint64_t da = a_mn ? sdesc(sA + s * 4 * 128, 128, 32 * 128) : sdesc(sA + s * 2 * 16 * 128, 16 * 128, 128);
        const uint64_t db = sdesc(sB + s * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
        mma_i8(t0 + (uint32_t)((it & 1) * 256), da, db, id, it > 1 || s > 0);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  unsigned long long c1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(t0, 512);
}

int main() {
  // (1) exactness
  std::vector<int8_t> A(M * KD), B(N * KD);
  srand(1);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  std::vector<int32_t> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t s = 0;
      for (int k = 0; k < KD; ++k) s += (int32_t)A[m * KD + k] * B[n * KD + k];
      ref[m * N + n] = s;
    }
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, ref.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  for (int a_mn = 0; a_mn < 2; ++a_mn) {
    CK(cudaMemset(dD, 0x55, ref.size() * 4));
    k_check<<<1, 128>>>(dA, dB, dD, a_mn);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(ref.size());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (size_t i = 0; i < D.size(); ++i) bad += D[i] != ref[i];
    printf("{\"check\": \"%s\", \"mismatches\": %d, \"d00\": %d, \"ref00\": %d}\n", a_mn ? "A MN-major" : "A K-major", bad,
           D[0], ref[0]);
  }
  // (2) rate
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, sms * 8));
  auto run = [&](auto kern, int NN, int a_mn) {
    const size_t smem = (size_t)(M + NN) * 256;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int iters = 4000;
    kern<<<sms, 128, smem>>>(10, a_mn, dc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<sms, 128, smem>>>(iters, a_mn, dc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * M * NN * 256.0 * iters * sms;
    std::vector<unsigned long long> c(sms);
    CK(cudaMemcpy(c.data(), dc, sms * 8, cudaMemcpyDeviceToHost));
    printf("{\"rate\": \"M128 N%d K32 %s\", \"ms\": %.3f, \"tops\": %.1f, \"cycles_per_mma\": %.1f}\n", NN,
           a_mn ? "A MN" : "A K", ms, ops / ms / 1e9, (double)c[0] / (iters * 8.0));
  };
  run(k_rate<256>, 256, 0);
  run(k_rate<256>, 256, 1);
  run(k_rate<128>, 128, 0);
  run(k_rate<96>, 96, 0);
  run(k_rate<96>, 96, 1);
  run(k_rate<8>, 8, 0);
  return 0;
}
