// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// FP64 tensor-core (DMMA via mma.sync.m8n8k4.f64), FP64 FMA (DFMA) and read-only HBM bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
  double x[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) x[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// DMMA with a 4 x 2 fragment tile per warp (distinct A and B operand registers, 8 accumulators), the
// pattern of the fused kernel's phase 1; operands are perturbed every iteration so nothing is hoisted.
__global__ void k_dmma_tile(double* out, int iters) {
  double a[4], b[2], c[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) c[m][n][0] = c[m][n][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 2; ++n)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[m][n][0]), "+d"(c[m][n][1]) : "d"(a[m]), "d"(b[n]));
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __longlong_as_double(__double_as_longlong(a[i]) ^ 1);
  }
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) s += c[m][n][0] + c[m][n][1];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA interleaved in one warp: if the two share the FP64 datapath the mix is no faster
// than the sum of the parts.
template <int NACC, int NF>
__global__ void k_mix(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC > 0 ? NACC : 1][2];
  double x[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
#pragma unroll
  for (int i = 0; i < NF; ++i) x[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_read(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int nsm = pr.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d", pr.name, nsm);
  // DMMA sweep over warps per SM and accumulator chains
  double best_dmma = 0;
  for (int tpb : {128, 256, 512, 1024}) {
    for (int blocks_per_sm : {1, 2}) {
      int iters = 4000;
      dim3 g(nsm * blocks_per_sm), b(tpb);
      k_dmma<8><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      k_dmma<8><<<g, b>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * 256 * 8 * (double)iters * (g.x * (tpb / 32));
      double tf = flops / (ms * 1e-3) / 1e12;
      printf(", \"dmma_tpb%d_bps%d_tflops\": %.2f", tpb, blocks_per_sm, tf);
      if (tf > best_dmma) best_dmma = tf;
    }
  }
  for (int tpb : {256, 512}) {
    int iters = 4000; dim3 g(nsm), b(tpb);
    k_dmma_tile<<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_dmma_tile<<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 256 * 8 * (double)iters * (g.x * (tpb / 32));
    double tf = flops / (ms * 1e-3) / 1e12;
    printf(", \"dmma_tile4x2_tpb%d_tflops\": %.2f", tpb, tf);
    if (tf > best_dmma) best_dmma = tf;
  }
  // DMMA single-warp-per-SMSP chain latency probe: 1 acc chain, 4 warps per SM
  {
    int iters = 20000; dim3 g(nsm), b(128);
    k_dmma<1><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_dmma<1><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double ns_per = ms * 1e6 / iters;
    printf(", \"dmma_dep_chain_ns\": %.3f", ns_per);
    k_dmma<2><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_dmma<2><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf(", \"dmma_2chain_ns_per_iter\": %.3f", ms * 1e6 / iters);
    k_dmma<4><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_dmma<4><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf(", \"dmma_4chain_ns_per_iter\": %.3f", ms * 1e6 / iters);
  }
  {
    // mix: per iteration 8 DMMA (8 x 256 FMA per warp) and/or 32 DFMA per thread (32 x 32 FMA per warp)
    int iters = 4000; dim3 g(nsm), b(256);
    float t_d, t_f, t_m;
    k_mix<8, 0><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_mix<8, 0><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&t_d, e0, e1));
    k_mix<0, 32><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_mix<0, 32><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&t_f, e0, e1));
    k_mix<8, 32><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); k_mix<8, 32><<<g, b>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&t_m, e0, e1));
    printf(", \"mix_dmma_only_ms\": %.3f, \"mix_dfma_only_ms\": %.3f, \"mix_both_ms\": %.3f", t_d, t_f, t_m);
  }
  double best_dfma = 0;
  for (int tpb : {256, 512, 1024}) {
    for (int blocks_per_sm : {1, 2}) {
      int iters = 20000;
      dim3 g(nsm * blocks_per_sm), b(tpb);
      k_dfma<8><<<g, b>>>(out, 10); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      k_dfma<8><<<g, b>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * 8 * (double)iters * g.x * tpb;
      double tf = flops / (ms * 1e-3) / 1e12;
      printf(", \"dfma_tpb%d_bps%d_tflops\": %.2f", tpb, blocks_per_sm, tf);
      if (tf > best_dfma) best_dfma = tf;
    }
  }
  // read-only HBM bandwidth over 8 GiB
  size_t bytes = (size_t)8 << 30; size_t n4 = bytes / sizeof(double2);
  double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  double best_bw = 0;
  for (int bps : {2, 4, 8}) {
    dim3 g(nsm * bps), b(512);
    k_read<<<g, b>>>(buf, n4, out); CK(cudaDeviceSynchronize());
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0)); k_read<<<g, b>>>(buf, n4, out); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = bytes / (ms * 1e-3) / 1e9;
      if (gbs > best_bw) best_bw = gbs;
    }
  }
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf(", \"sm_clock_attr_mhz\": %d", clk_khz / 1000);
  printf(", \"best_dmma_tflops\": %.2f, \"best_dfma_tflops\": %.2f, \"read_hbm_gbs\": %.1f}\n", best_dmma, best_dfma, best_bw);
  CK(cudaFree(buf));
  return 0;
}
