// cuBLAS DGEMM reference point for the FP64 roofline: C = A B with A, B, C n x n fp64,
// timed with CUDA events after warm-up; prints TFLOP/s. nvcc -O3 -o dgemm_ref dgemm_ref.cu -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 8192;
  const int reps = argc > 2 ? atoi(argv[2]) : 10;
  double *A, *B, *C;
  cudaMalloc(&A, (size_t)n * n * 8);
  cudaMalloc(&B, (size_t)n * n * 8);
  cudaMalloc(&C, (size_t)n * n * 8);
  std::vector<double> h((size_t)n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cublasHandle_t hd;
  cublasCreate(&hd);
  const double one = 1.0, zero = 0.0;
  for (int i = 0; i < 3; ++i) cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tf = 2.0 * n * (double)n * n * reps / (ms * 1e-3) / 1e12;
  printf("{\"cublas_dgemm_n\": %d, \"ms_per_gemm\": %.3f, \"tflops\": %.2f}\n", n, ms / reps, tf);
  cublasDestroy(hd);
  return 0;
}
