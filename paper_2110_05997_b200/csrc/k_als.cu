// Kernels of the CP-ALS sweep (NEXT #4, Alg. ALS) that are not GEMMs: the Khatri–Rao
// product chunk of Thm unfolding-formula2's reversed order (KR def 4780-4786) and the
// pseudo-inverse of the symmetric R x R Hadamard product of Grams (Thm special-products 11-12, 4815-4816)
// from its eigen-decomposition.
#include "../../include/tf.h"
#include "tf_device.cuh"
#include "tf_internal.h"

namespace tfk {

// KR[(y + ny*(x - x0)), r] = X[x, r] * Y[y, r] for x in [x0, x0 + xn): the rows of X ⊙ Y for a chunk of x
// (column-major, leading dimension ny*xn). X is nx x R (ld nx), Y is ny x R (ld ny).
__global__ void k_khatri_rao(int64_t nx, const double* __restrict__ X, int64_t x0, int64_t xn, int64_t ny,
                             const double* __restrict__ Y, int64_t R, double* __restrict__ KR) {
  const int64_t rows = ny * xn;
  const int64_t total = rows * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rows, row = e % rows;
    const int64_t y = row % ny, x = x0 + row / ny;
    KR[e] = X[x + nx * r] * Y[y + ny * r];
  }
}

// out = Q diag(theta_r^dagger) Q^T with theta^dagger = 1/theta if |theta| > 1e-15 max|theta| else 0
// (numpy.linalg.pinv's rule, reading R30); theta sorted by |theta| decreasing (k_jacobi_eig).
__global__ void k_pinv_from_eig(int R, const double* __restrict__ Q, const double* __restrict__ theta,
                                double* __restrict__ out) {
  const double cut = 1e-15 * fabs(theta[0]);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * R; e += gridDim.x * blockDim.x) {
    const int a = e % R, b = e / R;
    double s = 0.0;
    for (int r = 0; r < R; ++r) {
      const double t = theta[r];
      if (fabs(t) > cut) s += Q[a + R * r] * Q[b + R * r] / t;
    }
    out[e] = s;
  }
}

cudaError_t launch_khatri_rao(int64_t nx, const double* X, int64_t x0, int64_t xn, int64_t ny, const double* Y,
                              int64_t R, double* KR, cudaStream_t st) {
  const int64_t total = ny * xn * R;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_khatri_rao<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(nx, X, x0, xn, ny, Y, R, KR);
  return cudaGetLastError();
}

cudaError_t launch_pinv_from_eig(int R, const double* Q, const double* theta, double* out, cudaStream_t st) {
  k_pinv_from_eig<<<(R * R + 255) / 256, 256, 0, st>>>(R, Q, theta, out);
  return cudaGetLastError();
}

}  // namespace tfk
