/*
 * oracle.c -- plain, slow, obviously-correct CPU reference for the dGN
 * evaluation hot path of Tensor Fox (arxiv 2110.05997, PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2110_05997_b200/csrc) and never calls it.
 *
 * Conventions (PAPER.md:857-872 Alg. Unfolding; 1466-1473 vec/w layout):
 *   T[i + I*(j + J*k)]   first index fastest; frontal slice k contiguous.
 *   A[i + I*r], B[j + J*r], C[k + K*r]   column-major factor matrices.
 *   w = [vec A; vec B; vec C], length n = R*(I+J+K).
 *
 * Arithmetic: every accumulation and every intermediate is carried in x86
 * 80-bit `long double` (64-bit significand), so the oracle's own rounding
 * (~1e-19 relative per operation) is far below the 1e-10 parity bar and any
 * parity gap is attributable to the fp64 GPU path (R15).
 *
 * Pinning status of every function is listed in DESIGN.md §3 and tested in
 * tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;

static int clamp_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  return nthreads;
#else
  (void)nthreads;
  return 1;
#endif
}

/*
 * oracle_eval: F(w) and grad F(w) by their definitions.
 *   residual  f_ijk = t_ijk - sum_r a_ir b_jr c_kr        (eq. residual_function)
 *   objective F = 1/2 sum_ijk f_ijk^2                      (eq. error_function)
 *   gradient  grad F = J_f^T f                             (Lemma gradF)
 *             with d f_ijk / d a_ir = -b_jr c_kr, etc.     (Lemma partialf)
 * One pass over the entries in storage order; slices k are split over
 * OpenMP threads (static schedule), per-thread partial sums of gA, gB and F
 * are combined in thread order, so the result is deterministic for a fixed
 * thread count. gC row k is owned by the thread that owns slice k.
 */
int oracle_eval(int64_t I, int64_t J, int64_t K, int64_t R, const double *T,
                const double *A, const double *B, const double *C,
                double *f_out, double *gA, double *gB, double *gC, int nthreads) {
  if (I < 1 || J < 1 || K < 1 || R < 1 || !T || !A || !B || !C) return 1;
  int nt = clamp_threads(nthreads);
  ld *pA = (ld *)calloc((size_t)nt * I * R, sizeof(ld));
  ld *pB = (ld *)calloc((size_t)nt * J * R, sizeof(ld));
  ld *pF = (ld *)calloc((size_t)nt, sizeof(ld));
  ld *gCl = (ld *)calloc((size_t)K * R, sizeof(ld));
  if (!pA || !pB || !pF || !gCl) { free(pA); free(pB); free(pF); free(gCl); return 6; }

#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int tid = omp_get_thread_num();
#else
    int tid = 0;
#endif
    ld *myA = pA + (size_t)tid * I * R;
    ld *myB = pB + (size_t)tid * J * R;
    ld myF = 0.0L;
    ld *bc = (ld *)malloc(sizeof(ld) * R);
#pragma omp for schedule(static)
    for (int64_t k = 0; k < K; ++k) {
      for (int64_t j = 0; j < J; ++j) {
        for (int64_t r = 0; r < R; ++r) bc[r] = (ld)B[j + J * r] * (ld)C[k + K * r];
        for (int64_t i = 0; i < I; ++i) {
          /* residual f_ijk (eq. residual_function) */
          ld x = 0.0L;
          for (int64_t r = 0; r < R; ++r) x += (ld)A[i + I * r] * bc[r];
          ld e = (ld)T[i + I * (j + J * k)] - x;
          myF += e * e;
          /* J_f^T f, column by column (Lemma partialf) */
          for (int64_t r = 0; r < R; ++r) {
            myA[i + I * r] -= e * bc[r];
            myB[j + J * r] -= e * (ld)A[i + I * r] * (ld)C[k + K * r];
            gCl[k + K * r] -= e * (ld)A[i + I * r] * (ld)B[j + J * r];
          }
        }
      }
    }
    pF[tid] = myF;
    free(bc);
  }
  ld F = 0.0L;
  for (int t = 0; t < nt; ++t) F += pF[t];
  *f_out = (double)(0.5L * F);
  for (int64_t q = 0; q < I * R; ++q) {
    ld s = 0.0L;
    for (int t = 0; t < nt; ++t) s += pA[(size_t)t * I * R + q];
    gA[q] = (double)s;
  }
  for (int64_t q = 0; q < J * R; ++q) {
    ld s = 0.0L;
    for (int t = 0; t < nt; ++t) s += pB[(size_t)t * J * R + q];
    gB[q] = (double)s;
  }
  for (int64_t q = 0; q < K * R; ++q) gC[q] = (double)gCl[q];
  free(pA); free(pB); free(pF); free(gCl);
  return 0;
}

/*
 * oracle_slice_eval: the same definitions restricted to the entries that
 * share one fixed index, i.e. one slice of T (PAPER.md:401-416 slice defs;
 * 579-586 slice formulas). For the fixed index with factor row x (length R)
 * and the slice S (n1 x n2, column-major, S[a + n1*b]) with the other two
 * factor matrices X (n1 x R) and Y (n2 x R):
 *   e_ab = s_ab - sum_r x_r X_ar Y_br,  f = 1/2 sum e_ab^2,  g_r = -sum_ab e_ab X_ar Y_br.
 * g is the gradient row of the fixed index (row i of dF/dA for a horizontal
 * slice, row j of dF/dB for a lateral one, row k of dF/dC for a frontal one)
 * and f is that slice's share of F. Used for sampled checks at full size.
 */
int oracle_slice_eval(int64_t n1, int64_t n2, int64_t R, const double *S, int64_t lds1, int64_t lds2,
                      const double *x, const double *X, int64_t ldX, const double *Y, int64_t ldY,
                      double *f_out, double *g) {
  /* S element (a,b) lives at S[a*lds1 + b*lds2]; X(a,r) at X[a + ldX*r]; Y(b,r) at Y[b + ldY*r] */
  if (n1 < 1 || n2 < 1 || R < 1) return 1;
  ld *gl = (ld *)calloc((size_t)R, sizeof(ld));
  ld *xy = (ld *)malloc(sizeof(ld) * R);
  ld F = 0.0L;
  for (int64_t b = 0; b < n2; ++b) {
    for (int64_t r = 0; r < R; ++r) xy[r] = (ld)x[r] * (ld)Y[b + ldY * r];
    for (int64_t a = 0; a < n1; ++a) {
      ld v = 0.0L;
      for (int64_t r = 0; r < R; ++r) v += (ld)X[a + ldX * r] * xy[r];
      ld e = (ld)S[a * lds1 + b * lds2] - v;
      F += e * e;
      for (int64_t r = 0; r < R; ++r) gl[r] -= e * (ld)X[a + ldX * r] * (ld)Y[b + ldY * r];
    }
  }
  *f_out = (double)(0.5L * F);
  for (int64_t r = 0; r < R; ++r) g[r] = (double)gl[r];
  free(gl); free(xy);
  return 0;
}

/*
 * oracle_gn_matvec_plain: y = (J_f^T J_f + lambda I) v without Grams.
 *   u = J_f v with (J_f v)_ijk = -sum_r (vA_ir b_jr c_kr + a_ir vB_jr c_kr + a_ir b_jr vC_kr)
 *   (Lemma partialf), then y = J_f^T u + lambda v by the
 *   same column formulas as in oracle_eval. O(IJKR) per call.
 */
int oracle_gn_matvec_plain(int64_t I, int64_t J, int64_t K, int64_t R,
                           const double *A, const double *B, const double *C,
                           const double *v, double lambda, const double *damp, double *y, int nthreads) {
  if (I < 1 || J < 1 || K < 1 || R < 1) return 1;
  const double *vA = v, *vB = v + I * R, *vC = v + (I + J) * R;
  int nt = clamp_threads(nthreads);
  ld *pA = (ld *)calloc((size_t)nt * I * R, sizeof(ld));
  ld *pB = (ld *)calloc((size_t)nt * J * R, sizeof(ld));
  ld *yC = (ld *)calloc((size_t)K * R, sizeof(ld));
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int tid = omp_get_thread_num();
#else
    int tid = 0;
#endif
    ld *myA = pA + (size_t)tid * I * R;
    ld *myB = pB + (size_t)tid * J * R;
#pragma omp for schedule(static)
    for (int64_t k = 0; k < K; ++k)
      for (int64_t j = 0; j < J; ++j)
        for (int64_t i = 0; i < I; ++i) {
          ld u = 0.0L;
          for (int64_t r = 0; r < R; ++r) {
            ld a = A[i + I * r], b = B[j + J * r], c = C[k + K * r];
            u -= (ld)vA[i + I * r] * b * c + a * (ld)vB[j + J * r] * c + a * b * (ld)vC[k + K * r];
          }
          for (int64_t r = 0; r < R; ++r) {
            ld a = A[i + I * r], b = B[j + J * r], c = C[k + K * r];
            myA[i + I * r] -= u * b * c;
            myB[j + J * r] -= u * a * c;
            yC[k + K * r] -= u * a * b;
          }
        }
  }
  for (int64_t q = 0; q < I * R; ++q) {
    ld s = 0.0L;
    for (int t = 0; t < nt; ++t) s += pA[(size_t)t * I * R + q];
    const ld dmp = damp ? (ld)damp[q / I] : 1.0L;
    y[q] = (double)(s + (ld)lambda * dmp * (ld)vA[q]);
  }
  for (int64_t q = 0; q < J * R; ++q) {
    ld s = 0.0L;
    for (int t = 0; t < nt; ++t) s += pB[(size_t)t * J * R + q];
    const ld dmp = damp ? (ld)damp[R + q / J] : 1.0L;
    y[I * R + q] = (double)(s + (ld)lambda * dmp * (ld)vB[q]);
  }
  for (int64_t q = 0; q < K * R; ++q) {
    const ld dmp = damp ? (ld)damp[2 * R + q / K] : 1.0L;
    y[(I + J) * R + q] = (double)(yC[q] + (ld)lambda * dmp * (ld)vC[q]);
  }
  free(pA); free(pB); free(yC);
  return 0;
}

/* pi^(l) = W^(l)T W^(l). grams = [pi_A | pi_B | pi_C], each R x R column-major. */
static void gram_ld(int64_t n, int64_t R, const double *W, ld *out) {
  for (int64_t r = 0; r < R; ++r)
    for (int64_t s = 0; s < R; ++s) {
      ld acc = 0.0L;
      for (int64_t a = 0; a < n; ++a) acc += (ld)W[a + n * r] * (ld)W[a + n * s];
      out[r + R * s] = acc;
    }
}

int oracle_grams(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
                 const double *C, double *grams) {
  ld *g = (ld *)malloc(sizeof(ld) * 3 * R * R);
  gram_ld(I, R, A, g);
  gram_ld(J, R, B, g + R * R);
  gram_ld(K, R, C, g + 2 * R * R);
  for (int64_t q = 0; q < 3 * R * R; ++q) grams[q] = (double)g[q];
  free(g);
  return 0;
}

/*
 * Hadamard chains for L = 3:
 *   Pi^(1) = pi^(2) * pi^(3),  Pi^(2) = pi^(1) * pi^(3),  Pi^(3) = pi^(1) * pi^(2);
 *   Pi^(1,2) = pi^(3),  Pi^(1,3) = pi^(2),  Pi^(2,3) = pi^(1)  (product over l not in {l', l''}).
 * out = [Pi1 | Pi2 | Pi3 | Pi12 | Pi13 | Pi23].
 */
static void pi_ld(int64_t R, const ld *g, ld *out) {
  const ld *pA = g, *pB = g + R * R, *pC = g + 2 * R * R;
  for (int64_t q = 0; q < R * R; ++q) {
    out[q] = pB[q] * pC[q];
    out[R * R + q] = pA[q] * pC[q];
    out[2 * R * R + q] = pA[q] * pB[q];
    out[3 * R * R + q] = pC[q];
    out[4 * R * R + q] = pB[q];
    out[5 * R * R + q] = pA[q];
  }
}

int oracle_pi(int64_t R, const double *grams, double *pi) {
  ld *g = (ld *)malloc(sizeof(ld) * 3 * R * R), *p = (ld *)malloc(sizeof(ld) * 6 * R * R);
  for (int64_t q = 0; q < 3 * R * R; ++q) g[q] = grams[q];
  pi_ld(R, g, p);
  for (int64_t q = 0; q < 6 * R * R; ++q) pi[q] = (double)p[q];
  free(g); free(p);
  return 0;
}

/*
 * Thm Hv: for each mode l',
 *   Y^(l') = V^(l') Pi^(l') + sum_{l'' != l'} W^(l') (Pi^(l',l'') * (V^(l'')T W^(l'')))
 * then y = vec(Y) + lambda v. Written with explicit loops in the theorem's order.
 */
static void hv_ld(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
                  const double *C, const ld *v, ld lambda, const double *damp, ld *y) {
  const int64_t dims[3] = {I, J, K};
  const double *W[3] = {A, B, C};
  int64_t off[3] = {0, I * R, (I + J) * R};
  ld *g = (ld *)malloc(sizeof(ld) * 3 * R * R), *pi = (ld *)malloc(sizeof(ld) * 6 * R * R);
  gram_ld(I, R, A, g);
  gram_ld(J, R, B, g + R * R);
  gram_ld(K, R, C, g + 2 * R * R);
  pi_ld(R, g, pi);
  /* index of Pi^(l',l'') in pi[] for l' != l'' */
  int pair_idx[3][3] = {{-1, 3, 4}, {3, -1, 5}, {4, 5, -1}};
  ld *M = (ld *)malloc(sizeof(ld) * R * R);
  for (int l1 = 0; l1 < 3; ++l1) {
    int64_t n1 = dims[l1];
    const ld *P1 = pi + (int64_t)l1 * R * R;
    const ld *V1 = v + off[l1];
    ld *Y = y + off[l1];
    /* Case 2: V^(l') Pi^(l') */
    for (int64_t a = 0; a < n1; ++a)
      for (int64_t s = 0; s < R; ++s) {
        ld acc = 0.0L;
        for (int64_t r = 0; r < R; ++r) acc += V1[a + n1 * r] * P1[r + R * s];
        const ld dmp = damp ? (ld)damp[l1 * R + s] : 1.0L;  /* (J^T J + lambda D) v, D = diag(damp) */
        Y[a + n1 * s] = acc + lambda * dmp * V1[a + n1 * s];
      }
    /* Case 1: W^(l') (Pi^(l',l'') * (V^(l'')T W^(l''))) */
    for (int l2 = 0; l2 < 3; ++l2) {
      if (l2 == l1) continue;
      int64_t n2 = dims[l2];
      const ld *V2 = v + off[l2];
      const double *W2 = W[l2];
      const ld *P12 = pi + (int64_t)pair_idx[l1][l2] * R * R;
      for (int64_t r = 0; r < R; ++r)
        for (int64_t s = 0; s < R; ++s) {
          ld acc = 0.0L; /* (V2^T W2)_{rs} */
          for (int64_t b = 0; b < n2; ++b) acc += V2[b + n2 * r] * (ld)W2[b + n2 * s];
          M[r + R * s] = P12[r + R * s] * acc;
        }
      const double *W1 = W[l1];
      for (int64_t a = 0; a < n1; ++a)
        for (int64_t s = 0; s < R; ++s) {
          ld acc = 0.0L;
          for (int64_t r = 0; r < R; ++r) acc += (ld)W1[a + n1 * r] * M[r + R * s];
          Y[a + n1 * s] += acc;
        }
    }
  }
  free(g); free(pi); free(M);
}

int oracle_gn_matvec_hv(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
                        const double *C, const double *v, double lambda, const double *damp, double *y) {
  int64_t n = R * (I + J + K);
  ld *vl = (ld *)malloc(sizeof(ld) * n), *yl = (ld *)malloc(sizeof(ld) * n);
  for (int64_t q = 0; q < n; ++q) vl[q] = v[q];
  hv_ld(I, J, K, R, A, B, C, vl, (ld)lambda, damp, yl);
  for (int64_t q = 0; q < n; ++q) y[q] = (double)yl[q];
  free(vl); free(yl);
  return 0;
}

/*
 * Diagonal regularizer of Tensor Fox (Section "Diagonal regularization"), L = 3:
 *   G = max{ max_r' ||Y_r'|| ||Z_r'||, max_r' ||X_r'|| ||Z_r'||, max_r' ||X_r'|| ||Y_r'|| }
 *   gamma_X^(r) = ||Y_r|| ||Z_r|| G,  gamma_Y^(r) = ||X_r|| ||Z_r|| G,  gamma_Z^(r) = ||X_r|| ||Y_r|| G
 * with X, Y, Z = A, B, C and ||.|| the 2-norm of a factor column. gamma = [gX | gY | gZ], 3R values;
 * D = diag(gamma_l^(r) I_{I_l}) in w-layout.
 */
int oracle_reg_gamma(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B, const double *C,
                     double *gamma) {
  const int64_t dims[3] = {I, J, K};
  const double *W[3] = {A, B, C};
  ld *nrm = (ld *)malloc(sizeof(ld) * 3 * R);
  for (int l = 0; l < 3; ++l)
    for (int64_t r = 0; r < R; ++r) {
      ld s = 0.0L;
      for (int64_t a = 0; a < dims[l]; ++a) s += (ld)W[l][a + dims[l] * r] * (ld)W[l][a + dims[l] * r];
      nrm[l * R + r] = sqrtl(s);
    }
  ld G = 0.0L;
  for (int64_t r = 0; r < R; ++r) {
    const ld yz = nrm[R + r] * nrm[2 * R + r], xz = nrm[r] * nrm[2 * R + r], xy = nrm[r] * nrm[R + r];
    if (yz > G) G = yz;
    if (xz > G) G = xz;
    if (xy > G) G = xy;
  }
  for (int64_t r = 0; r < R; ++r) {
    gamma[r] = (double)(nrm[R + r] * nrm[2 * R + r] * G);
    gamma[R + r] = (double)(nrm[r] * nrm[2 * R + r] * G);
    gamma[2 * R + r] = (double)(nrm[r] * nrm[R + r] * G);
  }
  free(nrm);
  return 0;
}

/*
 * Diagonal of J_f^T J_f: entry (l, a, r) is the squared norm of the Jacobian
 * column d f / d w^(l)_{a r}, whose nonzeros are -prod_{l != l'} w (Lemma
 * partialf), i.e. prod_{l != l'} ||w_r^(l)||^2 (= Pi^(l)_rr).
 */
static void jtj_diag_ld(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
                        const double *C, ld *d) {
  const int64_t dims[3] = {I, J, K};
  const double *W[3] = {A, B, C};
  ld *nrm = (ld *)malloc(sizeof(ld) * 3 * R);
  for (int l = 0; l < 3; ++l)
    for (int64_t r = 0; r < R; ++r) {
      ld s = 0.0L;
      for (int64_t a = 0; a < dims[l]; ++a) s += (ld)W[l][a + dims[l] * r] * (ld)W[l][a + dims[l] * r];
      nrm[l * R + r] = s;
    }
  const int64_t off[3] = {0, I * R, (I + J) * R};
  for (int l = 0; l < 3; ++l)
    for (int64_t r = 0; r < R; ++r) {
      ld p = 1.0L;
      for (int m = 0; m < 3; ++m) if (m != l) p *= nrm[m * R + r];
      for (int64_t a = 0; a < dims[l]; ++a) d[off[l] + a + dims[l] * r] = p;
    }
  free(nrm);
}

int oracle_jtj_diag(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
                    const double *C, double *d) {
  int64_t n = R * (I + J + K);
  ld *dl = (ld *)malloc(sizeof(ld) * n);
  jtj_diag_ld(I, J, K, R, A, B, C, dl);
  for (int64_t q = 0; q < n; ++q) d[q] = (double)dl[q];
  free(dl);
  return 0;
}

/*
 * Alg. CG-dGN with damping lambda*D (D = diag(damp) per (mode, r); damp = NULL
 * is D = I, the north star's lambda*I, reading R2) and M = I (jacobi = 0) or
 * M = diag(J^T J) + lambda diag(D) (jacobi = 1):
 *   B = M^{-1/2} (J^T J + lambda D) M^{-1/2};  x0 = 0;  r0 = M^{-1/2} rhs;  p0 = r0
 *   for i = 1..maxiter:
 *     z = B p;  alpha = ||r||^2 / <p, z>;  x += alpha p;  r -= alpha z;
 *     eps = ||r||^2;  beta = eps / ||r_old||^2;  p = r + beta p;  if eps < tol: break
 * Returns x in w-coordinates, x = M^{-1/2} x_hat (reading R3).
 * x_hist (nullable): maxiter*n, the iterate after each iteration (w-coordinates);
 * r2/alpha/beta (nullable): per-iteration ||r||^2, alpha, beta. *iters = iterations done.
 * Returns 5 if alpha or beta is not finite.
 */
int oracle_cg(int64_t I, int64_t J, int64_t K, int64_t R, const double *A, const double *B,
              const double *C, const double *rhs, double lambda, const double *damp, int maxiter, double tol,
              int jacobi,
              double *x_out, double *x_hist, double *r2_hist, double *alpha_hist, double *beta_hist,
              int *iters) {
  int64_t n = R * (I + J + K);
  ld *x = (ld *)calloc(n, sizeof(ld)), *r = (ld *)malloc(sizeof(ld) * n), *p = (ld *)malloc(sizeof(ld) * n);
  ld *z = (ld *)malloc(sizeof(ld) * n), *tmp = (ld *)malloc(sizeof(ld) * n), *minv = (ld *)malloc(sizeof(ld) * n);
  int status = 0;
  if (jacobi) {
    /* M = diag(J^T J) + lambda diag(D) */
    jtj_diag_ld(I, J, K, R, A, B, C, minv);
    const int64_t dims[3] = {I, J, K}, off[3] = {0, I * R, (I + J) * R};
    for (int l = 0; l < 3; ++l)
      for (int64_t r = 0; r < R; ++r)
        for (int64_t a = 0; a < dims[l]; ++a) {
          const int64_t q = off[l] + a + dims[l] * r;
          const ld dmp = damp ? (ld)damp[l * R + r] : 1.0L;
          minv[q] = 1.0L / sqrtl(minv[q] + (ld)lambda * dmp);
        }
  } else {
    for (int64_t q = 0; q < n; ++q) minv[q] = 1.0L;
  }
  ld rr = 0.0L;
  for (int64_t q = 0; q < n; ++q) { r[q] = minv[q] * (ld)rhs[q]; p[q] = r[q]; rr += r[q] * r[q]; }
  int it = 0;
  /* reading R33: r^(0) = 0 (rhs = 0) is already solved by x^(0) = 0; the loop as printed would divide 0 by 0 */
  if (rr == 0.0L) maxiter = 0;
  for (int i = 1; i <= maxiter; ++i) {
    /* z = B p in three steps */
    for (int64_t q = 0; q < n; ++q) tmp[q] = minv[q] * p[q];
    hv_ld(I, J, K, R, A, B, C, tmp, (ld)lambda, damp, z);
    for (int64_t q = 0; q < n; ++q) z[q] *= minv[q];
    ld pz = 0.0L;
    for (int64_t q = 0; q < n; ++q) pz += p[q] * z[q];
    ld alpha = rr / pz;
    if (!isfinite((double)alpha)) { status = 5; break; }
    ld rr_new = 0.0L;
    for (int64_t q = 0; q < n; ++q) {
      x[q] += alpha * p[q];
      r[q] -= alpha * z[q];
      rr_new += r[q] * r[q];
    }
    ld beta = rr_new / rr;
    if (!isfinite((double)beta)) { status = 5; break; }
    for (int64_t q = 0; q < n; ++q) p[q] = r[q] + beta * p[q];
    rr = rr_new;
    it = i;
    if (x_hist) for (int64_t q = 0; q < n; ++q) x_hist[(int64_t)(i - 1) * n + q] = (double)(minv[q] * x[q]);
    if (r2_hist) r2_hist[i - 1] = (double)rr_new;
    if (alpha_hist) alpha_hist[i - 1] = (double)alpha;
    if (beta_hist) beta_hist[i - 1] = (double)beta;
    if (rr_new < (ld)tol) break;
  }
  for (int64_t q = 0; q < n; ++q) x_out[q] = (double)(minv[q] * x[q]);
  if (iters) *iters = it;
  free(x); free(r); free(p); free(z); free(tmp); free(minv);
  return status;
}

/*
 * ---- NEXT #2: the damped Gauss-Newton outer loop of Tensor Fox, step by step.
 * Per iteration k = 1..maxiter (the initial F, grad at w^(0) are evaluated first):
 *   gamma_k from w^(k-1) if use_gamma, else D = I
 *   x = CG-dGN on (J^T J + mu D) x = -grad F(w^(k-1)), cg_iters[k-1] iterations, tolerance tol,
 *       Jacobi M = diag(J^T J) + mu diag(D) if jacobi
 *   w^(k) = w^(k-1) + x
 *   norm balancing: for each r, every mode's column gets norm (prod_l ||w_r^(l)||)^(1/3)
 *   F(w^(k)); gain ratio g = (F(w^(k-1)) - F(w^(k))) / (F(w^(k-1)) - 1/2 ||f~||^2),
 *       f~ = f(w^(k-1)) + J_f(w^(k-1)) x, evaluated entry by entry (reading R19)
 *   damping: g < 0.25 -> mu = 3 mu; g > 0.75 -> mu = mu / 3
 *   stopping conditions 1-7 in the paper's order (readings R20-R22)
 * mu^(0) = mu0 if mu0 > 0 else tau * mean|T| with tau = 1.
 * hist (nullable): per iteration [F, rel_err, mu used, g, ||x||]. Returns the stop reason (0 = maxiter,
 * 1..7 = condition, 8 = non-finite) in *reason and the iterations done in *iters.
 */
static ld linearized_half_sq(int64_t I, int64_t J, int64_t K, int64_t R, const double *T, const double *A,
                             const double *B, const double *C, const double *x) {
  const double *xA = x, *xB = x + I * R, *xC = x + (I + J) * R;
  ld s = 0.0L;
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < J; ++j)
      for (int64_t i = 0; i < I; ++i) {
        ld rec = 0.0L, jx = 0.0L;
        for (int64_t r = 0; r < R; ++r) {
          const ld a = A[i + I * r], b = B[j + J * r], c = C[k + K * r];
          rec += a * b * c;
          jx -= (ld)xA[i + I * r] * b * c + a * (ld)xB[j + J * r] * c + a * b * (ld)xC[k + K * r];
        }
        const ld ft = ((ld)T[i + I * (j + J * k)] - rec) + jx;   /* f~ = f + J x (Lemma partialf) */
        s += ft * ft;
      }
  return 0.5L * s;
}

/*
 * The stopping conditions of the dGN loop, checked at iteration k >= 1 in the paper's
 * order; returns the first that holds (1..7) or 0. rel[0..k] = ||S - S^(k)|| / ||S|| (relative errors after
 * 0..k iterations), step = ||w^(k-1) - w^(k)|| (reading R20: the Gauss-Newton step x before balancing),
 * ginf = ||grad F(w^(k))||_inf, nT2 = ||T||^2.
 *   1 relative error          rel[k] < tol
 *   2 step size               step < tol
 *   3 rel. error improvement  |rel[k-1] - rel[k]| < tol
 *   4 gradient norm           ginf < tol
 *   5 average error           mean(rel over [k-2c, k-c)) - mean(rel over [k-c, k)) < tol
 *   6 average improvement     (1/c) sum_{t in [k-c, k)} |rel[t] - rel[t+1]| < 1e-3 (1/c) sum_{t in [k-c, k)} rel[t]
 *     (5 and 6 only when k > 2c and k = 0 mod c, c = 1 + ceil(maxiter / 10); reading R21)
 *   7 divergence              rel[k] > max(1, ||T||^2) / (1e-16 + tol)
 */
int oracle_dgn_stop(int k, const double *rel, int maxiter, double tol, double step, double ginf, double nT2) {
  const int c = 1 + (maxiter + 9) / 10;   /* c = 1 + ceil(maxiter / 10) */
  if (rel[k] < tol) return 1;
  if (step < tol) return 2;
  if (fabs(rel[k - 1] - rel[k]) < tol) return 3;
  if (ginf < tol) return 4;
  if (k > 2 * c && k % c == 0) {
    ld m1 = 0.0L, m2 = 0.0L, imp = 0.0L;
    for (int t = k - 2 * c; t < k - c; ++t) m1 += rel[t];
    for (int t = k - c; t < k; ++t) { m2 += rel[t]; imp += fabsl((ld)rel[t] - (ld)rel[t + 1]); }
    m1 /= c; m2 /= c; imp /= c;
    if (m1 - m2 < (ld)tol) return 5;
    if (imp < 1e-3L * m2) return 6;
  }
  if ((ld)rel[k] > ((ld)nT2 > 1.0L ? (ld)nT2 : 1.0L) / (1e-16L + (ld)tol)) return 7;
  return 0;
}

int oracle_dgn(int64_t I, int64_t J, int64_t K, int64_t R, const double *T, double *w, int maxiter, double tol,
               double mu0, int use_gamma, int jacobi, int balance, const int *cg_iters, int *iters, int *reason,
               double *f_out, double *hist, int nthreads) {
  const int64_t n = R * (I + J + K), N = I * J * K;
  double *grad = (double *)malloc(sizeof(double) * n), *x = (double *)malloc(sizeof(double) * n);
  double *gam = (double *)malloc(sizeof(double) * 3 * R), *wprev = (double *)malloc(sizeof(double) * n);
  double *rel = (double *)malloc(sizeof(double) * (maxiter + 1));
  ld nT2 = 0.0L, sabs = 0.0L;
  for (int64_t q = 0; q < N; ++q) {
    nT2 += (ld)T[q] * (ld)T[q];
    sabs += fabsl((ld)T[q]);
  }
  const ld normT = sqrtl(nT2);
  ld mu = mu0 > 0 ? (ld)mu0 : sabs / (ld)N;
  double F;
  double *gA = grad, *gB = grad + I * R, *gC = grad + (I + J) * R;
  oracle_eval(I, J, K, R, T, w, w + I * R, w + (I + J) * R, &F, gA, gB, gC, nthreads);
  rel[0] = (double)(sqrtl(2.0L * (ld)F) / normT);
  int it = 0, why = 0;
  for (int k = 1; k <= maxiter; ++k) {
    const double *A = w, *B = w + I * R, *C = w + (I + J) * R;
    if (use_gamma) oracle_reg_gamma(I, J, K, R, A, B, C, gam);
    double *rhs = (double *)malloc(sizeof(double) * n);
    for (int64_t q = 0; q < n; ++q) rhs[q] = -grad[q];
    int cgit = 0;
    int st = oracle_cg(I, J, K, R, A, B, C, rhs, (double)mu, use_gamma ? gam : NULL, cg_iters[k - 1], tol, jacobi, x,
                       NULL, NULL, NULL, NULL, &cgit);
    free(rhs);
    if (st) { why = 8; break; }
    const ld pred = (ld)F - linearized_half_sq(I, J, K, R, T, A, B, C, x);   /* predicted decrease */
    ld step2 = 0.0L;
    for (int64_t q = 0; q < n; ++q) {
      wprev[q] = w[q];
      w[q] = (double)((ld)w[q] + (ld)x[q]);
      step2 += (ld)x[q] * (ld)x[q];
    }
    if (balance) {
      const int64_t dims[3] = {I, J, K}, off[3] = {0, I * R, (I + J) * R};
      for (int64_t r = 0; r < R; ++r) {
        ld nr[3], prod = 1.0L;
        for (int l = 0; l < 3; ++l) {
          ld s = 0.0L;
          for (int64_t a = 0; a < dims[l]; ++a) s += (ld)w[off[l] + a + dims[l] * r] * (ld)w[off[l] + a + dims[l] * r];
          nr[l] = sqrtl(s);
          prod *= nr[l];
        }
        if (prod == 0.0L) continue;
        const ld alpha = cbrtl(prod);
        for (int l = 0; l < 3; ++l) {
          const ld sc = alpha / nr[l];
          for (int64_t a = 0; a < dims[l]; ++a) w[off[l] + a + dims[l] * r] = (double)((ld)w[off[l] + a + dims[l] * r] * sc);
        }
      }
    }
    double Fn;
    oracle_eval(I, J, K, R, T, w, w + I * R, w + (I + J) * R, &Fn, gA, gB, gC, nthreads);
    const ld g = ((ld)F - (ld)Fn) / pred;
    if (hist) {
      hist[5 * (k - 1) + 0] = Fn;
      hist[5 * (k - 1) + 1] = (double)(sqrtl(2.0L * (ld)Fn) / normT);
      hist[5 * (k - 1) + 2] = (double)mu;
      hist[5 * (k - 1) + 3] = (double)g;
      hist[5 * (k - 1) + 4] = (double)sqrtl(step2);
    }
    if (g < 0.25L) mu *= 3.0L;
    else if (g > 0.75L) mu /= 3.0L;
    F = Fn;
    it = k;
    rel[k] = (double)(sqrtl(2.0L * (ld)F) / normT);
    if (!isfinite(F)) { why = 8; break; }
    ld ginf = 0.0L;
    for (int64_t q = 0; q < n; ++q) if (fabsl((ld)grad[q]) > ginf) ginf = fabsl((ld)grad[q]);
    why = oracle_dgn_stop(k, rel, maxiter, tol, (double)sqrtl(step2), (double)ginf, (double)nT2);
    if (why) break;
  }
  if (iters) *iters = it;
  if (reason) *reason = why;
  if (f_out) *f_out = F;
  free(grad); free(x); free(gam); free(wprev); free(rel);
  return 0;
}
