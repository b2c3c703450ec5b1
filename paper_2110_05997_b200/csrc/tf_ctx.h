// Host-side context of the C ABI (include/tf.h) and the helpers every host translation unit uses.
#pragma once
#include <string>
#include <vector>

#include "../../include/tf.h"
#include "tf_internal.h"

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct tf_ctx;
inline int cg_grid(const tf_ctx* c);

struct tf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nsm = 148;
  std::string err;
  DevBuf gAp, gBp, gCp, fp;                 // eval partials
  DevBuf gram_part;                         // Gram split-K partials
  DevBuf mvG, mvS, mvPi, mvD, mvPart;       // matvec / CG scratch
  DevBuf cgR, cgP, cgZ, cgState;            // CG vectors and state
  DevBuf hostW, hostGrad, hostGradTmp, hostF, hostStage[2];  // host-streamed eval
  DevBuf dgnGrad, dgnX, dgnY, dgnGrams, dgnGamma, dgnScal, dgnPart;  // dGN outer loop
  DevBuf gemmPart;                          // compression: GEMM split-K partials
  DevBuf eigQ, eigZ, eigH, eigV, eigU, eigRes, eigScal, eigB;  // compression: subspace iteration
  DevBuf mlG, mlU, mlLam, mlX, mlY, mlRanks;
  DevBuf cpdU, cpdSig, cpdS, cpdW, cpdGrad, cpdScal;   // tf_cpd pipeline
  DevBuf alsKR, alsM, alsSmall, alsF;                 // CP-ALS
  DevBuf evGrams, evPart;                             // Pi-form evaluation: local Grams, guard partials
  int cg_grid = 0;                                    // 0: default CG launch; > 0: grid kernel with that many blocks
  int eval_form = 0;                                  // 0 auto, 1 residual form, 2 guarded Pi form
  int last_eval_tma = -1;                             // the last evaluation's slice loads: 1 TMA, 0 cooperative
  bool last_eval_pi = false;                          // the last evaluation ran the guarded Pi form
  bool force_residual = false;                        // dGN loop: the guard fell back, stay residual
  bool eval_f_only = false;                           // the caller needs F only (guard ignores grad)              // compression: Grams, U, core intermediates
  double* scal_host = nullptr;              // pinned, dGN scalars
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  tfk::CgState* cg_host = nullptr;          // pinned
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used_pairs = 0;
  int64_t eval_launches = 0;
  int64_t total_launches = 0;
};

namespace tfh {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn();
tf_status set_err(tf_ctx* c, tf_status s, const std::string& msg);
tf_status cuda_err(tf_ctx* c, cudaError_t e, const char* where);
tf_status ensure(tf_ctx* c, DevBuf& b, size_t bytes);
void free_buf(DevBuf& b);

// generic DMMA GEMM (k_gemm.cu) planning and launch, tf_mlsvd.cu
tfk::GemmOperand opnd(const double* p, int64_t ld, bool kc, int64_t bstride = 0);
tfk::GemmArgs gemm_args(tfk::GemmOperand a, tfk::GemmOperand b, int64_t M, int64_t N, int64_t Kd, double* C,
                        int64_t ldc);
tf_status gemm_run(tf_ctx* c, tfk::GemmArgs g);
// F at w (grad_scratch: n doubles of scratch), the Pi-form guard checking the expansion of F only (tf_api.cu)
tf_status eval_f_only(tf_ctx* c, tf_dims d, const double* T, const double* w, double* f, double* grad_scratch);

}  // namespace tfh

#define TF_CUDA(c, expr)                                          \
  do {                                                            \
    cudaError_t e_ = (expr);                                      \
    if (e_ != cudaSuccess) return tfh::cuda_err((c), e_, #expr);  \
  } while (0)

// blocks of the persistent CG / matvec launch: every SM, or the test cap of tf_ctx_set_cg_grid
inline int cg_grid(const tf_ctx* c) { return c->cg_grid > 0 && c->cg_grid < c->nsm ? c->cg_grid : c->nsm; }
