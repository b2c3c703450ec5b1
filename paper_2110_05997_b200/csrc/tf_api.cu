// C-ABI of the dGN evaluation hot path (include/tf.h): argument validation, context and workspace
// management, work decomposition and launch orchestration. No arithmetic of the method happens here;
// every step runs in the kernels of k_eval.cu, k_cg.cu and k_small.cu.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "tf_ctx.h"

using namespace tfk;

namespace tfh {

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

tf_status set_err(tf_ctx* c, tf_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

tf_status cuda_err(tf_ctx* c, cudaError_t e, const char* where) {
  return set_err(c, TF_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

tf_status ensure(tf_ctx* c, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (b.cap >= bytes) return TF_OK;
  if (b.p) {
    // the buffer may still be read or written by work on either library stream (the host-staged path copies
    // on copy_stream): both must be idle before it is freed
    cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
  }
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(c, TF_ERR_ALLOC, "workspace allocation of " + std::to_string(bytes) + " bytes failed: " +
                                        cudaGetErrorString(e));
  }
  b.cap = bytes;
  return TF_OK;
}

void free_buf(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

}  // namespace tfh

using namespace tfh;

namespace {
tf_status eval_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* w, double* f, double* grad);
}

namespace tfh {
// F alone (grad is scratch): the Pi-form guard then only asks the Gram expansion of F to be safe
tf_status eval_f_only(tf_ctx* c, tf_dims d, const double* T, const double* w, double* f, double* grad_scratch) {
  if (d.ldT == 0) d.ldT = d.I;
  if (d.K_total == 0) d.K_total = d.K + d.k_begin;
  c->eval_f_only = true;
  tf_status s = eval_impl(c, d, T, w, f, grad_scratch);
  c->eval_f_only = false;
  return s;
}
}  // namespace tfh

namespace {

tf_status check_dims(tf_ctx* c, tf_dims& d) {
  if (!c) return TF_ERR_ARG;
  if (d.ldT == 0) d.ldT = d.I;
  if (d.K_total == 0) d.K_total = d.K + d.k_begin;
  if (d.I < 1 || d.J < 1 || d.K < 1 || d.R < 1)
    return set_err(c, TF_ERR_ARG, "dimensions must be >= 1 (I=" + std::to_string(d.I) + " J=" +
                                      std::to_string(d.J) + " K=" + std::to_string(d.K) +
                                      " R=" + std::to_string(d.R) + ")");
  if (d.ldT < d.I) return set_err(c, TF_ERR_ARG, "ldT < I");
  if (d.k_begin < 0 || d.k_begin + d.K > d.K_total) return set_err(c, TF_ERR_ARG, "k_begin + K > K_total");
  if (d.R > TF_MAX_R) return set_err(c, TF_ERR_UNSUPPORTED, "R > TF_MAX_R (" + std::to_string(TF_MAX_R) + ")");
  if (d.I > (1LL << 31) - 1 || d.J > (1LL << 31) - 1 || d.K_total > (1LL << 31) - 1)
    return set_err(c, TF_ERR_UNSUPPORTED, "mode size >= 2^31");
  return TF_OK;
}

Modes make_modes(const tf_dims& d, const double* w) {
  Modes m;
  m.R = d.R;
  m.n[0] = d.I;
  m.n[1] = d.J;
  m.n[2] = d.K_total;
  m.off[0] = 0;
  m.off[1] = d.I * d.R;
  m.off[2] = (d.I + d.J) * d.R;
  for (int l = 0; l < 3; ++l) m.W[l] = w + m.off[l];
  return m;
}

// Choose the number of k-chunks per (i-tile, j-tile): minimise waves * (slices per chunk + overhead),
// where one CTA is resident per SM (the fused kernel uses ~190 KB of shared memory).
int choose_ksplit(int64_t tiles, int64_t K, int nsm) {
  // development overrides: TF_EVAL_KSPLIT (fixed split) and TF_EVAL_KSPLIT_OVH (the overhead constant)
  static const int force = [] {
    const char* e = getenv("TF_EVAL_KSPLIT");
    return e ? atoi(e) : 0;
  }();
  static const double ovh = [] {
    const char* e = getenv("TF_EVAL_KSPLIT_OVH");
    return e ? atof(e) : 2.0;
  }();
  if (force > 0) return (int)std::min<int64_t>(force, K);
  const double overhead = ovh;  // prologue + partial write-out, in slice-iterations
  int best = 1;
  double best_cost = 1e300;
  const int64_t kmax = std::min<int64_t>(K, 4096);
  for (int64_t ks = 1; ks <= kmax; ++ks) {
    const int64_t chunk = (K + ks - 1) / ks;
    const int64_t used = (K + chunk - 1) / chunk;  // non-empty chunks
    if (used != ks) continue;
    const int64_t units = tiles * ks;
    const int64_t waves = (units + nsm - 1) / nsm;
    const double cost = (double)waves * ((double)chunk + overhead);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = (int)ks;
    }
  }
  return best;
}

tf_status grams_impl(tf_ctx* c, const tf_dims& d, const double* w, double* grams) {
  Modes m = make_modes(d, w);
  tf_status s = ensure(c, c->gram_part, (size_t)gram_partial_slots(m) * 3 * d.R * d.R * 8);
  if (s) return s;
  TF_CUDA(c, launch_grams_ws(m, (double*)c->gram_part.p, grams, c->stream));
  c->total_launches += 2;
  return TF_OK;
}

// Stream-K decomposition of the fused kernel's (tile, slice) space: TF_EVAL_STREAMK=0 selects the k-chunk grid
// (development comparison); read per call.
static bool eval_streamk() {
  const char* e = getenv("TF_EVAL_STREAMK");
  return !(e && atoi(e) == 0);
}

// Decoupled warp groups in the Pi-form pass: 0 = the per-slice block barrier, 1 = decoupled with group 0
// throttled to about half a slice ahead, 2 = decoupled, unthrottled; TF_EVAL_DECOUPLE overrides (development).
// Default from the 500^3 sweep over R = 8..40 and c4/c5 (tools/gpu_r02dec4.sh): only NT = 3 gains (R = 24: 0.485 ->
// 0.473 ms, 2 CTAs per SM); every other NT loses 3-11%, c5 6%. The head start of group 0 in ns: TF_EVAL_SKEW_NS,
// default about half a slice (260 ns per r-tile; no measurable effect).
static int eval_decouple(int NT) {
  const char* e = getenv("TF_EVAL_DECOUPLE");
  return e ? atoi(e) : (NT == 3 ? 2 : 0);
}
static int eval_skew_ns(int NT) {
  const char* e = getenv("TF_EVAL_SKEW_NS");
  return e ? atoi(e) : 260 * NT;
}

// L2 promotion of the T tiles' TMA reads (TF_EVAL_L2PROMO = 0 | 64 | 128 | 256, development comparison).
static CUtensorMapL2promotion eval_l2_promotion() {
  const char* e = getenv("TF_EVAL_L2PROMO");
  const int v = e ? atoi(e) : 0;
  return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                  : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                             : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

// Tile size of the fused kernel: TF_EVAL_TILE=32|64 overrides (development); default 64.
int eval_tile() {
  static int bt = 0;
  if (!bt) {
    const char* e = getenv("TF_EVAL_TILE");
    bt = (e && atoi(e) == 32) ? 32 : 64;
  }
  return bt;
}

tf_status eval_impl(tf_ctx* c, const tf_dims& d, const double* T, const double* w, double* f, double* grad) {
  const int NT = (int)((d.R + 7) / 8);
  const int RP = 8 * NT;
  const int BT = eval_tile();
  // the form decides which kernel runs (and how many of its CTAs fit on an SM)
  const bool pi_form = BT == 64 && !c->force_residual &&
                       (c->eval_form == 2 || (c->eval_form == 0 && 6.0 * d.I * d.J * d.K * d.R >= 5e9));
  // co-resident CTAs only pay off when one CTA leaves the DMMA pipe mostly idle (R <= 16; measured: c2's
  // R = 10 gains 14%, c3's R = 20 loses 9% to the shorter k-chunks)
  const int ctas_per_sm = BT == 32 ? 2 : (NT <= 2 ? eval_ctas_per_sm(NT, !pi_form) : 1);
  EvalArgs p;
  memset(&p, 0, sizeof(p));
  p.run_if = nullptr;
  p.A = w;
  p.B = w + d.I * d.R;
  p.C = w + (d.I + d.J) * d.R;
  p.I = d.I;
  p.J = d.J;
  p.K = d.K;
  p.R = d.R;
  p.ldT = d.ldT;
  p.Ktot = d.K_total;
  p.kbeg = d.k_begin;
  p.nTi = (int)((d.I + BT - 1) / BT);
  p.nTj = (int)((d.J + BT - 1) / BT);
  p.Ipad = (int64_t)p.nTi * BT;
  p.Jpad = (int64_t)p.nTj * BT;
  p.decouple = eval_decouple(NT);
  p.skewNs = eval_skew_ns(NT);
  const int64_t tiles = (int64_t)p.nTi * p.nTj;
  if (eval_streamk() && d.K > 0) {
    // stream-K: a persistent grid of every co-resident CTA, each with an equal run of (tile, slice) units
    const char* ecps = getenv("TF_EVAL_PERSIST_CPS");   // development override of the CTAs per SM
    // the Pi pass runs two CTAs per SM where its launch bounds guarantee them (R <= 24), one otherwise (measured:
    // 500^3 R = 8/16/24 at two CTAs 0.242/0.351/0.485 ms vs one 0.294/0.385/0.526 ms; R = 32 one CTA 0.621 vs 0.636)
    const int cps = (ecps && atoi(ecps) > 0) ? atoi(ecps)
                                             : (BT == 32 ? 2 : pi_form ? (NT <= 3 ? 2 : 1) : eval_ctas_per_sm(NT, true));
    const int64_t units = tiles * d.K;
    int64_t grid = std::min<int64_t>(units, (int64_t)c->nsm * cps);
    p.unitsPerCta = (units + grid - 1) / grid;
    grid = (units + p.unitsPerCta - 1) / p.unitsPerCta;
    int smax = 1;
    for (int64_t t = 0; t < tiles; ++t) {
      const int64_t c0 = (t * d.K) / p.unitsPerCta, c1 = (t * d.K + d.K - 1) / p.unitsPerCta;
      smax = std::max<int>(smax, (int)(c1 - c0 + 1));
    }
    p.streamK = 1;
    p.kSplit = smax;
    p.kChunk = d.K;
    p.nCta = (int)grid;
  } else {
    p.streamK = 0;
    p.kSplit = choose_ksplit(tiles, d.K, c->nsm * ctas_per_sm);
    p.kChunk = (d.K + p.kSplit - 1) / p.kSplit;
    p.nCta = (int)(tiles * p.kSplit);
  }
  tf_status s;
  if ((s = ensure(c, c->gAp, (size_t)p.nTj * p.kSplit * p.Ipad * RP * 8))) return s;
  if ((s = ensure(c, c->gBp, (size_t)p.nTi * p.kSplit * p.Jpad * RP * 8))) return s;
  if ((s = ensure(c, c->gCp, (size_t)tiles * d.K * RP * 8))) return s;
  if ((s = ensure(c, c->fp, (size_t)p.nCta * 8))) return s;
  p.gAp = (double*)c->gAp.p;
  p.gBp = (double*)c->gBp.p;
  p.gCp = (double*)c->gCp.p;
  p.fp = (double*)c->fp.p;

  CUtensorMap map[2];   // [0] 3-D (I, J, K) view; [1] 4-D (i mod BT, i / BT, J, K) view of the whole i-tiles
  memset(map, 0, sizeof(map));
  bool tma = (d.ldT % 2 == 0) && ((reinterpret_cast<uintptr_t>(T) & 15) == 0);
  if (tma) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) {
      tma = false;
    } else {
      cuuint64_t gdim[3] = {(cuuint64_t)d.I, (cuuint64_t)d.J, (cuuint64_t)d.K};
      cuuint64_t gstride[2] = {(cuuint64_t)d.ldT * 8, (cuuint64_t)d.ldT * d.J * 8};
      cuuint32_t box[3] = {(cuuint32_t)(BT + 4), (cuuint32_t)BT, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      CUresult r = enc(&map[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(T), gdim, gstride, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, eval_l2_promotion(),
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) tma = false;
      const char* e4 = getenv("TF_EVAL_TMA4");   // development switch: 0 = 3-D map only
      if (tma && d.I >= BT && !(e4 && atoi(e4) == 0)) {
        cuuint64_t gdim4[4] = {(cuuint64_t)BT, (cuuint64_t)(d.I / BT), (cuuint64_t)d.J, (cuuint64_t)d.K};
        cuuint64_t gstride4[3] = {(cuuint64_t)BT * 8, (cuuint64_t)d.ldT * 8, (cuuint64_t)d.ldT * d.J * 8};
        cuuint32_t box4[4] = {(cuuint32_t)(BT + 4), 1, (cuuint32_t)BT, 1};
        cuuint32_t estr4[4] = {1, 1, 1, 1};
        r = enc(&map[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(T), gdim4, gstride4, box4, estr4,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, eval_l2_promotion(),
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        p.tma4 = r == CUDA_SUCCESS ? 1 : 0;
      }
    }
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    if (c->ev_used_pairs * 2 + 2 > c->ev_pool.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t ev;
        TF_CUDA(c, cudaEventCreate(&ev));
        c->ev_pool.push_back(ev);
      }
    }
    e0 = c->ev_pool[c->ev_used_pairs * 2];
    e1 = c->ev_pool[c->ev_used_pairs * 2 + 1];
    c->ev_used_pairs++;
    TF_CUDA(c, cudaEventRecord(e0, c->stream));
  }
  // (small problems are launch-bound: the Pi form's extra launches — Grams, guard, conditional fallback —
  // would cost more than the reconstruction flops it saves, hence the 5e9-flop threshold above)
  c->last_eval_pi = pi_form;
  c->last_eval_tma = tma ? 1 : 0;
  if (!pi_form) {
    TF_CUDA(c, launch_eval(map, T, p, NT, tma, BT, c->stream));
    if (c->timing) TF_CUDA(c, cudaEventRecord(e1, c->stream));
    TF_CUDA(c, launch_eval_finalize(p, RP, f, grad, c->nsm, c->stream));
    c->eval_launches += 1;
    c->total_launches += 2;
    return TF_OK;
  }
  // Pi form: one pass computes the three MTTKRPs of T (2 contractions per slice), then
  // grad = W Pi - M and f by the Gram expansion; if cancellation makes that unsafe the residual form runs
  // (the same kernel with the reconstruction phase; reading R31).
  const int nblk = eval_pi_blocks(c->nsm);
  if ((s = ensure(c, c->evGrams, (size_t)9 * d.R * d.R * 8))) return s;
  if ((s = ensure(c, c->evPart, (size_t)3 * nblk * 8 + 64))) return s;
  double* grams = (double*)c->evGrams.p;
  double* part = (double*)c->evPart.p;
  int* flag = reinterpret_cast<int*>(part + 3 * nblk);
  TF_CUDA(c, launch_eval(map, T, p, NT, tma, BT, c->stream, false));
  // Equal-size modes sit I*R apart in w (and their Grams / Pi blocks R*R apart), so their small GEMMs run as
  // one batched launch: the three Grams (whole tensor, I = J = K) or A^T A and B^T B (I = J).
  const bool cube = d.I == d.J && d.J == d.K && d.K == d.K_total;
  if (d.K == d.K_total && !cube) {
    if ((s = grams_impl(c, d, w, grams))) return s;
  } else {   // for a K-shard the C Gram is over the local slices only (the partial f and grad)
    const int64_t R = d.R, RR = R * R;
    const int nab = cube ? 3 : (d.I == d.J ? 2 : 1);
    GemmArgs ga = gemm_args(opnd(p.A, d.I, true, d.I * R), opnd(p.A, d.I, true, d.I * R), R, R, d.I, grams, R);
    ga.sym = true;
    ga.batch = nab;
    ga.sum_batch = nab == 1;
    ga.cstride = RR;
    if ((s = gemm_run(c, ga))) return s;
    if (nab == 1) {
      GemmArgs gb = gemm_args(opnd(p.B, d.J, true), opnd(p.B, d.J, true), R, R, d.J, grams + RR, R);
      gb.sym = true;
      if ((s = gemm_run(c, gb))) return s;
    }
    if (!cube) {
      GemmArgs gc = gemm_args(opnd(p.C + d.k_begin, d.K_total, true), opnd(p.C + d.k_begin, d.K_total, true), R,
                              R, d.K, grams + 2 * RR, R);
      gc.sym = true;
      if ((s = gemm_run(c, gc))) return s;
    }
  }
  // W Pi into grad: Pi = [Pi1 | Pi2 | Pi3 | ...] from the (local) Grams, then one small GEMM per mode
  double* pi = grams + 3 * d.R * d.R;
  TF_CUDA(c, launch_hadamard(d.R, grams, pi, c->stream));
  {
    const int64_t R = d.R, RR = R * R;
    const int nab = cube ? 3 : (d.I == d.J ? 2 : 1);
    GemmArgs ga = gemm_args(opnd(p.A, d.I, false, d.I * R), opnd(pi, R, true, RR), d.I, R, R, grad, d.I);
    ga.batch = nab;
    ga.sum_batch = nab == 1;
    ga.cstride = d.I * R;
    if ((s = gemm_run(c, ga))) return s;
    if (nab == 1 &&
        (s = gemm_run(c, gemm_args(opnd(p.B, d.J, false), opnd(pi + RR, R, true), d.J, R, R, grad + d.I * R, d.J))))
      return s;
    if (!cube && (s = gemm_run(c, gemm_args(opnd(p.C + d.k_begin, d.K_total, false), opnd(pi + 2 * RR, R, true), d.K,
                                            R, R, grad + (d.I + d.J) * R + d.k_begin, d.K_total))))
      return s;
  }
  TF_CUDA(c, launch_eval_finalize_pi(p, RP, grad, part, nblk, c->stream));
  TF_CUDA(c, launch_eval_pi_guard(p, grams, part, nblk, f, flag, c->stream, !c->eval_f_only));
  EvalArgs pr = p;
  pr.run_if = flag;
  TF_CUDA(c, launch_eval(map, T, pr, NT, tma, BT, c->stream, true));
  if (c->timing) TF_CUDA(c, cudaEventRecord(e1, c->stream));
  TF_CUDA(c, launch_eval_finalize(pr, RP, f, grad, c->nsm, c->stream));
  c->eval_launches += 1;
  c->total_launches += 5;
  return TF_OK;
}

}  // namespace

extern "C" {

int tf_version(void) { return 1; }

const char* tf_status_str(tf_status s) {
  switch (s) {
    case TF_OK: return "TF_OK";
    case TF_ERR_ARG: return "TF_ERR_ARG";
    case TF_ERR_ALIGN: return "TF_ERR_ALIGN";
    case TF_ERR_UNSUPPORTED: return "TF_ERR_UNSUPPORTED";
    case TF_ERR_CUDA: return "TF_ERR_CUDA";
    case TF_ERR_NONFINITE: return "TF_ERR_NONFINITE";
    case TF_ERR_ALLOC: return "TF_ERR_ALLOC";
  }
  return "TF_ERR_UNKNOWN";
}

const char* tf_last_error(const tf_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

tf_status tf_ctx_create(tf_ctx** out, int device, void* cuda_stream) {
  if (!out) return TF_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return TF_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return TF_ERR_CUDA;
  tf_ctx* c = new tf_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  {
    const char* e = getenv("TF_EVAL_FORM");
    c->eval_form = (e && std::string(e) == "residual") ? 1 : 0;
  }
  if (cudaMallocHost(&c->cg_host, sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost(&c->scal_host, 16 * sizeof(double)) != cudaSuccess) {
    delete c;
    return TF_ERR_ALLOC;
  }
  *out = c;
  return TF_OK;
}

tf_status tf_ctx_destroy(tf_ctx* c) {
  if (!c) return TF_ERR_ARG;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->gAp, &c->gBp, &c->gCp, &c->fp, &c->gram_part, &c->mvG, &c->mvS, &c->mvPi, &c->mvD,
                    &c->mvPart, &c->cgR, &c->cgP, &c->cgZ, &c->cgState, &c->hostW, &c->hostGrad,
                    &c->hostGradTmp, &c->hostF, &c->hostStage[0], &c->hostStage[1], &c->dgnGrad, &c->dgnX,
                    &c->dgnY, &c->dgnGrams, &c->dgnGamma, &c->dgnScal, &c->dgnPart, &c->gemmPart,
                    &c->eigQ, &c->eigZ, &c->eigH, &c->eigV, &c->eigU, &c->eigRes, &c->eigScal, &c->eigB, &c->mlG,
                    &c->mlU, &c->mlLam, &c->mlX, &c->mlY, &c->mlRanks, &c->cpdU, &c->cpdSig, &c->cpdS,
                    &c->cpdW, &c->cpdGrad, &c->cpdScal, &c->alsKR, &c->alsM, &c->alsSmall, &c->alsF, &c->evGrams, &c->evPart};
  for (DevBuf* b : bufs) free_buf(*b);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_used[i]) cudaEventDestroy(c->ev_used[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->cg_host) cudaFreeHost(c->cg_host);
  if (c->scal_host) cudaFreeHost(c->scal_host);
  delete c;
  return TF_OK;
}

tf_status tf_ctx_set_stream(tf_ctx* c, void* s) {
  if (!c) return TF_ERR_ARG;
  c->stream = static_cast<cudaStream_t>(s);
  return TF_OK;
}

tf_status tf_ctx_set_eval_form(tf_ctx* c, int form) {
  if (!c) return TF_ERR_ARG;
  if (form < 0 || form > 2)
    return set_err(c, TF_ERR_ARG, "eval form must be 0 (auto), 1 (residual) or 2 (guarded Pi form at any size)");
  c->eval_form = form;
  return TF_OK;
}

tf_status tf_ctx_eval_path(tf_ctx* c, int* tma) {
  if (!c || !tma) return TF_ERR_ARG;
  *tma = c->last_eval_tma;
  return TF_OK;
}

tf_status tf_ctx_set_cg_grid(tf_ctx* c, int nblocks) {
  if (!c) return TF_ERR_ARG;
  if (nblocks < 0) return set_err(c, TF_ERR_ARG, "nblocks must be >= 0");
  c->cg_grid = nblocks;
  return TF_OK;
}

tf_status tf_ctx_eval_fallback(tf_ctx* c, int* fell_back) {
  if (!c || !fell_back) return TF_ERR_ARG;
  *fell_back = -1;
  if (!c->evPart.p || !c->last_eval_pi) return TF_OK;   // -1: the last evaluation did not run the Pi form
  cudaSetDevice(c->device);
  const int nblk = eval_pi_blocks(c->nsm);
  int v = -1;
  TF_CUDA(c, cudaMemcpyAsync(&v, reinterpret_cast<int*>((double*)c->evPart.p + 3 * nblk), sizeof(int),
                             cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  *fell_back = v;
  return TF_OK;
}

tf_status tf_ctx_set_timing(tf_ctx* c, int enable) {
  if (!c) return TF_ERR_ARG;
  c->timing = enable != 0;
  return TF_OK;
}

tf_status tf_ctx_kernel_stats(tf_ctx* c, double* ms, int64_t* eval_launches, int64_t* total, int reset) {
  if (!c) return TF_ERR_ARG;
  cudaSetDevice(c->device);
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  double t = 0.0;
  for (size_t i = 0; i < c->ev_used_pairs; ++i) {
    float x = 0.f;
    TF_CUDA(c, cudaEventElapsedTime(&x, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
    t += x;
  }
  if (ms) *ms = t;
  if (eval_launches) *eval_launches = (int64_t)c->ev_used_pairs;
  if (total) *total = c->total_launches;
  if (reset) {
    c->ev_used_pairs = 0;
    c->total_launches = 0;
    c->eval_launches = 0;
  }
  return TF_OK;
}

tf_status tf_grams(tf_ctx* c, tf_dims d, const double* w, double* grams) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!w || !grams) return set_err(c, TF_ERR_ARG, "null pointer");
  cudaSetDevice(c->device);
  return grams_impl(c, d, w, grams);
}

tf_status tf_hadamard(tf_ctx* c, int64_t R, const double* grams, double* pi) {
  if (!c) return TF_ERR_ARG;
  if (R < 1 || !grams || !pi) return set_err(c, TF_ERR_ARG, "bad argument");
  cudaSetDevice(c->device);
  TF_CUDA(c, launch_hadamard(R, grams, pi, c->stream));
  c->total_launches += 1;
  return TF_OK;
}

tf_status tf_cpd_eval(tf_ctx* c, tf_dims d, const double* T, const double* w, double* f, double* grad,
                      double* grams) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!T || !w || !f || !grad) return set_err(c, TF_ERR_ARG, "null pointer");
  if (reinterpret_cast<uintptr_t>(T) & 7) return set_err(c, TF_ERR_ALIGN, "T not 8-byte aligned");
  cudaSetDevice(c->device);
  if ((s = eval_impl(c, d, T, w, f, grad))) return s;
  if (grams) {
    // the Pi-form pass already formed [A^T A | B^T B | C^T C] (the whole tensor: K == K_total); for a K-shard
    // it formed A^T A, B^T B and the local C Gram, so only the full C^T C remains (one symmetric GEMM)
    if (c->last_eval_pi) {
      const int64_t R = d.R;
      const size_t nb = (size_t)(d.K == d.K_total ? 3 : 2) * R * R * 8;
      TF_CUDA(c, cudaMemcpyAsync(grams, c->evGrams.p, nb, cudaMemcpyDeviceToDevice, c->stream));
      if (d.K == d.K_total) return TF_OK;
      const double* C = w + (d.I + d.J) * R;
      GemmArgs gc = gemm_args(opnd(C, d.K_total, true), opnd(C, d.K_total, true), R, R, d.K_total, grams + 2 * R * R,
                              R);
      gc.sym = true;
      return gemm_run(c, gc);
    }
    return grams_impl(c, d, w, grams);
  }
  return TF_OK;
}

tf_status tf_cpd_eval_host(tf_ctx* c, tf_dims d, const double* T_host, const double* w_host, double* f_host,
                           double* grad_host) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!T_host || !w_host || !f_host || !grad_host) return set_err(c, TF_ERR_ARG, "null pointer");
  cudaSetDevice(c->device);
  const int64_t n = d.R * (d.I + d.J + d.K_total);
  const size_t slice_bytes = (size_t)d.ldT * d.J * 8;
  const size_t slab_target = (size_t)512 << 20;
  int64_t kslab = std::max<int64_t>(1, (int64_t)(slab_target / slice_bytes));
  kslab = std::min<int64_t>(kslab, d.K);
  if ((s = ensure(c, c->hostW, n * 8))) return s;
  if ((s = ensure(c, c->hostGrad, n * 8))) return s;
  if ((s = ensure(c, c->hostGradTmp, n * 8))) return s;
  if ((s = ensure(c, c->hostF, 16))) return s;
  for (int i = 0; i < 2; ++i)
    if ((s = ensure(c, c->hostStage[i], kslab * slice_bytes))) return s;
  if (!c->copy_stream) TF_CUDA(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!c->ev_copied[i]) TF_CUDA(c, cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
    if (!c->ev_used[i]) TF_CUDA(c, cudaEventCreateWithFlags(&c->ev_used[i], cudaEventDisableTiming));
  }
  double* wd = (double*)c->hostW.p;
  double* gacc = (double*)c->hostGrad.p;
  double* gtmp = (double*)c->hostGradTmp.p;
  double* fd = (double*)c->hostF.p;  // fd[0] accumulated f, fd[1] per-slab f
  TF_CUDA(c, cudaMemcpyAsync(wd, w_host, n * 8, cudaMemcpyHostToDevice, c->stream));
  TF_CUDA(c, cudaMemsetAsync(gacc, 0, n * 8, c->stream));
  TF_CUDA(c, cudaMemsetAsync(fd, 0, 16, c->stream));
  // the copy stream must not overwrite a stage before the compute stream is done with it
  TF_CUDA(c, cudaEventRecord(c->ev_used[0], c->stream));
  TF_CUDA(c, cudaEventRecord(c->ev_used[1], c->stream));
  int slab = 0;
  for (int64_t k0 = 0; k0 < d.K; k0 += kslab, ++slab) {
    const int64_t kn = std::min<int64_t>(kslab, d.K - k0);
    const int b = slab & 1;
    TF_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->ev_used[b], 0));
    TF_CUDA(c, cudaMemcpyAsync(c->hostStage[b].p, T_host + (size_t)k0 * d.ldT * d.J, kn * slice_bytes,
                               cudaMemcpyHostToDevice, c->copy_stream));
    TF_CUDA(c, cudaEventRecord(c->ev_copied[b], c->copy_stream));
    TF_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
    tf_dims ds = d;
    ds.K = kn;
    ds.k_begin = d.k_begin + k0;
    if ((s = eval_impl(c, ds, (const double*)c->hostStage[b].p, wd, fd + 1, gtmp))) return s;
    TF_CUDA(c, cudaEventRecord(c->ev_used[b], c->stream));
    TF_CUDA(c, launch_axpy1(n, gtmp, gacc, c->stream));
    TF_CUDA(c, launch_axpy1(1, fd + 1, fd, c->stream));
    c->total_launches += 2;
  }
  TF_CUDA(c, cudaMemcpyAsync(grad_host, gacc, n * 8, cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaMemcpyAsync(f_host, fd, 8, cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  return TF_OK;
}

static tf_status matvec_ws(tf_ctx* c, const tf_dims& d, const Modes& m, MatvecWs& ws) {
  const size_t RR = (size_t)d.R * d.R;
  tf_status s;
  if ((s = ensure(c, c->mvG, cg_gram_partial_doubles(d.R) * 8))) return s;
  if ((s = ensure(c, c->mvS, 3 * RR * 8))) return s;
  if ((s = ensure(c, c->mvPi, 6 * RR * 8))) return s;
  if ((s = ensure(c, c->mvD, 3 * d.R * 8))) return s;
  const size_t part = (size_t)gram_partial_slots(m) * 3 * RR + (size_t)cg_partial_slots(m) + 2 * (size_t)c->nsm + 16;
  if ((s = ensure(c, c->mvPart, part * 8))) return s;
  ws.G = (double*)c->mvG.p;
  ws.S = (double*)c->mvS.p;
  ws.pi = (double*)c->mvPi.p;
  ws.dscale = (double*)c->mvD.p;
  ws.partial = (double*)c->mvPart.p;
  ws.nblk_dot = cg_partial_slots(m);
  return TF_OK;
}

tf_status tf_reg_gamma(tf_ctx* c, int64_t R, const double* grams, double* gamma) {
  if (!c) return TF_ERR_ARG;
  if (R < 1 || R > TF_MAX_R || !grams || !gamma) return set_err(c, TF_ERR_ARG, "bad argument");
  cudaSetDevice(c->device);
  TF_CUDA(c, launch_reg_gamma(R, grams, gamma, c->stream));
  c->total_launches += 1;
  return TF_OK;
}

tf_status tf_gn_matvec_damped(tf_ctx* c, tf_dims d, const double* grams, const double* w, const double* v, double lambda,
                              const double* damp, double* y) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!grams || !w || !v || !y) return set_err(c, TF_ERR_ARG, "null pointer");
  if (v == y) return set_err(c, TF_ERR_ARG, "y must not alias v");
  cudaSetDevice(c->device);
  Modes m = make_modes(d, w);
  MatvecWs ws;
  if ((s = matvec_ws(c, d, m, ws))) return s;
  TF_CUDA(c, launch_hadamard(d.R, grams, ws.pi, c->stream));
  TF_CUDA(c, launch_cg_persistent(m, ws.pi, nullptr, damp, lambda, 0.0, 0, nullptr, v, y, nullptr, nullptr, nullptr,
                                  ws.G, ws.S, ws.partial, nullptr, 1, cg_grid(c), c->cg_grid == 0, c->stream));
  c->total_launches += 2;
  return TF_OK;
}

tf_status tf_gn_matvec(tf_ctx* c, tf_dims d, const double* grams, const double* w, const double* v, double lambda,
                       double* y) {
  return tf_gn_matvec_damped(c, d, grams, w, v, lambda, nullptr, y);
}

// CG on (J^T J + lambda D) x = rhs; the state (iterations, ||r||^2, non-finite flag) lands in c->cgState.
static tf_status cg_impl(tf_ctx* c, const tf_dims& d, const double* grams, const double* w, const double* rhs,
                         double lambda, const double* damp, int maxiter, double tol, int jacobi, double* x) {
  Modes m = make_modes(d, w);
  const int64_t n = d.R * (d.I + d.J + d.K_total);
  MatvecWs ws;
  tf_status s;
  if ((s = matvec_ws(c, d, m, ws))) return s;
  if ((s = ensure(c, c->cgR, n * 8))) return s;
  if ((s = ensure(c, c->cgP, 2 * n * 8))) return s;   // current and next CG direction
  if ((s = ensure(c, c->cgZ, n * 8))) return s;
  if ((s = ensure(c, c->cgState, sizeof(CgState)))) return s;
  CgState* st = (CgState*)c->cgState.p;
  TF_CUDA(c, cudaMemsetAsync(st, 0, sizeof(CgState), c->stream));
  TF_CUDA(c, launch_hadamard(d.R, grams, ws.pi, c->stream));
  if (jacobi) TF_CUDA(c, launch_jacobi_scale(m, ws.pi, lambda, damp, ws.dscale, c->stream));
  TF_CUDA(c, launch_cg_persistent(m, ws.pi, jacobi ? ws.dscale : nullptr, damp, lambda, tol, maxiter, rhs, nullptr, x,
                                  (double*)c->cgR.p, (double*)c->cgP.p, (double*)c->cgZ.p, ws.G, ws.S, ws.partial, st,
                                  0, cg_grid(c), c->cg_grid == 0, c->stream));
  c->total_launches += 2 + (jacobi ? 1 : 0);
  return TF_OK;
}

tf_status tf_cg_solve_damped(tf_ctx* c, tf_dims d, const double* grams, const double* w, const double* rhs,
                             double lambda, const double* damp, int maxiter, double tol, int jacobi, double* x,
                             int* iters_done, double* res2) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!grams || !w || !rhs || !x) return set_err(c, TF_ERR_ARG, "null pointer");
  if (maxiter < 0) return set_err(c, TF_ERR_ARG, "maxiter < 0");
  cudaSetDevice(c->device);
  if ((s = cg_impl(c, d, grams, w, rhs, lambda, damp, maxiter, tol, jacobi, x))) return s;
  TF_CUDA(c, cudaMemcpyAsync(c->cg_host, c->cgState.p, sizeof(CgState), cudaMemcpyDeviceToHost, c->stream));
  TF_CUDA(c, cudaStreamSynchronize(c->stream));
  if (iters_done) *iters_done = c->cg_host->iters;
  if (res2) *res2 = c->cg_host->rr;
  if (c->cg_host->nonfinite)
    return set_err(c, TF_ERR_NONFINITE,
                   "CG: non-finite alpha/beta at iteration " + std::to_string(c->cg_host->nonfinite));
  return TF_OK;
}

}  // extern "C"

namespace {

// The dGN loop; with an exchange hook (K-sharded ranks) the partial [grad | F] of every evaluation and the
// tensor sums are summed over the ranks through xbuf, everything else runs replicated (identical inputs,
// deterministic kernels -> identical trajectories on every rank).
tf_status dgn_impl(tf_ctx* c, tf_dims d, const double* T, double* w, const tf_dgn_params* prm, tf_dgn_result* res,
                   double* hist, tf_allreduce_fn xfn, void* xuser, double* xbuf) {
  tf_status s;
  const int64_t n = d.R * (d.I + d.J + d.K_total), RR = d.R * d.R;
  if ((s = ensure(c, c->dgnGrad, (n + 1) * 8))) return s;
  if ((s = ensure(c, c->dgnX, n * 8))) return s;
  if ((s = ensure(c, c->dgnY, n * 8))) return s;
  if ((s = ensure(c, c->dgnGrams, 3 * RR * 8))) return s;
  if ((s = ensure(c, c->dgnGamma, 3 * d.R * 8))) return s;
  if ((s = ensure(c, c->dgnScal, 16 * 8))) return s;
  if ((s = ensure(c, c->dgnPart, (size_t)red_blocks() * 4 * 8))) return s;
  double* grad = (double*)c->dgnGrad.p;
  double* x = (double*)c->dgnX.p;
  double* y = (double*)c->dgnY.p;
  double* grams = (double*)c->dgnGrams.p;
  double* gamma = (double*)c->dgnGamma.p;
  double* scal = (double*)c->dgnScal.p;   // [0] F, [1..2] tensor sums, [4..7] dots
  double* part = (double*)c->dgnPart.p;
  double* hs = c->scal_host;
  const Modes m = make_modes(d, w);
  if ((s = ensure(c, c->cgState, sizeof(CgState)))) return s;
  TF_CUDA(c, cudaMemsetAsync(c->cgState.p, 0, sizeof(CgState), c->stream));
  // Once the guarded Pi-form evaluation falls back (the fit has become too close for the Gram expansion),
  // the remaining iterations evaluate in the residual form directly instead of paying for both passes.
  int* hflag = reinterpret_cast<int*>(hs + 14);
  auto sync_scalars = [&]() -> tf_status {
    TF_CUDA(c, cudaMemcpyAsync(hs, scal, 12 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaMemcpyAsync(c->cg_host, c->cgState.p, sizeof(CgState), cudaMemcpyDeviceToHost, c->stream));
    const bool pi = c->last_eval_pi;
    if (pi)
      TF_CUDA(c, cudaMemcpyAsync(hflag, reinterpret_cast<int*>((double*)c->evPart.p + 3 * eval_pi_blocks(c->nsm)),
                                 sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
    if (pi && *hflag == 1) c->force_residual = true;
    return TF_OK;
  };
  struct ResetForce {
    tf_ctx* c;
    ~ResetForce() { c->force_residual = false; }
  } reset_force{c};
  // exchange: xbuf <- src (cnt doubles), SUM over ranks by the hook, src <- xbuf
  auto exchange = [&](double* src, int64_t cnt) -> tf_status {
    if (!xfn) return TF_OK;
    TF_CUDA(c, cudaMemcpyAsync(xbuf, src, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
    TF_CUDA(c, cudaStreamSynchronize(c->stream));
    if (xfn(xbuf, cnt, xuser) != 0) return set_err(c, TF_ERR_CUDA, "the all-reduce hook reported a failure");
    TF_CUDA(c, cudaMemcpyAsync(src, xbuf, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
    return TF_OK;
  };
  // [grad | F] of the local slices -> global (grad is allocated with one spare slot for F)
  auto eval_global = [&]() -> tf_status {
    tf_status st;
    if (!xfn) return eval_impl(c, d, T, w, scal, grad);
    if ((st = eval_impl(c, d, T, w, grad + n, grad))) return st;
    if ((st = exchange(grad, n + 1))) return st;
    TF_CUDA(c, cudaMemcpyAsync(scal, grad + n, 8, cudaMemcpyDeviceToDevice, c->stream));
    return TF_OK;
  };
  // ||T||^2, mean |T|, F and grad at w0
  TF_CUDA(c, launch_tsums(d.I, d.J, d.K, d.ldT, T, part, scal + 1, c->stream));
  if ((s = exchange(scal + 1, 2))) return s;
  if ((s = eval_global())) return s;
  if ((s = grams_impl(c, d, w, grams))) return s;
  c->total_launches += 2;
  if ((s = sync_scalars())) return s;
  const double normT2 = hs[2], normT = sqrt(normT2);
  const double N = (double)d.I * d.J * d.K_total;
  double mu = prm->mu0 > 0 ? prm->mu0 : hs[1] / N;
  double F = hs[0];
  std::vector<double> rel(prm->maxiter + 1);
  rel[0] = normT > 0 ? sqrt(2.0 * F) / normT : 0.0;
  const int cc = 1 + (prm->maxiter + 9) / 10;   // c = 1 + ceil(maxiter / 10)
  const double tol = prm->tol;
  int it = 0, why = 0;
  for (int k = 1; k <= prm->maxiter; ++k) {
    if (prm->use_gamma) {
      TF_CUDA(c, launch_reg_gamma(d.R, grams, gamma, c->stream));
      c->total_launches += 1;
    }
    TF_CUDA(c, launch_scale_copy(n, -1.0, grad, y, c->stream));   // rhs = -grad F(w^(k-1))
    if ((s = cg_impl(c, d, grams, w, y, mu, prm->use_gamma ? gamma : nullptr, prm->cg_iters[k - 1], tol,
                     prm->jacobi, x)))
      return s;
    // x^T J^T J x for the predicted decrease: one GN matvec with lambda = 0 (rhs in y is consumed by now)
    {
      MatvecWs ws;
      if ((s = matvec_ws(c, d, m, ws))) return s;
      TF_CUDA(c, launch_hadamard(d.R, grams, ws.pi, c->stream));
      TF_CUDA(c, launch_cg_persistent(m, ws.pi, nullptr, nullptr, 0.0, 0.0, 0, nullptr, x, y, nullptr, nullptr,
                                      nullptr, ws.G, ws.S, ws.partial, nullptr, 1, cg_grid(c), c->cg_grid == 0, c->stream));
    }
    TF_CUDA(c, launch_dots(n, grad, x, y, part, scal + 4, c->stream));   // {g.x, x.JtJx, x.x, max|g_old|}
    // w^(k) = w^(k-1) + x; the step and the balancing are skipped on the device when the CG met a non-finite
    // alpha/beta (reason 8 below leaves w = w^(k-1), as Alg. CG-dGN's caller in the oracle does)
    const CgState* gate = (const CgState*)c->cgState.p;
    TF_CUDA(c, launch_axpy_inplace(n, x, w, gate, c->stream));
    if (prm->balance) {
      if ((s = grams_impl(c, d, w, grams))) return s;
      TF_CUDA(c, launch_balance(m, grams, w, gate, c->stream));
    }
    if ((s = eval_global())) return s;                                   // F, grad at w^(k)
    if ((s = grams_impl(c, d, w, grams))) return s;
    TF_CUDA(c, launch_dots(n, grad, grad, grad, part, scal + 8, c->stream));   // [11] = ||grad||_inf
    c->total_launches += 12;
    if ((s = sync_scalars())) return s;
    if (c->cg_host->nonfinite) {
      why = 8;
      break;
    }
    const double Fn = hs[0], gx = hs[4], xjjx = hs[5], step = sqrt(hs[6]), ginf = hs[11];
    const double pred = -gx - 0.5 * xjjx;          // F(w_old) - 1/2 ||f + J x||^2
    const double g = (F - Fn) / pred;
    if (hist) {
      hist[5 * (k - 1) + 0] = Fn;
      hist[5 * (k - 1) + 1] = normT > 0 ? sqrt(2.0 * Fn) / normT : 0.0;
      hist[5 * (k - 1) + 2] = mu;
      hist[5 * (k - 1) + 3] = g;
      hist[5 * (k - 1) + 4] = step;
    }
    if (g < 0.25) mu *= 3.0;
    else if (g > 0.75) mu /= 3.0;
    F = Fn;
    it = k;
    rel[k] = normT > 0 ? sqrt(2.0 * F) / normT : 0.0;
    if (!std::isfinite(F)) {
      why = 8;
      break;
    }
    // stopping conditions in the order of PAPER.md:2756-2773
    if (rel[k] < tol) { why = 1; break; }
    if (step < tol) { why = 2; break; }
    if (fabs(rel[k - 1] - rel[k]) < tol) { why = 3; break; }
    if (ginf < tol) { why = 4; break; }
    if (k > 2 * cc && k % cc == 0) {
      double m1 = 0.0, m2 = 0.0, imp = 0.0;
      for (int t = k - 2 * cc; t < k - cc; ++t) m1 += rel[t];
      for (int t = k - cc; t < k; ++t) {
        m2 += rel[t];
        imp += fabs(rel[t] - rel[t + 1]);
      }
      m1 /= cc;
      m2 /= cc;
      imp /= cc;
      if (m1 - m2 < tol) { why = 5; break; }
      if (imp < 1e-3 * m2) { why = 6; break; }
    }
    if (rel[k] > std::max(1.0, normT2) / (1e-16 + tol)) { why = 7; break; }
  }
  res->iters = it;
  res->reason = why;
  res->f = F;
  res->rel_err = normT > 0 ? sqrt(2.0 * F) / normT : 0.0;
  res->mu = mu;
  return TF_OK;
}

}  // namespace

extern "C" {

tf_status tf_cpd_dgn(tf_ctx* c, tf_dims d, const double* T, double* w, const tf_dgn_params* prm, tf_dgn_result* res,
                     double* hist) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!T || !w || !prm || !res || (prm->maxiter > 0 && !prm->cg_iters)) return set_err(c, TF_ERR_ARG, "null pointer");
  if (d.K != d.K_total || d.k_begin != 0)
    return set_err(c, TF_ERR_UNSUPPORTED, "tf_cpd_dgn needs the whole tensor (K == K_total); use tf_cpd_dgn_sharded");
  if (prm->maxiter < 0) return set_err(c, TF_ERR_ARG, "maxiter < 0");
  cudaSetDevice(c->device);
  return dgn_impl(c, d, T, w, prm, res, hist, nullptr, nullptr, nullptr);
}

tf_status tf_cpd_dgn_sharded(tf_ctx* c, tf_dims d, const double* T, double* w, const tf_dgn_params* prm,
                             tf_dgn_result* res, double* hist, tf_allreduce_fn allreduce, void* user, double* xbuf) {
  tf_status s = check_dims(c, d);
  if (s) return s;
  if (!T || !w || !prm || !res || !allreduce || !xbuf || (prm->maxiter > 0 && !prm->cg_iters))
    return set_err(c, TF_ERR_ARG, "null pointer");
  if (prm->maxiter < 0) return set_err(c, TF_ERR_ARG, "maxiter < 0");
  cudaSetDevice(c->device);
  return dgn_impl(c, d, T, w, prm, res, hist, allreduce, user, xbuf);
}

tf_status tf_cg_solve(tf_ctx* c, tf_dims d, const double* grams, const double* w, const double* rhs, double lambda,
                      int maxiter, double tol, int jacobi, double* x, int* iters_done, double* res2) {
  return tf_cg_solve_damped(c, d, grams, w, rhs, lambda, nullptr, maxiter, tol, jacobi, x, iters_done, res2);
}

}  // extern "C"
