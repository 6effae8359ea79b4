// Shared device/host helpers for libkst_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: ranges cost ~nothing without a tool

#include "../../include/kst_b200.h"

typedef double2 cplx;  // (re, im) == numpy complex128 memory

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__host__ __device__ __forceinline__ cplx cmulc(cplx a, cplx b) {
  return cmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += a * conj(b)
__device__ __forceinline__ void cfmac(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfmca(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }

constexpr int kNumSMs = 148;  // B200

// ---------------------------------------------------------------- context
struct kst_ctx {
  int device = 0;
  std::string err;
  // grow-only device workspace slots (never shrink; freed at destroy)
  struct Slot {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  Slot slots[32];
  // pinned host staging for small device->host reads
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* cusolver = nullptr;  // cusolverDnHandle_t, created lazily (heig.cu fallback)
  void* cublas = nullptr;    // cublasHandle_t for the int8 Gram (gram_ozaki.cu)
  // K1 engine: 0 = FP64 DMMA tiles (gram.cu), 1 = int8 tensor-core slices
  // (gram_ozaki.cu) with `gram_slices` 7-bit slices per operand, 2 = int8
  // modular residues (gram_crt.cu) with `gram_slices` moduli on the hand-written
  // tcgen05 kernel, 3 = the same CRT numerics with cuBLAS int8 GEMMs
  int gram_mode = 0;
  int gram_slices = 7;
  double last_int8_ops = 0.0;  // int8 ops issued by the last int8 Gram (bench roofline)
  // instrumentation: kernel launches issued, and per-stage CUDA events of the
  // last kst_pipeline call (recorded only when profiling is on)
  // detection constants resident in the WS_DET workspace (conj grid,
  // Dopplers, twiddles): the key they were uploaded for
  const void* det_base = nullptr;
  std::vector<double> det_key;
  // K5 precision: 32 = FP32 prime-factor transform (detect_f32.cu) where it
  // applies, 64 = the FP64 kernels; position maps resident for f32_D
  int det_bits = 32;
  const void* f32_base = nullptr;
  int f32_D = 0;
  long long launches = 0;
  int profiling = 0;
  // NVTX ranges of the kst_pipeline stages (kst.scm, kst.lrkron, kst.bases,
  // kst.detect) and of the Gram's tensor-core span, for ncu --nvtx filters
  nvtxRangeId_t nvtx_stage = 0, nvtx_sub = 0;
  cudaEvent_t ev[8] = {};
  int n_ev = 0;
  // pageable host <-> device staging ring (hostio.cu): pinned chunks and the
  // events that guard their reuse
  void* stage = nullptr;
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev[32] = {};
};

// record stage boundary k on `st` when profiling (kst_pipeline)
inline void stage_mark(kst_ctx* ctx, int k, cudaStream_t st) {
  static const char* const kStage[4] = {"kst.scm", "kst.lrkron", "kst.bases", "kst.detect"};
  if (k <= 4) {
    if (ctx->nvtx_stage) nvtxRangeEnd(ctx->nvtx_stage);
    ctx->nvtx_stage = k < 4 ? nvtxRangeStartA(kStage[k]) : 0;
  } else if (k == 5) {
    ctx->nvtx_sub = nvtxRangeStartA("kst.gram.tensor");
  } else if (k == 6 && ctx->nvtx_sub) {
    nvtxRangeEnd(ctx->nvtx_sub);
    ctx->nvtx_sub = 0;
  }
  if (!ctx->profiling || k >= 8) return;
  if (!ctx->ev[k]) cudaEventCreate(&ctx->ev[k]);
  // inside a CUDA-graph capture (FrameGraph) the marks become event-record
  // nodes, so every replay re-times its stages
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ctx->ev[k], st, cudaEventRecordExternal);
  else
    cudaEventRecord(ctx->ev[k], st);
  if (k + 1 > ctx->n_ev) ctx->n_ev = k + 1;
}

enum WsSlot {
  WS_S = 0,        // pq x pq covariance (pipeline)
  WS_B = 1,        // q x q temporal iterate
  WS_PART = 2,     // per-CTA partial sums
  WS_SMALL = 3,    // small matrices / scalars (spatial iterate, flags)
  WS_EIG = 4,      // eigensolver block vectors
  WS_EIG2 = 5,     // eigensolver scratch
  WS_DET = 6,      // detection scratch (spectra / coefficients)
  WS_DET2 = 7,     // detection constants (twiddles, grids, bases spectra)
  WS_PREP = 8,     // Gram operand planes
  WS_UB = 9,       // pipeline temporal basis
  WS_UA = 10,      // pipeline spatial basis
  WS_VALS = 11,    // misc
  WS_CUSOLVER = 12, // cuSOLVER workspace (fallback path only)
  WS_TMP = 13,      // short-lived copies
  WS_PIPE_UB = 14,  // pipeline: temporal basis (lives until detection)
  WS_PIPE_T = 15,   // pipeline: full temporal factor (rank_temporal == q only)
  WS_PIPE_SP = 16,  // pipeline: spatial factor + spatial basis
  WS_BZ = 17,       // eigensolver: split-K partials of B*Z
  WS_OZ_SLICES = 18, // int8 Gram: operand slices + column exponents
  WS_OZ_PROD = 19,  // int8 Gram: int32 diagonal products
  WS_LM_SPEC = 20,  // L-mode: bin spectra (+ twiddle / grid constants)
  WS_LM_W = 21,     // L-mode: banded snapshot Gram + row sums
  WS_LM_E = 22,     // L-mode: per-test-bin projection matrices + window info
  WS_LM_H = 23,     // L-mode: per-CTA eigen scratch (small Grams, residuals)
  WS_DET32 = 24,    // FP32 detection: prime-factor position maps
  WS_PIPE_REC = 25  // pipeline: device outcome record of the sync-free form
};

// Every extern "C" entry point runs on its context's device: the caller's
// stream and the workspace slots belong to ctx->device, whatever device the
// calling thread has current.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

#define CTX_GUARD(ctx)                          \
  if (!(ctx)) return KST_ERR_DIMENSION;         \
  DeviceGuard guard__((ctx)->device);           \
  (ctx)->err.clear();

void* ws_get(kst_ctx* ctx, int slot, size_t bytes);  // may return nullptr on OOM
void* pinned_get(kst_ctx* ctx, size_t bytes);
// Upload `bytes` of host data to a __constant__ `symbol` on the current
// device unless it already holds exactly these bytes (constant plans are
// device-global; repeated frames with the same plan skip the small
// host->device transfer, which costs tens of us when PCIe is saturated by a
// cube upload).
int const_upload(kst_ctx* ctx, const void* symbol, const void* src, size_t bytes, cudaStream_t st);
// Resident-state epoch: bumped whenever device state that a captured CUDA
// graph of a frame depends on changes outside the graph (a workspace or pinned
// buffer reallocated, a constant bank uploaded, resident detection tables
// restaged). kst_state_epoch exports it; a graph captured at epoch e replays
// correctly while the epoch is still e.
void epoch_bump(const char* why = nullptr, long long tag = 0);

int set_err(kst_ctx* ctx, int code, const char* fmt, ...);

#define KST_CUDA(ctx, call)                                                               \
  do {                                                                                    \
    cudaError_t e__ = (call);                                                             \
    if (e__ != cudaSuccess)                                                               \
      return set_err((ctx), KST_ERR_CUDA, "%s failed: %s (%s:%d)", #call,                 \
                     cudaGetErrorString(e__), __FILE__, __LINE__);                        \
  } while (0)

#define KST_LAUNCH(ctx)                                                                   \
  do {                                                                                    \
    ++(ctx)->launches;                                                                    \
    cudaError_t e__ = cudaGetLastError();                                                 \
    if (e__ != cudaSuccess)                                                               \
      return set_err((ctx), KST_ERR_CUDA, "kernel launch failed: %s (%s:%d)",             \
                     cudaGetErrorString(e__), __FILE__, __LINE__);                        \
  } while (0)

#define KST_TRY(expr)              \
  do {                             \
    int rc__ = (expr);             \
    if (rc__ != KST_OK) return rc__; \
  } while (0)

static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ---------------------------------------------------------------- device reductions
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block sum (deterministic): every thread gets the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// ---------------------------------------------------------------- async copies
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Compile-time channel count dispatch (P = 1..16) for the per-channel kernels.
#define KST_DISPATCH_P(P, CALL)                        \
  switch (P) {                                         \
    case 1: { constexpr int PP = 1; CALL; } break;     \
    case 2: { constexpr int PP = 2; CALL; } break;     \
    case 3: { constexpr int PP = 3; CALL; } break;     \
    case 4: { constexpr int PP = 4; CALL; } break;     \
    case 5: { constexpr int PP = 5; CALL; } break;     \
    case 6: { constexpr int PP = 6; CALL; } break;     \
    case 7: { constexpr int PP = 7; CALL; } break;     \
    case 8: { constexpr int PP = 8; CALL; } break;     \
    case 9: { constexpr int PP = 9; CALL; } break;     \
    case 10: { constexpr int PP = 10; CALL; } break;   \
    case 11: { constexpr int PP = 11; CALL; } break;   \
    case 12: { constexpr int PP = 12; CALL; } break;   \
    case 13: { constexpr int PP = 13; CALL; } break;   \
    case 14: { constexpr int PP = 14; CALL; } break;   \
    case 15: { constexpr int PP = 15; CALL; } break;   \
    default: { constexpr int PP = 16; CALL; } break;   \
  }

// ---------------------------------------------------------------- internal API between units
namespace kst {
// gram.cu (dispatches to gram_ozaki.cu when ctx->gram_mode == 1)
int scm(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, cudaStream_t st);
// gram_ozaki.cu
bool ozaki_available();
int scm_ozaki(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, int s, cudaStream_t st);
// gram_crt.cu: modular (CRT) int8 Gram with `nmod` moduli (8..16); crt_beta
// is the integer scaling it uses for n snapshots (-1 if unsupported)
int scm_crt(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, int nmod, bool use_tc,
            cudaStream_t st);
bool crt_tc_available();  // cuTensorMapEncodeTiled reachable (tcgen05 path)
int crt_beta(int nmod, int64_t n);
// heig.cu
struct TopEig {
  int r = 0;
  std::vector<double> values;  // descending, host
  cplx* vectors = nullptr;     // dev (n, r) row-major
};
int heig_top(kst_ctx* ctx, const cplx* M, int n, int r, double* values_host, cplx* vectors,
             cudaStream_t st, int* ok_dev = nullptr, const double** values_dev_out = nullptr,
             const double* mdiag = nullptr /* Re diag(M), contiguous (optional) */);
int small_heig(kst_ctx* ctx, const cplx* M, int n, double* values_dev, cplx* vectors_dev,
               cudaStream_t st);
int truncate_from_pairs(kst_ctx* ctx, const double* values_host, const cplx* vectors, int n,
                        int r, double top_abs, cplx* out, cudaStream_t st);
int eig_truncate(kst_ctx* ctx, const cplx* M, int n, int rank, cplx* out, cudaStream_t st);
int subspace_basis(kst_ctx* ctx, const cplx* M, int n, int rank, double tol, cplx* basis, int* keep,
                   cudaStream_t st);
int herm_check(kst_ctx* ctx, const cplx* M, int n, cudaStream_t st);  // DataError if not Hermitian
// lrkron.cu
struct FitOut {
  int iterations = 0, converged = 0, n_res = 0;
  std::vector<double> residuals;
};
int lrkron(kst_ctx* ctx, const cplx* S, int p, int q, int ra, int rb, double tol, int max_iter,
           int validate, cplx* spatial, cplx* temporal, cplx* tb_vectors, double* tb_values,
           FitOut* fit, cplx* iter_spatial, cplx* iter_b, cudaStream_t st);
int lrkron_async(kst_ctx* ctx, const cplx* S, int p, int q, int ra, int rb, double tol, int max_iter,
                 cplx* spatial, cplx* tb_vectors, int* heig_ok, const double** tb_vals_dev,
                 const double** dres_out, const double** diag_out, cudaStream_t st);
// detect.cu
int detect(kst_ctx* ctx, const cplx* cube, int64_t n, int p, int q, const cplx* ua, int ka,
           const cplx* ub, int kb, int kind, int spatial_only, const double* dop_host, int D,
           const cplx* grid_host, int G, int groups, double* values, cudaStream_t st,
           bool check_finite = true);
int spectra(kst_ctx* ctx, const cplx* x, int64_t rows, int q, const double* dop_host, int D,
            cplx* spec, void* consts, cudaStream_t st);
// detect_f32.cu: FP32 single-map detection (uniform grid); -1 = not taken
bool detect_f32_supported(int p, int q, int ka, int kb, int mode, int spatial, int D, int G);
int detect_f32(kst_ctx* ctx, const cplx* cube, int64_t n, int p, int q, const cplx* ua, int ka,
               const cplx* ub, int kb, int mode, int spatial, int D, const cplx* ubspec,
               const cplx* tw, const cplx* hconj, const cplx* grid_host, int G, bool dft,
               double* values, int* flag, cudaStream_t st);
}  // namespace kst
