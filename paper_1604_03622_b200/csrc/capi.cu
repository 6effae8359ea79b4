// C ABI of libkst_b200.so (declared in include/kst_b200.h): context,
// workspace and the extern "C" entry points. No C++ exception crosses it.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>

#include "common.cuh"

int set_err(kst_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

static std::atomic<long long> g_epoch{1};
void epoch_bump(const char* why, long long tag) {
  g_epoch.fetch_add(1);
  static const bool dbg = getenv("KST_EPOCH_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "[kst] state epoch bump: %s %lld\n", why ? why : "?", tag);
}

void* ws_get(kst_ctx* ctx, int slot, size_t bytes) {
  auto& s = ctx->slots[slot];
  if (bytes == 0) bytes = 1;
  if (s.bytes >= bytes) return s.ptr;
  epoch_bump("workspace", slot);
  if (s.ptr) {
    // in-flight kernels may still read the old buffer
    cudaDeviceSynchronize();
    cudaFree(s.ptr);
    s.ptr = nullptr;
    s.bytes = 0;
  }
  size_t want = bytes + bytes / 8 + 256;
  if (cudaMalloc(&s.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    s.ptr = nullptr;
    return nullptr;
  }
  s.bytes = want;
  return s.ptr;
}

int const_upload(kst_ctx* ctx, const void* symbol, const void* src, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, std::vector<char>> held;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto& cur = held[{dev, symbol}];
  if (cur.size() == bytes && std::memcmp(cur.data(), src, bytes) == 0) return KST_OK;
  epoch_bump("constant", (long long)(uintptr_t)symbol);
  const cudaError_t e = cudaMemcpyToSymbolAsync(symbol, src, bytes, 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cur.clear();
    return set_err(ctx, KST_ERR_CUDA, "constant upload: %s", cudaGetErrorString(e));
  }
  cur.assign((const char*)src, (const char*)src + bytes);
  return KST_OK;
}

void* pinned_get(kst_ctx* ctx, size_t bytes) {
  if (ctx->pinned_bytes >= bytes) return ctx->pinned;
  epoch_bump("pinned", (long long)bytes);
  if (ctx->pinned) {
    cudaDeviceSynchronize();
    cudaFreeHost(ctx->pinned);
  }
  size_t want = std::max<size_t>(bytes, 1 << 16);
  if (cudaMallocHost(&ctx->pinned, want) != cudaSuccess) {
    cudaGetLastError();
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    return nullptr;
  }
  ctx->pinned_bytes = want;
  return ctx->pinned;
}

// ---------------------------------------------------------------- optimistic pipeline
// Device forms of the host decisions of kst_pipeline's common case, so a frame
// runs without a stream synchronisation until its end:
//
// spatial_basis_kernel: subspace_basis(spatial, r_a) (src/filters.py:58-73)
//   from the Jacobi pairs of the P x P spatial factor: the Hermitian check of
//   herm_check, the kept count k (values > 1e-9 of the top one, <= r), and
//   the first r eigenvectors copied with pitch r (the caller assumed k = r).
__global__ void spatial_basis_kernel(const cplx* __restrict__ M, int p, const double* __restrict__ vals,
                                     const cplx* __restrict__ vecs, int r, cplx* __restrict__ ua,
                                     int* __restrict__ flags) {
  if (threadIdx.x == 0) {
    double f = 0.0, a = 0.0;
    int bad = 0;
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) {
        const cplx x = M[i * p + j], y = M[j * p + i];
        if (!isfinite(x.x) || !isfinite(x.y)) bad = 1;
        f += cabs2(x);
        a += cabs2(cmk(x.x - y.x, x.y + y.y));
      }
    const double scale = sqrt(f);
    flags[0] = (!bad && !(scale > 0 && sqrt(a) > 1e-8 * scale)) ? 1 : 0;  // Hermitian
    int k = 0;
    const double top = vals[0];
    if (top > 0.0)
      while (k < r && vals[k] > 1e-9 * top) ++k;
    flags[1] = k;
  }
  for (int e = threadIdx.x; e < p * r; e += blockDim.x) {
    const int i = e / r, c = e % r;
    ua[e] = vecs[i * p + c];
  }
}

// pipeline_check_kernel: the kept temporal rank from the top-r_b values of b
// (capi: clamp of src/linalg.py:138-140, keep rule src/filters.py:70) and the
// validation of every assumption of the optimistic schedule; rec =
// {ok, iterations, converged, ka, kb, last residual}.
__global__ void pipeline_check_kernel(const double* __restrict__ tbv, int rb, const double* __restrict__ dres,
                                      int max_iter, const double* __restrict__ diag,
                                      const int* __restrict__ heig_ok, const int* __restrict__ flags,
                                      int ka_assumed, double* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  double top = 0.0;
  for (int k = 0; k < rb; ++k) top = fmax(top, fabs(tbv[k]));
  double v0 = tbv[0];
  if (v0 < 0 && fabs(v0) <= 1e-10 * top) v0 = 0.0;
  int kb = 0;
  if (v0 > 0.0)
    while (kb < rb) {
      double v = tbv[kb];
      if (v < 0 && fabs(v) <= 1e-10 * top) v = 0.0;
      if (!(v > 1e-9 * v0)) break;
      ++kb;
    }
  const int status = (int)dres[max_iter], iters = (int)dres[max_iter + 1],
            conv = (int)dres[max_iter + 2];
  const bool ok = status == 0 && diag[0] == 0.0 && diag[3] > 0.0 && iters >= 1 && *heig_ok == 1 &&
                  flags[0] == 1 && flags[1] == ka_assumed && kb == rb;
  rec[0] = ok ? 1.0 : 0.0;
  rec[1] = iters;
  rec[2] = conv;
  rec[3] = flags[1];
  rec[4] = kb;
  rec[5] = iters >= 1 ? dres[iters - 1] : 0.0;
}

extern "C" {

int kst_version(void) { return 1; }

int kst_ctx_create(int device, kst_ctx** out) {
  if (!out) return KST_ERR_DIMENSION;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    return KST_ERR_CUDA;
  }
  kst_ctx* c = new (std::nothrow) kst_ctx();
  if (!c) return KST_ERR_CUDA;
  c->device = device;
  // K1 engine default: the CRT int8 Gram on the hand-written tcgen05 kernel
  // with 10 moduli (x rounded to >= 32 bits; measured at full size: spatial
  // factor 5e-13, projectors 1e-13, residuals at their 1e-10 floor, see
  // gram_crt.cu / DESIGN.md); else int8 slices (6) with cuBLAS; else FP64 DMMA.
  // Override: KST_GRAM=crt|crt-cublas|int8|dmma, KST_GRAM_SLICES (moduli or slices).
  const bool i8 = kst::ozaki_available(), tc = kst::crt_tc_available();
  c->gram_mode = tc ? 2 : i8 ? 1 : 0;
  c->gram_slices = tc ? 10 : 6;
  if (const char* e = getenv("KST_GRAM")) {
    c->gram_mode = (strcmp(e, "int8") == 0 && i8)               ? 1
                   : (strcmp(e, "crt") == 0 && tc)              ? 2
                   : (strcmp(e, "crt-cublas") == 0 && i8)       ? 3
                                                                : 0;
    c->gram_slices = c->gram_mode >= 2 ? 10 : 6;
  }
  if (const char* e = getenv("KST_GRAM_SLICES"))
    c->gram_slices = c->gram_mode >= 2 ? std::min(14, std::max(8, atoi(e)))
                                       : std::min(8, std::max(3, atoi(e)));
  // K5 precision default: FP32 transform; KST_DETECT=f64 overrides
  if (const char* e = getenv("KST_DETECT")) c->det_bits = strcmp(e, "f64") == 0 ? 64 : 32;
  DeviceGuard g(device);
  cudaFree(nullptr);  // establish the primary context
  *out = c;
  return KST_OK;
}

int kst_ctx_destroy(kst_ctx* ctx) {
  if (!ctx) return KST_OK;
  {
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    for (auto& s : ctx->slots)
      if (s.ptr) cudaFree(s.ptr);
    for (auto& e : ctx->ev)
      if (e) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->stage) cudaFreeHost(ctx->stage);
    for (auto& e : ctx->stage_ev)
      if (e) cudaEventDestroy(e);
  }
  delete ctx;
  return KST_OK;
}

const char* kst_last_error(const kst_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

long long kst_launch_count(const kst_ctx* ctx) { return ctx ? ctx->launches : -1; }

int kst_set_gram(kst_ctx* ctx, int mode, int slices) {
  if (!ctx) return KST_ERR_DIMENSION;
  if (mode < 0 || mode > 3) return set_err(ctx, KST_ERR_DIMENSION, "gram mode must be 0..3");
  if (mode == 1 && (slices < 3 || slices > 8))
    return set_err(ctx, KST_ERR_DIMENSION, "int8 Gram needs 3..8 slices, got %d", slices);
  if (mode == 2 && !kst::crt_tc_available())
    return set_err(ctx, KST_ERR_CUDA, "tcgen05 CRT Gram unavailable: no cuTensorMapEncodeTiled");
  if (mode >= 2 && (slices < 8 || slices > 14))
    return set_err(ctx, KST_ERR_DIMENSION, "CRT Gram needs 8..14 moduli, got %d", slices);
  if (mode != 0 && !kst::ozaki_available())
    return set_err(ctx, KST_ERR_CUDA, "int8 Gram unavailable: cuBLAS not loadable");
  ctx->gram_mode = mode;
  if (mode != 0) ctx->gram_slices = slices;
  return KST_OK;
}

int kst_set_detect(kst_ctx* ctx, int bits) {
  if (!ctx) return KST_ERR_DIMENSION;
  if (bits != 32 && bits != 64) return set_err(ctx, KST_ERR_DIMENSION, "detection precision must be 32 or 64");
  ctx->det_bits = bits;
  return KST_OK;
}

int kst_get_detect(const kst_ctx* ctx, int* bits) {
  if (!ctx) return KST_ERR_DIMENSION;
  if (bits) *bits = ctx->det_bits;
  return KST_OK;
}

double kst_gram_int8_ops(const kst_ctx* ctx) { return ctx ? ctx->last_int8_ops : 0.0; }

int kst_get_gram(const kst_ctx* ctx, int* mode, int* slices) {
  if (!ctx) return KST_ERR_DIMENSION;
  if (mode) *mode = ctx->gram_mode;
  if (slices) *slices = ctx->gram_slices;
  return KST_OK;
}

int kst_set_profiling(kst_ctx* ctx, int on) {
  if (!ctx) return KST_ERR_DIMENSION;
  ctx->profiling = on;
  ctx->n_ev = 0;
  return KST_OK;
}

int kst_stage_times(kst_ctx* ctx, double* ms, int max) {
  if (!ctx) return KST_ERR_DIMENSION;
  DeviceGuard g(ctx->device);
  int k = 0;
  for (; k + 1 < ctx->n_ev && k < max; ++k) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, ctx->ev[k], ctx->ev[k + 1]) != cudaSuccess) {
      cudaGetLastError();
      t = -1.f;
    }
    ms[k] = t;
  }
  return k;
}

int kst_scm(kst_ctx* ctx, const double* X, int64_t n, int64_t d, double* S, void* stream) {
  CTX_GUARD(ctx);
  return kst::scm(ctx, (const cplx*)X, n, d, (cplx*)S, (cudaStream_t)stream);
}

int kst_lrkron(kst_ctx* ctx, const double* S, int p, int q, int rank_spatial, int rank_temporal,
               double tol, int max_iter, int validate, double* spatial, double* temporal,
               double* tb_vectors, double* tb_values, double* residuals, int* n_residuals,
               int* iterations, int* converged, double* iter_spatial, double* iter_b,
               void* stream) {
  CTX_GUARD(ctx);
  kst::FitOut fit;
  int rc = kst::lrkron(ctx, (const cplx*)S, p, q, rank_spatial, rank_temporal, tol, max_iter,
                       validate, (cplx*)spatial, (cplx*)temporal, (cplx*)tb_vectors, tb_values,
                       &fit, (cplx*)iter_spatial, (cplx*)iter_b, (cudaStream_t)stream);
  if (iterations) *iterations = fit.iterations;
  if (converged) *converged = fit.converged;
  if (n_residuals) *n_residuals = fit.n_res;
  if (residuals)
    for (int k = 0; k < fit.n_res; ++k) residuals[k] = fit.residuals[k];
  return rc;
}

int kst_heig_top(kst_ctx* ctx, const double* M, int n, int r, double* values, double* vectors,
                 void* stream) {
  CTX_GUARD(ctx);
  KST_TRY(kst::herm_check(ctx, (const cplx*)M, n, (cudaStream_t)stream));
  return kst::heig_top(ctx, (const cplx*)M, n, r, values, (cplx*)vectors, (cudaStream_t)stream);
}

int kst_eig_truncate(kst_ctx* ctx, const double* M, int n, int rank, double* out, void* stream) {
  CTX_GUARD(ctx);
  return kst::eig_truncate(ctx, (const cplx*)M, n, rank, (cplx*)out, (cudaStream_t)stream);
}

int kst_subspace_basis(kst_ctx* ctx, const double* M, int n, int rank, double tol, double* basis,
                       int* keep, void* stream) {
  CTX_GUARD(ctx);
  return kst::subspace_basis(ctx, (const cplx*)M, n, rank, tol, (cplx*)basis, keep,
                             (cudaStream_t)stream);
}

int kst_detect(kst_ctx* ctx, const double* cube, int64_t n, int p, int q, const double* ua, int ka,
               const double* ub, int kb, int kind, int spatial_only, const double* dopplers, int D,
               const double* grid, int G, int groups, double* values, void* stream) {
  CTX_GUARD(ctx);
  return kst::detect(ctx, (const cplx*)cube, n, p, q, (const cplx*)ua, ka, (const cplx*)ub, kb, kind,
                     spatial_only, dopplers, D, (const cplx*)grid, G, groups, values,
                     (cudaStream_t)stream);
}

// The sync-free form of a frame applies (p <= 4, q > 64 for heig_top's
// block solver, r_b <= 24 and < q)
static bool pipeline_async_ok(int p, int q, int rank_spatial, int rank_temporal, int max_iter) {
  return rank_temporal != q && p <= 4 && q > 64 /* heig_top Jacobi limit */ && rank_spatial >= 1 &&
         rank_spatial <= p && rank_temporal >= 1 && rank_temporal <= 24 && max_iter >= 1;
}

// Enqueue the whole frame with every decision (convergence, kept ranks,
// validity) taken on the device; rec (device, 8 doubles) receives
// [ok, iterations, converged, ka, kb, last residual]. No host
// synchronisation, no allocation once the workspaces exist: capturable in a
// CUDA graph after one call with the same arguments.
static int pipeline_async_core(kst_ctx* ctx, const double* cube, int64_t n, int p, int q, int rank_spatial,
                               int rank_temporal, double tol, int max_iter, int kind,
                               const double* dopplers, int D, const double* grid, int G, int groups,
                               double* values, double* rec_out, cudaStream_t st) {
  const int64_t d = (int64_t)p * q;
  cplx* S = (cplx*)ws_get(ctx, WS_S, sizeof(cplx) * d * d);
  cplx* ubA = (cplx*)ws_get(ctx, WS_PIPE_UB, sizeof(cplx) * (size_t)q * rank_temporal * 2 + 64);
  // spatial (p^2) | ua (p^2) | Jacobi vectors (p^2) | values (p) | rec (8) | flags
  char* sp = (char*)ws_get(ctx, WS_PIPE_SP, sizeof(cplx) * p * p * 3 + sizeof(double) * (p + 8) + 64);
  if (!S || !ubA || !sp) return set_err(ctx, KST_ERR_CUDA, "pipeline: workspace");
  cplx* spA = (cplx*)sp;
  cplx* uaA = spA + p * p;
  cplx* vecA = uaA + p * p;
  double* valA = (double*)(vecA + p * p);
  double* rec = rec_out ? rec_out : valA + p;
  int* flags = (int*)(valA + p + 8);
  int* heig_ok = flags + 2;
  stage_mark(ctx, 0, st);
  KST_TRY(kst::scm(ctx, (const cplx*)cube, n, d, S, st));
  stage_mark(ctx, 1, st);
  const double* tbv_dev = nullptr;
  const double* dres = nullptr;
  const double* diag = nullptr;
  KST_TRY(kst::lrkron_async(ctx, S, p, q, rank_spatial, rank_temporal, tol, max_iter, spA, ubA, heig_ok,
                            &tbv_dev, &dres, &diag, st));
  stage_mark(ctx, 2, st);
  KST_TRY(kst::small_heig(ctx, spA, p, valA, vecA, st));
  const int ka = rank_spatial;
  spatial_basis_kernel<<<1, 32, 0, st>>>(spA, p, valA, vecA, ka, uaA, flags);
  KST_LAUNCH(ctx);
  stage_mark(ctx, 3, st);
  KST_TRY(kst::detect(ctx, (const cplx*)cube, n, p, q, uaA, ka, ubA, rank_temporal, kind, 0, dopplers, D,
                      (const cplx*)grid, G, groups, values, st, false));
  stage_mark(ctx, 4, st);
  pipeline_check_kernel<<<1, 32, 0, st>>>(tbv_dev, rank_temporal, dres, max_iter, diag, heig_ok, flags, ka,
                                          rec);
  KST_LAUNCH(ctx);
  return KST_OK;
}

int kst_pipeline_async(kst_ctx* ctx, const double* cube, int64_t n, int p, int q, int rank_spatial,
                       int rank_temporal, double tol, int max_iter, int kind, const double* dopplers,
                       int D, const double* grid, int G, int groups, double* values, double* rec,
                       void* stream) {
  CTX_GUARD(ctx);
  if (n < 1 || p < 1 || q < 1) return set_err(ctx, KST_ERR_DIMENSION, "pipeline: empty cube");
  if (!rec) return set_err(ctx, KST_ERR_DIMENSION, "pipeline_async: rec buffer required");
  if (!pipeline_async_ok(p, q, rank_spatial, rank_temporal, max_iter))
    return set_err(ctx, KST_ERR_DIMENSION,
                   "pipeline_async: shape outside the sync-free form (p <= 4, q > 64, "
                   "1 <= rank_temporal <= 24, rank_temporal < q)");
  return pipeline_async_core(ctx, cube, n, p, q, rank_spatial, rank_temporal, tol, max_iter, kind, dopplers,
                             D, grid, G, groups, values, rec, (cudaStream_t)stream);
}

long long kst_state_epoch(void) { return g_epoch.load(); }

int kst_pipeline(kst_ctx* ctx, const double* cube, int64_t n, int p, int q, int rank_spatial,
                 int rank_temporal, double tol, int max_iter, int kind, const double* dopplers,
                 int D, const double* grid, int G, int groups, double* values, double* summary,
                 void* stream) {
  CTX_GUARD(ctx);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t d = (int64_t)p * q;
  if (n < 1 || p < 1 || q < 1) return set_err(ctx, KST_ERR_DIMENSION, "pipeline: empty cube");
  const bool full_b = rank_temporal == q;
  // Optimistic host-sync-free form of the common case: estimator, bases and
  // detection are enqueued back to back with every decision taken on the
  // device (pipeline_async_core); ONE synchronisation reads the outcome.
  // When any assumption fails (non-finite or zero S, a degenerate iterate,
  // the eigensolver needing more than one round, k_A < r_A, k_B < r_B) the
  // frame is recomputed from S by the synchronous path below, so results
  // equal the synchronous path's either way.
  static const bool async_env = !(getenv("KST_PIPE_ASYNC") && atoi(getenv("KST_PIPE_ASYNC")) == 0);
  if (async_env && pipeline_async_ok(p, q, rank_spatial, rank_temporal, max_iter)) {
    double* hrec = (double*)pinned_get(ctx, 256);
    if (!hrec) return set_err(ctx, KST_ERR_CUDA, "pipeline: workspace");
    double* rec = (double*)ws_get(ctx, WS_PIPE_REC, 64 * sizeof(double));
    if (!rec) return set_err(ctx, KST_ERR_CUDA, "pipeline: workspace");
    KST_TRY(pipeline_async_core(ctx, cube, n, p, q, rank_spatial, rank_temporal, tol, max_iter, kind,
                                dopplers, D, grid, G, groups, values, rec, st));
    KST_CUDA(ctx, cudaMemcpyAsync(hrec, rec, sizeof(double) * 6, cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    if (hrec[0] == 1.0) {
      if (summary) {
        summary[0] = hrec[1];
        summary[1] = hrec[2];
        summary[2] = hrec[3];
        summary[3] = hrec[4];
        summary[4] = hrec[5];
        summary[5] = summary[6] = summary[7] = 0.0;
      }
      return KST_OK;
    }
    // an assumption failed: the synchronous path recomputes from S
  }
  cplx* S = (cplx*)ws_get(ctx, WS_S, sizeof(cplx) * d * d);
  cplx* spatial = (cplx*)ws_get(ctx, WS_PIPE_SP, sizeof(cplx) * p * p * 3 + sizeof(double) * (p + 8) + 64);
  if (!S || !spatial) return set_err(ctx, KST_ERR_CUDA, "pipeline: workspace");
  cplx* ua = spatial + p * p;
  const bool s_ready = async_env && pipeline_async_ok(p, q, rank_spatial, rank_temporal, max_iter);
  if (!s_ready) {
    stage_mark(ctx, 0, st);
    KST_TRY(kst::scm(ctx, (const cplx*)cube, n, d, S, st));
    stage_mark(ctx, 1, st);
  }
  // ub: the top-rb eigenvectors (q x rb), then the kept kb columns repacked (q x kb)
  cplx* ub = (cplx*)ws_get(ctx, WS_PIPE_UB, sizeof(cplx) * (size_t)q * rank_temporal * 2 + 64);
  cplx* temporal = full_b ? (cplx*)ws_get(ctx, WS_PIPE_T, sizeof(cplx) * (size_t)q * q) : nullptr;
  if (!ub || (full_b && !temporal)) return set_err(ctx, KST_ERR_CUDA, "pipeline: workspace");
  std::vector<double> tbv(rank_temporal > 0 ? rank_temporal : 1);
  kst::FitOut fit;
  KST_TRY(kst::lrkron(ctx, S, p, q, rank_spatial, rank_temporal, tol, max_iter, 0, spatial,
                      temporal, full_b ? nullptr : ub, full_b ? nullptr : tbv.data(), &fit,
                      nullptr, nullptr, st));
  stage_mark(ctx, 2, st);
  // build_filter (src/filters.py:164-175): U_A from the spatial factor
  int ka = 0, kb = 0;
  KST_TRY(kst::subspace_basis(ctx, spatial, p, rank_spatial, 1e-9, ua, &ka, st));
  if (full_b) {
    KST_TRY(kst::subspace_basis(ctx, temporal, q, rank_temporal, 1e-9, ub, &kb, st));
  } else if (tbv[0] > 0.0) {
    while (kb < rank_temporal && tbv[kb] > 1e-9 * tbv[0]) ++kb;
  }
  // kb < rb (b of rank below r_b): detect takes a q x kb basis
  const cplx* ubk = ub;
  if (!full_b && kb > 0 && kb < rank_temporal) {
    cplx* packed = ub + (size_t)q * rank_temporal;
    KST_CUDA(ctx, cudaMemcpy2DAsync(packed, sizeof(cplx) * kb, ub, sizeof(cplx) * rank_temporal,
                                    sizeof(cplx) * kb, q, cudaMemcpyDeviceToDevice, st));
    ubk = packed;
  }
  stage_mark(ctx, 3, st);
  KST_TRY(kst::detect(ctx, (const cplx*)cube, n, p, q, ka ? ua : nullptr, ka, kb ? ubk : nullptr, kb,
                      kind, 0, dopplers, D, (const cplx*)grid, G, groups, values, st,
                      /*check_finite=*/false));  // a non-finite cube already failed lrkron
  stage_mark(ctx, 4, st);
  if (summary) {
    summary[0] = fit.iterations;
    summary[1] = fit.converged;
    summary[2] = ka;
    summary[3] = kb;
    summary[4] = fit.residuals.empty() ? 0.0 : fit.residuals.back();
    summary[5] = summary[6] = summary[7] = 0.0;
  }
  return KST_OK;
}

int kst_windowed(kst_ctx* ctx, const double* cube, int64_t a, int64_t n_bins, int p, int q, int n_w,
                 int64_t lo, int64_t hi, int64_t s_begin, int64_t s_end, int64_t s_step,
                 int rank_spatial, int rank_temporal, double tol, int max_iter, int kind,
                 int drop_temporal, const double* dopplers, int D, const double* grid, int G,
                 double* values, void* stream) {
  CTX_GUARD(ctx);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t d = (int64_t)p * q;
  if (p < 1 || q < 1 || n_w < 1 || n_w > n_bins || lo < 0 || hi > n_bins || lo >= hi || s_step < 1 ||
      a < 0 || a > lo)
    return set_err(ctx, KST_ERR_DIMENSION, "windowed: bad window / tile arguments");
  if (rank_temporal == q)  // the fused path keeps only the top rb eigenvectors of b
    return set_err(ctx, KST_ERR_DIMENSION, "windowed: rank_temporal == q needs the step API");
  cplx* S = (cplx*)ws_get(ctx, WS_S, sizeof(cplx) * d * d);
  cplx* spatial = (cplx*)ws_get(ctx, WS_PIPE_SP, sizeof(cplx) * p * p * 2 + 64);
  // ub: the top-rb eigenvectors (q x rb), then the kept kb columns repacked (q x kb)
  cplx* ub = (cplx*)ws_get(ctx, WS_PIPE_UB, sizeof(cplx) * (size_t)q * rank_temporal * 2 + 64);
  if (!S || !spatial || !ub) return set_err(ctx, KST_ERR_CUDA, "windowed: workspace");
  cplx* ua = spatial + p * p;
  std::vector<double> tbv(rank_temporal > 0 ? rank_temporal : 1);
  const cplx* X = (const cplx*)cube;  // bin a of the frame at row 0
  const int h = n_w / 2;
  // Window Grams run on the FP64 DMMA engine whatever the context's K1
  // engine: a window's b can have rank n_w r_a < r_b, and the CRT engine's
  // 2^-32 column rounding lifts its null eigenvalues to ~1e-10 of the top
  // one -- close enough to the 1e-9 keep threshold (src/filters.py:70) to
  // admit a spurious basis vector. FP64 keeps them at ~1e-16 (measured at
  // n_w = 1, r_b = 2).
  struct EngineGuard {
    kst_ctx* c;
    int mode;
    ~EngineGuard() { c->gram_mode = mode; }
  } eg{ctx, ctx->gram_mode};
  ctx->gram_mode = 0;
  // and the per-window detection runs in FP64 like the batched L-mode
  // detector (lmode.cu lm_detect_kernel), whatever the context's K5 precision
  struct DetGuard {
    kst_ctx* c;
    int bits;
    ~DetGuard() { c->det_bits = bits; }
  } dg{ctx, ctx->det_bits};
  ctx->det_bits = 64;
  for (int64_t s = s_begin; s < s_end; s += s_step) {
    if (s < 0 || s + n_w > n_bins || s < a)
      return set_err(ctx, KST_ERR_DIMENSION, "windowed: window %lld outside the cube",
                     (long long)s);
    // training: bins [s, s + n_w) (SURVEY.md §8 L-mode definition)
    KST_TRY(kst::scm(ctx, X + (s - a) * d, n_w, d, S, st));
    kst::FitOut fit;
    std::fill(tbv.begin(), tbv.end(), 0.0);
    KST_TRY(kst::lrkron(ctx, S, p, q, rank_spatial, rank_temporal, tol, max_iter, 1, spatial,
                        nullptr, ub, tbv.data(), &fit, nullptr, nullptr, st));
    int ka = 0, kb = 0;
    KST_TRY(kst::subspace_basis(ctx, spatial, p, rank_spatial, 1e-9, ua, &ka, st));
    if (tbv[0] > 0.0)
      while (kb < rank_temporal && tbv[kb] > 1e-9 * tbv[0]) ++kb;
    // kb < rb (a window's b of rank n_w r_a < r_b): detect takes a q x kb basis
    const cplx* ubk = ub;
    if (kb > 0 && kb < rank_temporal) {
      cplx* packed = ub + (size_t)q * rank_temporal;
      KST_CUDA(ctx, cudaMemcpy2DAsync(packed, sizeof(cplx) * kb, ub, sizeof(cplx) * rank_temporal,
                                      sizeof(cplx) * kb, q, cudaMemcpyDeviceToDevice, st));
      ubk = packed;
    }
    // test bins sharing window s (windowed.window_bins), clipped to the tile
    int64_t t0 = (s == 0) ? 0 : s + h, t1 = (s == n_bins - n_w) ? n_bins : s + h + 1;
    t0 = std::max(t0, lo);
    t1 = std::min(t1, hi);
    if (t1 <= t0) continue;
    KST_TRY(kst::detect(ctx, X + (t0 - a) * d, t1 - t0, p, q, ka ? ua : nullptr, ka,
                        kb ? ubk : nullptr, kb, kind, drop_temporal, dopplers, D,
                        (const cplx*)grid, G, 1, values + (t0 - lo) * D, st, false));
  }
  return KST_OK;
}

}  // extern "C"
