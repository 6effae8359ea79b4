// "optimal" (covariance-whitening) filter -- src/filters.py:137-163 (build_filter
// kind "optimal": scipy cho_factor(sigma, lower=True)) and src/filters.py:98-100
// (apply_matrix: cho_solve). SURVEY.md §8f rank 4.
//
// The factor is the lower Cholesky factor of the Hermitian matrix defined by
// sigma's lower triangle (cho_factor reads only that triangle), kept on the
// device in column-major order; solves take the cube as it lies in HBM: an
// (n, p, q) C-order cube is the column-major (pq x n) right-hand-side matrix
// with one snapshot per column, so every bin is solved by one zpotrs call.
// Dense factorisation / triangular solves are plain library calls (cuSOLVER,
// bound with dlopen like the eigensolver fallback in heig.cu); the layout
// change and the validation scans are ours.
#include <cusolverDn.h>
#include <dlfcn.h>

#include "common.cuh"

namespace {

struct Chol {
  bool tried = false, ok = false;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*potrf_bufsize)(cusolverDnHandle_t, cublasFillMode_t, int, cuDoubleComplex*,
                                    int, int*) = nullptr;
  cusolverStatus_t (*potrf)(cusolverDnHandle_t, cublasFillMode_t, int, cuDoubleComplex*, int,
                            cuDoubleComplex*, int, int*) = nullptr;
  cusolverStatus_t (*potrs)(cusolverDnHandle_t, cublasFillMode_t, int, int, const cuDoubleComplex*,
                            int, cuDoubleComplex*, int, int*) = nullptr;
};
Chol g_chol;

bool load_chol() {
  if (g_chol.tried) return g_chol.ok;
  g_chol.tried = true;
  const char* names[] = {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return false;
  g_chol.create = (decltype(g_chol.create))dlsym(h, "cusolverDnCreate");
  g_chol.set_stream = (decltype(g_chol.set_stream))dlsym(h, "cusolverDnSetStream");
  g_chol.potrf_bufsize = (decltype(g_chol.potrf_bufsize))dlsym(h, "cusolverDnZpotrf_bufferSize");
  g_chol.potrf = (decltype(g_chol.potrf))dlsym(h, "cusolverDnZpotrf");
  g_chol.potrs = (decltype(g_chol.potrs))dlsym(h, "cusolverDnZpotrs");
  g_chol.ok = g_chol.create && g_chol.set_stream && g_chol.potrf_bufsize && g_chol.potrf &&
              g_chol.potrs;
  return g_chol.ok;
}

int solver_handle(kst_ctx* ctx, cudaStream_t st, cusolverDnHandle_t* out) {
  if (!load_chol()) return set_err(ctx, KST_ERR_CUDA, "optimal filter: cuSOLVER not loadable");
  if (!ctx->cusolver) {
    cusolverDnHandle_t h;
    if (g_chol.create(&h) != CUSOLVER_STATUS_SUCCESS)
      return set_err(ctx, KST_ERR_CUDA, "cusolverDnCreate failed");
    ctx->cusolver = (void*)h;
  }
  *out = (cusolverDnHandle_t)ctx->cusolver;
  g_chol.set_stream(*out, st);
  return KST_OK;
}

// A (column-major) lower triangle <- S (row-major) lower triangle, through a
// 32 x 32 smem tile (coalesced on both sides); strict upper of A zeroed;
// flag[0] |= any non-finite entry of S (as_matrix, src/linalg.py:25-33)
__global__ void lower_colmajor_kernel(const cplx* __restrict__ S, int d, cplx* __restrict__ A,
                                      int* __restrict__ flag) {
  __shared__ cplx tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  int bad = 0;
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;
    cplx v = cmk(0.0, 0.0);
    if (r < d && c < d) {
      v = S[(size_t)r * d + c];
      if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
    }
    tile[k][tx] = v;
  }
  if (bad) atomicOr(flag, 1);
  __syncthreads();
  // column-major A[i + j d] = S[i][j] (i >= j): thread tx walks rows i
  for (int k = ty; k < 32; k += 8) {
    const int j = c0 + k, i = r0 + tx;
    if (i < d && j < d) A[(size_t)j * d + i] = (i >= j) ? tile[tx][k] : cmk(0.0, 0.0);
  }
}

__global__ void finite_kernel(const cplx* __restrict__ x, int64_t count, int* __restrict__ flag) {
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const cplx v = x[e];
    if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

extern "C" int kst_chol(kst_ctx* ctx, const double* sigma, int d, double* L, void* stream) {
  CTX_GUARD(ctx);
  if (d < 1) return set_err(ctx, KST_ERR_DIMENSION, "chol: dimension %d", d);
  if ((const void*)sigma == (const void*)L)  // the tiled transpose cannot run in place
    return set_err(ctx, KST_ERR_DIMENSION, "chol: L must not alias sigma");
  cudaStream_t st = (cudaStream_t)stream;
  cplx* A = (cplx*)L;
  int* dflag = (int*)ws_get(ctx, WS_SMALL, 64);
  int* hflag = (int*)pinned_get(ctx, 64);
  if (!dflag || !hflag) return set_err(ctx, KST_ERR_CUDA, "chol: workspace");
  KST_CUDA(ctx, cudaMemsetAsync(dflag, 0, 2 * sizeof(int), st));
  lower_colmajor_kernel<<<dim3(cdiv(d, 32), cdiv(d, 32)), dim3(32, 8), 0, st>>>((const cplx*)sigma,
                                                                               d, A, dflag);
  KST_LAUNCH(ctx);
  cusolverDnHandle_t h;
  KST_TRY(solver_handle(ctx, st, &h));
  int lwork = 0;
  if (g_chol.potrf_bufsize(h, CUBLAS_FILL_MODE_LOWER, d, (cuDoubleComplex*)A, d, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, KST_ERR_CUDA, "zpotrf buffer size");
  char* wk = (char*)ws_get(ctx, WS_CUSOLVER, sizeof(cuDoubleComplex) * (size_t)lwork + 64);
  if (!wk) return set_err(ctx, KST_ERR_CUDA, "zpotrf workspace");
  int* info = (int*)(wk + sizeof(cuDoubleComplex) * (size_t)lwork);
  // a non-finite input is reported before factorising (scipy's check_finite)
  KST_CUDA(ctx, cudaMemcpyAsync(hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[0]) return set_err(ctx, KST_ERR_DATA, "covariance contains non-finite entries");
  if (g_chol.potrf(h, CUBLAS_FILL_MODE_LOWER, d, (cuDoubleComplex*)A, d, (cuDoubleComplex*)wk,
                   lwork, info) != CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, KST_ERR_CUDA, "zpotrf failed");
  KST_CUDA(ctx, cudaMemcpyAsync(hflag + 1, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[1] != 0) return set_err(ctx, KST_ERR_DATA, "covariance is not positive definite");
  return KST_OK;
}

extern "C" int kst_chol_solve(kst_ctx* ctx, const double* L, int d, const double* B, int64_t nrhs,
                              double* X, void* stream) {
  CTX_GUARD(ctx);
  if (d < 1 || nrhs < 0 || nrhs > 0x7fffffff)
    return set_err(ctx, KST_ERR_DIMENSION, "chol_solve: d=%d nrhs=%lld", d, (long long)nrhs);
  if (nrhs == 0) return KST_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t count = (int64_t)d * nrhs;
  int* dflag = (int*)ws_get(ctx, WS_SMALL, 64);
  int* hflag = (int*)pinned_get(ctx, 64);
  if (!dflag || !hflag) return set_err(ctx, KST_ERR_CUDA, "chol_solve: workspace");
  KST_CUDA(ctx, cudaMemsetAsync(dflag, 0, sizeof(int), st));
  finite_kernel<<<(unsigned)std::min<int64_t>(cdiv(count, 256), 4 * kNumSMs), 256, 0, st>>>(
      (const cplx*)B, count, dflag);
  KST_LAUNCH(ctx);
  if (X != B)
    KST_CUDA(ctx, cudaMemcpyAsync(X, B, sizeof(cplx) * (size_t)count, cudaMemcpyDeviceToDevice, st));
  cusolverDnHandle_t h;
  KST_TRY(solver_handle(ctx, st, &h));
  int* info = dflag + 1;
  if (g_chol.potrs(h, CUBLAS_FILL_MODE_LOWER, d, (int)nrhs, (const cuDoubleComplex*)L, d,
                   (cuDoubleComplex*)X, d, info) != CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, KST_ERR_CUDA, "zpotrs failed");
  KST_CUDA(ctx, cudaMemcpyAsync(hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[0]) return set_err(ctx, KST_ERR_DATA, "bin matrix contains non-finite entries");
  return KST_OK;
}
