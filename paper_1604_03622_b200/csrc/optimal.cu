// "optimal" (covariance-whitening) filter -- src/filters.py:137-163 (build_filter
// kind "optimal": scipy cho_factor(sigma, lower=True)) and src/filters.py:98-100
// (apply_matrix: cho_solve). SURVEY.md §8f rank 4.
//
// The factor is the lower Cholesky factor of the Hermitian matrix defined by
// sigma's lower triangle (cho_factor reads only that triangle, and LAPACK's
// zpotrf only the real part of the diagonal), kept on the device in
// column-major order. Hand-written blocked kernels, FP64 complex:
//
// factor (right-looking, panel width CB = 32), per panel k:
//   chol_diag_kernel    one CTA: unblocked Cholesky of the CB x CB diagonal
//                       block in shared memory; a pivot <= 0 or non-finite
//                       raises the not-positive-definite flag (zpotrf info > 0)
//   chol_panel_kernel   L21 = A21 L11^-H, thread per row, L11 in smem
//   chol_update_kernel  A22 -= L21 L21^H on the lower triangle, 64 x 64 tiles,
//                       4 x 4 register blocks, both panels staged in smem
// solve L L^H X = B (cho_solve): the right-hand sides (one snapshot per
// column of the (pq x n) matrix = the C-order cube) are transposed to
// row-major Y (d x nrhs, right-hand sides contiguous), then per CB-row block
// a triangular solve (thread per right-hand side, the block of L in smem)
// and a rank-CB update of the rows still to solve (64 x 64 tiles):
//   forward  L Y = B   blocks top to bottom,  Y_i -= L_ik Y_k      (i > k)
//   backward L^H X = Y blocks bottom to top,  Y_c -= L_kc^H X_k    (c < k)
// and transposed back.
#include "common.cuh"

namespace {

constexpr int CB = 32;  // panel / block width
constexpr int UT = 64;  // update tile edge (rows x columns)
constexpr int kTileSmem = (int)(sizeof(cplx) * 2 * CB * (UT + 1));  // two staged panels

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

// ---------------------------------------------------------------- factor
// Unblocked Cholesky of the diagonal block A[k:k+nb, k:k+nb] (already holding
// every earlier panel's update). Column j: l_jj = sqrt(a_jj) (real part, as
// zpotrf), l_ij = a_ij / l_jj, then a_il -= l_ij conj(l_lj) for j < l <= i.
__global__ void __launch_bounds__(256) chol_diag_kernel(cplx* __restrict__ A, int d, int k, int nb,
                                                        int* __restrict__ flag) {
  __shared__ cplx a[CB][CB + 1];  // a[row][col]
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e % nb;  // column-major walk: coalesced
    a[r][c] = A[(size_t)(k + c) * d + k + r];
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double ajj = a[j][j].x;
    if (tid == 0 && !(ajj > 0.0 && isfinite(ajj))) atomicOr(flag, 2);  // not positive definite
    const double ljj = sqrt(fmax(ajj, 0.0));
    const double inv = ljj > 0.0 ? 1.0 / ljj : 0.0;
    __syncthreads();
    if (tid == 0) a[j][j] = cmk(ljj, 0.0);
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) a[i][j] = cscale(a[i][j], inv);
    __syncthreads();
    const int m = nb - j - 1;  // trailing block (j+1 .. nb-1), lower triangle
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) a[i][l] = csub(a[i][l], cmulc(a[i][j], a[l][j]));
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e % nb;
    A[(size_t)(k + c) * d + k + r] = r >= c ? a[r][c] : cmk(0.0, 0.0);
  }
}

// L21 = A21 L11^-H: row x of A21 solves x L11^H = a, i.e.
// x_j = (a_j - sum_{l<j} x_l conj(L11[j][l])) / L11[j][j]
__global__ void __launch_bounds__(128) chol_panel_kernel(cplx* __restrict__ A, int d, int k, int nb) {
  __shared__ cplx l11[CB][CB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e % nb;
    l11[r][c] = A[(size_t)(k + c) * d + k + r];
  }
  __syncthreads();
  const int i = k + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  cplx x[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) x[j] = j < nb ? A[(size_t)(k + j) * d + i] : cmk(0, 0);
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    if (j >= nb) break;
    cplx v = x[j];
#pragma unroll
    for (int l = 0; l < CB; ++l)
      if (l < j) v = csub(v, cmulc(x[l], l11[j][l]));  // x_l conj(L11[j][l])
    x[j] = cscale(v, 1.0 / l11[j][j].x);
  }
#pragma unroll
  for (int j = 0; j < CB; ++j)
    if (j < nb) A[(size_t)(k + j) * d + i] = x[j];
}

// A22[i][l] -= sum_j L21[i][j] conj(L21[l][j]) for i >= l (lower triangle of
// the trailing matrix, rows/cols from t0 = k + nb). Tile (I, J), I >= J, of
// UT x UT; thread = 4 x 4 block (rows ty + 16 u, cols tx + 16 v).
__global__ void __launch_bounds__(256) chol_update_kernel(cplx* __restrict__ A, int d, int k, int nb) {
  extern __shared__ __align__(16) cplx upd_smem[];  // pi, pj: [j][row within tile]
  cplx(*pi)[UT + 1] = (cplx(*)[UT + 1])upd_smem;
  cplx(*pj)[UT + 1] = (cplx(*)[UT + 1])(upd_smem + CB * (UT + 1));
  const int t0 = k + nb;
  // lower-triangle tile enumeration: blockIdx.x -> (I, J), J <= I
  int I = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) / 2.0);
  while ((I + 1) * (I + 2) / 2 <= (int)blockIdx.x) ++I;
  while (I * (I + 1) / 2 > (int)blockIdx.x) --I;
  const int J = blockIdx.x - I * (I + 1) / 2;
  const int r0 = t0 + I * UT, c0 = t0 + J * UT;
  for (int e = threadIdx.x; e < nb * UT; e += blockDim.x) {
    const int j = e / UT, r = e % UT;
    pi[j][r] = r0 + r < d ? A[(size_t)(k + j) * d + r0 + r] : cmk(0, 0);
    pj[j][r] = c0 + r < d ? A[(size_t)(k + j) * d + c0 + r] : cmk(0, 0);
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  cplx acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = cmk(0, 0);
  for (int j = 0; j < nb; ++j) {
    cplx a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = pi[j][ty + 16 * u];
      b[u] = pj[j][tx + 16 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cfmac(acc[u][v], a[u], b[v]);  // a conj(b)
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int l = c0 + tx + 16 * v;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = r0 + ty + 16 * u;
      if (i < d && l < d && l <= i) {
        cplx* p = A + (size_t)l * d + i;
        *p = csub(*p, acc[u][v]);
      }
    }
  }
}

// ---------------------------------------------------------------- solve
// Y[r][c] (row-major, nrhs columns) <-> B[c][r] (the cube: one right-hand
// side of d entries per snapshot), 32 x 32 smem tiles; conj never applied
__global__ void transpose_tiles_kernel(const cplx* __restrict__ in, int64_t rows, int64_t cols,
                                       cplx* __restrict__ out) {
  __shared__ cplx tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8)
    if (r0 + k < rows && c0 + tx < cols) tile[k][tx] = in[(r0 + k) * cols + c0 + tx];
  __syncthreads();
  for (int k = ty; k < 32; k += 8)
    if (c0 + k < cols && r0 + tx < rows) out[(c0 + k) * rows + r0 + tx] = tile[tx][k];
}

// Block triangular solve on rows [k, k + nb) of Y, thread per right-hand side.
// forward: y_r = (y_r - sum_{c<r} L[r][c] y_c) / L[r][r]
// backward (L^H): y_r = (y_r - sum_{c>r} conj(L[c][r]) y_c) / L[r][r]
template <bool BACK>
__global__ void __launch_bounds__(128) trsm_block_kernel(const cplx* __restrict__ L, int d, int k,
                                                         int nb, cplx* __restrict__ Y, int64_t nrhs) {
  __shared__ cplx l[CB][CB + 1];  // l[r][c] = L[k + r][k + c]
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e % nb;
    l[r][c] = L[(size_t)(k + c) * d + k + r];
  }
  __syncthreads();
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= nrhs) return;
  cplx y[CB];
#pragma unroll
  for (int r = 0; r < CB; ++r) y[r] = r < nb ? Y[(size_t)(k + r) * nrhs + col] : cmk(0, 0);
  if (!BACK) {
#pragma unroll
    for (int r = 0; r < CB; ++r) {
      if (r >= nb) break;
      cplx v = y[r];
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (c < r) v = csub(v, cmul(l[r][c], y[c]));
      y[r] = cscale(v, 1.0 / l[r][r].x);
    }
  } else {
#pragma unroll
    for (int r = CB - 1; r >= 0; --r) {
      if (r >= nb) continue;
      cplx v = y[r];
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (c > r && c < nb) v = csub(v, cmulc(y[c], l[c][r]));  // conj(L[c][r]) y_c
      y[r] = cscale(v, 1.0 / l[r][r].x);
    }
  }
#pragma unroll
  for (int r = 0; r < CB; ++r)
    if (r < nb) Y[(size_t)(k + r) * nrhs + col] = y[r];
}

// Rank-nb update of the rows still to solve, tile = UT rows x UT right-hand
// sides (thread 4 x 4):
// forward  (rows i in [k + nb, d)):  Y[i] -= sum_j L[i][k + j] Y[k + j]
// backward (rows c in [0, k)):       Y[c] -= sum_j conj(L[k + j][c]) Y[k + j]
template <bool BACK>
__global__ void __launch_bounds__(256) trsm_update_kernel(const cplx* __restrict__ L, int d, int k,
                                                          int nb, cplx* __restrict__ Y,
                                                          int64_t nrhs) {
  extern __shared__ __align__(16) cplx trsm_smem[];
  cplx(*ls)[UT + 1] = (cplx(*)[UT + 1])trsm_smem;                  // [j][row] (conj for BACK)
  cplx(*ys)[UT + 1] = (cplx(*)[UT + 1])(trsm_smem + CB * (UT + 1));  // [j][rhs]
  const int row0 = (BACK ? 0 : k + nb) + blockIdx.y * UT;
  const int64_t c0 = (int64_t)blockIdx.x * UT;
  const int rend = BACK ? k : d;
  for (int e = threadIdx.x; e < CB * UT; e += blockDim.x) {
    // L panel: consecutive threads walk the contiguous (column-major) index
    const int j = BACK ? e % CB : e / UT, r = BACK ? e / CB : e % UT;
    const int row = row0 + r;
    cplx lv = cmk(0, 0);
    if (row < rend && j < nb)
      lv = BACK ? cconj(L[(size_t)row * d + k + j]) : L[(size_t)(k + j) * d + row];
    ls[j][r] = lv;
  }
  for (int e = threadIdx.x; e < nb * UT; e += blockDim.x) {
    const int j = e / UT, r = e % UT;
    ys[j][r] = c0 + r < nrhs ? Y[(size_t)(k + j) * nrhs + c0 + r] : cmk(0, 0);
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  cplx acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = cmk(0, 0);
  for (int j = 0; j < nb; ++j) {
    cplx a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = ls[j][ty + 16 * u];
      b[u] = ys[j][tx + 16 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cfma(acc[u][v], a[u], b[v]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int row = row0 + ty + 16 * u;
    if (row >= rend) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t col = c0 + tx + 16 * v;
      if (col < nrhs) {
        cplx* p = Y + (size_t)row * nrhs + col;
        *p = csub(*p, acc[u][v]);
      }
    }
  }
}

int tile_smem_attrs(kst_ctx* ctx) {
  static bool done = false;  // per process: the attribute is a property of the function
  if (done) return KST_OK;
  KST_CUDA(ctx, cudaFuncSetAttribute(chol_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kTileSmem));
  KST_CUDA(ctx, cudaFuncSetAttribute(trsm_update_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
  KST_CUDA(ctx, cudaFuncSetAttribute(trsm_update_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
  done = true;
  return KST_OK;
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
  // a non-finite input is reported before factorising (scipy's check_finite)
  KST_CUDA(ctx, cudaMemcpyAsync(hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[0]) return set_err(ctx, KST_ERR_DATA, "covariance contains non-finite entries");
  KST_TRY(tile_smem_attrs(ctx));
  for (int k = 0; k < d; k += CB) {
    const int nb = std::min(CB, d - k);
    chol_diag_kernel<<<1, 256, 0, st>>>(A, d, k, nb, dflag);
    KST_LAUNCH(ctx);
    const int rest = d - k - nb;
    if (rest <= 0) break;
    chol_panel_kernel<<<cdiv(rest, 128), 128, 0, st>>>(A, d, k, nb);
    KST_LAUNCH(ctx);
    const int t = cdiv(rest, UT);
    chol_update_kernel<<<t * (t + 1) / 2, 256, kTileSmem, st>>>(A, d, k, nb);
    KST_LAUNCH(ctx);
  }
  KST_CUDA(ctx, cudaMemcpyAsync(hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[0] & 2) return set_err(ctx, KST_ERR_DATA, "covariance is not positive definite");
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
  cplx* Y = (cplx*)ws_get(ctx, WS_CUSOLVER, sizeof(cplx) * (size_t)count + 64);
  if (!dflag || !hflag || !Y) return set_err(ctx, KST_ERR_CUDA, "chol_solve: workspace");
  KST_CUDA(ctx, cudaMemsetAsync(dflag, 0, sizeof(int), st));
  finite_kernel<<<(unsigned)std::min<int64_t>(cdiv(count, 256), 4 * kNumSMs), 256, 0, st>>>(
      (const cplx*)B, count, dflag);
  KST_LAUNCH(ctx);
  const cplx* Lc = (const cplx*)L;
  KST_TRY(tile_smem_attrs(ctx));
  // B (nrhs x d, row-major) -> Y (d x nrhs)
  transpose_tiles_kernel<<<dim3((unsigned)cdiv(d, 32), (unsigned)cdiv(nrhs, 32)), dim3(32, 8), 0, st>>>(
      (const cplx*)B, nrhs, d, Y);
  KST_LAUNCH(ctx);
  const unsigned gx = (unsigned)cdiv(nrhs, UT), gs = (unsigned)cdiv(nrhs, 128);
  for (int k = 0; k < d; k += CB) {  // L Y = B
    const int nb = std::min(CB, d - k);
    trsm_block_kernel<false><<<gs, 128, 0, st>>>(Lc, d, k, nb, Y, nrhs);
    KST_LAUNCH(ctx);
    const int rest = d - k - nb;
    if (rest > 0) {
      trsm_update_kernel<false><<<dim3(gx, (unsigned)cdiv(rest, UT)), 256, kTileSmem, st>>>(Lc, d, k, nb, Y, nrhs);
      KST_LAUNCH(ctx);
    }
  }
  for (int k = ((d - 1) / CB) * CB; k >= 0; k -= CB) {  // L^H X = Y
    const int nb = std::min(CB, d - k);
    trsm_block_kernel<true><<<gs, 128, 0, st>>>(Lc, d, k, nb, Y, nrhs);
    KST_LAUNCH(ctx);
    if (k > 0) {
      trsm_update_kernel<true><<<dim3(gx, (unsigned)cdiv(k, UT)), 256, kTileSmem, st>>>(Lc, d, k, nb, Y, nrhs);
      KST_LAUNCH(ctx);
    }
  }
  // Y (d x nrhs) -> X (nrhs x d)
  transpose_tiles_kernel<<<dim3((unsigned)cdiv(nrhs, 32), (unsigned)cdiv(d, 32)), dim3(32, 8), 0, st>>>(
      Y, d, nrhs, (cplx*)X);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaMemcpyAsync(hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag[0]) return set_err(ctx, KST_ERR_DATA, "bin matrix contains non-finite entries");
  return KST_OK;
}
