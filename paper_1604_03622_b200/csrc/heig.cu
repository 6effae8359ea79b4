// Hermitian eigen-helpers with the reference's conventions.
//
//  * n <= 64: one-CTA Jacobi (jacobi.cuh), all eigenpairs.
//  * n  > 64: top-r pairs by a restarted block-Krylov Rayleigh-Ritz
//    iteration (K4): basis V = [Z, W] with Z the current s Ritz
//    vectors and W the orthonormalised block residual (I - ZZ^H) B Z; RR on
//    V^H B V (<= 2s x 2s, Jacobi); keep the top s. One B-multiply per
//    iteration (B Z is carried as Y). Convergence when every wanted Ritz
//    residual |B z - theta z| <= 1e-12 max|theta|. cuSOLVER zheevd is the
//    fallback only for rank budgets above 24 or non-convergence.
//
// Replaces hermitian_eig / eig_truncate (src/linalg.py:82-144) and
// subspace_basis (src/filters.py:58-73).
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>

#include "jacobi.cuh"

namespace {

using namespace kstj;

__global__ void jacobi_eig_kernel(const cplx* __restrict__ M, int ldm, int n, double div,
                                  double* __restrict__ values, cplx* __restrict__ vectors,
                                  int ldv) {
  extern __shared__ __align__(16) char sm[];
  JacSmem j = jac_carve(sm, n);
  jac_load_sym(j, M, ldm, n, div);
  jac_sweeps(j, n);
  jac_finish(j, n);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e % n;
    vectors[(size_t)i * ldv + k] = j.V[i * j.ld + j.order[k]];
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) values[k] = j.val[j.order[k]];
}

// ---------------------------------------------------------------- tall-skinny kernels
// Y (n x s) = B (n x n) * Z (n x s); s <= 32, multiple of 8. 128 threads,
// 16 rows per CTA, K staged through shared memory in chunks of 32.
constexpr int BZ_ROWS = 16, BZ_K = 32;
__global__ void __launch_bounds__(128) bz_kernel(const cplx* __restrict__ B, int n,
                                                 const cplx* __restrict__ Z, int s,
                                                 cplx* __restrict__ Y) {
  __shared__ cplx sb[BZ_ROWS][BZ_K + 1];
  __shared__ cplx sz[BZ_K][32 + 1];
  const int r0 = blockIdx.x * BZ_ROWS;
  const int t = threadIdx.x;
  const int row = t >> 3, cg = t & 7;  // 16 rows x 8 column groups
  cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
  for (int k0 = 0; k0 < n; k0 += BZ_K) {
    for (int e = t; e < BZ_ROWS * BZ_K; e += 128) {
      const int rr = e / BZ_K, kk = e % BZ_K;
      const int gr = r0 + rr, gk = k0 + kk;
      sb[rr][kk] = (gr < n && gk < n) ? B[(size_t)gr * n + gk] : cmk(0, 0);
    }
    for (int e = t; e < BZ_K * s; e += 128) {
      const int kk = e / s, c = e % s;
      const int gk = k0 + kk;
      sz[kk][c] = gk < n ? Z[(size_t)gk * s + c] : cmk(0, 0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BZ_K; ++kk) {
      const cplx b = sb[row][kk];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = cg + 8 * c;
        if (col < s) cfma(acc[c], b, sz[kk][col]);
      }
    }
    __syncthreads();
  }
  const int gr = r0 + row;
  if (gr < n) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int col = cg + 8 * c;
      if (col < s) Y[(size_t)gr * s + col] = acc[c];
    }
  }
}

// partial[blk][a][b] = sum_{rows in chunk} conj(U[row][a]) * V[row][b]
constexpr int GP_ROWS = 64;
__global__ void gram_partial_kernel(const cplx* __restrict__ U, int ldu, int s1,
                                    const cplx* __restrict__ V, int ldv, int s2, int n,
                                    cplx* __restrict__ partial) {
  extern __shared__ __align__(16) cplx gsm[];
  cplx* su = gsm;
  cplx* sv = gsm + GP_ROWS * s1;
  const int r0 = blockIdx.x * GP_ROWS;
  const int rows = min(GP_ROWS, n - r0);
  for (int e = threadIdx.x; e < GP_ROWS * s1; e += blockDim.x) {
    const int rr = e / s1, a = e % s1;
    su[e] = rr < rows ? U[(size_t)(r0 + rr) * ldu + a] : cmk(0, 0);
  }
  for (int e = threadIdx.x; e < GP_ROWS * s2; e += blockDim.x) {
    const int rr = e / s2, b = e % s2;
    sv[e] = rr < rows ? V[(size_t)(r0 + rr) * ldv + b] : cmk(0, 0);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < s1 * s2; e += blockDim.x) {
    const int a = e / s2, b = e % s2;
    cplx acc = cmk(0, 0);
    for (int rr = 0; rr < GP_ROWS; ++rr) cfmca(acc, su[rr * s1 + a], sv[rr * s2 + b]);
    partial[(size_t)blockIdx.x * s1 * s2 + e] = acc;
  }
}

// out[e] = sum_blk partial[blk][e], fixed order
__global__ void reduce_partials_kernel(const cplx* __restrict__ partial, int nblk, int count,
                                       cplx* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    for (int b = 0; b < nblk; ++b) acc = cadd(acc, partial[(size_t)b * count + e]);
    out[e] = acc;
  }
}

// Out (n x s2, ld) = [X0 -] U (n x s1, ldu) * C (s1 x s2, ldc)
__global__ void ts_mul_kernel(const cplx* __restrict__ U, int ldu, int s1,
                              const cplx* __restrict__ C, int ldc, int s2,
                              const cplx* __restrict__ X0, int ldx, cplx* __restrict__ Out,
                              int ldo, int n) {
  extern __shared__ __align__(16) cplx csm[];
  for (int e = threadIdx.x; e < s1 * s2; e += blockDim.x) csm[e] = C[(e / s2) * ldc + e % s2];
  __syncthreads();
  const int64_t total = (int64_t)n * s2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / s2), col = (int)(e % s2);
    cplx acc = cmk(0, 0);
    for (int a = 0; a < s1; ++a) cfma(acc, U[(size_t)row * ldu + a], csm[a * s2 + col]);
    if (X0) acc = csub(X0[(size_t)row * ldx + col], acc);
    Out[(size_t)row * ldo + col] = acc;
  }
}

// SVQB coefficients: C = Q diag(1/sqrt(g)) with dropped directions zeroed.
// vals/vecs: Jacobi output of G (descending). mask[k] = 1 if kept.
__global__ void svqb_coeff_kernel(const double* __restrict__ vals, const cplx* __restrict__ vecs,
                                  int s, double rel_drop, cplx* __restrict__ C, int* mask) {
  const double gmax = vals[0];
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int k = e % s;
    const double g = vals[k];
    const bool keep = gmax > 0.0 && g > rel_drop * gmax;
    C[e] = keep ? cscale(vecs[e], 1.0 / sqrt(g)) : cmk(0, 0);
    if (mask && e < s) mask[e] = (gmax > 0.0 && vals[e] > rel_drop * gmax) ? 1 : 0;
  }
}

// Place Hred into the Jacobi input, forcing masked-out W directions to a
// large negative sentinel so they sort last.
__global__ void mask_hred_kernel(cplx* H, int s, const int* __restrict__ mask, double sentinel) {
  const int m = 2 * s;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int a = e / m, b = e % m;
    const bool da = a < s || mask[a - s], db = b < s || mask[b - s];
    if (!da || !db) H[e] = (a == b) ? cmk(sentinel, 0) : cmk(0, 0);
  }
}

// ||Y[:,k] - theta_k Z[:,k]||_2 for k < r  -> res[k]; plus theta copy.
__global__ void ritz_residual_kernel(const cplx* __restrict__ Y, const cplx* __restrict__ Z,
                                     int n, int s, const double* __restrict__ theta, int r,
                                     double* __restrict__ res) {
  __shared__ double sh[32];
  const int k = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const cplx y = Y[(size_t)i * s + k], z = Z[(size_t)i * s + k];
    acc += cabs2(cmk(y.x - theta[k] * z.x, y.y - theta[k] * z.y));
  }
  acc = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) res[k] = sqrt(acc);
}

__global__ void random_block_kernel(cplx* Z, int n, int s, uint64_t seed) {
  const int64_t total = (int64_t)n * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(e + 1));
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    const double u1 = ((x >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    uint64_t y = x * 0x2545F4914F6CDD1Dull + 0x632BE59BD9B4E019ull;
    y ^= y >> 29;
    const double u2 = ((y >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    Z[e] = cmk(u1 - 0.5, u2 - 0.5);
  }
}

// Final ordering (descending, reference tie rule) + pivot phase for the top r
// Ritz vectors; single CTA of 256 threads, s <= 32.
__global__ void finalize_top_kernel(const cplx* __restrict__ Z, int n, int s, int r,
                                    const double* __restrict__ theta, double* __restrict__ vals_out,
                                    cplx* __restrict__ vec_out) {
  __shared__ int piv[32];
  __shared__ int order[32];
  __shared__ double phr[32], phi[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int k = w; k < s; k += 8) {
    double bm = -1.0;
    int bi = 0;
    for (int i = l; i < n; i += 32) {
      const cplx v = Z[(size_t)i * s + k];
      const double a = hypot(v.x, v.y);
      if (a > bm) {
        bm = a;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, bm, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > bm || (ob == bm && oi < bi)) {
        bm = ob;
        bi = oi;
      }
    }
    if (l == 0) piv[k] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < s; ++k) order[k] = k;
    for (int a = 1; a < s; ++a) {
      const int key = order[a];
      int b = a - 1;
      while (b >= 0 && theta[order[b]] < theta[key]) {
        order[b + 1] = order[b];
        --b;
      }
      order[b + 1] = key;
    }
    double mx = 0.0;
    for (int k = 0; k < s; ++k) mx = fmax(mx, fabs(theta[k]));
    const double tie = mx * 1e-12;
    int a0 = 0;
    while (a0 < s) {
      int e = a0 + 1;
      while (e < s && fabs(theta[order[e]] - theta[order[e - 1]]) <= tie) ++e;
      for (int a = a0 + 1; a < e; ++a) {
        const int key = order[a];
        int b = a - 1;
        while (b >= a0 && piv[order[b]] > piv[key]) {
          order[b + 1] = order[b];
          --b;
        }
        order[b + 1] = key;
      }
      a0 = e;
    }
    for (int k = 0; k < s; ++k) {
      const cplx z = Z[(size_t)piv[k] * s + k];
      const double mag = hypot(z.x, z.y);
      phr[k] = mag > 0.0 ? z.x / mag : 1.0;
      phi[k] = mag > 0.0 ? -z.y / mag : 0.0;
    }
    for (int k = 0; k < r; ++k) vals_out[k] = theta[order[k]];
  }
  __syncthreads();
  const int64_t total = (int64_t)n * r;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = (int)(e / r), k = (int)(e % r);
    const int src = order[k];
    vec_out[e] = cmul(Z[(size_t)i * s + src], cmk(phr[src], phi[src]));
  }
}

// out = (U diag(lam) U^H + h.c.)/2, U (n x r)
__global__ void recon_kernel(const cplx* __restrict__ U, const double* __restrict__ lam, int n,
                             int r, cplx* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / n), b = (int)(e % n);
    cplx ab = cmk(0, 0), ba = cmk(0, 0);
    for (int k = 0; k < r; ++k) {
      const cplx ua = U[(size_t)a * r + k], ub = U[(size_t)b * r + k];
      cfmac(ab, cscale(ua, lam[k]), ub);
      cfmac(ba, cscale(ub, lam[k]), ua);
    }
    out[e] = cmk((ab.x + ba.x) / 2.0, (ab.y - ba.y) / 2.0);
  }
}

// (M + M^H)/2
__global__ void symmetrize_kernel(const cplx* __restrict__ M, int n, cplx* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / n), b = (int)(e % n);
    const cplx x = M[(size_t)a * n + b], y = M[(size_t)b * n + a];
    out[e] = cmk((x.x + y.x) / 2.0, (x.y - y.y) / 2.0);
  }
}

// per-block partials of [sum |M|^2, sum |M - M^H|^2, nonfinite count]
__global__ void herm_check_kernel(const cplx* __restrict__ M, int n, double* __restrict__ part) {
  __shared__ double sh[32];
  double f = 0.0, a = 0.0, bad = 0.0;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    const cplx x = M[e], y = M[(size_t)c * n + r];
    if (!isfinite(x.x) || !isfinite(x.y)) bad += 1.0;
    f += cabs2(x);
    a += cabs2(cmk(x.x - y.x, x.y + y.y));
  }
  f = block_sum<256>(f, sh);
  a = block_sum<256>(a, sh);
  bad = block_sum<256>(bad, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = f;
    part[blockIdx.x * 3 + 1] = a;
    part[blockIdx.x * 3 + 2] = bad;
  }
}

__global__ void conj_transpose_cols_kernel(const cplx* __restrict__ colmajor, int n, int first,
                                           int count, cplx* __restrict__ out) {
  // cuSOLVER ran on conj(M) (row-major read as column-major); eigenvector j of
  // conj(M) is column j (contiguous) -> out[i][k] = conj(vec_{first+k}[i])
  const int64_t total = (int64_t)n * count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / count), k = (int)(e % count);
    out[e] = cconj(colmajor[(size_t)(first + k) * n + i]);
  }
}

unsigned grid_for(int64_t total, int nt = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + nt - 1) / nt, kNumSMs * 8));
}

// ---------------------------------------------------------------- host helpers
struct TsCtx {
  kst_ctx* ctx;
  cudaStream_t st;
  cplx* partial;  // workspace for gram partials
};

int gram_ts(TsCtx& t, const cplx* U, int ldu, int s1, const cplx* V, int ldv, int s2, int n,
            cplx* out) {
  const int nblk = (n + GP_ROWS - 1) / GP_ROWS;
  const size_t smem = sizeof(cplx) * GP_ROWS * (s1 + s2);
  static bool configured = false;
  if (!configured) {
    KST_CUDA(t.ctx, cudaFuncSetAttribute(gram_partial_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(cplx) * GP_ROWS * 128)));
    configured = true;
  }
  gram_partial_kernel<<<nblk, 256, smem, t.st>>>(U, ldu, s1, V, ldv, s2, n, t.partial);
  KST_LAUNCH(t.ctx);
  reduce_partials_kernel<<<grid_for(s1 * s2), 256, 0, t.st>>>(t.partial, nblk, s1 * s2, out);
  KST_LAUNCH(t.ctx);
  return KST_OK;
}

int ts_mul(TsCtx& t, const cplx* U, int ldu, int s1, const cplx* C, int ldc, int s2,
           const cplx* X0, int ldx, cplx* Out, int ldo, int n) {
  ts_mul_kernel<<<grid_for((int64_t)n * s2), 256, sizeof(cplx) * s1 * s2, t.st>>>(
      U, ldu, s1, C, ldc, s2, X0, ldx, Out, ldo, n);
  KST_LAUNCH(t.ctx);
  return KST_OK;
}

int jacobi(kst_ctx* ctx, const cplx* M, int ldm, int n, double div, double* vals, cplx* vecs,
           int ldv, cudaStream_t st) {
  const size_t smem = jac_smem_bytes(n);
  static int configured = 0;
  if (!configured) {
    KST_CUDA(ctx, cudaFuncSetAttribute(jacobi_eig_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)jac_smem_bytes(kMaxN)));
    configured = 1;
  }
  jacobi_eig_kernel<<<1, 256, smem, st>>>(M, ldm, n, div, vals, vecs, ldv);
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace

namespace kst {

int small_heig(kst_ctx* ctx, const cplx* M, int n, double* values_dev, cplx* vectors_dev,
               cudaStream_t st) {
  if (n > kMaxN) return set_err(ctx, KST_ERR_DIMENSION, "small_heig: n=%d > %d", n, kMaxN);
  return jacobi(ctx, M, n, n, 1.0, values_dev, vectors_dev, n, st);
}

int herm_check(kst_ctx* ctx, const cplx* M, int n, cudaStream_t st) {
  const unsigned nb = grid_for((int64_t)n * n);
  double* part = (double*)ws_get(ctx, WS_PART, sizeof(double) * 3 * nb);
  double* host = (double*)pinned_get(ctx, sizeof(double) * 3 * nb);
  if (!part || !host) return set_err(ctx, KST_ERR_CUDA, "herm_check: allocation failed");
  herm_check_kernel<<<nb, 256, 0, st>>>(M, n, part);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaMemcpyAsync(host, part, sizeof(double) * 3 * nb, cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  double f = 0, a = 0, bad = 0;
  for (unsigned b = 0; b < nb; ++b) {
    f += host[3 * b];
    a += host[3 * b + 1];
    bad += host[3 * b + 2];
  }
  if (bad > 0) return set_err(ctx, KST_ERR_DATA, "matrix contains non-finite entries");
  const double scale = sqrt(f);
  if (scale > 0 && sqrt(a) > 1e-8 * scale)
    return set_err(ctx, KST_ERR_DATA, "matrix deviates from Hermitian beyond tolerance");
  return KST_OK;
}

// cuSOLVER is bound at run time (dlopen) so libkst_b200 has no link-time
// dependency on a cuSOLVER/cuBLAS pair that could clash with torch's copies.
namespace {
struct Solver {
  bool tried = false, ok = false;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*bufsize)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int,
                              const cuDoubleComplex*, int, const double*, int*) = nullptr;
  cusolverStatus_t (*heevd)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int,
                            cuDoubleComplex*, int, double*, cuDoubleComplex*, int, int*) = nullptr;
};
Solver g_solver;
bool load_solver() {
  if (g_solver.tried) return g_solver.ok;
  g_solver.tried = true;
  const char* names[] = {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return false;
  g_solver.create = (decltype(g_solver.create))dlsym(h, "cusolverDnCreate");
  g_solver.set_stream = (decltype(g_solver.set_stream))dlsym(h, "cusolverDnSetStream");
  g_solver.bufsize = (decltype(g_solver.bufsize))dlsym(h, "cusolverDnZheevd_bufferSize");
  g_solver.heevd = (decltype(g_solver.heevd))dlsym(h, "cusolverDnZheevd");
  g_solver.ok = g_solver.create && g_solver.set_stream && g_solver.bufsize && g_solver.heevd;
  return g_solver.ok;
}
}  // namespace

static int heig_top_cusolver(kst_ctx* ctx, const cplx* M, int n, int r, double* values_host,
                             cplx* vectors, cudaStream_t st) {
  if (!load_solver()) return set_err(ctx, KST_ERR_NOCONV, "eigensolver fallback: cuSOLVER not loadable");
  if (!ctx->cusolver) {
    cusolverDnHandle_t h;
    if (g_solver.create(&h) != CUSOLVER_STATUS_SUCCESS)
      return set_err(ctx, KST_ERR_CUDA, "cusolverDnCreate failed");
    ctx->cusolver = (void*)h;
  }
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  g_solver.set_stream(h, st);
  cplx* A = (cplx*)ws_get(ctx, WS_EIG2, sizeof(cplx) * (size_t)n * n + sizeof(double) * n + 64);
  if (!A) return set_err(ctx, KST_ERR_CUDA, "cusolver workspace");
  double* w = (double*)(A + (size_t)n * n);
  // symmetrise into A (row-major == column-major conj(M))
  symmetrize_kernel<<<grid_for((int64_t)n * n), 256, 0, st>>>(M, n, A);
  KST_LAUNCH(ctx);
  int lwork = 0;
  if (g_solver.bufsize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                  (cuDoubleComplex*)A, n, w, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, KST_ERR_CUDA, "zheevd buffer size");
  char* wk = (char*)ws_get(ctx, WS_CUSOLVER, sizeof(cuDoubleComplex) * (size_t)lwork + 64);
  if (!wk) return set_err(ctx, KST_ERR_CUDA, "zheevd workspace");
  int* info = (int*)(wk + sizeof(cuDoubleComplex) * (size_t)lwork);
  if (g_solver.heevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                       (cuDoubleComplex*)A, n, w, (cuDoubleComplex*)wk, lwork, info) !=
      CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, KST_ERR_CUDA, "zheevd failed");
  // ascending -> we need the top r (+ a few for the tie rule): take columns n-s..n-1
  const int s = std::min(n, std::max(r, 1) + 8);
  cplx* Zs = (cplx*)ws_get(ctx, WS_EIG, sizeof(cplx) * (size_t)n * s + sizeof(double) * (s + r) + 64);
  if (!Zs) return set_err(ctx, KST_ERR_CUDA, "eig workspace");
  double* theta = (double*)(Zs + (size_t)n * s);
  double* vout = theta + s;
  conj_transpose_cols_kernel<<<grid_for((int64_t)n * s), 256, 0, st>>>(A, n, n - s, s, Zs);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaMemcpyAsync(theta, w + (n - s), sizeof(double) * s, cudaMemcpyDeviceToDevice, st));
  finalize_top_kernel<<<1, 256, 0, st>>>(Zs, n, s, r, theta, vout, vectors);
  KST_LAUNCH(ctx);
  if (values_host) {
    KST_CUDA(ctx, cudaMemcpyAsync(values_host, vout, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
  }
  return KST_OK;
}

int heig_top(kst_ctx* ctx, const cplx* M, int n, int r, double* values_host, cplx* vectors,
             cudaStream_t st) {
  if (r < 1 || r > n) return set_err(ctx, KST_ERR_DIMENSION, "heig_top: r=%d n=%d", r, n);
  if (n <= kMaxN) {
    cplx* vec = (cplx*)ws_get(ctx, WS_EIG2, sizeof(cplx) * n * n + sizeof(double) * n);
    if (!vec) return set_err(ctx, KST_ERR_CUDA, "heig_top: workspace");
    double* val = (double*)(vec + n * n);
    KST_TRY(jacobi(ctx, M, n, n, 1.0, val, vec, n, st));
    // copy leading r columns
    KST_CUDA(ctx, cudaMemcpy2DAsync(vectors, sizeof(cplx) * r, vec, sizeof(cplx) * n,
                                    sizeof(cplx) * r, n, cudaMemcpyDeviceToDevice, st));
    if (values_host) {
      KST_CUDA(ctx, cudaMemcpyAsync(values_host, val, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
      KST_CUDA(ctx, cudaStreamSynchronize(st));
    }
    return KST_OK;
  }
  if (r > 24) return heig_top_cusolver(ctx, M, n, r, values_host, vectors, st);

  int s = std::max(r + 6, 8);
  s = ((s + 7) / 8) * 8;
  if (s > 32) s = 32;
  const int s2 = 2 * s;
  // workspace layout
  const size_t nb = (size_t)n * s;
  size_t bytes = sizeof(cplx) * (nb * 8 + (size_t)s2 * s2 * 3 + (size_t)s * s * 4) +
                 sizeof(double) * (s2 * 2 + s * 4) + sizeof(int) * (s + 8) + 256;
  char* base = (char*)ws_get(ctx, WS_EIG, bytes);
  const int nblk = (n + GP_ROWS - 1) / GP_ROWS;
  cplx* partial = (cplx*)ws_get(ctx, WS_EIG2, sizeof(cplx) * (size_t)nblk * s2 * s2);
  double* hres = (double*)pinned_get(ctx, sizeof(double) * 2 * s2);
  if (!base || !partial || !hres) return set_err(ctx, KST_ERR_CUDA, "heig_top: workspace");
  cplx* Vb = (cplx*)base;    // [Z | W]   n x 2s
  cplx* Tb = Vb + 2 * nb;    // [Y | BW]  n x 2s
  cplx* Zn = Tb + 2 * nb;    // new Z     n x s
  cplx* Yn = Zn + nb;        // new Y     n x s
  cplx* Wt = Yn + nb;        // temp      n x s
  cplx* Wt2 = Wt + nb;       // temp2     n x s
  cplx* H = Wt2 + nb;        // s2 x s2
  cplx* Hv = H + s2 * s2;    // s2 x s2 eigenvectors
  cplx* Cs = Hv + s2 * s2;   // s x s coefficients
  cplx* Gs = Cs + s * s;     // s x s gram
  cplx* Gv = Gs + s * s;     // s x s eigvecs
  cplx* Cs2 = Gv + s * s;    // s x s
  double* Hval = (double*)(Cs2 + s * s);
  double* Gval = Hval + s2;
  double* theta = Gval + s2;
  double* res = theta + s;
  double* vout = res + s;
  int* mask = (int*)(vout + s);
  TsCtx t{ctx, st, partial};

  // Z stored at ld 2s inside Vb (columns 0..s-1), W at columns s..2s-1
  const int ldV = s2;
  // Orthonormalise a block X (n x s, ld ldx) in place via two SVQB passes,
  // optionally against Z first. Returns via mask which columns survived.
  auto svqb = [&](cplx* X, int ldx, bool against_z, int* msk) -> int {
    for (int pass = 0; pass < 2; ++pass) {
      if (against_z) {
        // X -= Z (Z^H X)
        KST_TRY(gram_ts(t, Vb, ldV, s, X, ldx, s, n, Cs));
        KST_TRY(ts_mul(t, Vb, ldV, s, Cs, s, s, X, ldx, Wt, s, n));
        KST_CUDA(ctx, cudaMemcpy2DAsync(X, sizeof(cplx) * ldx, Wt, sizeof(cplx) * s,
                                        sizeof(cplx) * s, n, cudaMemcpyDeviceToDevice, st));
      }
      KST_TRY(gram_ts(t, X, ldx, s, X, ldx, s, n, Gs));
      KST_TRY(jacobi(ctx, Gs, s, s, 1.0, Gval, Gv, s, st));
      svqb_coeff_kernel<<<1, 256, 0, st>>>(Gval, Gv, s, 1e-24, Cs2, pass == 1 ? msk : nullptr);
      KST_LAUNCH(ctx);
      KST_TRY(ts_mul(t, X, ldx, s, Cs2, s, s, nullptr, 0, Wt2, s, n));
      KST_CUDA(ctx, cudaMemcpy2DAsync(X, sizeof(cplx) * ldx, Wt2, sizeof(cplx) * s,
                                      sizeof(cplx) * s, n, cudaMemcpyDeviceToDevice, st));
    }
    return KST_OK;
  };

  // Z0 = orth(random); Y0 = B Z0
  random_block_kernel<<<grid_for((int64_t)n * s), 256, 0, st>>>(Wt, n, s, 0x5EEDull + n);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaMemcpy2DAsync(Vb, sizeof(cplx) * ldV, Wt, sizeof(cplx) * s, sizeof(cplx) * s,
                                  n, cudaMemcpyDeviceToDevice, st));
  KST_TRY(svqb(Vb, ldV, false, mask));
  KST_CUDA(ctx, cudaMemcpy2DAsync(Zn, sizeof(cplx) * s, Vb, sizeof(cplx) * ldV, sizeof(cplx) * s,
                                  n, cudaMemcpyDeviceToDevice, st));
  bz_kernel<<<cdiv(n, BZ_ROWS), 128, 0, st>>>(M, n, Zn, s, Yn);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaMemcpy2DAsync(Tb, sizeof(cplx) * ldV, Yn, sizeof(cplx) * s, sizeof(cplx) * s, n,
                                  cudaMemcpyDeviceToDevice, st));

  bool converged = false;
  double prev_worst = 1e300;
  int stall = 0;
  for (int it = 0; it < 80 && !converged; ++it) {
    // W = Y - Z (Z^H Y), orthonormalised against Z
    cplx* W = Vb + s;
    KST_TRY(gram_ts(t, Vb, ldV, s, Tb, ldV, s, n, Cs));
    KST_TRY(ts_mul(t, Vb, ldV, s, Cs, s, s, Tb, ldV, W, ldV, n));
    KST_TRY(svqb(W, ldV, true, mask));
    // BW
    KST_CUDA(ctx, cudaMemcpy2DAsync(Wt, sizeof(cplx) * s, W, sizeof(cplx) * ldV, sizeof(cplx) * s,
                                    n, cudaMemcpyDeviceToDevice, st));
    bz_kernel<<<cdiv(n, BZ_ROWS), 128, 0, st>>>(M, n, Wt, s, Wt2);
    KST_LAUNCH(ctx);
    KST_CUDA(ctx, cudaMemcpy2DAsync(Tb + s, sizeof(cplx) * ldV, Wt2, sizeof(cplx) * s,
                                    sizeof(cplx) * s, n, cudaMemcpyDeviceToDevice, st));
    // Hred = V^H T, masked; eig
    KST_TRY(gram_ts(t, Vb, ldV, s2, Tb, ldV, s2, n, H));
    mask_hred_kernel<<<1, 256, 0, st>>>(H, s, mask, -1e300);
    KST_LAUNCH(ctx);
    KST_TRY(jacobi(ctx, H, s2, s2, 1.0, Hval, Hv, s2, st));
    // Z = V C[:, :s], Y = T C[:, :s]
    KST_TRY(ts_mul(t, Vb, ldV, s2, Hv, s2, s, nullptr, 0, Zn, s, n));
    KST_TRY(ts_mul(t, Tb, ldV, s2, Hv, s2, s, nullptr, 0, Yn, s, n));
    KST_CUDA(ctx, cudaMemcpy2DAsync(Vb, sizeof(cplx) * ldV, Zn, sizeof(cplx) * s, sizeof(cplx) * s,
                                    n, cudaMemcpyDeviceToDevice, st));
    KST_CUDA(ctx, cudaMemcpy2DAsync(Tb, sizeof(cplx) * ldV, Yn, sizeof(cplx) * s, sizeof(cplx) * s,
                                    n, cudaMemcpyDeviceToDevice, st));
    KST_CUDA(ctx, cudaMemcpyAsync(theta, Hval, sizeof(double) * s, cudaMemcpyDeviceToDevice, st));
    ritz_residual_kernel<<<r, 256, 0, st>>>(Yn, Zn, n, s, theta, r, res);
    KST_LAUNCH(ctx);
    KST_CUDA(ctx, cudaMemcpyAsync(hres, res, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaMemcpyAsync(hres + r, theta, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    double tmax = 0.0, worst = 0.0;
    for (int k = 0; k < s; ++k) tmax = std::max(tmax, std::fabs(hres[r + k]));
    for (int k = 0; k < r; ++k) worst = std::max(worst, hres[k]);
    if (tmax == 0.0 || worst <= 1e-12 * tmax) converged = true;
    else if (worst <= 1e-9 * tmax) {
      // accept a stalled residual floor once it stops improving
      stall = (worst > 0.5 * prev_worst) ? stall + 1 : 0;
      if (stall >= 3) converged = true;
    }
    prev_worst = worst;
  }
  if (!converged) return heig_top_cusolver(ctx, M, n, r, values_host, vectors, st);
  finalize_top_kernel<<<1, 256, 0, st>>>(Zn, n, s, r, theta, vout, vectors);
  KST_LAUNCH(ctx);
  if (values_host) {
    KST_CUDA(ctx, cudaMemcpyAsync(values_host, vout, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
  }
  return KST_OK;
}

int truncate_from_pairs(kst_ctx* ctx, const double* values_host, const cplx* vectors, int n, int r,
                        double top_abs, cplx* out, cudaStream_t st) {
  double* lam = (double*)ws_get(ctx, WS_VALS, sizeof(double) * r);
  double* hl = (double*)pinned_get(ctx, sizeof(double) * r);
  if (!lam || !hl) return set_err(ctx, KST_ERR_CUDA, "truncate: workspace");
  for (int k = 0; k < r; ++k) {
    double v = values_host[k];
    if (v < 0 && std::fabs(v) <= 1e-10 * top_abs) v = 0.0;  // src/linalg.py:138-140
    hl[k] = v;
  }
  KST_CUDA(ctx, cudaMemcpyAsync(lam, hl, sizeof(double) * r, cudaMemcpyHostToDevice, st));
  recon_kernel<<<grid_for((int64_t)n * n), 256, 0, st>>>(vectors, lam, n, r, out);
  KST_LAUNCH(ctx);
  KST_CUDA(ctx, cudaStreamSynchronize(st));  // hl is reused by later calls
  return KST_OK;
}

int eig_truncate(kst_ctx* ctx, const cplx* M, int n, int rank, cplx* out, cudaStream_t st) {
  KST_TRY(herm_check(ctx, M, n, st));
  if (rank < 1 || rank > n) return set_err(ctx, KST_ERR_DIMENSION, "rank must be in [1, %d], got %d", n, rank);
  if (rank == n) {
    symmetrize_kernel<<<grid_for((int64_t)n * n), 256, 0, st>>>(M, n, out);
    KST_LAUNCH(ctx);
    return KST_OK;
  }
  std::vector<double> vals(n);
  const int want = n <= kMaxN ? n : rank;  // small: all pairs (exact max|lambda|)
  cplx* U = (cplx*)ws_get(ctx, WS_UB, sizeof(cplx) * (size_t)n * want);
  if (!U) return set_err(ctx, KST_ERR_CUDA, "eig_truncate: workspace");
  KST_TRY(heig_top(ctx, M, n, want, vals.data(), U, st));
  double top = 0.0;
  for (int k = 0; k < want; ++k) top = std::max(top, std::fabs(vals[k]));
  if (want != rank) {
    // keep the leading `rank` columns contiguous
    cplx* U2 = (cplx*)ws_get(ctx, WS_TMP, sizeof(cplx) * (size_t)n * rank);
    if (!U2) return set_err(ctx, KST_ERR_CUDA, "eig_truncate: workspace");
    KST_CUDA(ctx, cudaMemcpy2DAsync(U2, sizeof(cplx) * rank, U, sizeof(cplx) * want,
                                    sizeof(cplx) * rank, n, cudaMemcpyDeviceToDevice, st));
    U = U2;
  }
  return truncate_from_pairs(ctx, vals.data(), U, n, rank, top, out, st);
}

int subspace_basis(kst_ctx* ctx, const cplx* M, int n, int rank, double tol, cplx* basis, int* keep,
                   cudaStream_t st) {
  KST_TRY(herm_check(ctx, M, n, st));
  *keep = 0;
  const int r = std::min(rank, n);
  if (r < 1) return KST_OK;  // no budget -> None
  std::vector<double> vals(r);
  cplx* U = (cplx*)ws_get(ctx, WS_UA, sizeof(cplx) * (size_t)n * r);
  if (!U) return set_err(ctx, KST_ERR_CUDA, "subspace_basis: workspace");
  KST_TRY(heig_top(ctx, M, n, r, vals.data(), U, st));
  const double top = vals[0];
  if (top <= 0.0) return KST_OK;
  int k = 0;
  while (k < r && vals[k] > tol * top) ++k;
  if (k > 0)
    KST_CUDA(ctx, cudaMemcpy2DAsync(basis, sizeof(cplx) * k, U, sizeof(cplx) * r, sizeof(cplx) * k,
                                    n, cudaMemcpyDeviceToDevice, st));
  *keep = k;
  return KST_OK;
}

}  // namespace kst
