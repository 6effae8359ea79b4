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
  jac_solve(j, M, ldm, n, div);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e % n;
    vectors[(size_t)i * ldv + k] = j.V[i * j.ld + j.order[k]];
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) values[k] = j.val[j.order[k]];
}

// ---------------------------------------------------------------- tall-skinny kernels
// Ypart[ks] (n x s) = B[:, kslice] * Z[kslice, :]; s <= 32. Split-K over
// blockIdx.y (BZ_KSPLIT columns of B each) so ~1000 CTAs stream the 64 MB
// matrix; the partials are summed in a fixed order afterwards.
constexpr int BZ_ROWS = 16, BZ_K = 32, BZ_KSPLIT = 256;
__global__ void __launch_bounds__(128) bz_kernel(const cplx* __restrict__ B, int n,
                                                 const cplx* __restrict__ Z, int s,
                                                 cplx* __restrict__ Ypart) {
  __shared__ cplx sb[BZ_ROWS][BZ_K + 1];
  __shared__ cplx sz[BZ_K][32 + 1];
  const int r0 = blockIdx.x * BZ_ROWS;
  const int kbeg = blockIdx.y * BZ_KSPLIT, kend = min(n, kbeg + BZ_KSPLIT);
  const int t = threadIdx.x;
  const int row = t >> 3, cg = t & 7;  // 16 rows x 8 column groups
  cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
  // register prefetch of the next chunk (global loads overlap the compute)
  cplx pb[4], pz[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = t + 128 * u;
      const int rr = e / BZ_K, kk = e % BZ_K;
      const int gr = r0 + rr, gk = k0 + kk;
      pb[u] = (gr < n && gk < kend) ? B[(size_t)gr * n + gk] : cmk(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = t + 128 * u;
      if (e < BZ_K * s) {
        const int kk = e / s, c = e % s;
        const int gk = k0 + kk;
        pz[u] = gk < kend ? Z[(size_t)gk * s + c] : cmk(0, 0);
      }
    }
  };
  fetch(kbeg);
  for (int k0 = kbeg; k0 < kend; k0 += BZ_K) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = t + 128 * u;
      sb[e / BZ_K][e % BZ_K] = pb[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = t + 128 * u;
      if (e < BZ_K * s) sz[e / s][e % s] = pz[u];
    }
    __syncthreads();
    if (k0 + BZ_K < kend) fetch(k0 + BZ_K);
    // only the column groups this thread owns (no predicated-off DFMAs)
    const int ncol = (s - cg + 7) >> 3;
#define BZ_CASE(NC)                                                      \
  for (int kk = 0; kk < BZ_K; ++kk) {                                    \
    const cplx b = sb[row][kk];                                          \
    _Pragma("unroll") for (int c = 0; c < NC; ++c) cfma(acc[c], b, sz[kk][cg + 8 * c]); \
  }
    switch (ncol) {
      case 1: BZ_CASE(1) break;
      case 2: BZ_CASE(2) break;
      case 3: BZ_CASE(3) break;
      case 4: BZ_CASE(4) break;
      default: break;
    }
#undef BZ_CASE
    __syncthreads();
  }
  const int gr = r0 + row;
  cplx* Y = Ypart + (size_t)blockIdx.y * n * s;
  if (gr < n) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int col = cg + 8 * c;
      if (col < s) Y[(size_t)gr * s + col] = acc[c];
    }
  }
}

// Y = B Z for Hermitian B via Y[i, c] = conj(sum_k conj(Z[k, c]) B[k, i]):
// thread i streams column i of B down rows k (coalesced across the warp, each
// element read once, 8 loads in flight per thread), Z rows broadcast from
// shared memory. Split-K over blockIdx.y; partials summed in fixed order.
#ifndef KST_BZ2_U
#define KST_BZ2_U 8  // rows of B in flight per thread
#endif
#ifndef KST_BZ2_COLS
#define KST_BZ2_COLS 128
#endif
constexpr int BZ2_COLS = KST_BZ2_COLS;
#ifndef KST_BZ2_K8
#define KST_BZ2_K8 128
#endif
template <int S>
struct Bz2K {
  // K chunk per CTA: more chunks = more CTAs in flight (B is L2-resident, the
  // kernel is latency-bound); sz stays under 48 KB
  static constexpr int value = S <= 8 ? KST_BZ2_K8 : S <= 16 ? 128 : 64;
};
template <int S>
__global__ void __launch_bounds__(BZ2_COLS) bz2_kernel(const cplx* __restrict__ B, int n,
                                                        const cplx* __restrict__ Z,
                                                        cplx* __restrict__ Ypart) {
  constexpr int BZ2_K = Bz2K<S>::value;
  __shared__ cplx sz[BZ2_K * S];
  const int i = blockIdx.x * BZ2_COLS + threadIdx.x;
  const int kbeg = blockIdx.y * BZ2_K, kend = min(n, kbeg + BZ2_K);
  for (int e = threadIdx.x; e < (kend - kbeg) * S; e += BZ2_COLS)
    sz[e] = cconj(Z[(size_t)kbeg * S + e]);
  __syncthreads();
  cplx acc[S];
#pragma unroll
  for (int c = 0; c < S; ++c) acc[c] = cmk(0, 0);
  if (i < n) {
    const cplx* col = B + i;
    int k = kbeg;
    for (; k + KST_BZ2_U <= kend; k += KST_BZ2_U) {
      cplx bv[KST_BZ2_U];
#pragma unroll
      for (int u = 0; u < KST_BZ2_U; ++u) bv[u] = col[(size_t)(k + u) * n];
#pragma unroll
      for (int u = 0; u < KST_BZ2_U; ++u) {
        const cplx* zr = sz + (k + u - kbeg) * S;
#pragma unroll
        for (int c = 0; c < S; ++c) cfma(acc[c], zr[c], bv[u]);
      }
    }
    for (; k < kend; ++k) {
      const cplx bv = col[(size_t)k * n];
      const cplx* zr = sz + (k - kbeg) * S;
#pragma unroll
      for (int c = 0; c < S; ++c) cfma(acc[c], zr[c], bv);
    }
    cplx* Y = Ypart + (size_t)blockIdx.y * n * S + (size_t)i * S;
#pragma unroll
    for (int c = 0; c < S; ++c) Y[c] = cconj(acc[c]);
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

// out[e] = sum_blk partial[blk][e], fixed order (eight loads in flight, the
// additions in block order)
__global__ void reduce_partials_kernel(const cplx* __restrict__ partial, int nblk, int count,
                                       cplx* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    int b = 0;
    for (; b + 8 <= nblk; b += 8) {
      cplx v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = partial[(size_t)(b + u) * count + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = cadd(acc, v[u]);
    }
    for (; b < nblk; ++b) acc = cadd(acc, partial[(size_t)b * count + e]);
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

// Z0 (n x s) = unit vectors e_i for the s largest Re(B_ii) (ties -> lower i).
// One CTA (1024 threads); the diagonal is gathered into smem once (all its
// strided loads in flight together) when it fits (dyn_n > 0), and the s
// selection rounds then read smem.
__global__ void __launch_bounds__(1024) unit_start_kernel(const cplx* __restrict__ B, int n, int s,
                                                          cplx* __restrict__ Z, int dyn_n,
                                                          const double* __restrict__ mdiag,
                                                          int* __restrict__ picked_out) {
  extern __shared__ double dg[];
  __shared__ int picked[32];
  __shared__ double bv[32];
  __shared__ int bi[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = threadIdx.x; i < dyn_n; i += blockDim.x) dg[i] = mdiag ? mdiag[i] : B[(size_t)i * n + i].x;
  __syncthreads();  // Z was zeroed by the caller (memset: the whole GPU, not one SM)
  // s rounds of a block argmax (ties -> lower i): thread -> warp (shuffles)
  // -> warp 0 over the 32 warp winners (shuffles), two barriers per round
  const int nw = (int)(blockDim.x >> 5);
  for (int k = 0; k < s; ++k) {
    double best = -INFINITY;
    int besti = n;
    if (dyn_n) {  // picked entries are knocked out of the staged diagonal (finite values)
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = dg[i];
        if (v > best || (v == best && i < besti)) {
          best = v;
          besti = i;
        }
      }
    } else {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool used = false;
        for (int j = 0; j < k; ++j) used |= picked[j] == i;
        const double v = B[(size_t)i * n + i].x;
        if (!used && (v > best || (v == best && i < besti))) {
          best = v;
          besti = i;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
      if (ob > best || (ob == best && oi < besti)) {
        best = ob;
        besti = oi;
      }
    }
    if (l == 0) {
      bv[w] = best;
      bi[w] = besti;
    }
    __syncthreads();
    if (w == 0) {
      double b0 = l < nw ? bv[l] : -INFINITY;
      int i0 = l < nw ? bi[l] : n;
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b0, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i0, o);
        if (ob > b0 || (ob == b0 && oi < i0)) {
          b0 = ob;
          i0 = oi;
        }
      }
      if (l == 0) {
        picked[k] = i0 >= n ? k : i0;  // fewer candidates than s (cannot happen for n > 64)
        if (dyn_n && i0 < n) dg[i0] = -INFINITY;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < s) {
    Z[(size_t)picked[threadIdx.x] * s + threadIdx.x] = cmk(1.0, 0.0);
    picked_out[threadIdx.x] = picked[threadIdx.x];
  }
}

// Y = B Z0 for the unit-vector start block: Y[i][c] = conj(B[p_c][i]) (row p_c
// of the Hermitian B read contiguously), the value bz2_kernel forms as
// conj(sum_k B[k][i] conj(Z0[k][c])) -- no pass over all of B
__global__ void start_cols_kernel(const cplx* __restrict__ B, int n, int s, const int* __restrict__ picked,
                                  cplx* __restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * s;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n), i = (int)(e % n);
    Y[(size_t)i * s + c] = cconj(B[(size_t)picked[c] * n + i]);
  }
}

// heig_top's Rayleigh-Ritz convergence test, on the device for both the
// synchronous loop and the sync-free form: res_red[k] = sum over the row-
// block partials of the k-th squared residual (one warp, fixed-order lane
// sums + xor tree: both paths see identical values), then every wanted pair
// with residual <= 1e-12 max|theta|, or <= 1e-9 max|theta| and <= 1e-8 of
// its gap, and kept > 0 -> *ok = 1.
__global__ void rr_check_kernel(const double* __restrict__ res_part, int nup, int r,
                                const double* __restrict__ th, int s, const int* __restrict__ info,
                                double* __restrict__ res_red, int* __restrict__ ok) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < r; ++k) {
    double acc = 0.0;
    for (int b = lane; b < nup; b += 32) acc += res_part[(size_t)b * r + k];
    acc = warp_sum(acc);
    if (lane == 0) res_red[k] = acc;
  }
  __syncwarp();
  if (lane != 0) return;
  double tmax = 0.0;
  for (int k = 0; k < s; ++k) tmax = fmax(tmax, fabs(th[k]));
  bool all_ok = true;
  for (int k = 0; k < r; ++k) {
    const double res = sqrt(res_red[k]);
    double gap = 1e300;
    for (int jx = 0; jx < s; ++jx)
      if (jx != k) gap = fmin(gap, fabs(th[k] - th[jx]));
    all_ok = all_ok && (res <= 1e-12 * tmax || (res <= 1e-9 * tmax && res <= 1e-8 * gap));
  }
  *ok = (info[0] != 0 && (tmax == 0.0 || all_ok)) ? 1 : 0;
}

// Final ordering (descending, reference tie rule) + pivot phase for the top r
// Ritz vectors; single CTA of 1024 threads, s <= 32. The pivot search (argmax
// |Z[i][k]| per column, lowest index on ties) maps thread t to column t % s and
// rows t / s, t / s + 1024 / s, ... (row-contiguous, coalesced loads), then
// one warp per column reduces the row groups.
__global__ void __launch_bounds__(1024) finalize_top_kernel(
    const cplx* __restrict__ Z, int n, int s, int r, const double* __restrict__ theta,
    double* __restrict__ vals_out, cplx* __restrict__ vec_out) {
  __shared__ int piv[32];
  __shared__ int order[32];
  __shared__ double phr[32], phi[32];
  __shared__ double sbm[1024];
  __shared__ int sbi[1024];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  {
    const int ng = (int)blockDim.x / s;  // row groups
    const int k = threadIdx.x % s, g = threadIdx.x / s;
    double bm = -1.0;
    int bi = n;
    if (g < ng) {
      int i = g;
      for (; i + 3 * ng < n; i += 4 * ng) {  // four loads in flight, rows in ascending order
        cplx v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = Z[(size_t)(i + u * ng) * s + k];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double a = hypot(v[u].x, v[u].y);
          if (a > bm) {
            bm = a;
            bi = i + u * ng;
          }
        }
      }
      for (; i < n; i += ng) {
        const cplx v = Z[(size_t)i * s + k];
        const double a = hypot(v.x, v.y);
        if (a > bm) {
          bm = a;
          bi = i;
        }
      }
    }
    sbm[threadIdx.x] = bm;
    sbi[threadIdx.x] = bi;
    __syncthreads();
    for (int kc = w; kc < s; kc += (int)(blockDim.x >> 5)) {
      double b2 = -1.0;
      int i2 = n;
      for (int gg = l; gg < ng; gg += 32) {  // ascending groups: first maximum kept
        const double ob = sbm[gg * s + kc];
        const int oi = sbi[gg * s + kc];
        if (ob > b2 || (ob == b2 && oi < i2)) {
          b2 = ob;
          i2 = oi;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b2, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i2, o);
        if (ob > b2 || (ob == b2 && oi < i2)) {
          b2 = ob;
          i2 = oi;
        }
      }
      if (l == 0) piv[kc] = i2 < n ? i2 : 0;
    }
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
// ---------------------------------------------------------------- K4 v2 kernels
// Block power iteration with Rayleigh-Ritz and scaled-SVQB orthonormalisation:
//   Y = B Z;  H = Z^H Y = Q Theta Q^H (Ritz);  G' = (YQ)^H (YQ);
//   D = diag(G')^-1/2;  D G' D = V S^2 V^H;  Z <- Y Q D V S^-1.
// Ritz residuals |Y q_k - theta_k Z q_k| are formed directly (no Gram
// cancellation). All small-matrix work runs in one CTA (k4_small_kernel).
constexpr int K4_ROWS = 16;

// partial[blk] = {Z^H Y1, Y2^H Y2} over a chunk of rows (s x s each)
__global__ void __launch_bounds__(256) k4_gram_kernel(const cplx* __restrict__ Z,
                                                      const cplx* __restrict__ Y1,
                                                      const cplx* __restrict__ Y2, int n, int s,
                                                      cplx* __restrict__ partial) {
  __shared__ cplx sz[K4_ROWS][33];
  __shared__ cplx sy[K4_ROWS][33];
  __shared__ cplx s2[K4_ROWS][33];
  // each CTA walks row tiles blockIdx.x, +gridDim.x, ... (few partials to reduce)
  cplx acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = cmk(0, 0);
  for (int r0 = blockIdx.x * K4_ROWS; r0 < n; r0 += gridDim.x * K4_ROWS) {
    const int rows = min(K4_ROWS, n - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < K4_ROWS * s; e += 256) {
      const int rr = e / s, a = e % s;
      sz[rr][a] = rr < rows ? Z[(size_t)(r0 + rr) * s + a] : cmk(0, 0);
      sy[rr][a] = rr < rows ? Y1[(size_t)(r0 + rr) * s + a] : cmk(0, 0);
      s2[rr][a] = rr < rows ? Y2[(size_t)(r0 + rr) * s + a] : cmk(0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + 256 * u;
      if (e < 2 * s * s) {
        const int which = e / (s * s), ab = e % (s * s);
        const int a = ab / s, b = ab % s;
        if (which == 0)
          for (int rr = 0; rr < K4_ROWS; ++rr) cfmca(acc[u], sz[rr][a], sy[rr][b]);
        else
          for (int rr = 0; rr < K4_ROWS; ++rr) cfmca(acc[u], s2[rr][a], s2[rr][b]);
      }
    }
  }
  cplx* out = partial + (size_t)blockIdx.x * 2 * s * s;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + 256 * u;
    if (e < 2 * s * s) out[e] = acc[u];
  }
}

// One CTA. mode 0: Rayleigh-Ritz + orthonormalise Y; mode 1: orthonormalise
// only (Q = I). Writes C (s x s), Q (s x s), theta (s), info[0] = kept columns,
// info[1] = Jacobi sweeps (diagnostic).
__global__ void __launch_bounds__(256) k4_small_kernel(const cplx* __restrict__ partial, int nblk,
                                                       int s, int mode, cplx* __restrict__ Cout,
                                                       cplx* __restrict__ Qout,
                                                       double* __restrict__ theta,
                                                       int* __restrict__ info) {
  extern __shared__ __align__(16) char sm[];
  __shared__ double dsc[32], th[32];
  cplx* H = (cplx*)(sm + ((jac_smem_bytes(s) + 15) / 16) * 16);
  cplx* G = H + s * s;
  cplx* Q = G + s * s;
  cplx* T = Q + s * s;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  (void)w;
  (void)l;
  // fixed-order reduction of the partials: one thread per complex entry, the
  // nblk loads of an entry are independent and issued back to back
  for (int e = tid; e < 2 * s * s; e += blockDim.x) {
    cplx acc = cmk(0, 0);
#pragma unroll 8
    for (int b = 0; b < nblk; ++b) acc = cadd(acc, partial[(size_t)b * 2 * s * s + e]);
    if (e < s * s) H[e] = acc;
    else G[e - s * s] = acc;
  }
  __syncthreads();
  JacSmem j = jac_carve(sm, s);
  if (mode == 0) {
    jac_solve(j, H, s, s, 1.0);
    for (int e = tid; e < s * s; e += blockDim.x) {
      const int i = e / s, k = e % s;
      Q[e] = j.V[i * j.ld + j.order[k]];
    }
    for (int k = tid; k < s; k += blockDim.x) th[k] = j.val[j.order[k]];
  } else {
    for (int e = tid; e < s * s; e += 256) Q[e] = cmk((e / s) == (e % s) ? 1.0 : 0.0, 0.0);
    for (int k = tid; k < s; k += blockDim.x) th[k] = 0.0;
  }
  __syncthreads();
  // T = G Q, then G' = Q^H T (reuse H)
  for (int e = tid; e < s * s; e += blockDim.x) {
    const int a = e / s, k = e % s;
    cplx acc = cmk(0, 0);
    for (int b = 0; b < s; ++b) cfma(acc, G[a * s + b], Q[b * s + k]);
    T[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < s * s; e += blockDim.x) {
    const int a = e / s, k = e % s;
    cplx acc = cmk(0, 0);
    for (int b = 0; b < s; ++b) cfmca(acc, Q[b * s + a], T[b * s + k]);
    H[e] = acc;
  }
  __syncthreads();
  for (int k = tid; k < s; k += blockDim.x) {
    const double g = H[k * s + k].x;
    dsc[k] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < s * s; e += blockDim.x) {
    const int a = e / s, b = e % s;
    G[e] = cscale(H[e], dsc[a] * dsc[b]);
  }
  __syncthreads();
  // Fast path: scaled Cholesky QR. G~ = R^H R (R upper, in T), C = Q D R^-1.
  // mode 0: taken when every pivot stays >= 1e-10 (well-conditioned block, all
  // iterations after the warm-up), else SVQB by Jacobi. mode 1 (warm-up
  // orthonormalisation, always followed by another pass): shifted Cholesky QR,
  // G~ + 1e-11 I, never needs the Jacobi -- nearly dependent directions come
  // out short instead of unit length and the next pass re-normalises them.
  {
    __shared__ int chol_ok;
    const double shift = mode == 1 ? 1e-11 : 0.0, pmin = mode == 1 ? 0.0 : 1e-10;
    for (int e = tid; e < s * s; e += blockDim.x)
      T[e] = (e / s == e % s) ? cmk(G[e].x + shift, G[e].y) : G[e];
    if (tid == 0) chol_ok = 1;
    __syncthreads();
    for (int k = 0; k < s; ++k) {
      const double dkk = T[k * s + k].x;
      if (!(dkk >= pmin) || !(dkk > 0.0)) {
        if (tid == 0) chol_ok = 0;
        break;  // uniform across the block (all threads read the same dkk)
      }
      const double rkk = sqrt(dkk);
      __syncthreads();
      // row k of R: R[k][j] = T[k][j] / rkk (j > k); R[k][k] = rkk
      for (int jj = k + 1 + tid; jj < s; jj += blockDim.x) T[k * s + jj] = cscale(T[k * s + jj], 1.0 / rkk);
      __syncthreads();
      if (tid == 0) T[k * s + k] = cmk(rkk, 0.0);
      // trailing update T[i][jj] -= conj(R[k][i]) R[k][jj], i, jj > k
      const int m = s - k - 1;
      for (int e = tid; e < m * m; e += blockDim.x) {
        const int i = k + 1 + e / m, jj = k + 1 + e % m;
        const cplx a = T[k * s + i], b = T[k * s + jj];
        T[i * s + jj] = csub(T[i * s + jj], cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x));
      }
      __syncthreads();
    }
    __syncthreads();
    if (chol_ok) {
      // Rinv (upper) by column-parallel back substitution, stored in G
      for (int col = tid; col < s; col += blockDim.x) {
        for (int i = s - 1; i >= 0; --i) {
          cplx acc = cmk(i == col ? 1.0 : 0.0, 0.0);
          for (int jj = i + 1; jj <= col; ++jj) acc = csub(acc, cmul(T[i * s + jj], G[jj * s + col]));
          G[i * s + col] = i > col ? cmk(0, 0) : cscale(acc, 1.0 / T[i * s + i].x);
        }
      }
      __syncthreads();
      for (int e = tid; e < s * s; e += blockDim.x) {
        const int a = e / s, k = e % s;
        cplx acc = cmk(0, 0);
        for (int b = 0; b <= k; ++b) cfma(acc, Q[a * s + b], cscale(G[b * s + k], dsc[b]));
        Cout[e] = acc;
        Qout[e] = Q[e];
      }
      if (tid == 0) {
        info[0] = s;
        info[1] = 2;  // Cholesky path
      }
      if (mode == 0)
        for (int k = tid; k < s; k += blockDim.x) theta[k] = th[k];
      return;
    }
  }
  jac_solve(j, G, s, s, 1.0);
  // C = Q D V S^-1. Nearly dependent directions are NOT dropped: their tiny
  // singular values are floored, so they come back as amplified rounding
  // noise -- fresh trial directions -- and the next pass orthonormalises them.
  const double smax = j.val[j.order[0]];
  for (int e = tid; e < s * s; e += blockDim.x) {
    const int a = e / s, k = e % s;
    const double sg = fmax(j.val[j.order[k]], 1e-30 * smax);
    cplx acc = cmk(0, 0);
    if (smax > 0.0) {
      const double inv = 1.0 / sqrt(sg);
      for (int b = 0; b < s; ++b)
        cfma(acc, Q[a * s + b], cscale(j.V[b * j.ld + j.order[k]], dsc[b] * inv));
    }
    Cout[e] = acc;
    Qout[e] = Q[e];
  }
  if (tid == 0) {
    int kept = 0;
    for (int k = 0; k < s; ++k) kept += (smax > 0.0 && j.val[j.order[k]] > 1e-26 * smax) ? 1 : 0;
    info[0] = kept;  // diagnostic: numerically independent directions
    info[1] = smax > 0.0 ? 1 : 0;
  }
  if (mode == 0)
    for (int k = tid; k < s; k += blockDim.x) theta[k] = th[k];
}

// Z_new = Y C; X = Z Q (Ritz vectors); residual partials sum_rows |Y q_k - th_k X_k|^2
// blockDim (32, 8): x = column, y = row in block. mode 1: only Z_new = Y C.
__global__ void __launch_bounds__(256) k4_update_kernel(
    const cplx* __restrict__ Y, const cplx* __restrict__ Y2, const cplx* __restrict__ Z, int n,
    int s, int r, int mode,
    const cplx* __restrict__ C, const cplx* __restrict__ Q, const double* __restrict__ theta,
    cplx* __restrict__ Znew, cplx* __restrict__ X, double* __restrict__ res_part) {
  __shared__ cplx sC[32 * 32], sQ[32 * 32];
  __shared__ double sres[8][32];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < s * s; e += 256) {
    sC[e] = C[e];
    sQ[e] = Q[e];
  }
  __syncthreads();
  const int row = blockIdx.x * 8 + threadIdx.y, k = threadIdx.x;
  double rr = 0.0;
  if (row < n && k < s) {
    cplx zn = cmk(0, 0), x = cmk(0, 0), yq = cmk(0, 0);
    for (int a = 0; a < s; ++a) {
      const cplx y = Y[(size_t)row * s + a];
      cfma(zn, Y2[(size_t)row * s + a], sC[a * s + k]);
      if (mode == 0) {
        cfma(yq, y, sQ[a * s + k]);
        cfma(x, Z[(size_t)row * s + a], sQ[a * s + k]);
      }
    }
    Znew[(size_t)row * s + k] = zn;
    if (mode == 0) {
      X[(size_t)row * s + k] = x;
      if (k < r) rr = cabs2(cmk(yq.x - theta[k] * x.x, yq.y - theta[k] * x.y));
    }
  }
  sres[threadIdx.y][threadIdx.x] = rr;
  __syncthreads();
  if (mode == 0 && threadIdx.y == 0 && k < r) {
    double acc = 0.0;
    for (int i = 0; i < 8; ++i) acc += sres[i][k];
    res_part[(size_t)blockIdx.x * r + k] = acc;
  }
}

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

int bz(kst_ctx* ctx, const cplx* B, int n, const cplx* Z, int s, cplx* Y, cudaStream_t st) {
  if (s % 8 == 0 && s <= 32) {
    const int kc = s <= 8 ? KST_BZ2_K8 : s <= 16 ? 128 : 64;  // == Bz2K<s>
    const int ks = (n + kc - 1) / kc;
    cplx* part = (cplx*)ws_get(ctx, WS_BZ, sizeof(cplx) * (size_t)ks * n * s);
    if (!part) return set_err(ctx, KST_ERR_CUDA, "bz: workspace");
    const dim3 grid(cdiv(n, BZ2_COLS), ks);
    switch (s) {
      case 8: bz2_kernel<8><<<grid, BZ2_COLS, 0, st>>>(B, n, Z, part); break;
      case 16: bz2_kernel<16><<<grid, BZ2_COLS, 0, st>>>(B, n, Z, part); break;
      case 24: bz2_kernel<24><<<grid, BZ2_COLS, 0, st>>>(B, n, Z, part); break;
      default: bz2_kernel<32><<<grid, BZ2_COLS, 0, st>>>(B, n, Z, part); break;
    }
    KST_LAUNCH(ctx);
    reduce_partials_kernel<<<grid_for((int64_t)n * s), 256, 0, st>>>(part, ks, n * s, Y);
    KST_LAUNCH(ctx);
    return KST_OK;
  }
  const int ks = (n + BZ_KSPLIT - 1) / BZ_KSPLIT;
  cplx* part = (cplx*)ws_get(ctx, WS_BZ, sizeof(cplx) * (size_t)ks * n * s);
  if (!part) return set_err(ctx, KST_ERR_CUDA, "bz: workspace");
  bz_kernel<<<dim3(cdiv(n, BZ_ROWS), ks), 128, 0, st>>>(B, n, Z, s, part);
  KST_LAUNCH(ctx);
  reduce_partials_kernel<<<grid_for((int64_t)n * s), 256, 0, st>>>(part, ks, n * s, Y);
  KST_LAUNCH(ctx);
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

// ok_dev != nullptr (host-sync-free form, n > kMaxN, r <= 24): the fixed
// schedule of the common case -- warm-up, ONE Rayleigh-Ritz round -- with the
// round-0 convergence test on the device (rr_check_kernel: 1 in *ok_dev when
// the host loop would have stopped after that round, 0 otherwise), values
// left on the device (*values_dev_out); no stream synchronisation.
int heig_top(kst_ctx* ctx, const cplx* M, int n, int r, double* values_host, cplx* vectors,
             cudaStream_t st, int* ok_dev, const double** values_dev_out, const double* mdiag) {
  if (r < 1 || r > n) return set_err(ctx, KST_ERR_DIMENSION, "heig_top: r=%d n=%d", r, n);
  if (ok_dev && (n <= kMaxN || r > 24))
    return set_err(ctx, KST_ERR_DIMENSION, "heig_top: no sync-free form for n=%d r=%d", n, r);
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

  // block: r wanted + >= 5 guard vectors (convergence rate lambda_{s+1}/lambda_r)
  const int s = std::min(32, ((std::max(8, r + 5) + 7) / 8) * 8);
  const size_t nb = (size_t)n * s;
  const int nblk = std::min((n + K4_ROWS - 1) / K4_ROWS, 32);
  const int nup = (n + 7) / 8;
  size_t bytes = sizeof(cplx) * (nb * 5 + (size_t)s * s * 2) +
                 sizeof(double) * ((size_t)nup * r + 2 * s + r + 4) + sizeof(int) * 8 + 256;
  char* base = (char*)ws_get(ctx, WS_EIG, bytes);
  cplx* partial = (cplx*)ws_get(ctx, WS_EIG2, sizeof(cplx) * (size_t)nblk * 2 * s * s +
                                                  sizeof(double) * (size_t)nup * r + 64);
  double* hres = (double*)pinned_get(ctx, sizeof(double) * (2 * s + r + 8));
  if (!base || !partial || !hres) return set_err(ctx, KST_ERR_CUDA, "heig_top: workspace");
  cplx* Z = (cplx*)base;
  cplx* Y = Z + nb;
  cplx* Y2 = Y + nb;
  cplx* Zn = Y2 + nb;
  cplx* X = Zn + nb;
  cplx* Cm = X + nb;
  cplx* Qm = Cm + s * s;
  // [residual partials | theta | vout | info (2 ints) | reduced residuals | ok]:
  // theta .. ok contiguous, one readback per Rayleigh-Ritz round
  double* res_part = (double*)(Qm + s * s);
  double* theta = res_part + (size_t)nup * r;
  double* vout = theta + s;
  int* info = (int*)(vout + s);
  double* res_red = (double*)(info + 2);
  int* ok_loop = (int*)(res_red + r);
  const size_t small_smem = ((jac_smem_bytes(s) + 15) / 16) * 16 + sizeof(cplx) * 4 * s * s;
  static bool small_attr = false;
  if (!small_attr) {
    KST_CUDA(ctx, cudaFuncSetAttribute(k4_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(((jac_smem_bytes(32) + 15) / 16) * 16 +
                                             sizeof(cplx) * 4 * 32 * 32)));
    small_attr = true;
  }
  // mode 0: Ritz pairs of span(Zc) from Y1 = B Zc; next block = orth(Y2), Y2 = B Y1
  // mode 1: Zc <- orth(Y2) only
  auto step = [&](const cplx* Zc, const cplx* Y1, const cplx* Y2c, int mode) -> int {
    k4_gram_kernel<<<nblk, 256, 0, st>>>(Zc, Y1, Y2c, n, s, partial);
    KST_LAUNCH(ctx);
    k4_small_kernel<<<1, 128, small_smem, st>>>(partial, nblk, s, mode, Cm, Qm, theta, info);
    KST_LAUNCH(ctx);
    k4_update_kernel<<<nup, dim3(32, 8), 0, st>>>(Y1, Y2c, Zc, n, s, r, mode, Cm, Qm, theta, Zn,
                                                   X, res_part);
    KST_LAUNCH(ctx);
    std::swap(Z, Zn);  // Zn (= Y2 C) becomes the current block
    return KST_OK;
  };
  // Z0 = unit vectors at the s largest diagonal entries of B (orthonormal by
  // construction; B e_i is the i-th column, rich in the dominant directions)
  {
    const int dyn_n = n <= 24 * 1024 ? n : 0;  // diagonal staged in smem up to 192 KB
    if (dyn_n > 6 * 1024)
      KST_CUDA(ctx, cudaFuncSetAttribute(unit_start_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(double) * dyn_n)));
    KST_CUDA(ctx, cudaMemsetAsync(Z, 0, sizeof(cplx) * (size_t)n * s, st));
    int* picked = (int*)partial;  // scratch: consumed before k4_gram writes the partials
    unit_start_kernel<<<1, 1024, sizeof(double) * dyn_n, st>>>(M, n, s, Z, dyn_n, mdiag, picked);
    KST_LAUNCH(ctx);
    start_cols_kernel<<<grid_for((int64_t)n * s), 256, 0, st>>>(M, n, s, picked, Y);  // Y = B Z0
  }
  KST_LAUNCH(ctx);
  // Warm-up without Rayleigh-Ritz (Ritz pairs of the start block are useless):
  // Z <- orth(B^4 Z0), two orthonormalisation passes (SVQB when the block is
  // ill-conditioned, Cholesky-QR once it is not).
  KST_TRY(bz(ctx, M, n, Y, s, Y2, st));
  KST_TRY(bz(ctx, M, n, Y2, s, Y, st));
  KST_TRY(bz(ctx, M, n, Y, s, Y2, st));
  KST_TRY(step(Z, Z, Y2, 1));
  KST_TRY(step(Z, Z, Z, 1));

  if (ok_dev) {
    KST_TRY(bz(ctx, M, n, Z, s, Y, st));
    KST_TRY(bz(ctx, M, n, Y, s, Y2, st));
    cplx* Zcur = Z;
    KST_TRY(step(Zcur, Y, Y2, 0));
    rr_check_kernel<<<1, 32, 0, st>>>(res_part, nup, r, theta, s, info, res_red, ok_dev);
    KST_LAUNCH(ctx);
    finalize_top_kernel<<<1, 1024, 0, st>>>(X, n, s, r, theta, vout, vectors);
    KST_LAUNCH(ctx);
    if (values_dev_out) *values_dev_out = vout;
    return KST_OK;
  }
  bool converged = false;
  double prev_worst = 1e300;
  int stall = 0;
  for (int it = 0; it < 60 && !converged; ++it) {
    // two power steps per Rayleigh-Ritz (halves the sequential small steps)
    KST_TRY(bz(ctx, M, n, Z, s, Y, st));
    KST_TRY(bz(ctx, M, n, Y, s, Y2, st));
    cplx* Zcur = Z;
    KST_TRY(step(Zcur, Y, Y2, 0));  // X = Ritz vectors of span(Zcur); Z <- orth(B^2 Zcur)
    rr_check_kernel<<<1, 32, 0, st>>>(res_part, nup, r, theta, s, info, res_red, ok_loop);
    KST_LAUNCH(ctx);
    KST_CUDA(ctx, cudaMemcpyAsync(hres, theta, sizeof(double) * (2 * s + r) + 2 * sizeof(int),
                                  cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    const double* th = hres;
    const int kept = *(int*)(hres + 2 * s);
    const int path = *((int*)(hres + 2 * s) + 1);
    const double* hred = hres + 2 * s + 1;  // the device-reduced squared residuals
    double tmax = 0.0, worst = 0.0;
    for (int k = 0; k < s; ++k) tmax = std::max(tmax, std::fabs(th[k]));
    // Converged when every wanted Ritz pair has residual <= 1e-12 max|theta|
    // (the FP64 floor), or <= 1e-9 max|theta| AND <= 1e-8 of its gap to the
    // other Ritz values: eigenvector error <= residual / gap <= 1e-8.
    bool all_ok = true;
    for (int k = 0; k < r; ++k) {
      const double res = std::sqrt(hred[k]);
      worst = std::max(worst, res);
      double gap = 1e300;
      for (int jx = 0; jx < s; ++jx)
        if (jx != k) gap = std::min(gap, std::fabs(th[k] - th[jx]));
      all_ok = all_ok && (res <= 1e-12 * tmax || (res <= 1e-9 * tmax && res <= 1e-8 * gap));
    }
    {
      static const bool dbg = getenv("KST_HEIG_DEBUG") != nullptr;  // convergence margins
      if (dbg)
        for (int k = 0; k < r; ++k) {
          double gap = 1e300;
          for (int jx = 0; jx < s; ++jx)
            if (jx != k) gap = std::min(gap, std::fabs(th[k] - th[jx]));
          fprintf(stderr, "[heig_top] round %d pair %d: res/tmax %.3e (1e-12), res/gap %.3e (1e-8)\n",
                  it, k, std::sqrt(hred[k]) / tmax, std::sqrt(hred[k]) / gap);
        }
    }
    if (kept == 0) break;  // B^2 Z vanished: leave it to the dense solver
    if (tmax == 0.0 || all_ok) {
      converged = true;
    } else if (worst <= 1e-9 * tmax) {
      // accept a residual floor once it stops improving
      stall = (worst > 0.5 * prev_worst) ? stall + 1 : 0;
      if (stall >= 3) converged = true;
    }
    prev_worst = worst;
    // the SVQB path (ill-conditioned block) regenerates noise directions that
    // need a second orthonormalisation; the Cholesky path is already orthonormal
    if (!converged && path != 2) KST_TRY(step(Z, Z, Z, 1));
  }
  if (!converged) return heig_top_cusolver(ctx, M, n, r, values_host, vectors, st);
  finalize_top_kernel<<<1, 1024, 0, st>>>(X, n, s, r, theta, vout, vectors);
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
