// K1 on the int8 tensor cores: Ozaki-style error-free slicing of the FP64
// Gram S = (1/n) X^T conj(X) (`sample_covariance`, src/lrkron.py:53-78).
//
// Each snapshot column a (real and imaginary parts together) is scaled by a
// power of two 2^-E_a (|x| < 2^E_a) and cut into s signed 7-bit slices
// (truncation; every remainder is exact in FP64):
//     x[k,a] = 2^E_a * sum_t sigma_t[k,a] * 2^(-7t) + O(2^(E_a - 7s)).
// Products of slices are exact in int32, so with the K-stacking trick
//     G_e = sum_{t+u=e} sigma_t^T sigma_u = [sigma_1..sigma_{e-1}]^T [sigma_{e-1}..sigma_1]
// one int8 GEMM per diagonal e = 2..s+1 yields every kept pair exactly
// (|G_e| <= (e-1) K 127^2 < 2^31). Then
//     Re S = 2^(E_a+E_b)/n * sum_e 2^-7e (GR_e + GI_e)       (GR: Xr.Xr, GI: Xi.Xi)
//     Im S = 2^(E_a+E_b)/n * sum_e 2^-7e (M_e[a,b] - M_e[b,a]) (M: Xi.Xr)
// so S is exactly Hermitian with a real diagonal. Dropped pairs (t+u > s+1)
// and the truncated tail bound the relative error by ~(s+1) 2^(-7s)
// (s = 6: ~2e-12; s = 7: ~1e-14) of max|x_a| max|x_b| K.
//
// The int8 GEMMs are plain library GEMMs (cuBLAS, int8 x int8 -> int32 on
// the B200 tensor cores, bound with dlopen); slicing and recombination are
// hand-written kernels. Non-finite columns poison their S entries with NaN so
// the estimator's finite check raises DataError exactly like the FP64 path.
#include <dlfcn.h>

#include <algorithm>

#include "gram_i8.cuh"

namespace kst {
namespace i8 {

// E_a per column: smallest E with max_k max(|re|, |im|) < 2^E; NaN sentinel
// for non-finite columns; 0 for all-zero columns (slices are then zero).
// CTA = 32 columns x 8 row groups (coalesced over columns), smem max-reduce.
__global__ void colmax_kernel(const cplx* __restrict__ X, int64_t n, int64_t d,
                              int* __restrict__ expo) {
  __shared__ double sm[8][33];
  __shared__ int sb[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t a = blockIdx.x * 32 + tx;
  double m = 0.0;
  int bad = 0;
  if (a < d)
    for (int64_t k = ty; k < n; k += 8) {
      const cplx v = X[k * d + a];
      bad |= !isfinite(v.x) || !isfinite(v.y);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
  sm[ty][tx] = m;
  sb[ty][tx] = bad;
  __syncthreads();
  if (ty == 0 && a < d) {
    for (int r = 1; r < 8; ++r) {
      m = fmax(m, sm[r][tx]);
      bad |= sb[r][tx];
    }
    expo[a] = bad ? kNaNExpo : (m > 0.0 ? ilogb(m) + 1 : 0);
  }
}

}  // namespace i8
}  // namespace kst

namespace {

using kst::i8::kNaNExpo;
using kst::i8::colmax_kernel;

// Slices, column-major per snapshot element a (K blocks of npad contiguous):
//   RIf[a][2t + c][k] = sigma_{t+1}(part c)[k,a]       (c = 0 real, 1 imag)
//   RIr[a][2(s-1-t) + c][k] = sigma_{t+1}(part c)[k,a]  (reversed slice order)
//   If [a][t][k] = sigma_{t+1}(imag),  Rr[a][s-1-t][k] = sigma_{t+1}(real)
// A prefix of RIf against the matching suffix of RIr pairs (sigma_t, sigma_{e-t})
// of the same part for every t, so Re = GR_e + GI_e is ONE int8 GEMM per e.
// CTA = 16 columns a x 128 rows k. Phase 1 reads X coalesced over a and cuts
// each element into its 2s slice bytes, staged in smem as [part][t][a][k];
// phase 2 writes every (a, slice) row segment with 4-byte stores coalesced
// over k (128 contiguous bytes per warp store). Padded rows/columns
// (k >= n, a >= d) are written as zero slices.
constexpr int SL_A = 16, SL_K = 128, SL_KP = SL_K + 4;
template <int SS>
__global__ void __launch_bounds__(256) slice_kernel(
    const cplx* __restrict__ X, int64_t n, int64_t npad, int64_t d, int64_t dpad,
    const int* __restrict__ expo, int8_t* __restrict__ RIf, int8_t* __restrict__ RIr,
    int8_t* __restrict__ If, int8_t* __restrict__ Rr) {
  constexpr int s = SS;
  __shared__ __align__(16) int8_t sb[2][s][SL_A][SL_KP];
  const int64_t k0 = (int64_t)blockIdx.y * SL_K, a0 = (int64_t)blockIdx.x * SL_A;
  const int tid = threadIdx.x;
  {
    const int c = tid & (SL_A - 1);
    const int64_t a = a0 + c;
    const int e = a < d ? expo[a] : 0;
    const double sc = (e == kNaNExpo) ? 0.0 : ldexp(1.0, -e);
    for (int r = tid / SL_A; r < SL_K; r += 256 / SL_A) {
      const int64_t k = k0 + r;
      const cplx v = (k < n && a < d) ? X[k * d + a] : cmk(0, 0);
      double rr = v.x * sc, ri = v.y * sc;  // |.| < 1
#pragma unroll
      for (int t = 0; t < s; ++t) {
        rr *= 128.0;
        ri *= 128.0;
        const double qr = trunc(rr), qi = trunc(ri);
        rr -= qr;  // exact
        ri -= qi;
        sb[0][t][c][r] = (int8_t)qr;
        sb[1][t][c][r] = (int8_t)qi;
      }
    }
  }
  __syncthreads();
  const int lane = tid & 31, w = tid >> 5;
  const int64_t k = k0 + 4 * lane;
  if (k >= npad) return;  // npad is a multiple of 16: whole words only
  for (int c = w; c < SL_A; c += 8) {
    const int64_t a = a0 + c;
    if (a >= dpad) break;
    const int64_t b2 = a * (int64_t)(2 * s) * npad + k, b1 = a * (int64_t)s * npad + k;
#pragma unroll
    for (int t = 0; t < s; ++t) {
      const uint32_t qr = *(const uint32_t*)&sb[0][t][c][4 * lane];
      const uint32_t qi = *(const uint32_t*)&sb[1][t][c][4 * lane];
      *(uint32_t*)(RIf + b2 + (int64_t)(2 * t) * npad) = qr;
      *(uint32_t*)(RIf + b2 + (int64_t)(2 * t + 1) * npad) = qi;
      *(uint32_t*)(RIr + b2 + (int64_t)(2 * (s - 1 - t)) * npad) = qr;
      *(uint32_t*)(RIr + b2 + (int64_t)(2 * (s - 1 - t) + 1) * npad) = qi;
      *(uint32_t*)(If + b1 + (int64_t)t * npad) = qi;
      *(uint32_t*)(Rr + b1 + (int64_t)(s - 1 - t) * npad) = qr;
    }
  }
}

// S from the int32 diagonal products (column-major, ld = dpad).
// CTA per (bi <= bj) pair of 32x32 tiles; writes both S[a][b] and S[b][a].
// Templated on the slice count so the per-element plane loads are unrolled.
template <int SS>
__global__ void __launch_bounds__(256, 2) ozaki_combine_kernel(
    const int32_t* __restrict__ GRe, const int32_t* __restrict__ GM, int64_t dpad, int64_t d,
    const int* __restrict__ expo, double dn, int T, cplx* __restrict__ S) {
  constexpr int s = SS;
  __shared__ double mt[32][33];  // mt[i][j] = sum_e w_e M_e[b0+i][a0+j]
  __shared__ cplx vt[32][33];    // vt[i][j] = S[a0+i][b0+j]
  // upper-triangle tile enumeration
  const int t = blockIdx.x;
  double disc = (2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * t;
  int bi = (int)floor(((2.0 * T + 1.0) - sqrt(disc)) * 0.5);
  if (bi < 0) bi = 0;
  while (bi > 0 && bi * T - bi * (bi - 1) / 2 > t) --bi;
  while ((bi + 1) * T - (bi + 1) * bi / 2 <= t) ++bi;
  const int bj = bi + (t - (bi * T - bi * (bi - 1) / 2));
  const int64_t a0 = (int64_t)bi * 32, b0 = (int64_t)bj * 32;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const int q4 = 4 * (tid & 7), r = tid >> 3;  // 4 consecutive column-major entries per thread
  const size_t plane = (size_t)dpad * dpad;
  // exact weights 2^-7e, accumulated from the smallest term (e = s+1) up.
  // Each thread issues all its 16-byte plane loads before consuming any.
  const double w0 = ldexp(1.0, -7 * (s + 1));
  {  // transposed M block: mt[i][j] = M[b0+i][a0+j], column-major index (b0+i) + (a0+j)*dpad
    const size_t idx = (size_t)(b0 + q4) + (size_t)(a0 + r) * dpad;
    int4 v[s];
#pragma unroll
    for (int u = 0; u < s; ++u) v[u] = *(const int4*)(GM + (size_t)(s - 1 - u) * plane + idx);
    double acc[4] = {0.0, 0.0, 0.0, 0.0}, w = w0;
#pragma unroll
    for (int u = 0; u < s; ++u) {
      acc[0] += (double)v[u].x * w;
      acc[1] += (double)v[u].y * w;
      acc[2] += (double)v[u].z * w;
      acc[3] += (double)v[u].w * w;
      w *= 128.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) mt[q4 + c][r] = acc[c];
  }
  __syncthreads();
  {  // (a = a0 + q4 + c, b = b0 + r): column-major G[a][b] at a + b*dpad
    const int64_t b = b0 + r;
    const size_t idx = (size_t)(a0 + q4) + (size_t)b * dpad;
    int4 vr[s], vm[s];
#pragma unroll
    for (int u = 0; u < s; ++u) {
      vr[u] = *(const int4*)(GRe + (size_t)(s - 1 - u) * plane + idx);
      vm[u] = *(const int4*)(GM + (size_t)(s - 1 - u) * plane + idx);
    }
    double re[4] = {0.0, 0.0, 0.0, 0.0}, m_ab[4] = {0.0, 0.0, 0.0, 0.0}, w = w0;
#pragma unroll
    for (int u = 0; u < s; ++u) {
      re[0] += (double)vr[u].x * w;
      re[1] += (double)vr[u].y * w;
      re[2] += (double)vr[u].z * w;
      re[3] += (double)vr[u].w * w;
      m_ab[0] += (double)vm[u].x * w;
      m_ab[1] += (double)vm[u].y * w;
      m_ab[2] += (double)vm[u].z * w;
      m_ab[3] += (double)vm[u].w * w;
      w *= 128.0;
    }
    const int eb = (b < d) ? expo[b] : 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t a = a0 + q4 + c;
      const double im = m_ab[c] - mt[r][q4 + c];  // M[a][b] - M[b][a]
      const int ea = (a < d) ? expo[a] : 0;
      cplx v;
      if (ea == kNaNExpo || eb == kNaNExpo) {
        v = cmk(NAN, NAN);
      } else {
        v = cmk(ldexp(re[c], ea + eb) / dn, ldexp(im, ea + eb) / dn);
      }
      vt[q4 + c][r] = v;
    }
  }
  __syncthreads();
  // row-major S writes, coalesced over the column index
  for (int r = ty; r < 32; r += 8) {
    {  // S[a0 + r][b0 + tx] = vt[r][tx]
      const int64_t a = a0 + r, b = b0 + tx;
      if (a < d && b < d && (bi != bj || a <= b)) {
        const cplx v = vt[r][tx];
        S[a * d + b] = (a == b) ? cmk(v.x, 0.0) : v;
      }
    }
    {  // S[b0 + r][a0 + tx] = conj(vt[tx][r])
      const int64_t b = b0 + r, a = a0 + tx;
      if (a < d && b < d && (bi != bj || a < b)) {
        const cplx v = vt[tx][r];
        S[b * d + a] = cmk(v.x, -v.y);
      }
    }
  }
}

}  // namespace

namespace kst {
namespace i8 {
// ---------------------------------------------------------------- cuBLAS binding
Blas g_blas;
bool load_blas() {
  if (g_blas.tried) return g_blas.ok;
  g_blas.tried = true;
  const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return false;
  g_blas.create = (decltype(g_blas.create))dlsym(h, "cublasCreate_v2");
  g_blas.set_stream = (decltype(g_blas.set_stream))dlsym(h, "cublasSetStream_v2");
  g_blas.gemm_ex = (decltype(g_blas.gemm_ex))dlsym(h, "cublasGemmEx");
  g_blas.gemm_batched_ex = (decltype(g_blas.gemm_batched_ex))dlsym(h, "cublasGemmBatchedEx");
  g_blas.ok = g_blas.create && g_blas.set_stream && g_blas.gemm_ex && g_blas.gemm_batched_ex;
  return g_blas.ok;
}

cublasHandle_t blas_handle(kst_ctx* ctx, cudaStream_t st) {
  if (!ctx->cublas) {
    cublasHandle_t h;
    if (g_blas.create(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    ctx->cublas = (void*)h;
  }
  cublasHandle_t h = (cublasHandle_t)ctx->cublas;
  g_blas.set_stream(h, st);
  return h;
}

}  // namespace i8

using i8::g_blas;
using i8::load_blas;

bool ozaki_available() { return load_blas(); }

int scm_ozaki(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, int s, cudaStream_t st) {
  if (!load_blas()) return set_err(ctx, KST_ERR_CUDA, "scm_ozaki: cuBLAS not loadable");
  cublasHandle_t h = i8::blas_handle(ctx, st);
  if (!h) return set_err(ctx, KST_ERR_CUDA, "cublasCreate failed");
  const int64_t npad = ((n + 15) / 16) * 16;  // K multiple of 16 (int8 tensor-op alignment)
  // Re = GR + GI is symmetric: for large d only the NB(NB+1)/2 upper blocks of
  // an NB x NB block grid are multiplied (one batched GEMM per diagonal e).
  constexpr int NB = 4;
  const bool blocked = d >= 1024;
  const int64_t dpad = blocked ? ((d + 32 * NB - 1) / (32 * NB)) * (32 * NB) : ((d + 31) / 32) * 32;
  const int64_t bsz = dpad / NB;
  constexpr int NBLK = NB * (NB + 1) / 2;
  const size_t slice_bytes = (size_t)dpad * s * npad;
  const size_t plane = (size_t)dpad * dpad;
  char* sl = (char*)ws_get(ctx, WS_OZ_SLICES, 6 * slice_bytes + sizeof(int) * dpad +
                                                   sizeof(void*) * 3 * NBLK * 8 + 512);
  int32_t* G = (int32_t*)ws_get(ctx, WS_OZ_PROD, sizeof(int32_t) * 2 * s * plane);
  if (!sl || !G) return set_err(ctx, KST_ERR_CUDA, "scm_ozaki: workspace");
  int8_t* RIf = (int8_t*)sl;
  int8_t* RIr = RIf + 2 * slice_bytes;
  int8_t* If = RIr + 2 * slice_bytes;
  int8_t* Rr = If + slice_bytes;
  int* expo = (int*)(Rr + slice_bytes);
  void** dptr = (void**)(((uintptr_t)(expo + dpad) + 255) & ~(uintptr_t)255);  // batched pointers
  int32_t* GRe = G;
  int32_t* GM = G + (size_t)s * plane;
  if (blocked) {
    // pointer arrays for every (e, upper block): A, B, C
    void** hp = (void**)pinned_get(ctx, sizeof(void*) * 6 * NBLK * 8);
    if (!hp) return set_err(ctx, KST_ERR_CUDA, "scm_ozaki: pinned staging");
    const int lda2 = (int)(2 * s * npad);
    for (int e = 2; e <= s + 1; ++e) {
      const int64_t off2 = (int64_t)2 * (s - (e - 1)) * npad;
      int k = 0;
      for (int I = 0; I < NB; ++I)
        for (int J = I; J < NB; ++J, ++k) {
          void** row = hp + ((size_t)(e - 2) * NBLK + k) * 3;
          row[0] = (void*)(RIf + (size_t)I * bsz * lda2);
          row[1] = (void*)(RIr + off2 + (size_t)J * bsz * lda2);
          row[2] = (void*)(GRe + (size_t)(e - 2) * plane + I * bsz + (size_t)J * bsz * dpad);
        }
    }
    // de-interleave into A[], B[], C[] arrays per e on the host buffer tail
    void** ha = hp + 3 * NBLK * s;
    for (int e = 0; e < s; ++e)
      for (int k = 0; k < NBLK; ++k)
        for (int c = 0; c < 3; ++c) ha[((size_t)c * s + e) * NBLK + k] = hp[((size_t)e * NBLK + k) * 3 + c];
    KST_CUDA(ctx, cudaMemcpyAsync(dptr, ha, sizeof(void*) * 3 * NBLK * s, cudaMemcpyHostToDevice, st));
  }

  colmax_kernel<<<cdiv(d, 32), dim3(32, 8), 0, st>>>(X, n, d, expo);
  KST_LAUNCH(ctx);
  {
    const dim3 grid(cdiv(dpad, SL_A), cdiv(npad, SL_K));
#define KST_SLICE(S_)                                                                            \
  slice_kernel<S_><<<grid, 256, 0, st>>>(X, n, npad, d, dpad, expo, RIf, RIr, If, Rr)
    switch (s) {
      case 3: KST_SLICE(3); break;
      case 4: KST_SLICE(4); break;
      case 5: KST_SLICE(5); break;
      case 6: KST_SLICE(6); break;
      case 7: KST_SLICE(7); break;
      default: KST_SLICE(8); break;
    }
#undef KST_SLICE
    KST_LAUNCH(ctx);
  }
  stage_mark(ctx, 5, st);  // profiling: int8 GEMM span (events 5..6)
  const int32_t one = 1, zero = 0;
  const int lda2 = (int)(2 * s * npad), lda1 = (int)(s * npad);
  for (int e = 2; e <= s + 1; ++e) {
    int32_t* ore = GRe + (size_t)(e - 2) * plane;
    int32_t* om = GM + (size_t)(e - 2) * plane;
    // Re: GR_e + GI_e in one GEMM over the interleaved real/imag slice blocks
    const int K2 = (int)(2 * (e - 1) * npad);
    const int64_t off2 = (int64_t)2 * (s - (e - 1)) * npad;  // reversed suffix start
    cublasStatus_t r1;
    if (blocked) {
      void** A = dptr + (size_t)(0 * s + (e - 2)) * NBLK;
      void** B = dptr + (size_t)(1 * s + (e - 2)) * NBLK;
      void** Cc = dptr + (size_t)(2 * s + (e - 2)) * NBLK;
      r1 = g_blas.gemm_batched_ex(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)bsz, (int)bsz, K2, &one,
                                  (const void* const*)A, CUDA_R_8I, lda2, (const void* const*)B,
                                  CUDA_R_8I, lda2, &zero, Cc, CUDA_R_32I, (int)dpad, NBLK,
                                  CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
    } else {
      r1 = g_blas.gemm_ex(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)dpad, (int)dpad, K2, &one, RIf,
                          CUDA_R_8I, lda2, RIr + off2, CUDA_R_8I, lda2, &zero, ore, CUDA_R_32I,
                          (int)dpad, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
    }
    // M_e = sum_{t+u=e} sigma_t(Xi)^T sigma_u(Xr)
    const int K1 = (int)((e - 1) * npad);
    const int64_t off1 = (int64_t)(s - (e - 1)) * npad;
    cublasStatus_t r3 = g_blas.gemm_ex(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)dpad, (int)dpad, K1, &one,
                                       If, CUDA_R_8I, lda1, Rr + off1, CUDA_R_8I, lda1, &zero, om,
                                       CUDA_R_32I, (int)dpad, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
    if (r1 != CUBLAS_STATUS_SUCCESS || r3 != CUBLAS_STATUS_SUCCESS)
      return set_err(ctx, KST_ERR_CUDA, "cublasGemmEx (int8) failed: %d %d", (int)r1, (int)r3);
    ctx->launches += 2;
  }
  stage_mark(ctx, 6, st);
  {
    const double re_frac = blocked ? (double)NBLK / (NB * NB) : 1.0;  // Re: upper blocks only
    const double k_re = 2.0 * npad * s * (s + 1) / 2.0, k_m = (double)npad * s * (s + 1) / 2.0;
    ctx->last_int8_ops = 2.0 * (double)dpad * (double)dpad * (re_frac * k_re + k_m);
  }
  const int T = (int)(dpad / 32);
  const unsigned nt = T * (T + 1) / 2;
  const unsigned blk = 256;
  switch (s) {
    case 3: ozaki_combine_kernel<3><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
    case 4: ozaki_combine_kernel<4><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
    case 5: ozaki_combine_kernel<5><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
    case 6: ozaki_combine_kernel<6><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
    case 7: ozaki_combine_kernel<7><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
    default: ozaki_combine_kernel<8><<<nt, blk, 0, st>>>(GRe, GM, dpad, d, expo, (double)n, T, S); break;
  }
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace kst
