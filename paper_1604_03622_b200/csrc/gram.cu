// K1: Hermitian sample-covariance Gram on the FP64 tensor cores, for
// `sample_covariance` (src/lrkron.py:53-78):  S = (1/n) X^T conj(X),
// X = (n, d) snapshots, d = p*q.
//
// Design:
//  * FP64 DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4): B200 runs FP64 at
//    the same peak on the tensor pipe as on the DFMA pipe (measured 37 vs
//    34 TFLOP/s, tools/fp64_peak), with 8x fewer issue slots per FMA.
//  * 3M complex product: with planes xr, xi, s = xr + xi, d = xr - xi,
//      Re = sum xr_a xr_b + xi_a xi_b,  Im = sum s_a d_b - xr_a xr_b + xi_a xi_b,
//    three real GEMMs instead of four.
//  * Only upper-triangle 64x64 tiles are computed; each writes itself and its
//    conjugate transpose, so S is exactly Hermitian with a real diagonal (the
//    reference symmetrises with (S + S^H)/2, src/lrkron.py:77).
//  * Operand planes come from gram_prep (zero padded to the tile grid) and
//    stream through a 4-stage cp.async ring; smem rows padded to 68 doubles
//    so every fragment load is bank-conflict free. 8 warps, warp tile 32x16.
#include "common.cuh"

namespace {

constexpr int BM = 64;                  // tile edge (rows == cols)
constexpr int BK = 8;                   // snapshots per pipeline stage
constexpr int LD = BM + 4;              // padded smem row (doubles)
constexpr int STAGES = 4;
constexpr int NT = 256;
constexpr int PLANE = BK * LD;          // doubles per plane per stage
constexpr int STAGE_DOUBLES = 6 * PLANE;  // A: xr, xi, s   B: xr, xi, d

// planes[4][npad][dpad]: xr, xi, xr+xi, xr-xi
__global__ void gram_prep(const cplx* __restrict__ X, int64_t n, int64_t d, int64_t npad,
                          int64_t dpad, double* __restrict__ planes) {
  const int64_t total = npad * dpad;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx / dpad, a = idx - m * dpad;
    cplx v = cmk(0.0, 0.0);
    if (m < n && a < d) v = X[m * d + a];
    planes[idx] = v.x;
    planes[total + idx] = v.y;
    planes[2 * total + idx] = v.x + v.y;
    planes[3 * total + idx] = v.x - v.y;
  }
}

// D(8x8) += A(8x4, row) * B(4x8, col); lane (g = lane/4, t = lane%4) holds
// a = A[g][t], b = B[t][g], c = {C[g][2t], C[g][2t+1]}.
__device__ __forceinline__ void dmma(double2& c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c.x), "+d"(c.y)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tile_of(int t, int T, int& bi, int& bj) {
  // row-major enumeration of the upper triangle: row i holds T - i tiles
  double disc = (2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * t;
  int i = (int)floor(((2.0 * T + 1.0) - sqrt(disc)) * 0.5);
  if (i < 0) i = 0;
  while (i > 0 && i * T - i * (i - 1) / 2 > t) --i;
  while ((i + 1) * T - (i + 1) * i / 2 <= t) ++i;
  bi = i;
  bj = i + (t - (i * T - i * (i - 1) / 2));
}

__global__ void __launch_bounds__(NT, 2)
gram_herm_dmma(const double* __restrict__ planes, int64_t npad, int64_t dpad, int64_t n,
               int64_t d, int T, cplx* __restrict__ S) {
  extern __shared__ __align__(16) double smem[];
  int bi, bj;
  tile_of(blockIdx.x, T, bi, bj);
  const int a0 = bi * BM, b0 = bj * BM;
  const int64_t plane = npad * dpad;
  const int tid = threadIdx.x;

  // loader: 6 planes x BK rows x 32 chunks(16 B) = 1536 chunks, 6 per thread
  auto load_stage = [&](int stage, int kb) {
    double* base = smem + stage * STAGE_DOUBLES;
    const int64_t m0 = (int64_t)kb * BK;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int chunk = tid + NT * c;
      const int pl = chunk >> 8;
      const int within = chunk & 255;
      const int row = within >> 5;
      const int col = (within & 31) * 2;
      const int src_plane = pl < 3 ? pl : (pl == 5 ? 3 : pl - 3);  // A: xr xi s  B: xr xi d
      const int colbase = pl < 3 ? a0 : b0;
      cp_async16(base + pl * PLANE + row * LD + col,
                 planes + src_plane * plane + (m0 + row) * dpad + colbase + col);
    }
  };

  const int w = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (w >> 2) * 32;  // warp tile rows  [wr, wr+32)
  const int wc = (w & 3) * 16;   // warp tile cols  [wc, wc+16)

  double2 t1[4][2], t2[4][2], t3[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) t1[i][j] = t2[i][j] = t3[i][j] = make_double2(0.0, 0.0);

  const int nk = (int)(npad / BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kb + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, nxt);
      cp_async_commit();
    }
    const double* st = smem + (kb % STAGES) * STAGE_DOUBLES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int ro = (kk + t) * LD;
      double xr[4], xi[4], xs[4], yr[2], yi[2], yd[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int a = ro + wr + 8 * i + g;
        xr[i] = st[0 * PLANE + a];
        xi[i] = st[1 * PLANE + a];
        xs[i] = st[2 * PLANE + a];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = ro + wc + 8 * j + g;
        yr[j] = st[3 * PLANE + b];
        yi[j] = st[4 * PLANE + b];
        yd[j] = st[5 * PLANE + b];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(t1[i][j], xr[i], yr[j]);
          dmma(t2[i][j], xi[i], yi[j]);
          dmma(t3[i][j], xs[i], yd[j]);
        }
    }
  }
  cp_async_wait<0>();

  const double dn = (double)n;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + wr + 8 * i + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = b0 + wc + 8 * j + 2 * t + e;
        if (a >= d || b >= d) continue;
        const double v1 = e ? t1[i][j].y : t1[i][j].x;
        const double v2 = e ? t2[i][j].y : t2[i][j].x;
        const double v3 = e ? t3[i][j].y : t3[i][j].x;
        const double re = (v1 + v2) / dn;
        const double im = (v3 - v1 + v2) / dn;
        if (bi != bj || a < b) {
          S[(int64_t)a * d + b] = cmk(re, im);
          S[(int64_t)b * d + a] = cmk(re, -im);
        } else if (a == b) {
          S[(int64_t)a * d + a] = cmk(re, 0.0);
        }
      }
    }
  }
}

}  // namespace

namespace kst {

int scm(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, cudaStream_t st) {
  if (n < 1 || d < 1) return set_err(ctx, KST_ERR_DIMENSION, "scm: need n >= 1 and d >= 1");
  if (ctx->gram_mode == 1) return scm_ozaki(ctx, X, n, d, S, ctx->gram_slices, st);
  if (ctx->gram_mode == 2 || ctx->gram_mode == 3)
    return scm_crt(ctx, X, n, d, S, ctx->gram_slices, ctx->gram_mode == 2, st);
  const int64_t npad = ((n + BK - 1) / BK) * BK;
  const int64_t dpad = ((d + BM - 1) / BM) * BM;
  double* planes = (double*)ws_get(ctx, WS_PREP, sizeof(double) * 4 * npad * dpad);
  if (!planes) return set_err(ctx, KST_ERR_CUDA, "scm: workspace allocation failed");
  {
    const int64_t total = npad * dpad;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 16);
    gram_prep<<<blocks, 256, 0, st>>>(X, n, d, npad, dpad, planes);
    KST_LAUNCH(ctx);
  }
  const int T = (int)(dpad / BM);
  const int tiles = T * (T + 1) / 2;
  const size_t smem = sizeof(double) * STAGES * STAGE_DOUBLES;
  static bool attr = false;
  if (!attr) {
    KST_CUDA(ctx, cudaFuncSetAttribute(gram_herm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    attr = true;
  }
  gram_herm_dmma<<<tiles, NT, smem, st>>>(planes, npad, dpad, n, d, T, S);
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace kst
