// K1: Hermitian sample-covariance Gram, FP64, for `sample_covariance`
// (src/lrkron.py:53-78):  S = (1/n) X^T conj(X),  X = (n, d) snapshots.
//
// Design:
//  * Only upper-triangle 64x64 tiles are computed; each tile writes itself
//    and its conjugate transpose, so S is exactly Hermitian (the reference
//    symmetrises with (S + S^H)/2, src/lrkron.py:77) and the diagonal is real.
//  * 3M complex product: with planes xr, xi, s = xr + xi, d = xr - xi,
//      Re = sum xr_a xr_b + xi_a xi_b,  Im = sum s_a d_b - xr_a xr_b + xi_a xi_b,
//    i.e. three real FP64 FMAs per complex MAC instead of four.
//  * Operand planes are produced once by gram_prep (zero-padded to the tile
//    grid so the main loop has no bounds checks) and streamed into a
//    3-stage cp.async shared-memory ring; 256 threads, 4x4 outputs each.
#include "common.cuh"

namespace {

constexpr int BM = 64;          // tile edge (rows == cols)
constexpr int BK = 8;           // snapshots per pipeline stage
constexpr int STAGES = 3;
constexpr int NT = 256;
constexpr int PLANE = BK * BM;  // doubles per plane per stage
constexpr int STAGE_DOUBLES = 6 * PLANE;  // A: xr, xi, s   B: xr, xi, d

// planes[4][npad][dpad]: xr, xi, xr+xi, xr-xi
__global__ void gram_prep(const cplx* __restrict__ X, int64_t n, int64_t d, int64_t npad,
                          int64_t dpad, double* __restrict__ planes) {
  const int64_t total = npad * dpad;
  const int64_t plane = total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx / dpad, a = idx - m * dpad;
    cplx v = cmk(0.0, 0.0);
    if (m < n && a < d) v = X[m * d + a];
    planes[idx] = v.x;
    planes[plane + idx] = v.y;
    planes[2 * plane + idx] = v.x + v.y;
    planes[3 * plane + idx] = v.x - v.y;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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

__global__ void __launch_bounds__(NT, 1)
gram_herm_3m(const double* __restrict__ planes, int64_t npad, int64_t dpad, int64_t n,
             int64_t d, int T, cplx* __restrict__ S) {
  extern __shared__ __align__(16) double smem[];
  int bi, bj;
  tile_of(blockIdx.x, T, bi, bj);
  const int a0 = bi * BM, b0 = bj * BM;
  const int64_t plane = npad * dpad;
  const double* gxr = planes;
  const double* gxi = planes + plane;
  const double* gs = planes + 2 * plane;
  const double* gd = planes + 3 * plane;

  const int tid = threadIdx.x;
  // loader mapping: each stage moves 6 planes x BK rows x 64 doubles = 1536
  // 16-byte chunks; thread handles chunks tid + 256*c, c < 6.
  auto load_stage = [&](int stage, int kb) {
    double* base = smem + stage * STAGE_DOUBLES;
    const int64_t m0 = (int64_t)kb * BK;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int chunk = tid + NT * c;      // 0..1535
      const int pl = chunk >> 8;           // 256 chunks per plane
      const int within = chunk & 255;
      const int row = within >> 5;         // 32 chunks per row (64 doubles)
      const int col = (within & 31) * 2;
      const double* src;
      int colbase;
      switch (pl) {
        case 0: src = gxr; colbase = a0; break;
        case 1: src = gxi; colbase = a0; break;
        case 2: src = gs; colbase = a0; break;
        case 3: src = gxr; colbase = b0; break;
        case 4: src = gxi; colbase = b0; break;
        default: src = gd; colbase = b0; break;
      }
      cp_async16(base + pl * PLANE + row * BM + col, src + (m0 + row) * dpad + colbase + col);
    }
  };

  const int w = tid >> 5, lane = tid & 31;
  const int r0 = (w >> 1) * 16 + (lane >> 3) * 4;  // 4 contiguous rows
  const int c0 = (w & 1) * 32 + (lane & 7) * 4;    // 4 contiguous cols

  double t1[4][4], t2[4][4], t3[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) t1[i][j] = t2[i][j] = t3[i][j] = 0.0;

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
    for (int k = 0; k < BK; ++k) {
      const double* ar = st + 0 * PLANE + k * BM + r0;
      const double* ai = st + 1 * PLANE + k * BM + r0;
      const double* as = st + 2 * PLANE + k * BM + r0;
      const double* br = st + 3 * PLANE + k * BM + c0;
      const double* bi_ = st + 4 * PLANE + k * BM + c0;
      const double* bd = st + 5 * PLANE + k * BM + c0;
      double xr[4], xi[4], xs[4], yr[4], yi[4], yd[4];
      *(double2*)&xr[0] = *(const double2*)&ar[0];
      *(double2*)&xr[2] = *(const double2*)&ar[2];
      *(double2*)&xi[0] = *(const double2*)&ai[0];
      *(double2*)&xi[2] = *(const double2*)&ai[2];
      *(double2*)&xs[0] = *(const double2*)&as[0];
      *(double2*)&xs[2] = *(const double2*)&as[2];
      *(double2*)&yr[0] = *(const double2*)&br[0];
      *(double2*)&yr[2] = *(const double2*)&br[2];
      *(double2*)&yi[0] = *(const double2*)&bi_[0];
      *(double2*)&yi[2] = *(const double2*)&bi_[2];
      *(double2*)&yd[0] = *(const double2*)&bd[0];
      *(double2*)&yd[2] = *(const double2*)&bd[2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          t1[i][j] = fma(xr[i], yr[j], t1[i][j]);
          t2[i][j] = fma(xi[i], yi[j], t2[i][j]);
          t3[i][j] = fma(xs[i], yd[j], t3[i][j]);
        }
    }
  }
  cp_async_wait<0>();

  const double dn = (double)n;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + r0 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = b0 + c0 + j;
      if (a >= d || b >= d) continue;
      const double re = (t1[i][j] + t2[i][j]) / dn;
      const double im = (t3[i][j] - t1[i][j] + t2[i][j]) / dn;
      if (bi != bj || a < b) {
        S[(int64_t)a * d + b] = cmk(re, im);
        S[(int64_t)b * d + a] = cmk(re, -im);
      } else if (a == b) {
        S[(int64_t)a * d + a] = cmk(re, 0.0);
      }
    }
  }
}

}  // namespace

namespace kst {

int scm(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, cudaStream_t st) {
  if (n < 1 || d < 1) return set_err(ctx, KST_ERR_DIMENSION, "scm: need n >= 1 and d >= 1");
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
    KST_CUDA(ctx, cudaFuncSetAttribute(gram_herm_3m, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    attr = true;
  }
  gram_herm_3m<<<tiles, NT, smem, st>>>(planes, npad, dpad, n, d, T, S);
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace kst
