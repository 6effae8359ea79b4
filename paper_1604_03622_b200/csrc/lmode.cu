// K7: the batched L-mode (windowed) estimator and detector -- BASELINE
// configs[3], SURVEY.md §8 "L-mode definition": for test bin m the training
// bins are [s, s + n_w), s = clamp(m - n_w // 2, 0, n_bins - n_w), and
//
//   est_m     = lr_kron_estimate(sample_covariance(X[s:s+n_w]), r_a, r_b)  (src/lrkron.py:53,118)
//   values[m] = detection_image(build_filter(kind, est_m), X[m:m+1], ...)  (src/filters.py:137,243)
//
// Nothing of size (pq)^2 or q^2 is formed per window. Everything follows from
// the banded snapshot Gram W_{m,m'} = X_m X_m'^H (P x P blocks, |m - m'| < n_w)
// and the row sums s_m = X_m 1_q:
//
//   ||S||_F^2 = (1/n^2) sum_{m,m'} |tr W_{mm'}|^2                      (A.4)
//   A0        = (1/(n q^2)) sum_m s_m s_m^H                              (A.1)
//   M = R R^H = (1/n^2) sum_{m,m'} W_{mm'} (x) conj(W_{mm'})   (P^2 x P^2; b/V steps, A.2/A.3)
//
// so every LR-Kron iteration runs on P^2-sized quantities (the same M-path
// iteration as the global estimate, lrkron_dev.cuh). The final b is
// b = U Omega U^H with U = [X_m^T conj(a_k)] (q x n_w r) from A_prev =
// sum_k lambda_k a_k a_k^H; its top-r_b eigenpairs come from the (n_w r)^2
// Hermitian H = Omega^1/2 Gamma Omega^1/2, Gamma_{(m,k),(m',k')} =
// a_k^H W_{mm'} a_k' (A.7), by block subspace iteration + Rayleigh-Ritz
// (Jacobi) in one CTA per window. The temporal basis v_j = U Omega^1/2
// conj(z_j) / sqrt(theta_j) is never materialised: a test bin's filtered
// spectrum is a P x (n_w P) matrix E_m applied to the spectra of its
// window's bins,
//
//   yhat_m = E_m [xhat_{s}; ...; xhat_{s+n_w-1}],  E_m = Q1 e_m - Q2 C_m Gamma_w^T
//
// (Q1/Q2 the spatial projector of the filter kind, C_m = X_m conj(V_B) from
// W, Gamma_w the spectral combination of v_j), followed by the spatial
// candidates and max|.| of detection_image.
//
// Kernels: band_gram_kernel (halo-reusing smem staging of the window rows),
// window_kernel (one CTA per window: record, iterations, eigensolves, E),
// lm_detect_kernel (smem-staged window spectra shared by consecutive test
// bins, the north_star "training-patch gather with halo reuse"). Spectra:
// kst::spectra (detect.cu). A window whose small eigensolve does not converge
// (or exceeds the batched limits) is recomputed by the per-window step path.
#include <algorithm>
#include <cstring>

#include "lrkron_dev.cuh"

namespace kst {
int lrkron(kst_ctx* ctx, const cplx* S, int p, int q, int ra, int rb, double tol, int max_iter,
           int validate, cplx* spatial, cplx* temporal, cplx* tb_vectors, double* tb_values,
           FitOut* fit, cplx* iter_spatial, cplx* iter_b, cudaStream_t st);
}

namespace {

#ifdef KST_LM_PROF
// phase clock stamps of every window (A/B builds only: -DKST_LM_PROF)
__device__ long long lm_prof[4096][16];
#define LM_STAMP(w, k) \
  do {                 \
    __syncthreads();   \
    if (threadIdx.x == 0 && (w) < 4096) lm_prof[w][k] = clock64(); \
  } while (0)
#else
#define LM_STAMP(w, k) \
  do {                 \
  } while (0)
#endif

constexpr int LM_NWMAX = 128;  // training window of the batched path
constexpr int LM_KBMAX = 3;    // temporal basis width of the batched path (r_b <= LM_S - 2)
// subspace block: the r_b <= 3 wanted pairs + 2 guard vectors (A/B on
// configs[3]: s = 5 converges in the same 2 rounds as s = 8 with eig(H) 173 ->
// 96 us per window; CGS and the Rayleigh-Ritz Jacobi scale with s^2). Larger
// r_b run on the per-window step path.
constexpr int LM_S = 5;
constexpr int LM_JAC = 16;     // n_w r <= this: dense Jacobi instead of subspace iteration
constexpr int LM_NBMAX = 256;  // n_w r limit (block vectors in smem)
constexpr int LM_MAXR = 24;    // Rayleigh-Ritz rounds before falling back
constexpr int LM_FALLBACK = 64;  // window status: redo on the step path

__host__ __device__ __forceinline__ int64_t win_start(int64_t m, int n_w, int64_t n_bins) {
  int64_t s = m - n_w / 2;
  s = s < 0 ? 0 : s;
  return s > n_bins - n_w ? n_bins - n_w : s;
}

// ---------------------------------------------------------------- band Gram
// W[m][o] = X_m X_{m+o}^H (P x P), o < n_w, and rs[m] = X_m 1_q, for the
// bins of the tile+halo cube. One CTA = tb consecutive bins m and every
// offset: the rows of bins [m0, m0 + tb + n_w - 1) are staged in smem in
// chunks of BG_TQ pulses (each bin row read once per CTA, not once per
// pair); thread = (m, group of KT offsets), its P x P x KT accumulators in
// registers.
// P = 3: 2 offsets per thread (36 accumulator doubles) and 2 CTAs per SM:
// the kernel is shared-memory-latency bound, so warps beat register reuse
// (A/B at Gotcha scale: KT 4 / 1 CTA 2.01 ms, KT 2 / 2 CTAs 1.39 ms, KT 1 /
// 3 CTAs 1.49 ms)
#ifndef KST_BG_KT3
#define KST_BG_KT3 2
#endif
#ifndef KST_BG_MINB
#define KST_BG_MINB 2
#endif
template <int P>
struct BG {
  static constexpr int KT = P <= 2 ? 8 : P == 3 ? KST_BG_KT3 : 2;
  static constexpr int MINB = P == 3 ? KST_BG_MINB : 1;
};
constexpr int BG_TQ = 16;
constexpr int BG_LD = BG_TQ + 1;  // padded smem row (bank spread)

// Split-K: blockIdx.y takes pulses [y qs, (y + 1) qs); with nsplit > 1 each
// split writes its own partial (W + y * wstride, rs + y * rstride) and
// band_reduce_kernel sums them in split order. nsplit and qs depend on q only
// (never on the tile), so a tile's W equals the full frame's bitwise.
template <int P>
__global__ void __launch_bounds__(NT, BG<P>::MINB) band_gram_kernel(const cplx* __restrict__ X, int nb, int q,
                                                       int n_w, int tb, int qs, int64_t wstride,
                                                       cplx* __restrict__ W, cplx* __restrict__ rs) {
  constexpr int KT = BG<P>::KT;
  extern __shared__ __align__(16) cplx xs[];  // [bin][channel][BG_LD]
  const int m0 = blockIdx.x * tb;
  const int qa = blockIdx.y * qs, qb = min(q, qa + qs);
  W += blockIdx.y * wstride;
  rs += blockIdx.y * (int64_t)nb * P;
  const int nrb = min(tb + n_w - 1, nb - m0);
  const int ngrp = (n_w + KT - 1) / KT;
  const int ml = threadIdx.x / ngrp, og = threadIdx.x % ngrp;
  const bool active = ml < tb && m0 + ml < nb;
  cplx acc[KT][P][P];
  cplx racc[P];
#pragma unroll
  for (int k = 0; k < KT; ++k)
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) acc[k][i][j] = cmk(0, 0);
#pragma unroll
  for (int i = 0; i < P; ++i) racc[i] = cmk(0, 0);
  for (int t0 = qa; t0 < qb; t0 += BG_TQ) {
    const int tl = min(BG_TQ, qb - t0);
    __syncthreads();  // previous chunk consumed
    for (int e = threadIdx.x; e < nrb * P * BG_TQ; e += NT) {
      const int r = e / BG_TQ, c = e - r * BG_TQ;
      if (c < tl)
        cp_async16(&xs[r * BG_LD + c], &X[((int64_t)m0 * P + r) * q + t0 + c]);
      else
        xs[r * BG_LD + c] = cmk(0, 0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (active) {
      for (int c = 0; c < tl; ++c) {
        cplx xm[P];
#pragma unroll
        for (int i = 0; i < P; ++i) xm[i] = xs[(ml * P + i) * BG_LD + c];
        if (og == 0)
#pragma unroll
          for (int i = 0; i < P; ++i) racc[i] = cadd(racc[i], xm[i]);
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const int o = og * KT + k;
          if (o < n_w && ml + o < nrb) {
            cplx xo[P];
#pragma unroll
            for (int j = 0; j < P; ++j) xo[j] = xs[((ml + o) * P + j) * BG_LD + c];
#pragma unroll
            for (int i = 0; i < P; ++i)
#pragma unroll
              for (int j = 0; j < P; ++j) cfmac(acc[k][i][j], xm[i], xo[j]);
          }
        }
      }
    }
  }
  if (!active) return;
  const int m = m0 + ml;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    const int o = og * KT + k;
    if (o < n_w && m + o < nb) {
      cplx* w = W + ((int64_t)m * n_w + o) * P * P;
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) w[i * P + j] = acc[k][i][j];
    }
  }
  if (og == 0)
#pragma unroll
    for (int i = 0; i < P; ++i) rs[(int64_t)m * P + i] = racc[i];
}

// W = sum over splits in split order (and the row sums)
__global__ void band_reduce_kernel(const cplx* __restrict__ Wp, int nsplit, int64_t wcount,
                                   int64_t wstride, int64_t rcount, cplx* __restrict__ W,
                                   cplx* __restrict__ rs) {
  const cplx* rsp = Wp + nsplit * wstride;  // partial row sums follow the W partials
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < wcount + rcount;
       e += (int64_t)gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    if (e < wcount) {
      for (int k = 0; k < nsplit; ++k) acc = cadd(acc, Wp[k * wstride + e]);
      W[e] = acc;
    } else {
      const int64_t r = e - wcount;
      for (int k = 0; k < nsplit; ++k) acc = cadd(acc, rsp[k * rcount + r]);
      rs[r] = acc;
    }
  }
}

// Band-prefix record rows: for bin m and length L = 1..n_w,
//   Qp[m][slot][L-1] = sum_{o < L} g(m, o)[slot],  g(m, o) = the record
//   contribution of the pair (m, m + o): [(o ? 2 : 1) |tr B|^2, #non-finite
//   entries of B, M upper triangle re/im: B[i,k] conj(B[j,l]) (+ conj(B[k,i])
//   B[l,j] for o > 0)] with B = W_{m, m+o}. A window [s, s + n_w) owns exactly
//   the pairs (s + ml, s + ml + o), o < n_w - ml, so its record is the sum of
//   the n_w entries Qp[s + ml][.][n_w - ml - 1] -- n_w reads instead of
//   n_w (n_w + 1) / 2 pair products per window (consecutive windows share all
//   but 2 n_w - 1 pairs). Warp per (bin, record item): lanes take offsets
//   o = 32 c + lane, warp inclusive scan per 32-offset chunk plus the running
//   carry (fixed shuffle tree: deterministic, tile-independent).
template <int P>
__global__ void __launch_bounds__(256) band_prefix_kernel(const cplx* __restrict__ W, int nb, int n_w,
                                                          double* __restrict__ Qp) {
  constexpr int U = P * P, E = U * (U + 1) / 2, NQ = 2 + 2 * E, NI = 2 + E;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= (int64_t)nb * NI) return;
  const int m = (int)(wid / NI), it = (int)(wid - (int64_t)m * NI);
  const cplx* wm = W + (int64_t)m * n_w * U;
  int i = 0, j = 0, k = 0, l = 0;
  if (it >= 2) {  // upper-triangle entry it - 2 -> (u, x), u <= x
    int u = 0, rem = it - 2;
    while (rem >= U - u) {
      rem -= U - u;
      ++u;
    }
    const int x = u + rem;
    i = u / P, j = u % P, k = x / P, l = x % P;
  }
  const int ns = it < 2 ? 1 : 2;  // output slots of this item
  double* out0 = Qp + ((int64_t)m * NQ + (it < 2 ? it : 2 + 2 * (it - 2))) * n_w;
  double carry0 = 0.0, carry1 = 0.0;
  for (int c0 = 0; c0 < n_w; c0 += 32) {
    const int o = c0 + lane;
    double v0 = 0.0, v1 = 0.0;
    if (o < n_w && m + o < nb) {
      const cplx* B = wm + (int64_t)o * U;
      if (it == 0) {
        cplx tr = cmk(0, 0);
#pragma unroll
        for (int ii = 0; ii < P; ++ii) tr = cadd(tr, B[ii * P + ii]);
        v0 = (o ? 2.0 : 1.0) * cabs2(tr);
      } else if (it == 1) {
#pragma unroll
        for (int kk = 0; kk < U; ++kk) v0 += (isfinite(B[kk].x) && isfinite(B[kk].y)) ? 0.0 : 1.0;
      } else {
        cplx t = cmulc(B[i * P + k], B[j * P + l]);
        if (o) t = cadd(t, cmulc(B[l * P + j], B[k * P + i]));
        v0 = t.x;
        v1 = t.y;
      }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // inclusive warp scan
      const double a0 = __shfl_up_sync(0xffffffffu, v0, d);
      const double a1 = __shfl_up_sync(0xffffffffu, v1, d);
      if (lane >= d) {
        v0 += a0;
        v1 += a1;
      }
    }
    v0 += carry0;
    v1 += carry1;
    if (o < n_w) {
      out0[o] = v0;
      if (ns == 2) out0[n_w + o] = v1;
    }
    carry0 = __shfl_sync(0xffffffffu, v0, 31);
    carry1 = __shfl_sync(0xffffffffu, v1, 31);
  }
}

// W_{mA,mB}[i][j] from the band (mA, mB bin indices of the tile cube)
template <int P>
__device__ __forceinline__ cplx wget(const cplx* __restrict__ W, int n_w, int mA, int mB, int i,
                                     int j) {
  return mA <= mB ? W[((int64_t)mA * n_w + (mB - mA)) * P * P + i * P + j]
                  : cconj(W[((int64_t)mB * n_w + (mA - mB)) * P * P + j * P + i]);
}

// ---------------------------------------------------------------- window kernel
struct WinArgs {
  int64_t a, n_bins, lo, hi;  // tile cube starts at bin a; test bins [lo, hi)
  int64_t s0;                 // first window (absolute)
  int nwin, n_w, q, ra, rb, max_iter, kind, spatial_only, nslot, nbmax;
  double tol;
};

// fixed-order block reduction of NV values per thread (warp shuffles, then
// warps in index order); result in out[0..NV) (smem), all threads see it
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* scratch, double* out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double x = warp_sum(v[k]);
    if (l == 0) scratch[w * NV + k] = x;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NV; k += NT) {
    double s = 0.0;
    for (int ww = 0; ww < NT / 32; ++ww) s += scratch[ww * NV + k];
    out[k] = s;
  }
  __syncthreads();
}

// Y (nb x LM_S, smem, row-major) <- H Y  with H (nb x nb, global, row-major);
// thread = row
__device__ __forceinline__ void hmul(const cplx* __restrict__ H, int nb, const cplx* Y, cplx* Z,
                                     int s) {
  for (int r = threadIdx.x; r < nb; r += NT) {
    cplx acc[LM_S];
#pragma unroll
    for (int k = 0; k < LM_S; ++k) acc[k] = cmk(0, 0);
    const cplx* h = H + (int64_t)r * nb;
    for (int c = 0; c < nb; ++c) {
      const cplx hv = h[c];
#pragma unroll
      for (int k = 0; k < LM_S; ++k)
        if (k < s) cfma(acc[k], hv, Y[c * LM_S + k]);
    }
#pragma unroll
    for (int k = 0; k < LM_S; ++k)
      if (k < s) Z[r * LM_S + k] = acc[k];
  }
  __syncthreads();
}

// G = A^H B (s x s, full) of two nb x s blocks (smem): warp j forms row j of
// G (lanes stride the nb rows, fixed shuffle tree: deterministic)
__device__ __forceinline__ void block_gram(const cplx* A, const cplx* B, int nb, int s, cplx* G) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int jr = wid; jr < s; jr += NT / 32) {
    cplx acc[LM_S];
#pragma unroll
    for (int k = 0; k < LM_S; ++k) acc[k] = cmk(0, 0);
    for (int r = lane; r < nb; r += 32) {
      const cplx x = A[r * LM_S + jr];
#pragma unroll
      for (int k = 0; k < LM_S; ++k)
        if (k < s) cfmca(acc[k], x, B[r * LM_S + k]);  // conj(x) y
    }
#pragma unroll
    for (int k = 0; k < LM_S; ++k) {
      const double re = warp_sum(acc[k].x), im = warp_sum(acc[k].y);
      if (lane == 0 && k < s) G[jr * LM_S + k] = cmk(re, im);
    }
  }
  __syncthreads();
}

// Orthonormalise the nb x s block Y in place by classical Gram-Schmidt with
// selective reorthogonalisation (a second pass when the first cancelled more
// than half of the norm -- "twice is enough"), column by column: stable for
// the very ill-conditioned blocks a dominant mover produces after one H step (where
// Cholesky-QR, which squares the condition number, breaks down). A column
// that vanishes after projection (relative 1e-13) is replaced by the next
// unused unit vector and re-projected. Warp j forms coefficient j (lanes
// stride the rows, fixed shuffle tree: deterministic).
__device__ void cgs2(cplx* Y, int nb, int s, cplx* coef, double* nrm, int* next_unit) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // y_k -= sum_{j<k} <y_j, y_k> y_j: warps j < k form the coefficients (warp
  // NT/32 - 1 meanwhile |y_k|^2 into nrm[0] when want_n0), then every row
  // updates; ends with |y_k|^2 in nrm[1] visible to all
  auto project = [&](int k, bool want_n0) {
    if (wid < k) {
      cplx acc = cmk(0, 0);
      for (int r = lane; r < nb; r += 32) cfmca(acc, Y[r * LM_S + wid], Y[r * LM_S + k]);
      acc.x = warp_sum(acc.x);
      acc.y = warp_sum(acc.y);
      if (lane == 0) coef[wid] = acc;
    } else if (want_n0 && wid == NT / 32 - 1) {
      double a = 0.0;
      for (int r = lane; r < nb; r += 32) a += cabs2(Y[r * LM_S + k]);
      a = warp_sum(a);
      if (lane == 0) nrm[0] = a;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nb; r += NT) {
      cplx y = Y[r * LM_S + k];
      for (int j2 = 0; j2 < k; ++j2) y = csub(y, cmul(Y[r * LM_S + j2], coef[j2]));
      Y[r * LM_S + k] = y;
    }
    __syncthreads();
    if (wid == 0) {
      double a = 0.0;
      for (int r = lane; r < nb; r += 32) a += cabs2(Y[r * LM_S + k]);
      a = warp_sum(a);
      if (lane == 0) nrm[1] = a;
    }
    __syncthreads();
  };
  for (int k = 0; k < s; ++k) {
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (k == 0) {
        if (wid == 0) {
          double a = 0.0;
          for (int r = lane; r < nb; r += 32) a += cabs2(Y[r * LM_S + k]);
          a = warp_sum(a);
          if (lane == 0) nrm[0] = nrm[1] = a;
        }
        __syncthreads();
      } else {
        project(k, true);
        // "twice is enough" (Kahan-Parlett): reorthogonalise only when the
        // projection cancelled more than half of the norm
        if (nrm[1] <= 0.25 * nrm[0]) project(k, false);  // nrm[0] keeps |y_k|^2 before
      }
      const bool ok = nrm[1] > 1e-26 * nrm[0] && nrm[1] > 0.0;
      if (ok || attempt == 1) break;
      // dependent column: restart it as the next unit vector
      __syncthreads();
      const int u = *next_unit % nb;
      for (int r = threadIdx.x; r < nb; r += NT) Y[r * LM_S + k] = cmk(r == u ? 1.0 : 0.0, 0.0);
      __syncthreads();
      if (threadIdx.x == 0) *next_unit = u + 1;
    }
    const double inv = nrm[1] > 0.0 ? 1.0 / sqrt(nrm[1]) : 0.0;
    for (int r = threadIdx.x; r < nb; r += NT) Y[r * LM_S + k] = cscale(Y[r * LM_S + k], inv);
    __syncthreads();
  }
}

// Y <- Y Q (nb x s times s x s, Q taken as column `order[k]` of the Jacobi V)
__device__ __forceinline__ void rotate_block(cplx* Y, int nb, int s, const JacSmem& j) {
  for (int r = threadIdx.x; r < nb; r += NT) {
    cplx y[LM_S], o[LM_S];
#pragma unroll
    for (int k = 0; k < LM_S; ++k) y[k] = k < s ? Y[r * LM_S + k] : cmk(0, 0);
#pragma unroll
    for (int k = 0; k < LM_S; ++k) {
      o[k] = cmk(0, 0);
      if (k < s) {
        const int c = j.order[k];
#pragma unroll
        for (int i = 0; i < LM_S; ++i)
          if (i < s) cfma(o[k], y[i], j.V[i * j.ld + c]);
      }
    }
#pragma unroll
    for (int k = 0; k < LM_S; ++k)
      if (k < s) Y[r * LM_S + k] = o[k];
  }
  __syncthreads();
}

// info per window (ints): status, iterations, converged, ka, kb, eig rounds, r, nb
constexpr int WI = 8;

#ifndef KST_WIN_MINB
#define KST_WIN_MINB 2
#endif
template <int P>
__global__ void __launch_bounds__(NT, KST_WIN_MINB) window_kernel(const cplx* __restrict__ W,
                                                       const cplx* __restrict__ rs,
                                                       const double* __restrict__ Qp, WinArgs g,
                                                       cplx* __restrict__ Hscr,
                                                       double* __restrict__ resid_scr,
                                                       cplx* __restrict__ Eout,
                                                       int* __restrict__ info_out,
                                                       double* __restrict__ res_out) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E, NREC = 1 + 2 * E;
  constexpr int NPW = P * P;
  extern __shared__ __align__(16) char dyn[];
  // dynamic smem: [jacobi scratch | reduction scratch | Y (nbmax x LM_S) | Z]
  char* jsm = dyn;
  const size_t jbytes = (kstj::jac_smem_bytes(LM_JAC) + 15) / 16 * 16;
  double* scratch = (double*)(dyn + jbytes);  // 256 doubles
  cplx* Y = (cplx*)(scratch + 256);
  cplx* Z = Y + (size_t)g.nbmax * LM_S;
  cplx* gam = Z + (size_t)g.nbmax * LM_S;  // n_w P x LM_KBMAX
  cplx* cmall = gam + (size_t)g.n_w * P * LM_KBMAX;  // (n_w / 2 + 1) x P x LM_KBMAX
  __shared__ double red[4 + 2 * U + 2 * E];
  __shared__ double recv[NREC + 1];
  __shared__ double a0s[2 * U];
  __shared__ IterState st;
  __shared__ cplx spatial[kMaxP * kMaxP];
  __shared__ double dinfo[4], hdiag[8];
  __shared__ cplx ua[P * P], av[P * P], Q1[P * P], Q2[P * P];
  __shared__ double lamv[P], omega[P], theta[LM_S];
  __shared__ cplx G8[LM_S * LM_S];
  __shared__ int ka_s, r_s, kb_s, flag_s, status_s, rounds_s, mode_s, spat_s, kk_s;
  __shared__ int sel[LM_S];
  __shared__ double nrm2[2];
  __shared__ cplx coefs[LM_S];
  __shared__ int unit_s;
  const int tid = threadIdx.x;
  const int n_w = g.n_w;
  const double nn = (double)n_w;
  for (int w = blockIdx.x; w < g.nwin; w += gridDim.x) {
    const int64_t s_abs = g.s0 + w;
    const int s = (int)(s_abs - g.a);  // window's first bin in the tile cube
    LM_STAMP(w, 0);
    // ---------------------------------------------------------- (1) record
    // the window's pairs (m, m'), m <= m' in [s, s + n_w): for each of its
    // bins m = s + ml the offsets o < n_w - ml, i.e. the band-prefix entry
    // Qp[m][slot][n_w - ml - 1] (band_prefix_kernel); warp = record slot,
    // lanes over the bins, fixed warp_sum tree (deterministic, tile-independent)
    {
      constexpr int NQ = 2 + 2 * E;
      const int wid = tid >> 5, lane = tid & 31;
      // warp per 4 slots (12 independent loads in flight per lane), lanes over the bins
      for (int k0 = 4 * wid; k0 < NQ; k0 += 4 * (NT / 32)) {
        double x[4] = {0.0, 0.0, 0.0, 0.0};
        for (int ml = lane; ml < n_w; ml += 32) {
          const double* qb = Qp + (int64_t)(s + ml) * NQ * n_w + (n_w - 1 - ml);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (k0 + c < NQ) x[c] += qb[(int64_t)(k0 + c) * n_w];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double t = warp_sum(x[c]);
          if (lane == 0 && k0 + c < NQ) recv[k0 + c] = t;
        }
      }
      // A0 block sums (1/n) sum_m s_m[i] conj(s_m[j]): warp per block entry
      for (int u = wid; u < U; u += NT / 32) {
        const int i = u / P, j = u % P;
        cplx acc = cmk(0, 0);
        for (int ml = lane; ml < n_w; ml += 32)
          cfmac(acc, rs[(int64_t)(s + ml) * P + i], rs[(int64_t)(s + ml) * P + j]);
        acc.x = warp_sum(acc.x);
        acc.y = warp_sum(acc.y);
        if (lane == 0) {
          a0s[2 * u] = acc.x;
          a0s[2 * u + 1] = acc.y;
        }
      }
      __syncthreads();
      const double inv_n2 = 1.0 / (nn * nn);
      for (int k = tid; k < 4 + 2 * U + 2 * E; k += NT) {
        double x;
        if (k == 0) x = recv[0] * inv_n2;
        else if (k == 1) x = recv[1] != 0.0 ? 1.0 : 0.0;  // non-finite window data
        else if (k == 2) x = 0.0;  // window S diagonal = (1/n) sum |x|^2 >= 0
        else if (k == 3) x = 1.0;
        else if (k < 4 + 2 * U) {
          x = a0s[k - 4] / nn;  // A0 block sums (re at even, im at odd)
        } else {
          x = recv[2 + (k - 4 - 2 * U)] * inv_n2;
        }
        red[k] = x;
      }
      __syncthreads();
    }
    LM_STAMP(w, 1);
    // ---------------------------------------------------------- (2) LR-Kron iterations
    double* resid = resid_scr + (size_t)blockIdx.x * (g.max_iter + 1);
    m_iterations<P>(red, g.q, g.ra, g.tol, g.max_iter, &st, jsm, spatial, resid, dinfo, hdiag);
    __syncthreads();
    if (tid == 0) {
      int status = (int)dinfo[0];
      if (red[1] > 0.0) status = 200;  // non-finite window data
      else if (status == 4) status = KST_ERR_DEGENERATE + 100;  // spatial collapse (own message)
      status_s = status;
      ka_s = 0;
      kb_s = 0;
      r_s = 0;
      rounds_s = 0;
      kk_s = 0;
    }
    __syncthreads();
    const int iters = (int)dinfo[1], conv = (int)dinfo[2];
    const bool zero_s = red[0] == 0.0 && red[1] == 0.0;
    int* inf = info_out + (size_t)w * WI;
    if (status_s != 0) {
      if (tid == 0) {
        inf[0] = status_s;
        inf[1] = iters;
        inf[2] = conv;
      }
      continue;
    }
    LM_STAMP(w, 2);
    // ---------------------------------------------------------- (3) U_A = subspace_basis(A)
    if (!zero_s) {
      JacSmem j = jac_carve(jsm, P);
      jac_solve(j, spatial, P, P, 1.0);
      if (tid == 0) {
        int keep = 0;
        const double top = j.val[j.order[0]];
        if (top > 0.0) {
          for (int k = 0; k < P; ++k) keep += j.val[k] > 1e-9 * top;
          keep = min(keep, g.ra);
        }
        ka_s = keep;
      }
      __syncthreads();
      for (int e = tid; e < P * P; e += NT) {
        const int i = e / P, k = e % P;
        ua[e] = k < ka_s ? j.V[i * j.ld + j.order[k]] : cmk(0, 0);  // ua[i*P + k]
      }
      __syncthreads();
      // ------------------------------------------------------ (4) A_prev = sum lambda_k a_k a_k^H
      for (int e = tid; e < P * P; e += NT) spatial[e] = cconj(st.Aconj[e]);
      __syncthreads();
      jac_solve(j, spatial, P, P, 1.0);
      if (tid == 0) {
        double mx = 0.0;
        for (int k = 0; k < P; ++k) mx = fmax(mx, fabs(j.val[k]));
        int r = 0;
        for (int k = 0; k < P; ++k) {
          const double lam = j.val[j.order[k]];
          if (lam > 1e-13 * mx) {
            lamv[r] = lam;
            omega[r] = lam / (nn * st.na2);
            ++r;
          }
        }
        r_s = r;
      }
      __syncthreads();
      for (int e = tid; e < P * P; e += NT) {
        const int i = e / P, k = e % P;
        av[e] = k < r_s ? j.V[i * j.ld + j.order[k]] : cmk(0, 0);  // av[i*P + k] = a_k[i]
      }
      __syncthreads();
    }
    const int r = r_s, nb = n_w * r;
    if (!zero_s && (nb > g.nbmax || nb < 1)) {
      if (tid == 0) {
        inf[0] = LM_FALLBACK;
        inf[1] = iters;
        inf[2] = conv;
        inf[3] = 1;  // reason: n_w r outside the batched limit
        inf[6] = r;
        inf[7] = nb;
      }
      continue;
    }
    LM_STAMP(w, 3);
    // ---------------------------------------------------------- (5) H and its top pairs
    const int kk = zero_s ? 0 : min(g.rb, nb);
    cplx* H = Hscr + (size_t)blockIdx.x * g.nbmax * g.nbmax;
    if (!zero_s) {
      // upper block pairs (m1 = ml, m2 = ml + o) of the band, each W block read
      // once: H[(m1,k1),(m2,k2)] = sqrt(om_k1 om_k2) a_k1^H W_{m1 m2} a_k2 and the
      // mirror H[(m2,k2),(m1,k1)] = conj (H Hermitian by construction)
      for (int e = tid; e < n_w * n_w; e += NT) {
        const int ml = e / n_w, o = e - ml * n_w;
        if (o >= n_w - ml) continue;
        const cplx* bp = W + ((int64_t)(s + ml) * n_w + o) * NPW;
        cplx B[NPW];
#pragma unroll
        for (int k = 0; k < NPW; ++k) B[k] = bp[k];
        for (int k2 = 0; k2 < r; ++k2) {
          cplx wa[P];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            wa[i] = cmk(0, 0);
#pragma unroll
            for (int jj = 0; jj < P; ++jj) cfma(wa[i], B[i * P + jj], av[jj * P + k2]);
          }
          for (int k1 = 0; k1 < r; ++k1) {
            cplx acc = cmk(0, 0);
#pragma unroll
            for (int i = 0; i < P; ++i) cfmca(acc, av[i * P + k1], wa[i]);
            const cplx h = cscale(acc, sqrt(omega[k1] * omega[k2]));
            const int row = ml * r + k1, col = (ml + o) * r + k2;
            H[(int64_t)row * nb + col] = h;
            if (o) H[(int64_t)col * nb + row] = cconj(h);
          }
        }
      }
      __syncthreads();
      LM_STAMP(w, 4);
      if (nb <= LM_JAC) {
        JacSmem j = jac_carve(jsm, nb);
        jac_solve(j, H, nb, nb, 1.0);
        for (int e = tid; e < nb * LM_S; e += NT) {
          const int row = e / LM_S, k = e % LM_S;
          Y[e] = k < kk ? j.V[row * j.ld + j.order[k]] : cmk(0, 0);
        }
        if (tid < kk) theta[tid] = j.val[j.order[tid]];
        __syncthreads();
      } else {
        const int sb = min(LM_S, nb);
        // start block: unit vectors at the sb largest diagonal entries (ties:
        // lower index); warp 0, lane l holds rows l + 32 i (nb <= LM_NBMAX),
        // sb rounds of a warp argmax
        if (tid < 32) {
          constexpr int RPL = LM_NBMAX / 32;
          double dv[RPL];
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int row = tid + 32 * i;
            dv[i] = row < nb ? H[(int64_t)row * nb + row].x : -INFINITY;
          }
          for (int k = 0; k < sb; ++k) {
            double bv = -INFINITY;
            int bi = nb;
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              if (dv[i] > bv) {
                bv = dv[i];
                bi = tid + 32 * i;
              }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
              if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
              }
            }
            if (tid == 0) sel[k] = bi;
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              if (tid + 32 * i == bi) dv[i] = -INFINITY;
          }
        }
        __syncthreads();
        for (int e = tid; e < nb * LM_S; e += NT) {
          const int row = e / LM_S, k = e % LM_S;
          Y[e] = cmk((k < sb && sel[k] == row) ? 1.0 : 0.0, 0.0);
        }
        if (tid == 0) unit_s = 0;
        __syncthreads();
        LM_STAMP(w, 14);
        bool done = false;
        int round = 0;
        double prev_worst = 1e300;
        int stall = 0;
        for (; round < LM_MAXR && !done; ++round) {
          // two power steps, each followed by CGS2 orthonormalisation
          LM_STAMP(w, 8);
          hmul(H, nb, Y, Z, sb);
          LM_STAMP(w, 9);
          cgs2(Z, nb, sb, coefs, nrm2, &unit_s);
          LM_STAMP(w, 10);
          hmul(H, nb, Z, Y, sb);
          cgs2(Y, nb, sb, coefs, nrm2, &unit_s);
          if (round < 1) continue;  // H^4 warm-up before the first Rayleigh-Ritz
          LM_STAMP(w, 11);
          hmul(H, nb, Y, Z, sb);
          block_gram(Y, Z, nb, sb, G8);  // T = Y^H H Y
          LM_STAMP(w, 12);
          JacSmem j = jac_carve(jsm, sb);
          jac_solve(j, G8, LM_S, sb, 1.0);
          LM_STAMP(w, 13);
          rotate_block(Y, nb, sb, j);
          rotate_block(Z, nb, sb, j);
          if (tid < sb) theta[tid] = j.val[j.order[tid]];
          __syncthreads();
          // residuals |H y_k - theta_k y_k| for the wanted pairs
          double v[LM_S];
#pragma unroll
          for (int k = 0; k < LM_S; ++k) v[k] = 0.0;
          for (int row = tid; row < nb; row += NT)
#pragma unroll
            for (int k = 0; k < LM_S; ++k)
              if (k < kk) v[k] += cabs2(csub(Z[row * LM_S + k], cscale(Y[row * LM_S + k], theta[k])));
          double* out = scratch + (NT / 32) * LM_S;
          block_reduce<LM_S>(v, scratch, out);
          if (tid == 0) {
            double tmax = 0.0, worst = 0.0;
            for (int k = 0; k < sb; ++k) tmax = fmax(tmax, fabs(theta[k]));
            bool all_ok = true;
            for (int k = 0; k < kk; ++k) {
              const double res = sqrt(out[k]);
              worst = fmax(worst, res);
              double gap = 1e300;
              for (int k2 = 0; k2 < sb; ++k2)
                if (k2 != k) gap = fmin(gap, fabs(theta[k] - theta[k2]));
              all_ok = all_ok && (res <= 1e-12 * tmax || (res <= 1e-9 * tmax && res <= 1e-8 * gap));
            }
            int ok = (tmax == 0.0 || all_ok) ? 1 : 0;
            if (!ok && worst <= 1e-9 * tmax) {
              stall = (worst > 0.5 * prev_worst) ? stall + 1 : 0;
              if (stall >= 3) ok = 1;
            }
            prev_worst = worst;
            flag_s = ok;
          }
          __syncthreads();
          done = flag_s != 0;
        }
        __syncthreads();
        if (!done) {
          if (tid == 0) {
            inf[0] = LM_FALLBACK;
            inf[1] = iters;
            inf[2] = conv;
            inf[3] = rounds_s < 0 ? 2 : 3;  // reason: Cholesky-QR breakdown / no convergence
            inf[5] = rounds_s < 0 ? -rounds_s - 1 : round;
            inf[6] = r;
            inf[7] = nb;
          }
          continue;
        }
        if (tid == 0) rounds_s = round;
      }
      // ------------------------------------------------------ (6) kept temporal rank
      if (tid == 0) {
        double top = 0.0;
        for (int k = 0; k < kk; ++k) top = fmax(top, fabs(theta[k]));
        for (int k = 0; k < kk; ++k)
          if (theta[k] < 0 && fabs(theta[k]) <= 1e-10 * top) theta[k] = 0.0;  // eig_truncate clamp
        int keep = 0;
        if (kk > 0 && theta[0] > 0.0) {
          for (int k = 0; k < kk; ++k) keep += theta[k] > 1e-9 * theta[0];
          keep = min(keep, g.rb);
        }
        kb_s = keep;
        kk_s = kk;
      }
      __syncthreads();
    }
    LM_STAMP(w, 5);
    // ---------------------------------------------------------- (7) filter kind -> Q1, Q2
    if (tid == 0) {
      const bool has_a = ka_s > 0, has_b = kb_s > 0;
      int mode = 2, spatial_f = 0;  // mode 0: temporal (kron), 1: classical, 2: none
      if (g.kind == KST_KIND_KRON) {
        mode = (has_b && !g.spatial_only) ? 0 : 2;
        spatial_f = has_a ? 1 : 0;
      } else if (has_a) {
        if (g.spatial_only) spatial_f = 1;
        else if (has_b) mode = 1;
      }
      mode_s = mode;
      spat_s = spatial_f;
    }
    __syncthreads();
    for (int e = tid; e < P * P; e += NT) {
      const int i = e / P, l = e % P;
      cplx uu = cmk(0, 0);  // (U_A U_A^H)[i, l]
      for (int k = 0; k < ka_s; ++k) cfmac(uu, ua[i * P + k], ua[l * P + k]);
      const cplx id = cmk(i == l ? 1.0 : 0.0, 0.0);
      const cplx pa = spat_s ? csub(id, uu) : id;
      Q1[e] = mode_s == 1 ? id : pa;
      Q2[e] = mode_s == 1 ? uu : pa;
    }
    __syncthreads();
    const int kb = mode_s == 2 ? 0 : kb_s;
    // gamma[(m', l), j] = sum_k' alpha[(m'k'), j] conj(a_k'[l]),
    // alpha[(m'k'), j] = sqrt(omega_k') conj(z_j[m' r + k']) / sqrt(theta_j)   (in Z)
    if (kb > 0) {
      for (int e = tid; e < n_w * P * kb; e += NT) {
        const int row = e / kb, jj = e - row * kb, m2 = row / P, l = row - m2 * P;
        const double it = 1.0 / sqrt(theta[jj]);
        cplx acc = cmk(0, 0);
        for (int k2 = 0; k2 < r; ++k2) {
          const cplx al = cscale(cconj(Y[(m2 * r + k2) * LM_S + jj]), sqrt(omega[k2]) * it);
          cfmac(acc, al, av[l * P + k2]);
        }
        gam[row * LM_KBMAX + jj] = acc;
      }
      __syncthreads();
    }
    LM_STAMP(w, 6);
    // ---------------------------------------------------------- (8) E for the window's test bins
    const int h = n_w / 2;
    int64_t t0 = (s_abs == 0) ? 0 : s_abs + h;
    int64_t t1 = (s_abs == g.n_bins - n_w) ? g.n_bins : s_abs + h + 1;
    t0 = max(t0, g.lo);
    t1 = min(t1, g.hi);
    const int nwp = n_w * P;
    // test bins of this window: <= n_w / 2 + 1, except a lone window
    // (n_w = n_bins) that owns every bin -- C_t is staged CH bins at a time
    const int CH = n_w / 2 + 1;
    for (int64_t c0 = t0; c0 < t1; c0 += CH) {
      const int64_t c1 = min(t1, c0 + CH);
      const int ntw = (int)(c1 - c0);
      if (kb > 0 && ntw > 0) {
        // C_t[i, j] = sum_{m'k'} conj(alpha[(m'k'), j]) (W_{ml m'} a_k')[i], all test bins:
        // warp per test bin, lanes stride the n_w r window columns; each lane
        // reads its W block once for all (i, j) (P x kb accumulators); per
        // (i, j) the same lane order and warp_sum tree as a per-output warp
        const int wid = tid >> 5, lane = tid & 31;
        for (int tb = wid; tb < ntw; tb += NT / 32) {
          const int ml = (int)(c0 + tb - s_abs);
          cplx acc[P][LM_KBMAX];
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int jj = 0; jj < LM_KBMAX; ++jj) acc[i][jj] = cmk(0, 0);
          for (int c = lane; c < nb; c += 32) {
            const int m2 = c / r, k2 = c - m2 * r;
            cplx wa[P];
#pragma unroll
            for (int i = 0; i < P; ++i) {
              wa[i] = cmk(0, 0);
#pragma unroll
              for (int l = 0; l < P; ++l)
                cfma(wa[i], wget<P>(W, n_w, s + ml, s + m2, i, l), av[l * P + k2]);
            }
            const double so = sqrt(omega[k2]);
#pragma unroll
            for (int jj = 0; jj < LM_KBMAX; ++jj) {
              if (jj >= kb) break;
              const cplx alc = cscale(Y[c * LM_S + jj], so * (1.0 / sqrt(theta[jj])));  // conj(alpha)
#pragma unroll
              for (int i = 0; i < P; ++i) cfma(acc[i][jj], alc, wa[i]);
            }
          }
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int jj = 0; jj < LM_KBMAX; ++jj) {
              if (jj >= kb) break;
              const double ax = warp_sum(acc[i][jj].x), ay = warp_sum(acc[i][jj].y);
              if (lane == 0) cmall[(tb * P + i) * LM_KBMAX + jj] = cmk(ax, ay);
            }
        }
        __syncthreads();
      }
      // E_t[i, (m', l)] = Q1[i, l] [m' = ml] - sum_i2 Q2[i, i2] sum_j C_t[i2, j] gamma[(m' l), j]
      // thread = window column (m', l) with its gamma row in registers, all
      // (test bin, channel) rows; stores coalesced over the columns
      for (int col = tid; col < nwp; col += NT) {
        const int m2 = col / P, l = col - m2 * P;
        cplx gv[LM_KBMAX];
#pragma unroll
        for (int jj = 0; jj < LM_KBMAX; ++jj) gv[jj] = jj < kb ? gam[col * LM_KBMAX + jj] : cmk(0, 0);
        for (int row = 0; row < ntw * P; ++row) {
          const int tb = row / P, i = row - tb * P;
          const int ml = (int)(c0 + tb - s_abs);
          cplx x = m2 == ml ? Q1[i * P + l] : cmk(0, 0);
          if (kb > 0) {
            cplx dl = cmk(0, 0);
            for (int i2 = 0; i2 < P; ++i2) {
              cplx cg = cmk(0, 0);
#pragma unroll
              for (int jj = 0; jj < LM_KBMAX; ++jj)
                if (jj < kb) cfma(cg, cmall[(tb * P + i2) * LM_KBMAX + jj], gv[jj]);
              cfma(dl, Q2[i * P + i2], cg);
            }
            x = csub(x, dl);
          }
          Eout[(size_t)(c0 + tb - g.lo) * P * nwp + (size_t)i * nwp + col] = x;
        }
      }
      __syncthreads();
    }
    LM_STAMP(w, 7);
    if (tid == 0) {
      inf[0] = 0;
      inf[1] = zero_s ? 0 : iters;
      inf[2] = zero_s ? 1 : conv;
      inf[3] = ka_s;
      inf[4] = kb_s;
      inf[5] = rounds_s;
      inf[6] = r;
      inf[7] = nb;
      res_out[w] = zero_s ? 0.0 : (iters > 0 ? resid[iters - 1] : 0.0);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- detection
// Test bins [t0, t0 + DT_TB) per CTA: their E rows stay in smem; the spectra
// of the union of their windows (<= DT_TB + n_w - 1 bins: consecutive test
// bins share n_w - 1 training bins) are staged chunk by chunk of DT_TD
// Doppler bins; yhat = E xhat per (bin, channel, Doppler), then the spatial
// candidates and max|.| (src/filters.py:269-272).
constexpr int DT_TB = 4;
constexpr int DT_TD = 16;
constexpr int DT_LD = DT_TD + 1;

struct DetArgs {
  int64_t a, n_bins, lo, hi;
  int n_w, D, G;
  double inv_sqrt_q;
};

// Thread = (test bin b, K quarter kq, Doppler dd): the three channel outputs
// of bin b at Doppler dd over window rows [kq K4, (kq + 1) K4), three
// independent FP64 chains sharing each X load (E rows broadcast within the
// warp); the four K partials are summed in quarter order by the candidate
// pass (deterministic). The X chunk of the next DT_TD Dopplers is staged by
// cp.async into the second buffer while the current one is consumed (when
// both fit the smem budget).
constexpr int DT_KQ = 4;  // K split of the window rows
template <int P>
__global__ void __launch_bounds__(NT) lm_detect_kernel(const cplx* __restrict__ spec,
                                                       const cplx* __restrict__ Ein,
                                                       const cplx* __restrict__ hconj, DetArgs g,
                                                       int nbuf, double* __restrict__ values) {
  extern __shared__ __align__(16) cplx dsm[];
  const int n_w = g.n_w, nwp = n_w * P;
  cplx* Es = dsm;                    // DT_TB x P x nwp
  cplx* Xb = Es + DT_TB * P * nwp;   // nbuf x (span x P x DT_LD)
  __shared__ cplx Hs[64 * 4];
  __shared__ cplx Yp[DT_KQ * DT_TB * P * DT_TD];  // K-quarter partials
  const int64_t t0 = g.lo + (int64_t)blockIdx.x * DT_TB;
  const int nt = (int)min((int64_t)DT_TB, g.hi - t0);
  const int64_t sf = win_start(t0, n_w, g.n_bins);
  const int span = (int)(win_start(t0 + nt - 1, n_w, g.n_bins) + n_w - sf);
  const size_t xsz = (size_t)span * P * DT_LD;
  for (int e = threadIdx.x; e < nt * P * nwp; e += NT)
    cp_async16(&Es[e], &Ein[(size_t)(t0 - g.lo) * P * nwp + e]);
  for (int e = threadIdx.x; e < g.G * P; e += NT) Hs[e] = hconj[e];
  const int b = threadIdx.x / (DT_KQ * DT_TD), kq = (threadIdx.x / DT_TD) % DT_KQ,
            dd = threadIdx.x % DT_TD;
  const int kqn = (nwp + DT_KQ - 1) / DT_KQ, k0 = kq * kqn, k1 = min(nwp, k0 + kqn);
  const int base = b < nt ? (int)(win_start(t0 + b, n_w, g.n_bins) - sf) * P : 0;
  auto stage = [&](int d0, cplx* Xs) {
    const int dl = min(DT_TD, g.D - d0);
    for (int e = threadIdx.x; e < span * P * DT_TD; e += NT) {
      const int row = e / DT_TD, c = e - row * DT_TD;
      if (c < dl)
        cp_async16(&Xs[row * DT_LD + c], &spec[((sf - g.a) * P + row) * (int64_t)g.D + d0 + c]);
    }
    cp_async_commit();
  };
  stage(0, Xb);
  int buf = 0;
  for (int d0 = 0; d0 < g.D; d0 += DT_TD) {
    const int dl = min(DT_TD, g.D - d0);
    const bool next = d0 + DT_TD < g.D;
    if (nbuf == 2 && next) {
      stage(d0 + DT_TD, Xb + (size_t)(buf ^ 1) * xsz);  // its slot was freed by the last barrier
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk d0 (and E) visible
    const cplx* Xs = Xb + (size_t)buf * xsz;
    if (b < nt && dd < dl) {
      cplx acc[P];
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = cmk(0, 0);
      const cplx* er = Es + (size_t)b * P * nwp;
      const cplx* xr = Xs + (size_t)base * DT_LD + dd;
#pragma unroll 4
      for (int jx = k0; jx < k1; ++jx) {
        const cplx x = xr[jx * DT_LD];
#pragma unroll
        for (int i = 0; i < P; ++i) cfma(acc[i], er[i * nwp + jx], x);
      }
#pragma unroll
      for (int i = 0; i < P; ++i) Yp[((kq * DT_TB + b) * P + i) * DT_TD + dd] = acc[i];
    }
    __syncthreads();  // partials ready; chunk d0's X slot may be refilled
    for (int o = threadIdx.x; o < nt * DT_TD; o += NT) {
      const int bb = o / DT_TD, d2 = o % DT_TD;
      if (d2 >= dl) continue;
      cplx y[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        cplx v = Yp[((0 * DT_TB + bb) * P + i) * DT_TD + d2];
#pragma unroll
        for (int k = 1; k < DT_KQ; ++k) v = cadd(v, Yp[((k * DT_TB + bb) * P + i) * DT_TD + d2]);
        y[i] = v;
      }
      double best2 = -1.0;
      cplx zb = cmk(0, 0);
      for (int gg = 0; gg < g.G; ++gg) {
        cplx z = cmk(0, 0);
#pragma unroll
        for (int i = 0; i < P; ++i) cfma(z, Hs[gg * P + i], y[i]);
        const double m2 = cabs2(z);
        if (m2 > best2) {
          best2 = m2;
          zb = z;
        }
      }
      values[(t0 + bb - g.lo) * (int64_t)g.D + d0 + d2] = hypot(zb.x * g.inv_sqrt_q, zb.y * g.inv_sqrt_q);
    }
    if (nbuf == 2) buf ^= 1;
    else if (next) {
      __syncthreads();  // single buffer: every read of chunk d0 done before restaging
      stage(d0 + DT_TD, Xb);
    }
  }
}

size_t window_smem(int nbmax, int n_w, int p) {
  const size_t jbytes = (kstj::jac_smem_bytes(LM_JAC) + 15) / 16 * 16;
  return jbytes + sizeof(double) * 256 +
         sizeof(cplx) * (2 * (size_t)nbmax * LM_S + (size_t)n_w * p * LM_KBMAX +
                         (size_t)(n_w / 2 + 1) * p * LM_KBMAX);
}

int band_splits(int q) { return std::max(1, std::min(8, q / 32)); }

template <int P>
int launch_band(kst_ctx* ctx, const cplx* X, int nb, int q, int n_w, cplx* W, cplx* rs,
                cplx* Wp, cudaStream_t st) {
  constexpr int KT = BG<P>::KT;
  const int ngrp = (n_w + KT - 1) / KT;
  const int tb = std::max(1, NT / ngrp);
  const size_t smem = sizeof(cplx) * (size_t)(tb + n_w - 1) * P * BG_LD;
  const int nsplit = band_splits(q);
  const int qs = ((q + nsplit - 1) / nsplit + BG_TQ - 1) / BG_TQ * BG_TQ;
  const int64_t wcount = (int64_t)nb * n_w * P * P, rcount = (int64_t)nb * P;
  KST_CUDA(ctx, cudaFuncSetAttribute(band_gram_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  if (nsplit == 1) {
    band_gram_kernel<P><<<dim3(cdiv(nb, tb), 1), NT, smem, st>>>(X, nb, q, n_w, tb, qs, 0, W, rs);
    KST_LAUNCH(ctx);
    return KST_OK;
  }
  const int ny = (q + qs - 1) / qs;
  band_gram_kernel<P><<<dim3(cdiv(nb, tb), ny), NT, smem, st>>>(X, nb, q, n_w, tb, qs, wcount, Wp,
                                                                Wp + ny * wcount);
  KST_LAUNCH(ctx);
  band_reduce_kernel<<<(unsigned)std::min<int64_t>(cdiv(wcount + rcount, 256), 4096), 256, 0, st>>>(
      Wp, ny, wcount, wcount, rcount, W, rs);
  KST_LAUNCH(ctx);
  return KST_OK;
}

template <int P>
int launch_prefix(kst_ctx* ctx, const cplx* W, int nb, int n_w, double* Qp, cudaStream_t st) {
  constexpr int NI = 2 + P * P * (P * P + 1) / 2;  // one warp per (bin, record item)
  band_prefix_kernel<P><<<(unsigned)cdiv((int64_t)nb * NI * 32, 256), 256, 0, st>>>(W, nb, n_w, Qp);
  KST_LAUNCH(ctx);
  return KST_OK;
}

template <int P>
int launch_win(kst_ctx* ctx, const cplx* W, const cplx* rs, const double* Qp, const WinArgs& wa,
               cplx* H, double* rscr, cplx* E, int* dinfo, double* dres, size_t wsm,
               cudaStream_t st) {
  KST_CUDA(ctx, cudaFuncSetAttribute(window_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)wsm));
  window_kernel<P><<<wa.nslot, NT, wsm, st>>>(W, rs, Qp, wa, H, rscr, E, dinfo, dres);
  KST_LAUNCH(ctx);
  return KST_OK;
}

template <int P>
int launch_det(kst_ctx* ctx, const cplx* spec, const cplx* E, const cplx* hconj, const DetArgs& da,
               double* values, int64_t n_test, size_t dsm, int nbuf, cudaStream_t st) {
  KST_CUDA(ctx, cudaFuncSetAttribute(lm_detect_kernel<P>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  lm_detect_kernel<P><<<cdiv(n_test, DT_TB), NT, dsm, st>>>(spec, E, hconj, da, nbuf, values);
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace

#ifdef KST_LM_PROF
extern "C" __attribute__((visibility("default"))) int kst_lm_prof(long long* out, int nwin) {
  return (int)cudaMemcpyFromSymbol(out, lm_prof, sizeof(long long) * 16 * std::min(nwin, 4096));
}
#endif

extern "C" int kst_windowed(kst_ctx* ctx, const double* cube, int64_t a, int64_t n_bins, int p,
                            int q, int n_w, int64_t lo, int64_t hi, int64_t s_begin, int64_t s_end,
                            int64_t s_step, int rank_spatial, int rank_temporal, double tol,
                            int max_iter, int kind, int drop_temporal, const double* dopplers,
                            int D, const double* grid, int G, double* values, void* stream);

extern "C" int kst_lmode(kst_ctx* ctx, const double* cube, int64_t a, int64_t n_bins, int p, int q,
                         int n_w, int64_t lo, int64_t hi, int rank_spatial, int rank_temporal,
                         double tol, int max_iter, int kind, int drop_temporal,
                         const double* dopplers, int D, const double* grid, int G, double* values,
                         int* window_info, void* stream) {
  CTX_GUARD(ctx);
  cudaStream_t st = (cudaStream_t)stream;
  if (p < 1 || q < 1 || n_w < 1 || n_w > n_bins || lo < 0 || hi > n_bins || lo >= hi || a < 0 ||
      D < 1 || G < 1)
    return set_err(ctx, KST_ERR_DIMENSION, "lmode: bad window / tile arguments");
  if (rank_spatial < 1 || rank_spatial > p)
    return set_err(ctx, KST_ERR_DIMENSION, "spatial rank must be in [1, %d], got %d", p,
                   rank_spatial);
  if (rank_temporal < 1 || rank_temporal > q)
    return set_err(ctx, KST_ERR_DIMENSION, "temporal rank must be in [1, %d], got %d", q,
                   rank_temporal);
  if (max_iter < 1) return set_err(ctx, KST_ERR_DIMENSION, "max_iter must be >= 1, got %d", max_iter);
  const int64_t s_lo = win_start(lo, n_w, n_bins), s_hi = win_start(hi - 1, n_w, n_bins);
  if (a > s_lo) return set_err(ctx, KST_ERR_DIMENSION, "lmode: tile cube starts after its halo");
  const int nwin = (int)(s_hi - s_lo + 1);
  static const bool batched_env = !(getenv("KST_LMODE") && strcmp(getenv("KST_LMODE"), "serial") == 0);
  const bool supported = batched_env && p <= 3 && n_w <= LM_NWMAX && rank_temporal <= LM_S - 2 &&
                         rank_temporal < q && G <= 64 &&
                         (kind == KST_KIND_KRON || kind == KST_KIND_CLASSICAL);
  if (!supported) {
    if (window_info) std::fill(window_info, window_info + (size_t)nwin * WI, -1);
    return kst_windowed(ctx, cube, a, n_bins, p, q, n_w, lo, hi, s_lo, s_hi + 1, 1, rank_spatial,
                        rank_temporal, tol, max_iter, kind, drop_temporal, dopplers, D, grid, G,
                        values, stream);
  }
  const int64_t b_end = s_hi + n_w;  // tile cube bins [a, b_end) are read
  const int nb = (int)(b_end - a);
  const int nwp = n_w * p;
  const int64_t n_test = hi - lo;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int nslot = std::min(nwin, KST_WIN_MINB * nsm);
  // n_w r, r = rank of the b-producing spatial iterate: r_a, or p when the
  // loop stops after its first iteration (A_prev = A0)
  const int nbmax = std::min(LM_NBMAX, n_w * (max_iter == 1 ? p : rank_spatial));
  // workspace
  char* wspec = (char*)ws_get(ctx, WS_LM_SPEC, sizeof(cplx) * ((size_t)nb * p * D + D + (size_t)G * p) +
                                                   sizeof(double) * D + 256);
  const int nsplit = band_splits(q);
  // W + row sums, then (split-K) nsplit partial copies of both
  // band-prefix record rows (nb x n_w x (2 + 2E) doubles), then W + row sums,
  // then (split-K) nsplit partial copies of both
  const size_t nq = 2 + (size_t)p * p * (p * p + 1);
  const size_t qbytes = (sizeof(double) * (size_t)nb * n_w * nq + 255) / 256 * 256;
  char* wW = (char*)ws_get(ctx, WS_LM_W, qbytes + sizeof(cplx) * ((size_t)nb * n_w * p * p + (size_t)nb * p) *
                                                      (nsplit > 1 ? nsplit + 1 : 1) + 256);
  char* wE = (char*)ws_get(ctx, WS_LM_E, sizeof(cplx) * (size_t)n_test * p * nwp +
                                             sizeof(int) * (size_t)nwin * WI + sizeof(double) * nwin + 256);
  char* wH = (char*)ws_get(ctx, WS_LM_H, sizeof(cplx) * (size_t)nslot * nbmax * nbmax +
                                             sizeof(double) * (size_t)nslot * (max_iter + 1) + 256);
  int* hinfo = (int*)pinned_get(ctx, sizeof(int) * (size_t)nwin * WI + sizeof(cplx) * G * p + 64);
  if (!wspec || !wW || !wE || !wH || !hinfo) return set_err(ctx, KST_ERR_CUDA, "lmode: workspace");
  cplx* spec = (cplx*)wspec;
  cplx* hconj = spec + (size_t)nb * p * D;
  void* consts = hconj + (size_t)G * p;
  double* Qp = (double*)wW;
  cplx* W = (cplx*)(wW + qbytes);
  cplx* rs = W + (size_t)nb * n_w * p * p;
  cplx* Wp = rs + (size_t)nb * p;  // split-K partials (nsplit > 1)
  cplx* E = (cplx*)wE;
  int* dinfo = (int*)(E + (size_t)n_test * p * nwp);
  double* dres = (double*)(((uintptr_t)(dinfo + (size_t)nwin * WI) + 15) & ~(uintptr_t)15);
  cplx* H = (cplx*)wH;
  double* rscr = (double*)(H + (size_t)nslot * nbmax * nbmax);
  // conj(grid) (pinned staging, then the stream owns it until the sync below)
  cplx* hg = (cplx*)(hinfo + (size_t)nwin * WI);
  hg = (cplx*)(((uintptr_t)hg + 15) & ~(uintptr_t)15);
  for (int e = 0; e < G * p; ++e) hg[e] = cconj(((const cplx*)grid)[e]);
  KST_CUDA(ctx, cudaMemcpyAsync(hconj, hg, sizeof(cplx) * G * p, cudaMemcpyHostToDevice, st));
  const cplx* X = (const cplx*)cube;  // bin a at row 0
  // 1. spectra of every bin the tile reads
  KST_TRY(kst::spectra(ctx, X, (int64_t)nb * p, q, dopplers, D, spec, consts, st));
  // 2. banded snapshot Gram + row sums
  switch (p) {
    case 1: KST_TRY(launch_band<1>(ctx, X, nb, q, n_w, W, rs, Wp, st)); break;
    case 2: KST_TRY(launch_band<2>(ctx, X, nb, q, n_w, W, rs, Wp, st)); break;
    default: KST_TRY(launch_band<3>(ctx, X, nb, q, n_w, W, rs, Wp, st)); break;
  }
  KST_LAUNCH(ctx);
  switch (p) {
    case 1: KST_TRY(launch_prefix<1>(ctx, W, nb, n_w, Qp, st)); break;
    case 2: KST_TRY(launch_prefix<2>(ctx, W, nb, n_w, Qp, st)); break;
    default: KST_TRY(launch_prefix<3>(ctx, W, nb, n_w, Qp, st)); break;
  }
  // 3. one CTA per window (persistent over nslot CTAs)
  WinArgs wa;
  wa.a = a;
  wa.n_bins = n_bins;
  wa.lo = lo;
  wa.hi = hi;
  wa.s0 = s_lo;
  wa.nwin = nwin;
  wa.n_w = n_w;
  wa.q = q;
  wa.ra = rank_spatial;
  wa.rb = rank_temporal;
  wa.max_iter = max_iter;
  wa.kind = kind;
  wa.spatial_only = drop_temporal;
  wa.nslot = nslot;
  wa.nbmax = nbmax;
  wa.tol = tol;
  const size_t wsm = window_smem(nbmax, n_w, p);
  switch (p) {
    case 1: KST_TRY(launch_win<1>(ctx, W, rs, Qp, wa, H, rscr, E, dinfo, dres, wsm, st)); break;
    case 2: KST_TRY(launch_win<2>(ctx, W, rs, Qp, wa, H, rscr, E, dinfo, dres, wsm, st)); break;
    default: KST_TRY(launch_win<3>(ctx, W, rs, Qp, wa, H, rscr, E, dinfo, dres, wsm, st)); break;
  }
  KST_LAUNCH(ctx);
  // 4. detection of the tile's test bins
  DetArgs da;
  da.a = a;
  da.n_bins = n_bins;
  da.lo = lo;
  da.hi = hi;
  da.n_w = n_w;
  da.D = D;
  da.G = G;
  da.inv_sqrt_q = 1.0 / sqrt((double)q);
  // E rows + one or two X chunks (double-buffered when both fit 200 KB)
  const size_t xchunk = sizeof(cplx) * (size_t)(DT_TB + n_w - 1) * p * DT_LD;
  const size_t ebytes = sizeof(cplx) * (size_t)DT_TB * p * nwp;
  const int nbuf = ebytes + 2 * xchunk <= 200 * 1024 ? 2 : 1;
  const size_t dsm = ebytes + nbuf * xchunk;
  switch (p) {
    case 1: KST_TRY(launch_det<1>(ctx, spec, E, hconj, da, values, n_test, dsm, nbuf, st)); break;
    case 2: KST_TRY(launch_det<2>(ctx, spec, E, hconj, da, values, n_test, dsm, nbuf, st)); break;
    default: KST_TRY(launch_det<3>(ctx, spec, E, hconj, da, values, n_test, dsm, nbuf, st)); break;
  }
  KST_LAUNCH(ctx);
  // 5. window statuses: errors raise in window order (the reference's loop
  //    order); windows the batched solver handed back run on the step path
  KST_CUDA(ctx, cudaMemcpyAsync(hinfo, dinfo, sizeof(int) * (size_t)nwin * WI, cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  std::vector<int> info(hinfo, hinfo + (size_t)nwin * WI);
  for (int w = 0; w < nwin; ++w) {
    const int sc = info[(size_t)w * WI];
    if (sc == 200) return set_err(ctx, KST_ERR_DATA, "covariance contains non-finite entries");
    if (sc == KST_ERR_DATA)
      return set_err(ctx, KST_ERR_DATA, "matrix deviates from Hermitian beyond tolerance");
    if (sc == KST_ERR_DEGENERATE + 100)
      return set_err(ctx, KST_ERR_DEGENERATE, "spatial iterate collapsed to zero");
    if (sc == KST_ERR_DEGENERATE)
      return set_err(ctx, KST_ERR_DEGENERATE, "temporal iterate collapsed to zero");
    if (sc != 0 && sc != LM_FALLBACK)
      return set_err(ctx, sc, "lmode: window %lld failed", (long long)(s_lo + w));
  }
  for (int w = 0; w < nwin; ++w)
    if (info[(size_t)w * WI] == LM_FALLBACK) {
      KST_TRY(kst_windowed(ctx, cube, a, n_bins, p, q, n_w, lo, hi, s_lo + w, s_lo + w + 1, 1,
                           rank_spatial, rank_temporal, tol, max_iter, kind, drop_temporal,
                           dopplers, D, grid, G, values, stream));
    }
  if (window_info) std::copy(info.begin(), info.end(), window_info);
  return KST_OK;
}
