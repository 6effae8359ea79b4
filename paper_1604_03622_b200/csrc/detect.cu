// K5/K6: detection image for the projection filters, FP64.
//
// Reference (src/filters.py:243-275, 88-116): per bin m,
//   F = filter(X_m)                       (kron: X - (X conj(U_B)) U_B^T, then
//                                          X - U_A (U_A^H X); classical: joint)
//   values[m, d] = max_g | sum_i conj(H[g,i]) sum_t F[i,t] conj(T[t,d]) |,
//   T[t,d] = exp(2 pi i t f_d) / sqrt(q).
//
// B200 formulation: the filter is linear and acts on the
// channel and pulse axes separately, so it commutes with the pulse-axis
// transform. Per (bin, channel) row we
//   1. compute the temporal coefficients c[k] = sum_t x[t] conj(U_B[t,k]),
//   2. fold t mod D and run a length-D mixed-radix Stockham DFT in shared
//      memory (exact integer twiddle indices into an FP64 table), which for
//      the uniform grid f_d = d/D equals sum_t x[t] exp(-2 pi i t d / D);
//      any other Doppler set takes a direct sum,
// then per (bin, Doppler) subtract sum_k c[k] DFT(U_B[:,k])[d], apply the
// spatial projector, the spatial candidates, |.|, max, and write f64.
// Multipass (`pass_images`, src/multipass.py:83-102) filters once and
// emits one map per row block of the stacked grid (`groups`).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace {

#ifndef KST_FFT_GRP
#define KST_FFT_GRP 0
#endif
constexpr int NT = 256;
constexpr int kMaxFactors = 32;
constexpr int kMaxP = 16;
constexpr int kMaxKB = 64;

// Odd radices with register-resident butterflies; their W_R^m = (cos, -sin)
// of 2 pi m / R live in the plan (constant bank) at offset rtw_off(R).
constexpr int kRegRadix[] = {3, 5, 7, 11, 13, 23, 29};
__host__ __device__ constexpr int rtw_off(int R) {
  return R == 3 ? 0 : R == 5 ? 3 : R == 7 ? 8 : R == 11 ? 15 : R == 13 ? 26 : R == 23 ? 39 : 62;
}
constexpr int kRtwCount = 91;  // sum of kRegRadix

struct Plan {
  int D;
  int nf;
  int radix[kMaxFactors];
  double rtw[2 * kRtwCount];
};

__constant__ Plan c_plan;

// twiddle table w[k] = exp(-2 pi i k / D)
__global__ void twiddle_kernel(cplx* w, int D) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < D; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)D, &s, &c);
    w[k] = cmk(c, s);
  }
}

// One odd-radix Stockham stage with the butterfly inputs held in registers:
// each work item j < D/R loads its R inputs once (stage twiddles applied),
// forms s_r = t_r + t_{R-r}, d_r = t_r - t_{R-r} in place, and emits all R
// outputs -- shared-memory traffic ~2D per stage instead of ~R*D.
template <int R>
__device__ __forceinline__ void stage_reg(const cplx* __restrict__ a, cplx* __restrict__ b,
                                          const cplx* __restrict__ w, int D, int Ns) {
  constexpr int h = (R - 1) / 2;
  constexpr int off = rtw_off(R);
  const int DR = D / R, step = D / (Ns * R);
  for (int j = threadIdx.x; j < DR; j += blockDim.x) {
    const int k = j % Ns;
    cplx t[R];
    t[0] = a[j];
#pragma unroll
    for (int r = 1; r < R; ++r) t[r] = cmul(a[j + r * DR], w[r * k * step]);
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const cplx sr = cadd(t[r], t[R - r]), dr = csub(t[r], t[R - r]);
      t[r] = sr;
      t[R - r] = dr;
    }
    const int dst = (j / Ns) * Ns * R + k;
    cplx x0 = t[0];
#pragma unroll
    for (int r = 1; r <= h; ++r) x0 = cadd(x0, t[r]);
    b[dst] = x0;
    // fully unrolled: (r u) mod R is a compile-time constant, so every
    // W_R^m operand is a constant-bank read folded into the DFMA
#pragma unroll
    for (int u = 1; u <= h; ++u) {
      double ax = t[0].x, ay = t[0].y, bx = 0.0, by = 0.0;
#pragma unroll
      for (int r = 1; r <= h; ++r) {
        const int m = (r * u) % R;
        const double wc = c_plan.rtw[2 * (off + m)], ws = c_plan.rtw[2 * (off + m) + 1];
        ax = fma(wc, t[r].x, ax);
        ay = fma(wc, t[r].y, ay);
        bx = fma(-ws, t[R - r].x, bx);
        by = fma(-ws, t[R - r].y, by);
      }
      b[dst + u * Ns] = cmk(ax + by, ay - bx);        // A - iB
      b[dst + (R - u) * Ns] = cmk(ax - by, ay + bx);  // A + iB
    }
  }
}

// Large odd radices (11, 13, 23, 29) in two phases, so the R-point
// butterflies neither pin 2R doubles per thread nor leave most threads idle
// (the radix-29 stage of D = 2001 has only 69 butterflies):
//   A (one thread per butterfly j): twiddled t_r, pairs s_r = t_r + t_{R-r},
//     d_r = t_r - t_{R-r} written back in place, X_0 = t_0 + sum s_r;
//   B (one thread per (j, group of GU output pairs)): streams (s_r, d_r)
//     from smem and keeps 4 GU independent accumulator chains in registers.
// Same operation order per output as stage_reg (bitwise identical results).
template <int R, int GU, int G>
__device__ __forceinline__ void grp_unit(const cplx* __restrict__ a, cplx* __restrict__ b, int j,
                                         int DR, int Ns) {
  constexpr int h = (R - 1) / 2, off = rtw_off(R);
  constexpr int U0 = 1 + G * GU, U1 = (U0 + GU - 1 < h) ? U0 + GU - 1 : h, NU = U1 - U0 + 1;
  const int k = j % Ns, dst = (j / Ns) * Ns * R + k;
  const cplx t0 = a[j];
  double ax[NU], ay[NU], bx[NU], by[NU];
#pragma unroll
  for (int v = 0; v < NU; ++v) {
    ax[v] = t0.x;
    ay[v] = t0.y;
    bx[v] = 0.0;
    by[v] = 0.0;
  }
#pragma unroll
  for (int r = 1; r <= h; ++r) {
    const cplx sr = a[j + r * DR], dr = a[j + (R - r) * DR];
#pragma unroll
    for (int v = 0; v < NU; ++v) {
      const int m = (r * (U0 + v)) % R;
      const double wc = c_plan.rtw[2 * (off + m)], ws = c_plan.rtw[2 * (off + m) + 1];
      ax[v] = fma(wc, sr.x, ax[v]);
      ay[v] = fma(wc, sr.y, ay[v]);
      bx[v] = fma(-ws, dr.x, bx[v]);
      by[v] = fma(-ws, dr.y, by[v]);
    }
  }
#pragma unroll
  for (int v = 0; v < NU; ++v) {
    const int u = U0 + v;
    b[dst + u * Ns] = cmk(ax[v] + by[v], ay[v] - bx[v]);        // A - iB
    b[dst + (R - u) * Ns] = cmk(ax[v] - by[v], ay[v] + bx[v]);  // A + iB
  }
}

template <int R, int GU>
__device__ void stage_grp(cplx* __restrict__ a, cplx* __restrict__ b, const cplx* __restrict__ w,
                          int D, int Ns) {
  constexpr int h = (R - 1) / 2, NGR = (h + GU - 1) / GU;
  static_assert(NGR >= 1 && NGR <= 3, "stage_grp: 1..3 output groups");
  const int DR = D / R, step = D / (Ns * R);
  for (int j = threadIdx.x; j < DR; j += blockDim.x) {  // phase A
    const int k = j % Ns, dst = (j / Ns) * Ns * R + k;
    cplx x0 = a[j];
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const cplx tr = cmul(a[j + r * DR], w[r * k * step]);
      const cplx tm = cmul(a[j + (R - r) * DR], w[(R - r) * k * step]);
      const cplx sr = cadd(tr, tm);
      a[j + r * DR] = sr;
      a[j + (R - r) * DR] = csub(tr, tm);
      x0 = cadd(x0, sr);
    }
    b[dst] = x0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < DR * NGR; e += blockDim.x) {  // phase B
    const int j = e % DR, g = e / DR;
    if (g == 0) grp_unit<R, GU, 0>(a, b, j, DR, Ns);
    if (NGR > 1 && g == 1) grp_unit<R, GU, (NGR > 1 ? 1 : 0)>(a, b, j, DR, Ns);
    if (NGR > 2 && g == 2) grp_unit<R, GU, (NGR > 2 ? 2 : 0)>(a, b, j, DR, Ns);
  }
}

// Ping-pong Stockham DFT (decimation in time) of length D over shared
// buffers; w[k] = exp(-2 pi i k / D). Stage (radix R, Ns = product of the
// previous radices, DR = D / R, step = D / (Ns R)), for j < DR, k = j mod Ns:
//   t_r = a[j + r DR] * w[r k step],   X_u = sum_r t_r W_R^{ru},
//   b[(j / Ns) Ns R + k + u Ns] = X_u.
// Radix 2 and 4 use explicit butterflies. Odd radices pair outputs u, R-u:
// with s_r = t_r + t_{R-r}, d_r = t_r - t_{R-r},
//   X_u = t_0 + sum_r cos(2 pi r u / R) s_r -+ i sum_r sin(2 pi r u / R) d_r,
// a quarter of the real multiply-adds of the direct R-point sum. All twiddle
// indices are exact integers (no float phase accumulation).
// Returns the buffer holding the result.
__device__ cplx* stockham(cplx* a, cplx* b, const cplx* __restrict__ w, int D) {
  int Ns = 1;
  const int nt = blockDim.x;
  for (int f = 0; f < c_plan.nf; ++f) {
    const int R = c_plan.radix[f];
    const int DR = D / R;
    const int step = D / (Ns * R);
    if (R == 2 || R == 4) {
      for (int j = threadIdx.x; j < DR; j += nt) {
        const int k = j % Ns;
        const int dst = (j / Ns) * Ns * R + k;
        if (R == 2) {
          const cplx t0 = a[j], t1 = cmul(a[j + DR], w[k * step]);
          b[dst] = cadd(t0, t1);
          b[dst + Ns] = csub(t0, t1);
        } else {
          const cplx t0 = a[j];
          const cplx t1 = cmul(a[j + DR], w[k * step]);
          const cplx t2 = cmul(a[j + 2 * DR], w[2 * k * step]);
          const cplx t3 = cmul(a[j + 3 * DR], w[3 * k * step]);
          const cplx s02 = cadd(t0, t2), d02 = csub(t0, t2);
          const cplx s13 = cadd(t1, t3), d13 = csub(t1, t3);
          // -i * d13 = (d13.y, -d13.x)
          b[dst] = cadd(s02, s13);
          b[dst + Ns] = cmk(d02.x + d13.y, d02.y - d13.x);
          b[dst + 2 * Ns] = csub(s02, s13);
          b[dst + 3 * Ns] = cmk(d02.x - d13.y, d02.y + d13.x);
        }
      }
    } else if (R == 3 || R == 5 || R == 7 || R == 11 || R == 13 || R == 23 || R == 29) {
      switch (R) {
        case 3: stage_reg<3>(a, b, w, D, Ns); break;
        case 5: stage_reg<5>(a, b, w, D, Ns); break;
        case 7: stage_reg<7>(a, b, w, D, Ns); break;
#if KST_FFT_GRP
        case 11: stage_grp<11, 5>(a, b, w, D, Ns); break;
        case 13: stage_grp<13, 6>(a, b, w, D, Ns); break;
        case 23: stage_grp<23, 6>(a, b, w, D, Ns); break;
        default: stage_grp<29, 7>(a, b, w, D, Ns); break;
#else
        case 11: stage_reg<11>(a, b, w, D, Ns); break;
        case 13: stage_reg<13>(a, b, w, D, Ns); break;
        case 23: stage_reg<23>(a, b, w, D, Ns); break;
        default: stage_reg<29>(a, b, w, D, Ns); break;
#endif
      }
    } else {
      const int h = (R - 1) / 2;
      // phase A: stage twiddles, folded into (s_r, d_r) in place
      for (int e = threadIdx.x; e < DR * h; e += nt) {
        const int j = e % DR, r = 1 + e / DR;
        const int k = j % Ns;
        const cplx tr = cmul(a[j + r * DR], w[r * k * step]);
        const cplx tm = cmul(a[j + (R - r) * DR], w[(R - r) * k * step]);
        a[j + r * DR] = cadd(tr, tm);
        a[j + (R - r) * DR] = csub(tr, tm);
      }
      __syncthreads();
      // phase B: output pairs (u, R - u) and u = 0
      const int DRR = D / R;  // W_R^m = w[m * D / R]
      for (int e = threadIdx.x; e < DR * (h + 1); e += nt) {
        const int j = e % DR, u = e / DR;
        const int k = j % Ns;
        const int dst = (j / Ns) * Ns * R + k;
        const cplx t0 = a[j];
        if (u == 0) {
          cplx acc0 = t0, acc1 = cmk(0, 0);
          int r = 1;
          for (; r + 1 <= h; r += 2) {
            acc0 = cadd(acc0, a[j + r * DR]);
            acc1 = cadd(acc1, a[j + (r + 1) * DR]);
          }
          if (r <= h) acc0 = cadd(acc0, a[j + r * DR]);
          b[dst] = cadd(acc0, acc1);
        } else {
          double ax = t0.x, ay = t0.y, bx = 0.0, by = 0.0;
          int m = 0;
          for (int r = 1; r <= h; ++r) {
            m += u;
            if (m >= R) m -= R;
            const cplx wm = w[m * DRR];  // (cos, -sin)
            const cplx sr = a[j + r * DR], dr = a[j + (R - r) * DR];
            ax = fma(wm.x, sr.x, ax);
            ay = fma(wm.x, sr.y, ay);
            bx = fma(-wm.y, dr.x, bx);
            by = fma(-wm.y, dr.y, by);
          }
          // X_u = A - iB, X_{R-u} = A + iB
          b[dst + u * Ns] = cmk(ax + by, ay - bx);
          b[dst + (R - u) * Ns] = cmk(ax - by, ay + bx);
        }
      }
    }
    __syncthreads();
    cplx* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

// One CTA per row (bin m, channel i) of `src` (rows x q, row stride q):
// coefficients against U_B and the folded DFT (uniform) or direct sum.
// 128-thread CTAs: the register-resident radix-23/29 butterflies need ~150
// registers, so two row-CTAs per SM beat one 256-thread CTA.
#ifndef KST_NTS
#define KST_NTS 128
#endif
constexpr int NTS = KST_NTS;
#ifndef KST_RS_GTW
#define KST_RS_GTW 0
#endif
#ifndef KST_RS_MINB
#define KST_RS_MINB 1
#endif
#ifndef KST_CB_MINB
#define KST_CB_MINB 1
#endif
__global__ void __launch_bounds__(NTS, KST_RS_MINB) row_spectrum_kernel(
    const cplx* __restrict__ src, int64_t rows, int q, const cplx* __restrict__ ub, int kb,
    const cplx* __restrict__ w, int D, int uniform, const double* __restrict__ dop,
    cplx* __restrict__ spec, cplx* __restrict__ coef, int* __restrict__ nonfinite) {
  constexpr int NT = NTS;  // shadows the file-wide 256
  extern __shared__ __align__(16) cplx smem[];
  __shared__ double red[32];
  const int64_t row = blockIdx.x;
  const cplx* x = src + row * q;
  // 0. stage the row (and the twiddle table) in smem with one batch of
  //    cp.async copies: every load is in flight at once instead of one
  //    dependent global load per loop trip.
  //    Uniform grid with q <= D: the row lands in the FFT input buffer
  //    (zero-padded to D); otherwise in the first q entries of smem.
  const bool staged_fft = uniform && q <= D;
  cplx* xs = smem;  // staged row (both paths start at smem[0])
  if (uniform) {
#if KST_RS_GTW
    for (int k = threadIdx.x; k < D; k += NT) {
      if (staged_fft) {
#else
    cplx* tw = smem + 2 * D;
    for (int k = threadIdx.x; k < D; k += NT) {
      cp_async16(&tw[k], &w[k]);
      if (staged_fft) {
#endif
        if (k < q)
          cp_async16(&xs[k], &x[k]);
        else
          xs[k] = cmk(0, 0);
      }
    }
  } else {
    for (int t = threadIdx.x; t < q; t += NT) cp_async16(&xs[t], &x[t]);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const bool in_smem = staged_fft || !uniform;
  const cplx* xr = in_smem ? xs : x;
  // 1. temporal coefficients c[k] = sum_t x[t] conj(ub[t, k]), 4 at a time,
  //    one fixed-order multi-value block reduction per group
  int bad = 0;
  __shared__ double red4[8][NT / 32];
  for (int k0 = 0; k0 < kb; k0 += 4) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 4
    for (int t = threadIdx.x; t < q; t += NT) {
      const cplx v = xr[t];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < kb) {
          const cplx w_ = ub[(int64_t)t * kb + k0 + u];
          acc[2 * u] = fma(v.x, w_.x, acc[2 * u]);
          acc[2 * u] = fma(v.y, w_.y, acc[2 * u]);
          acc[2 * u + 1] = fma(v.y, w_.x, acc[2 * u + 1]);
          acc[2 * u + 1] = fma(-v.x, w_.y, acc[2 * u + 1]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = warp_sum(acc[u]);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
      for (int u = 0; u < 8; ++u) red4[u][wid] = acc[u];
    __syncthreads();
    if (threadIdx.x < 8) {
      double s_ = 0.0;
      for (int w2 = 0; w2 < NT / 32; ++w2) s_ += red4[threadIdx.x][w2];
      const int u = threadIdx.x >> 1;
      if (k0 + u < kb) {
        double* cp = (double*)&coef[row * kb + k0 + u];
        cp[threadIdx.x & 1] = s_;
      }
    }
    __syncthreads();
  }
  (void)red;
  if (uniform) {
    cplx* a = smem;
    cplx* b = smem + D;
#if KST_RS_GTW
    const cplx* tw = w;  // twiddle table read through L1 (frees 1/3 of the smem)
#else
    cplx* tw = smem + 2 * D;
#endif
    if (staged_fft) {
      for (int t = threadIdx.x; t < q; t += NT) {
        const cplx v = a[t];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
      }
    } else {
      // 2. fold t mod D (ascending t: deterministic)
      for (int tp = threadIdx.x; tp < D; tp += NT) {
        cplx acc = cmk(0, 0);
        for (int t = tp; t < q; t += D) {
          const cplx v = x[t];
          if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
          acc = cadd(acc, v);
        }
        a[tp] = acc;
      }
    }
    __syncthreads();
    cplx* res = stockham(a, b, tw, D);
    for (int d = threadIdx.x; d < D; d += NT) spec[row * D + d] = res[d];
  } else {
    // direct sum with the reference's phase: theta = 2 pi (t f_d)
    for (int t = threadIdx.x; t < q; t += NT) {
      const cplx v = xs[t];
      if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
    }
    const double twopi = 6.283185307179586;
    for (int d = threadIdx.x; d < D; d += NT) {
      const double f = dop[d];
      cplx acc = cmk(0, 0);
      for (int t = 0; t < q; ++t) {
        double s, c;
        sincos(twopi * ((double)t * f), &s, &c);
        cfmac(acc, xs[t], cmk(c, s));  // x * conj(exp(i theta))
      }
      spec[row * D + d] = acc;
    }
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

// Transpose U_B (q x kb) into kb rows of length q.
__global__ void transpose_kernel(const cplx* __restrict__ ub, int q, int kb, cplx* __restrict__ out) {
  const int64_t total = (int64_t)q * kb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / kb), k = (int)(e % kb);
    out[(int64_t)k * q + t] = ub[e];
  }
}

struct CombineArgs {
  int P, D, ka, kb, G, groups;
  int mode;  // 0: temporal coef (kron), 1: joint coef (classical), 2: none
  int spatial;  // apply spatial projector
  double inv_sqrt_q;
};

// grid: (ceil(D / NT), ceil(n / CB_BINS)). One thread per Doppler; each CTA
// walks CB_BINS consecutive bins so the per-CTA setup (projector, candidate
// grid in smem) is amortised. Templated on the channel count so the
// per-pixel channel loops are fully unrolled in registers.
constexpr int CB_BINS = 8;
template <int PT>
__global__ void __launch_bounds__(NT, KST_CB_MINB) combine_kernel(
    const cplx* __restrict__ spec, const cplx* __restrict__ coef, const cplx* __restrict__ ubspec,
    const cplx* __restrict__ ua, const cplx* __restrict__ hconj, CombineArgs a,
    double* __restrict__ values, int64_t n) {
  __shared__ cplx s_ua[kMaxP * kMaxP];
  __shared__ cplx s_c[kMaxP * kMaxKB];
  __shared__ cplx s_e[kMaxP * kMaxKB];
  extern __shared__ __align__(16) cplx s_h[];  // G x P conj grid
  constexpr int P = PT;
  for (int e = threadIdx.x; e < P * a.ka; e += NT) s_ua[e] = ua[e];
  for (int e = threadIdx.x; e < a.G * P; e += NT) s_h[e] = hconj[e];
  const int d = blockIdx.x * NT + threadIdx.x;
  const int per = a.G / a.groups;
  // bin blocks stride over gridDim.y (capped at 65535 by the launch)
  for (int64_t mb = blockIdx.y; mb * CB_BINS < n; mb += gridDim.y)
  for (int64_t m = mb * CB_BINS, m_end = min((mb + 1) * CB_BINS, n); m < m_end; ++m) {
    __syncthreads();  // previous bin's s_c fully consumed
    if (a.mode != 2) {
      for (int e = threadIdx.x; e < P * a.kb; e += NT) s_c[e] = coef[m * P * a.kb + e];
    }
    __syncthreads();
    if (a.mode == 1) {
      // classical: E = U_A (U_A^H c)  (src/filters.py:115-116)
      for (int e = threadIdx.x; e < P * a.kb; e += NT) {
        const int i = e / a.kb, k = e % a.kb;
        cplx acc = cmk(0, 0);
        for (int al = 0; al < a.ka; ++al) {
          cplx inner = cmk(0, 0);
          for (int j = 0; j < P; ++j) cfmca(inner, s_ua[j * a.ka + al], s_c[j * a.kb + k]);
          cfma(acc, s_ua[i * a.ka + al], inner);
        }
        s_e[e] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < P * a.kb; e += NT) s_c[e] = s_e[e];
      __syncthreads();
    }
    if (d >= a.D) continue;
    cplx y[kMaxP];
#pragma unroll
    for (int i = 0; i < kMaxP; ++i)
      if (i < P) y[i] = spec[(m * P + i) * a.D + d];
    if (a.mode != 2) {
      for (int k = 0; k < a.kb; ++k) {
        const cplx u = ubspec[(int64_t)k * a.D + d];
#pragma unroll
        for (int i = 0; i < kMaxP; ++i)
          if (i < P) {
            const cplx cu = cmul(s_c[i * a.kb + k], u);
            y[i] = csub(y[i], cu);
          }
      }
    }
    if (a.spatial) {
      for (int al = 0; al < a.ka; ++al) {
        cplx alpha = cmk(0, 0);
#pragma unroll
        for (int i = 0; i < kMaxP; ++i)
          if (i < P) cfmca(alpha, s_ua[i * a.ka + al], y[i]);
#pragma unroll
        for (int i = 0; i < kMaxP; ++i)
          if (i < P) y[i] = csub(y[i], cmul(s_ua[i * a.ka + al], alpha));
      }
    }
    for (int gr = 0; gr < a.groups; ++gr) {
      // max_g |z_g|: select by |z|^2, then one hypot (|.| as numpy computes it)
      double best2 = -1.0;
      cplx zb = cmk(0, 0);
      for (int g = gr * per; g < (gr + 1) * per; ++g) {
        cplx z = cmk(0, 0);
#pragma unroll
        for (int i = 0; i < kMaxP; ++i)
          if (i < P) cfma(z, s_h[g * P + i], y[i]);
        const double m2 = cabs2(z);
        if (m2 > best2) {
          best2 = m2;
          zb = z;
        }
      }
      values[((int64_t)gr * n + m) * a.D + d] = hypot(zb.x * a.inv_sqrt_q, zb.y * a.inv_sqrt_q);
    }
  }
}

__global__ void change_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              int64_t count, int is_signed, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = a[e] - b[e];
    out[e] = is_signed ? v : fabs(v);
  }
}

// c[row][k] = sum_t x[t] conj(U_B[t,k]); one CTA per (bin, channel) row
__global__ void __launch_bounds__(NT) coef_kernel(const cplx* __restrict__ src, int q,
                                                  const cplx* __restrict__ ub, int kb,
                                                  cplx* __restrict__ coef, int* __restrict__ nonfinite) {
  __shared__ double red[32];
  const int64_t row = blockIdx.x;
  const cplx* x = src + row * q;
  int bad = 0;
  for (int t = threadIdx.x; t < q; t += NT) {
    const cplx v = x[t];
    if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
  }
  if (bad) atomicOr(nonfinite, 1);
  for (int k = 0; k < kb; ++k) {
    double cr = 0.0, ci = 0.0;
    for (int t = threadIdx.x; t < q; t += NT) {
      const cplx v = x[t], u = ub[(int64_t)t * kb + k];
      cr = fma(v.x, u.x, cr);
      cr = fma(v.y, u.y, cr);
      ci = fma(v.y, u.x, ci);
      ci = fma(-v.x, u.y, ci);
    }
    cr = block_sum<NT>(cr, red);
    ci = block_sum<NT>(ci, red);
    if (threadIdx.x == 0) coef[row * kb + k] = cmk(cr, ci);
  }
}

// Time-domain projection filter (StapFilter.apply_matrix, src/filters.py:88-116):
// grid (ceil(q / NT), n); one thread per pulse t of bin m.
__global__ void __launch_bounds__(NT) filter_apply_kernel(
    const cplx* __restrict__ cube, const cplx* __restrict__ coef, const cplx* __restrict__ ub,
    const cplx* __restrict__ ua, int P, int q, int ka, int kb, int mode, int spatial,
    cplx* __restrict__ out, int64_t n) {
  __shared__ cplx s_ua[kMaxP * kMaxP];
  __shared__ cplx s_c[kMaxP * kMaxKB];
  __shared__ cplx s_e[kMaxP * kMaxKB];
  for (int e = threadIdx.x; e < P * ka; e += NT) s_ua[e] = ua[e];
  // bins stride over gridDim.y (capped at 65535 by the launch)
  for (int64_t m = blockIdx.y; m < n; m += gridDim.y) {
  __syncthreads();  // previous bin's s_c consumed
  if (mode != 2)
    for (int e = threadIdx.x; e < P * kb; e += NT) s_c[e] = coef[m * P * kb + e];
  __syncthreads();
  if (mode == 1) {
    for (int e = threadIdx.x; e < P * kb; e += NT) {
      const int i = e / kb, k = e % kb;
      cplx acc = cmk(0, 0);
      for (int al = 0; al < ka; ++al) {
        cplx inner = cmk(0, 0);
        for (int j = 0; j < P; ++j) cfmca(inner, s_ua[j * ka + al], s_c[j * kb + k]);
        cfma(acc, s_ua[i * ka + al], inner);
      }
      s_e[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < P * kb; e += NT) s_c[e] = s_e[e];
    __syncthreads();
  }
  const int t = blockIdx.x * NT + threadIdx.x;
  if (t >= q) continue;
  cplx y[kMaxP];
#pragma unroll
  for (int i = 0; i < kMaxP; ++i)
    if (i < P) y[i] = cube[(m * P + i) * q + t];
  if (mode != 2) {
    for (int k = 0; k < kb; ++k) {
      const cplx u = ub[(int64_t)t * kb + k];
#pragma unroll
      for (int i = 0; i < kMaxP; ++i)
        if (i < P) y[i] = csub(y[i], cmul(s_c[i * kb + k], u));
    }
  }
  if (spatial) {
    for (int al = 0; al < ka; ++al) {
      cplx alpha = cmk(0, 0);
#pragma unroll
      for (int i = 0; i < kMaxP; ++i)
        if (i < P) cfmca(alpha, s_ua[i * ka + al], y[i]);
#pragma unroll
      for (int i = 0; i < kMaxP; ++i)
        if (i < P) y[i] = csub(y[i], cmul(s_ua[i * ka + al], alpha));
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxP; ++i)
    if (i < P) out[(m * P + i) * q + t] = y[i];
  }
}

#define KST_DISPATCH_P4(P, ...)                           \
  switch (P) {                                            \
    case 1: { constexpr int PP = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int PP = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int PP = 3; __VA_ARGS__; } break; \
    default: { constexpr int PP = 4; __VA_ARGS__; } break; \
  }

// ---------------------------------------------------------------- fused per-bin detection
// Uniform Doppler grid, q <= D, P <= 4, radices in {2, 3, 4, 5, 7, 11, 13, 23,
// 29}: persistent CTAs (one per SM) walk the range bins. A bin's P channel
// rows are staged in smem by bulk async copies (the next bin's rows are
// prefetched into the free ping-pong buffer while this bin's pixels are
// formed), transformed together by a multi-row Stockham FFT (every stage
// has P x more independent butterflies than a one-row CTA), the temporal
// coefficients come from Parseval on the spectra,
//   c_ik = sum_t x_i[t] conj(U_B[t,k]) = (1/D) sum_d X_i[d] conj(U^_k[d])
// (exact identity for the zero-padded length-D transform), and the per-pixel
// projection, spatial candidates and max run straight from smem: the spectra
// never round-trip through HBM and one launch replaces two.
#ifndef KST_FB_NT
#define KST_FB_NT 512
#endif
constexpr int FB_NT = KST_FB_NT;
constexpr int FB_MAXP = 4;
constexpr int FB_MAXKB = 4;
constexpr int FB_MAXG = 64;
#ifndef KST_FB_PDT
#define KST_FB_PDT 2
#endif
constexpr int FB_PDT = KST_FB_PDT;  // Parseval: d values per thread with loads in flight

struct FusedArgs {
  int P, q, D, ka, kb, G, groups, mode, spatial;
  double inv_sqrt_q, inv_D;
  // dft = 1: the spatial grid is make_spatial_grid(P, G) (src/filters.py:208-217)
  // with G % 4 == 0, so z_g = (1/sqrt P) sum_i y_i W^{g i}, W = e^{-2 pi i/G},
  // splits as g = g0 + (G/4) g1 into twiddles W^{g0 i} and a 4-point DFT over
  // i; w4[g0][i] = W^{g0 i}, scale = 1/sqrt(P q)
  int dft;
  double scale;
  double w4[FB_MAXG / 4][FB_MAXP][2];
};

// sums v[0..31] over the warp; lane l returns the warp total of value l
// (transposing butterfly: 31 exchanges instead of 32 x 5)
__device__ __forceinline__ double warp_transpose_reduce32(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const double send = up ? v[j] : v[j + o];
      const double keep = up ? v[j + o] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

// radix-R Stockham stage over P rows (row stride D): small radices in registers
template <int R>
__device__ __forceinline__ void mr_stage_small(const cplx* __restrict__ a, cplx* __restrict__ b,
                                               const cplx* __restrict__ w, int D, int Ns, int P) {
  const int DR = D / R, step = D / (Ns * R);
  for (int it = threadIdx.x; it < P * DR; it += FB_NT) {
    const int row = it / DR, j = it - row * DR;
    const cplx* ar = a + (size_t)row * D;
    cplx* br = b + (size_t)row * D;
    const int k = j % Ns, dst = (j / Ns) * Ns * R + k;
    cplx t[R];
    t[0] = ar[j];
#pragma unroll
    for (int r = 1; r < R; ++r) t[r] = cmul(ar[j + r * DR], w[r * k * step]);
    if (R == 2) {
      br[dst] = cadd(t[0], t[1]);
      br[dst + Ns] = csub(t[0], t[1]);
    } else if (R == 4) {
      const cplx s02 = cadd(t[0], t[2]), d02 = csub(t[0], t[2]);
      const cplx s13 = cadd(t[1], t[3]), d13 = csub(t[1], t[3]);
      br[dst] = cadd(s02, s13);
      br[dst + Ns] = cmk(d02.x + d13.y, d02.y - d13.x);
      br[dst + 2 * Ns] = csub(s02, s13);
      br[dst + 3 * Ns] = cmk(d02.x - d13.y, d02.y + d13.x);
    } else {
      constexpr int h = (R - 1) / 2, off = rtw_off(R);
#pragma unroll
      for (int r = 1; r <= h; ++r) {
        const cplx sr = cadd(t[r], t[R - r]), dr = csub(t[r], t[R - r]);
        t[r] = sr;
        t[R - r] = dr;
      }
      cplx x0 = t[0];
#pragma unroll
      for (int r = 1; r <= h; ++r) x0 = cadd(x0, t[r]);
      br[dst] = x0;
#pragma unroll
      for (int u = 1; u <= h; ++u) {
        double ax = t[0].x, ay = t[0].y, bx = 0.0, by = 0.0;
#pragma unroll
        for (int r = 1; r <= h; ++r) {
          const int m = (r * u) % R;
          const double wc = c_plan.rtw[2 * (off + m)], ws = c_plan.rtw[2 * (off + m) + 1];
          ax = fma(wc, t[r].x, ax);
          ay = fma(wc, t[r].y, ay);
          bx = fma(-ws, t[R - r].x, bx);
          by = fma(-ws, t[R - r].y, by);
        }
        br[dst + u * Ns] = cmk(ax + by, ay - bx);
        br[dst + (R - u) * Ns] = cmk(ax - by, ay + bx);
      }
    }
  }
}

// large odd radix over P rows: phase A (twiddled pairs in place, X_0 out),
// barrier, phase B (grouped output pairs, grp_unit per row)
template <int R, int GU>
__device__ void mr_stage_grp(cplx* __restrict__ a, cplx* __restrict__ b, const cplx* __restrict__ w,
                             int D, int Ns, int P) {
  constexpr int h = (R - 1) / 2, NGR = (h + GU - 1) / GU;
  const int DR = D / R, step = D / (Ns * R);
  for (int it = threadIdx.x; it < P * DR; it += FB_NT) {
    const int row = it / DR, j = it - row * DR;
    cplx* ar = a + (size_t)row * D;
    const int k = j % Ns, dst = (j / Ns) * Ns * R + k;
    cplx x0 = ar[j];
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const cplx tr = cmul(ar[j + r * DR], w[r * k * step]);
      const cplx tm = cmul(ar[j + (R - r) * DR], w[(R - r) * k * step]);
      const cplx sr = cadd(tr, tm);
      ar[j + r * DR] = sr;
      ar[j + (R - r) * DR] = csub(tr, tm);
      x0 = cadd(x0, sr);
    }
    b[(size_t)row * D + dst] = x0;
  }
  __syncthreads();
  for (int un = threadIdx.x; un < P * DR * NGR; un += FB_NT) {
    const int g = un / (P * DR), it = un - g * (P * DR);
    const int row = it / DR, j = it - row * DR;
    const cplx* ar = a + (size_t)row * D;
    cplx* br = b + (size_t)row * D;
    if (g == 0) grp_unit<R, GU, 0>(ar, br, j, DR, Ns);
    if (NGR > 1 && g == 1) grp_unit<R, GU, (NGR > 1 ? 1 : 0)>(ar, br, j, DR, Ns);
    if (NGR > 2 && g == 2) grp_unit<R, GU, (NGR > 2 ? 2 : 0)>(ar, br, j, DR, Ns);
  }
}

// P-row Stockham FFT, a -> (a or b); returns the buffer holding the spectra
__device__ cplx* mr_fft(cplx* a, cplx* b, const cplx* __restrict__ w, int D, int P) {
  int Ns = 1;
  for (int f = 0; f < c_plan.nf; ++f) {
    const int R = c_plan.radix[f];
    switch (R) {
      case 2: mr_stage_small<2>(a, b, w, D, Ns, P); break;
      case 3: mr_stage_small<3>(a, b, w, D, Ns, P); break;
      case 4: mr_stage_small<4>(a, b, w, D, Ns, P); break;
      case 5: mr_stage_small<5>(a, b, w, D, Ns, P); break;
      case 7: mr_stage_small<7>(a, b, w, D, Ns, P); break;
      case 11: mr_stage_grp<11, 5>(a, b, w, D, Ns, P); break;
      case 13: mr_stage_grp<13, 6>(a, b, w, D, Ns, P); break;
      case 23: mr_stage_grp<23, 4>(a, b, w, D, Ns, P); break;
      default: mr_stage_grp<29, 7>(a, b, w, D, Ns, P); break;
    }
    __syncthreads();
    cplx* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

__device__ __forceinline__ void fb_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t ad = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(ad), "r"(parity)
        : "memory");
}
// one thread: bulk-copy bin m's P rows (q entries each) to rows of length D at dst
__device__ __forceinline__ void fb_issue(const cplx* __restrict__ cube, int64_t m, int P, int q,
                                         int D, cplx* dst, uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
               "r"((uint32_t)(P * q * sizeof(cplx)))
               : "memory");
  for (int i = 0; i < P; ++i)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst + (size_t)i * D)),
        "l"(cube + (m * P + i) * q), "r"((uint32_t)(q * sizeof(cplx))), "r"(b)
        : "memory");
}

template <int PT>
__global__ void __launch_bounds__(FB_NT, 1) detect_bin_kernel(
    const cplx* __restrict__ cube, int64_t n, const cplx* __restrict__ w,
    const cplx* __restrict__ ubspec, const cplx* __restrict__ ua, const cplx* __restrict__ hconj,
    FusedArgs fa, double* __restrict__ values, int* __restrict__ nonfinite) {
  constexpr int P = PT, NC = P * FB_MAXKB;
  extern __shared__ __align__(128) unsigned char fb_smem[];
  const int D = fa.D, q = fa.q;
  cplx* buf0 = (cplx*)fb_smem;
  cplx* buf1 = buf0 + (size_t)P * D;
  __shared__ cplx s_ua[FB_MAXP * FB_MAXP];
  __shared__ cplx s_c[NC], s_e[NC];
  __shared__ cplx s_h[FB_MAXG * FB_MAXP];
  __shared__ cplx s_w4[FB_MAXG / 4 * FB_MAXP];
  __shared__ double red[FB_NT / 32][2 * NC];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int e = tid; e < P * fa.ka; e += FB_NT) s_ua[e] = ua[e];
  for (int e = tid; e < fa.G * P; e += FB_NT) s_h[e] = hconj[e];
  for (int e = tid; e < FB_MAXG / 4 * FB_MAXP; e += FB_NT)
    s_w4[e] = cmk(fa.w4[e / FB_MAXP][e % FB_MAXP][0], fa.w4[e / FB_MAXP][e % FB_MAXP][1]);
  if (tid == 0) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < n) fb_issue(cube, blockIdx.x, P, q, D, buf0, &bar);
  }
  cplx* in = buf0;
  cplx* other = buf1;
  uint32_t phase = 0;
  const int per = fa.G / fa.groups;
  for (int64_t m = blockIdx.x; m < n; m += gridDim.x, phase ^= 1u) {
    // zero padding [q, D) of the input rows (the FFT overwrote it last bin)
    for (int e = tid; e < P * (D - q); e += FB_NT) {
      const int i = e / (D - q), t = q + e % (D - q);
      in[(size_t)i * D + t] = cmk(0.0, 0.0);
    }
    __syncthreads();
    fb_mbar_wait(&bar, phase);
    if (nonfinite) {
      int bad = 0;
      for (int e = tid; e < P * q; e += FB_NT) {
        const cplx v = in[(size_t)(e / q) * D + e % q];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
      }
      if (bad) atomicOr(nonfinite, 1);
    }
    cplx* X = mr_fft(in, other, w, D, P);
    cplx* fr = (X == in) ? other : in;  // free buffer: prefetch the next bin
    if (tid == 0 && m + gridDim.x < n) fb_issue(cube, m + gridDim.x, P, q, D, fr, &bar);
    // coefficients by Parseval (fixed-order reduction: deterministic)
    if (fa.mode != 2) {
      double acc[2 * NC];
#pragma unroll
      for (int c = 0; c < 2 * NC; ++c) acc[c] = 0.0;
      // the basis spectra come from L2 (__ldcg: L1 keeps the twiddles): all
      // FB_PDT x kb loads of a chunk are issued before its FMAs, so the L2
      // latency is paid once per chunk, not once per d (same summation order)
      for (int d0 = tid; d0 < D; d0 += FB_PDT * FB_NT) {
        cplx u[FB_PDT][FB_MAXKB];
#pragma unroll
        for (int t = 0; t < FB_PDT; ++t)
#pragma unroll
          for (int k = 0; k < FB_MAXKB; ++k) {
            const int d = d0 + t * FB_NT;
            u[t][k] = (k < fa.kb && d < D) ? __ldcg(&ubspec[(int64_t)k * D + d]) : cmk(0.0, 0.0);
          }
#pragma unroll
        for (int t = 0; t < FB_PDT; ++t) {
          const int d = d0 + t * FB_NT;
          if (d >= D) break;
#pragma unroll
          for (int k = 0; k < FB_MAXKB; ++k) {
            if (k < fa.kb) {
#pragma unroll
              for (int i = 0; i < P; ++i) {
                cplx c = cmk(acc[2 * (i * FB_MAXKB + k)], acc[2 * (i * FB_MAXKB + k) + 1]);
                cfmac(c, X[(size_t)i * D + d], u[t][k]);
                acc[2 * (i * FB_MAXKB + k)] = c.x;
                acc[2 * (i * FB_MAXKB + k) + 1] = c.y;
              }
            }
          }
        }
      }
      const int wid = tid >> 5, lane = tid & 31;
      {
        double v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = (c < 2 * NC) ? acc[c] : 0.0;
        const double tot = warp_transpose_reduce32(v);
        if (lane < 2 * NC) red[wid][lane] = tot;
      }
      __syncthreads();
      if (tid < P * fa.kb) {
        const int i = tid / fa.kb, k = tid % fa.kb;
        double re = 0.0, im = 0.0;
        for (int w2 = 0; w2 < FB_NT / 32; ++w2) {
          re += red[w2][2 * (i * FB_MAXKB + k)];
          im += red[w2][2 * (i * FB_MAXKB + k) + 1];
        }
        s_c[i * fa.kb + k] = cmk(re * fa.inv_D, im * fa.inv_D);
      }
      __syncthreads();
      if (fa.mode == 1) {  // classical: E = U_A (U_A^H c)  (src/filters.py:115-116)
        if (tid < P * fa.kb) {
          const int i = tid / fa.kb, k = tid % fa.kb;
          cplx acc2 = cmk(0, 0);
          for (int al = 0; al < fa.ka; ++al) {
            cplx inner = cmk(0, 0);
            for (int j = 0; j < P; ++j) cfmca(inner, s_ua[j * fa.ka + al], s_c[j * fa.kb + k]);
            cfma(acc2, s_ua[i * fa.ka + al], inner);
          }
          s_e[tid] = acc2;
        }
        __syncthreads();
        if (tid < P * fa.kb) s_c[tid] = s_e[tid];
        __syncthreads();
      }
    }
    // per pixel: projection, spatial candidates, max |z|
    for (int d = tid; d < D; d += FB_NT) {
      cplx y[P];
#pragma unroll
      for (int i = 0; i < P; ++i) y[i] = X[(size_t)i * D + d];
      if (fa.mode != 2) {
        for (int k = 0; k < fa.kb; ++k) {
          const cplx u = __ldcg(&ubspec[(int64_t)k * D + d]);  // L2 only: L1 keeps the twiddles
#pragma unroll
          for (int i = 0; i < P; ++i) y[i] = csub(y[i], cmul(s_c[i * fa.kb + k], u));
        }
      }
      if (fa.spatial) {
        for (int al = 0; al < fa.ka; ++al) {
          cplx alpha = cmk(0, 0);
#pragma unroll
          for (int i = 0; i < P; ++i) cfmca(alpha, s_ua[i * fa.ka + al], y[i]);
#pragma unroll
          for (int i = 0; i < P; ++i) y[i] = csub(y[i], cmul(s_ua[i * fa.ka + al], alpha));
        }
      }
      if (fa.dft) {
        // max_g |z_g|^2 via g = g0 + (G/4) g1: t_i = y_i W^{g0 i}, then the
        // 4-point DFT over i in pairs, max(|a + c|^2, |a - c|^2) =
        // |a|^2 + |c|^2 + 2 |Re(a conj c)| (a = t0 + t2, c = t1 + t3) and
        // max(|b - ie|^2, |b + ie|^2) = |b|^2 + |e|^2 + 2 |Im(b conj e)|
        double best2 = 0.0;
        const int G4 = fa.G >> 2;
        for (int g0 = 0; g0 < G4; ++g0) {
          cplx t[4];
          t[0] = y[0];
#pragma unroll
          for (int i = 1; i < 4; ++i)
            t[i] = (i < P) ? cmul(y[i], s_w4[g0 * FB_MAXP + i]) : cmk(0.0, 0.0);
          const cplx a = cadd(t[0], t[2]), b = csub(t[0], t[2]);
          const cplx c = (P > 3) ? cadd(t[1], t[3]) : t[1];
          const cplx e = (P > 3) ? csub(t[1], t[3]) : t[1];
          const double aa = fma(a.x, a.x, a.y * a.y), bb = fma(b.x, b.x, b.y * b.y);
          const double cc = fma(c.x, c.x, c.y * c.y);
          const double ee = (P > 3) ? fma(e.x, e.x, e.y * e.y) : cc;
          const double re = fma(a.x, c.x, a.y * c.y), im = fma(b.y, e.x, -b.x * e.y);
          best2 = fmax(best2, fma(2.0, fabs(re), aa + cc));
          best2 = fmax(best2, fma(2.0, fabs(im), bb + ee));
        }
        values[m * D + d] = sqrt(best2) * fa.scale;
        continue;
      }
      for (int gr = 0; gr < fa.groups; ++gr) {
        double best2 = -1.0;
        cplx zb = cmk(0, 0);
        for (int g = gr * per; g < (gr + 1) * per; ++g) {
          cplx z = cmk(0, 0);
#pragma unroll
          for (int i = 0; i < P; ++i) cfma(z, s_h[g * P + i], y[i]);
          const double m2 = cabs2(z);
          if (m2 > best2) {
            best2 = m2;
            zb = z;
          }
        }
        values[((int64_t)gr * n + m) * D + d] = hypot(zb.x * fa.inv_sqrt_q, zb.y * fa.inv_sqrt_q);
      }
    }
    __syncthreads();  // X and the coefficient smem are free for the next bin
    in = fr;
    other = X;
  }
}

// host: is grid[g, i] = exp(2 pi i (g / G) i) / sqrt(p) (make_spatial_grid,
// src/filters.py:208-217) to within rounding (numpy rounds the phase
// 2 pi (g / G) i before exp: ~1e-15 absolute; 1e-12 separates the uniform
// grid from any other while staying far inside the map tolerance)
bool dft_grid(const cplx* grid, int G, int p) {
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double s = 1.0L / sqrtl((long double)p);
  for (int g = 0; g < G; ++g)
    for (int i = 0; i < p; ++i) {
      const long double th = 2.0L * pi * ((long double)g / G) * i;
      const long double dx = (long double)grid[g * p + i].x - s * cosl(th);
      const long double dy = (long double)grid[g * p + i].y - s * sinl(th);
      if (fabsl(dx) > 1e-12L || fabsl(dy) > 1e-12L) return false;
    }
  return true;
}

// host: can the fused kernel take this problem
bool fused_ok(const Plan& plan, int P, int q, int D, int kb, int G) {
  if (P > FB_MAXP || q > D || kb > FB_MAXKB || G > FB_MAXG) return false;
  if ((size_t)2 * P * D * sizeof(cplx) > 200 * 1024) return false;
  for (int f = 0; f < plan.nf; ++f) {
    const int R = plan.radix[f];
    if (R != 2 && R != 3 && R != 4 && R != 5 && R != 7 && R != 11 && R != 13 && R != 23 && R != 29)
      return false;
  }
  return true;
}

// filter semantics -> (mode, spatial) (src/filters.py:98-116)
// mode 0: temporal projection coefficients, 1: joint (classical), 2: none
void filter_mode(int kind, bool has_a, bool has_b, int spatial_only, int& mode, int& spatial) {
  mode = 2;
  spatial = 0;
  if (kind == KST_KIND_KRON) {
    mode = (has_b && !spatial_only) ? 0 : 2;
    spatial = has_a ? 1 : 0;
  } else if (has_a) {
    if (spatial_only) spatial = 1;
    else if (has_b) mode = 1;
  }
}

int plan_factors(int D, Plan& p) {
  p = Plan{};  // every byte defined: const_upload compares the whole struct
  p.D = D;
  p.nf = 0;
  int x = D;
  while (x % 4 == 0) {
    p.radix[p.nf++] = 4;
    x /= 4;
  }
  while (x % 2 == 0) {
    p.radix[p.nf++] = 2;
    x /= 2;
  }
  for (int f = 3; (int64_t)f * f <= x; f += 2)
    while (x % f == 0) {
      p.radix[p.nf++] = f;
      x /= f;
    }
  if (x > 1) p.radix[p.nf++] = x;
  for (int R : kRegRadix)
    for (int m = 0; m < R; ++m) {
      const long double th = 2.0L * 3.141592653589793238462643383279502884L * m / R;
      p.rtw[2 * (rtw_off(R) + m)] = (double)cosl(th);
      p.rtw[2 * (rtw_off(R) + m) + 1] = (double)-sinl(th);
    }
  return p.nf <= kMaxFactors;
}

}  // namespace

namespace kst {

int detect(kst_ctx* ctx, const cplx* cube, int64_t n, int p, int q, const cplx* ua, int ka,
           const cplx* ub, int kb, int kind, int spatial_only, const double* dop_host, int D,
           const cplx* grid_host, int G, int groups, double* values, cudaStream_t st,
           bool check_finite) {
  if (p < 1 || q < 1 || D < 1 || G < 1 || groups < 1 || G % groups)
    return set_err(ctx, KST_ERR_DIMENSION, "detect: bad shape p=%d q=%d D=%d G=%d groups=%d", p, q,
                   D, G, groups);
  if (p > kMaxP) return set_err(ctx, KST_ERR_DIMENSION, "detect: p=%d exceeds %d", p, kMaxP);
  if (ka < 0 || ka > p || kb < 0 || kb > std::min(q, kMaxKB))
    return set_err(ctx, KST_ERR_DIMENSION, "detect: basis widths ka=%d kb=%d unsupported", ka, kb);
  if (n == 0) return KST_OK;
  const bool has_a = ua && ka > 0, has_b = ub && kb > 0;
  int mode = 2, spatial = 0;
  filter_mode(kind, has_a, has_b, spatial_only, mode, spatial);
  const int kb_used = (mode == 2) ? 0 : kb;
  bool uniform = true;
  for (int d = 0; d < D && uniform; ++d) uniform = dop_host[d] == (double)d / (double)D;
  Plan plan{};
  if (uniform && (!plan_factors(D, plan) || (size_t)3 * D * sizeof(cplx) > 200 * 1024)) uniform = false;
  if (!uniform && (size_t)q * sizeof(cplx) > 200 * 1024)
    return set_err(ctx, KST_ERR_DIMENSION, "detect: q=%d too long for the direct-sum path", q);

  const int64_t rows = n * p;
  // fused per-bin kernel (no spectra in HBM) when the plan fits it
  FusedArgs fa;
  static const bool fused_on = !(getenv("KST_DET_FUSED") && atoi(getenv("KST_DET_FUSED")) == 0);
  // FP32 prime-factor kernel (detect_f32.cu) at det_bits = 32, else the FP64 kernels
  const bool f32 = uniform && ctx->det_bits == 32 && groups == 1 &&
                   detect_f32_supported(p, q, has_a ? ka : 0, kb_used, mode, spatial, D, G);
  const bool fused = !f32 && uniform && fused_on && fused_ok(plan, p, q, D, kb_used, G);
  const int64_t srows = (fused || f32) ? 0 : rows;  // spectra / coefficient rows in HBM
  // workspace: spec (srows x D), coef (srows x kb), ubspec (kb x D), ubT (kb x q),
  // twiddles (D), hconj (G x p), dop (D), flag (2), perm (D)
  const size_t bytes = sizeof(cplx) * ((size_t)srows * D + (size_t)srows * std::max(kb_used, 1) +
                                       (size_t)std::max(kb_used, 1) * (D + q) + D + (size_t)G * p) +
                       sizeof(double) * D + sizeof(int) * (D + 4) + 256;
  char* base = (char*)ws_get(ctx, WS_DET, bytes);
  cplx* hstage = (cplx*)pinned_get(ctx, sizeof(cplx) * (size_t)G * p + sizeof(double) * D +
                                            sizeof(int) * D + 64);
  if (!base || !hstage) return set_err(ctx, KST_ERR_CUDA, "detect: workspace");
  cplx* spec = (cplx*)base;
  cplx* coef = spec + (size_t)srows * D;
  cplx* ubspec = coef + (size_t)srows * std::max(kb_used, 1);
  cplx* ubT = ubspec + (size_t)std::max(kb_used, 1) * D;
  cplx* tw = ubT + (size_t)std::max(kb_used, 1) * q;
  cplx* hconj = tw + D;
  double* dop = (double*)(hconj + (size_t)G * p);
  int* flag = (int*)(dop + D);

  // conj(grid), Dopplers and the twiddle table stay resident in the
  // workspace: re-uploaded only when the grid, the layout or the buffer change
  std::vector<double> key;
  key.reserve(8 + D + 2 * (size_t)G * p);
  for (double v : {(double)D, (double)G, (double)p, (double)q, (double)kb_used, (double)uniform,
                   (double)srows, (double)fused})
    key.push_back(v);
  key.insert(key.end(), dop_host, dop_host + D);
  key.insert(key.end(), (const double*)grid_host, (const double*)grid_host + 2 * (size_t)G * p);
  if (ctx->det_base != base || ctx->det_key != key) {
    epoch_bump("detect tables", D);
    for (int e = 0; e < G * p; ++e) hstage[e] = cconj(grid_host[e]);
    double* hdop = (double*)(hstage + (size_t)G * p);
    for (int d = 0; d < D; ++d) hdop[d] = dop_host[d];
    KST_CUDA(ctx, cudaMemcpyAsync(hconj, hstage, sizeof(cplx) * G * p, cudaMemcpyHostToDevice, st));
    KST_CUDA(ctx, cudaMemcpyAsync(dop, hdop, sizeof(double) * D, cudaMemcpyHostToDevice, st));
    if (uniform) {
      twiddle_kernel<<<cdiv(D, 256), 256, 0, st>>>(tw, D);
      KST_LAUNCH(ctx);
    }
    // the staging buffer is reused by the next call: wait for the copies
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    ctx->det_base = base;
    ctx->det_key.swap(key);
  }
  if (uniform) KST_TRY(const_upload(ctx, (const void*)&c_plan, &plan, sizeof(Plan), st));
  if (check_finite) KST_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), st));
  const size_t smem = uniform ? sizeof(cplx) * (KST_RS_GTW ? 2 : 3) * D : sizeof(cplx) * q;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    KST_CUDA(ctx, cudaFuncSetAttribute(row_spectrum_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    configured = 226 * 1024;
  }
  if (kb_used > 0 && !f32) {  // (the FP32 kernel takes its basis spectra by a direct DFT)
    transpose_kernel<<<cdiv((int64_t)q * kb_used, 256), 256, 0, st>>>(ub, q, kb_used, ubT);
    KST_LAUNCH(ctx);
    // spectra of the temporal basis columns (coefficients unused)
    row_spectrum_kernel<<<kb_used, NTS, smem, st>>>(ubT, kb_used, q, nullptr, 0, tw, D, uniform, dop,
                                                   ubspec, nullptr, flag + 1);
    KST_LAUNCH(ctx);
  }
  if (f32) {
    const bool dft = G % 4 == 0 && dft_grid(grid_host, G, p);
    const int rc = detect_f32(ctx, cube, n, p, q, has_a ? ua : nullptr, has_a ? ka : 0, ub, kb_used,
                              mode, spatial, D, nullptr, tw, hconj, grid_host, G, dft, values,
                              check_finite ? flag : nullptr, st);
    if (rc != KST_OK) return rc == -1 ? set_err(ctx, KST_ERR_CUDA, "detect_f32: plan rejected") : rc;
  } else if (fused) {
    fa.P = p;
    fa.q = q;
    fa.D = D;
    fa.ka = has_a ? ka : 0;
    fa.kb = kb_used;
    fa.G = G;
    fa.groups = groups;
    fa.mode = mode;
    fa.spatial = spatial;
    fa.inv_sqrt_q = 1.0 / sqrt((double)q);
    fa.inv_D = 1.0 / (double)D;
    fa.dft = (groups == 1 && G % 4 == 0 && dft_grid(grid_host, G, p)) ? 1 : 0;
    fa.scale = 1.0 / sqrt((double)p * (double)q);
    for (int g0 = 0; g0 < FB_MAXG / 4; ++g0)
      for (int i = 0; i < FB_MAXP; ++i) {
        const long double th =
            -2.0L * 3.141592653589793238462643383279502884L * (long double)(g0 * i) / (long double)G;
        fa.w4[g0][i][0] = (double)cosl(th);
        fa.w4[g0][i][1] = (double)sinl(th);
      }
    const int fsm = (int)(2 * sizeof(cplx) * p * D);
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    KST_DISPATCH_P4(p, {
      static bool attr = false;
      if (!attr) {
        KST_CUDA(ctx, cudaFuncSetAttribute(detect_bin_kernel<PP>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
      }
      detect_bin_kernel<PP><<<(unsigned)std::min<int64_t>(n, nsm), FB_NT, fsm, st>>>(
          cube, n, tw, ubspec, has_a ? ua : hconj, hconj, fa, values,
          check_finite ? flag : nullptr);
    });
    KST_LAUNCH(ctx);
  } else {
  row_spectrum_kernel<<<(unsigned)rows, NTS, smem, st>>>(cube, rows, q, ub, kb_used, tw, D, uniform,
                                                        dop, spec, coef,
                                                        check_finite ? flag : nullptr);
  KST_LAUNCH(ctx);
  CombineArgs a;
  a.P = p;
  a.D = D;
  a.ka = has_a ? ka : 0;
  a.kb = kb_used;
  a.G = G;
  a.groups = groups;
  a.mode = mode;
  a.spatial = spatial;
  a.inv_sqrt_q = 1.0 / sqrt((double)q);
  KST_DISPATCH_P(p, (combine_kernel<PP><<<dim3(cdiv(D, NT), (unsigned)std::min<int64_t>(cdiv(n, CB_BINS), 65535)), NT,
                                          sizeof(cplx) * G * p, st>>>(
                        spec, coef, ubspec, has_a ? ua : hconj, hconj, a, values, n)));
  KST_LAUNCH(ctx);
  }
  if (!check_finite) return KST_OK;
  int hflag = 0;
  KST_CUDA(ctx, cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag) return set_err(ctx, KST_ERR_DATA, "bin matrix contains non-finite entries");
  return KST_OK;
}

// Unnormalised Doppler spectra of `rows` time rows (length q) at the D
// Doppler bins: spec[row][d] = sum_t x[t] e^{-2 pi i t f_d} -- the folded
// Stockham FFT on a uniform grid f_d = d / D, the direct
// sum with the reference's phase otherwise (src/filters.py:262-264). `consts`
// is caller-owned device scratch of D complex + D doubles (twiddles, grid).
// Used by the batched L-mode path (lmode.cu), whose per-bin projections act
// on these spectra.
int spectra(kst_ctx* ctx, const cplx* x, int64_t rows, int q, const double* dop_host, int D,
            cplx* spec, void* consts, cudaStream_t st) {
  if (rows == 0) return KST_OK;
  bool uniform = true;
  for (int d = 0; d < D && uniform; ++d) uniform = dop_host[d] == (double)d / (double)D;
  Plan plan{};
  if (uniform && (!plan_factors(D, plan) || (size_t)3 * D * sizeof(cplx) > 200 * 1024)) uniform = false;
  if (!uniform && (size_t)q * sizeof(cplx) > 200 * 1024)
    return set_err(ctx, KST_ERR_DIMENSION, "spectra: q=%d too long for the direct-sum path", q);
  cplx* tw = (cplx*)consts;
  double* dop = (double*)(tw + D);
  if (uniform) {
    twiddle_kernel<<<cdiv(D, 256), 256, 0, st>>>(tw, D);
    KST_LAUNCH(ctx);
    KST_TRY(const_upload(ctx, (const void*)&c_plan, &plan, sizeof(Plan), st));
  } else {
    KST_CUDA(ctx, cudaMemcpyAsync(dop, dop_host, sizeof(double) * D, cudaMemcpyHostToDevice, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));  // dop_host is pageable caller memory
  }
  const size_t smem = uniform ? sizeof(cplx) * (KST_RS_GTW ? 2 : 3) * D : sizeof(cplx) * q;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    KST_CUDA(ctx, cudaFuncSetAttribute(row_spectrum_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    configured = 226 * 1024;
  }
  row_spectrum_kernel<<<(unsigned)rows, NTS, smem, st>>>(x, rows, q, nullptr, 0, tw, D, uniform, dop,
                                                        spec, nullptr, nullptr);
  KST_LAUNCH(ctx);
  return KST_OK;
}

int filter_cube(kst_ctx* ctx, const cplx* cube, int64_t n, int p, int q, const cplx* ua, int ka,
                const cplx* ub, int kb, int kind, int spatial_only, cplx* out, cudaStream_t st) {
  if (p < 1 || q < 1 || p > kMaxP || ka < 0 || ka > p || kb < 0 || kb > std::min(q, kMaxKB))
    return set_err(ctx, KST_ERR_DIMENSION, "filter: unsupported shape p=%d q=%d ka=%d kb=%d", p, q,
                   ka, kb);
  if (n == 0) return KST_OK;
  const bool has_a = ua && ka > 0, has_b = ub && kb > 0;
  int mode = 2, spatial = 0;
  filter_mode(kind, has_a, has_b, spatial_only, mode, spatial);
  const int kb_used = mode == 2 ? 0 : kb;
  const int64_t rows = n * p;
  char* base = (char*)ws_get(ctx, WS_DET, sizeof(cplx) * (size_t)rows * std::max(kb_used, 1) + 256);
  if (!base) return set_err(ctx, KST_ERR_CUDA, "filter: workspace");
  ctx->det_base = nullptr;  // overwrites detect's resident grid / twiddles
  epoch_bump("filter", 0);
  cplx* coef = (cplx*)base;
  int* flag = (int*)(coef + (size_t)rows * std::max(kb_used, 1));
  KST_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), st));
  coef_kernel<<<(unsigned)rows, NT, 0, st>>>(cube, q, ub, kb_used, coef, flag);
  KST_LAUNCH(ctx);
  filter_apply_kernel<<<dim3(cdiv(q, NT), (unsigned)std::min<int64_t>(n, 65535)), NT, 0, st>>>(
      cube, coef, ub, has_a ? ua : coef, p, q, has_a ? ka : 0, kb_used, mode, spatial, out, n);
  KST_LAUNCH(ctx);
  int hflag = 0;
  KST_CUDA(ctx, cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  if (hflag) return set_err(ctx, KST_ERR_DATA, "bin matrix contains non-finite entries");
  return KST_OK;
}

}  // namespace kst

extern "C" int kst_filter(kst_ctx* ctx, const double* cube, int64_t n, int p, int q,
                          const double* ua, int ka, const double* ub, int kb, int kind,
                          int spatial_only, double* out, void* stream) {
  CTX_GUARD(ctx);
  return kst::filter_cube(ctx, (const cplx*)cube, n, p, q, (const cplx*)ua, ka, (const cplx*)ub, kb,
                          kind, spatial_only, (cplx*)out, (cudaStream_t)stream);
}

extern "C" int kst_change(kst_ctx* ctx, const double* a, const double* b, int64_t count,
                          int is_signed, double* out, void* stream) {
  CTX_GUARD(ctx);
  if (count <= 0) return KST_OK;
  change_kernel<<<cdiv(count, 256) > 4096 ? 4096 : cdiv(count, 256), 256, 0, (cudaStream_t)stream>>>(
      a, b, count, is_signed, out);
  KST_LAUNCH(ctx);
  return KST_OK;
}
