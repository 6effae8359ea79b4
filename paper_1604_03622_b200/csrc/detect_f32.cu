// K5, FP32 detection (default precision):
// FP64 estimation, FP32 transform. Same semantics as detect_bin_kernel
// (src/filters.py:243-275 over StapFilter.apply_matrix, src/filters.py:88-116)
// for single-map projection filters on a uniform Doppler grid f_d = d / D.
//
// Per range bin m (persistent CTAs walk the bins, two CTAs share an SM):
//  1. load pass (FP64): the bin's P channel rows are read once from HBM
//     (c128, coalesced, prefetched into L2 two bins ahead) and reduced to
//     NR = rank of the spatial projector rows y' = Q^H x, Q an orthonormal
//     basis of range(I - U_A U_A^H) (the spatial projection is y = Q y', so
//     the transform runs on NR < P rows); the temporal-projection
//     coefficients c_ak = sum_t y'_a[t] conj(U_B[t,k]) accumulate in FP64 in
//     the same pass; y' is stored as c64 in shared memory at its
//     prime-factor position;
//  2. length-D DFT in FP32 by the Good-Thomas prime-factor algorithm: D is a
//     product of coprime factors F_j (each <= 32, or a * b with a, b <= 32
//     done Cooley-Tukey inside the factor); the row is viewed as a
//     multi-dimensional array and every stage is a set of independent
//     in-place pencil DFTs of length <= 32 held in registers -- no twiddles
//     between coprime factors, exact W_R^m values from a per-stage table,
//     one barrier per stage; zero padding t in [q, D) is the input map;
//  3. per pixel: Y'_a[d] - sum_k c_ak U^_k[d], y = Q Y', the spatial
//     candidates and max |z|, written as float64.
// Software pipeline: the pixel pass of bin m and the load pass of the CTA's
// next bin share one loop (HBM loads in flight during pixel work), the
// transformed rows and coefficients are double-buffered.
//
// Arithmetic per pixel (P = 3, r = (1, 3), D = 2001 = 3 * 23 * 29): ~48 FP64
// FMA in the load pass, ~120 FP32 FMA of transform, ~90 FP32 FMA of pixel
// work; HBM: the c128 cube once (48 B/px) and the f64 map (8 B/px).
// Error: FP32 rounding of the transform relative to the bin's spectrum
// (measured: max |err| ~3e-8 M0, >200x inside the §8c comparator).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

#ifndef KST_F32_NT
#define KST_F32_NT 256
#endif
constexpr int F32_NT = KST_F32_NT;
#ifndef KST_F32_MINB
#define KST_F32_MINB 2
#endif
constexpr int F32_MAXP = 4;
constexpr int F32_MAXKB = 3;
constexpr int F32_MAXG = 64;
constexpr int F32_MAXDIM = 8;
constexpr int kPencils[] = {2, 3, 4, 5, 7, 8, 9, 11, 13, 16, 17, 19, 23, 25, 27, 29, 31, 32};

__host__ __device__ constexpr int pencil_h(int R) { return (R % 2) ? (R - 1) / 2 : R / 2 - 1; }

struct F32Stage {
  int R;      // pencil length
  int st;     // element stride of the pencil (product of later dims)
  int npen;   // pencils per row (D / R)
  int boff;   // offset of this stage's pencil bases in the base table
  int woff;   // offset of its h x h table W_R^{u r mod R} (u, r = 1..h)
  int twF;    // Cooley-Tukey factor F = a * b (0: none) ...
  int twst;   // ... stride and length of the partner dim a (k1 = (base / twst) % twlen)
  int twlen;
  int twoff;  // offset of W_F^m, m < F, in the Cooley-Tukey twiddle table
};
struct F32Plan {
  int D, nst, nbase, nw;
  F32Stage s[F32_MAXDIM];
};
__constant__ F32Plan c_f32;

struct F32Args {
  int P, q, D, kb, G, mode, dft, ka;
  float scalef;  // dft: 1 / sqrt(P q); generic: 1 / sqrt(q)
};
// spatial-DFT candidate twiddles W_G^{g0 i} (dft grid): constant bank, so the
// unrolled candidate loop reads them as immediate FFMA operands
__constant__ float c_w4[F32_MAXG / 4][F32_MAXP][2];

// In-place DFT of one pencil (R elements at base + r * st) in registers.
// Pairs: X_u = A - iB, X_{R-u} = A + iB with s_r = t_r + t_{R-r},
// d_r = t_r - t_{R-r}, A = t_0 [+ (-1)^u t_{R/2}] + sum cos s_r,
// B = sum sin d_r. The inputs stay in registers (r unrolled); the output
// loop over u is a runtime loop over rows of the shared-memory table
// wt[(u-1) h + (r-1)] = W_R^{u r mod R} = (cos, -sin) (warp-uniform
// addresses: broadcast reads). ctw (Cooley-Tukey b-dim stages):
// W_F^{r k1} = ctw[(r k1) mod F].
// W_R^m = (cos, -sin)(2 pi m / R), m < R, of the fixed plan's factors: with
// the output loop fully unrolled every twiddle is a constant-bank operand
__constant__ float2 c_w3[3], c_w23[23], c_w29[29];
template <int R>
__device__ __forceinline__ float2 cw(int m) {
  return R == 3 ? c_w3[m] : R == 23 ? c_w23[m] : c_w29[m];
}

template <int R, int ST = 0, bool CT = false>  // ST > 0: compile-time element stride (fixed
                                               // plans); CT: constant-bank twiddles, unrolled u
__device__ __forceinline__ void pencil(float2* __restrict__ a, int base, int st_rt,
                                       const float2* __restrict__ wt,
                                       const float2* __restrict__ ctw, int twF, int k1) {
  const int st = ST > 0 ? ST : st_rt;
  constexpr bool even = (R % 2) == 0;
  constexpr int h = pencil_h(R);
  float2 t[R];
#pragma unroll
  for (int r = 0; r < R; ++r) t[r] = a[base + r * st];
  if (twF) {
    int idx = 0;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      idx += k1;
      if (idx >= twF) idx -= twF;
      const float2 c = __ldg(&ctw[idx]);
      const float2 v = t[r];
      t[r] = make_float2(v.x * c.x - v.y * c.y, v.x * c.y + v.y * c.x);
    }
  }
#pragma unroll
  for (int r = 1; r <= h; ++r) {
    const float2 s = make_float2(t[r].x + t[R - r].x, t[r].y + t[R - r].y);
    const float2 d = make_float2(t[r].x - t[R - r].x, t[r].y - t[R - r].y);
    t[r] = s;
    t[R - r] = d;
  }
  {
    float2 x0 = t[0];
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      x0.x += t[r].x;
      x0.y += t[r].y;
    }
    if (even) {
      x0.x += t[R / 2].x;
      x0.y += t[R / 2].y;
    }
    a[base] = x0;
  }
  if (even) {  // X_{R/2} = t_0 + sum (-1)^r s_r + (-1)^{R/2} t_{R/2}
    float2 xn = t[0];
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const float sg = (r & 1) ? -1.0f : 1.0f;
      xn.x = fmaf(sg, t[r].x, xn.x);
      xn.y = fmaf(sg, t[r].y, xn.y);
    }
    const float sn = ((R / 2) & 1) ? -1.0f : 1.0f;
    xn.x = fmaf(sn, t[R / 2].x, xn.x);
    xn.y = fmaf(sn, t[R / 2].y, xn.y);
    a[base + (R / 2) * st] = xn;
  }
  if (CT) {  // same operations, twiddles from the constant bank
#pragma unroll
    for (int u = 1; u <= h; ++u) {
      float ax = t[0].x, ay = t[0].y, bx = 0.0f, by = 0.0f;
      if (even) {
        const float sg = (u & 1) ? -1.0f : 1.0f;
        ax = fmaf(sg, t[R / 2].x, ax);
        ay = fmaf(sg, t[R / 2].y, ay);
      }
#pragma unroll
      for (int r = 1; r <= h; ++r) {
        const float2 wm = cw<R>((u * r) % R);  // (cos, -sin)
        ax = fmaf(wm.x, t[r].x, ax);
        ay = fmaf(wm.x, t[r].y, ay);
        bx = fmaf(-wm.y, t[R - r].x, bx);
        by = fmaf(-wm.y, t[R - r].y, by);
      }
      a[base + u * st] = make_float2(ax + by, ay - bx);        // A - iB
      a[base + (R - u) * st] = make_float2(ax - by, ay + bx);  // A + iB
    }
    return;
  }
#pragma unroll 1
  for (int u = 1; u <= h; ++u) {
    float ax = t[0].x, ay = t[0].y, bx = 0.0f, by = 0.0f;
    if (even) {
      const float sg = (u & 1) ? -1.0f : 1.0f;
      ax = fmaf(sg, t[R / 2].x, ax);
      ay = fmaf(sg, t[R / 2].y, ay);
    }
    const float2* wr = wt + (u - 1) * h;
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const float2 wm = wr[r - 1];  // (cos, -sin)
      ax = fmaf(wm.x, t[r].x, ax);
      ay = fmaf(wm.x, t[r].y, ay);
      bx = fmaf(-wm.y, t[R - r].x, bx);
      by = fmaf(-wm.y, t[R - r].y, by);
    }
    a[base + u * st] = make_float2(ax + by, ay - bx);        // A - iB
    a[base + (R - u) * st] = make_float2(ax - by, ay + bx);  // A + iB
  }
}

// one stage over nr <= 3 rows (row stride D); pencil bases from the table
template <int R>
__device__ __forceinline__ void stage_rows(float2* buf, int nr, int D, const F32Stage& s,
                                           const uint16_t* bases, const float2* wt,
                                           const float2* __restrict__ ctw) {
  const int npen = s.npen, st = s.st;
  for (int wi = threadIdx.x; wi < nr * npen; wi += F32_NT) {
    const int row = (wi >= npen) + (wi >= 2 * npen), pn = wi - row * npen;
    const int base = bases[pn];
    const int k1 = s.twF ? (base / s.twst) % s.twlen : 0;
    pencil<R>(buf + (size_t)row * D, base, st, wt, ctw + s.twoff, s.twF, k1);
  }
}

// fixed-plan stage: R, stride and pencil count are compile-time constants, the
// pencil bases ((pn / ST) R ST + pn % ST) are computed, no Cooley-Tukey factor
template <int R, int ST, int NPEN>
__device__ __forceinline__ void stage_fixed(float2* buf, int nr, int D, const float2* wt) {
  for (int wi = threadIdx.x; wi < nr * NPEN; wi += F32_NT) {
    const int row = (wi >= NPEN) + (wi >= 2 * NPEN), pn = wi - row * NPEN;
    const int base = (pn / ST) * (R * ST) + pn % ST;
    pencil<R, ST, true>(buf + (size_t)row * D, base, ST, wt, nullptr, 0, 0);
  }
}

__device__ __forceinline__ void run_stage(float2* buf, int nr, int D, const F32Stage& s,
                                          const uint16_t* bases, const float2* wt,
                                          const float2* __restrict__ ctw) {
  const uint16_t* b = bases + s.boff;
  const float2* w = wt + s.woff;
  switch (s.R) {
#define KST_F32_CASE(RR) \
  case RR: stage_rows<RR>(buf, nr, D, s, b, w, ctw); break;
    KST_F32_CASE(2) KST_F32_CASE(3) KST_F32_CASE(4) KST_F32_CASE(5) KST_F32_CASE(7)
    KST_F32_CASE(8) KST_F32_CASE(9) KST_F32_CASE(11) KST_F32_CASE(13) KST_F32_CASE(16)
    KST_F32_CASE(17) KST_F32_CASE(19) KST_F32_CASE(23) KST_F32_CASE(25) KST_F32_CASE(27)
    KST_F32_CASE(29) KST_F32_CASE(31) KST_F32_CASE(32)
#undef KST_F32_CASE
    default: break;
  }
}

// lane l returns the warp total of value (l mod NV), NV a power of two
template <int NV>
__device__ __forceinline__ double warp_reduce_tr(double (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= NV; o >>= 1)
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
  for (int o = NV / 2; o >= 1; o >>= 1) {
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

// L2 prefetch of bin m's P rows (contiguous P q c128 in the (n, P, q) cube)
__device__ __forceinline__ void prefetch_bin(const cplx* cube, int64_t m, int P, int q) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cube + m * P * q),
               "r"((uint32_t)(P * q * sizeof(cplx)))
               : "memory");
}

// max over g1 of |z_{g0 + (G/4) g1}|^2 for the spatial DFT grid: t_i = y_i W^{g0 i},
// then the 4-point DFT over i in pairs (see detect_bin_kernel)
__device__ __forceinline__ float dft_cand(const float2 (&y)[F32_MAXP], int P, int g0,
                                          const F32Args& fa) {
  float2 t[4];
  t[0] = y[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    const float wx = c_w4[g0][i][0], wy = c_w4[g0][i][1];
    t[i] = (i < P) ? make_float2(y[i].x * wx - y[i].y * wy, y[i].x * wy + y[i].y * wx)
                   : make_float2(0.0f, 0.0f);
  }
  const float2 a = make_float2(t[0].x + t[2].x, t[0].y + t[2].y);
  const float2 b = make_float2(t[0].x - t[2].x, t[0].y - t[2].y);
  const float2 c = make_float2(t[1].x + t[3].x, t[1].y + t[3].y);
  const float2 e = make_float2(t[1].x - t[3].x, t[1].y - t[3].y);
  const float aa = fmaf(a.x, a.x, a.y * a.y), bb = fmaf(b.x, b.x, b.y * b.y);
  const float cc = fmaf(c.x, c.x, c.y * c.y), ee = fmaf(e.x, e.x, e.y * e.y);
  const float re = fmaf(a.x, c.x, a.y * c.y), im = fmaf(b.y, e.x, -b.x * e.y);
  return fmaxf(fmaf(2.0f, fabsf(re), aa + cc), fmaf(2.0f, fabsf(im), bb + ee));
}

// pixel d: Y'_a[d] - sum_k c_ak U^_k[d], y = Q Y', candidates, max |z| -> f64
template <int NR, int PF = 0>  // PF > 0: compile-time channel count
__device__ __forceinline__ void pixel(const float2* __restrict__ src, int D, int ps, int d,
                                      const float2 (&uf)[F32_MAXKB], const float2* cf,
                                      const float2* s_q, const float2* s_h, const F32Args& fa,
                                      double* __restrict__ vrow) {
  const int P = PF > 0 ? PF : fa.P, kb = PF > 0 ? F32_MAXKB : fa.kb;
  float2 yq[NR];
#pragma unroll
  for (int a = 0; a < NR; ++a) yq[a] = src[(size_t)a * D + ps];
#pragma unroll
  for (int k = 0; k < F32_MAXKB; ++k) {
    if (k < kb) {
#pragma unroll
      for (int a = 0; a < NR; ++a) {
        const float2 c = cf[a * F32_MAXKB + k];
        yq[a].x = fmaf(-c.x, uf[k].x, fmaf(c.y, uf[k].y, yq[a].x));
        yq[a].y = fmaf(-c.x, uf[k].y, fmaf(-c.y, uf[k].x, yq[a].y));
      }
    }
  }
  float2 y[F32_MAXP];
#pragma unroll
  for (int i = 0; i < F32_MAXP; ++i) {
    y[i] = make_float2(0.0f, 0.0f);
    if (i < P) {
#pragma unroll
      for (int a = 0; a < NR; ++a) {
        const float2 qq = s_q[i * NR + a];
        y[i].x = fmaf(qq.x, yq[a].x, fmaf(-qq.y, yq[a].y, y[i].x));
        y[i].y = fmaf(qq.x, yq[a].y, fmaf(qq.y, yq[a].x, y[i].y));
      }
    }
  }
  float best2 = 0.0f;
  if (fa.dft) {
    if (fa.G == 16) {
#pragma unroll
      for (int g0 = 0; g0 < 4; ++g0) best2 = fmaxf(best2, dft_cand(y, P, g0, fa));
    } else {
      for (int g0 = 0; g0 < (fa.G >> 2); ++g0) best2 = fmaxf(best2, dft_cand(y, P, g0, fa));
    }
  } else {
    for (int g = 0; g < fa.G; ++g) {
      float2 z = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < F32_MAXP; ++i) {
        if (i < P) {
          const float2 h = s_h[g * P + i];
          z.x = fmaf(h.x, y[i].x, fmaf(-h.y, y[i].y, z.x));
          z.y = fmaf(h.x, y[i].y, fmaf(h.y, y[i].x, z.y));
        }
      }
      best2 = fmaxf(best2, fmaf(z.x, z.x, z.y * z.y));
    }
  }
  vrow[d] = (double)(sqrtf(best2) * fa.scalef);
}

// One pass over t = d in [0, D): issue the HBM loads of bin `mload` (t < q),
// form pixel d of bin `mpix` from `src` meanwhile (its basis spectra loaded
// one iteration ahead), then reduce the loaded channels to y' = Q^H x
// (FP64), accumulate the temporal coefficients (FP64) and scatter y' (c64)
// into `dst` at the prime-factor input positions. Ends with a barrier (OR of
// the non-finite test).
template <int NR, int PF = 0>  // PF > 0: compile-time channel count
__device__ __forceinline__ void load_bin(
    const cplx* __restrict__ cube, int64_t mload, int P_rt, int q, int D, int kb,
    const cplx* __restrict__ ub, const double2* s_qh, const uint16_t* pos_in,
    const uint16_t* pos_out, float2* dst, double (&acc)[NR * F32_MAXKB][2], int64_t mpix,
    const float2* src, const float2* cf, const float2* s_q, const float2* s_h,
    const float2* __restrict__ ubf, const F32Args& fa, double* __restrict__ values,
    int* __restrict__ nonfinite) {
  constexpr int NC = NR * F32_MAXKB;
  const int P = PF > 0 ? PF : P_rt;
  if (PF > 0) kb = F32_MAXKB;  // the fixed plan also fixes k_B = 3
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c][0] = acc[c][1] = 0.0;
  int bad = 0;
  const cplx* xb = cube + (mload >= 0 ? mload : 0) * P * q;
  float2 ufn[F32_MAXKB];
#pragma unroll
  for (int k = 0; k < F32_MAXKB; ++k)
    ufn[k] = (mpix >= 0 && k < kb && (int)threadIdx.x < D) ? __ldg(&ubf[(size_t)k * D + threadIdx.x])
                                                           : make_float2(0.0f, 0.0f);
  for (int t = threadIdx.x; t < D; t += F32_NT) {
    const bool ld = mload >= 0 && t < q;
    cplx x[F32_MAXP], u[F32_MAXKB];
#pragma unroll
    for (int i = 0; i < F32_MAXP; ++i)
      x[i] = (ld && i < P) ? __ldcs(&xb[(size_t)i * q + t]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < F32_MAXKB; ++k)
      u[k] = (ld && k < kb) ? __ldg(&ub[(size_t)t * kb + k]) : make_double2(0.0, 0.0);
    if (mpix >= 0) {
      float2 uf[F32_MAXKB];
      const int tn = t + F32_NT;
#pragma unroll
      for (int k = 0; k < F32_MAXKB; ++k) {
        uf[k] = ufn[k];
        ufn[k] = (k < kb && tn < D) ? __ldg(&ubf[(size_t)k * D + tn]) : make_float2(0.0f, 0.0f);
      }
      pixel<NR, PF>(src, D, pos_out[t], t, uf, cf, s_q, s_h, fa, values + mpix * D);
    }
    if (mload < 0) continue;
    double2 yq[NR];
#pragma unroll
    for (int a = 0; a < NR; ++a) yq[a] = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < F32_MAXP; ++i) {
      if (i < P) {
#pragma unroll
        for (int a = 0; a < NR; ++a) {
          const double2 w = s_qh[a * F32_MAXP + i];
          yq[a].x = fma(w.x, x[i].x, fma(-w.y, x[i].y, yq[a].x));
          yq[a].y = fma(w.x, x[i].y, fma(w.y, x[i].x, yq[a].y));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < F32_MAXKB; ++k) {
      if (k < kb) {
#pragma unroll
        for (int a = 0; a < NR; ++a) {  // += y' conj(u)
          double* ac = acc[a * F32_MAXKB + k];
          ac[0] = fma(yq[a].x, u[k].x, fma(yq[a].y, u[k].y, ac[0]));
          ac[1] = fma(yq[a].y, u[k].x, fma(-yq[a].x, u[k].y, ac[1]));
        }
      }
    }
    // every x_i enters every y'_a (0 * NaN = NaN, 0 * Inf = NaN): a
    // non-finite input bin shows as a non-finite sum of y'
    double chk = 0.0;
#pragma unroll
    for (int a = 0; a < NR; ++a) chk += yq[a].x + yq[a].y;
    bad |= !isfinite(chk);
    const int ps = pos_in[t];
#pragma unroll
    for (int a = 0; a < NR; ++a) dst[(size_t)a * D + ps] = make_float2((float)yq[a].x, (float)yq[a].y);
  }
  if (__syncthreads_or(bad) && nonfinite && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

// coefficients: warp partials -> fixed-order sum over warps (deterministic);
// FP64 copy in s_c (classical transform), FP32 copy in cf
template <int NR, int NV>
__device__ __forceinline__ void reduce_coef(double (&acc)[NR * F32_MAXKB][2], double (*red)[NV],
                                            int kb, double* s_c, float2* cf) {
  constexpr int NC = NR * F32_MAXKB;
  if (kb == 0) return;
  const int tid = threadIdx.x;
  double v[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = (c < 2 * NC) ? acc[c >> 1][c & 1] : 0.0;
  const double tot = warp_reduce_tr<NV>(v);
  if ((tid & 31) < NV) red[tid >> 5][tid & 31] = tot;
  __syncthreads();
  if (tid < 2 * NC) {
    double sum = 0.0;
    for (int w = 0; w < F32_NT / 32; ++w) sum += red[w][tid];
    s_c[tid] = sum;
    ((float*)cf)[tid] = (float)sum;
  }
}

// classical kind: C <- U_A (U_A^H C) (src/filters.py:114-116), FP64
template <int NR>
__device__ __forceinline__ void classical_coef(const double* s_c, float2* cf, const double2* s_ua,
                                               int P, int ka, int kb) {
  __syncthreads();
  const int tid = threadIdx.x, i = tid / F32_MAXKB, k = tid % F32_MAXKB;
  if (tid < NR * F32_MAXKB && k < kb) {
    double2 e = make_double2(0.0, 0.0);
    for (int al = 0; al < ka; ++al) {
      double2 inner = make_double2(0.0, 0.0);
      for (int j = 0; j < P; ++j) {  // conj(U_A[j,al]) C[j,k]
        const double2 a = s_ua[j * ka + al];
        const double cx = s_c[2 * (j * F32_MAXKB + k)], cy = s_c[2 * (j * F32_MAXKB + k) + 1];
        inner.x += a.x * cx + a.y * cy;
        inner.y += a.x * cy - a.y * cx;
      }
      const double2 a = s_ua[i * ka + al];
      e.x += a.x * inner.x - a.y * inner.y;
      e.y += a.x * inner.y + a.y * inner.x;
    }
    cf[tid] = make_float2((float)e.x, (float)e.y);
  }
}

// Q (P x NR, orthonormal columns spanning range(I - U_A U_A^H), or I) by
// pivoted Gram-Schmidt on the projector's columns; one thread, FP64.
// qh = Q^H (NR x F32_MAXP, FP64), qf = Q (P x NR, FP32)
__global__ void f32_q_kernel(const cplx* __restrict__ ua, int P, int ka, int spat, int nr,
                             double2* __restrict__ qh, float2* __restrict__ qf) {
  if (threadIdx.x != 0) return;
  double2 pm[F32_MAXP][F32_MAXP];
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      double2 v = make_double2(i == j ? 1.0 : 0.0, 0.0);
      if (spat)
        for (int al = 0; al < ka; ++al) {  // - U_A[i,al] conj(U_A[j,al])
          const double2 a = ua[i * ka + al], b = ua[j * ka + al];
          v.x -= a.x * b.x + a.y * b.y;
          v.y -= a.y * b.x - a.x * b.y;
        }
      pm[i][j] = v;
    }
  for (int a = 0; a < nr; ++a) {
    int best = 0;
    double bn = -1.0;
    for (int j = 0; j < P; ++j) {
      double nn = 0.0;
      for (int i = 0; i < P; ++i) nn += pm[i][j].x * pm[i][j].x + pm[i][j].y * pm[i][j].y;
      if (nn > bn) {
        bn = nn;
        best = j;
      }
    }
    const double inv = bn > 0.0 ? 1.0 / sqrt(bn) : 0.0;
    double2 qa[F32_MAXP];
    for (int i = 0; i < P; ++i) qa[i] = make_double2(pm[i][best].x * inv, pm[i][best].y * inv);
    for (int j = 0; j < P; ++j) {  // pm -= q (q^H pm[:, j])
      double2 dot = make_double2(0.0, 0.0);
      for (int i = 0; i < P; ++i) {
        dot.x += qa[i].x * pm[i][j].x + qa[i].y * pm[i][j].y;
        dot.y += qa[i].x * pm[i][j].y - qa[i].y * pm[i][j].x;
      }
      for (int i = 0; i < P; ++i) {
        pm[i][j].x -= qa[i].x * dot.x - qa[i].y * dot.y;
        pm[i][j].y -= qa[i].x * dot.y + qa[i].y * dot.x;
      }
    }
    for (int i = 0; i < F32_MAXP; ++i) {
      qh[a * F32_MAXP + i] = i < P ? make_double2(qa[i].x, -qa[i].y) : make_double2(0.0, 0.0);
      if (i < P) qf[i * nr + a] = make_float2((float)qa[i].x, (float)qa[i].y);
    }
  }
}

// Basis spectra for the FP32 transform straight from the time-domain basis:
// U^_k[d] = sum_t U_B[t, k] W_D^{t d} (uniform grid, exact index t d mod D
// into the FP64 twiddle table), FP64 sums rounded once to c64. CTA = 16
// Dopplers x 32 pulse chunks, the chunks summed in fixed order (replaces the
// transpose + one-CTA-per-row FFT + conversion: 3 launches, ~26 us).
constexpr int BD_D = 8, BD_C = 32;
__global__ void __launch_bounds__(BD_D * BD_C) f32_basis_dft_kernel(
    const cplx* __restrict__ ub, int kb, int q, const cplx* __restrict__ tw, int D,
    float2* __restrict__ ubf) {
  __shared__ cplx part[BD_C][BD_D];
  const int dl = threadIdx.x % BD_D, ch = threadIdx.x / BD_D;
  const int d = blockIdx.x * BD_D + dl, k = blockIdx.y;
  const int tl = (q + BD_C - 1) / BD_C, t0 = ch * tl, t1 = min(q, t0 + tl);
  cplx acc = cmk(0, 0);
  if (d < D) {
    // twiddles by rotation, w_{t+1} = w_t W^d, re-seeded from the exact
    // table every 16 pulses (a warp's table gathers hit 32 scattered
    // addresses: one per 16 steps instead of one per step); the rotation
    // error stays below 16 ulp of FP64, far under the c64 rounding of the sum
    const cplx step = tw[d];
    int idx = (int)(((int64_t)t0 * d) % D);
    const int d16 = (int)(((int64_t)16 * d) % D);
    for (int t = t0; t < t1; t += 16) {
      cplx w = tw[idx];
      const int te = min(t1, t + 16);
      for (int u = t; u < te; ++u) {
        cfma(acc, ub[(size_t)u * kb + k], w);
        w = cmul(w, step);
      }
      idx += d16;
      if (idx >= D) idx -= D;
    }
  }
  part[ch][dl] = acc;
  __syncthreads();
  if (ch == 0 && d < D) {
    cplx s = part[0][dl];
    for (int c = 1; c < BD_C; ++c) s = cadd(s, part[c][dl]);
    ubf[(size_t)k * D + d] = make_float2((float)s.x, (float)s.y);
  }
}

__global__ void f32_spec_kernel(const cplx* __restrict__ in, float2* __restrict__ out, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = make_float2((float)in[i].x, (float)in[i].y);
}

// Dynamic shared memory: two NR x D c64 row buffers | W tables (nw c64) |
// pos_in, pos_out (D u16 each) | pencil bases (nbase u16).
// PL = 0: any plan (stages from c_f32); PL = 1: P = 3 channels, k_B = 3 and
// D = 2001 = 3 x 23 x 29 (the Gotcha frame), every stage, channel and basis
// loop a compile-time instantiation
template <int NR, int PL>
__global__ void __launch_bounds__(F32_NT, KST_F32_MINB) detect_f32_kernel(
    const cplx* __restrict__ cube, int64_t n, const cplx* __restrict__ ub,
    const float2* __restrict__ ubf, const cplx* __restrict__ ua, const cplx* __restrict__ hconj,
    const uint16_t* __restrict__ tab_u16, const float2* __restrict__ tab_w,
    const float2* __restrict__ ctw, const double2* __restrict__ qh_g,
    const float2* __restrict__ qf_g, F32Args fa, double* __restrict__ values,
    int* __restrict__ nonfinite) {
  constexpr int NC = NR * F32_MAXKB;  // coefficient count (complex)
  constexpr int NV = NC * 2 <= 8 ? 8 : NC * 2 <= 16 ? 16 : 32;
  extern __shared__ __align__(16) unsigned char f32_smem[];
  const int D = PL == 1 ? 2001 : fa.D, q = fa.q, P = PL == 1 ? 3 : fa.P,
            kb = PL == 1 ? F32_MAXKB : fa.kb;
  float2* buf = (float2*)f32_smem;
  float2* s_wt = buf + (size_t)2 * NR * D;
  uint16_t* pos_in = (uint16_t*)(s_wt + c_f32.nw);
  uint16_t* pos_out = pos_in + D;
  uint16_t* s_base = pos_out + D;
  __shared__ double2 s_qh[NR * F32_MAXP];
  __shared__ float2 s_q[F32_MAXP * NR];
  __shared__ double2 s_ua[F32_MAXP * F32_MAXP];
  __shared__ double s_c[2 * NC];
  __shared__ float2 s_cf[2][NC];
  __shared__ float2 s_h[F32_MAXG * F32_MAXP];
  __shared__ double red[F32_NT / 32][NV];
  const int tid = threadIdx.x;
  for (int e = tid; e < c_f32.nw; e += F32_NT) s_wt[e] = tab_w[e];
  for (int e = tid; e < 2 * D + c_f32.nbase; e += F32_NT) pos_in[e] = tab_u16[e];
  for (int e = tid; e < fa.G * P; e += F32_NT) {
    const cplx h = hconj[e];
    s_h[e] = make_float2((float)h.x, (float)h.y);
  }
  for (int e = tid; e < P * fa.ka; e += F32_NT) s_ua[e] = ua[e];
  for (int e = tid; e < NR * F32_MAXP; e += F32_NT) s_qh[e] = qh_g[e];
  for (int e = tid; e < P * NR; e += F32_NT) s_q[e] = qf_g[e];
  float2* bufs[2] = {buf, buf + (size_t)NR * D};
  const int64_t g = gridDim.x;
  int64_t m = blockIdx.x;
  if (tid == 0 && m < n) {
    prefetch_bin(cube, m, P, q);
    if (m + g < n) prefetch_bin(cube, m + g, P, q);
  }
  __syncthreads();
  if (m >= n) return;
  {  // prologue: bin m0 -> bufs[0]
    double acc[NC][2];
    load_bin<NR, PL == 1 ? 3 : 0>(cube, m, P, q, D, kb, ub, s_qh, pos_in, pos_out, bufs[0], acc,
                                  -1, nullptr, s_cf[0], s_q, s_h, ubf, fa, values, nonfinite);
    reduce_coef<NR, NV>(acc, red, kb, s_c, s_cf[0]);
  }
  int cur = 0;
  for (;; m += g, cur ^= 1) {
    if (fa.mode == 1) classical_coef<NR>(s_c, s_cf[cur], s_ua, P, fa.ka, kb);
    if (PL == 1) {  // prime-factor DFT of bin m (FP32), 2001 = 3 x 23 x 29
      stage_fixed<3, 667, 667>(bufs[cur], NR, 2001, s_wt + c_f32.s[0].woff);
      __syncthreads();
      stage_fixed<23, 29, 87>(bufs[cur], NR, 2001, s_wt + c_f32.s[1].woff);
      __syncthreads();
      stage_fixed<29, 1, 69>(bufs[cur], NR, 2001, s_wt + c_f32.s[2].woff);
      __syncthreads();
    } else {
      for (int s = 0; s < c_f32.nst; ++s) {  // prime-factor DFT of bin m (FP32)
        run_stage(bufs[cur], NR, D, c_f32.s[s], s_base, s_wt, ctw);
        __syncthreads();
      }
    }
    const int64_t mn = m + g;
    if (tid == 0 && mn + g < n) prefetch_bin(cube, mn + g, P, q);
    double acc[NC][2];
    // pixels of bin m (+ the load pass of bin mn when it exists)
    load_bin<NR, PL == 1 ? 3 : 0>(cube, mn < n ? mn : -1, P, q, D, kb, ub, s_qh, pos_in, pos_out,
                                  bufs[cur ^ 1], acc, m, bufs[cur], s_cf[cur], s_q, s_h, ubf, fa,
                                  values, nonfinite);
    if (mn >= n) break;
    reduce_coef<NR, NV>(acc, red, kb, s_c, s_cf[cur ^ 1]);
  }
}

int modinv(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  a %= m;
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return m == 1 ? 0 : -1;
}

bool pencil_ok(int R) {
  for (int r : kPencils)
    if (r == R) return true;
  return false;
}

// D -> stages, the in/out position maps, the per-stage pencil bases and W
// tables, and the Cooley-Tukey twiddles (Good-Thomas across coprime prime
// powers, Cooley-Tukey a x b inside a factor above 32)
struct CachedPlan {
  bool ok = false;
  F32Plan plan{};
  std::vector<uint16_t> u16;  // pos_in (D), pos_out (D), bases (nbase)
  std::vector<float2> w;      // per-stage W tables (nw)
  std::vector<float2> ctw;    // Cooley-Tukey twiddles
};

bool f32_plan(int D, CachedPlan& cp) {
  F32Plan& pl = cp.plan;
  if (D < 2 || D > 65535) return false;
  std::vector<int> F;
  int x = D;
  for (int f = 2; f * f <= x; ++f)
    if (x % f == 0) {
      int pe = 1;
      while (x % f == 0) {
        x /= f;
        pe *= f;
      }
      F.push_back(pe);
    }
  if (x > 1) F.push_back(x);
  std::vector<std::pair<int, int>> ab;  // (a, b) per factor; b = 1: one pencil dim
  for (size_t j = 0; j < F.size(); ++j) {
    const int f = F[j];
    if (f <= 32) {
      if (!pencil_ok(f)) return false;
      ab.push_back({f, 1});
      continue;
    }
    int a = 0;
    for (int c = 32; c >= 2; --c)
      if (f % c == 0 && f / c <= 32 && pencil_ok(c) && pencil_ok(f / c)) {
        a = c;
        break;
      }
    if (!a) return false;
    ab.push_back({a, f / a});
  }
  std::vector<int> dims, fid, role;  // role 0: whole factor / a-dim, 1: b-dim
  for (size_t j = 0; j < F.size(); ++j) {
    dims.push_back(ab[j].first);
    fid.push_back((int)j);
    role.push_back(0);
    if (ab[j].second > 1) {
      dims.push_back(ab[j].second);
      fid.push_back((int)j);
      role.push_back(1);
    }
  }
  const int nd = (int)dims.size();
  if (nd > F32_MAXDIM) return false;
  std::vector<int> st(nd, 1);
  for (int i = nd - 2; i >= 0; --i) st[i] = st[i + 1] * dims[i + 1];
  pl.D = D;
  pl.nst = nd;
  cp.u16.assign(2 * (size_t)D, 0);
  cp.w.clear();
  cp.ctw.assign(1, make_float2(1.0f, 0.0f));
  const long double two_pi = 2.0L * 3.141592653589793238462643383279502884L;
  for (int i = 0; i < nd; ++i) {
    F32Stage& s = pl.s[i];
    const int R = dims[i], h = pencil_h(R);
    s.R = R;
    s.st = st[i];
    s.npen = D / R;
    s.boff = (int)cp.u16.size() - 2 * D;
    for (int pn = 0; pn < s.npen; ++pn)
      cp.u16.push_back((uint16_t)((pn / st[i]) * (R * st[i]) + pn % st[i]));
    s.woff = (int)cp.w.size();
    for (int u = 1; u <= h; ++u)
      for (int r = 1; r <= h; ++r) {
        const long double th = two_pi * ((u * r) % R) / R;
        cp.w.push_back(make_float2((float)cosl(th), (float)-sinl(th)));
      }
    s.twF = 0;
    s.twst = 1;
    s.twlen = 1;
    s.twoff = 0;
    if (role[i] == 1) {  // b-dim of a Cooley-Tukey factor: twiddle by W_F^{n2 k1}
      const int f = F[fid[i]];
      s.twF = f;
      s.twst = st[i - 1];
      s.twlen = dims[i - 1];
      s.twoff = (int)cp.ctw.size();
      for (int m = 0; m < f; ++m) {  // W_F^m = exp(-2 pi i m / F)
        const long double th = -two_pi * m / f;
        cp.ctw.push_back(make_float2((float)cosl(th), (float)sinl(th)));
      }
    }
  }
  if (cp.w.empty()) cp.w.push_back(make_float2(0.0f, 0.0f));
  pl.nbase = (int)cp.u16.size() - 2 * D;
  pl.nw = (int)cp.w.size();
  // position of x[t] (Ruritanian input map n_j = t (D/F_j)^-1 mod F_j) and of
  // X[d] (CRT output map k_j = d mod F_j); n_j = b n1 + n2, k_j = k1 + a k2
  std::vector<int> inv(F.size());
  for (size_t j = 0; j < F.size(); ++j) inv[j] = modinv((D / F[j]) % F[j], F[j]);
  for (int t = 0; t < D; ++t) {
    int pin = 0, pout = 0, di = 0;
    for (size_t j = 0; j < F.size(); ++j) {
      const int f = F[j], a = ab[j].first, b = ab[j].second;
      const int nj = (int)(((int64_t)t * inv[j]) % f);
      const int kj = t % f;
      if (b == 1) {
        pin += nj * st[di];
        pout += kj * st[di];
        di += 1;
      } else {
        pin += (nj / b) * st[di] + (nj % b) * st[di + 1];
        pout += (kj % a) * st[di] + (kj / a) * st[di + 1];
        di += 2;
      }
    }
    cp.u16[t] = (uint16_t)pin;
    cp.u16[D + t] = (uint16_t)pout;
  }
  return true;
}

// plans by D, per host thread (contexts are per thread)
const CachedPlan& cached_plan(int D) {
  static thread_local std::vector<std::pair<int, CachedPlan>> cache;
  for (auto& e : cache)
    if (e.first == D) return e.second;
  if (cache.size() > 16) cache.erase(cache.begin());
  cache.emplace_back(D, CachedPlan());
  CachedPlan& c = cache.back().second;
  c.ok = f32_plan(D, c);
  return c;
}

size_t f32_smem_bytes(const CachedPlan& cp, int nr, int D) {
  return sizeof(float2) * (2 * (size_t)nr * D + cp.plan.nw) +
         sizeof(uint16_t) * (2 * (size_t)D + cp.plan.nbase);
}

}  // namespace

namespace kst {

bool detect_f32_supported(int p, int q, int ka, int kb, int mode, int spatial, int D, int G) {
  if (p > F32_MAXP || kb > F32_MAXKB || G > F32_MAXG || q > D || ka > F32_MAXP) return false;
  const int nr = (mode == 1 || !spatial) ? p : p - ka;
  if (nr < 1 || nr > 3 || D < 2) return false;
  const CachedPlan& cp = cached_plan(D);
  return cp.ok && f32_smem_bytes(cp, nr, D) <= 100 * 1024;
}

// Returns KST_OK, an error, or -1 when the FP32 kernel does not take this
// problem (the caller runs the FP64 path).
int detect_f32(kst_ctx* ctx, const cplx* cube, int64_t n, int p, int q, const cplx* ua, int ka,
               const cplx* ub, int kb, int mode, int spatial, int D, const cplx* ubspec,
               const cplx* tw, const cplx* hconj, const cplx* grid_host, int G, bool dft,
               double* values, int* flag, cudaStream_t st) {
  (void)grid_host;
  if (!detect_f32_supported(p, q, ka, kb, mode, spatial, D, G)) return -1;
  const int nr = (mode == 1 || !spatial) ? p : p - ka;
  const CachedPlan& cp = cached_plan(D);
  const size_t smem = f32_smem_bytes(cp, nr, D);
  // workspace: u16 tables | W tables | CT twiddles | basis spectra (FP32) | Q
  auto al16 = [](size_t b) { return (b + 15) / 16 * 16; };
  const size_t b_u16 = al16(sizeof(uint16_t) * cp.u16.size());
  const size_t b_w = al16(sizeof(float2) * cp.w.size());
  const size_t b_ctw = al16(sizeof(float2) * cp.ctw.size());
  const size_t tab_bytes = b_u16 + b_w + b_ctw;
  const size_t b_ubf = al16(sizeof(float2) * (size_t)std::max(kb, 1) * D);
  const size_t b_q = sizeof(double2) * 4 * F32_MAXP + sizeof(float2) * F32_MAXP * 4;
  char* ws = (char*)ws_get(ctx, WS_DET32, tab_bytes + b_ubf + b_q);
  if (!ws) return set_err(ctx, KST_ERR_CUDA, "detect_f32: workspace");
  const uint16_t* u16_d = (const uint16_t*)ws;
  const float2* w_d = (const float2*)(ws + b_u16);
  const float2* ctw_d = (const float2*)(ws + b_u16 + b_w);
  float2* ubf = (float2*)(ws + tab_bytes);
  double2* qh = (double2*)(ws + tab_bytes + b_ubf);
  float2* qf = (float2*)(qh + 4 * F32_MAXP);
  if (ctx->f32_base != (const void*)ws || ctx->f32_D != D) {  // tables resident per (buffer, D)
    epoch_bump("f32 tables", D);
    char* hs = (char*)pinned_get(ctx, tab_bytes);
    if (!hs) return set_err(ctx, KST_ERR_CUDA, "detect_f32: pinned staging");
    memcpy(hs, cp.u16.data(), sizeof(uint16_t) * cp.u16.size());
    memcpy(hs + b_u16, cp.w.data(), sizeof(float2) * cp.w.size());
    memcpy(hs + b_u16 + b_w, cp.ctw.data(), sizeof(float2) * cp.ctw.size());
    KST_CUDA(ctx, cudaMemcpyAsync(ws, hs, tab_bytes, cudaMemcpyHostToDevice, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));  // staging buffer reused by later calls
    ctx->f32_base = ws;
    ctx->f32_D = D;
  }
  KST_TRY(const_upload(ctx, (const void*)&c_f32, &cp.plan, sizeof(F32Plan), st));
  if (kb > 0 && ubspec) {
    f32_spec_kernel<<<cdiv((int64_t)kb * D, 256), 256, 0, st>>>(ubspec, ubf, kb * D);
    KST_LAUNCH(ctx);
  } else if (kb > 0) {  // spectra straight from the basis (uniform grid twiddles)
    f32_basis_dft_kernel<<<dim3((unsigned)cdiv(D, BD_D), (unsigned)kb), BD_D * BD_C, 0, st>>>(
        ub, kb, q, tw, D, ubf);
    KST_LAUNCH(ctx);
  }
  const int spat = (mode != 1 && spatial && ka > 0) ? 1 : 0;
  f32_q_kernel<<<1, 32, 0, st>>>(ua ? ua : hconj, p, ka, spat, nr, qh, qf);
  KST_LAUNCH(ctx);
  F32Args fa;
  memset(&fa, 0, sizeof(fa));
  fa.P = p;
  fa.q = q;
  fa.D = D;
  fa.kb = kb;
  fa.G = G;
  fa.mode = mode;
  fa.ka = (mode == 1 || spatial) ? ka : 0;
  fa.dft = dft ? 1 : 0;
  fa.scalef = (float)(dft ? 1.0 / sqrt((double)p * (double)q) : 1.0 / sqrt((double)q));
  {
    float w4[F32_MAXG / 4][F32_MAXP][2];
    for (int g0 = 0; g0 < F32_MAXG / 4; ++g0)
      for (int i = 0; i < F32_MAXP; ++i) {
        const long double th = -2.0L * 3.141592653589793238462643383279502884L *
                               (long double)((g0 * i) % G) / (long double)G;
        w4[g0][i][0] = (float)cosl(th);
        w4[g0][i][1] = (float)sinl(th);
      }
    KST_TRY(const_upload(ctx, (const void*)&c_w4, w4, sizeof(w4), st));
  }
  {  // constant-bank twiddles of the fixed plan's factors (same values as the W tables)
    const long double two_pi = 2.0L * 3.141592653589793238462643383279502884L;
    float2 w3[3], w23[23], w29[29];
    auto fill = [&](float2* w, int R) {
      for (int m = 0; m < R; ++m) {
        const long double th = two_pi * m / R;
        w[m] = make_float2((float)cosl(th), (float)-sinl(th));
      }
    };
    fill(w3, 3);
    fill(w23, 23);
    fill(w29, 29);
    KST_TRY(const_upload(ctx, (const void*)&c_w3, w3, sizeof(w3), st));
    KST_TRY(const_upload(ctx, (const void*)&c_w23, w23, sizeof(w23), st));
    KST_TRY(const_upload(ctx, (const void*)&c_w29, w29, sizeof(w29), st));
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)nsm * KST_F32_MINB);
  // the Gotcha Doppler bank has a compile-time plan (stage order 3, 23, 29)
  static const bool fixed_on = !(getenv("KST_F32_FIXED") && atoi(getenv("KST_F32_FIXED")) == 0);
  const F32Plan& pl = cp.plan;
  const int PLv = (fixed_on && p == 3 && kb == F32_MAXKB && D == 2001 && pl.nst == 3 &&
                   pl.s[0].R == 3 && pl.s[0].st == 667 &&
                   pl.s[1].R == 23 && pl.s[1].st == 29 && pl.s[2].R == 29 && pl.s[2].st == 1)
                      ? 1
                      : 0;
  switch (nr * 2 + PLv) {
#define KST_F32_LAUNCH(NRR, PLL)                                                                 \
  case NRR * 2 + PLL: {                                                                          \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      KST_CUDA(ctx, cudaFuncSetAttribute(detect_f32_kernel<NRR, PLL>,                            \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024)); \
      attr = true;                                                                               \
    }                                                                                            \
    detect_f32_kernel<NRR, PLL><<<grid, F32_NT, smem, st>>>(cube, n, ub, ubf, ua ? ua : hconj,   \
                                                            hconj, u16_d, w_d, ctw_d, qh, qf, fa, \
                                                            values, flag);                        \
  } break;
    KST_F32_LAUNCH(1, 0)
    KST_F32_LAUNCH(2, 0)
    KST_F32_LAUNCH(3, 0)
    KST_F32_LAUNCH(1, 1)
    KST_F32_LAUNCH(2, 1)
    KST_F32_LAUNCH(3, 1)
#undef KST_F32_LAUNCH
  }
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace kst
