// K1 on the int8 tensor cores, modular form: the complex Gram
// S = (1/n) X^T conj(X) (`sample_covariance`, src/lrkron.py:53-78) by the
// Chinese remainder theorem over int8 residues (the "Ozaki scheme II" idea).
//
// Each column a is scaled by 2^(beta - E_a) (|x| < 2^E_a) and rounded to
// integers x' (|x'| <= 2^beta, real and imaginary parts separately). For N
// pairwise-coprime moduli m_i <= 256 (product P) the residues x' mod m_i fit
// int8, so per modulus two int8 GEMMs give exact int32 products
//     Re_i = [Xr Xi]^T [Xr Xi]   (K-stacked, depth 2n)      M_i = Xi^T Xr   (depth n)
// and the exact integer Gram entries follow from
//     V = sum_i c_i w_i - k P,   w_i = (P/m_i) ((P/m_i)^-1 mod m_i) < P,
//     c_i = Re_i mod m_i    (Im: c_i = (M_i[a,b] - M_i[b,a]) mod m_i),
//     k = round(sum_i c_i w_i / P)   (from the top chunk alone, see crt_finish).
// beta is the largest value with 2n 2^(2 beta) <= P/4, so |V| <= P/4 and V is
// the exact integer product; w_i and P are cut into 40-bit (<= 10 moduli) or
// 39-bit chunks so every chunk sum is exact in FP64 and V costs one or two
// roundings. The only error is rounding x to beta bits: ~n 2^-beta of
// max|x_a| max|x_b| (10 moduli, n = 2001: beta = 32; rounding, unlike slice
// truncation, is unbiased). N moduli cost 3N units of int8 GEMM depth-n work
// against 3 s(s+1)/2 for s slices (10 vs 21 at s = 6).
//
// S is exactly Hermitian with a real diagonal (Im V[a,a] = 0 by construction);
// non-finite columns poison their S entries with NaN (DataError upstream).
#include <cuda.h>  // CUtensorMap types; the encoder is fetched with cudaGetDriverEntryPoint

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gram_i8.cuh"

namespace {

using kst::i8::kNaNExpo;

constexpr int kMaxMod = 16;  // table size; 3 x 39-bit chunks bound the product P < 2^117: <= 14 used
constexpr int kMaxUsed = 14;
// pairwise coprime: 2^8, 3.5.17, 11.23, 251, 13.19, 241, 239, 233, 229, 227,
// 223, 7.31, 211, 199, 197, 193
constexpr int kModuli[kMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233,
                                  229, 227, 223, 217, 211, 199, 197, 193};
// device-side view (a select chain that folds to a constant in unrolled loops)
__host__ __device__ constexpr int modulus(int i) {
  return i == 0 ? 256 : i == 1 ? 255 : i == 2 ? 253 : i == 3 ? 251 : i == 4 ? 247 : i == 5 ? 241
       : i == 6 ? 239 : i == 7 ? 233 : i == 8 ? 229 : i == 9 ? 227 : i == 10 ? 223 : i == 11 ? 217
       : i == 12 ? 211 : i == 13 ? 199 : i == 14 ? 197 : 193;
}

// CRT weights cut into NCH chunks of CB bits: NCH = 2, CB = 40 while P < 2^80
// (<= 10 moduli), else NCH = 3, CB = 39 (P < 2^117).
__host__ __device__ constexpr int crt_nch(int nmod) { return nmod <= 10 ? 2 : 3; }
__host__ __device__ constexpr int crt_cb(int nmod) { return nmod <= 10 ? 40 : 39; }
struct CrtConst {
  double w[kMaxMod][3];  // w_i chunks, most significant first
  double p[3];           // P, same chunks
  double kscale;         // 2^CB / P: quotient estimate from the upper chunks
};
__constant__ CrtConst c_crt;

// ---------------------------------------------------------------- residues
// R[a][i][part][k] = x'[k,a] mod m_i (part 0 real, 1 imag), centred in
// [-(m-1)/2, (m-1)/2] for odd m and two's complement [-128, 127] for 256.
// CTA = 16 columns x 64 rows; phase 1 reads X coalesced over a and cuts each
// element into its 2N residue bytes (smem [i][part][a][k]); phase 2 writes
// every (a, i, part) row segment with 4-byte stores coalesced over k.
#ifndef KST_CR_SUB
#define KST_CR_SUB 1
#endif
constexpr int CR_A = 16, CR_K = 64, CR_KP = CR_K + 4, CR_SUB = KST_CR_SUB;

// (h 2^32 + mid 2^16 + lo - 2^48) mod m as an int8 in [-128, 127]; m is a
// compile-time constant after unrolling, so "% m" is a multiply-high sequence.
// UNSIGNED: the residue in [0, m) as a uint8 (tcgen05 kind::i8 with unsigned
// operands); else centred into [-128, 127] (cuBLAS signed int8 GEMMs).
template <bool UNSIGNED>
__device__ __forceinline__ uint8_t crt_residue8(int m, uint32_t h, uint32_t mid, uint32_t lo) {
  const uint32_t um = (uint32_t)m;
  const uint32_t c16 = 65536u % um, c32 = (c16 * c16) % um, c48 = (c32 * c16) % um;
  const uint32_t t = h * c32 + mid * c16 + lo + (um - c48);  // < 2^27, == x' mod m
  const uint32_t r = t % um;                                   // [0, m)
  if (UNSIGNED) return (uint8_t)r;
  return (uint8_t)(int8_t)(r >= 128u ? (int)r - m : (int)r);  // |r| <= 128
}

// NEG (two-SM tcgen05 path) adds a third part per modulus, -Xr' mod m.
template <int NM, bool UNSIGNED, bool NEG>
__global__ void __launch_bounds__(256) crt_residue_kernel(
    const cplx* __restrict__ X, int64_t n, int64_t npad, int64_t d, int64_t dpad,
    const int* __restrict__ expo, int beta, int8_t* __restrict__ R) {
  constexpr int NP = NEG ? 3 : 2;  // parts per modulus
  // smem [column][modulus, part][row]: a column's NM NP row segments are
  // contiguous, so phase 2's segment index maps to global memory with no
  // division; +4 bytes per column keeps phase 1's byte stores conflict-free
  constexpr int CC = NM * NP * CR_KP + 4;
  __shared__ __align__(16) int8_t sb[CR_A * CC];
  const int64_t a0 = (int64_t)blockIdx.x * CR_A;
  const int tid = threadIdx.x;
  const int c = tid & (CR_A - 1), r_first = tid / CR_A;
  constexpr int RPT = CR_K / (256 / CR_A);  // rows per thread per sub-block (4)
  const int64_t a = a0 + c;
  const int e = a < d ? expo[a] : 0;
  // 2^(beta - E) as two spliced factors (each a normal double); 0 for NaN columns
  const int sh = max(-2044, min(2046, beta - e)), h1 = sh / 2, h2 = sh - h1;
  const double s1 = (e == kNaNExpo) ? 0.0 : __longlong_as_double((long long)(h1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(h2 + 1023) << 52);
  const int lw = tid & 15;
  // CR_SUB consecutive 64-row sub-blocks per CTA; the next sub-block's X
  // values are loaded while the current one is cut and written
  cplx v[RPT];
  int64_t kb0 = (int64_t)blockIdx.y * CR_K * CR_SUB;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int64_t k = kb0 + r_first + j * (256 / CR_A);
    v[j] = (k < n && a < d) ? X[k * d + a] : cmk(0, 0);
  }
#pragma unroll 1
  for (int sub = 0; sub < CR_SUB; ++sub, kb0 += CR_K) {
    if (kb0 >= npad) break;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int r = r_first + j * (256 / CR_A);
      // x' = rint(x 2^(beta - E)), |x'| <= 2^48, read off the mantissa of
      // x + 1.5 2^52 (round to nearest even, FP64 adder only), then biased by
      // 2^48 and cut into 17 + 16 + 16 bits for 32-bit modular arithmetic
      const long long magic = 0x4338000000000000ll;
      const long long xr =
          __double_as_longlong(fma(v[j].x * s1, s2, 6755399441055744.0)) - magic;
      const long long xi =
          __double_as_longlong(fma(v[j].y * s1, s2, 6755399441055744.0)) - magic;
      const unsigned long long ur = (unsigned long long)(xr + (1ll << 48));
      const unsigned long long ui = (unsigned long long)(xi + (1ll << 48));
      const uint32_t hr = (uint32_t)(ur >> 32), mr = (uint32_t)(ur >> 16) & 0xFFFFu,
                     lr = (uint32_t)ur & 0xFFFFu;
      const uint32_t hi = (uint32_t)(ui >> 32), mi = (uint32_t)(ui >> 16) & 0xFFFFu,
                     li = (uint32_t)ui & 0xFFFFu;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        const uint8_t rr = crt_residue8<UNSIGNED>(modulus(i), hr, mr, lr);
        int8_t* sp = sb + c * CC + (i * NP) * CR_KP + r;
        sp[0] = (int8_t)rr;
        sp[CR_KP] = (int8_t)crt_residue8<UNSIGNED>(modulus(i), hi, mi, li);
        if (NEG) sp[2 * CR_KP] = (int8_t)(rr ? (uint8_t)(modulus(i) - rr) : (uint8_t)0);
      }
    }
    if (sub + 1 < CR_SUB) {  // prefetch the next sub-block
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t k = kb0 + CR_K + r_first + j * (256 / CR_A);
        v[j] = (k < n && a < d) ? X[k * d + a] : cmk(0, 0);
      }
    }
    __syncthreads();
    const int64_t k = kb0 + 4 * lw;
    if (k < npad) {  // npad is a multiple of 16: whole words only
      // segment seg = (column cc, modulus i, part): R row ((a0 + cc) NM + i) NP
      // + part = a0 NM NP + seg
      int8_t* dst = R + (size_t)a0 * NM * NP * npad + k;
      const int segs = (int)(dpad - a0 < CR_A ? dpad - a0 : CR_A) * NM * NP;
      for (int seg = tid >> 4; seg < segs; seg += 16) {
        const int cc = seg / (NP * NM), rem = seg - cc * (NP * NM);
        *(uint32_t*)(dst + (size_t)seg * npad) = *(const uint32_t*)&sb[cc * CC + rem * CR_KP + 4 * lw];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- reconstruction
// chunk sums s_j = sum_i c_i w_ij (exact) -> V = sum_i c_i w_i - k P with
// k = round(sum_i c_i w_i / P) estimated from all but the lowest chunk:
// (s_0 [2^CB + s_1]) 2^CB / P; the dropped chunk moves the quotient by
// < nmod 2^9 2^CB / P < 1e-8, far inside the |V| <= P/4 margin. |k| < 2 nmod,
// so every s_j - k P_j is exact; V costs NCH - 1 roundings.
template <int NCH>
__device__ __forceinline__ double crt_finish(double s0, double s1, double s2) {
  const double est = (NCH == 2) ? s0 : fma(s0, 549755813888.0, s1);
  const double k = rint(est * c_crt.kscale);
  s0 = fma(-k, c_crt.p[0], s0);
  s1 = fma(-k, c_crt.p[1], s1);
  if (NCH == 2) return fma(s0, 1099511627776.0, s1);  // 2^40
  s2 = fma(-k, c_crt.p[2], s2);
  const double t = fma(s0, 549755813888.0, s1);  // 2^39
  return fma(t, 549755813888.0, s2);
}

// v 2^sh / n: exact power-of-two scaling as two multiplications by spliced
// powers 2^(sh/2), 2^(sh - sh/2) (each a normal double for |sh| <= 2044), then
// the quotient by one Newton correction of v (1/n) (within an ulp of the
// correctly rounded v / n; no FP64 divide or ldexp per entry)
// |sh| > 1022 (extreme column scales): out of line, so the common path is
// not predicated through ldexp's instruction sequence
__device__ __noinline__ double crt_scale_far(double v, int sh, double dn, double rn) {
  const double x = ldexp(v, sh);
  const double q = x * rn;
  return fma(fma(-q, dn, x), rn, q);
}
__device__ __forceinline__ double crt_scale(double v, int sh, double dn, double rn) {
#ifdef KST_SCALE_SPLIT
  sh = max(-2044, min(2046, sh));
  const int h1 = sh >> 1, h2 = sh - h1;
  const double x = v * __longlong_as_double((long long)(h1 + 1023) << 52) *
                   __longlong_as_double((long long)(h2 + 1023) << 52);
#else  // measured faster (A/B, tools/ab_kernels.sh)
  if (sh < -1022 || sh > 1023) return crt_scale_far(v, sh, dn, rn);
  const double x = v * __longlong_as_double((long long)(sh + 1023) << 52);
#endif
  const double q = x * rn;
  return fma(fma(-q, dn, x), rn, q);
}

// S from the per-modulus int32 products (column-major, ld = dpad): CTA per
// (bi <= bj) pair of 32x32 tiles, writes S[a][b] and S[b][a] = conj.
template <int NM>
__global__ void __launch_bounds__(256, 2) crt_combine_kernel(
    const int32_t* __restrict__ GRe, const int32_t* __restrict__ GM, int64_t dpad, int64_t d,
    const int* __restrict__ expo, int beta, double dn, int T, cplx* __restrict__ S) {
  __shared__ uint8_t mt[NM][32][33];  // mt[i][j][l] = M_i[b0+j][a0+l] mod m_i
  __shared__ cplx vt[32][33];         // vt[j][l] = S[a0+j][b0+l]
  const double rn = 1.0 / dn;
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
  const int q4 = 4 * (tid & 7), r = tid >> 3;
  const size_t plane = (size_t)dpad * dpad;
  {  // transposed M block residues
    const size_t idx = (size_t)(b0 + q4) + (size_t)(a0 + r) * dpad;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const int m = modulus(i);
      const int4 v = *(const int4*)(GM + (size_t)i * plane + idx);
      const int u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int rr = u[c] % m;
        mt[i][q4 + c][r] = (uint8_t)(rr < 0 ? rr + m : rr);
      }
    }
  }
  __syncthreads();
  {
    const int64_t b = b0 + r;
    const size_t idx = (size_t)(a0 + q4) + (size_t)b * dpad;
    constexpr int NCH = crt_nch(NM);
    double re0[4], re1[4], re2[4], im0[4], im1[4], im2[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) re0[c] = re1[c] = re2[c] = im0[c] = im1[c] = im2[c] = 0.0;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const int m = modulus(i);
      const int4 vr = *(const int4*)(GRe + (size_t)i * plane + idx);
      const int4 vm = *(const int4*)(GM + (size_t)i * plane + idx);
      const int ur[4] = {vr.x, vr.y, vr.z, vr.w}, um[4] = {vm.x, vm.y, vm.z, vm.w};
      const double w0 = c_crt.w[i][0], w1 = c_crt.w[i][1], w2 = c_crt.w[i][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cre = ur[c] % m;  // (-m, m)
        int cim = um[c] % m;
        cim = (cim < 0 ? cim + m : cim) - (int)mt[i][r][q4 + c];  // (-m, m)
        const double dre = (double)cre, dim = (double)cim;
        re0[c] = fma(dre, w0, re0[c]);
        re1[c] = fma(dre, w1, re1[c]);
        im0[c] = fma(dim, w0, im0[c]);
        im1[c] = fma(dim, w1, im1[c]);
        if (NCH == 3) {
          re2[c] = fma(dre, w2, re2[c]);
          im2[c] = fma(dim, w2, im2[c]);
        }
      }
    }
    const int eb = (b < d) ? expo[b] : 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t a = a0 + q4 + c;
      const int ea = (a < d) ? expo[a] : 0;
      cplx v;
      if (ea == kNaNExpo || eb == kNaNExpo) {
        v = cmk(NAN, NAN);
      } else {
        const double vre = crt_finish<NCH>(re0[c], re1[c], re2[c]);
        const double vim = crt_finish<NCH>(im0[c], im1[c], im2[c]);
        const int sh = ea + eb - 2 * beta;
        v = cmk(crt_scale(vre, sh, dn, rn), crt_scale(vim, sh, dn, rn));
      }
      vt[q4 + c][r] = v;
    }
  }
  __syncthreads();
  for (int rr = ty; rr < 32; rr += 8) {
    {  // S[a0 + rr][b0 + tx]
      const int64_t a = a0 + rr, b = b0 + tx;
      if (a < d && b < d && (bi != bj || a <= b)) {
        const cplx v = vt[rr][tx];
        S[a * d + b] = (a == b) ? cmk(v.x, 0.0) : v;
      }
    }
    {  // S[b0 + rr][a0 + tx] = conj(S[a0 + tx][b0 + rr])
      const int64_t b = b0 + rr, a = a0 + tx;
      if (a < d && b < d && (bi != bj || a < b)) {
        const cplx v = vt[tx][rr];
        S[b * d + a] = cmk(v.x, -v.y);
      }
    }
  }
}

// ---------------------------------------------------------------- host constants
struct HostCrt {
  int nmod = 0;
  CrtConst c;
  double log2p = 0.0;
};

int modinv(int a, int m) {  // a^-1 mod m (a, m coprime)
  int t = 0, nt = 1, r = m, nr = a % m;
  while (nr) {
    const int q = r / nr;
    int tmp = t - q * nt;
    t = nt;
    nt = tmp;
    tmp = r - q * nr;
    r = nr;
    nr = tmp;
  }
  return t < 0 ? t + m : t;
}

const HostCrt& host_crt(int nmod) {
  static HostCrt cache[kMaxMod + 1];
  HostCrt& h = cache[nmod];
  if (h.nmod == nmod) return h;
  typedef unsigned __int128 u128;
  u128 P = 1;
  double lp = 0.0;
  for (int i = 0; i < nmod; ++i) {
    P *= (u128)kModuli[i];
    lp += std::log2((double)kModuli[i]);
  }
  const int nch = crt_nch(nmod), cb = crt_cb(nmod);
  const u128 mask = ((u128)1 << cb) - 1;
  auto chunks = [&](u128 v, double* out) {  // most significant chunk first
    out[2] = 0.0;
    for (int j = nch - 1; j >= 0; --j) {
      out[j] = (double)(unsigned long long)(j == 0 ? v : (v & mask));
      v >>= cb;
    }
  };
  for (int i = 0; i < kMaxMod; ++i) {
    if (i < nmod) {
      const int m = kModuli[i];
      const u128 Q = P / (u128)m;
      const int y = modinv((int)(Q % (u128)m), m);
      chunks(Q * (u128)y, h.c.w[i]);
    } else {
      h.c.w[i][0] = h.c.w[i][1] = h.c.w[i][2] = 0.0;
    }
  }
  chunks(P, h.c.p);
  h.c.kscale = std::ldexp(1.0, cb) / (double)P;  // units of the estimate: 2^CB
  h.log2p = lp;
  h.nmod = nmod;
  return h;
}

// Column exponents (i8::colmax_kernel semantics) with the rows split over
// CM_SLICES CTAs per 32-column block, so the pass has ~8x the CTAs in flight
// (the one-CTA-per-block form ran at 16 % occupancy, 3.2 TB/s). Each slice
// folds its exponent into code[a] by atomicMax on an order-preserving code
// (0 = all zero, E + 2048 otherwise, INT_MAX = non-finite); max is order
// independent, so the result is deterministic. The last slice to finish a
// block (counter) decodes it into expo. work = code (d ints) + counters.
constexpr int CM_SLICES = 8;
__global__ void __launch_bounds__(256) colmax_split_kernel(const cplx* __restrict__ X, int64_t n,
                                                           int64_t d, int* __restrict__ expo,
                                                           int* __restrict__ work) {
  __shared__ double sm[8][33];
  __shared__ int sb[8][33];
  __shared__ int last;
  int* code = work;
  int* cnt = work + d;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t a = blockIdx.x * 32 + tx;
  const int64_t per = (n + CM_SLICES - 1) / CM_SLICES;
  const int64_t k0 = blockIdx.y * per, k1 = min(n, k0 + per);
  double m = 0.0;
  int bad = 0;
  if (a < d) {
    int64_t k = k0 + ty;
    for (; k + 24 < k1; k += 32) {  // four independent loads in flight
      cplx v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(&X[(k + 8 * u) * d + a]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bad |= !isfinite(v[u].x) || !isfinite(v[u].y);
        m = fmax(m, fmax(fabs(v[u].x), fabs(v[u].y)));
      }
    }
    for (; k < k1; k += 8) {
      const cplx v = __ldcs(&X[k * d + a]);
      bad |= !isfinite(v.x) || !isfinite(v.y);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
  }
  sm[ty][tx] = m;
  sb[ty][tx] = bad;
  __syncthreads();
  if (ty == 0 && a < d) {
    for (int r = 1; r < 8; ++r) {
      m = fmax(m, sm[r][tx]);
      bad |= sb[r][tx];
    }
    const int c = bad ? INT_MAX : (m > 0.0 ? ilogb(m) + 1 + 2048 : 0);
    if (c) atomicMax(&code[a], c);
  }
  __threadfence();
  __syncthreads();
  if (tx == 0 && ty == 0) last = (atomicAdd(&cnt[blockIdx.x], 1) == CM_SLICES - 1);
  __syncthreads();
  if (last && ty == 0 && a < d) {
    __threadfence();
    const int c = atomicAdd(&code[a], 0);
    expo[a] = c == INT_MAX ? kNaNExpo : (c == 0 ? 0 : c - 2048);
  }
}

int colmax_split(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, int* expo, int* work,
                 cudaStream_t st) {
  KST_CUDA(ctx, cudaMemsetAsync(work, 0, sizeof(int) * ((size_t)d + cdiv(d, 32)), st));
  colmax_split_kernel<<<dim3(cdiv(d, 32), CM_SLICES), dim3(32, 8), 0, st>>>(X, n, d, expo, work);
  KST_LAUNCH(ctx);
  return KST_OK;
}

// parts: 2 = {Xr', Xi'} (signed for cuBLAS, unsigned for the single-CTA
// kernel), 3 = {Xr', Xi', -Xr'} unsigned (two-SM kernel)
template <int NM>
void launch_crt(const cplx* X, int64_t n, int64_t npad, int64_t d, int64_t dpad, const int* expo,
                int beta, int8_t* R, bool uns, int parts, cudaStream_t st) {
  const dim3 grid(cdiv(dpad, CR_A), cdiv(npad, CR_K * CR_SUB));
  if (parts == 3)
    crt_residue_kernel<NM, true, true><<<grid, 256, 0, st>>>(X, n, npad, d, dpad, expo, beta, R);
  else if (uns)
    crt_residue_kernel<NM, true, false><<<grid, 256, 0, st>>>(X, n, npad, d, dpad, expo, beta, R);
  else
    crt_residue_kernel<NM, false, false><<<grid, 256, 0, st>>>(X, n, npad, d, dpad, expo, beta, R);
}
template <int NM>
void launch_combine(const int32_t* GRe, const int32_t* GM, int64_t dpad, int64_t d, const int* expo,
                    int beta, double dn, cplx* S, cudaStream_t st) {
  const int T = (int)(dpad / 32);
  crt_combine_kernel<NM><<<(unsigned)(T * (T + 1) / 2), 256, 0, st>>>(GRe, GM, dpad, d, expo, beta,
                                                                      dn, T, S);
}

// ============================================================================
// Hand-written tcgen05 path (sm_100a): the per-modulus products and their
// modular reduction in one persistent kernel, no int32 planes.
//
// Work unit: an upper-triangle tile (I <= J) of 128 x 128 Gram entries. Per
// modulus i and K block (128 snapshots) one TMA stage brings four 16 KB
// operand tiles into smem (128B-swizzled, K-major):
//   Ar = Xr'_I, Ai = Xi'_I, Br = Xr'_J, Bi = Xi'_J       (residues mod m_i)
// and the MMA thread issues 16 tcgen05.mma.kind::i8 (M = N = 128, K = 32)
// into three TMEM accumulators (int32, 128 lanes x 384 columns):
//   Re += Ar.Br + Ai.Bi,   M += Ai.Br,   MT += Ar.Bi      (Im = M - MT)
// Every operand byte feeds two products (128 int8 MACs per smem byte, the
// same intensity as a 256 x 256 two-SM GEMM tile). After the last K block
// of a modulus the four epilogue warps drain TMEM (tcgen05.ld, one TMEM lane
// = one Gram row per thread), reduce Re and M - MT mod m_i and store uint8
// residues; the next modulus starts as soon as TMEM is read. A separate
// kernel then runs the CRT reconstruction on the residues (20 bytes per
// entry for 10 moduli instead of 120 bytes of int32 products).
//
// Warp roles (576 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2-17 = epilogue (warp w reads TMEM
// lanes 32 (w % 4) .. +31, columns 32 ((w - 2) / 4) .. +31). Pipelines: smem
// full/empty mbarriers (TMA <-> MMA, 3 stages of 64 KB), TMEM full/empty
// (MMA <-> epilogue).
constexpr int TC_BM = 128;                   // tile edge (rows = TMEM lanes, cols = N)
constexpr int TC_BK = 128;                   // K bytes per stage (one 128B swizzle row)
constexpr int TC_STAGES = 3;
constexpr int TC_OPER = TC_BM * TC_BK;       // 16 KB operand tile
constexpr int TC_STAGE_BYTES = 4 * TC_OPER;  // Ar, Ai, Br, Bi
constexpr int TC_THREADS = 576;            // 2 control warps + 16 epilogue warps
constexpr int TC_EPI_THREADS = 512;
constexpr int TC_TMEM_COLS = 512;            // Re | M | MT (3 x 128), power-of-2 allocation
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + 1024 + 256;
// instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B unsigned 8-bit
// (bits 7-9, 10-12 = 0; residues in [0, m)), both K-major, N >> 3 at bit 17,
// M >> 4 at bit 24. Products < 2^16, so |Re| < 2n 2^16 and |M|, |MT| < n 2^16.
constexpr uint32_t kTcIdesc = (2u << 4) | ((uint32_t)(TC_BM >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);
constexpr int64_t kTcMaxN = 8192;  // keeps every accumulator inside tc_mod's range

__constant__ int c_tc_mod[kMaxMod];
__constant__ uint32_t c_tc_magic[kMaxMod];  // ceil(2^39 / m), 2^31 for m = 256

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity))
    if (clock64() - t0 > (1ll << 33)) asm volatile("trap;");  // ~4 s at 2 GHz
}
__device__ __forceinline__ void tma_load3(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                          int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major operand in the canonical 128B-swizzled layout: 8-row groups of
// 1024 B (SBO), LBO unused (1), descriptor version 1, layout SWIZZLE_128B (2)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kTcIdesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// row-major enumeration of the upper triangle of a T x T tile grid
__host__ __device__ __forceinline__ void upper_tile(int t, int T, int& I, int& J) {
  double disc = (2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * t;
  int i = (int)floor(((2.0 * T + 1.0) - sqrt(disc)) * 0.5);
  if (i < 0) i = 0;
  while (i > 0 && i * T - i * (i - 1) / 2 > t) --i;
  while ((i + 1) * T - (i + 1) * i / 2 <= t) ++i;
  I = i;
  J = i + (t - (i * T - i * (i - 1) / 2));
}

// Visiting order of the persistent kernel: bands of KST_TC_BAND tile rows,
// each walked column by column (the diagonal triangle first), so the 148
// tiles in flight cover a ~12 x 12 block of the grid and each operand tile
// is fetched from HBM about once per band instead of once per tile row
// (row-major order re-reads every column tile T times once the residues
// outgrow L2: 92 GB at d = 24012). Results are stored by the row-major
// index (upper_tile), so only the order changes.
#ifndef KST_TC_BAND
#define KST_TC_BAND 12
#endif
__host__ __device__ __forceinline__ void band_tile(int v, int T, int& I, int& J) {
  int b0 = 0;
  for (;;) {
    const int h = T - b0 < KST_TC_BAND ? T - b0 : KST_TC_BAND;
    const int tri = h * (h + 1) / 2;
    const int cnt = tri + (T - b0 - h) * h;
    if (v < cnt) {
      if (v < tri) {  // triangle, column c holds rows b0 .. b0 + c
        int c = (int)((sqrt(8.0 * v + 1.0) - 1.0) * 0.5);
        while (c > 0 && c * (c + 1) / 2 > v) --c;
        while ((c + 1) * (c + 2) / 2 <= v) ++c;
        J = b0 + c;
        I = b0 + (v - c * (c + 1) / 2);
      } else {
        const int u = v - tri;
        J = b0 + h + u / h;
        I = b0 + u % h;
      }
      return;
    }
    v -= cnt;
    b0 += h;
  }
}
__host__ __device__ __forceinline__ int upper_index(int I, int J, int T) {
  return I * T - I * (I - 1) / 2 + (J - I);
}

// v mod m in [0, m), integer pipes only (no conversions): u = v + m 2^22,
// q = floor(u / m) = umulhi(u, ceil(2^39 / m)) >> 7, exact for u < 2^31 and
// 128 < m <= 256 (magic = 2^31 for m = 256). n <= kTcMaxN keeps
// -m 2^22 < v < 2^31 - m 2^22 for every Re / Im accumulator.
__device__ __forceinline__ uint32_t tc_mod(int v, int m, uint32_t magic) {
  const uint32_t u = (uint32_t)(v + (m << 22));
  return u - (uint32_t)m * (__umulhi(u, magic) >> 7);
}

// res[t][i][comp][row][col] (uint8; comp 0 = Re, 1 = Im), t = upper tile index
__global__ void __launch_bounds__(TC_THREADS, 1) gram_tc_kernel(
    const __grid_constant__ CUtensorMap tmap, int T, int ntiles, int nmod, int nkb,
    uint8_t* __restrict__ res, unsigned long long* __restrict__ prof) {
  // prof (debug, KST_TC_PROF=1): cycles the producer waits for free slots, the
  // MMA thread waits for data / for TMEM, and the MMA thread's total span
  long long w_empty = 0, w_full = 0, w_tmem = 0, t_begin = clock64();
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + TC_STAGES * TC_STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = (uint32_t*)(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, TC_EPI_THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int v = blockIdx.x; v < ntiles; v += gridDim.x) {
        int I, J;
        band_tile(v, T, I, J);
        for (int i = 0; i < nmod; ++i)
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % TC_STAGES;
            const uint32_t ph = (uint32_t)(it / TC_STAGES) & 1u;
            if (prof) {
              const long long c0 = clock64();
              mbar_wait(&empty[s], ph ^ 1u);
              w_empty += clock64() - c0;
            } else {
              mbar_wait(&empty[s], ph ^ 1u);
            }
            uint8_t* st = base + s * TC_STAGE_BYTES;
            mbar_expect_tx(&full[s], TC_STAGE_BYTES);
            tma_load3(&tmap, &full[s], st, kb * TC_BK, 2 * i, I * TC_BM);
            tma_load3(&tmap, &full[s], st + TC_OPER, kb * TC_BK, 2 * i + 1, I * TC_BM);
            tma_load3(&tmap, &full[s], st + 2 * TC_OPER, kb * TC_BK, 2 * i, J * TC_BM);
            tma_load3(&tmap, &full[s], st + 3 * TC_OPER, kb * TC_BK, 2 * i + 1, J * TC_BM);
          }
      }
      if (prof) atomicAdd(&prof[0], (unsigned long long)w_empty);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int it = 0, pass = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int i = 0; i < nmod; ++i, ++pass) {
          {
            const long long c0 = prof ? clock64() : 0;
            mbar_wait(tempty, ((uint32_t)pass & 1u) ^ 1u);  // epilogue drained TMEM
            if (prof) w_tmem += clock64() - c0;
          }
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % TC_STAGES;
            const uint32_t ph = (uint32_t)(it / TC_STAGES) & 1u;
            {
              const long long c0 = prof ? clock64() : 0;
              mbar_wait(&full[s], ph);
              if (prof) w_full += clock64() - c0;
            }
            tc_fence_after();
            const uint32_t sa = smem_u32(base + s * TC_STAGE_BYTES);
#ifdef KST_TC_INTERLEAVE
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk) {
              const uint64_t ar = sw128_desc(sa + 32 * kk);
              const uint64_t ai = sw128_desc(sa + TC_OPER + 32 * kk);
              const uint64_t br = sw128_desc(sa + 2 * TC_OPER + 32 * kk);
              const uint64_t bi = sw128_desc(sa + 3 * TC_OPER + 32 * kk);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              tc_mma_i8(tmem, ar, br, acc);          // Re  = Xr_a Xr_b
              tc_mma_i8(tmem, ai, bi, 1u);           //     + Xi_a Xi_b
              tc_mma_i8(tmem + 128, ai, br, acc);    // M   = Xi_a Xr_b
              tc_mma_i8(tmem + 256, ar, bi, acc);    // MT  = Xr_a Xi_b
            }
#else
            // runs of MMAs into the same accumulator: Re (8), M (4), MT (4)
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk)  // Re = Xr_a Xr_b
              tc_mma_i8(tmem, sw128_desc(sa + 32 * kk), sw128_desc(sa + 2 * TC_OPER + 32 * kk),
                        (kb | kk) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk)  //    + Xi_a Xi_b
              tc_mma_i8(tmem, sw128_desc(sa + TC_OPER + 32 * kk),
                        sw128_desc(sa + 3 * TC_OPER + 32 * kk), 1u);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk)  // M = Xi_a Xr_b
              tc_mma_i8(tmem + 128, sw128_desc(sa + TC_OPER + 32 * kk),
                        sw128_desc(sa + 2 * TC_OPER + 32 * kk), (kb | kk) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk)  // MT = Xr_a Xi_b
              tc_mma_i8(tmem + 256, sw128_desc(sa + 32 * kk),
                        sw128_desc(sa + 3 * TC_OPER + 32 * kk), (kb | kk) ? 1u : 0u);
#endif
            tc_commit(&empty[s]);  // smem slot reusable once these MMAs retire
          }
          tc_commit(tfull);  // accumulators of modulus i complete
        }
      if (prof) {
        atomicAdd(&prof[1], (unsigned long long)w_full);
        atomicAdd(&prof[2], (unsigned long long)w_tmem);
        atomicAdd(&prof[3], (unsigned long long)(clock64() - t_begin));
      }
    }
  } else {  // ---------------- epilogue: TMEM -> residues
    // 16 warps: lane quarter q = warp % 4 (TMEM lanes 32q..32q+31 = tile rows),
    // column block cb = (warp - 2) / 4 (32 of the 128 columns). Each thread
    // loads its 32 Re, M and MT words, releases TMEM, and only then reduces
    // and stores, so the next modulus' MMAs overlap the modular arithmetic.
    const int q = warp & 3, cb = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + 32 * cb;
    int pass = 0;
    for (int v = blockIdx.x; v < ntiles; v += gridDim.x) {
      int I, J;
      band_tile(v, T, I, J);
      const int t = upper_index(I, J, T);
      for (int i = 0; i < nmod; ++i, ++pass) {
        mbar_wait(tfull, (uint32_t)pass & 1u);
        tc_fence_after();
        uint32_t vre[32], vm[32], vmt[32];
        tc_ld32(taddr, vre);
        tc_ld32(taddr + 128, vm);
        tc_ld32(taddr + 256, vmt);
        tc_wait_ld();
        tc_fence_before();
        mbar_arrive(tempty);  // TMEM free for modulus i + 1
        const int m = c_tc_mod[i];
        const uint32_t magic = c_tc_magic[i];
        uint32_t pre[8], pim[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          uint32_t a = 0, b = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * w + e;
            a |= tc_mod((int)vre[j], m, magic) << (8 * e);
            b |= tc_mod((int)vm[j] - (int)vmt[j], m, magic) << (8 * e);
          }
          pre[w] = a;
          pim[w] = b;
        }
        uint8_t* out_re = res + (((size_t)t * nmod + i) * 2) * (TC_BM * TC_BM) +
                          (size_t)row * TC_BM + 32 * cb;
        uint4* dre = (uint4*)out_re;
        uint4* dim = (uint4*)(out_re + TC_BM * TC_BM);
        dre[0] = make_uint4(pre[0], pre[1], pre[2], pre[3]);
        dre[1] = make_uint4(pre[4], pre[5], pre[6], pre[7]);
        dim[0] = make_uint4(pim[0], pim[1], pim[2], pim[3]);
        dim[1] = make_uint4(pim[4], pim[5], pim[6], pim[7]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TC_TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- two-SM form
// gram_tc2_kernel: the products on CTA pairs (cluster of 2, one CTA per SM)
// with tcgen05.mma.cta_group::2, M = 256 and N = 256: work unit = rows
// [256 I2, 256 I2 + 256) x columns [256 Jp, 256 Jp + 256), Jp >= I2. CTA rank
// r holds its 128 rows of A (Xr', Xi' and the negated -Xr') and the 128 B rows
// of column tile J = 2 Jp + r (Xr', Xi') in its own smem at the same offsets;
// the leader (rank 0) issues every MMA for the pair and each CTA's TMEM
// receives its 128 rows x 256 columns of two accumulators:
//   Re += Ar.Br + Ai.Bi        Im += Ai.Br + An.Bi    (An = -Xr' mod m)
// so Im = M - MT needs no third accumulator and TMEM (512 columns) holds
// [Re | Im] for 256 columns. Per SM and 64-snapshot K block the operands are
// 40 KB for 16 MMA units of 128 x 128 x 32 (2.5 KB per unit against 4 KB in
// the single-CTA kernel: 40 B/clk per SM at full MMA rate, under the ~42 B/clk
// the L2 delivers), and every instruction is a 256 x 256 MMA, which amortises
// the per-instruction cost that holds the 128-wide MMAs at ~2/3 of the pipe
// rate. Both CTAs' TMA loads complete on
// the leader's full barrier (.cta_group::2); the leader's commits multicast
// to both CTAs' empty / tfull barriers; both epilogues arrive on the leader's
// tempty barrier. Sub-tiles below the diagonal (J < I) are computed and not
// stored.
#ifndef KST_TC2_BK
#define KST_TC2_BK 64
#endif
constexpr int TC2_BK = KST_TC2_BK;               // K bytes per stage = swizzle row (64 or 128 B)
constexpr int TC2_STAGES = TC2_BK == 64 ? 5 : 2;  // <= 200 KB of stages
constexpr int TC2_TILE = TC_BM * TC2_BK;                    // 8 KB: 128 rows x 64 B
constexpr int TC2_STAGE_BYTES = 5 * TC2_TILE;               // Ar, Ai, An | Br, Bi: 40 KB
constexpr size_t TC2_SMEM = (size_t)TC2_STAGES * TC2_STAGE_BYTES + 1024 + 256;
// kind::i8, D s32, A/B unsigned, K-major, N = 256, M = 256 (pair)
constexpr uint32_t kTc2Idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA into this CTA's smem completing on an mbarrier of either CTA of the pair
// (.cta_group::2 -- here always the leader's full barrier)
__device__ __forceinline__ void tma_load3_to(const CUtensorMap* map, uint32_t mbar_cluster, void* dst,
                                             int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(mbar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// K-major operand, 64B-swizzled rows of 64 bytes: 8-row groups 512 B apart;
// with 128-byte rows the 128B-swizzled layout (sw128_desc)
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  if (TC2_BK == 128) return sw128_desc(saddr);
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void tc2_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kTc2Idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in both CTAs once the issued MMAs retire
__device__ __forceinline__ void tc2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1) gram_tc2_kernel(
    const __grid_constant__ CUtensorMap tmap, int T, int nunits, int nmod, int nkb,
    uint8_t* __restrict__ res) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + TC2_STAGES * TC2_STAGE_BYTES);
  uint64_t* empty = full + TC2_STAGES;
  uint64_t* tfull = empty + TC2_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = (uint32_t*)(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int T2 = T >> 1;  // pair tiles per side
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TC2_STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: one expect_tx arrival for both CTAs' bytes
      mbar_init(&empty[s], 1);  // one multicast commit per use
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * TC_EPI_THREADS);  // both CTAs' epilogues (the leader's copy is used)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const uint32_t full_l0 = mapa_shared(&full[0], 0);
      int it = 0;
      for (int u = cid; u < nunits; u += ncl) {
        int I2, Jp;
        upper_tile(u, T2, I2, Jp);
        const int arow = 256 * I2 + 128 * (int)rank, brow = 256 * Jp + 128 * (int)rank;
        for (int i = 0; i < nmod; ++i)
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % TC2_STAGES;
            const uint32_t ph = (uint32_t)(it / TC2_STAGES) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            uint8_t* st = base + s * TC2_STAGE_BYTES;
            const uint32_t fb = full_l0 + (uint32_t)(s * sizeof(uint64_t));  // leader's full[s]
            if (leader) mbar_expect_tx(&full[s], 2 * TC2_STAGE_BYTES);
            const int k0 = kb * TC2_BK, pl = 3 * i;  // planes Xr', Xi', -Xr' of modulus i
            tma_load3_to(&tmap, fb, st, k0, pl, arow);                     // Ar
            tma_load3_to(&tmap, fb, st + TC2_TILE, k0, pl + 1, arow);      // Ai
            tma_load3_to(&tmap, fb, st + 2 * TC2_TILE, k0, pl + 2, arow);  // An
            tma_load3_to(&tmap, fb, st + 3 * TC2_TILE, k0, pl, brow);      // Br (this CTA's half)
            tma_load3_to(&tmap, fb, st + 4 * TC2_TILE, k0, pl + 1, brow);  // Bi
          }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---------------- MMA issuer (leader only)
      int it = 0, pass = 0;
      for (int u = cid; u < nunits; u += ncl)
        for (int i = 0; i < nmod; ++i, ++pass) {
          mbar_wait(tempty, ((uint32_t)pass & 1u) ^ 1u);  // both epilogues drained TMEM
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % TC2_STAGES;
            const uint32_t ph = (uint32_t)(it / TC2_STAGES) & 1u;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(base + s * TC2_STAGE_BYTES);
            const uint32_t a_r = sa, a_i = sa + TC2_TILE, a_n = sa + 2 * TC2_TILE;
            const uint32_t b_r = sa + 3 * TC2_TILE, b_i = sa + 4 * TC2_TILE;
#pragma unroll
            for (int kk = 0; kk < TC2_BK / 32; ++kk) {
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              tc2_mma_i8(tmem, sw64_desc(a_r + 32 * kk), sw64_desc(b_r + 32 * kk), acc);  // Re
              tc2_mma_i8(tmem, sw64_desc(a_i + 32 * kk), sw64_desc(b_i + 32 * kk), 1u);
              tc2_mma_i8(tmem + 256, sw64_desc(a_i + 32 * kk), sw64_desc(b_r + 32 * kk), acc);  // Im
              tc2_mma_i8(tmem + 256, sw64_desc(a_n + 32 * kk), sw64_desc(b_i + 32 * kk), 1u);
            }
            tc2_commit_both(&empty[s]);  // both CTAs' slot s reusable
          }
          tc2_commit_both(tfull);  // both CTAs' accumulators of modulus i complete
        }
    }
  } else {  // ---------------- epilogue (both CTAs, own 128 rows x 256 columns)
    // 16 warps: lane quarter q = warp % 4, column block cb = (warp - 2) / 4 of
    // 64 columns = column tile J = 2 Jp + cb / 2, offset 64 (cb % 2); two
    // rounds of 32 columns; TMEM is released after the second round's loads.
    const int q = warp & 3, cb = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + 64 * cb;
    const uint32_t tempty_l0 = mapa_shared(tempty, 0);
    int pass = 0;
    for (int u = cid; u < nunits; u += ncl) {
      int I2, Jp;
      upper_tile(u, T2, I2, Jp);
      const int I = 2 * I2 + (int)rank, J = 2 * Jp + (cb >> 1);
      const bool store = J >= I;
      const int t = I * T - I * (I - 1) / 2 + (J - I);  // upper-tile index (when store)
      for (int i = 0; i < nmod; ++i, ++pass) {
        mbar_wait(tfull, (uint32_t)pass & 1u);
        tc_fence_after();
        const int m = c_tc_mod[i];
        const uint32_t magic = c_tc_magic[i];
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t vre[32], vim[32];
          tc_ld32(taddr + 32 * h, vre);
          tc_ld32(taddr + 256 + 32 * h, vim);
          tc_wait_ld();
          if (h == 1) {
            tc_fence_before();
            mbar_arrive_cluster(tempty_l0);  // this CTA's TMEM free for modulus i + 1
          }
          if (!store) continue;
          uint32_t pre[8], pim[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * w + e;
              a |= tc_mod((int)vre[j], m, magic) << (8 * e);
              b |= tc_mod((int)vim[j], m, magic) << (8 * e);
            }
            pre[w] = a;
            pim[w] = b;
          }
          uint8_t* out_re = res + (((size_t)t * nmod + i) * 2) * (TC_BM * TC_BM) +
                            (size_t)row * TC_BM + 64 * (cb & 1) + 32 * h;
          uint4* dre = (uint4*)out_re;
          uint4* dim = (uint4*)(out_re + TC_BM * TC_BM);
          dre[0] = make_uint4(pre[0], pre[1], pre[2], pre[3]);
          dre[1] = make_uint4(pre[4], pre[5], pre[6], pre[7]);
          dim[0] = make_uint4(pim[0], pim[1], pim[2], pim[3]);
          dim[1] = make_uint4(pim[4], pim[5], pim[6], pim[7]);
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the leader's last MMAs into the peer's TMEM have retired
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TC_TMEM_COLS)
                 : "memory");
  }
}

// CRT reconstruction from the uint8 residue tiles: CTA per (tile, 32 x 32
// sub-block); writes S[a][b] and the conjugate mirror S[b][a] (coalesced via
// an smem transpose). Diagonal tiles keep a <= b only.
template <int NM>
__global__ void __launch_bounds__(256, 2) crt_tile_combine_kernel(
    const uint8_t* __restrict__ res, int T, const int* __restrict__ expo, int beta, double dn,
    int64_t d, cplx* __restrict__ S) {
  __shared__ cplx vt[32][33];
  const double rn = 1.0 / dn;
  const int t = blockIdx.x >> 4, sb = blockIdx.x & 15;
  int I, J;
  upper_tile(t, T, I, J);
  const int sr = sb >> 2, sc = sb & 3;
  const int tid = threadIdx.x;
  const int q4 = 4 * (tid & 7), r = tid >> 3;
  const int lr = 32 * sr + r, lc = 32 * sc + q4;  // tile-local row / first column
  const int64_t a = (int64_t)I * TC_BM + lr;
  constexpr int NCH = crt_nch(NM);
  double re0[4], re1[4], re2[4], im0[4], im1[4], im2[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) re0[c] = re1[c] = re2[c] = im0[c] = im1[c] = im2[c] = 0.0;
  const uint8_t* src = res + (size_t)t * NM * 2 * (TC_BM * TC_BM) + (size_t)lr * TC_BM + lc;
  uint32_t pr[NM], pm[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    pr[i] = *(const uint32_t*)(src + (size_t)(2 * i) * (TC_BM * TC_BM));
    pm[i] = *(const uint32_t*)(src + (size_t)(2 * i + 1) * (TC_BM * TC_BM));
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const double w0 = c_crt.w[i][0], w1 = c_crt.w[i][1], w2 = c_crt.w[i][2];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // byte -> double by exponent splicing (FP64 adder, not the conversion
      // unit): (2^52 + c) - 2^52
      const uint32_t cr = __byte_perm(pr[i], 0, 0x4440 + c), cm = __byte_perm(pm[i], 0, 0x4440 + c);
      const double dr = __longlong_as_double(0x4330000000000000ll | cr) - 4503599627370496.0;
      const double dm = __longlong_as_double(0x4330000000000000ll | cm) - 4503599627370496.0;
      re0[c] = fma(dr, w0, re0[c]);
      re1[c] = fma(dr, w1, re1[c]);
      im0[c] = fma(dm, w0, im0[c]);
      im1[c] = fma(dm, w1, im1[c]);
      if (NCH == 3) {
        re2[c] = fma(dr, w2, re2[c]);
        im2[c] = fma(dm, w2, im2[c]);
      }
    }
  }
  const int ea = (a < d) ? expo[a] : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int64_t b = (int64_t)J * TC_BM + lc + c;
    const int eb = (b < d) ? expo[b] : 0;
    cplx v;
    if (ea == kNaNExpo || eb == kNaNExpo) {
      v = cmk(NAN, NAN);
    } else {
      const double vre = crt_finish<NCH>(re0[c], re1[c], re2[c]);
      const double vim = crt_finish<NCH>(im0[c], im1[c], im2[c]);
      const int sh = ea + eb - 2 * beta;
      v = cmk(crt_scale(vre, sh, dn, rn), crt_scale(vim, sh, dn, rn));
    }
    vt[r][q4 + c] = v;
  }
  __syncthreads();
  const int tx = tid & 31, ty = tid >> 5;
  const int64_t a0 = (int64_t)I * TC_BM + 32 * sr, b0 = (int64_t)J * TC_BM + 32 * sc;
  for (int rr = ty; rr < 32; rr += 8) {
    {  // S[a0 + rr][b0 + tx]
      const int64_t aa = a0 + rr, bb = b0 + tx;
      if (aa < d && bb < d && aa <= bb) {
        const cplx v = vt[rr][tx];
        S[aa * d + bb] = (aa == bb) ? cmk(v.x, 0.0) : v;
      }
    }
    {  // S[b0 + rr][a0 + tx] = conj(S[a0 + tx][b0 + rr])
      const int64_t bb = b0 + rr, aa = a0 + tx;
      if (aa < d && bb < d && aa < bb) {
        const cplx v = vt[tx][rr];
        S[bb * d + aa] = cmk(v.x, -v.y);
      }
    }
  }
}

// Strip variant (default): persistent CTAs, item = (tile, 8-row strip). A
// producer lane streams each item's 2 NM residue planes (8 rows x 128 B =
// 1 KB, contiguous) into an mbarrier ring with bulk async copies, so the
// loads run ahead of the FP64 reconstruction instead of stalling it (the
// per-thread-load kernel above spends most of its time on long-scoreboard
// waits at 25 % occupancy). 8 consumer warps: row r = warp, 4 columns per
// lane; S rows (2 KB segments) and the conjugate mirror (128 B segments)
// are written from an smem transpose.
constexpr int CS_ROWS = 8, CS_CONS = 256;
#ifndef KST_CS_STAGES
#define KST_CS_STAGES 2
#endif
// 2 stages x 20 KB: three CTAs per SM (A/B: 232 us vs 247 us at 4 stages, 2 CTAs)
__host__ __device__ constexpr int cs_stages(int nm) { return nm <= 10 ? KST_CS_STAGES : 2; }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CS_CONS) : "memory");
}

template <int NM>
__global__ void __launch_bounds__(CS_CONS + 32, 3) crt_strip_combine_kernel(
    const uint8_t* __restrict__ res, int T, int nitems, const int* __restrict__ expo, int beta,
    double dn, int64_t d, cplx* __restrict__ S) {
  constexpr int PLANE = CS_ROWS * TC_BM, STAGE = 2 * NM * PLANE, NS = cs_stages(NM);
  constexpr int VLD = TC_BM + 1;  // padded vt row (conflict-free column reads)
  extern __shared__ __align__(128) unsigned char cs_smem[];
  __shared__ uint64_t full[NS], empty[NS];
  uint8_t* ring = cs_smem;
  cplx* vt = (cplx*)(cs_smem + NS * STAGE);  // [CS_ROWS][VLD]
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CS_CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr int SPT = TC_BM / CS_ROWS;  // strips per tile
  if (tid >= CS_CONS) {  // ------------------------------ producer lane
    if (tid == CS_CONS) {
      int it = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
        const int s = it % NS;
        mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
        mbar_expect_tx(&full[s], STAGE);
        const uint8_t* src = res + (size_t)(item / SPT) * NM * 2 * (TC_BM * TC_BM) +
                             (size_t)(item % SPT) * PLANE;
        for (int pl = 0; pl < 2 * NM; ++pl)
          bulk_load(ring + s * STAGE + pl * PLANE, src + (size_t)pl * (TC_BM * TC_BM), PLANE, &full[s]);
      }
    }
    return;
  }
  // ------------------------------------------------------ consumers
  constexpr int NCH = crt_nch(NM);
  const double rn = 1.0 / dn;
  const int r = tid >> 5, l = tid & 31;
  int it = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
    const int s = it % NS;
    const int t = item / SPT;
    int I, J;
    upper_tile(t, T, I, J);
    const int64_t a0 = (int64_t)I * TC_BM + (item % SPT) * CS_ROWS, b0 = (int64_t)J * TC_BM;
    const int64_t a = a0 + r;
    // column exponents first: their global latency overlaps the ring wait
    const int ea = (a < d) ? __ldg(&expo[a]) : 0;
    int eb[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) eb[c] = (b0 + 4 * l + c < d) ? __ldg(&expo[b0 + 4 * l + c]) : 0;
    mbar_wait(&full[s], (uint32_t)(it / NS) & 1u);
    uint32_t pr[NM], pm[NM];
    const uint8_t* src = ring + s * STAGE + r * TC_BM + 4 * l;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      pr[i] = *(const uint32_t*)(src + (2 * i) * PLANE);
      pm[i] = *(const uint32_t*)(src + (2 * i + 1) * PLANE);
    }
    __syncwarp();
    if (l == 0) mbar_arrive(&empty[s]);  // residues are in registers: release the slot
    double re0[4], re1[4], re2[4], im0[4], im1[4], im2[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) re0[c] = re1[c] = re2[c] = im0[c] = im1[c] = im2[c] = 0.0;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const double w0 = c_crt.w[i][0], w1 = c_crt.w[i][1], w2 = c_crt.w[i][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t cr = __byte_perm(pr[i], 0, 0x4440 + c), cm = __byte_perm(pm[i], 0, 0x4440 + c);
        const double dr = __longlong_as_double(0x4330000000000000ll | cr) - 4503599627370496.0;
        const double dm = __longlong_as_double(0x4330000000000000ll | cm) - 4503599627370496.0;
        re0[c] = fma(dr, w0, re0[c]);
        re1[c] = fma(dr, w1, re1[c]);
        im0[c] = fma(dm, w0, im0[c]);
        im1[c] = fma(dm, w1, im1[c]);
        if (NCH == 3) {
          re2[c] = fma(dr, w2, re2[c]);
          im2[c] = fma(dm, w2, im2[c]);
        }
      }
    }
    cons_sync();  // previous item's vt reads are done
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cplx v;
      if (ea == kNaNExpo || eb[c] == kNaNExpo) {
        v = cmk(NAN, NAN);
      } else {
        const int sh = ea + eb[c] - 2 * beta;
        v = cmk(crt_scale(crt_finish<NCH>(re0[c], re1[c], re2[c]), sh, dn, rn),
                crt_scale(crt_finish<NCH>(im0[c], im1[c], im2[c]), sh, dn, rn));
      }
      vt[r * VLD + 4 * l + c] = v;
    }
    cons_sync();
    // S[a][b], a <= b: one 2 KB row segment per warp trip
#pragma unroll
    for (int k = 0; k < CS_ROWS * TC_BM / CS_CONS; ++k) {
      const int idx = tid + k * CS_CONS, rr = idx >> 7, cc = idx & (TC_BM - 1);
      const int64_t aa = a0 + rr, bb = b0 + cc;
      if (aa < d && bb < d && aa <= bb) {
        const cplx v = vt[rr * VLD + cc];
        S[aa * d + bb] = (aa == bb) ? cmk(v.x, 0.0) : v;
      }
    }
    // S[b][a] = conj(S[a][b]), a < b: 128 B row segments
#pragma unroll
    for (int k = 0; k < CS_ROWS * TC_BM / CS_CONS; ++k) {
      const int idx = tid + k * CS_CONS, cc = idx / CS_ROWS, rr = idx % CS_ROWS;
      const int64_t aa = a0 + rr, bb = b0 + cc;
      if (aa < d && bb < d && aa < bb) {
        const cplx v = vt[rr * VLD + cc];
        S[bb * d + aa] = cmk(v.x, -v.y);
      }
    }
  }
}

template <int NM>
void launch_tile_combine(const uint8_t* res, int T, int ntiles, const int* expo, int beta, double dn,
                         int64_t d, cplx* S, cudaStream_t st) {
  static const bool strip = !(getenv("KST_CTC") && atoi(getenv("KST_CTC")) == 0);
  if (!strip) {
    crt_tile_combine_kernel<NM><<<(unsigned)ntiles * 16, 256, 0, st>>>(res, T, expo, beta, dn, d, S);
    return;
  }
  constexpr int smem = cs_stages(NM) * 2 * NM * CS_ROWS * TC_BM + CS_ROWS * (TC_BM + 1) * 16;
  static int grid = 0;
  if (!grid) {
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(crt_strip_combine_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, crt_strip_combine_kernel<NM>, CS_CONS + 32, smem);
    grid = nsm * std::max(per, 1);
  }
  const int nitems = ntiles * (TC_BM / CS_ROWS);
  crt_strip_combine_kernel<NM><<<(unsigned)std::min(grid, nitems), CS_CONS + 32, smem, st>>>(
      res, T, nitems, expo, beta, dn, d, S);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

#define KST_CRT_DISPATCH(NMV, CALL)                \
  switch (NMV) {                                   \
    case 8: { constexpr int NM_ = 8; CALL; } break;   \
    case 9: { constexpr int NM_ = 9; CALL; } break;   \
    case 10: { constexpr int NM_ = 10; CALL; } break; \
    case 11: { constexpr int NM_ = 11; CALL; } break; \
    case 12: { constexpr int NM_ = 12; CALL; } break; \
    case 13: { constexpr int NM_ = 13; CALL; } break; \
    default: { constexpr int NM_ = 14; CALL; } break; \
  }

}  // namespace

namespace kst {

int crt_beta(int nmod, int64_t n) {
  if (nmod < 8 || nmod > kMaxUsed || n < 1) return -1;
  const double lp = host_crt(nmod).log2p;
  // 2n 2^(2 beta) <= P / 4 (exact products, |V| <= P/4); small safety margin
  const int beta = (int)std::floor((lp - 3.0 - std::log2((double)n) - 1e-6) / 2.0);
  return std::min(beta, 48);
}

bool crt_tc_available() { return encode_tiled() != nullptr; }

// tcgen05 path: residues -> gram_tc_kernel (products + modular reduction) ->
// crt_tile_combine_kernel (reconstruction). Caller validated nmod / n.
static int scm_crt_tc(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, int nmod, int beta,
                      cudaStream_t st) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return set_err(ctx, KST_ERR_CUDA, "scm_crt: cuTensorMapEncodeTiled unavailable");
  // KST_TC2=1 selects the two-SM (cta_group::2, 256x256) kernel: same exact
  // products, but measured ~5% slower end to end on B200 (3-plane residues,
  // 256-row padding, below-diagonal sub-tiles) -- the single-CTA kernel runs
  // at ~87% of the power-capped int8 rate already.
  const char* tc2 = getenv("KST_TC2");
  const bool pair = tc2 && atoi(tc2) == 1;
  const int64_t npad = ((n + 15) / 16) * 16;
  const int64_t dal = pair ? 2 * TC_BM : TC_BM;  // pair units span two row tiles
  const int64_t dpad = ((d + dal - 1) / dal) * dal;
  const int parts = pair ? 3 : 2;  // residue planes per modulus
  const int T = (int)(dpad / TC_BM);
  const int ntiles = T * (T + 1) / 2;
  const int bk = pair ? TC2_BK : TC_BK;
  const int nkb = (int)((npad + bk - 1) / bk);
  const int64_t ldr = (int64_t)nmod * parts * npad;
  char* sl = (char*)ws_get(ctx, WS_OZ_SLICES,
                          (size_t)dpad * ldr + sizeof(int) * (2 * (size_t)dpad + 64) + 256);
  uint8_t* res = (uint8_t*)ws_get(ctx, WS_OZ_PROD, (size_t)ntiles * nmod * 2 * TC_BM * TC_BM);
  if (!sl || !res) return set_err(ctx, KST_ERR_CUDA, "scm_crt: workspace");
  int8_t* R = (int8_t*)sl;
  int* expo = (int*)(R + (size_t)dpad * ldr);
  {
    static int mods[kMaxMod];
    static uint32_t magic[kMaxMod];
    for (int i = 0; i < kMaxMod; ++i) {
      mods[i] = kModuli[i];
      magic[i] = kModuli[i] == 256 ? (1u << 31)
                                   : (uint32_t)((((uint64_t)1 << 39) + kModuli[i] - 1) / kModuli[i]);
    }
    KST_TRY(const_upload(ctx, (const void*)&c_tc_mod, mods, sizeof(mods), st));
    KST_TRY(const_upload(ctx, (const void*)&c_tc_magic, magic, sizeof(magic), st));
  }
  CUtensorMap map;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)npad, (cuuint64_t)(parts * nmod), (cuuint64_t)dpad};
    const cuuint64_t strides[2] = {(cuuint64_t)npad, (cuuint64_t)ldr};  // bytes, dims 1 and 2
    const cuuint32_t box[3] = {(cuuint32_t)bk, 1, TC_BM};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)R, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, KST_ERR_CUDA, "cuTensorMapEncodeTiled failed: %d", (int)r);
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = kNumSMs;
  }
  KST_TRY(colmax_split(ctx, X, n, d, expo, expo + dpad, st));
  KST_CRT_DISPATCH(nmod, (launch_crt<NM_>(X, n, npad, d, dpad, expo, beta, R, true, parts, st)));
  KST_LAUNCH(ctx);
  if (pair) {
    KST_CUDA(ctx, cudaFuncSetAttribute(gram_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)TC2_SMEM));
    const int nunits = (T / 2) * (T / 2 + 1) / 2;  // upper 256 x 256 super-tiles
    const int nclusters = std::min(nunits, nsm / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * nclusters));
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = TC2_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    stage_mark(ctx, 5, st);
    KST_CUDA(ctx, cudaLaunchKernelEx(&cfg, gram_tc2_kernel, map, T, nunits, nmod, nkb, res));
    KST_LAUNCH(ctx);
    stage_mark(ctx, 6, st);
    ctx->last_int8_ops = 2.0 * 4.0 * 4.0 * (double)TC_BM * TC_BM * (double)nkb * bk * nmod * nunits;
    KST_CRT_DISPATCH(nmod, (launch_tile_combine<NM_>(res, T, ntiles, expo, beta, (double)n, d, S, st)));
    KST_LAUNCH(ctx);
    return KST_OK;
  }
  KST_CUDA(ctx, cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)TC_SMEM));
  stage_mark(ctx, 5, st);  // profiling: int8 tensor-core span (events 5..6)
  static const bool prof_on = getenv("KST_TC_PROF") && atoi(getenv("KST_TC_PROF")) != 0;
  unsigned long long* prof = nullptr;
  if (prof_on) {
    prof = (unsigned long long*)ws_get(ctx, WS_TMP, 64);
    if (!prof) return set_err(ctx, KST_ERR_CUDA, "scm_crt: profile buffer");
    KST_CUDA(ctx, cudaMemsetAsync(prof, 0, 64, st));
  }
  const int grid = std::min(ntiles, nsm);
  gram_tc_kernel<<<(unsigned)grid, TC_THREADS, TC_SMEM, st>>>(map, T, ntiles, nmod, nkb, res, prof);
  KST_LAUNCH(ctx);
  stage_mark(ctx, 6, st);
  if (prof_on) {  // debug: where the pipeline waits (cycles summed over CTAs)
    unsigned long long h[4];
    KST_CUDA(ctx, cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    fprintf(stderr,
            "[gram_tc] per CTA (cycles): span %.0f, MMA waits data %.0f (%.1f%%), TMEM %.0f "
            "(%.1f%%), producer waits slots %.0f\n",
            (double)h[3] / grid, (double)h[1] / grid, 100.0 * h[1] / h[3], (double)h[2] / grid,
            100.0 * h[2] / h[3], (double)h[0] / grid);
  }
  ctx->last_int8_ops = 2.0 * 4.0 * (double)TC_BM * TC_BM * (double)nkb * TC_BK * nmod * ntiles;
  KST_CRT_DISPATCH(nmod, (launch_tile_combine<NM_>(res, T, ntiles, expo, beta, (double)n, d, S, st)));
  KST_LAUNCH(ctx);
  return KST_OK;
}

int scm_crt(kst_ctx* ctx, const cplx* X, int64_t n, int64_t d, cplx* S, int nmod, bool use_tc,
            cudaStream_t st) {
  if (nmod < 8 || nmod > kMaxUsed)
    return set_err(ctx, KST_ERR_DIMENSION, "CRT Gram needs 8..%d moduli, got %d", kMaxUsed, nmod);
  const int beta = crt_beta(nmod, n);
  if (beta < 8) return set_err(ctx, KST_ERR_DIMENSION, "CRT Gram: n=%lld too large for %d moduli",
                               (long long)n, nmod);
  if (2 * n > (int64_t)1 << 17)
    return set_err(ctx, KST_ERR_DIMENSION, "CRT Gram: int32 products need n <= 65536");
  const HostCrt& hc = host_crt(nmod);
  KST_TRY(const_upload(ctx, (const void*)&c_crt, &hc.c, sizeof(CrtConst), st));
  // n > kTcMaxN (beyond every configuration here) takes the library-GEMM form
  // of the same numerics
  if (use_tc && n <= kTcMaxN) return scm_crt_tc(ctx, X, n, d, S, nmod, beta, st);
  if (!i8::load_blas()) return set_err(ctx, KST_ERR_CUDA, "scm_crt: cuBLAS not loadable");
  cublasHandle_t h = i8::blas_handle(ctx, st);
  if (!h) return set_err(ctx, KST_ERR_CUDA, "cublasCreate failed");

  const int64_t npad = ((n + 15) / 16) * 16;
  constexpr int NB = 4;  // Re is symmetric: upper blocks of an NB x NB grid
  const bool blocked = d >= 1024;
  const int64_t dpad = blocked ? ((d + 32 * NB - 1) / (32 * NB)) * (32 * NB) : ((d + 31) / 32) * 32;
  const int64_t bsz = dpad / NB;
  constexpr int NBLK = NB * (NB + 1) / 2;
  const size_t plane = (size_t)dpad * dpad;
  const int64_t ldr = (int64_t)nmod * 2 * npad;  // bytes per column a
  char* sl = (char*)ws_get(ctx, WS_OZ_SLICES, (size_t)dpad * ldr + sizeof(int) * dpad +
                                                   sizeof(void*) * 3 * NBLK * kMaxMod + 512);
  int32_t* G = (int32_t*)ws_get(ctx, WS_OZ_PROD, sizeof(int32_t) * 2 * nmod * plane);
  if (!sl || !G) return set_err(ctx, KST_ERR_CUDA, "scm_crt: workspace");
  int8_t* R = (int8_t*)sl;
  int* expo = (int*)(R + (size_t)dpad * ldr);
  void** dptr = (void**)(((uintptr_t)(expo + dpad) + 255) & ~(uintptr_t)255);
  int32_t* GRe = G;
  int32_t* GM = G + (size_t)nmod * plane;
  if (blocked) {
    void** hp = (void**)pinned_get(ctx, sizeof(void*) * 3 * NBLK * kMaxMod);
    if (!hp) return set_err(ctx, KST_ERR_CUDA, "scm_crt: pinned staging");
    // [A | B | C] pointer arrays, each nmod x NBLK
    for (int i = 0; i < nmod; ++i) {
      int k = 0;
      for (int I = 0; I < NB; ++I)
        for (int J = I; J < NB; ++J, ++k) {
          const size_t e = (size_t)i * NBLK + k;
          hp[e] = (void*)(R + (size_t)i * 2 * npad + (size_t)I * bsz * ldr);
          hp[(size_t)nmod * NBLK + e] = (void*)(R + (size_t)i * 2 * npad + (size_t)J * bsz * ldr);
          hp[(size_t)2 * nmod * NBLK + e] =
              (void*)(GRe + (size_t)i * plane + I * bsz + (size_t)J * bsz * dpad);
        }
    }
    KST_CUDA(ctx, cudaMemcpyAsync(dptr, hp, sizeof(void*) * 3 * NBLK * nmod, cudaMemcpyHostToDevice, st));
  }
  i8::colmax_kernel<<<cdiv(d, 32), dim3(32, 8), 0, st>>>(X, n, d, expo);
  KST_LAUNCH(ctx);
  KST_CRT_DISPATCH(nmod, (launch_crt<NM_>(X, n, npad, d, dpad, expo, beta, R, false, 2, st)));
  KST_LAUNCH(ctx);
  stage_mark(ctx, 5, st);  // profiling: int8 GEMM span (events 5..6)
  const int32_t one = 1, zero = 0;
  for (int i = 0; i < nmod; ++i) {
    const int8_t* Ri = R + (size_t)i * 2 * npad;
    cublasStatus_t r1;
    if (blocked) {
      void** A = dptr + (size_t)i * NBLK;
      void** B = dptr + (size_t)(nmod + i) * NBLK;
      void** Cc = dptr + (size_t)(2 * nmod + i) * NBLK;
      r1 = i8::g_blas.gemm_batched_ex(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)bsz, (int)bsz, (int)(2 * npad),
                                      &one, (const void* const*)A, CUDA_R_8I, (int)ldr,
                                      (const void* const*)B, CUDA_R_8I, (int)ldr, &zero, Cc,
                                      CUDA_R_32I, (int)dpad, NBLK, CUBLAS_COMPUTE_32I,
                                      CUBLAS_GEMM_DEFAULT);
    } else {
      r1 = i8::g_blas.gemm_ex(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)dpad, (int)dpad, (int)(2 * npad), &one,
                              Ri, CUDA_R_8I, (int)ldr, Ri, CUDA_R_8I, (int)ldr, &zero,
                              GRe + (size_t)i * plane, CUDA_R_32I, (int)dpad, CUBLAS_COMPUTE_32I,
                              CUBLAS_GEMM_DEFAULT);
    }
    // M_i[a][b] = sum_k Xi'[k,a] Xr'[k,b] (mod-m_i residues)
    const cublasStatus_t r2 = i8::g_blas.gemm_ex(
        h, CUBLAS_OP_T, CUBLAS_OP_N, (int)dpad, (int)dpad, (int)npad, &one, Ri + npad, CUDA_R_8I,
        (int)ldr, Ri, CUDA_R_8I, (int)ldr, &zero, GM + (size_t)i * plane, CUDA_R_32I, (int)dpad,
        CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
    if (r1 != CUBLAS_STATUS_SUCCESS || r2 != CUBLAS_STATUS_SUCCESS)
      return set_err(ctx, KST_ERR_CUDA, "cublasGemmEx (int8 CRT) failed: %d %d", (int)r1, (int)r2);
    ctx->launches += 2;
  }
  stage_mark(ctx, 6, st);
  {
    const double re_frac = blocked ? (double)NBLK / (NB * NB) : 1.0;
    ctx->last_int8_ops = 2.0 * (double)dpad * (double)dpad * (double)npad * nmod * (2.0 * re_frac + 1.0);
  }
  KST_CRT_DISPATCH(nmod, (launch_combine<NM_>(GRe, GM, dpad, d, expo, beta, (double)n, S, st)));
  KST_LAUNCH(ctx);
  return KST_OK;
}

}  // namespace kst
