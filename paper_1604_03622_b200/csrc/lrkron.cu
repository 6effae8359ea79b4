// K2 + K3: the LR-Kron alternating estimator, `lr_kron_estimate`
// (src/lrkron.py:118-230), on a device-resident covariance S (pq x pq).
//
// Streaming passes over S (HBM-bound), with S4[i,r,j,c] =
// S[i*q + r, j*q + c]:
//   stats  : |S|_F^2, block sums A0 = sum_rc S4 / q^2, non-finite count,
//            diagonal min/max                     (src/lrkron.py:100-115,151,173-175)
//   b-step : b[r,c] = sum_ij S4[i,r,j,c] conj(A[i,j]) / |A|^2, plus |b|^2 partials
//                                                  (src/lrkron.py:185-195)
//   V-step : V[i,j] = sum_rc S4[i,r,j,c] conj(b[r,c])  (src/lrkron.py:197-205)
//   tail   : one CTA: A = EIG_ra(V / |b|^2) by Jacobi, expanded-norm residual,
//            stall test                           (src/lrkron.py:207-221)
// Every reduction is per-CTA partials + one fixed-order pass: bitwise
// reproducible. The final temporal factor is EIG_rb(b) (src/lrkron.py:223),
// computed once by heig_top and reused by build_filter.
#include <algorithm>

#include "lrkron_dev.cuh"

namespace {
constexpr int ST_ROWS = 8;   // rows of S per stats CTA
constexpr int V_ROWS = 8;    // rows of S per V-step CTA
constexpr int STAT_STRIDE = 4 + 2 * kMaxP;

// Deterministic warp-strided sum of vals[k * stride], k < count: lane-fixed
// partial sums then a fixed shuffle tree. Result valid in every lane.
__device__ __forceinline__ double warp_sum_strided(const double* __restrict__ vals, int count,
                                                   int stride) {
  const int l = threadIdx.x & 31;
  double acc = 0.0;
  for (int k = l; k < count; k += 32) acc += vals[(size_t)k * stride];
  return warp_sum(acc);
}

// partial layout per CTA: [fro2, nonfinite, dmin, dmax, blocksum(j).re/im ...]
template <int P>
__global__ void __launch_bounds__(NT) stats_kernel(const cplx* __restrict__ S, int q,
                                                   double* __restrict__ part) {
  __shared__ double sh[32];
  const int64_t d = (int64_t)P * q;
  const int i = blockIdx.y;                    // block row
  const int r0 = blockIdx.x * ST_ROWS;         // row within block
  const int rows = min(ST_ROWS, q - r0);
  double fro = 0.0, bad = 0.0, dmin = 1e308, dmax = -1e308;
  double bs[2 * P];
#pragma unroll
  for (int j = 0; j < 2 * P; ++j) bs[j] = 0.0;
  for (int rr = 0; rr < rows; ++rr) {
    const int64_t a = (int64_t)i * q + r0 + rr;
    const cplx* row = S + a * d;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      // four independent streaming loads in flight per thread (S is read once here)
      for (int c0 = threadIdx.x; c0 < q; c0 += 4 * NT) {
        cplx v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = (c0 + u * NT < q) ? __ldcs(&row[(int64_t)j * q + c0 + u * NT]) : cmk(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!isfinite(v[u].x) || !isfinite(v[u].y)) bad += 1.0;
          fro = fma(v[u].x, v[u].x, fro);
          fro = fma(v[u].y, v[u].y, fro);
          bs[2 * j] += v[u].x;
          bs[2 * j + 1] += v[u].y;
        }
      }
    }
    if (threadIdx.x == 0) {
      const double dv = row[a].x;
      dmin = fmin(dmin, dv);
      dmax = fmax(dmax, dv);
    }
  }
  double* out = part + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * STAT_STRIDE;
  fro = block_sum<NT>(fro, sh);
  bad = block_sum<NT>(bad, sh);
  if (threadIdx.x == 0) {
    out[0] = fro;
    out[1] = bad;
    out[2] = dmin;
    out[3] = dmax;
  }
#pragma unroll
  for (int j = 0; j < 2 * P; ++j) {
    const double v = block_sum<NT>(bs[j], sh);
    if (threadIdx.x == 0) out[4 + j] = v;
  }
}

// Reduce stats partials -> fro, A0 (= blocksum / q^2), |A0|^2; diag stats.
// One CTA; every sum is a fixed-order warp reduction (deterministic).
__global__ void __launch_bounds__(NT) init_kernel(const double* __restrict__ part, int nblk_x,
                                                  int P, int q, IterState* st, double* host_diag) {
  __shared__ double red[4 + 2 * kMaxP * kMaxP];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nrec = nblk_x * P;
  const int nq = 2 + 2 * P * P;  // fro2, bad, then A0 re/im per (i, j)
  for (int k = w; k < nq; k += NT / 32) {
    double v;
    if (k < 2) {
      v = warp_sum_strided(part + k, nrec, STAT_STRIDE);
    } else {
      const int e = (k - 2) >> 1, ri = (k - 2) & 1;
      const int i = e / P, j = e % P;
      v = warp_sum_strided(part + (size_t)i * nblk_x * STAT_STRIDE + 4 + 2 * j + ri, nblk_x,
                           STAT_STRIDE);
    }
    if (l == 0) red[k] = v;
  }
  if (w == 0) {
    double mn = 1e308, mx = -1e308;
    for (int k = l; k < nrec; k += 32) {
      mn = fmin(mn, part[(size_t)k * STAT_STRIDE + 2]);
      mx = fmax(mx, part[(size_t)k * STAT_STRIDE + 3]);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (l == 0) {
      red[nq] = mn;
      red[nq + 1] = mx;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double qq = (double)q * (double)q;
    double na2 = 0.0;
    for (int e = 0; e < P * P; ++e) {
      const cplx a = cmk(red[2 + 2 * e] / qq, red[3 + 2 * e] / qq);
      st->A[e] = a;
      st->Aconj[e] = cmk(a.x, -a.y);
      na2 += cabs2(a);
    }
    st->fro2 = red[0];
    st->fro = sqrt(red[0]);
    st->na2 = na2;
    st->eta_prev = INFINITY;
    st->status = 0;
    st->converged = 0;
    st->iteration = 0;
    host_diag[0] = red[1];
    host_diag[1] = red[nq];
    host_diag[2] = red[nq + 1];
    host_diag[3] = st->fro;
    host_diag[4] = na2;
  }
}

// b[r,c] = sum_ij S4[i,r,j,c] conj(A[i,j]) / |A|^2 ; partial |b|^2 per CTA
template <int P>
__global__ void __launch_bounds__(NT) bstep_kernel(const cplx* __restrict__ S, int q,
                                                   const IterState* __restrict__ st,
                                                   cplx* __restrict__ b, double* __restrict__ part,
                                                   double* __restrict__ bdiag = nullptr) {
  __shared__ cplx ca[P * P];
  __shared__ double sh[32];
  for (int e = threadIdx.x; e < P * P; e += NT) ca[e] = st->Aconj[e];
  __syncthreads();
  const double na2 = st->na2;
  const int64_t d = (int64_t)P * q;
  const int r = blockIdx.y;
  const int c = blockIdx.x * NT + threadIdx.x;
  double nb = 0.0;
  if (c < q) {
    cplx acc = cmk(0, 0);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const cplx* row = S + ((int64_t)i * q + r) * d + c;
#pragma unroll
      for (int j = 0; j < P; ++j) cfma(acc, row[(int64_t)j * q], ca[i * P + j]);
    }
    acc = cmk(acc.x / na2, acc.y / na2);
    b[(int64_t)r * q + c] = acc;
    if (bdiag && c == r) bdiag[r] = acc.x;  // Re diag(b), contiguous for the eigensolver's start block
    nb = cabs2(acc);
  }
  nb = block_sum<NT>(nb, sh);
  if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = nb;
}

// V partials: CTA (x = row chunk, y = block row i) -> part[(i, x)][j]
template <int P>
__global__ void __launch_bounds__(NT) vstep_kernel(const cplx* __restrict__ S, int q,
                                                   const cplx* __restrict__ b,
                                                   cplx* __restrict__ part) {
  __shared__ double sh[32];
  const int64_t d = (int64_t)P * q;
  const int i = blockIdx.y;
  const int r0 = blockIdx.x * V_ROWS;
  const int rows = min(V_ROWS, q - r0);
  double ar[P], ai[P];
#pragma unroll
  for (int j = 0; j < P; ++j) ar[j] = ai[j] = 0.0;
  for (int rr = 0; rr < rows; ++rr) {
    const int r = r0 + rr;
    const cplx* row = S + ((int64_t)i * q + r) * d;
    const cplx* brow = b + (int64_t)r * q;
    for (int c = threadIdx.x; c < q; c += NT) {
      const cplx bv = brow[c];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const cplx s = row[(int64_t)j * q + c];
        // s * conj(bv)
        ar[j] = fma(s.x, bv.x, ar[j]);
        ar[j] = fma(s.y, bv.y, ar[j]);
        ai[j] = fma(s.y, bv.x, ai[j]);
        ai[j] = fma(-s.x, bv.y, ai[j]);
      }
    }
  }
  cplx* out = part + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * P;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const double re = block_sum<NT>(ar[j], sh);
    const double im = block_sum<NT>(ai[j], sh);
    if (threadIdx.x == 0) out[j] = cmk(re, im);
  }
}

// One CTA: reduce V and |b|^2, then spatial_update (streaming path).
__global__ void __launch_bounds__(NT) tail_kernel(const cplx* __restrict__ vpart, int nvx,
                                                  const double* __restrict__ bpart, int nbp,
                                                  int P, int ra, double tol, IterState* st,
                                                  cplx* __restrict__ spatial_out,
                                                  double* __restrict__ host_out) {
  extern __shared__ __align__(16) char sm[];
  __shared__ cplx V[kMaxP * kMaxP];
  __shared__ cplx Anew[kMaxP * kMaxP];
  __shared__ double lam[kMaxP];
  __shared__ double nb2_s, eta_s;
  __shared__ int bad_s, conv_s;
  __shared__ double red_sh[32];
  const int tid = threadIdx.x;
  {
    double acc = 0.0;
    for (int k = tid; k < nbp; k += NT) acc += bpart[k];
    acc = block_sum<NT>(acc, red_sh);
    if (tid == 0) nb2_s = acc;
  }
  {
    const int w = tid >> 5, l = tid & 31;
    for (int k = w; k < 2 * P * P; k += NT / 32) {
      const int e = k >> 1, ri = k & 1;
      const int i = e / P, j = e % P;
      const double v = warp_sum_strided((const double*)vpart + ((size_t)i * nvx * P + j) * 2 + ri,
                                        nvx, 2 * P);
      if (l == 0) {
        if (ri) V[e].y = v;
        else V[e].x = v;
      }
    }
  }
  __syncthreads();
  const double nb2 = nb2_s;
  if (nb2 == 0.0) {
    if (tid == 0) {
      st->status = KST_ERR_DEGENERATE;
      host_out[0] = KST_ERR_DEGENERATE;
    }
    return;
  }
  const int rc = spatial_update(V, nb2, P, ra, tol, st, sm, Anew, lam, &bad_s, &eta_s, &conv_s);
  if (tid == 0) {
    if (rc) {
      host_out[0] = rc;
    } else {
      for (int e = 0; e < P * P; ++e) spatial_out[e] = Anew[e];
      host_out[0] = 0;
      host_out[1] = eta_s;
      host_out[2] = conv_s;
      host_out[3] = st->na2;
    }
  }
}

// ---------------------------------------------------------------- M path (P <= 4)
// b = R^T conj(a) / |a|^2 and V = R conj(b) with R the P^2 x q^2 rearrangement
// (src/rearrange.py:1-20), so with M = R R^H (P^2 x P^2, Hermitian):
//   |b|^2 = a^H M a / |a|^4,   V = M a / |a|^2.
// One pass over S yields M together with |S|_F^2, the block sums A0 and the
// validation scans; every iteration then runs on the device with no pass
// over S and no host round trip. The final b needs one last b-step pass.
constexpr int MG_ROWS = 4;   // rows r per CTA
constexpr int MG_TILE = 64;  // positions c per smem tile


// partial: [fro2, bad, dmin, dmax, A0 re/im (2U), M upper re/im (2E)]
template <int P>
__global__ void __launch_bounds__(NT) mgram_kernel(const cplx* __restrict__ S, int q,
                                                   double* __restrict__ part) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E;
  constexpr int G = NT / E > 0 ? NT / E : 1;  // position groups for the M entries
  __shared__ cplx sv[MG_TILE][U + 1];
  __shared__ double sh[32];
  __shared__ int eu[E], ev[E];
  const int64_t d = (int64_t)P * q;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int k = 0;
    for (int u = 0; u < U; ++u)
      for (int v = u; v < U; ++v) {
        eu[k] = u;
        ev[k] = v;
        ++k;
      }
  }
  const int my_e = tid % E, my_g = tid / E;
  const bool m_active = my_g < G && tid < G * E;
  double mr = 0.0, mi = 0.0, fro = 0.0, bad = 0.0, dmin = 1e308, dmax = -1e308;
  double bs[2 * U];
#pragma unroll
  for (int u = 0; u < 2 * U; ++u) bs[u] = 0.0;
  const int r0 = blockIdx.x * MG_ROWS;
  for (int rr = 0; rr < MG_ROWS && r0 + rr < q; ++rr) {
    const int r = r0 + rr;
    for (int c0 = 0; c0 < q; c0 += MG_TILE) {
      __syncthreads();
      for (int e = tid; e < MG_TILE * U; e += NT) {
        const int u = e / MG_TILE, p = e % MG_TILE;  // consecutive threads -> consecutive c
        const int i = u / P, j = u % P, c = c0 + p;
        cplx v = cmk(0, 0);
        if (c < q) {
          v = S[((int64_t)i * q + r) * d + (int64_t)j * q + c];
          if (!isfinite(v.x) || !isfinite(v.y)) bad += 1.0;
          fro = fma(v.x, v.x, fro);
          fro = fma(v.y, v.y, fro);
          if (i == j && c == r) {
            dmin = fmin(dmin, v.x);
            dmax = fmax(dmax, v.x);
          }
        }
        sv[p][u] = v;
      }
      __syncthreads();
      // block sums: thread u-owner accumulates over the tile in fixed order
      if (tid < U) {
        double sr = 0.0, si = 0.0;
        for (int p = 0; p < MG_TILE; ++p) {
          sr += sv[p][tid].x;
          si += sv[p][tid].y;
        }
        bs[2 * tid] += sr;
        bs[2 * tid + 1] += si;
      }
      if (m_active) {
        const int u = eu[my_e], v = ev[my_e];
        for (int p = my_g; p < MG_TILE; p += G) {
          const cplx a = sv[p][u], b = sv[p][v];  // M_uv += s_u conj(s_v)
          mr = fma(a.x, b.x, mr);
          mr = fma(a.y, b.y, mr);
          mi = fma(a.y, b.x, mi);
          mi = fma(-a.x, b.y, mi);
        }
      }
    }
  }
  double* out = part + (size_t)blockIdx.x * Dm::STRIDE;
  fro = block_sum<NT>(fro, sh);
  bad = block_sum<NT>(bad, sh);
  // dmin/dmax: fixed-order smem reduction
  __shared__ double smn[NT], smx[NT];
  smn[tid] = dmin;
  smx[tid] = dmax;
  __syncthreads();
  if (tid == 0) {
    double a = 1e308, b = -1e308;
    for (int k = 0; k < NT; ++k) {
      a = fmin(a, smn[k]);
      b = fmax(b, smx[k]);
    }
    out[0] = fro;
    out[1] = bad;
    out[2] = a;
    out[3] = b;
  }
  if (tid < U) {
    out[4 + 2 * tid] = bs[2 * tid];
    out[4 + 2 * tid + 1] = bs[2 * tid + 1];
  }
  // M: sum the G position groups of each entry in fixed order
  __syncthreads();
  smn[tid] = m_active ? mr : 0.0;
  smx[tid] = m_active ? mi : 0.0;
  __syncthreads();
  if (tid < E) {
    double ar = 0.0, ai = 0.0;
    for (int g = 0; g < G; ++g) {
      ar += smn[g * E + tid];
      ai += smx[g * E + tid];
    }
    out[4 + 2 * U + 2 * tid] = ar;
    out[4 + 2 * U + 2 * tid + 1] = ai;
  }
}

// Register variant for P <= 3: each thread owns positions (r, c) (loads
// coalesced over c), keeps its s-vector and the whole upper triangle of its
// partial M in registers, then one fixed-order CTA reduction. Same partial
// record as mgram_kernel. ~2x fewer instructions than the smem variant and no
// shared-memory traffic in the hot loop.
template <int P>
__global__ void __launch_bounds__(NT, 1) mgram_reg_kernel(const cplx* __restrict__ S, int q,
                                                          double* __restrict__ part) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E, R = Dm::STRIDE;
  __shared__ double red[NT / 32][R];
  const int64_t d = (int64_t)P * q;
  const int tid = threadIdx.x;
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  acc[2] = 1e308;
  acc[3] = -1e308;
  const int r0 = blockIdx.x * MG_ROWS;
  for (int rr = 0; rr < MG_ROWS && r0 + rr < q; ++rr) {
    const int r = r0 + rr;
    for (int c = tid; c < q; c += NT) {
      cplx sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = u / P, j = u % P;
        sv[u] = S[((int64_t)i * q + r) * d + (int64_t)j * q + c];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const cplx v = sv[u];
        if (!isfinite(v.x) || !isfinite(v.y)) acc[1] += 1.0;
        acc[0] = fma(v.x, v.x, acc[0]);
        acc[0] = fma(v.y, v.y, acc[0]);
        acc[4 + 2 * u] += v.x;
        acc[4 + 2 * u + 1] += v.y;
        if (u / P == u % P && c == r) {
          acc[2] = fmin(acc[2], v.x);
          acc[3] = fmax(acc[3], v.x);
        }
      }
      int k = 0;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = u; v < U; ++v, ++k) {
          const cplx a = sv[u], b = sv[v];  // M_uv += s_u conj(s_v)
          double& mr = acc[4 + 2 * U + 2 * k];
          double& mi = acc[4 + 2 * U + 2 * k + 1];
          mr = fma(a.x, b.x, mr);
          mr = fma(a.y, b.y, mr);
          mi = fma(a.y, b.x, mi);
          mi = fma(-a.x, b.y, mi);
        }
    }
  }
  // fixed-order reduction: warp shuffle tree, then warps in order
  const int w = tid >> 5, l = tid & 31;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, v, o);
      v = (k == 2) ? fmin(v, x) : (k == 3) ? fmax(v, x) : v + x;
    }
    if (l == 0) red[w][k] = v;
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * R;
  for (int k = tid; k < R; k += NT) {
    double v = red[0][k];
    for (int ww = 1; ww < NT / 32; ++ww)
      v = (k == 2) ? fmin(v, red[ww][k]) : (k == 3) ? fmax(v, red[ww][k]) : v + red[ww][k];
    out[k] = v;
  }
  (void)E;
}

// Split register variant (P = 3: 45 complex M entries do not fit one thread's
// registers). The CTA is NG groups of 128 threads over `rows` rows of S4.
// Tiles of 128 positions x U blocks stream through an MS_STAGES-deep cp.async
// ring in smem (loads decoupled from registers, so the SM keeps ~55 KB in
// flight); every group reads each position's s-vector from the ring and
// group g owns a contiguous chunk [ms_bound(g), ms_bound(g+1)) of the upper
// triangle; group 0 also owns the scans and block sums. Same partial record
// as mgram_kernel.
constexpr int MS_NTG = 128;  // threads per group = positions per tile
#ifndef KST_MS_STAGES
#define KST_MS_STAGES 4
#endif
#ifndef KST_MS_NG
#define KST_MS_NG 2  // thread groups splitting M's upper triangle (P = 3; A/B: 2 159 us, 3 169, 4 177)
#endif
constexpr int MS_STAGES = KST_MS_STAGES;
// chunk bounds: group 0 (which also carries the scans) takes a smaller share
__host__ __device__ constexpr int ms_bound(int E, int NG, int g) {
  return g <= 0 ? 0
         : g >= NG ? E
         : (E / NG - (E / NG / 2 < 6 ? E / NG / 2 : 6)) +
               (E - (E / NG - (E / NG / 2 < 6 ? E / NG / 2 : 6))) * (g - 1) / (NG - 1);
}
template <int P, int NG, int G>
__device__ __forceinline__ void mgram_split_group(const cplx* __restrict__ S, int q, int r0,
                                                  int rows, int tg, cplx* __restrict__ ring,
                                                  double (*red)[MDims<P>::STRIDE]) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E;
  constexpr int K0 = ms_bound(E, NG, G), K1 = ms_bound(E, NG, G + 1), NK = K1 - K0;
  constexpr int NS = (G == 0) ? 4 + 2 * U : 0;  // scan + block-sum slots
  const int64_t d = (int64_t)P * q;
  double st[NS > 0 ? NS : 1], m[2 * NK];
#pragma unroll
  for (int k = 0; k < NS; ++k) st[k] = 0.0;
  if (NS) {
    st[2] = 1e308;
    st[3] = -1e308;
  }
#pragma unroll
  for (int k = 0; k < 2 * NK; ++k) m[k] = 0.0;
  const int nct = (q + MS_NTG - 1) / MS_NTG;
  const int ntile = rows * nct;
  // every thread of the CTA issues its share of each tile: KPT fixed (u, pp)
  // slots whose global offsets are computed once (no index division per tile)
  constexpr int KPT = (U + NG - 1) / NG;
  int64_t goff[KPT];
  int eoff[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int e = threadIdx.x + k * NG * MS_NTG;
    eoff[k] = e < U * MS_NTG ? e : -1;
    const int u = e / MS_NTG, pp = e % MS_NTG;
    goff[k] = (int64_t)(u / P) * q * d + (int64_t)(u % P) * q + pp;
  }
  int is_r = r0, is_c = 0, is_s = 0, is_t = 0;  // next tile to issue: row, col tile, stage
  auto issue = [&]() {
    if (is_t < ntile) {
      cplx* buf = ring + (size_t)is_s * U * MS_NTG;
      const cplx* src = S + (int64_t)is_r * d + is_c * MS_NTG;
#pragma unroll
      for (int k = 0; k < KPT; ++k)
        if (eoff[k] >= 0 && is_c * MS_NTG + (eoff[k] % MS_NTG) < q)
          cp_async16(buf + eoff[k], src + goff[k]);
    }
    cp_async_commit();
    ++is_t;
    is_s = (is_s + 1 == MS_STAGES) ? 0 : is_s + 1;
    if (++is_c == nct) {
      is_c = 0;
      ++is_r;
    }
  };
#pragma unroll 1
  for (int t = 0; t < MS_STAGES - 1; ++t) issue();
  int cr = r0, ccol = 0, cs = 0;  // tile being consumed
#pragma unroll 1
  for (int t = 0; t < ntile; ++t) {
    cp_async_wait<MS_STAGES - 2>();
    __syncthreads();  // tile t visible to all; buffer of tile t-1 free
    issue();
    const int r = cr, c = ccol * MS_NTG + tg;
    const cplx* buf = ring + (size_t)cs * U * MS_NTG + tg;
    cs = (cs + 1 == MS_STAGES) ? 0 : cs + 1;
    if (++ccol == nct) {
      ccol = 0;
      ++cr;
    }
    if (c < q) {
      cplx sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) sv[u] = buf[u * MS_NTG];
      if (NS) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const cplx v = sv[u];
          if (!isfinite(v.x) || !isfinite(v.y)) st[1] += 1.0;
          st[0] = fma(v.x, v.x, st[0]);
          st[0] = fma(v.y, v.y, st[0]);
          st[4 + 2 * u] += v.x;
          st[4 + 2 * u + 1] += v.y;
          if (u / P == u % P && c == r) {
            st[2] = fmin(st[2], v.x);
            st[3] = fmax(st[3], v.x);
          }
        }
      }
      int k = 0;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = u; v < U; ++v, ++k)
          if (k >= K0 && k < K1) {
            const cplx a = sv[u], b = sv[v];  // M_uv += s_u conj(s_v)
            double& mr = m[2 * (k - K0)];
            double& mi = m[2 * (k - K0) + 1];
            mr = fma(a.x, b.x, mr);
            mr = fma(a.y, b.y, mr);
            mi = fma(a.y, b.x, mi);
            mi = fma(-a.x, b.y, mi);
          }
    }
  }
  cp_async_wait<0>();
  const int w = tg >> 5, l = tg & 31, wrow = G * (MS_NTG / 32) + w;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    double v = st[k];
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, v, o);
      v = (k == 2) ? fmin(v, x) : (k == 3) ? fmax(v, x) : v + x;
    }
    if (l == 0) red[wrow][k] = v;
  }
#pragma unroll
  for (int k = 0; k < 2 * NK; ++k) {
    double v = m[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[wrow][4 + 2 * U + 2 * K0 + k] = v;
  }
}

template <int P, int NG>
__global__ void __launch_bounds__(NG * MS_NTG, 1) mgram_split_kernel(const cplx* __restrict__ S,
                                                                     int q, int rows_per,
                                                                     double* __restrict__ part) {
  static_assert(NG >= 1 && NG <= 4, "mgram_split_kernel: 1..4 groups");
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E, R = Dm::STRIDE, WG = MS_NTG / 32;
  __shared__ double red[NG * WG][R];
  extern __shared__ __align__(16) unsigned char ms_dyn[];
  cplx* ring = (cplx*)ms_dyn;  // MS_STAGES x U x MS_NTG
  const int g = threadIdx.x / MS_NTG, tg = threadIdx.x % MS_NTG;
  const int r0 = blockIdx.x * rows_per;
  const int rows = min(rows_per, q - r0);
  // the groups run different instantiations; their barriers are CTA-wide bar.sync 0
  // reached the same number of times by every warp
  if (g == 0) mgram_split_group<P, NG, 0>(S, q, r0, rows, tg, ring, red);
  if (NG > 1 && g == 1) mgram_split_group<P, NG, (NG > 1 ? 1 : 0)>(S, q, r0, rows, tg, ring, red);
  if (NG > 2 && g == 2) mgram_split_group<P, NG, (NG > 2 ? 2 : 0)>(S, q, r0, rows, tg, ring, red);
  if (NG > 3 && g == 3) mgram_split_group<P, NG, (NG > 3 ? 3 : 0)>(S, q, r0, rows, tg, ring, red);
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * R;
  for (int k = threadIdx.x; k < R; k += NG * MS_NTG) {
    // owner group: the largest g with ms_bound(g) <= entry (scans belong to group 0)
    int owner = 0;
    if (k >= 4 + 2 * U) {
      const int ent = (k - 4 - 2 * U) >> 1;
      for (int gg = 1; gg < NG; ++gg)
        if (ms_bound(E, NG, gg) <= ent) owner = gg;
    }
    double v = red[owner * WG][k];
    for (int ww = 1; ww < WG; ++ww) {
      const double x = red[owner * WG + ww][k];
      v = (k == 2) ? fmin(v, x) : (k == 3) ? fmax(v, x) : v + x;
    }
    out[k] = v;
  }
}

// Reduce mgram partials (fixed order) and run ALL iterations in one CTA.
// Outputs: spatial (final A), residuals[max_iter], info[0..3] = {status,
// iterations, converged, pad}, host_diag[0..4] = {bad, dmin, dmax, fro, na2_0};
// st->Aconj / st->na2 are left holding the A that produced the final b.
template <int P>
__global__ void __launch_bounds__(NT) m_iterate_kernel(const double* __restrict__ part, int nblk,
                                                       int q, int ra, double tol, int max_iter,
                                                       IterState* st, cplx* __restrict__ spatial_out,
                                                       double* __restrict__ residuals,
                                                       double* __restrict__ info,
                                                       double* __restrict__ host_diag) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E;
  extern __shared__ __align__(16) char sm[];
  __shared__ double red[4 + 2 * U + 2 * E];
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int k = w; k < Dm::STRIDE; k += NT / 32) {
    double v;
    if (k == 2 || k == 3) {
      double m = (k == 2) ? 1e308 : -1e308;
      for (int b = l; b < nblk; b += 32)
        m = (k == 2) ? fmin(m, part[(size_t)b * Dm::STRIDE + k]) : fmax(m, part[(size_t)b * Dm::STRIDE + k]);
      v = (k == 2) ? warp_min(m) : warp_max(m);
    } else {
      v = warp_sum_strided(part + k, nblk, Dm::STRIDE);
    }
    if (l == 0) red[k] = v;
  }
  __syncthreads();
  m_iterations<P>(red, q, ra, tol, max_iter, st, sm, spatial_out, residuals, info, host_diag);
}

__global__ void zero_kernel(cplx* p, int64_t count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = cmk(0, 0);
}

}  // namespace

namespace kst {

int lrkron(kst_ctx* ctx, const cplx* S, int p, int q, int ra, int rb, double tol, int max_iter,
           int validate, cplx* spatial, cplx* temporal, cplx* tb_vectors, double* tb_values,
           FitOut* fit, cplx* iter_spatial, cplx* iter_b, cudaStream_t st) {
  if (p < 1 || q < 1) return set_err(ctx, KST_ERR_DIMENSION, "block shape must be positive");
  if (p > kMaxP) return set_err(ctx, KST_ERR_DIMENSION, "p=%d exceeds the supported %d channels", p, kMaxP);
  const int64_t d = (int64_t)p * q;
  // stats pass
  const int nbx = (q + ST_ROWS - 1) / ST_ROWS;
  const size_t stat_stride = STAT_STRIDE;
  const int nvx = (q + V_ROWS - 1) / V_ROWS;
  const int nbb = (q + NT - 1) / NT;
  // M path: small P, valid ranks, no per-iteration b copies requested
  static const bool mpath_env = !(getenv("KST_LRKRON_MPATH") && atoi(getenv("KST_LRKRON_MPATH")) == 0);
  const bool mpath = mpath_env && p <= 4 && !iter_b && !iter_spatial && ra >= 1 && ra <= p &&
                     rb >= 1 && rb <= q && max_iter >= 1;
  // P = 3: one wave of pipelined CTAs (rows_per rows each); others MG_ROWS rows
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int rows_per = p == 3 ? (q + nsm - 1) / nsm : MG_ROWS;
  const int nblk = (q + rows_per - 1) / rows_per;
  size_t rec = 0;
  KST_DISPATCH_P(p, (rec = MDims<PP>::STRIDE));
  // WS_PART is taken ONCE, sized for every use below (stats / V / b partials and
  // the M-path records): a second ws_get on a grown slot would free the buffer
  // the b-step partials still point into.
  size_t part_bytes = std::max(sizeof(double) * stat_stride * p * nbx,
                               sizeof(cplx) * (size_t)p * nvx * p + sizeof(double) * (size_t)q * (nbb + 1) + 64);
  if (mpath) part_bytes = std::max(part_bytes, sizeof(double) * rec * nblk + 64);
  char* small = (char*)ws_get(ctx, WS_SMALL, sizeof(IterState) + 256);
  double* part = (double*)ws_get(ctx, WS_PART, part_bytes);
  cplx* b = (cplx*)ws_get(ctx, WS_B, sizeof(cplx) * (size_t)q * q);
  // one pinned staging buffer: [0, 64) small scalars, [64, ...) M-path residuals
  double* hbuf = (double*)pinned_get(ctx, sizeof(double) * (64 + std::max(max_iter, 1) + 32));
  if (!small || !part || !b || !hbuf) return set_err(ctx, KST_ERR_CUDA, "lrkron: workspace");
  IterState* state = (IterState*)small;

  double* mres = nullptr;
  double* minfo = nullptr;
  if (mpath) {
    double* mpart = part;  // consumed by m_iterate_kernel before bstep reuses the slot (same stream)
    double* dres = (double*)ws_get(ctx, WS_VALS, sizeof(double) * (max_iter + 8));
    mres = hbuf ? hbuf + 64 : nullptr;
    if (!mpart || !dres || !mres) return set_err(ctx, KST_ERR_CUDA, "lrkron: workspace");
    minfo = dres + max_iter;
    const size_t jsm = jac_smem_bytes(p);
    switch (p) {
      case 1:
        mgram_reg_kernel<1><<<nblk, NT, 0, st>>>(S, q, mpart);
        m_iterate_kernel<1><<<1, NT, jsm, st>>>(mpart, nblk, q, ra, tol, max_iter, state, spatial,
                                                 dres, minfo, (double*)(small + sizeof(IterState)));
        break;
      case 2:
        mgram_reg_kernel<2><<<nblk, NT, 0, st>>>(S, q, mpart);
        m_iterate_kernel<2><<<1, NT, jsm, st>>>(mpart, nblk, q, ra, tol, max_iter, state, spatial,
                                                 dres, minfo, (double*)(small + sizeof(IterState)));
        break;
      case 3:
      {
        constexpr size_t ring = sizeof(cplx) * MS_STAGES * 9 * MS_NTG;
        KST_CUDA(ctx, cudaFuncSetAttribute(mgram_split_kernel<3, KST_MS_NG>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring));
        mgram_split_kernel<3, KST_MS_NG><<<nblk, KST_MS_NG * MS_NTG, ring, st>>>(S, q, rows_per, mpart);
      }
        m_iterate_kernel<3><<<1, NT, jsm, st>>>(mpart, nblk, q, ra, tol, max_iter, state, spatial,
                                                 dres, minfo, (double*)(small + sizeof(IterState)));
        break;
      default:
        mgram_kernel<4><<<nblk, NT, 0, st>>>(S, q, mpart);
        m_iterate_kernel<4><<<1, NT, jsm, st>>>(mpart, nblk, q, ra, tol, max_iter, state, spatial,
                                                 dres, minfo, (double*)(small + sizeof(IterState)));
        break;
    }
    ctx->launches += 1;  // + 1 in KST_LAUNCH: mgram + m_iterate
    KST_LAUNCH(ctx);
    KST_CUDA(ctx, cudaMemcpyAsync(mres, dres, sizeof(double) * (max_iter + 3), cudaMemcpyDeviceToHost, st));
  } else {
    KST_DISPATCH_P(p, (stats_kernel<PP><<<dim3(nbx, p), NT, 0, st>>>(S, q, part)));
    KST_LAUNCH(ctx);
    init_kernel<<<1, NT, 0, st>>>(part, nbx, p, q, state, (double*)(small + sizeof(IterState)));
    KST_LAUNCH(ctx);
  }
  KST_CUDA(ctx, cudaMemcpyAsync(hbuf, small + sizeof(IterState), 5 * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  const double bad = hbuf[0], dmin = hbuf[1], dmax = hbuf[2], fro = hbuf[3];
  double na2 = hbuf[4];
  if (bad > 0) return set_err(ctx, KST_ERR_DATA, "covariance contains non-finite entries");
  if (validate) {
    KST_TRY(herm_check(ctx, S, (int)d, st));
    if (dmin < -1e-8 * std::max(dmax, 0.0))
      return set_err(ctx, KST_ERR_DATA, "covariance has a negative diagonal, not PSD");
  }
  if (ra < 1 || ra > p)
    return set_err(ctx, KST_ERR_DIMENSION, "spatial rank must be in [1, %d], got %d", p, ra);
  if (rb < 1 || rb > q)
    return set_err(ctx, KST_ERR_DIMENSION, "temporal rank must be in [1, %d], got %d", q, rb);
  if (max_iter < 1) return set_err(ctx, KST_ERR_DIMENSION, "max_iter must be >= 1, got %d", max_iter);

  fit->residuals.clear();
  if (fro == 0.0) {
    zero_kernel<<<1, 256, 0, st>>>(spatial, (int64_t)p * p);
    KST_LAUNCH(ctx);
    if (temporal) {
      zero_kernel<<<cdiv((int64_t)q * q, 256), 256, 0, st>>>(temporal, (int64_t)q * q);
      KST_LAUNCH(ctx);
    }
    fit->iterations = 0;
    fit->converged = 1;
    fit->residuals.push_back(0.0);
    fit->n_res = 1;
    if (tb_values)
      for (int k = 0; k < rb; ++k) tb_values[k] = 0.0;
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    return KST_OK;
  }

  cplx* vpart = (cplx*)part;
  double* bpart = (double*)(vpart + (size_t)p * nvx * p);
  double* hout = (double*)(small + sizeof(IterState) + 64);
  const size_t tail_smem = jac_smem_bytes(p);
  int iters = 0, conv = 0;
  if (mpath) {
    // all iterations already ran on the device (m_iterate_kernel)
    const int status = (int)mres[max_iter];
    iters = (int)mres[max_iter + 1];
    conv = (int)mres[max_iter + 2];
    if (status == 4) return set_err(ctx, KST_ERR_DEGENERATE, "spatial iterate collapsed to zero");
    if (status == KST_ERR_DEGENERATE)
      return set_err(ctx, KST_ERR_DEGENERATE, "temporal iterate collapsed to zero");
    if (status == KST_ERR_DATA)
      return set_err(ctx, KST_ERR_DATA, "matrix deviates from Hermitian beyond tolerance");
    for (int it = 0; it < iters; ++it) fit->residuals.push_back(mres[it]);
    // final b from the A that entered the last iteration (st->Aconj / st->na2)
    KST_DISPATCH_P(p, (bstep_kernel<PP><<<dim3(nbb, q), NT, 0, st>>>(S, q, state, b, bpart)));
    KST_LAUNCH(ctx);
  }
  for (int it = 0; it < max_iter && !mpath; ++it) {
    if (na2 == 0.0) return set_err(ctx, KST_ERR_DEGENERATE, "spatial iterate collapsed to zero");
    ++iters;
    KST_DISPATCH_P(p, (bstep_kernel<PP><<<dim3(nbb, q), NT, 0, st>>>(S, q, state, b, bpart)));
    KST_LAUNCH(ctx);
    KST_DISPATCH_P(p, (vstep_kernel<PP><<<dim3(nvx, p), NT, 0, st>>>(S, q, b, vpart)));
    KST_LAUNCH(ctx);
    tail_kernel<<<1, NT, tail_smem, st>>>(vpart, nvx, bpart, nbb * q, p, ra, tol, state, spatial, hout);
    KST_LAUNCH(ctx);
    KST_CUDA(ctx, cudaMemcpyAsync(hbuf, hout, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (iter_spatial)
      KST_CUDA(ctx, cudaMemcpyAsync(iter_spatial + (size_t)it * p * p, spatial,
                                    sizeof(cplx) * p * p, cudaMemcpyDeviceToDevice, st));
    if (iter_b)
      KST_CUDA(ctx, cudaMemcpyAsync(iter_b + (size_t)it * q * q, b, sizeof(cplx) * (size_t)q * q,
                                    cudaMemcpyDeviceToDevice, st));
    KST_CUDA(ctx, cudaStreamSynchronize(st));
    const int status = (int)hbuf[0];
    if (status == KST_ERR_DEGENERATE)
      return set_err(ctx, KST_ERR_DEGENERATE, "temporal iterate collapsed to zero");
    if (status == KST_ERR_DATA)
      return set_err(ctx, KST_ERR_DATA, "matrix deviates from Hermitian beyond tolerance");
    fit->residuals.push_back(hbuf[1]);
    na2 = hbuf[3];
    if (hbuf[2] != 0.0) {
      conv = 1;
      break;
    }
  }
  fit->iterations = iters;
  fit->converged = conv;
  fit->n_res = (int)fit->residuals.size();

  // temporal = EIG_rb(b)   (src/lrkron.py:223)
  if (validate) KST_TRY(herm_check(ctx, b, q, st));
  if (rb == q) {
    if (temporal) {
      // (b + b^H)/2 without eig (src/linalg.py:135-136)
      KST_TRY(eig_truncate(ctx, b, q, q, temporal, st));
    }
    return KST_OK;
  }
  const int want = q <= kMaxN ? q : rb;
  std::vector<double> vals(want);
  cplx* U = (cplx*)ws_get(ctx, WS_UB, sizeof(cplx) * (size_t)q * want);
  if (!U) return set_err(ctx, KST_ERR_CUDA, "lrkron: workspace");
  KST_TRY(heig_top(ctx, b, q, want, vals.data(), U, st));
  double top = 0.0;
  for (int k = 0; k < want; ++k) top = std::max(top, std::fabs(vals[k]));
  cplx* Ur = U;
  if (want != rb) {
    Ur = tb_vectors ? tb_vectors : (cplx*)ws_get(ctx, WS_EIG2, sizeof(cplx) * (size_t)q * rb);
    KST_CUDA(ctx, cudaMemcpy2DAsync(Ur, sizeof(cplx) * rb, U, sizeof(cplx) * want,
                                    sizeof(cplx) * rb, q, cudaMemcpyDeviceToDevice, st));
  } else if (tb_vectors) {
    KST_CUDA(ctx, cudaMemcpyAsync(tb_vectors, U, sizeof(cplx) * (size_t)q * rb,
                                  cudaMemcpyDeviceToDevice, st));
    Ur = tb_vectors;
  }
  if (tb_values)
    for (int k = 0; k < rb; ++k) {
      double v = vals[k];
      if (v < 0 && std::fabs(v) <= 1e-10 * top) v = 0.0;
      tb_values[k] = v;
    }
  if (temporal) KST_TRY(truncate_from_pairs(ctx, vals.data(), Ur, q, rb, top, temporal, st));
  KST_CUDA(ctx, cudaStreamSynchronize(st));
  return KST_OK;
}

// Host-sync-free form of lrkron's M-path (p <= 4, rb < q, q > 64), for the
// optimistic kst_pipeline: the same kernels -- mgram, m_iterate (every
// iteration on the device), the final b-step, the top-rb eigenpairs of b by
// heig_top's fixed common-case schedule -- with every outcome left on the
// device: *dres_out = residuals[max_iter] then {status, iterations,
// converged}; *diag_out = {bad, dmin, dmax, fro, na2_0}; *heig_ok = 1 when
// the eigensolver converged in its first round. The caller validates these
// on the device and re-runs the synchronous path when any check fails.
int lrkron_async(kst_ctx* ctx, const cplx* S, int p, int q, int ra, int rb, double tol, int max_iter,
                 cplx* spatial, cplx* tb_vectors, int* heig_ok, const double** tb_vals_dev,
                 const double** dres_out, const double** diag_out, cudaStream_t st) {
  if (p < 1 || p > 4 || q <= kMaxN || ra < 1 || ra > p || rb < 1 || rb >= q || rb > 24 ||
      max_iter < 1)
    return set_err(ctx, KST_ERR_DIMENSION, "lrkron_async: unsupported shape");
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int rows_per = p == 3 ? (q + nsm - 1) / nsm : MG_ROWS;
  const int nblk = (q + rows_per - 1) / rows_per;
  const int nvx = (q + V_ROWS - 1) / V_ROWS, nbb = (q + NT - 1) / NT, nbx = (q + ST_ROWS - 1) / ST_ROWS;
  size_t rec = 0;
  KST_DISPATCH_P(p, (rec = MDims<PP>::STRIDE));
  // the same slots and sizes as lrkron (WS_PART taken once for every use)
  size_t part_bytes = std::max(sizeof(double) * STAT_STRIDE * p * nbx,
                               sizeof(cplx) * (size_t)p * nvx * p + sizeof(double) * (size_t)q * (nbb + 1) + 64);
  part_bytes = std::max(part_bytes, sizeof(double) * rec * nblk + 64);
  char* small = (char*)ws_get(ctx, WS_SMALL, sizeof(IterState) + 256);
  double* part = (double*)ws_get(ctx, WS_PART, part_bytes);
  cplx* b = (cplx*)ws_get(ctx, WS_B, sizeof(cplx) * (size_t)q * q);
  double* dres = (double*)ws_get(ctx, WS_VALS, sizeof(double) * (max_iter + 8));
  if (!small || !part || !b || !dres) return set_err(ctx, KST_ERR_CUDA, "lrkron_async: workspace");
  IterState* state = (IterState*)small;
  double* minfo = dres + max_iter;
  double* diag = (double*)(small + sizeof(IterState));
  const size_t jsm = jac_smem_bytes(p);
  switch (p) {
    case 1:
      mgram_reg_kernel<1><<<nblk, NT, 0, st>>>(S, q, part);
      m_iterate_kernel<1><<<1, NT, jsm, st>>>(part, nblk, q, ra, tol, max_iter, state, spatial,
                                               dres, minfo, diag);
      break;
    case 2:
      mgram_reg_kernel<2><<<nblk, NT, 0, st>>>(S, q, part);
      m_iterate_kernel<2><<<1, NT, jsm, st>>>(part, nblk, q, ra, tol, max_iter, state, spatial,
                                               dres, minfo, diag);
      break;
    case 3: {
      constexpr size_t ring = sizeof(cplx) * MS_STAGES * 9 * MS_NTG;
      KST_CUDA(ctx, cudaFuncSetAttribute(mgram_split_kernel<3, KST_MS_NG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring));
      mgram_split_kernel<3, KST_MS_NG><<<nblk, KST_MS_NG * MS_NTG, ring, st>>>(S, q, rows_per, part);
      m_iterate_kernel<3><<<1, NT, jsm, st>>>(part, nblk, q, ra, tol, max_iter, state, spatial,
                                               dres, minfo, diag);
    } break;
    default:
      mgram_kernel<4><<<nblk, NT, 0, st>>>(S, q, part);
      m_iterate_kernel<4><<<1, NT, jsm, st>>>(part, nblk, q, ra, tol, max_iter, state, spatial,
                                               dres, minfo, diag);
      break;
  }
  ctx->launches += 1;  // + 1 in KST_LAUNCH: mgram + m_iterate
  KST_LAUNCH(ctx);
  // final b from the A that entered the last iteration (st->Aconj / st->na2)
  cplx* vpart = (cplx*)part;
  double* bpart = (double*)(vpart + (size_t)p * nvx * p);
  double* bdiag = bpart + (size_t)q * nbb;
  KST_DISPATCH_P(p, (bstep_kernel<PP><<<dim3(nbb, q), NT, 0, st>>>(S, q, state, b, bpart, bdiag)));
  KST_LAUNCH(ctx);
  KST_TRY(heig_top(ctx, b, q, rb, nullptr, tb_vectors, st, heig_ok, tb_vals_dev, bdiag));
  *dres_out = dres;
  *diag_out = diag;
  return KST_OK;
}

}  // namespace kst
