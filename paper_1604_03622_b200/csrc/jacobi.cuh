// K3: block-cooperative cyclic Jacobi for small complex Hermitian matrices
// (n <= 64), FP64, in shared memory, with the reference's output
// conventions (src/linalg.py:82-121): values descending; runs of values
// within 1e-12 * max|lambda| re-ordered by each vector's dominant index
// (stable); every vector rotated so its dominant entry is real positive.
//
// Parallel ordering: round-robin tournament, m/2 disjoint (p, q) pairs per
// round; each round = rotation parameters -> column update (A and V) ->
// row update (A), separated by __syncthreads.
#pragma once
#include "common.cuh"

#ifndef KST_JAC_BLOCK
#define KST_JAC_BLOCK 0  // 1: the block rounds for n = 3 as well (A/B)
#endif

namespace kstj {

constexpr int kMaxN = 64;

__host__ __device__ inline int jac_ld(int n) { return ((n + 7) / 8) * 8 + 1; }

// shared-memory layout needed by jacobi_smem for dimension n
__host__ __device__ inline size_t jac_smem_bytes(int n) {
  const int ld = jac_ld(n);
  return sizeof(cplx) * 2 * (size_t)n * ld      // A, V
         + sizeof(double) * 4 * (kMaxN / 2)     // c, s, cos/sin phase per pair
         + sizeof(int) * 2 * (kMaxN / 2)        // p, q per pair
         + sizeof(double) * 4 * kMaxN           // values, scratch, phase re/im
         + sizeof(int) * 2 * kMaxN + 64;        // order, pivots, flags
}

struct JacSmem {
  cplx* A;
  cplx* V;
  double *c, *s, *ec, *es;
  int *pp, *pq;
  double* val;
  double* scratch;
  double *phr, *phi;
  int* order;
  int* piv;
  int* flag;
  int ld;
};

__device__ inline JacSmem jac_carve(void* base, int n) {
  JacSmem j;
  j.ld = jac_ld(n);
  char* p = (char*)base;
  j.A = (cplx*)p;
  p += sizeof(cplx) * (size_t)n * j.ld;
  j.V = (cplx*)p;
  p += sizeof(cplx) * (size_t)n * j.ld;
  j.c = (double*)p;
  j.s = j.c + kMaxN / 2;
  j.ec = j.s + kMaxN / 2;
  j.es = j.ec + kMaxN / 2;
  p += sizeof(double) * 4 * (kMaxN / 2);
  j.pp = (int*)p;
  j.pq = j.pp + kMaxN / 2;
  p += sizeof(int) * 2 * (kMaxN / 2);
  j.val = (double*)p;
  j.scratch = j.val + kMaxN;
  j.phr = j.scratch + kMaxN;
  j.phi = j.phr + kMaxN;
  p += sizeof(double) * 4 * kMaxN;
  j.order = (int*)p;
  j.piv = j.order + kMaxN;
  j.flag = j.piv + kMaxN;
  return j;
}

// Load (M/div + (M/div)^H)/2 into A, V = I. M: global or shared, row-major,
// leading dim ldm. div reproduces e.g. eig_truncate(v / |b|^2) (src/lrkron.py:207).
__device__ inline void jac_load_sym(JacSmem& j, const cplx* M, int ldm, int n, double div) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    const cplx x = M[(size_t)r * ldm + c], y = M[(size_t)c * ldm + r];
    // (x + conj(y)) / 2, matching the reference's symmetrisation order
    j.A[r * j.ld + c] = cmk(((x.x / div) + (y.x / div)) / 2.0, ((x.y / div) - (y.y / div)) / 2.0);
    j.V[r * j.ld + c] = cmk(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- n = 3, one thread
// For n = 3 the tournament has one real pair per round -- (0,1), (0,2),
// (1,2) -- so a sweep is three sequential rotations. One thread runs them on
// registers with compile-time indices: the same parameter formulas,
// thresholds, column-then-row update and exact 2x2 diagonal as the block
// rounds, without their four barriers per round (the P x P spatial
// eigenproblems of every LR-Kron iteration and L-mode window).
template <int P_, int Q_>
__device__ __forceinline__ bool jac3_rot(cplx (&a)[3][3], cplx (&v)[3][3], double fro) {
  const double app = a[P_][P_].x, aqq = a[Q_][Q_].x;
  const cplx apq = a[P_][Q_];
  const double r2 = apq.x * apq.x + apq.y * apq.y;
  const double thr2 = fmax(4.84e-32 * fabs(app) * fabs(aqq), 1e-600 + 1e-30 * fro * fro);
  if (!(r2 > thr2)) return false;
  const double rinv = rsqrt(r2);
  const double r = r2 * rinv;
  const double ec = apq.x * rinv, es = apq.y * rinv;
  const double tau = (aqq - app) * (0.5 * rinv);
  const double t = copysign(1.0, tau) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
  const double c = rsqrt(fma(t, t, 1.0));
  const double sn = t * c;
  const cplx emi = cmk(ec, -es), epi = cmk(ec, es);
#pragma unroll
  for (int row = 0; row < 3; ++row) {  // A <- A U, V <- V U on columns (P_, Q_)
    {
      const cplx xp = a[row][P_], wq = cmul(emi, a[row][Q_]);
      a[row][P_] = cmk(c * xp.x - sn * wq.x, c * xp.y - sn * wq.y);
      a[row][Q_] = cmk(sn * xp.x + c * wq.x, sn * xp.y + c * wq.y);
    }
    {
      const cplx xp = v[row][P_], wq = cmul(emi, v[row][Q_]);
      v[row][P_] = cmk(c * xp.x - sn * wq.x, c * xp.y - sn * wq.y);
      v[row][Q_] = cmk(sn * xp.x + c * wq.x, sn * xp.y + c * wq.y);
    }
  }
#pragma unroll
  for (int col = 0; col < 3; ++col) {  // A <- U^H A on rows (P_, Q_)
    const cplx xp = a[P_][col], wq = cmul(epi, a[Q_][col]);
    a[P_][col] = cmk(c * xp.x - sn * wq.x, c * xp.y - sn * wq.y);
    a[Q_][col] = cmk(sn * xp.x + c * wq.x, sn * xp.y + c * wq.y);
  }
  a[P_][P_] = cmk(app - t * r, 0.0);
  a[Q_][Q_] = cmk(aqq + t * r, 0.0);
  a[P_][Q_] = cmk(0.0, 0.0);
  a[Q_][P_] = cmk(0.0, 0.0);
  return true;
}

static __device__ __noinline__ void jac3_thread(JacSmem& j) {
  cplx a[3][3], v[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[r][c] = j.A[r * j.ld + c];
      v[r][c] = j.V[r * j.ld + c];
    }
  double f = 0.0;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) f += cabs2(a[r][c]);
  const double fro = sqrt(f);
  int sweeps = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool any = jac3_rot<0, 1>(a, v, fro);
    any |= jac3_rot<0, 2>(a, v, fro);
    any |= jac3_rot<1, 2>(a, v, fro);
    sweeps = sweep + 1;
    if (!any) break;
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      j.A[r * j.ld + c] = a[r][c];
      j.V[r * j.ld + c] = v[r][c];
    }
    j.val[r] = a[r][r].x;
  }
  j.flag[1] = sweeps;  // diagnostic: sweeps used
}

// Run Jacobi sweeps on j.A (Hermitian), accumulating j.V. On return
// j.val holds the (unsorted) diagonal.
__device__ inline void jac_sweeps(JacSmem& j, int n) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n == 1) {
    if (tid == 0) j.val[0] = j.A[0].x;
    __syncthreads();
    return;
  }
  if (n == 3 && !KST_JAC_BLOCK) {
    if (tid == 0) jac3_thread(j);
    __syncthreads();
    return;
  }
  const int m = (n + 1) & ~1;  // even player count (index n is a bye when n is odd)
  const int npairs = m / 2;
  // Frobenius norm for the absolute rotation floor
  if (tid == 0) {
    double f = 0.0;
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) f += cabs2(j.A[r * j.ld + c]);
    j.scratch[0] = sqrt(f);
  }
  __syncthreads();
  const double fro = j.scratch[0];
  // exact reciprocal-multiply division for the task maps (indices < 2^13, divisors <= 2^12)
  const unsigned magic_n = 0xFFFFFFFFu / (unsigned)n + 1u;
  const unsigned magic_pn = 0xFFFFFFFFu / (unsigned)(npairs * n) + 1u;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (sweep > 0) {
      // would this sweep rotate at all? Every pair's test on the current A
      // (a sweep that rotates nothing leaves A unchanged, so its per-round
      // tests all see this A): the final, empty sweep -- n - 1 rounds of four
      // barriers -- becomes one parallel check with the same thresholds
      int rot = 0;
      for (int e = tid; e < n * n; e += nt) {
        const int a = (int)__umulhi((unsigned)e, magic_n), b = e - a * n;
        if (a < b) {
          const double app = j.A[a * j.ld + a].x, aqq = j.A[b * j.ld + b].x;
          const cplx apq = j.A[a * j.ld + b];
          const double r2 = apq.x * apq.x + apq.y * apq.y;
          const double thr2 = fmax(4.84e-32 * fabs(app) * fabs(aqq), 1e-600 + 1e-30 * fro * fro);
          rot |= r2 > thr2;
        }
      }
      if (!__syncthreads_or(rot)) {
        if (tid == 0) j.flag[1] = sweep;  // diagnostic: sweeps used
        break;
      }
    }
    if (tid == 0) *j.flag = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round) {
      // tournament pairing: player 0 fixed, others rotate
      if (tid < npairs) {
        int a, b;
        if (tid == 0) {
          a = 0;
          b = 1 + (round % (m - 1));
        } else {
          a = 1 + ((round + tid) % (m - 1));
          b = 1 + ((round + m - 1 - tid) % (m - 1));
        }
        if (a > b) {
          int t = a;
          a = b;
          b = t;
        }
        double c = 1.0, s = 0.0, ec = 1.0, es = 0.0;
        if (b < n) {
          const double app = j.A[a * j.ld + a].x, aqq = j.A[b * j.ld + b].x;
          const cplx apq = j.A[a * j.ld + b];
          const double r2 = apq.x * apq.x + apq.y * apq.y;
          // skip rotations already at the rounding floor (relative to the pair
          // and to |A|_F); a tighter floor only cycles on rounding noise.
          // Compared squared: r > max(2.2e-16 sqrt|app aqq|, 1e-15 |A|_F).
          const double thr2 = fmax(4.84e-32 * fabs(app) * fabs(aqq), 1e-600 + 1e-30 * fro * fro);
          if (r2 > thr2) {
            // rsqrt-based parameters: one division on the critical path
            const double rinv = rsqrt(r2);
            const double r = r2 * rinv;
            ec = apq.x * rinv;
            es = apq.y * rinv;  // e^{i phi}
            const double tau = (aqq - app) * (0.5 * rinv);
            const double t = copysign(1.0, tau) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            // post-rotation diagonal (exact 2x2 values)
            j.scratch[2 * tid] = app - t * r;
            j.scratch[2 * tid + 1] = aqq + t * r;
            *j.flag = 1;
          }
        }
        j.pp[tid] = a;
        j.pq[tid] = b;
        j.c[tid] = c;
        j.s[tid] = s;
        j.ec[tid] = ec;
        j.es[tid] = es;
      }
      __syncthreads();
      // column update: A <- A U, V <- V U on columns (p, q)
      for (int e = tid; e < npairs * n * 2; e += nt) {
        const int mat = (int)__umulhi((unsigned)e, magic_pn);  // e / (npairs * n)
        const int rem = e - mat * npairs * n;
        const int k = (int)__umulhi((unsigned)rem, magic_n);   // rem / n
        const int row = rem - k * n;
        const int p = j.pp[k], q = j.pq[k];
        if (q >= n || j.s[k] == 0.0) continue;
        cplx* M = mat ? j.V : j.A;
        const double c = j.c[k], s = j.s[k];
        const cplx emi = cmk(j.ec[k], -j.es[k]);  // e^{-i phi}
        const cplx xp = M[row * j.ld + p], xq = M[row * j.ld + q];
        const cplx wq = cmul(emi, xq);
        M[row * j.ld + p] = cmk(c * xp.x - s * wq.x, c * xp.y - s * wq.y);
        M[row * j.ld + q] = cmk(s * xp.x + c * wq.x, s * xp.y + c * wq.y);
      }
      __syncthreads();
      // row update: A <- U^H A on rows (p, q)
      for (int e = tid; e < npairs * n; e += nt) {
        const int k = (int)__umulhi((unsigned)e, magic_n), col = e - k * n;
        const int p = j.pp[k], q = j.pq[k];
        if (q >= n || j.s[k] == 0.0) continue;
        // the pair's own 2 x 2 block takes its exact post-rotation values
        // (real diagonal, zero off-diagonal) in the same pass
        if (col == p) {
          j.A[p * j.ld + p] = cmk(j.scratch[2 * k], 0.0);
          j.A[q * j.ld + p] = cmk(0.0, 0.0);
          continue;
        }
        if (col == q) {
          j.A[p * j.ld + q] = cmk(0.0, 0.0);
          j.A[q * j.ld + q] = cmk(j.scratch[2 * k + 1], 0.0);
          continue;
        }
        const double c = j.c[k], s = j.s[k];
        const cplx epi = cmk(j.ec[k], j.es[k]);  // e^{i phi}
        const cplx xp = j.A[p * j.ld + col], xq = j.A[q * j.ld + col];
        const cplx wq = cmul(epi, xq);
        j.A[p * j.ld + col] = cmk(c * xp.x - s * wq.x, c * xp.y - s * wq.y);
        j.A[q * j.ld + col] = cmk(s * xp.x + c * wq.x, s * xp.y + c * wq.y);
      }
      __syncthreads();
    }
    const int any = *j.flag;
    __syncthreads();
    if (tid == 0) j.flag[1] = sweep + 1;  // diagnostic: sweeps used
    if (!any) break;
  }
  for (int i = tid; i < n; i += nt) j.val[i] = j.A[i * j.ld + i].x;
  __syncthreads();
}

// ---------------------------------------------------------------- warp Jacobi
// Register-resident cyclic Jacobi for n <= N (N in {4, 8, 16}) run by ONE warp:
// lane l < N owns column l of A and of V; the N-1 rounds of a sweep are
// unrolled at compile time so every row index is static; partner columns and
// the rotation parameters move by warp shuffles (no shared memory, no block
// barriers). Same rotation formulas, thresholds and exact 2x2 diagonal
// update as jac_sweeps. Matrices with n < N are zero-padded; the padded
// indices never rotate (their off-diagonals are exact zeros).
// Reads (M/div + (M/div)^H)/2 (M row-major, leading dim ldm); writes j.V and
// j.val for the first n indices. Call from warp 0 only; follow with
// __syncthreads() and jac_finish(j, n).
template <int N>
__device__ inline void warp_jacobi(JacSmem& j, const cplx* M, int ldm, int n, double div) {
  const int l = threadIdx.x & 31;
  cplx a[N], v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    cplx x = cmk(0, 0);
    if (l < n && k < n) {
      const cplx m1 = M[(size_t)k * ldm + l], m2 = M[(size_t)l * ldm + k];
      x = cmk(((m1.x / div) + (m2.x / div)) / 2.0, ((m1.y / div) - (m2.y / div)) / 2.0);
    }
    a[k] = x;
    v[k] = cmk((k == l) ? 1.0 : 0.0, 0.0);
  }
  // Frobenius norm (absolute rotation floor), identical in every lane
  double f = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) f += cabs2(a[k]);
  f = warp_sum(f);
  const double fro2 = f;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0;
#pragma unroll
    for (int round = 0; round < N - 1; ++round) {
      // partner of lane l in this round (tournament, player 0 fixed)
      int m;
      if (l == 0) m = 1 + round % (N - 1);
      else if (l == 1 + round % (N - 1)) m = 0;
      else {
        const int pos = (l - 1 - round + 2 * (N - 1)) % (N - 1);  // circle position of l
        const int mpos = (N - 1 - pos) % (N - 1);                   // opposite position
        m = 1 + (mpos + round) % (N - 1);
      }
      if (l >= N) m = l;
      const bool is_p = l < m;
      // own diagonal a[l] and the cross element a[m] (row m of own column)
      cplx dl = cmk(0, 0), xm = cmk(0, 0);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (k == l) dl = a[k];
        if (k == m) xm = a[k];
      }
      const double dm = __shfl_sync(0xffffffffu, dl.x, m & 31);
      const double app = is_p ? dl.x : dm, aqq = is_p ? dm : dl.x;
      const cplx apq = is_p ? cconj(xm) : xm;  // A[p][q]
      double c = 1.0, s = 0.0, ec = 1.0, es = 0.0, tr = 0.0;
      const double r2 = apq.x * apq.x + apq.y * apq.y;
      const double thr2 = fmax(4.84e-32 * fabs(app) * fabs(aqq), 1e-30 * fro2);
      if (l < N && m != l && r2 > thr2) {
        const double rinv = rsqrt(r2);
        const double r = r2 * rinv;
        ec = apq.x * rinv;
        es = apq.y * rinv;
        const double tau = (aqq - app) * (0.5 * rinv);
        const double t = copysign(1.0, tau) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
        c = rsqrt(fma(t, t, 1.0));
        s = t * c;
        tr = t * r;
      }
      {  // both lanes of a pair use the p-lane's parameters (exactly one rotation)
        const int src = is_p ? l : (m & 31);
        c = __shfl_sync(0xffffffffu, c, src);
        s = __shfl_sync(0xffffffffu, s, src);
        ec = __shfl_sync(0xffffffffu, ec, src);
        es = __shfl_sync(0xffffffffu, es, src);
        tr = __shfl_sync(0xffffffffu, tr, src);
        if (s != 0.0) rotated = 1;
      }
      // column update with the partner's column (A and V)
      const cplx emi = cmk(ec, -es);  // e^{-i phi}
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double yx = __shfl_sync(0xffffffffu, a[k].x, m & 31);
        const double yy = __shfl_sync(0xffffffffu, a[k].y, m & 31);
        const double vx = __shfl_sync(0xffffffffu, v[k].x, m & 31);
        const double vy = __shfl_sync(0xffffffffu, v[k].y, m & 31);
        if (s != 0.0) {
          if (is_p) {  // col_p' = c col_p - s e^{-i phi} col_q
            const cplx wq = cmul(emi, cmk(yx, yy)), wv = cmul(emi, cmk(vx, vy));
            a[k] = cmk(c * a[k].x - s * wq.x, c * a[k].y - s * wq.y);
            v[k] = cmk(c * v[k].x - s * wv.x, c * v[k].y - s * wv.y);
          } else {     // col_q' = s col_p + c e^{-i phi} col_q
            const cplx wq = cmul(emi, a[k]), wv = cmul(emi, v[k]);
            a[k] = cmk(s * yx + c * wq.x, s * yy + c * wq.y);
            v[k] = cmk(s * vx + c * wv.x, s * vy + c * wv.y);
          }
        }
      }
      // row update: every pair's rows (p, q) in every owned column
#pragma unroll
      for (int k2 = 0; k2 < N / 2; ++k2) {
        int pa, pb;  // the pair k2 of this round (compile-time indices)
        if (k2 == 0) {
          pa = 0;
          pb = 1 + round % (N - 1);
        } else {
          pa = 1 + (round + k2) % (N - 1);
          pb = 1 + (round + N - 1 - k2) % (N - 1);
        }
        if (pa > pb) {
          const int t_ = pa;
          pa = pb;
          pb = t_;
        }
        const double pc = __shfl_sync(0xffffffffu, c, pa);
        const double ps = __shfl_sync(0xffffffffu, s, pa);
        const double pex = __shfl_sync(0xffffffffu, ec, pa);
        const double pey = __shfl_sync(0xffffffffu, es, pa);
        if (ps != 0.0) {
          const cplx epi = cmk(pex, pey);  // e^{i phi}
          const cplx xp = a[pa], xq = a[pb];
          const cplx wq = cmul(epi, xq);
          a[pa] = cmk(pc * xp.x - ps * wq.x, pc * xp.y - ps * wq.y);
          a[pb] = cmk(ps * xp.x + pc * wq.x, ps * xp.y + pc * wq.y);
        }
      }
      // exact 2x2 block of the own pair
      if (s != 0.0) {
        const double nd = is_p ? app - tr : aqq + tr;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          if (k == l) a[k] = cmk(nd, 0.0);
          if (k == m) a[k] = cmk(0.0, 0.0);
        }
      }
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  if (l < n) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if (k < n) j.V[k * j.ld + l] = v[k];
      if (k == l) j.val[l] = a[k].x;
    }
  }
}

__device__ inline void jac_finish(JacSmem& j, int n);

// Block Jacobi + the reference ordering/phase conventions. All threads of the
// CTA must call. (The register-resident warp_jacobi above measured slower on
// B200 -- 82 vs 49 us at n = 8, 517 vs 121 us at n = 16 -- because its
// critical path is the same FP64 rotation chain plus ~60 shuffles per
// round, so the block version stays the default.)
__device__ inline void jac_solve(JacSmem& j, const cplx* M, int ldm, int n, double div) {
  jac_load_sym(j, M, ldm, n, div);
  jac_sweeps(j, n);
  jac_finish(j, n);
}

// Descending order + tie rule + pivot phase. Produces j.order (column of V
// for output position k) and rotates V's columns in place.
__device__ inline void jac_finish(JacSmem& j, int n) {
  const int tid = threadIdx.x;
  // pivot (first argmax |v_ik|) of every column
  for (int k = tid; k < n; k += blockDim.x) {
    int best = 0;
    double bm = -1.0;
    for (int i = 0; i < n; ++i) {
      const cplx v = j.V[i * j.ld + k];
      const double a = hypot(v.x, v.y);
      if (a > bm) {
        bm = a;
        best = i;
      }
    }
    j.piv[k] = best;
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < n; ++k) j.order[k] = k;
    // stable insertion sort, descending by value
    for (int a = 1; a < n; ++a) {
      const int key = j.order[a];
      int b = a - 1;
      while (b >= 0 && j.val[j.order[b]] < j.val[key]) {
        j.order[b + 1] = j.order[b];
        --b;
      }
      j.order[b + 1] = key;
    }
    double mx = 0.0;
    for (int k = 0; k < n; ++k) mx = fmax(mx, fabs(j.val[k]));
    const double tie = mx * 1e-12;
    int s = 0;
    while (s < n) {
      int e = s + 1;
      while (e < n && fabs(j.val[j.order[e]] - j.val[j.order[e - 1]]) <= tie) ++e;
      if (e - s > 1) {  // stable sort of the run by dominant index
        for (int a = s + 1; a < e; ++a) {
          const int key = j.order[a];
          int b = a - 1;
          while (b >= s && j.piv[j.order[b]] > j.piv[key]) {
            j.order[b + 1] = j.order[b];
            --b;
          }
          j.order[b + 1] = key;
        }
      }
      s = e;
    }
  }
  __syncthreads();
  // pivot phase: v_k *= conj(z)/|z|, z = v[piv_k, k] (factors first, then apply)
  for (int k = tid; k < n; k += blockDim.x) {
    const cplx z = j.V[j.piv[k] * j.ld + k];
    const double mag = hypot(z.x, z.y);
    j.phr[k] = mag > 0.0 ? z.x / mag : 1.0;
    j.phi[k] = mag > 0.0 ? -z.y / mag : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e % n;
    j.V[i * j.ld + k] = cmul(j.V[i * j.ld + k], cmk(j.phr[k], j.phi[k]));
  }
  __syncthreads();
}

}  // namespace kstj
