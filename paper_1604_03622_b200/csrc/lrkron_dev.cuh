// Device-side pieces of the LR-Kron iteration shared by lrkron.cu (global
// estimate) and lmode.cu (batched L-mode windows): the iteration state, the
// spatial update (src/lrkron.py:207-221) and the M-path iteration loop.
// Internal linkage (anonymous namespace): each unit gets its own copy.
#pragma once
#include "jacobi.cuh"

namespace {

using namespace kstj;

constexpr int NT = 256;
constexpr int kMaxP = 16;

// State block shared by the iteration kernels (device memory).
struct IterState {
  double fro, fro2, na2, nb2, eta_prev, eta;
  int status;      // 0 ok, KST_ERR_DATA / KST_ERR_DEGENERATE
  int converged;
  int iteration;
  int pad;
  cplx A[kMaxP * kMaxP];     // current spatial iterate (row-major P x P)
  cplx Aconj[kMaxP * kMaxP]; // conj(A) (b-step operand)
};


template <int P>
struct MDims {
  static constexpr int U = P * P;
  static constexpr int E = U * (U + 1) / 2;          // upper-triangle entries of M
  static constexpr int STRIDE = 4 + 2 * U + 2 * E;   // partial record length
};

// Shared by the streaming and the M-path iterations. On entry V (smem, P x P)
// = <S4, conj(b)>_{rc} and nb2 = |b|^2 > 0. Performs A = EIG_ra(V / nb2)
// (src/lrkron.py:207), the expanded-norm residual (src/lrkron.py:210-213) and
// the stall test (src/lrkron.py:218-221); updates *st. Every thread of the CTA
// must call it. Returns 0 or KST_ERR_DATA (V not Hermitian), uniformly.
__device__ __noinline__ int spatial_update(const cplx* V, double nb2, int P, int ra, double tol, IterState* st,
                              char* sm, cplx* Anew, double* lam, int* bad_s, double* eta_out,
                              int* conv_out) {
  const int tid = threadIdx.x;
  // eig_truncate(V / nb2, ra): Hermitian check first (src/linalg.py:68-79);
  // the P^2 quotients by all threads, the sums in order by one
  __shared__ cplx vq[kMaxP * kMaxP];
  for (int e = tid; e < P * P; e += NT) vq[e] = cmk(V[e].x / nb2, V[e].y / nb2);
  __syncthreads();
  if (tid == 0) {
    double f = 0.0, a = 0.0;
    for (int r = 0; r < P; ++r)
      for (int c = 0; c < P; ++c) {
        const cplx x = vq[r * P + c];
        const cplx y = vq[c * P + r];
        f += cabs2(x);
        a += cabs2(cmk(x.x - y.x, x.y + y.y));
        if (!isfinite(x.x) || !isfinite(x.y)) a = INFINITY;
      }
    *bad_s = (sqrt(f) > 0 && !(sqrt(a) <= 1e-8 * sqrt(f))) ? 1 : 0;
  }
  __syncthreads();
  if (*bad_s) {
    if (tid == 0) st->status = KST_ERR_DATA;
    return KST_ERR_DATA;
  }
  if (ra == P) {
    for (int e = tid; e < P * P; e += NT) {
      const int r = e / P, c = e % P;
      const cplx x = V[r * P + c], y = V[c * P + r];
      Anew[e] = cmk(((x.x / nb2) + (y.x / nb2)) / 2.0, ((x.y / nb2) - (y.y / nb2)) / 2.0);
    }
  } else {
    JacSmem j = jac_carve(sm, P);
    jac_solve(j, V, P, P, nb2);
    if (tid == 0) {
      double top = 0.0;
      for (int k = 0; k < P; ++k) top = fmax(top, fabs(j.val[k]));
      for (int k = 0; k < ra; ++k) {
        double v = j.val[j.order[k]];
        if (v < 0 && fabs(v) <= 1e-10 * top) v = 0.0;
        lam[k] = v;
      }
    }
    __syncthreads();
    for (int e = tid; e < P * P; e += NT) {
      const int a = e / P, c = e % P;
      cplx ab = cmk(0, 0), ba = cmk(0, 0);
      for (int k = 0; k < ra; ++k) {
        const cplx ua = j.V[a * j.ld + j.order[k]], uc = j.V[c * j.ld + j.order[k]];
        cfmac(ab, cscale(ua, lam[k]), uc);
        cfmac(ba, cscale(uc, lam[k]), ua);
      }
      Anew[e] = cmk((ab.x + ba.x) / 2.0, (ab.y - ba.y) / 2.0);
    }
  }
  __syncthreads();
  if (tid == 0) {
    double cross = 0.0, na2 = 0.0;
    for (int e = 0; e < P * P; ++e) {
      cross += Anew[e].x * V[e].x + Anew[e].y * V[e].y;  // Re vdot(A, V)
      na2 += cabs2(Anew[e]);
    }
    const double fro = st->fro;
    const double eta2 = st->fro2 + na2 * nb2 - 2.0 * cross;
    const double eta = sqrt(fmax(eta2, 0.0)) / fro;
    const int conv = fabs(st->eta_prev - eta) <= tol;
    st->eta_prev = eta;
    st->eta = eta;
    st->nb2 = nb2;
    st->na2 = na2;
    st->converged = conv;
    st->iteration += 1;
    for (int e = 0; e < P * P; ++e) {
      st->A[e] = Anew[e];
      st->Aconj[e] = cmk(Anew[e].x, -Anew[e].y);
    }
    *eta_out = eta;
    *conv_out = conv;
  }
  __syncthreads();
  return 0;
}

// M-path iterations (P <= 4) on a reduced record in shared memory,
// red = [fro2, bad, dmin, dmax, A0 block sums re/im (2U), M upper re/im (2E)]
// with M = R R^H (R the Pitsianis-Van Loan rearrangement of S): every
// iteration of src/lrkron.py:184-221 runs on P^2-sized quantities. Shared by
// m_iterate_kernel (global estimate) and the batched L-mode window kernel.
// Outputs: spatial (final A), residuals[max_iter], info[0..2] = {status,
// iterations, converged}, host_diag[0..4] = {bad, dmin, dmax, fro, na2_0};
// st->Aconj / st->na2 are left holding the A that produced the final b.
// All threads of the (NT-thread) CTA must call.
template <int P>
__device__ void m_iterations(const double* red, int q, int ra, double tol, int max_iter,
                             IterState* st, char* sm, cplx* __restrict__ spatial_out,
                             double* __restrict__ residuals, double* __restrict__ info,
                             double* __restrict__ host_diag) {
  using Dm = MDims<P>;
  constexpr int U = Dm::U, E = Dm::E;
  __shared__ cplx M[U * U];
  __shared__ cplx V[kMaxP * kMaxP];
  __shared__ cplx Anew[kMaxP * kMaxP];
  __shared__ cplx Ma[U];
  __shared__ cplx Aprev[kMaxP * kMaxP];
  __shared__ double lam[kMaxP];
  __shared__ double eta_s, scal[4];
  __shared__ int bad_s, conv_s, stop_s;
  const int tid = threadIdx.x;
  __syncthreads();
  for (int k = tid; k < E; k += NT) {
    // unpack the upper triangle into the full Hermitian M
    int u = 0, rem = k;
    while (rem >= U - u) {
      rem -= U - u;
      ++u;
    }
    const int v = u + rem;
    const cplx m = cmk(red[4 + 2 * U + 2 * k], red[4 + 2 * U + 2 * k + 1]);
    M[u * U + v] = m;
    M[v * U + u] = cconj(m);
  }
  {  // A0 = block sums / q^2: the quotients by all threads, |A0|^2 in order by one
    const double qq = (double)q * (double)q;
    for (int e = tid; e < U; e += NT) {
      const cplx a = cmk(red[4 + 2 * e] / qq, red[5 + 2 * e] / qq);
      st->A[e] = a;
      st->Aconj[e] = cconj(a);
    }
  }
  __syncthreads();
  if (tid == 0) {
    double na2 = 0.0;
    for (int e = 0; e < U; ++e) na2 += cabs2(st->A[e]);
    st->fro2 = red[0];
    st->fro = sqrt(red[0]);
    st->na2 = na2;
    st->eta_prev = INFINITY;
    st->status = 0;
    st->converged = 0;
    st->iteration = 0;
    host_diag[0] = red[1];
    host_diag[1] = red[2];
    host_diag[2] = red[3];
    host_diag[3] = st->fro;
    host_diag[4] = na2;
    stop_s = (red[1] > 0.0 || red[0] == 0.0) ? 1 : 0;  // host handles bad input / zero S
  }
  __syncthreads();
  int status = 0, iters = 0, conv = 0;
  if (!stop_s) {
    for (int it = 0; it < max_iter; ++it) {
      if (tid == 0) {
        scal[0] = st->na2;
        stop_s = 0;
      }
      __syncthreads();
      const double na2 = scal[0];
      if (na2 == 0.0) {
        status = 4;  // spatial iterate collapsed (reference raises at iteration start)
        break;
      }
      // Ma = M a ; nb2 = Re(a^H M a) / na2^2 ; V = Ma / na2
      for (int u = tid; u < U; u += NT) {
        cplx acc = cmk(0, 0);
        for (int v = 0; v < U; ++v) cfma(acc, M[u * U + v], st->A[v]);
        Ma[u] = acc;
      }
      __syncthreads();
      if (tid == 0) {
        double q2 = 0.0;
        for (int u = 0; u < U; ++u) q2 += st->A[u].x * Ma[u].x + st->A[u].y * Ma[u].y;
        scal[1] = q2 / (na2 * na2);
        // the A that produces this iteration's b (kept for the final b-step)
        scal[2] = na2;
      }
      for (int u = tid; u < U; u += NT) V[u] = cmk(Ma[u].x / na2, Ma[u].y / na2);
      __syncthreads();
      const double nb2 = scal[1];
      ++iters;
      if (nb2 == 0.0) {
        status = KST_ERR_DEGENERATE;
        break;
      }
      // keep the b-producing A for the final b-step before spatial_update overwrites it
      for (int e = tid; e < U; e += NT) Aprev[e] = st->A[e];
      __syncthreads();
      const int rc = spatial_update(V, nb2, P, ra, tol, st, sm, Anew, lam, &bad_s, &eta_s, &conv_s);
      if (rc) {
        status = rc;
        break;
      }
      if (tid == 0) residuals[it] = eta_s;
      const int c_now = conv_s;
      __syncthreads();
      if (c_now) {
        conv = 1;
        // leave Aconj / na2 describing the b-producing A
        if (tid == 0) {
          for (int e = 0; e < U; ++e) {
            spatial_out[e] = st->A[e];
            st->Aconj[e] = cconj(Aprev[e]);
          }
          st->na2 = scal[2];
        }
        break;
      }
      if (it == max_iter - 1 && tid == 0) {
        for (int e = 0; e < U; ++e) {
          spatial_out[e] = st->A[e];
          st->Aconj[e] = cconj(Aprev[e]);
        }
        st->na2 = scal[2];
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    info[0] = status;
    info[1] = iters;
    info[2] = conv;
  }
}


}  // namespace
