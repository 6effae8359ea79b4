"""CPU oracle for the Kron-STAP hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product. Only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference`
legs of `bench.py` may import it. The package `paper_1604_03622_b200`
never imports it and has no CPU fallback.

It restates, in plain numpy, the algorithm of the reference package
`kronstap` (pure Python; /root/reference/pkg/src/kronstap, abbreviated
`src/`) for the path

    cube (n, P, q) c128 -> sample covariance -> LR-Kron estimate
         -> projection filter -> detection map (n, D) f64

plus the multipass stacking / pass images / change map. Every function
cites the reference lines it follows. Arithmetic is float64/complex128
like the reference.

Parity pin: tests/golden/*.npz hold outputs of the unmodified reference
run in the build container (script: oracle/gen_golden.py); the CPU test
`tests/test_oracle_golden.py` checks this restatement against them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

HERM_RTOL = 1e-8        # src/linalg.py:19, src/lrkron.py:21
CLAMP_RTOL = 1e-10      # src/linalg.py:22
TIE_RTOL = 1e-12        # src/linalg.py:99
RANK_TOL = 1e-9         # src/filters.py:58 (subspace_basis default tol)


class OracleError(Exception):
    """Raised where the reference raises; `kind` names the reference class."""

    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# dense Hermitian helpers -- src/linalg.py:82-144


def _herm_check(m):
    m = np.asarray(m, dtype=np.complex128)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise OracleError("DimensionError", "square matrix expected")
    if not np.all(np.isfinite(m)):
        raise OracleError("DataError", "non-finite entries")
    nrm = np.linalg.norm(m)
    if nrm > 0 and np.linalg.norm(m - m.conj().T) > HERM_RTOL * nrm:
        raise OracleError("DataError", "not Hermitian")
    return m


def heig(m):
    """Descending eigenpairs with the reference's tie and phase rules.

    src/linalg.py:82-121: symmetrise, eigh, reverse to descending; runs
    of values within 1e-12*max|lambda| are re-ordered by the index of
    each vector's largest |component| (stable); each vector is rotated
    so that component is real positive.
    """
    m = _herm_check(m)
    lam, vec = np.linalg.eigh(0.5 * (m + m.conj().T))
    lam = np.ascontiguousarray(lam[::-1])
    vec = np.ascontiguousarray(vec[:, ::-1])
    n = lam.size
    if n > 1:
        thr = TIE_RTOL * np.max(np.abs(lam))
        s = 0
        while s < n:
            e = s + 1
            while e < n and abs(lam[e] - lam[e - 1]) <= thr:
                e += 1
            if e - s > 1:
                piv = [int(np.argmax(np.abs(vec[:, k]))) for k in range(s, e)]
                perm = s + np.argsort(piv, kind="stable")
                lam[s:e] = lam[perm]
                vec[:, s:e] = vec[:, perm]
            s = e
    for k in range(n):
        z = vec[int(np.argmax(np.abs(vec[:, k]))), k]
        if abs(z) > 0:
            vec[:, k] *= np.conj(z) / abs(z)
    return lam, vec


def truncate(m, rank):
    """Top-`rank` Hermitian reconstruction -- src/linalg.py:124-144."""
    m = _herm_check(m)
    n = m.shape[0]
    if not 1 <= rank <= n:
        raise OracleError("DimensionError", "rank out of range")
    if rank == n:
        return 0.5 * (m + m.conj().T)
    lam, vec = heig(m)
    top = np.max(np.abs(lam)) if lam.size else 0.0
    lam = np.where((lam < 0) & (np.abs(lam) <= CLAMP_RTOL * top), 0.0, lam)
    u = vec[:, :rank]
    out = (u * lam[:rank]) @ u.conj().T
    return 0.5 * (out + out.conj().T)


def basis(m, rank, tol=RANK_TOL):
    """Leading eigenvectors kept by the reference -- src/filters.py:58-73.

    Returns None for an empty subspace.
    """
    lam, vec = heig(m)
    if lam.size == 0 or lam[0] <= 0.0:
        return None
    keep = min(int(np.sum(lam > tol * lam[0])), rank)
    return None if keep == 0 else vec[:, :keep]


# --------------------------------------------------------------------------
# estimation -- src/lrkron.py


def scm(snapshots, p, q):
    """S = (1/n) X^T conj(X), symmetrised -- src/lrkron.py:53-78."""
    x = np.asarray(snapshots, dtype=np.complex128)
    if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] != p * q:
        raise OracleError("DimensionError", "bad snapshot matrix")
    s = (x.T @ np.conj(x)) / x.shape[0]
    return 0.5 * (s + s.conj().T)


@dataclass
class Fit:
    """Mirror of KronCovEstimate (src/lrkron.py:36-50)."""

    spatial: np.ndarray
    temporal: np.ndarray
    rank_spatial: int
    rank_temporal: int
    iterations: int
    residuals: list = field(default_factory=list)
    converged: bool = True
    last_b: np.ndarray = None          # b of the final iteration (pre-truncation)
    iterates: list = field(default_factory=list)


def _validate(s, p, q):
    """src/lrkron.py:81-115 (asymmetry via a dense difference here)."""
    s = np.asarray(s, dtype=np.complex128)
    if s.shape != (p * q, p * q):
        raise OracleError("DimensionError", "covariance shape")
    if not np.all(np.isfinite(s)):
        raise OracleError("DataError", "non-finite covariance")
    fro = math.sqrt(np.vdot(s, s).real)
    if fro > 0 and np.linalg.norm(s - s.conj().T) > HERM_RTOL * fro:
        raise OracleError("DataError", "covariance not Hermitian")
    d = s.diagonal().real
    if d.size and d.min() < -HERM_RTOL * max(d.max(), 0.0):
        raise OracleError("DataError", "negative diagonal")
    return s, fro


def lrkron(s, p, q, ra, rb, tol=1e-4, max_iter=100, keep_iterates=False):
    """Alternating LR-Kron fit -- src/lrkron.py:118-230.

    S4[i, r, j, c] = S[i*q + r, j*q + c]. Start A0 = block sums / q^2
    (:173-175). Per iteration: b = <S4, conj A>_{ij} / |A|^2 (:191-195),
    V = <S4, conj b>_{rc} (:202-205), A = EIG_ra(V / |b|^2) (:207),
    eta from the expanded norm (:210-213), stop on |eta_prev - eta| <= tol
    (:218-221). Finally temporal = EIG_rb(b) (:223).
    """
    s, fro = _validate(s, p, q)
    if not 1 <= ra <= p or not 1 <= rb <= q or max_iter < 1:
        raise OracleError("DimensionError", "rank / max_iter out of range")
    if fro == 0.0:
        return Fit(np.zeros((p, p), complex), np.zeros((q, q), complex),
                   ra, rb, 0, [0.0], True)
    s4 = s.reshape(p, q, p, q)
    a = np.einsum("irjc->ij", s4) / float(q * q)
    res, its = [], []
    eta_prev = math.inf
    converged = False
    n_it = 0
    b = None
    for _ in range(max_iter):
        n_it += 1
        na2 = np.vdot(a, a).real
        if na2 == 0.0:
            raise OracleError("DegenerateInputError", "spatial iterate zero")
        b = np.einsum("irjc,ij->rc", s4, np.conj(a)) / na2
        nb2 = np.vdot(b, b).real
        if nb2 == 0.0:
            raise OracleError("DegenerateInputError", "temporal iterate zero")
        v = np.einsum("irjc,rc->ij", s4, np.conj(b))
        a = truncate(v / nb2, ra)
        cross = np.vdot(a, v).real
        eta2 = fro * fro + np.vdot(a, a).real * nb2 - 2.0 * cross
        eta = math.sqrt(max(eta2, 0.0)) / fro
        res.append(eta)
        if keep_iterates:
            its.append((a.copy(), b.copy()))
        if abs(eta_prev - eta) <= tol:
            converged = True
            break
        eta_prev = eta
    fit = Fit(a, truncate(b, rb), ra, rb, n_it, res, converged, b, its)
    return fit


# --------------------------------------------------------------------------
# filtering and detection -- src/filters.py


def filter_bases(fit, rank_tol=RANK_TOL):
    """(U_A, U_B) as build_filter pulls them -- src/filters.py:164-175."""
    return (basis(fit.spatial, fit.rank_spatial, rank_tol),
            basis(fit.temporal, fit.rank_temporal, rank_tol))


def apply_filter(kind, ua, ub, x, spatial_only=False):
    """One bin through a projection filter -- src/filters.py:88-116."""
    x = np.asarray(x, dtype=np.complex128)
    if not np.all(np.isfinite(x)):
        raise OracleError("DataError", "non-finite bin")
    if kind == "kron":
        y = x
        if ub is not None and not spatial_only:
            y = y - (y @ ub.conj()) @ ub.T
        if ua is not None:
            y = y - ua @ (ua.conj().T @ y)
        return np.array(y)
    if kind != "classical":
        raise OracleError("DimensionError", "kind")
    if ua is None:
        return np.array(x)
    if spatial_only:
        return x - ua @ (ua.conj().T @ x)
    if ub is None:
        return np.array(x)
    return x - ua @ (ua.conj().T @ x @ ub.conj()) @ ub.T


def doppler_grid(count):
    """src/filters.py:201-205."""
    return np.arange(count, dtype=np.float64) / count


def spatial_grid(p, count=16):
    """src/filters.py:208-217."""
    ph = np.outer(np.arange(count, dtype=np.float64) / count, np.arange(p))
    return np.exp(2j * np.pi * ph) / np.sqrt(p)


def stacked_grid(p, k, count=16):
    """Block-diagonal per-pass embedding -- src/filters.py:220-231."""
    g = np.zeros((k * count, k * p), dtype=np.complex128)
    base = spatial_grid(p, count)
    for j in range(k):
        g[j * count:(j + 1) * count, j * p:(j + 1) * p] = base
    return g


def detect(kind, ua, ub, cube, dopplers, grid, spatial_only=False):
    """max_g |conj(H) F(X_m) conj(T)| per bin -- src/filters.py:243-275."""
    cube = np.asarray(cube, dtype=np.complex128)
    dop = np.asarray(dopplers, dtype=np.float64).ravel()
    h = np.asarray(grid, dtype=np.complex128)
    n, p, q = cube.shape
    t = np.exp(2j * np.pi * np.outer(np.arange(q), dop)) / np.sqrt(q)
    tc, hc = t.conj(), h.conj()
    out = np.empty((n, dop.size))
    for m in range(n):
        f = apply_filter(kind, ua, ub, cube[m], spatial_only)
        out[m] = np.abs(hc @ (f @ tc)).max(axis=0)
    return out


# --------------------------------------------------------------------------
# "optimal" kind, steering, SINR -- src/filters.py:27-55, 98-100, 144-163, 178-198


def optimal_whiten(sigma, cube):
    """sigma^-1 x per bin: cho_factor(sigma, lower=True) (src/filters.py:156-162)
    then cho_solve per bin (src/filters.py:98-100); all bins as one solve."""
    from scipy.linalg import cho_factor, cho_solve
    c = cho_factor(np.asarray(sigma, dtype=np.complex128), lower=True)
    cube = np.asarray(cube, dtype=np.complex128)
    n, p, q = cube.shape
    return np.ascontiguousarray(cho_solve(c, cube.reshape(n, p * q).T).T).reshape(n, p, q)


def steering(doppler, p, q, kappa=0.5):
    """Unit-norm kron(spatial, temporal) steering snapshot (src/filters.py:38-55)."""
    sp = np.exp(2j * np.pi * kappa * doppler * np.arange(p))
    tm = np.exp(2j * np.pi * doppler * np.arange(q)) / np.sqrt(q)
    full = np.kron(sp, tm)
    return full / np.linalg.norm(full)


def sinr(w, d, amplitude, sigma):
    """|a|^2 |w^H d|^2 / (w^H sigma w) (src/filters.py:185-198)."""
    w, d = np.asarray(w).ravel(), np.asarray(d).ravel()
    denom = np.vdot(w, np.asarray(sigma) @ w).real
    return float((abs(amplitude) ** 2) * abs(np.vdot(w, d)) ** 2 / denom)


# --------------------------------------------------------------------------
# multipass -- src/multipass.py


def stack(data):
    """(K, n, p, q) -> (n, K*p, q), pass-major channels -- src/multipass.py:40-52."""
    k, n, p, q = data.shape
    return np.ascontiguousarray(np.transpose(data, (1, 0, 2, 3))).reshape(n, k * p, q)


def pass_maps(kind, ua, ub, stacked, n_passes, p, dopplers, count=16):
    """One map per pass through the stacked grid -- src/multipass.py:83-102."""
    g = stacked_grid(p, n_passes, count)
    return [detect(kind, ua, ub, stacked, dopplers, g[k * count:(k + 1) * count])
            for k in range(n_passes)]


def change(a, b, signed=False):
    """src/multipass.py:105-123."""
    d = np.asarray(a) - np.asarray(b)
    return d if signed else np.abs(d)


def pipeline(cube, ra, rb, n_doppler, n_spatial=16, tol=1e-4, max_iter=100,
             kind="kron"):
    """README library sequence (pkg/README.md:144-161) on one cube."""
    n, p, q = cube.shape
    s = scm(cube.reshape(n, p * q), p, q)
    fit = lrkron(s, p, q, ra, rb, tol, max_iter)
    ua, ub = filter_bases(fit)
    vals = detect(kind, ua, ub, cube, doppler_grid(n_doppler),
                  spatial_grid(p, n_spatial))
    return fit, ua, ub, vals


def windowed(cube, n_w, ra, rb, n_doppler, n_spatial=16, tol=1e-4, max_iter=100,
             kind="kron", bins=None):
    """L-mode (SURVEY.md §8 "L-mode definition"; no reference equivalent): for
    each test bin m, estimate on training bins [s, s + n_w) with
    s = clamp(m - n_w // 2, 0, n_bins - n_w) and detect bin m with that
    estimate. `bins` restricts the loop to a sample of test bins (rows of the
    returned map outside it stay NaN)."""
    n, p, q = cube.shape
    dop, grid = doppler_grid(n_doppler), spatial_grid(p, n_spatial)
    vals = np.full((n, n_doppler), np.nan)
    fits = {}
    for m in (range(n) if bins is None else bins):
        s0 = min(max(m - n_w // 2, 0), n - n_w)
        if s0 not in fits:
            w = cube[s0:s0 + n_w]
            fit = lrkron(scm(w.reshape(n_w, p * q), p, q), p, q, ra, rb, tol, max_iter)
            fits[s0] = (fit, filter_bases(fit))
        ua, ub = fits[s0][1]
        vals[m] = detect(kind, ua, ub, cube[m:m + 1], dop, grid)[0]
    return vals, {s0: f[0] for s0, f in fits.items()}
