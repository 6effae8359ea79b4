"""Clutter-cancellation filters and detection maps on the GPU.

Mirrors `kronstap.filters` (src/filters.py) for the projection filters:
`subspace_basis`, `StapFilter`, `projection_filter`, `build_filter`,
`detection_image`, `DetectionMap` and the grids. Kernels: kst_subspace_basis
(K3/K4), kst_detect (K5), kst_filter (whole-cube apply_matrix).

The "optimal" (covariance-whitening) kind factors
sigma once on the device (kst_chol) and whitens every bin with one solve
(kst_chol_solve); steering vectors are host constructions like the grids,
and filter_output / sinr evaluate on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np

from . import _native as nat
from ._dual import Dual
from .errors import DataError, DimensionError
from .linalg import subspace_basis_device

FILTER_KINDS = ("optimal", "classical", "kron")


def _basis_dual(b):
    if b is None or isinstance(b, Dual):
        return b
    return Dual(b)


def subspace_basis(matrix, rank, tol=1e-9):
    """Orthonormal basis of the top eigen-subspace, or None (src/filters.py:58-73)."""
    out = subspace_basis_device(matrix, rank, tol)
    if out is None:
        return None
    return out if nat.is_device(matrix) else nat.to_host(out)


class StapFilter:
    """Factored clutter filter for p-channel, q-pulse snapshots (src/filters.py:76-120).

    Bases may be numpy arrays or CUDA tensors; they are uploaded once."""

    def __init__(self, kind, p, q, spatial_basis=None, temporal_basis=None, spatial_only=False):
        self.kind = kind
        self.p = p
        self.q = q
        self._ua = _basis_dual(spatial_basis)
        self._ub = _basis_dual(temporal_basis)
        self.spatial_only = spatial_only
        self._chol = None  # kind "optimal": device (pq, pq) column-major lower factor

    @property
    def spatial_basis(self):
        return None if self._ua is None else self._ua.value()

    @spatial_basis.setter
    def spatial_basis(self, v):
        self._ua = _basis_dual(v)

    @property
    def temporal_basis(self):
        return None if self._ub is None else self._ub.value()

    @temporal_basis.setter
    def temporal_basis(self, v):
        self._ub = _basis_dual(v)

    def _dev_bases(self):
        ua = None if self._ua is None else self._ua.dev()
        ub = None if self._ub is None else self._ub.dev()
        return ua, ub

    def _kind_code(self):
        if self.kind not in nat.KIND:
            raise DimensionError(f"unknown filter kind {self.kind!r}")
        return nat.KIND[self.kind]

    def apply_cube(self, cube):
        """Filter every bin of an (n, p, q) cube (kst_filter)."""
        import torch
        shp = tuple(cube.shape) if hasattr(cube, "shape") else np.shape(cube)
        if len(shp) != 3 or shp[1:] != (self.p, self.q):
            raise DimensionError(f"cube shape {shp} does not match filter ({self.p}, {self.q})")
        x = nat.to_device(cube)
        if self.kind == "optimal":
            out = self._whiten(x)
            return out if nat.is_device(cube) else nat.to_host(out)
        kind = self._kind_code()
        ua, ub = self._dev_bases()
        out = torch.empty_like(x)
        c = nat.ctx(x.device)
        nat.check(nat.lib().kst_filter(
            c, nat.ptr(x), shp[0], self.p, self.q, nat.ptr(ua), 0 if ua is None else ua.shape[1],
            nat.ptr(ub), 0 if ub is None else ub.shape[1], kind, int(bool(self.spatial_only)),
            nat.ptr(out), nat.stream_of(x.device)), c)
        return out if nat.is_device(cube) else nat.to_host(out)

    def _whiten(self, x):
        """sigma^-1 applied to every bin of the device cube x (cho_solve,
        src/filters.py:98-100): one kst_chol_solve over all bins."""
        import torch
        if self._chol is None:
            raise DimensionError("optimal filter has no factor (use build_filter)")
        L = self._chol if self._chol.device == x.device else self._chol.to(x.device)
        out = torch.empty_like(x)
        c = nat.ctx(x.device)
        nat.check(nat.lib().kst_chol_solve(c, nat.ptr(L), self.p * self.q, nat.ptr(x), x.shape[0],
                                           nat.ptr(out), nat.stream_of(x.device)), c)
        return out

    def apply_matrix(self, x):
        """Filter one bin given as its (p, q) matrix (src/filters.py:88-116)."""
        shp = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
        if len(shp) != 2:
            raise DimensionError(f"bin matrix must be 2-D, got shape {shp}")
        if shp != (self.p, self.q):
            raise DimensionError(f"bin shape {shp} does not match filter ({self.p}, {self.q})")
        out = self.apply_cube(x.reshape(1, self.p, self.q) if nat.is_device(x)
                              else np.asarray(x, dtype=np.complex128).reshape(1, self.p, self.q))
        return out[0]

    def apply(self, x):
        """Filter one channel-major snapshot vector (src/filters.py:118-120)."""
        v = x.reshape(-1) if nat.is_device(x) else np.asarray(x).ravel()
        if v.shape[0] != self.p * self.q:
            raise DimensionError(f"snapshot length {v.shape[0]} does not match {self.p}x{self.q}")
        return self.apply_matrix(v.reshape(self.p, self.q)).reshape(-1)


def projection_filter(kind, spatial_basis, temporal_basis, p, q, spatial_only=False):
    """src/filters.py:123-134."""
    if kind not in ("classical", "kron"):
        raise DimensionError(f"unknown projection filter kind {kind!r}")
    for name, basis, dim in (("spatial", spatial_basis, p), ("temporal", temporal_basis, q)):
        if basis is not None and basis.shape[0] != dim:
            raise DimensionError(f"{name} basis has {basis.shape[0]} rows, expected {dim}")
    return StapFilter(kind, p, q, spatial_basis, temporal_basis, spatial_only)


def build_filter(kind, estimate=None, sigma=None, p=None, q=None, drop_temporal=False, rank_tol=1e-9):
    """src/filters.py:137-175. The temporal basis reuses the eigenpairs the
    estimator already computed for `temporal` (one q x q eigensolve, not two)."""
    if kind not in FILTER_KINDS:
        raise DimensionError(f"unknown filter kind {kind!r}")
    if kind == "optimal":
        return _optimal_filter(sigma, p, q)
    if estimate is None:
        raise DimensionError(f"{kind} filter needs a covariance estimate")
    device_mode = estimate._sp.device_mode if hasattr(estimate, "_sp") else nat.is_device(estimate.spatial)
    sp = estimate._sp.dev() if hasattr(estimate, "_sp") else nat.to_device(estimate.spatial)
    ua = subspace_basis_device(sp, estimate.rank_spatial, rank_tol)
    tb = getattr(estimate, "_tb", None)
    tp = None
    if tb is not None:
        vecs, vals = tb
        keep = 0
        if vals[0] > 0.0:
            while keep < min(estimate.rank_temporal, len(vals)) and vals[keep] > rank_tol * vals[0]:
                keep += 1
        ub = None if keep == 0 else vecs[:, :keep].contiguous()
    else:
        tp = estimate._tp.dev() if hasattr(estimate, "_tp") else nat.to_device(estimate.temporal)
        ub = subspace_basis_device(tp, estimate.rank_temporal, rank_tol)
    p_, q_ = sp.shape[0], (tb[0].shape[0] if tb is not None else tp.shape[0])
    f = StapFilter(kind, p_, q_,
                   None if ua is None else Dual.from_device(ua, device_mode),
                   None if ub is None else Dual.from_device(ub, device_mode),
                   spatial_only=drop_temporal)
    return f


def _optimal_filter(sigma, p, q):
    """build_filter(kind="optimal") (src/filters.py:144-163): the lower Cholesky
    factor of sigma on the device; DataError when sigma is non-finite or not
    positive definite."""
    import torch
    if sigma is None or p is None or q is None:
        raise DimensionError("optimal filter needs sigma and its bin shape")
    shp = tuple(sigma.shape) if hasattr(sigma, "shape") else np.shape(sigma)
    if len(shp) != 2:
        raise DimensionError(f"covariance must be 2-D, got shape {shp}")
    if shp != (p * q, p * q):
        # as_matrix's finite check comes first in the reference (src/linalg.py:25-33)
        host = sigma.cpu().numpy() if nat.is_device(sigma) else np.asarray(sigma)
        if not np.all(np.isfinite(host)):
            raise DataError("covariance contains non-finite entries")
        raise DimensionError(f"covariance shape {shp} does not match p*q = {p * q}")
    s = nat.to_device(sigma)
    L = torch.empty_like(s)
    c = nat.ctx(s.device)
    nat.check(nat.lib().kst_chol(c, nat.ptr(s), p * q, nat.ptr(L), nat.stream_of(s.device)), c)
    filt = StapFilter("optimal", p, q)
    filt._chol = L
    return filt


@dataclass
class SteeringVector:
    """Spatial and temporal steering for one normalized Doppler (src/filters.py:27-41)."""

    spatial: np.ndarray
    temporal: np.ndarray
    doppler: float
    kappa: float

    @property
    def vector(self):
        """Unit-norm channel-major steering snapshot."""
        full = np.kron(self.spatial, self.temporal)
        return full / np.linalg.norm(full)


def make_steering(doppler, p, q, kappa=0.5):
    """src/filters.py:44-55 (a host construction of p + q phase ramps, like the grids)."""
    if p < 1 or q < 1:
        raise DimensionError(f"steering needs positive dims, got p={p}, q={q}")
    spatial = np.exp(2j * np.pi * kappa * doppler * np.arange(p))
    temporal = np.exp(2j * np.pi * doppler * np.arange(q)) / np.sqrt(q)
    return SteeringVector(spatial, temporal, float(doppler), float(kappa))


def _dev_vector(v, dev):
    import torch
    if nat.is_device(v):
        return v.reshape(-1).to(dev, torch.complex128)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.complex128).ravel())).to(dev)


def filter_output(filt, steering, x):
    """(F d)^H x for one snapshot (src/filters.py:178-182): F d through the
    filter's device path, the inner product on the device."""
    import torch
    d = steering.vector if isinstance(steering, SteeringVector) else steering
    dev = torch.device("cuda", torch.cuda.current_device())
    w = _dev_vector(filt.apply(_dev_vector(d, dev)), dev)
    return complex(torch.vdot(w, _dev_vector(x, dev)).item())


def sinr(weights, steering, amplitude, sigma):
    """Output SINR of a weight vector (src/filters.py:185-198), on the device:
    |amplitude|^2 |w^H d|^2 / (w^H sigma w); scale invariant in w."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    w = _dev_vector(weights, dev)
    d = steering.vector if isinstance(steering, SteeringVector) else steering
    d = _dev_vector(d, dev)
    shp = tuple(sigma.shape) if hasattr(sigma, "shape") else np.shape(sigma)
    if len(shp) != 2:
        raise DimensionError(f"covariance must be 2-D, got shape {shp}")
    s = nat.to_device(sigma) if nat.is_device(sigma) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(sigma, dtype=np.complex128))).to(dev)
    if not bool(torch.isfinite(torch.view_as_real(s)).all()):
        raise DataError("covariance contains non-finite entries")
    denom = float(torch.vdot(w, s.to(dev) @ w).real.item())
    if denom <= 0.0:
        raise DataError("weights have no response power under this covariance")
    num = (abs(amplitude) ** 2) * abs(complex(torch.vdot(w, d).item())) ** 2
    return float(num / denom)


def make_doppler_grid(count):
    """src/filters.py:201-205."""
    if count < 1:
        raise DimensionError(f"doppler grid needs at least one bin, got {count}")
    return np.arange(count, dtype=np.float64) / count


def make_spatial_grid(p, count=16):
    """src/filters.py:208-217."""
    if count < 1:
        raise DimensionError(f"spatial grid needs at least one point, got {count}")
    slopes = np.arange(count, dtype=np.float64) / count
    return np.exp(2j * np.pi * np.outer(slopes, np.arange(p))) / np.sqrt(p)


def make_stacked_spatial_grid(p, n_passes, count=16):
    """src/filters.py:220-231."""
    base = make_spatial_grid(p, count)
    out = np.zeros((n_passes * count, n_passes * p), dtype=np.complex128)
    for k in range(n_passes):
        out[k * count:(k + 1) * count, k * p:(k + 1) * p] = base
    return out


@dataclass
class DetectionMap:
    """Per-bin, per-Doppler detection magnitudes with their grids (src/filters.py:234-240)."""

    values: object
    dopplers: np.ndarray
    spatial_grid: np.ndarray


def _host_grid_args(filt, dopplers, spatial_grid):
    dop = np.ascontiguousarray(np.asarray(dopplers.cpu() if nat.is_device(dopplers) else dopplers,
                                          dtype=np.float64).ravel())
    grid = np.ascontiguousarray(np.asarray(spatial_grid.cpu() if nat.is_device(spatial_grid)
                                           else spatial_grid, dtype=np.complex128))
    if grid.ndim != 2 or grid.shape[1] != filt.p:
        raise DimensionError(f"spatial grid shape {grid.shape} does not match p = {filt.p}")
    return dop, grid


def run_detect(filt, cube, dop, grid, groups=1, precision=None):
    """kst_detect -> device tensor (groups, n, D) float64. `precision`
    ("f32"/"f64") overrides the context's K5 precision for this call; the
    optimal kind always detects in FP64 (its whitened bins feed the SINR
    analysis of src/filters.py:185-198, not the hot path)."""
    import torch
    shp = tuple(cube.shape) if hasattr(cube, "shape") else np.shape(cube)
    if len(shp) != 3 or shp[1:] != (filt.p, filt.q):
        raise DimensionError(f"cube shape {shp} does not match filter ({filt.p}, {filt.q})")
    x = nat.to_device(cube)
    if filt.kind == "optimal":
        # whitened bins, then the identity projection (mode "kron", no bases)
        x, kind, ua, ub = filt._whiten(x), nat.KIND["kron"], None, None
    else:
        kind = filt._kind_code()
        ua, ub = filt._dev_bases()
    n, D, G = shp[0], dop.size, grid.shape[0]
    vals = torch.empty((groups, n, D), dtype=torch.float64, device=x.device)
    c = nat.ctx(x.device)
    if filt.kind == "optimal":
        precision = "f64"
    prev = None
    if precision is not None:
        b = C.c_int(0)
        nat.check(nat.lib().kst_get_detect(c, C.byref(b)), c)
        prev = b.value
        nat.check(nat.lib().kst_set_detect(c, {"f32": 32, "f64": 64}[precision]), c)
    try:
        nat.check(nat.lib().kst_detect(
            c, nat.ptr(x), n, filt.p, filt.q, nat.ptr(ua), 0 if ua is None else ua.shape[1],
            nat.ptr(ub), 0 if ub is None else ub.shape[1], kind, int(bool(filt.spatial_only)),
            dop.ctypes.data_as(nat.C.c_void_p), D, grid.ctypes.data_as(nat.C.c_void_p), G, groups,
            nat.ptr(vals), nat.stream_of(x.device)), c)
    finally:
        if prev is not None:
            nat.lib().kst_set_detect(c, prev)
    return vals


def detection_image(filt, cube, dopplers, spatial_grid, pool=None):
    """max_g |conj(H) F(X_m) conj(T)| per bin and Doppler (src/filters.py:243-275)."""
    shp = tuple(cube.shape) if hasattr(cube, "shape") else np.shape(cube)
    if len(shp) != 3 or shp[1:] != (filt.p, filt.q):
        raise DimensionError(f"cube shape {shp} does not match filter ({filt.p}, {filt.q})")
    dop, grid = _host_grid_args(filt, dopplers, spatial_grid)
    vals = run_detect(filt, cube, dop, grid)[0]
    return DetectionMap(vals if nat.is_device(cube) else nat.to_host(vals), dop, grid)


def set_detect_precision(precision="f32", device=None):
    """Select the detection (K5) arithmetic for this thread's context:
    "f32" (default: FP64 load pass -- spatial reduction and temporal
    coefficients -- then an FP32 prime-factor Doppler transform and pixel
    stage, within the SURVEY.md §8c map comparator; single-map uniform-grid
    cases, the rest run in FP64) or "f64" (FP64 kernels everywhere; maps to
    ~1e-12 of the reference)."""
    c = nat.ctx(device)
    bits = {"f32": 32, "f64": 64}[precision]
    nat.check(nat.lib().kst_set_detect(c, bits), c)


def get_detect_precision(device=None):
    c = nat.ctx(device)
    b = C.c_int(0)
    nat.check(nat.lib().kst_get_detect(c, C.byref(b)), c)
    return "f32" if b.value == 32 else "f64"
