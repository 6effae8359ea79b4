"""Hermitian eigen-helpers with the reference conventions, on the GPU.

Mirrors `kronstap.linalg.hermitian_eig / eig_truncate` (src/linalg.py:82-144):
values descending, ties ordered by dominant index, pivot entry real positive,
negative rounding-level eigenvalues clamped in truncation. Backed by
kst_heig_top / kst_eig_truncate (Jacobi for n <= 64, block-Krylov
Rayleigh-Ritz above).
"""

from __future__ import annotations

import ctypes as C
from collections import namedtuple

import numpy as np

from . import _native as nat
from .errors import DataError, DimensionError

EigenPairs = namedtuple("EigenPairs", ["values", "vectors"])


def _square(m, name="matrix"):
    shp = tuple(m.shape) if hasattr(m, "shape") else np.shape(m)
    if len(shp) != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {shp}")
    if shp[0] != shp[1]:
        raise DimensionError(f"{name} must be square, got {shp}")
    return shp[0]


def as_matrix(m, name="matrix"):
    """Validate and return a 2-D complex128 array with finite entries
    (src/linalg.py:25-33). Host-side helper for small inputs."""
    arr = np.asarray(m.cpu() if nat.is_device(m) else m)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {arr.shape}")
    arr = arr.astype(np.complex128, copy=False)
    if not np.all(np.isfinite(arr)):
        raise DataError(f"{name} contains non-finite entries")
    return arr


def hermitian_eig(m):
    """Full eigendecomposition with the reference conventions."""
    import torch
    n = _square(m)
    device_mode = nat.is_device(m)
    x = nat.to_device(m)
    if n == 0:
        v = np.zeros(0), np.zeros((0, 0), complex)
        return EigenPairs(*v)
    c = nat.ctx(x.device)
    vals = np.zeros(n)
    vecs = torch.empty((n, n), dtype=torch.complex128, device=x.device)
    nat.check(nat.lib().kst_heig_top(c, nat.ptr(x), n, n, vals.ctypes.data_as(C.c_void_p),
                                     nat.ptr(vecs), nat.stream_of(x.device)), c)
    return EigenPairs(vals, vecs if device_mode else nat.to_host(vecs))


def eig_truncate(m, rank):
    """Best Hermitian approximation keeping the top `rank` eigenpairs."""
    import torch
    n = _square(m)
    x = nat.to_device(m)
    c = nat.ctx(x.device)
    out = torch.empty((n, n), dtype=torch.complex128, device=x.device)
    nat.check(nat.lib().kst_eig_truncate(c, nat.ptr(x), n, int(rank), nat.ptr(out),
                                         nat.stream_of(x.device)), c)
    return out if nat.is_device(m) else nat.to_host(out)


def subspace_basis_device(m, rank, tol=1e-9):
    """Device tensor (n, keep) or None -- src/filters.py:58-73."""
    import torch
    n = _square(m)
    x = nat.to_device(m)
    c = nat.ctx(x.device)
    r = max(min(int(rank), n), 1)
    out = torch.empty(n * r, dtype=torch.complex128, device=x.device)
    keep = C.c_int(0)
    nat.check(nat.lib().kst_subspace_basis(c, nat.ptr(x), n, int(rank), float(tol), nat.ptr(out),
                                           C.byref(keep), nat.stream_of(x.device)), c)
    k = keep.value
    if k == 0:
        return None
    return out[:n * k].view(n, k)  # written densely as (n, keep)
