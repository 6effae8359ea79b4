"""Fused frame pipeline: cube -> detection map in one C-ABI call.

The README library sequence (pkg/README.md:144-161)

    sample_covariance(cube_to_snapshots(cube)) -> lr_kron_estimate(scm, ra, rb)
      -> build_filter(kind) -> detection_image(filt, cube, dopplers, grid)

as one `kst_pipeline` call with every intermediate (S, b, bases, spectra)
kept in the context's HBM workspace. `process_frame` accepts numpy (host
buffers: H2D + D2H included) or CUDA tensors.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .errors import DimensionError
from .filters import make_doppler_grid, make_spatial_grid


def process_frame_device(cube, rank_spatial=1, rank_temporal=3, dopplers=None, spatial_grid=None,
                         tol=1e-4, max_iter=100, kind="kron", groups=1, out=None, summary=None):
    """Device-resident cube (n, p, q) complex128 -> values (groups, n, D) float64 tensor.

    Returns (values, summary ndarray[8])."""
    import torch
    if cube.dim() != 3:
        raise DimensionError(f"cube must be 3-D, got shape {tuple(cube.shape)}")
    n, p, q = cube.shape
    dop = np.ascontiguousarray(make_doppler_grid(q) if dopplers is None else
                               np.asarray(dopplers, dtype=np.float64).ravel())
    grid = np.ascontiguousarray(make_spatial_grid(p) if spatial_grid is None else
                                np.asarray(spatial_grid, dtype=np.complex128))
    if grid.ndim != 2 or grid.shape[1] != p:
        raise DimensionError(f"spatial grid shape {grid.shape} does not match p = {p}")
    if kind not in nat.KIND:
        raise DimensionError(f"unknown projection filter kind {kind!r}")
    D, G = dop.size, grid.shape[0]
    if out is None:
        out = torch.empty((groups, n, D), dtype=torch.float64, device=cube.device)
    if summary is None:
        summary = np.zeros(8)
    c = nat.ctx(cube.device)
    nat.check(nat.lib().kst_pipeline(
        c, nat.ptr(cube), n, p, q, int(rank_spatial), int(rank_temporal), float(tol), int(max_iter),
        nat.KIND[kind], dop.ctypes.data_as(C.c_void_p), D, grid.ctypes.data_as(C.c_void_p), G,
        groups, nat.ptr(out), summary.ctypes.data_as(C.c_void_p), nat.stream_of(cube.device)), c)
    return out, summary


def process_frame(cube, rank_spatial=1, rank_temporal=3, dopplers=None, spatial_grid=None,
                  tol=1e-4, max_iter=100, kind="kron"):
    """cube (n, p, q) numpy or tensor -> (values (n, D) float64, summary dict)."""
    dev_in = nat.is_device(cube)
    x = nat.to_device(cube)
    vals, s = process_frame_device(x, rank_spatial, rank_temporal, dopplers, spatial_grid, tol,
                                   max_iter, kind)
    info = dict(iterations=int(s[0]), converged=bool(s[1]), ka=int(s[2]), kb=int(s[3]),
                residual=float(s[4]))
    v = vals[0]
    return (v if dev_in else nat.to_host(v)), info
