"""L-mode: windowed Kron-STAP estimation (BASELINE.json configs[3]).

The reference estimates one covariance from all bins of a frame; it has no
windowed mode. SURVEY.md §8 ("L-mode definition") fixes the windowed variant
as this loop over the reference's own functions: for each test bin m the
training bins are [s, s + n_w) with s = clamp(m - n_w // 2, 0, n_bins - n_w),

    est_m     = lr_kron_estimate(sample_covariance(cube_to_snapshots(cube[s:s+n_w]), p, q),
                                 r_a, r_b)                         (src/lrkron.py:53, 118)
    values[m] = detection_image(build_filter(kind, est_m), cube[m:m+1], dopplers,
                                grid).values[0]                    (src/filters.py:137, 243)

Here every step runs on the device (no host round trip of S or the cube):
the n_bins - n_w + 1 distinct windows are estimated once each, and the bins
that share a window (the first and last n_w // 2 + 1 bins share the edge
windows) are detected together in one call.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _native as nat
from .errors import DimensionError
from .filters import DetectionMap, StapFilter, _host_grid_args, build_filter, run_detect
from .layout import cube_to_snapshots
from .lrkron import get_gram_engine, lr_kron_estimate, sample_covariance, set_gram_engine


_local = threading.local()
_pools = {}
_pool_lock = threading.Lock()


def _pool(n):
    """Process-wide worker threads for concurrent windows (kept alive so each
    thread's kst context, workspace and stream are created once)."""
    with _pool_lock:
        p = _pools.get(n)
        if p is None:
            p = _pools[n] = ThreadPoolExecutor(max_workers=n, thread_name_prefix="kst-window")
        return p


def last_window_info():
    """Per-window records of this thread's last batched windowed call: rows
    {status, iterations, converged, ka, kb, Rayleigh-Ritz rounds, r, n_w r}
    (include/kst_b200.h kst_lmode); status 64 = recomputed on the step path."""
    return getattr(_local, "last_window_info", None)


def window_start(m, n_w, n_bins):
    """First training bin of test bin m: clamp(m - n_w // 2, 0, n_bins - n_w)."""
    return int(min(max(m - n_w // 2, 0), n_bins - n_w))


def window_bins(s, n_w, n_bins):
    """Test bins [lo, hi) whose training window starts at s."""
    h = n_w // 2
    lo = 0 if s == 0 else s + h
    hi = n_bins if s == n_bins - n_w else s + h + 1
    return lo, hi


def halo_range(lo, hi, n_w, n_bins):
    """Bins [a, b) a tile of test bins [lo, hi) reads: its own bins plus the
    halo its training windows reach (windowed L-mode)."""
    if not 0 <= lo < hi <= n_bins:
        raise DimensionError(f"test bins [{lo}, {hi}) outside [0, {n_bins})")
    return window_start(lo, n_w, n_bins), window_start(hi - 1, n_w, n_bins) + n_w


def windowed_detection_image(cube, n_w, rank_spatial, rank_temporal, dopplers, spatial_grid,
                             kind="kron", tol=1e-4, max_iter=100, drop_temporal=False,
                             return_estimates=False, bins=None, workers=8):
    """Detection map of the windowed (L-mode) estimator; cube (n_bins, p, q).

    Returns a DetectionMap (host arrays for numpy input, device tensor values
    for CUDA input); with return_estimates=True also the list of
    (window start, KronCovEstimate) pairs. bins=(lo, hi) computes only test
    bins [lo, hi) (map rows lo..hi-1, shape (hi - lo, D)); a host cube then
    has only the tile plus its halo (`halo_range`) copied to the device, so
    a tile-sharded frame moves each bin to at most the GPUs whose windows
    read it. `workers` host threads estimate windows concurrently (results
    are identical for any value).
    """
    import torch
    shp = tuple(cube.shape) if hasattr(cube, "shape") else np.shape(cube)
    if len(shp) != 3:
        raise DimensionError(f"cube must be (n_bins, p, q), got {shp}")
    n_bins, p, q = shp
    if not 1 <= n_w <= n_bins:
        raise DimensionError(f"window n_w={n_w} must be in [1, {n_bins}]")
    lo, hi = (0, n_bins) if bins is None else (int(bins[0]), int(bins[1]))
    a, b = halo_range(lo, hi, n_w, n_bins)
    x = nat.to_device(cube[a:b])  # the tile and its halo; a view for CUDA input
    snaps = cube_to_snapshots(x)
    dev_out = nat.is_device(cube)
    D = int(np.asarray(dopplers.cpu() if nat.is_device(dopplers) else dopplers).size)
    vals = torch.empty((hi - lo, D), dtype=torch.float64, device=x.device)
    starts = list(range(window_start(lo, n_w, n_bins), window_start(hi - 1, n_w, n_bins) + 1))
    ests = {}
    grids = {}
    # estimates not requested: the whole tile in ONE C call (kst_lmode: the
    # batched window estimator and detector; it hands windows outside its
    # limits to the per-window step path itself). The step-API loop below
    # keeps the per-window estimates (return_estimates) and serves as the
    # A/B reference path (KST_LMODE=serial).
    fused = not return_estimates and rank_temporal < q and kind in nat.KIND
    if fused:
        grids["dop"], grids["grid"] = _host_grid_args(StapFilter(kind, p, q), dopplers, spatial_grid)
        xc = x.contiguous()
        if os.environ.get("KST_LMODE", "batched") != "serial":
            dop, grid = grids["dop"], grids["grid"]
            c = nat.ctx(x.device)
            nwin = window_start(hi - 1, n_w, n_bins) - window_start(lo, n_w, n_bins) + 1
            info = np.zeros((nwin, 8), dtype=np.int32)
            nat.check(nat.lib().kst_lmode(
                c, nat.ptr(xc), a, n_bins, p, q, n_w, lo, hi, int(rank_spatial),
                int(rank_temporal), float(tol), int(max_iter), nat.KIND[kind],
                int(bool(drop_temporal)), dop.ctypes.data_as(nat.C.c_void_p), dop.size,
                grid.ctypes.data_as(nat.C.c_void_p), grid.shape[0], nat.ptr(vals),
                info.ctypes.data_as(nat.C.c_void_p), nat.stream_of(x.device)), c)
            _local.last_window_info = info
            dmap = DetectionMap(vals if dev_out else nat.to_host(vals), dop, grid)
            return dmap

    def run_fused(s_begin, s_end, step):
        dop, grid = grids["dop"], grids["grid"]
        c = nat.ctx(x.device)
        nat.check(nat.lib().kst_windowed(
            c, nat.ptr(xc), a, n_bins, p, q, n_w, lo, hi, s_begin, s_end, step,
            int(rank_spatial), int(rank_temporal), float(tol), int(max_iter), nat.KIND[kind],
            int(bool(drop_temporal)), dop.ctypes.data_as(nat.C.c_void_p), dop.size,
            grid.ctypes.data_as(nat.C.c_void_p), grid.shape[0], nat.ptr(vals),
            nat.stream_of(x.device)), c)

    def one_window(s):
        if fused:
            run_fused(s, s + 1, 1)
            return
        scm = sample_covariance(snaps[s - a:s - a + n_w], p, q)
        est = lr_kron_estimate(scm, rank_spatial, rank_temporal, tol=tol, max_iter=max_iter)
        filt = build_filter(kind, estimate=est, drop_temporal=drop_temporal)
        if "dop" not in grids:
            grids["dop"], grids["grid"] = _host_grid_args(filt, dopplers, spatial_grid)
        t0, t1 = window_bins(s, n_w, n_bins)
        t0, t1 = max(t0, lo), min(t1, hi)
        # L-mode detects in FP64 on every path (the batched lm_detect_kernel
        # and kst_windowed do)
        vals[t0 - lo:t1 - lo] = run_detect(filt, x[t0 - a:t1 - a], grids["dop"], grids["grid"],
                                           precision="f64")[0]
        if return_estimates:
            ests[s] = est

    # the first window runs alone (it uploads the device-global constant
    # plans); the rest run on `workers` host threads, each with its own CUDA
    # stream and kst context (one ctx per device and thread, include/kst_b200.h),
    # so the small per-window kernels and host round trips of different
    # windows overlap. Every window is computed exactly as in the serial loop.
    # Window Grams run on the FP64 DMMA engine on every path (kst_windowed
    # and the batched kst_lmode do: the CRT engine's 2^-32 column rounding can
    # lift a window's null b eigenvalues to the 1e-9 keep threshold)
    caller_engine = get_gram_engine(x.device)
    engine = ("dmma", caller_engine[1])
    set_gram_engine(*engine, device=x.device)
    try:
        _run_windows(starts, workers, one_window, run_fused, fused, x, engine)
    finally:
        set_gram_engine(*caller_engine, device=x.device)
    dop, grid = grids["dop"], grids["grid"]
    ests = [(s, ests[s]) for s in starts] if return_estimates else []
    dmap = DetectionMap(vals if dev_out else nat.to_host(vals), dop, grid)
    return (dmap, ests) if return_estimates else dmap


def _run_windows(starts, workers, one_window, run_fused, fused, x, engine):
    import torch
    one_window(starts[0])
    rest = starts[1:]
    nw = max(1, min(int(workers), len(rest)))
    if nw == 1:
        for s in rest:
            one_window(s)
    else:
        main = torch.cuda.current_stream(x.device)
        pool = _pool(nw)
        local = _local

        def worker(k):
            # persistent pool threads: their kst contexts and streams are reused
            torch.cuda.set_device(x.device)
            if get_gram_engine(x.device) != engine:
                set_gram_engine(*engine, device=x.device)
            streams = local.__dict__.setdefault("streams", {})
            st = streams.get(x.device.index)
            if st is None:
                st = streams[x.device.index] = torch.cuda.Stream(x.device)
            st.wait_stream(main)
            with torch.cuda.stream(st):
                if fused:
                    run_fused(rest[k], rest[-1] + 1, nw)
                else:
                    for s in rest[k::nw]:
                        one_window(s)
            return st

        futs = [pool.submit(worker, k) for k in range(nw)]
        done = [f.result() for f in futs]  # re-raises a worker's exception here
        for st in done:
            main.wait_stream(st)
