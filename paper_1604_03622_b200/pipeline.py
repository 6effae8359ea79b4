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
from .errors import DimensionError, KronStapError
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


class FrameGraph:
    """One frame of the fused pipeline as a replayable CUDA graph.

    The sync-free schedule of kst_pipeline (kst_pipeline_async: every
    decision on the device, ~40 kernels, no host round trip) is captured once
    for a fixed device cube buffer and replayed per frame: the host cost of a
    frame is one graph launch. Write each frame into `cube` (same shape,
    device-resident), then

        fg = FrameGraph(cube)            # warm-up + capture
        fg.replay()                      # enqueue the frame (current stream)
        values, summary = fg.result()    # synchronise, read the outcome

    result() checks the device outcome record; a frame outside the
    sync-free assumptions (degenerate iterate, eigensolver needing a second
    round, k_A < r_A, k_B < r_B) is recomputed by kst_pipeline's synchronous
    path, so values and errors equal process_frame_device's either way. The
    graph is re-captured automatically when resident device state it depends
    on changed since capture (kst_state_epoch: a workspace reallocated, a
    constant bank or detection table restaged by another call on the GPU).
    """

    def __init__(self, cube, rank_spatial=1, rank_temporal=3, dopplers=None, spatial_grid=None,
                 tol=1e-4, max_iter=100, kind="kron", groups=1, out=None):
        import torch
        if cube.dim() != 3 or not cube.is_cuda or cube.dtype != torch.complex128:
            raise DimensionError("FrameGraph needs a device complex128 cube (n, p, q)")
        self.cube = cube
        n, p, q = cube.shape
        self.dop = np.ascontiguousarray(make_doppler_grid(q) if dopplers is None else
                                        np.asarray(dopplers, dtype=np.float64).ravel())
        self.grid = np.ascontiguousarray(make_spatial_grid(p) if spatial_grid is None else
                                         np.asarray(spatial_grid, dtype=np.complex128))
        if self.grid.ndim != 2 or self.grid.shape[1] != p:
            raise DimensionError(f"spatial grid shape {self.grid.shape} does not match p = {p}")
        if kind not in nat.KIND:
            raise DimensionError(f"unknown projection filter kind {kind!r}")
        self.args = (int(rank_spatial), int(rank_temporal), float(tol), int(max_iter), nat.KIND[kind])
        self.kwargs = dict(rank_spatial=rank_spatial, rank_temporal=rank_temporal, dopplers=self.dop,
                           spatial_grid=self.grid, tol=tol, max_iter=max_iter, kind=kind, groups=groups)
        self.groups = int(groups)
        D = self.dop.size
        self.values = out if out is not None else torch.empty((groups, n, D), dtype=torch.float64,
                                                              device=cube.device)
        self.rec = torch.zeros(8, dtype=torch.float64, device=cube.device)
        self.graph = None
        self.epoch = None
        self.captures = 0
        self.launches = 0

    def _enqueue(self):
        n, p, q = self.cube.shape
        ra, rb, tol, max_iter, kind = self.args
        c = nat.ctx(self.cube.device)
        nat.check(nat.lib().kst_pipeline_async(
            c, nat.ptr(self.cube), n, p, q, ra, rb, tol, max_iter, kind,
            self.dop.ctypes.data_as(C.c_void_p), self.dop.size,
            self.grid.ctypes.data_as(C.c_void_p), self.grid.shape[0], self.groups,
            nat.ptr(self.values), nat.ptr(self.rec), nat.stream_of(self.cube.device)), c)

    def _capture(self):
        import torch
        # warm-up: allocates the workspaces, uploads the constant banks and
        # stages the detection tables this shape needs, outside the capture
        self._enqueue()
        torch.cuda.synchronize(self.cube.device)
        before = nat.lib().kst_state_epoch()
        c = nat.ctx(self.cube.device)
        l0 = nat.lib().kst_launch_count(c)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            self._enqueue()
        self.launches = nat.lib().kst_launch_count(c) - l0  # kernels per replay
        after = nat.lib().kst_state_epoch()
        if after != before:  # the capture itself changed resident state: not replayable
            raise KronStapError("FrameGraph: resident state changed during capture")
        self.graph, self.epoch = g, after
        self.captures += 1

    def replay(self):
        """Enqueue the frame now in `cube` on the current stream."""
        if self.graph is None or nat.lib().kst_state_epoch() != self.epoch:
            self._capture()
        self.graph.replay()

    def result(self):
        """Synchronise; (values (groups, n, D) device tensor, summary ndarray[8])."""
        rec = self.rec.cpu().numpy()
        if rec[0] == 1.0:
            summary = np.zeros(8)
            summary[:5] = rec[1:6]
            return self.values, summary
        # an assumption of the sync-free form failed: the synchronous path
        return process_frame_device(self.cube, out=self.values, **self.kwargs)


class FrameStream:
    """Host-buffer frame sequence with copy/compute overlap.

    Frame i+1's host-to-device copy runs on an upload stream while frame i is
    processed on the compute stream; each map is copied back on a separate
    download stream once its frame is done, so the two PCIe directions (two
    copy engines) overlap each other and the compute. With pinned host buffers
    the traffic (192 MB in + 32 MB out per Gotcha frame) hides under the
    compute up to the host-to-device bandwidth. `nbuf` device cube buffers
    (default 3) let the upload of frame i+1 start as soon as frame i-2 is
    done, so the copy engine never waits on a frame whose compute (with its
    host round trips) ran long; with 2 it waits for frame i-1.

        fs = FrameStream(shape, device)
        for i, cube in enumerate(host_cubes):
            fs.submit(cube)          # returns the previous frame's map (or None)
        last = fs.flush()
    """

    def __init__(self, shape, device=None, rank_spatial=1, rank_temporal=3, dopplers=None,
                 spatial_grid=None, tol=1e-4, max_iter=100, kind="kron", out_pinned=None, nbuf=3,
                 groups=1, gather_group=None):
        import torch
        self.dev = torch.device("cuda", nat.device_index(device))
        n, p, q = shape
        if nbuf < 2:
            raise ValueError("FrameStream needs at least 2 buffers")
        self.nbuf = nbuf
        self.args = (rank_spatial, rank_temporal, dopplers, spatial_grid, tol, max_iter, kind,
                     groups)
        self.groups = groups
        D = q if dopplers is None else len(np.asarray(dopplers).ravel())
        self.bufs = [torch.empty(shape, dtype=torch.complex128, device=self.dev) for _ in range(nbuf)]
        self.outs = [torch.empty((groups, n, D), dtype=torch.float64, device=self.dev)
                     for _ in range(nbuf)]
        hshape = (n, D) if groups == 1 else (groups, n, D)
        # gather_group (torch.distributed, NCCL): every frame's maps are
        # all-gathered over NVLink into a (world, groups, n, D) device stack
        # right after the frame, and rank 0 downloads the whole gathered
        # stack (the other ranks download nothing): the SURVEY.md §8e map
        # gather inside the end-to-end stream
        self.gather = gather_group
        self.rank0 = True
        if gather_group is not None:
            import torch.distributed as dist
            self.world = dist.get_world_size(gather_group)
            self.rank0 = dist.get_rank(gather_group) == 0
            self.gbufs = [torch.empty((self.world, groups, n, D), dtype=torch.float64,
                                      device=self.dev) for _ in range(nbuf)]
            hshape = (self.world,) + ((n, D) if groups == 1 else (groups, n, D))
        self.host_out = out_pinned if out_pinned is not None else [
            torch.empty(hshape, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
        if len(self.host_out) < nbuf:
            raise ValueError(f"out_pinned needs {nbuf} host buffers")
        self.copy = torch.cuda.Stream(self.dev)       # host -> device
        self.copy_back = torch.cuda.Stream(self.dev)  # device -> host
        self.comp = torch.cuda.current_stream(self.dev)
        self.ready = [torch.cuda.Event() for _ in range(nbuf)]
        self.done = [torch.cuda.Event() for _ in range(nbuf)]
        self.back = [torch.cuda.Event() for _ in range(nbuf)]
        self.i = 0
        self.pending = None
        self.summary = np.zeros(8)

    def _upload(self, host_cube, slot):
        import torch
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.done[slot])  # buffer free once its frame finished
            self.bufs[slot].copy_(host_cube, non_blocking=True)
            self.ready[slot].record(self.copy)

    def submit(self, host_cube):
        """Queue one pinned host cube; process the previously queued one."""
        import torch
        slot = self.i % self.nbuf
        self._upload(host_cube, slot)
        result = self._process_pending()
        self.pending = slot
        self.i += 1
        return result

    def _process_pending(self):
        import torch
        if self.pending is None:
            return None
        slot = self.pending
        self.comp.wait_event(self.ready[slot])
        self.comp.wait_event(self.back[slot])  # map buffer read back (frame i - nbuf)
        process_frame_device(self.bufs[slot], *self.args, out=self.outs[slot], summary=self.summary)
        if self.gather is not None:
            import torch.distributed as dist
            # NCCL all-gather on its own stream, ordered after this frame; the
            # compute stream waits for it before reusing gbufs/outs
            dist.all_gather_into_tensor(self.gbufs[slot], self.outs[slot], group=self.gather)
        self.done[slot].record(self.comp)
        with torch.cuda.stream(self.copy_back):
            self.copy_back.wait_event(self.done[slot])
            if self.gather is None:
                src = self.outs[slot][0] if self.groups == 1 else self.outs[slot]
                self.host_out[slot].copy_(src, non_blocking=True)
            elif self.rank0:
                src = self.gbufs[slot][:, 0] if self.groups == 1 else self.gbufs[slot]
                self.host_out[slot].copy_(src, non_blocking=True)
            self.back[slot].record(self.copy_back)
        self.pending = None
        return self.host_out[slot], self.back[slot]

    def flush(self):
        return self._process_pending()


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
