"""Multi-GPU frame sharding (SURVEY.md §8e, configs[2]).

Frames of a sequence are independent units: rank r processes frames
r, r + W, r + 2W, ... (round robin) with the single-GPU pipeline and no
data-path collective. The only collective is the optional gather of the
detection maps to rank 0 (NCCL over NVLink on the GPU box; gloo works the
same way for the CPU tests). One process per GPU, launched by torchrun.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def frame_assignment(n_frames, world):
    """Frame indices per rank, round robin (deterministic)."""
    if n_frames < 0 or world < 1:
        raise ValueError("n_frames >= 0 and world >= 1 required")
    return [list(range(r, n_frames, world)) for r in range(world)]


def local_frames(n_frames, rank, world):
    return frame_assignment(n_frames, world)[rank]


def gather_maps(local_maps, n_frames, group=None, dst_all=True):
    """All-gather per-rank map stacks into the global frame order.

    local_maps: tensor (k_local, n, D) holding this rank's frames in the order
    of `local_frames`. Ranks with fewer frames are padded to the per-rank
    maximum (all_gather needs equal shapes). Returns (n_frames, n, D) on
    every rank (or None off rank 0 when dst_all is False).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_frames // world) if n_frames else 0
    k_local, *tail = local_maps.shape
    assert k_local == len(local_frames(n_frames, rank, world))
    pad = torch.zeros((per, *tail), dtype=local_maps.dtype, device=local_maps.device)
    pad[:k_local] = local_maps
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if not dst_all and rank != 0:
        return None
    out = torch.empty((n_frames, *tail), dtype=local_maps.dtype, device=local_maps.device)
    for r, frames in enumerate(frame_assignment(n_frames, world)):
        for j, f in enumerate(frames):
            out[f] = bufs[r][j]
    return out


def process_sequence(frames, rank_spatial=1, rank_temporal=3, dopplers=None, spatial_grid=None,
                     group=None, gather=True, tol=1e-4, max_iter=100, kind="kron", device=None):
    """Run the fused pipeline over this rank's share of `frames` (a sequence
    of (n, p, q) cubes: numpy, CPU tensors -- pinned or not -- or CUDA
    tensors) and optionally all-gather every rank's maps.

    Uploads overlap compute: frame j+1 is staged into a pinned host buffer
    and copied host -> device on a side stream while frame j runs on the
    compute stream (two device cube buffers, event-ordered). Maps are written
    straight into one device stack (k_local, n, D), which is what the NCCL
    all-gather sends -- no device -> host -> device round trip.
    Returns the (n_frames, n, D) float64 tensor on this rank's device
    (gather and world > 1), else this rank's (k_local, n, D) stack.
    """
    from . import _native as nat
    from .pipeline import process_frame_device
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = local_frames(len(frames), rank, world)
    dev = torch.device("cuda", nat.device_index(device))
    if len(frames):
        n, p, q = (int(s) for s in frames[0].shape)
    else:
        n = p = q = 0
    D = len(np.ravel(dopplers)) if dopplers is not None else q
    maps = torch.empty((len(mine), n, D), dtype=torch.float64, device=dev)
    if mine:
        comp = torch.cuda.current_stream(dev)
        up = torch.cuda.Stream(dev)
        bufs = [torch.empty((n, p, q), dtype=torch.complex128, device=dev) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        staged = [None, None]
        pins, pin_free = [None, None], [torch.cuda.Event() for _ in range(2)]

        def upload(j):
            slot = j % 2
            src = frames[mine[j]]
            if isinstance(src, torch.Tensor) and src.is_cuda:
                staged[slot] = src  # already resident: no copy
                ready[slot].record(comp)
                return
            if isinstance(src, torch.Tensor) and src.is_pinned():
                host = src
            else:
                if pins[slot] is None:
                    pins[slot] = torch.empty((n, p, q), dtype=torch.complex128).pin_memory()
                pin_free[slot].synchronize()  # previous upload out of this pin buffer done
                pins[slot].copy_(torch.as_tensor(np.asarray(src, dtype=np.complex128))
                                 if not isinstance(src, torch.Tensor) else src)
                host = pins[slot]
            with torch.cuda.stream(up):
                up.wait_event(done[slot])  # device buffer free once frame j-2 finished
                bufs[slot].copy_(host, non_blocking=True)
                ready[slot].record(up)
                pin_free[slot].record(up)
            staged[slot] = bufs[slot]

        upload(0)
        for j in range(len(mine)):
            if j + 1 < len(mine):
                upload(j + 1)
            slot = j % 2
            comp.wait_event(ready[slot])
            process_frame_device(staged[slot], rank_spatial, rank_temporal, dopplers, spatial_grid,
                                 tol, max_iter, kind, out=maps[j:j + 1])
            done[slot].record(comp)
    if not gather or world == 1:
        return maps
    if dist.get_backend(group) != "nccl":
        maps = maps.cpu()
    return gather_maps(maps, len(frames), group)


def local_stack(maps, frames, dopplers, dev):
    """This rank's maps as one (k_local, n, D) tensor on `dev`. A rank with no
    frames (fewer frames than ranks) contributes an EMPTY stack of the same
    trailing shape, so all_gather sees equal (per, n, D) pads on every rank."""
    if maps:
        return torch.stack([torch.as_tensor(m).to(dev) for m in maps])
    n_bins = int(frames[0].shape[0]) if len(frames) else 0
    n_dop = (len(np.ravel(dopplers)) if dopplers is not None
             else (int(frames[0].shape[2]) if len(frames) else 0))
    return torch.zeros((0, n_bins, n_dop), dtype=torch.float64, device=dev)


# ----------------------------------------------------------------- L-mode tiles
def tile_bounds(n_bins, world):
    """Contiguous test-bin tiles [lo, hi) per rank, sizes differing by at most
    one (windowed L-mode shards by bin tile + halo)."""
    if n_bins < 0 or world < 1:
        raise ValueError("n_bins >= 0 and world >= 1 required")
    base, extra = divmod(n_bins, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def gather_tiles(local_rows, n_rows, group=None):
    """All-gather row tiles (tile_bounds order) into the full (n_rows, ...) map
    on every rank; tiles are padded to the largest tile for all_gather."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = tile_bounds(n_rows, world)
    per = max(hi - lo for lo, hi in bounds)
    k, *tail = local_rows.shape
    assert k == bounds[rank][1] - bounds[rank][0]
    pad = torch.zeros((per, *tail), dtype=local_rows.dtype, device=local_rows.device)
    pad[:k] = local_rows
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[r][:hi - lo] for r, (lo, hi) in enumerate(bounds)])


def windowed_sharded(cube, n_w, rank_spatial, rank_temporal, dopplers, spatial_grid, group=None,
                     gather=True, **kw):
    """L-mode detection of one frame tiled over the ranks of `group`: rank r
    detects test bins tile_bounds(n_bins, W)[r], reading only its tile plus
    the halo its training windows reach (windowed.halo_range); no exchange on
    the data path. Returns the full (n_bins, D) map on every rank (gather) or
    this rank's (hi - lo, D) tile."""
    from .windowed import windowed_detection_image
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_bins = int(cube.shape[0])
    lo, hi = tile_bounds(n_bins, world)[rank]
    if hi > lo:
        vals = torch.as_tensor(windowed_detection_image(
            cube, n_w, rank_spatial, rank_temporal, dopplers, spatial_grid, bins=(lo, hi),
            **kw).values)
    else:
        vals = torch.zeros((0, len(dopplers)), dtype=torch.float64)
    if not gather or world == 1:
        return vals
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    return gather_tiles(vals.to(dev), n_bins, group)
