"""CPU, world_size 2 over gloo: the frame-sharding host logic of the N > 1
path (paper_1604_03622_b200/parallel.py). Each rank computes its frames'
maps with the CPU oracle standing in for the GPU pipeline (test only), then
the maps are gathered into global frame order and checked on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_03622_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _frames():
    from paper_1604_03622_b200 import scenes
    return [scenes.bench_scene(3, 16, 24, seed=100 + f, movers=1).data[0] for f in range(5)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kron_oracle as orc
        frames = _frames()
        mine = parallel.local_frames(len(frames), rank, world)
        maps = [torch.from_numpy(orc.pipeline(frames[f], 1, 3, 16)[3]) for f in mine]
        local = torch.stack(maps)
        full = parallel.gather_maps(local, len(frames))
        want = np.stack([orc.pipeline(fr, 1, 3, 16)[3] for fr in frames])
        q.put((rank, bool(np.array_equal(full.numpy(), want)), mine))
    finally:
        dist.destroy_process_group()


def _few_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kron_oracle as orc
        frames = _frames()[:1]  # one frame, two ranks: rank 1 holds nothing
        mine = parallel.local_frames(len(frames), rank, world)
        maps = [orc.pipeline(frames[f], 1, 3, 16)[3] for f in mine]
        local = parallel.local_stack(maps, frames, np.arange(16) / 16, torch.device("cpu"))
        full = parallel.gather_maps(local, len(frames))
        want = orc.pipeline(frames[0], 1, 3, 16)[3][None]
        q.put((rank, tuple(local.shape), bool(np.array_equal(full.numpy(), want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_fewer_frames_than_ranks_gathers_equal_shapes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_few_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = {r: rest for r, *rest in res}
    assert res[0][0] == (1, 24, 16) and res[1][0] == (0, 24, 16)
    assert res[0][1] and res[1][1]


def test_frame_assignment_is_a_partition():
    for n, w in ((0, 1), (5, 2), (100, 8), (3, 4)):
        parts = parallel.frame_assignment(n, w)
        flat = sorted(f for p in parts for f in p)
        assert flat == list(range(n))
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


@pytest.mark.timeout(300)
def test_two_rank_gather_reassembles_frame_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == [0, 1]
    assert all(ok for _, ok, _ in res)
    assert {r: m for r, _, m in res} == {0: [0, 2, 4], 1: [1, 3]}


# ------------------------------------------------------------ L-mode bin tiles
def test_tile_bounds_and_halo_cover_every_window():
    from paper_1604_03622_b200.windowed import halo_range, window_start
    for n, w in ((24, 2), (256, 8), (7, 3), (5, 8)):
        tiles = parallel.tile_bounds(n, w)
        assert tiles[0][0] == 0 and tiles[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(tiles, tiles[1:]))
        assert max(h - l for l, h in tiles) - min(h - l for l, h in tiles) <= 1
        for n_w in (1, 2, 5, n):
            if n_w > n:
                continue
            for lo, hi in tiles:
                if hi == lo:
                    continue
                a, b = halo_range(lo, hi, n_w, n)
                assert 0 <= a <= lo and hi <= b <= n
                for m in range(lo, hi):
                    s = window_start(m, n_w, n)
                    assert a <= s and s + n_w <= b
                # the halo is minimal: the first and last windows touch its ends
                assert window_start(lo, n_w, n) == a and window_start(hi - 1, n_w, n) + n_w == b


def _tile_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kron_oracle as orc
        from paper_1604_03622_b200.windowed import halo_range
        from paper_1604_03622_b200 import scenes
        cube = scenes.bench_scene(3, 16, 24, seed=7, movers=1).data[0]
        n_w = 5
        lo, hi = parallel.tile_bounds(cube.shape[0], world)[rank]
        a, b = halo_range(lo, hi, n_w, cube.shape[0])
        # this rank may only read its tile and halo: poison everything else
        seen = np.full_like(cube, np.nan)
        seen[a:b] = cube[a:b]
        tile = orc.windowed(seen, n_w, 1, 3, 16, bins=range(lo, hi))[0][lo:hi]
        full = parallel.gather_tiles(torch.from_numpy(tile), cube.shape[0]).numpy()
        want = orc.windowed(cube, n_w, 1, 3, 16)[0]
        q.put((rank, bool(np.isfinite(tile).all()), bool(np.array_equal(full, want)), (lo, hi, a, b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_lmode_tiles_with_halo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tile_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = {r: rest for r, *rest in res}
    assert set(res) == {0, 1}
    assert all(fin and eq for fin, eq, _ in res.values())
    assert res[0][2] == (0, 12, 0, 14) and res[1][2] == (12, 24, 10, 24)
