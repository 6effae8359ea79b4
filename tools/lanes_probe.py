"""Throughput of 1 vs 2 concurrent frame pipelines (threads + streams + contexts)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
from paper_1604_03622_b200.pipeline import process_frame_device
dev = torch.device("cuda:0")
cubes = [torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17 + i).data[0]).to(dev) for i in range(2)]
dop, grid = kst.make_doppler_grid(2001), kst.make_spatial_grid(3)
NF = int(sys.argv[1]) if len(sys.argv) > 1 else 12

def lane(idx, nfr, out):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for i in range(nfr):
            v, _ = process_frame_device(cubes[idx % 2], 1, 3, dop, grid)
        s.synchronize()
    out[idx] = v

for lanes in (1, 2, 3, 1, 2):
    out = {}
    ths = [threading.Thread(target=lane, args=(k, 2, out)) for k in range(lanes)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=lane, args=(k, NF // lanes, out)) for k in range(lanes)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"lanes {lanes}: {dt / (NF // lanes * lanes) * 1e3:.3f} ms/frame")
ref = process_frame_device(cubes[0], 1, 3, dop, grid)[0]
print("lane result equal:", bool(torch.equal(out[0], ref)))
