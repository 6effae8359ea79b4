"""Frames/s with 1 or 2 compute lanes while a background pinned H2D loop saturates PCIe."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
from paper_1604_03622_b200.pipeline import process_frame_device
dev = torch.device("cuda:0")
host = torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17).data[0]).pin_memory()
cubes = [host.to(dev), host.to(dev)]
dst = torch.empty_like(cubes[0])
dop, grid = kst.make_doppler_grid(2001), kst.make_spatial_grid(3)
stop = False
def bg():
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        while not stop:
            dst.copy_(host, non_blocking=True)
            s.synchronize()
class Lane(threading.Thread):
    def __init__(self, k):
        super().__init__(); self.k = k; self.go = threading.Event(); self.done = threading.Event(); self.n = 0
        self.daemon = True
    def run(self):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            while True:
                self.go.wait(); self.go.clear()
                for _ in range(self.n):
                    process_frame_device(cubes[self.k], 1, 3, dop, grid)
                s.synchronize(); self.done.set()
lanes = [Lane(0), Lane(1)]
[l.start() for l in lanes]
def run(nl, nf):
    for l in lanes[:nl]:
        l.n = nf // nl; l.done.clear(); l.go.set()
    t0 = time.perf_counter()
    for l in lanes[:nl]: l.done.wait()
    return (time.perf_counter() - t0) / (nf // nl * nl) * 1e3
for background in (False, True):
    stop = False
    th = threading.Thread(target=bg) if background else None
    if th: th.start()
    for nl in (1, 2, 1, 2):
        run(nl, 4)
        print(f"background h2d={background} lanes={nl}: {run(nl, 12):.3f} ms/frame")
    stop = True
    if th: th.join()
