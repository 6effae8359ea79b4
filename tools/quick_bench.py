"""Stage timing on one GPU (CUDA events), for development; bench.py is the contract."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes

q = int(sys.argv[1]) if len(sys.argv) > 1 else 2001
t0 = time.time()
hist = scenes.bench_scene(3, q, q, seed=17)
cube = torch.from_numpy(hist.data[0]).cuda()
print(f"scene gen {time.time()-t0:.1f}s", flush=True)
n, p, q = cube.shape
dop, grid = kst.make_doppler_grid(q), kst.make_spatial_grid(p)

def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e

for rep in range(3):
    e0 = ev()
    scm = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    e1 = ev()
    est = kst.lr_kron_estimate(scm, 1, 3)
    e2 = ev()
    filt = kst.build_filter("kron", estimate=est)
    e3 = ev()
    img = kst.detection_image(filt, cube, dop, grid)
    e4 = ev()
    torch.cuda.synchronize()
    print(f"scm {e0.elapsed_time(e1):.3f} ms  lrkron {e1.elapsed_time(e2):.3f} ms (iters {est.iterations})  "
          f"build {e2.elapsed_time(e3):.3f} ms  detect {e3.elapsed_time(e4):.3f} ms", flush=True)
for rep in range(3):
    e0 = ev()
    vals, s = kst.process_frame_device(cube, 1, 3, dop, grid)
    e1 = ev(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"pipeline {ms:.3f} ms  -> {n*q/ms*1e3:.3e} px/s  summary {s[:5]}", flush=True)
flops = 4.0 * n * (p * q) ** 2
print(f"gram algorithmic {flops:.3e} flop")
