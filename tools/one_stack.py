"""Run the fused pipeline on one 4-pass stacked cube `reps` times (configs[4], for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
from paper_1604_03622_b200.pipeline import process_frame_device
q = int(sys.argv[1]) if len(sys.argv) > 1 else 2001
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
K = 4
hist = scenes.bench_scene(3, q, q, seed=17, n_passes=K)
x = torch.from_numpy(np.ascontiguousarray(kst.stack_passes(hist).data)).cuda()
dop, grid = kst.make_doppler_grid(q), kst.make_stacked_spatial_grid(3, K, 16)
for _ in range(reps):
    vals, s = process_frame_device(x, K, 3, dop, grid, groups=K)
torch.cuda.synchronize()
print("ok", s[:5])
