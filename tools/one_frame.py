"""Run the fused pipeline on one Gotcha-scale frame `reps` times (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
q = int(sys.argv[1]) if len(sys.argv) > 1 else 2001
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cube = torch.from_numpy(scenes.bench_scene(3, q, q, seed=17).data[0]).cuda()
dop, grid = kst.make_doppler_grid(q), kst.make_spatial_grid(3)
for _ in range(reps):
    vals, s = kst.process_frame_device(cube, 1, 3, dop, grid)
torch.cuda.synchronize()
print("ok", s[:5])
