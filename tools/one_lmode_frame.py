"""Batched L-mode (kst_lmode) on the configs[3] 256 x 256 frame `reps` times (ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cube = torch.from_numpy(scenes.bench_scene(3, q, q, seed=17, movers=8).data[0]).cuda()
dop, grid = kst.make_doppler_grid(q), kst.make_spatial_grid(3, 16)
for _ in range(reps):
    v = kst.windowed_detection_image(cube, 81, 1, 3, dop, grid)
torch.cuda.synchronize()
print("ok", float(v.values.cpu().numpy().max()))  # host-side max: no library kernel in the launch list
