"""L-mode windows on one 3 x 256 frame restricted to `nb` bins (ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 90
cube = torch.from_numpy(scenes.bench_scene(3, 256, 256, seed=17, movers=8).data[0][:nb]).cuda()
dop, grid = kst.make_doppler_grid(256), kst.make_spatial_grid(3, 16)
v = kst.windowed_detection_image(cube, 81, 1, 3, dop, grid, workers=1)
torch.cuda.synchronize()
print("ok", float(v.values.max()))
