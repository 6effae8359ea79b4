import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes, windowed
p, q, nb, D, G, n_w = 3, 2001, 2001, 2001, 16, 81
cube = torch.from_numpy(scenes.bench_scene(p, q, nb, seed=17, movers=8).data[0]).cuda()
dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid)
info = windowed.last_window_info()
fb = np.nonzero(info[:, 0] != 0)[0]
print("fallback windows", fb.tolist())
print(info[fb].tolist())
print("rounds hist", np.bincount(info[info[:, 0] == 0, 5]).tolist())
