"""One int8-engine sample_covariance on a Gotcha frame (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes, lrkron
s = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cube = torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17).data[0]).cuda()
lrkron.set_gram_engine("int8", s)
for _ in range(2):
    S = kst.sample_covariance(kst.cube_to_snapshots(cube), 3, 2001).matrix
torch.cuda.synchronize(); print("ok")
