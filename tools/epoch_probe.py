"""Which resident-state changes happen between consecutive identical frames (KST_EPOCH_DEBUG)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
from paper_1604_03622_b200 import _native as nat
p, q, n = 3, 96, 40
cube = torch.from_numpy(scenes.bench_scene(p, q, n, seed=3, movers=2).data[0]).cuda()
for i in range(3):
    e = nat.lib().kst_state_epoch()
    kst.process_frame_device(cube, 1, 3)
    torch.cuda.synchronize()
    print(f"frame {i}: epoch {e} -> {nat.lib().kst_state_epoch()}", file=sys.stderr, flush=True)
print("--- kst_pipeline_async x3", file=sys.stderr, flush=True)
fg = kst.FrameGraph(cube, 1, 3)
for i in range(3):
    e = nat.lib().kst_state_epoch()
    fg._enqueue()
    torch.cuda.synchronize()
    print(f"async {i}: epoch {e} -> {nat.lib().kst_state_epoch()} rec {fg.rec.cpu().numpy()[:6]}",
          file=sys.stderr, flush=True)
big = torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17).data[0]).cuda()
fg = kst.FrameGraph(big, 1, 3)
for i in range(3):
    e = nat.lib().kst_state_epoch()
    fg._enqueue()
    torch.cuda.synchronize()
    print(f"gotcha async {i}: epoch {e} -> {nat.lib().kst_state_epoch()} rec {fg.rec.cpu().numpy()[:6]}",
          file=sys.stderr, flush=True)
