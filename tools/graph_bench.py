"""Gotcha frame: back-to-back process_frame_device vs FrameGraph replay (CUDA events, 20 frames)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
cube = torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17).data[0]).cuda()
out = torch.empty((1, 2001, 2001), dtype=torch.float64, device="cuda")
K = 20


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for rep in range(3):
    for _ in range(3):
        kst.process_frame_device(cube, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0 = ev()
    for _ in range(K):
        kst.process_frame_device(cube, out=out)
    e1 = ev(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"direct: {e0.elapsed_time(e1) / K:.3f} ms/frame (events), host {1e3 * (t1 - t0) / K:.3f} ms",
          flush=True)
fg = kst.FrameGraph(cube, out=out)
ref = out.clone()
for rep in range(3):
    for _ in range(3):
        fg.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0 = ev()
    for _ in range(K):
        fg.replay()
    e1 = ev(); torch.cuda.synchronize(); t1 = time.perf_counter()
    ok = float(fg.rec[0])
    print(f"graph:  {e0.elapsed_time(e1) / K:.3f} ms/frame (events), host {1e3 * (t1 - t0) / K:.3f} ms, "
          f"rec ok {ok}, captures {fg.captures}", flush=True)
vals, summ = fg.result()
print("equal to direct:", bool(torch.equal(vals, ref)), summ[:5])
