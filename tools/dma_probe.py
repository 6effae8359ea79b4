"""Frame compute time alone vs with a concurrent pinned H2D / D2D copy loop."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes, _native as nat
from paper_1604_03622_b200.pipeline import process_frame_device
dev = torch.device("cuda:0")
host = torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17).data[0]).pin_memory()
cube = host.to(dev)
dst = torch.empty_like(cube)
dop, grid = kst.make_doppler_grid(2001), kst.make_spatial_grid(3)
nat.lib().kst_set_profiling(nat.ctx(dev), 1)
stop = False
def bg(kind):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        while not stop:
            if kind == "h2d":
                dst.copy_(host, non_blocking=True)
            else:
                dst.copy_(cube, non_blocking=True)
            s.synchronize()
for kind in ("none", "h2d", "d2d", "none"):
    stop = False
    th = threading.Thread(target=bg, args=(kind,)) if kind != "none" else None
    if th: th.start()
    time.sleep(0.05)
    ts, sts = [], []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        process_frame_device(cube, 1, 3, dop, grid)
        e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        st = np.zeros(8); k = nat.lib().kst_stage_times(nat.ctx(dev), st.ctypes.data_as(nat.C.c_void_p), 8)
        sts.append(st[:4])
    stop = True
    if th: th.join()
    print(f"{kind:5s}: {np.median(ts):.3f} ms  stages {np.median(np.array(sts), axis=0).round(3).tolist()}")
