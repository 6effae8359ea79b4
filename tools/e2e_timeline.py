"""Timeline of FrameStream (upload / compute / download per frame) from CUDA events.

    python tools/e2e_timeline.py [frames]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes
from paper_1604_03622_b200.pipeline import FrameStream, process_frame_device

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda:0")
cubes = [torch.from_numpy(scenes.bench_scene(3, 2001, 2001, seed=17 + i).data[0]).pin_memory() for i in range(2)]
dop, grid = kst.make_doppler_grid(2001), kst.make_spatial_grid(3)
fs = FrameStream((2001, 3, 2001), dev, 1, 3, dop, grid)
ev = lambda: torch.cuda.Event(enable_timing=True)
# instrument: wrap the streams' work with events
up, comp, down, stages = [], [], [], []
from paper_1604_03622_b200 import _native as nat
nat.lib().kst_set_profiling(nat.ctx(dev), 1)
orig_upload, orig_proc = fs._upload, fs._process_pending
def _upload(host, slot):
    a, b = ev(), ev()
    a.record(fs.copy)
    orig_upload(host, slot)
    b.record(fs.copy)
    up.append((a, b))
def _proc():
    if fs.pending is None:
        return None
    a, b = ev(), ev()
    fs.comp.wait_event(fs.ready[fs.pending])
    a.record(fs.comp)
    t0 = time.perf_counter()
    r = orig_proc()
    host_ms = (time.perf_counter() - t0) * 1e3
    st = np.zeros(8)
    k = nat.lib().kst_stage_times(nat.ctx(dev), st.ctypes.data_as(nat.C.c_void_p), 8)
    stages.append(st[:k].round(3).tolist())
    b.record(fs.comp)
    c = ev(); c.record(fs.copy_back)
    comp.append((a, b, host_ms))
    down.append(c)
    return r
fs._upload, fs._process_pending = _upload, _proc
for i in range(3):
    fs.submit(cubes[i % 2])
fs.flush()
torch.cuda.synchronize()
up.clear(); comp.clear(); down.clear(); stages.clear()
z = ev(); z.record(fs.comp)
t0 = time.perf_counter()
for i in range(nf):
    fs.submit(cubes[i % 2])
fs.flush()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"wall {wall:.2f} ms for {nf} frames = {wall / nf:.3f} ms/frame")
for i in range(nf):
    u0, u1 = (z.elapsed_time(e) for e in up[i])
    c0, c1, hm = comp[i]
    print(f"frame {i}: upload {u0:8.3f}-{u1:8.3f} ({u1 - u0:.3f})  compute {z.elapsed_time(c0):8.3f}-"
          f"{z.elapsed_time(c1):8.3f} ({c0.elapsed_time(c1):.3f}, host call {hm:.3f})  "
          f"map back {z.elapsed_time(down[i]):8.3f}  stages {stages[i]}")
# the same frames without concurrent uploads
for i in range(3):
    x = torch.empty_like(cubes[0], device=dev); x.copy_(cubes[i % 2])
    torch.cuda.synchronize()
    a, b = ev(), ev(); a.record()
    process_frame_device(x, 1, 3, dop, grid)
    b.record(); torch.cuda.synchronize()
    st = np.zeros(8)
    k = nat.lib().kst_stage_times(nat.ctx(dev), st.ctypes.data_as(nat.C.c_void_p), 8)
    print(f"alone: {a.elapsed_time(b):.3f} ms stages {st[:k].round(3).tolist()}")
