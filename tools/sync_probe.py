"""Host round trip (tiny kernel + stream sync) and launch cost, with and without a background pinned H2D loop."""
import os, sys, threading, time
import numpy as np
import torch
dev = torch.device("cuda:0")
host = torch.empty(192 * 2**20 // 8, dtype=torch.float64).pin_memory()
dst = torch.empty_like(host, device=dev)
x = torch.zeros(16, device=dev)
stop = False
def bg():
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        while not stop:
            dst.copy_(host, non_blocking=True)
            s.synchronize()
s = torch.cuda.Stream(dev)
for background in (False, True, False):
    stop = False
    th = threading.Thread(target=bg) if background else None
    if th: th.start()
    time.sleep(0.05)
    with torch.cuda.stream(s):
        rt = []
        for _ in range(200):
            t0 = time.perf_counter(); x.add_(1); s.synchronize(); rt.append(time.perf_counter() - t0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.synchronize(); e0.record(s)
        for _ in range(200): x.add_(1)
        e1.record(s); e1.synchronize()
        back = torch.empty(16, pin_memory=True)
        d2h = []
        for _ in range(100):
            t0 = time.perf_counter(); back.copy_(x, non_blocking=True); s.synchronize(); d2h.append(time.perf_counter() - t0)
    stop = True
    if th: th.join()
    print(f"background={background}: kernel+sync round trip median {np.median(rt)*1e6:.1f} us, "
          f"p90 {np.percentile(rt, 90)*1e6:.1f} us; 200 back-to-back tiny kernels {e0.elapsed_time(e1)*1e3/200:.2f} us each; "
          f"tiny D2H+sync {np.median(d2h)*1e6:.1f} us")
