"""kst_copy_staged throughput vs host threads (192 MB cube up, 32 MB map down)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1604_03622_b200 import _native as nat
x = np.random.default_rng(0).standard_normal(2 * 2001 * 3 * 2001).view(np.complex128)
y = np.empty(2001 * 2001, dtype=np.float64)
dev = torch.empty(x.shape, dtype=torch.complex128, device="cuda")
dy = torch.zeros(y.shape, dtype=torch.float64, device="cuda")
c = nat.ctx(0)
for nth in (4, 8, 12, 16):
    for direction, (dst, src, nb) in (("h2d", (nat.ptr(dev), x.ctypes.data_as(nat.C.c_void_p), x.nbytes)),
                                      ("d2h", (y.ctypes.data_as(nat.C.c_void_p), nat.ptr(dy), y.nbytes))):
        d = 0 if direction == "h2d" else 1
        best = 1e9
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nat.check(nat.lib().kst_copy_staged(c, dst, src, nb, d, nth, nat.stream_of(0)), c)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{direction} {nth:2d} threads: {nb / best / 1e9:6.1f} GB/s", flush=True)
print("cores", os.cpu_count())
