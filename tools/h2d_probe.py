"""Host->device bandwidth for a 192 MB complex128 cube: pageable torch copy,
pinned copy, and chunked staging through a pinned ring with host threads."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 2001 * 3 * 2001
x = (np.random.default_rng(0).standard_normal(2 * n).view(np.complex128)).reshape(2001, 3, 2001)
nbytes = x.nbytes
dev = torch.empty(x.shape, dtype=torch.complex128, device="cuda")


def bw(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9


print(f"pageable torch copy   {bw(lambda: dev.copy_(torch.from_numpy(x))):6.1f} GB/s")
pin = torch.empty(x.shape, dtype=torch.complex128, pin_memory=True)
pin.numpy()[...] = x
print(f"pinned copy           {bw(lambda: dev.copy_(pin, non_blocking=True)):6.1f} GB/s")
print(f"host memcpy 1 thread  {bw(lambda: np.copyto(pin.numpy(), x)):6.1f} GB/s")
flat_src = x.reshape(-1).view(np.uint8)
flat_pin = pin.numpy().reshape(-1).view(np.uint8)
flat_dev = dev.view(-1).view(torch.uint8)
for nth in (2, 4, 8):
    for chunk_mb in (4, 16):
        ch = chunk_mb << 20
        nch = (nbytes + ch - 1) // ch
        pool = ThreadPoolExecutor(nth)
        st = torch.cuda.Stream()

        def staged():
            def cp(i):
                a, b = i * ch, min(nbytes, (i + 1) * ch)
                np.copyto(flat_pin[a:b], flat_src[a:b])
                return i
            # copies complete in order of submission windows; issue H2D as each lands
            futs = [pool.submit(cp, i) for i in range(nch)]
            with torch.cuda.stream(st):
                for f in futs:
                    i = f.result()
                    a, b = i * ch, min(nbytes, (i + 1) * ch)
                    flat_dev[a:b].copy_(torch.from_numpy(flat_pin[a:b]), non_blocking=True)
            st.synchronize()
        print(f"staged {nth} threads {chunk_mb:2d} MB chunks {bw(staged):6.1f} GB/s")
        pool.shutdown()
print("cores", os.cpu_count())
