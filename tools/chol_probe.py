"""Hand-written Cholesky factor / solve (kst_chol, kst_chol_solve) against
torch.linalg (cuSOLVER) on random HPD matrices: relative error and time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1604_03622_b200 import _native as nat  # noqa: E402

for d, nrhs in ((5, 3), (33, 7), (200, 64), (768, 64), (1536, 256), (6003, 2001)):
    g = torch.Generator(device="cuda").manual_seed(d)
    x = torch.randn(d, d + 16, dtype=torch.complex128, device="cuda", generator=g)
    s = x @ x.conj().T / (d + 16) + 0.1 * torch.eye(d, dtype=torch.complex128, device="cuda")
    b = torch.randn(nrhs, d, dtype=torch.complex128, device="cuda", generator=g)
    L = torch.empty_like(s)
    c = nat.ctx(s.device)
    st = nat.stream_of(s.device)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nat.check(nat.lib().kst_chol(c, nat.ptr(s), d, nat.ptr(L), st), c)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X = torch.empty_like(b)
        nat.check(nat.lib().kst_chol_solve(c, nat.ptr(L), d, nat.ptr(b), nrhs, nat.ptr(X), st), c)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    Lcol = L.reshape(d, d).T  # stored column-major
    Lref = torch.linalg.cholesky(s)
    el = ((Lcol - Lref).abs().max() / Lref.abs().max()).item()
    xr = torch.cholesky_solve(b.T, Lref).T
    ex = ((X - xr).abs().max() / xr.abs().max()).item()
    print(f"d={d:5d} nrhs={nrhs:5d} factor {1e3*(t1-t0):8.2f} ms err {el:.1e}  solve {1e3*(t2-t1):8.2f} ms err {ex:.1e}")
