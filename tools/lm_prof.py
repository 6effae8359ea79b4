"""Phase breakdown of the batched L-mode window kernel (clock64 stamps of an
A/B build: make -C paper_1604_03622_b200/csrc EXTRA=-DKST_LM_PROF
OUT=../_lib/prof/libkst_b200.so OBJDIR=../_lib/prof/obj; run with
KST_LIB_PATH=paper_1604_03622_b200/_lib/prof/libkst_b200.so)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1604_03622_b200 as kst  # noqa: E402
from paper_1604_03622_b200 import _native as nat, scenes, windowed  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_w = int(sys.argv[2]) if len(sys.argv) > 2 else 81
cube = torch.from_numpy(scenes.bench_scene(3, q, q, seed=17, movers=8).data[0]).cuda()
dop, grid = kst.make_doppler_grid(q), kst.make_spatial_grid(3, 16)
for _ in range(2):
    kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid)
torch.cuda.synchronize()
info = windowed.last_window_info()
nwin = info.shape[0]
buf = np.zeros((nwin, 16), dtype=np.int64)
lib = nat.lib()
lib.kst_lm_prof.argtypes = [C.c_void_p, C.c_int]
assert lib.kst_lm_prof(buf.ctypes.data_as(C.c_void_p), nwin) == 0
ph = np.diff(buf[:, :8], axis=1) / 1.965e3  # us at 1965 MHz
names = ["record", "iterations", "ua+Aprev", "H build", "eig(H)", "Q1Q2+gamma", "E"]
print(f"{nwin} windows; info columns: status it conv ka kb rounds r nb")
print("iterations hist", np.bincount(info[:, 1]), "rounds hist", np.bincount(np.maximum(info[:, 5], 0)),
      "nb", np.unique(info[:, 7]))
for k, nm in enumerate(names):
    print(f"{nm:12s} mean {ph[:, k].mean():8.2f} us  max {ph[:, k].max():8.2f} us")
tot = (buf[:, 7] - buf[:, 0]) / 1.965e3
print(f"{'total':12s} mean {tot.mean():8.2f} us  max {tot.max():8.2f} us")
sub = np.diff(buf[:, 8:14], axis=1) / 1.965e3
for k, nm in enumerate(["hmul", "cgs2", "hmul+cgs2", "hmul+gram", "jacobi 8x8"]):
    print(f"  last round {nm:12s} mean {sub[:, k].mean():8.2f} us  max {sub[:, k].max():8.2f} us")
print(f"  last round rest     mean {((buf[:, 5] - buf[:, 13]) / 1.965e3).mean():8.2f} us")
print(f"  start block select   mean {((buf[:, 14] - buf[:, 4]) / 1.965e3).mean():8.2f} us")
