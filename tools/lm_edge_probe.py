"""Probe: batched L-mode vs the serial per-window path vs the oracle for n_w r < r_b."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes, windowed  # noqa: E402

p, q, nb, D, G = 3, 32, 24, 32, 16
dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
cube = scenes.bench_scene(p, q, nb, seed=9, movers=1).data[0]
for nw, ra, rb in ((1, 1, 2), (2, 1, 3), (1, 1, 3)):
    got = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid).values
    os.environ["KST_LMODE"] = "serial"
    ser = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid).values
    ser2, ests = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid, return_estimates=True)
    del os.environ["KST_LMODE"]
    ref, fits = orc.windowed(cube, nw, ra, rb, D, G)
    sc = np.abs(ref).max()
    print(f"n_w={nw} r=({ra},{rb}): batched-oracle {np.abs(got-ref).max()/sc:.2e} "
          f"serial-oracle {np.abs(ser-ref).max()/sc:.2e} steploop-oracle {np.abs(ser2.values-ref).max()/sc:.2e}")
    e = ests[0][1]
    tv = e.temporal.cpu().numpy() if hasattr(e.temporal, "cpu") else e.temporal
    w = np.linalg.eigvalsh(tv)[::-1][:4]
    print("  step-loop temporal eig", w, " oracle fit0 temporal eig", np.linalg.eigvalsh(fits[0].temporal)[::-1][:4])
