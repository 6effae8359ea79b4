import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes, windowed
from oracle import kron_oracle as orc
p, q, nb, D, G = 3, 32, 24, 32, 16
dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
cube = scenes.bench_scene(p, q, nb, seed=9, movers=1).data[0]
for nw, ra, rb in ((24, 1, 2), (1, 1, 2), (24, 1, 3), (23, 1, 2), (2, 1, 2), (1, 1, 1)):
    got = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid).values
    info = windowed.last_window_info()
    ref, fits = orc.windowed(cube, nw, ra, rb, D, G)
    err = np.abs(got - ref).max(axis=1) / np.abs(ref).max()
    print(nw, ra, rb, "maxrel", err.max(), "rows bad", np.nonzero(err > 1e-8)[0][:10], "info", info[:3].tolist())
os.environ["KST_LMODE"] = "serial"
for nw, ra, rb in ((24, 1, 2), (1, 1, 2), (2, 1, 2), (1, 1, 1)):
    got = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid).values
    ref, fits = orc.windowed(cube, nw, ra, rb, D, G)
    err = np.abs(got - ref).max(axis=1) / np.abs(ref).max()
    print("serial", nw, ra, rb, "maxrel", err.max(), "rows bad", np.nonzero(err > 1e-8)[0][:10])
    _, ests = kst.windowed_detection_image(cube, nw, ra, rb, dop, grid, return_estimates=True)
    e0 = ests[0][1]
    print("   step est iters", e0.iterations, "oracle", fits[0].iterations, fits[0].residuals, e0.residuals)
