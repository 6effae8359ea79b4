"""FP32 vs FP64 detection (K5) on the GPU: map error against the FP64 path
(itself ~1e-12 of the reference) under the SURVEY.md §8c comparator, over a
spread of shapes / kinds / grids, plus CUDA-event timing of detection_image."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_03622_b200 as kst  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402


def case(p, q, n, D, ra, rb, kind="kron", grid="dft", G=16, seed=17, spatial_only=False, reps=5):
    cube = torch.from_numpy(scenes.bench_scene(p, q, n, seed=seed, movers=8).data[0]).cuda()
    scm = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    est = kst.lr_kron_estimate(scm, ra, rb)
    filt = kst.build_filter(kind, estimate=est, drop_temporal=spatial_only)
    dop = kst.make_doppler_grid(D)
    if grid == "dft":
        gr = kst.make_spatial_grid(p, G)
    else:
        rng = np.random.default_rng(5)
        gr = (rng.standard_normal((G, p)) + 1j * rng.standard_normal((G, p))) / np.sqrt(2 * p)
    ident = kst.projection_filter("kron", None, None, p, q)
    out = {}
    for prec in ("f64", "f32"):
        kst.set_detect_precision(prec)
        v = kst.detection_image(filt, cube, dop, gr).values
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for _ in range(reps):
            kst.detection_image(filt, cube, dop, gr)
        en.record()
        torch.cuda.synchronize()
        out[prec] = (v.cpu().numpy(), st.elapsed_time(en) / reps)
        if prec == "f64":
            m0 = float(kst.detection_image(ident, cube, dop, gr).values.max())
    ref, got = out["f64"][0], out["f32"][0]
    err = np.abs(got - ref)
    tol = 1e-4 * np.abs(ref) + 1e-5 * m0
    print(f"p={p} q={q} n={n} D={D} r=({ra},{rb}) {kind}{'/so' if spatial_only else ''} grid={grid}:"
          f" max|err|/M0={err.max() / m0:.2e} budget={np.max(err / tol):.3f}"
          f" f64 {out['f64'][1]:.3f} ms  f32 {out['f32'][1]:.3f} ms", flush=True)
    return np.max(err / tol)


if __name__ == "__main__":
    worst = 0.0
    worst = max(worst, case(3, 2001, 2001, 2001, 1, 3))
    worst = max(worst, case(3, 256, 256, 256, 1, 3))
    worst = max(worst, case(3, 256, 256, 256, 2, 2))
    worst = max(worst, case(3, 256, 256, 64, 1, 1))
    worst = max(worst, case(3, 200, 256, 2001, 1, 3))
    worst = max(worst, case(3, 256, 128, 256, 1, 3, kind="classical"))
    worst = max(worst, case(3, 256, 128, 256, 1, 3, spatial_only=True))
    worst = max(worst, case(3, 256, 128, 256, 1, 3, grid="rand", G=7))
    worst = max(worst, case(2, 500, 300, 1000, 1, 2))
    worst = max(worst, case(4, 120, 100, 2000, 1, 3))
    print("worst budget", worst)
