"""Full-size golden fixtures from the UNMODIFIED reference (BASELINE configs
[1], [3] at Gotcha scale, [4], and a high-dynamic-range scene).

TEST INFRASTRUCTURE. Run in the build container only (the reference is not
present on the GPU box); needs ~30 GB RAM and a few minutes of 8 cores:

    python oracle/gen_golden_full.py [gotcha] [multipass] [lmode] [hdr]

Cubes are NOT stored: each case records its scene recipe and the SHA-256 of
the cube the reference simulator produced, and the tests regenerate the cube
with `paper_1604_03622_b200.scenes.bench_scene` (hash-checked, so the GPU
sees exactly the bytes the reference processed). The recipe is the one of
`scenes.bench_scene`: SceneConfig defaults + `movers` targets at bins/Dopplers
drawn from default_rng(seed + 1000) -- restated here with the reference's own
simulate.inject_target. Full detection maps (32 MB each) are summarised:
every row's max / sum / sum of squares, the reference map's quantiles at
the thresholds the tests use, plus full rows at a seeded bin sample and at
every mover bin.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
sys.path.insert(0, REF)

import kronstap as ks  # noqa: E402
from kronstap import filters, lrkron, multipass, simulate  # noqa: E402
from kronstap.layout import cube_to_snapshots  # noqa: E402
from kronstap.parallel import WorkerPool  # noqa: E402

QUANTS = np.array([0.5, 0.9, 0.99, 0.9999])


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scene(p, q, n_bins, seed, movers, n_passes=1, amplitude=10.0, **cfg_kw):
    """scenes.bench_scene restated on the reference simulator."""
    cfg = simulate.SceneConfig(p=p, q=q, n_bins=n_bins, rank_temporal=3, noise_power=1e-2,
                               seed=seed, **cfg_kw)
    hist = simulate.gen_clutter(cfg) if n_passes == 1 else simulate.gen_multipass(cfg, n_passes)
    rng = np.random.default_rng(seed + 1000)
    targets = []
    for _ in range(movers):
        b = int(rng.integers(0, n_bins))
        d = int(rng.integers(0, q)) / q
        k = int(rng.integers(0, n_passes))
        hist = simulate.inject_target(hist, b, d, amplitude, pass_index=k)
        targets.append((b, d, k))
    return hist, targets


def map_summary(prefix, vals, rows, out):
    out[prefix + "_rowmax"] = vals.max(axis=1)
    out[prefix + "_rowsum"] = vals.sum(axis=1)
    out[prefix + "_rowsq"] = (vals * vals).sum(axis=1)
    out[prefix + "_quant"] = np.quantile(vals, QUANTS)
    out[prefix + "_rows"] = np.asarray(rows, dtype=np.int64)
    out[prefix + "_rowvals"] = vals[rows]
    out[prefix + "_max"] = vals.max()
    out[prefix + "_argmax"] = np.array(np.unravel_index(int(np.argmax(vals)), vals.shape))


def sample_rows(n, k, seed, extra=()):
    rng = np.random.default_rng(seed)
    rows = set(int(x) for x in rng.choice(n, size=k, replace=False))
    rows |= {0, n - 1} | set(int(x) for x in extra)
    return sorted(rows)


def frame_case(name, p, q, n, D, G, ra, rb, seed, movers, pool, **cfg_kw):
    t0 = time.time()
    hist, targets = scene(p, q, n, seed, movers, **cfg_kw)
    cube = hist.data[0]
    scm = lrkron.sample_covariance(cube_to_snapshots(cube), p, q, pool=pool)
    est = lrkron.lr_kron_estimate(scm, ra, rb, pool=pool)
    filt = filters.build_filter("kron", estimate=est)
    dop, grid = filters.make_doppler_grid(D), filters.make_spatial_grid(p, G)
    vals = filters.detection_image(filt, cube, dop, grid, pool=pool).values
    ident = filters.projection_filter("kron", None, None, p, q)
    m0 = filters.detection_image(ident, cube, dop, grid, pool=pool).values.max()
    out = dict(recipe=np.array(repr(dict(p=p, q=q, n_bins=n, seed=seed, movers=movers, **cfg_kw))),
               D=D, G=G, ra=ra, rb=rb, cube_sha=np.array(sha(cube)),
               targets=np.array(targets, dtype=float).reshape(-1, 3),
               spatial=est.spatial, iterations=est.iterations,
               residuals=np.array(est.residuals), converged=est.converged, m0=m0,
               ua=filt.spatial_basis, ub=filt.temporal_basis,
               scm_fro=np.linalg.norm(scm.matrix), scm_diag=np.diag(scm.matrix).real.copy())
    map_summary("map", vals, sample_rows(n, 48, seed, [t[0] for t in targets]), out)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, f"{time.time() - t0:.1f}s iters", est.iterations, "res", est.residuals, flush=True)


def gotcha(pool):
    """configs[1]: the seed-17 Gotcha frame the bench measures."""
    frame_case("full_gotcha_s17", 3, 2001, 2001, 2001, 16, 1, 3, 17, 8, pool)


def hdr(pool):
    """High dynamic range: inverse-gamma texture
    (src/simulate.py:147-153, shape 1.5: heavy-tailed bin powers) and movers
    at |alpha| = 1e4 -- the CRT Gram rounds each column to 32 bits, so the
    per-column scale and the heavy tail are exactly what stresses it."""
    t0 = time.time()
    p, q, n, D, G, ra, rb, seed = 3, 512, 512, 512, 16, 1, 3, 29
    for name, amp, shape in (("hdr_invgamma_q512", 1e4, 1.5), ("hdr_invgamma_q512_a1e6", 1e6, 1.2)):
        hist, targets = scene(p, q, n, seed, 6, amplitude=amp, texture="inverse_gamma",
                              texture_shape=shape)
        cube = hist.data[0]
        scm = lrkron.sample_covariance(cube_to_snapshots(cube), p, q, pool=pool)
        est = lrkron.lr_kron_estimate(scm, ra, rb, pool=pool)
        filt = filters.build_filter("kron", estimate=est)
        dop, grid = filters.make_doppler_grid(D), filters.make_spatial_grid(p, G)
        vals = filters.detection_image(filt, cube, dop, grid, pool=pool).values
        ident = filters.projection_filter("kron", None, None, p, q)
        m0 = filters.detection_image(ident, cube, dop, grid, pool=pool).values.max()
        out = dict(recipe=np.array(repr(dict(p=p, q=q, n_bins=n, seed=seed, movers=6,
                                             amplitude=amp, texture="inverse_gamma",
                                             texture_shape=shape))),
                   D=D, G=G, ra=ra, rb=rb, cube_sha=np.array(sha(cube)),
                   targets=np.array(targets, dtype=float).reshape(-1, 3),
                   spatial=est.spatial, iterations=est.iterations,
                   residuals=np.array(est.residuals), converged=est.converged, m0=m0,
                   ua=filt.spatial_basis, ub=filt.temporal_basis, values=vals,
                   scm_fro=np.linalg.norm(scm.matrix), scm_diag=np.diag(scm.matrix).real.copy(),
                   col_power=np.abs(cube).max(axis=(1, 2)))
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
        print(name, f"{time.time() - t0:.1f}s iters", est.iterations, "res", est.residuals,
              "bin power range", float(out["col_power"].min()), float(out["col_power"].max()),
              flush=True)


def multipass_full(pool):
    """configs[4]: a 4-pass 3-channel 2001 x 2001 stack (seed 17, 8 movers),
    stacked to (n, 12, q); joint fit with ranks (K, 3) on the 24012^2
    covariance; 4 pass maps through the stacked grid and the 3 consecutive
    change maps (src/multipass.py:40-123)."""
    t0 = time.time()
    p, q, n, D, G, K, rb, seed = 3, 2001, 2001, 2001, 16, 4, 3, 17
    hist, targets = scene(p, q, n, seed, 8, n_passes=K)
    st = multipass.stack_passes(hist)
    est = multipass.multipass_estimate(st, rb, pool=pool)
    print("  estimate", f"{time.time() - t0:.1f}s", flush=True)
    filt = filters.build_filter("kron", estimate=est)
    dop = filters.make_doppler_grid(D)
    imgs = multipass.pass_images(filt, st, dop, spatial_count=G, pool=pool)
    ident = filters.projection_filter("kron", None, None, K * p, q)
    m0 = filters.detection_image(ident, st.data, dop, filters.make_spatial_grid(K * p, G),
                                 pool=pool).values.max()
    out = dict(recipe=np.array(repr(dict(p=p, q=q, n_bins=n, seed=seed, movers=8, n_passes=K))),
               D=D, G=G, K=K, rb=rb, cube_sha=np.array(sha(hist.data)),
               targets=np.array(targets, dtype=float).reshape(-1, 3),
               spatial=est.spatial, iterations=est.iterations,
               residuals=np.array(est.residuals), converged=est.converged, m0=m0,
               ua=filt.spatial_basis, ub=filt.temporal_basis)
    rows = sample_rows(n, 32, seed, [t[0] for t in targets])
    for k, im in enumerate(imgs):
        map_summary(f"pass{k}", im.values, rows, out)
    for k in range(K - 1):
        ch = multipass.change_detect(imgs[k], imgs[k + 1])
        chv = ch.values if hasattr(ch, "values") else np.asarray(ch)
        map_summary(f"change{k}", chv, rows, out)
    np.savez_compressed(os.path.join(OUT, "full_multipass_s17.npz"), **out)
    print("full_multipass_s17", f"{time.time() - t0:.1f}s iters", est.iterations, "res",
          est.residuals, flush=True)


def lmode(pool):
    """configs[3] L-mode at Gotcha scale (SURVEY.md §8 L-mode definition):
    training bins [s, s + n_w), s = clamp(m - n_w // 2, 0, n - n_w), n_w = 81,
    one reference estimate + filter per test bin, on the seed-17 Gotcha frame.
    A seeded sample of test bins: both edges (clamped windows), the first and
    last unclamped ones, and interior bins including mover bins."""
    t0 = time.time()
    p, q, n, D, G, ra, rb, seed, n_w = 3, 2001, 2001, 2001, 16, 1, 3, 17, 81
    hist, targets = scene(p, q, n, seed, 8)
    cube = hist.data[0]
    dop, grid = filters.make_doppler_grid(D), filters.make_spatial_grid(p, G)
    h = n_w // 2
    movers = sorted({t[0] for t in targets})
    bins = sorted({0, 1, h - 1, h, n - h - 1, n - h, n - 2, n - 1, 1000} | set(movers[:3]))
    rows, fits = [], []
    for m in bins:
        s = min(max(m - h, 0), n - n_w)
        win = cube[s:s + n_w]
        scm = lrkron.sample_covariance(cube_to_snapshots(win), p, q, pool=pool)
        est = lrkron.lr_kron_estimate(scm, ra, rb, pool=pool)
        filt = filters.build_filter("kron", estimate=est)
        rows.append(filters.detection_image(filt, cube[m:m + 1], dop, grid, pool=pool).values[0])
        fits.append((s, est.iterations, est.converged, est.residuals[-1], len(est.residuals)))
        print(f"  bin {m} window {s} iters {est.iterations} {time.time() - t0:.1f}s", flush=True)
    ident = filters.projection_filter("kron", None, None, p, q)
    m0 = filters.detection_image(ident, cube, dop, grid, pool=pool).values.max()
    np.savez_compressed(
        os.path.join(OUT, "full_lmode_s17_nw81.npz"),
        recipe=np.array(repr(dict(p=p, q=q, n_bins=n, seed=seed, movers=8))),
        D=D, G=G, ra=ra, rb=rb, n_w=n_w, cube_sha=np.array(sha(cube)),
        bins=np.array(bins, dtype=np.int64), values=np.stack(rows),
        window_start=np.array([f[0] for f in fits]), iterations=np.array([f[1] for f in fits]),
        converged=np.array([f[2] for f in fits]), last_residual=np.array([f[3] for f in fits]),
        m0=m0)
    print("full_lmode_s17_nw81", f"{time.time() - t0:.1f}s", flush=True)


def main():
    which = sys.argv[1:] or ["gotcha", "hdr", "lmode", "multipass"]
    with WorkerPool(os.cpu_count() or 1) as pool:
        for w in which:
            {"gotcha": gotcha, "hdr": hdr, "lmode": lmode, "multipass": multipass_full}[w](pool)


if __name__ == "__main__":
    main()
