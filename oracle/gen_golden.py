"""Generate tests/golden/*.npz by running the UNMODIFIED reference here.

TEST INFRASTRUCTURE. Run in the build container only (the reference is
not present on the GPU box):

    python oracle/gen_golden.py            # writes tests/golden/

It imports `kronstap` from /root/reference/pkg/src via sys.path (nothing
is copied), builds seeded cases through the reference's own public API,
and saves inputs + outputs. Large cubes are stored as a SHA-256 of their
bytes plus the seed, and regenerated in tests by
`paper_1604_03622_b200.scenes` (bit-exactness is itself a golden check).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import kronstap  # noqa: F401
    from kronstap import filters, lrkron, multipass, simulate
    from kronstap.layout import cube_to_snapshots
    return kronstap, filters, lrkron, multipass, simulate, cube_to_snapshots


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _pack_basis(prefix, u, d):
    if u is None:
        d[prefix + "_none"] = np.array(True)
        d[prefix] = np.zeros((0, 0), complex)
    else:
        d[prefix + "_none"] = np.array(False)
        d[prefix] = u


def pipeline_case(name, cfg_kw, ra, rb, D, G, targets, store_cube=True,
                  tol=1e-4, max_iter=100, kind="kron", drop_temporal=False,
                  store_scm=False, extra=None):
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    cfg = simulate.SceneConfig(**cfg_kw)
    hist = simulate.gen_clutter(cfg)
    for (b, f, amp) in targets:
        hist = simulate.inject_target(hist, b, f, amp)
    cube = hist.data[0]
    p, q = cfg.p, cfg.q
    scm = lrkron.sample_covariance(c2s(cube), p, q)
    est = lrkron.lr_kron_estimate(scm, ra, rb, tol=tol, max_iter=max_iter)
    filt = filters.build_filter(kind, estimate=est, drop_temporal=drop_temporal)
    dop = filters.make_doppler_grid(D)
    grid = filters.make_spatial_grid(p, G)
    img = filters.detection_image(filt, cube, dop, grid)
    ident = filters.projection_filter("kron", None, None, p, q)
    m0 = filters.detection_image(ident, cube, dop, grid).values.max()
    d = dict(cfg=np.array(repr(cfg_kw)), ra=ra, rb=rb, D=D, G=G, tol=tol,
             max_iter=max_iter, kind=np.array(kind), drop_temporal=drop_temporal,
             targets=np.array(targets, dtype=float).reshape(-1, 3),
             cube_sha=np.array(sha(cube)), spatial=est.spatial,
             iterations=est.iterations, residuals=np.array(est.residuals),
             converged=est.converged, values=img.values, m0=m0,
             scm_fro=np.linalg.norm(scm.matrix), scm_diag=np.diag(scm.matrix).real.copy())
    if q <= 64:
        d["temporal"] = est.temporal
    _pack_basis("ua", filt.spatial_basis, d)
    _pack_basis("ub", filt.temporal_basis, d)
    if store_cube:
        d["cube"] = cube
    if store_scm:
        d["scm"] = scm.matrix
    if extra:
        d.update(extra)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print(name, "iters", est.iterations, "res", est.residuals[-1],
          "ka", None if filt.spatial_basis is None else filt.spatial_basis.shape[1],
          "kb", None if filt.temporal_basis is None else filt.temporal_basis.shape[1])


def estimator_cases():
    """Direct lr_kron_estimate cases on explicit covariances (edge cases of
    tests/test_lrkron.py:79-228)."""
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    rng = np.random.default_rng(2024)
    cases = {}

    def cg(shape):
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)

    def psd(n, r=None):
        g = cg((n, n if r is None else r))
        m = g @ g.conj().T
        return (m + m.conj().T) / 2

    def run(key, s, p, q, ra, rb, tol=1e-4, max_iter=100):
        sc = lrkron.SampleCovariance(np.asarray(s, complex), 1, p, q)
        try:
            est = lrkron.lr_kron_estimate(sc, ra, rb, tol=tol, max_iter=max_iter)
            cases[key] = dict(s=s, p=p, q=q, ra=ra, rb=rb, tol=tol, max_iter=max_iter,
                              error="", spatial=est.spatial, temporal=est.temporal,
                              iterations=est.iterations, residuals=np.array(est.residuals),
                              converged=est.converged)
        except ks.KronStapError as exc:
            cases[key] = dict(s=s, p=p, q=q, ra=ra, rb=rb, tol=tol, max_iter=max_iter,
                              error=type(exc).__name__)

    for t in range(6):
        p = int(rng.integers(2, 5)); q = int(rng.integers(2, 9))
        ra = int(rng.integers(1, p + 1)); rb = int(rng.integers(1, q + 1))
        a, b = psd(p, ra), psd(q, rb)
        run(f"kron{t}", np.kron(a, b), p, q, ra, rb, tol=1e-6)
    for t in range(4):
        p, q = 3, 10
        snaps = cg((25, p * q))
        s = lrkron.sample_covariance(snaps, p, q).matrix
        run(f"noisy{t}", s, p, q, 1 + t % 3, 3, tol=1e-12, max_iter=60)
    snaps = cg((8, 6))
    run("fixed17", lrkron.sample_covariance(snaps, 2, 3).matrix, 2, 3, 1, 2, tol=-1.0, max_iter=17)
    run("white", 0.7 * np.eye(15, dtype=complex), 3, 5, 3, 5, tol=1e-6)
    run("zero", np.zeros((6, 6), complex), 2, 3, 1, 2)
    bm = np.array([[1.0, -1.0], [-1.0, 1.0]], complex)
    run("degenerate", np.kron(np.eye(2, dtype=complex), bm), 2, 2, 1, 1)
    s = psd(6)
    skew = s.copy(); skew[0, 1] += 1.0
    run("skew", skew, 2, 3, 1, 1)
    neg = np.eye(6, dtype=complex); neg[5, 5] = -1
    run("negdiag", neg, 2, 3, 1, 1)
    run("maxiter1", lrkron.sample_covariance(cg((20, 24)), 3, 8).matrix, 3, 8, 1, 3, tol=1e-15, max_iter=1)
    for t in range(3):
        snaps = cg((10, 6))
        run(f"svdfix{t}", lrkron.sample_covariance(snaps, 2, 3).matrix, 2, 3, 2, 3, tol=-1.0, max_iter=400)
    flat = {}
    for key, c in cases.items():
        for k, v in c.items():
            flat[f"{key}__{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, "estimator_cases.npz"), keys=np.array(sorted(cases)), **flat)
    print("estimator cases", len(cases))


def eig_cases():
    """hermitian_eig / eig_truncate / subspace_basis known answers."""
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    from kronstap import linalg
    rng = np.random.default_rng(77)
    out = {}
    mats = []
    for n in (1, 2, 3, 5, 8, 12, 24, 40):
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        mats.append((g + g.conj().T) / 2)
    mats.append(np.diag([3.0, 1.0, 1.0, 0.5]).astype(complex))       # tie
    mats.append(np.diag([1.0, 1e-12, 0.0]).astype(complex))          # rank tol
    mats.append(np.zeros((4, 4), complex))
    for i, m in enumerate(mats):
        lam, vec = linalg.hermitian_eig(m)
        out[f"m{i}"] = m
        out[f"lam{i}"] = lam
        out[f"vec{i}"] = vec
        n = m.shape[0]
        for r in sorted({1, max(1, n // 2), n}):
            out[f"trunc{i}_{r}"] = linalg.eig_truncate(m, r)
            b = filters.subspace_basis(m, r)
            out[f"basis{i}_{r}"] = np.zeros((0, 0), complex) if b is None else b
    out["count"] = np.array(len(mats))
    np.savez_compressed(os.path.join(OUT, "eig_cases.npz"), **out)


def detect_cases():
    """detection_image over the filter-kind / basis / grid argument space."""
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    rng = np.random.default_rng(99)
    out = {}

    def orth(n, r):
        g = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
        return np.linalg.qr(g)[0]

    specs = []
    n, p, q = 9, 3, 12
    cube = (rng.standard_normal((n, p, q)) + 1j * rng.standard_normal((n, p, q))) / np.sqrt(2)
    ua, ub = orth(p, 1), orth(q, 3)
    uniform = filters.make_doppler_grid(20)
    nonuni = np.sort(rng.random(7))
    grid = filters.make_spatial_grid(p, 16)
    rgrid = rng.standard_normal((5, p)) + 1j * rng.standard_normal((5, p))
    for kind in ("kron", "classical"):
        for (a, b) in ((ua, ub), (None, ub), (ua, None), (None, None)):
            for so in (False, True):
                specs.append((kind, a, b, so, uniform, grid))
    specs.append(("kron", ua, ub, False, nonuni, grid))
    specs.append(("kron", ua, ub, False, filters.make_doppler_grid(5), rgrid))
    specs.append(("kron", ua, ub, False, filters.make_doppler_grid(q), grid))
    specs.append(("classical", orth(p, 2), orth(q, 4), False, nonuni, rgrid))
    specs.append(("kron", np.eye(p, dtype=complex), np.eye(q, dtype=complex), False, uniform, grid))
    for i, (kind, a, b, so, dop, g) in enumerate(specs):
        filt = filters.projection_filter(kind, a, b, p, q, spatial_only=so)
        img = filters.detection_image(filt, cube, dop, g)
        out[f"kind{i}"] = np.array(kind)
        _pack_basis(f"ua{i}", a, out)
        _pack_basis(f"ub{i}", b, out)
        out[f"so{i}"] = np.array(so)
        out[f"dop{i}"] = dop
        out[f"grid{i}"] = g
        out[f"values{i}"] = img.values
    out["cube"] = cube
    out["count"] = np.array(len(specs))
    np.savez_compressed(os.path.join(OUT, "detect_cases.npz"), **out)
    print("detect cases", len(specs))


def multipass_cases():
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    out = {}
    specs = [
        ("k2", dict(p=2, q=8, n_bins=40, rank_temporal=2, noise_power=0.02, seed=12), 2, 16, 8, [(5, 0.25, 3.0, 1)], {}),
        ("k2same", dict(p=2, q=8, n_bins=24, rank_temporal=2, noise_power=0.0, seed=12), 2, 16, 16, [],
         dict(shared_calibration=True, unit_gains=True)),
        ("k4", dict(p=3, q=32, n_bins=64, rank_temporal=3, noise_power=0.01, seed=17), 4, 32, 16, [(7, 0.25, 5.0, 2), (40, 0.5, 5.0, 0)], {}),
    ]
    for name, ckw, k, D, G, targets, gkw in specs:
        cfg = simulate.SceneConfig(**ckw)
        hist = simulate.gen_multipass(cfg, k, **gkw)
        for (b, f, amp, kk) in targets:
            hist = simulate.inject_target(hist, b, f, amp, pass_index=kk)
        st = multipass.stack_passes(hist)
        est = multipass.multipass_estimate(st, cfg.rank_temporal)
        filt = filters.build_filter("kron", estimate=est)
        dop = filters.make_doppler_grid(D)
        imgs = multipass.pass_images(filt, st, dop, spatial_count=G)
        out[f"{name}__data"] = hist.data
        out[f"{name}__k"] = k
        out[f"{name}__D"] = D
        out[f"{name}__G"] = G
        out[f"{name}__rb"] = cfg.rank_temporal
        out[f"{name}__spatial"] = est.spatial
        out[f"{name}__iterations"] = est.iterations
        out[f"{name}__residuals"] = np.array(est.residuals)
        out[f"{name}__maps"] = np.stack([im.values for im in imgs])
        out[f"{name}__change01"] = multipass.change_detect(imgs[0], imgs[1]).values
        out[f"{name}__signed01"] = multipass.change_detect(imgs[0], imgs[1], signed=True).values
        print(name, est.iterations)
    out["names"] = np.array([s[0] for s in specs])
    np.savez_compressed(os.path.join(OUT, "multipass_cases.npz"), **out)


def optimal_cases():
    """kind "optimal" (src/filters.py:144-163, 98-100), steering, filter_output
    and SINR (src/filters.py:44-55, 178-198) on seeded scenes: the whitened
    detection map against the scene's true covariance, and the SINR of the
    kron / classical / optimal weights (acceptance criteria 6/7 shape)."""
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    out = {}
    cfg = simulate.SceneConfig(p=3, q=32, n_bins=48, rank_temporal=4, noise_power=1e-2, seed=1000)
    sigma = simulate.scene_model(cfg).total_covariance()
    hist = simulate.inject_target(simulate.gen_clutter(cfg), 9, 0.25, 3.0)
    cube = hist.data[0]
    filt = filters.build_filter("optimal", sigma=sigma, p=3, q=32)
    dop, grid = filters.make_doppler_grid(32), filters.make_spatial_grid(3, 8)
    out["sigma"] = sigma
    out["cube"] = cube
    out["whitened"] = np.stack([filt.apply_matrix(cube[m]) for m in range(cube.shape[0])])
    out["map"] = filters.detection_image(filt, cube, dop, grid).values
    est = lrkron.lr_kron_estimate(lrkron.sample_covariance(c2s(cube[:5]), 3, 32), 1, 4)
    sv = filters.make_steering(0.25, 3, 32, kappa=2.0)
    out["steering"] = sv.vector
    vals, outs = [], []
    for kind in ("kron", "classical"):
        f = filters.build_filter(kind, estimate=est)
        vals.append(filters.sinr(f.apply(sv.vector), sv, 2.0, sigma))
        outs.append(filters.filter_output(f, sv, cube[9].ravel()))
    vals.append(filters.sinr(filt.apply(sv.vector), sv, 2.0, sigma))
    outs.append(filters.filter_output(filt, sv, cube[9].ravel()))
    out["sinr"] = np.array(vals)
    out["filter_output"] = np.array(outs)
    out["est_spatial"] = est.spatial
    out["est_temporal"] = est.temporal
    np.savez_compressed(os.path.join(OUT, "optimal_cases.npz"), **out)


def scene_hashes():
    """SHA-256 of reference-simulated cubes; pins scenes.py bit-exactly."""
    ks, filters, lrkron, multipass, simulate, c2s = _ref()
    rows = []
    specs = [
        (dict(p=3, q=16, n_bins=200, rank_temporal=3, noise_power=0.01, seed=17), 1, {}),
        (dict(p=3, q=256, n_bins=256, rank_temporal=3, seed=17), 1, {}),
        (dict(p=2, q=8, n_bins=40, rank_temporal=2, seed=12, texture="inverse_gamma"), 3,
         dict(change_fraction=0.25)),
        (dict(p=3, q=20, n_bins=30, rank_temporal=2, seed=5, calibration_phase=0.3), 2,
         dict(shared_calibration=True, unit_gains=False, gain_spread=0.2)),
    ]
    for ckw, k, gkw in specs:
        cfg = simulate.SceneConfig(**ckw)
        hist = simulate.gen_clutter(cfg) if k == 1 and not gkw else simulate.gen_multipass(cfg, k, **gkw)
        hist = simulate.inject_target(hist, 3, 0.25, 2.0 - 1.0j, pass_index=k - 1)
        rows.append((repr(ckw), k, repr(gkw), sha(hist.data)))
    np.savez_compressed(os.path.join(OUT, "scene_hashes.npz"),
                        cfg=np.array([r[0] for r in rows]), k=np.array([r[1] for r in rows]),
                        gen=np.array([r[2] for r in rows]), sha=np.array([r[3] for r in rows]))


def main():
    os.makedirs(OUT, exist_ok=True)
    readme = dict(p=3, q=16, n_bins=200, rank_temporal=3, noise_power=0.01, seed=17)
    pipeline_case("readme_q16", readme, 1, 3, 64, 16, [(11, 0.25, 10.0)], store_scm=True)
    small = dict(p=3, q=64, n_bins=96, rank_temporal=3, noise_power=0.01, seed=17)
    movers = [(11, 0.25, 10.0), (40, 0.5, 10.0), (70, 0.125, 10.0), (90, 0.75, 10.0)]
    for ra in (1, 2, 3):
        for rb in (1, 2, 3):
            pipeline_case(f"sweep_q64_ra{ra}_rb{rb}", small, ra, rb, 64, 16, movers,
                          store_cube=(ra == 1 and rb == 1))
    pipeline_case("classical_q64", small, 1, 3, 48, 8, movers, store_cube=False, kind="classical")
    pipeline_case("droptemporal_q64", small, 1, 3, 80, 16, movers, store_cube=False, drop_temporal=True)
    cfg1 = dict(p=3, q=256, n_bins=256, rank_temporal=3, noise_power=0.01, seed=17)
    m8 = [(int(b), float(d) / 256, 10.0) for b, d in
          zip(np.random.default_rng(1017).integers(0, 256, 8), np.random.default_rng(2017).integers(0, 256, 8))]
    pipeline_case("cfg1_q256", cfg1, 1, 3, 256, 16, m8, store_cube=False)
    estimator_cases()
    eig_cases()
    detect_cases()
    multipass_cases()
    optimal_cases()
    scene_hashes()


if __name__ == "__main__":
    main()
