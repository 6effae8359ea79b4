"""GPU parity: the CUDA path (through the package API / C ABI) against the
reference's own outputs (tests/golden, from the unmodified reference) and
the oracle, on the same inputs.

Tolerances (FP64 estimation; detection in FP64 or the default FP32 transform,
the map tests run at both precisions -- conftest.precision):
  * iterations / converged / kept ranks: identical;
  * residuals: 1e-9 relative; spatial factor: 1e-9 relative (Frobenius);
  * subspace projectors U U^H: 1e-8 max-abs;
  * maps: SURVEY.md §8c rule |v - v_ref| <= 1e-4 |v_ref| + 1e-5 M0 (M0 = max of
    the identity-filter map), and on well-conditioned rank points the much
    tighter conftest.tight_tolerance (FP64: 1e-9 |v_ref| + 1e-10 M0; FP32:
    1e-5 |v_ref| + 1e-6 M0).
"""

import numpy as np
import pytest

from conftest import PIPELINE_CASES, basis_of, golden, map_tolerance, scene_cube, tight_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402


MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def crt_beta(nmod, n):
    """gram_crt.cu crt_beta: largest beta with 2n 2^(2 beta) <= P/4 (capped at 48)."""
    log2p = sum(np.log2(MODULI[:nmod]))
    return min(int(np.floor((log2p - 3 - np.log2(n) - 1e-6) / 2)), 48)


def _proj(u):
    u = np.asarray(u)
    return u @ u.conj().T


def _well_conditioned(name):
    return "ra1" in name or name in ("readme_q16", "classical_q64", "droptemporal_q64", "cfg1_q256")


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_step_api_matches_reference(name, precision):
    d = golden(name)
    cube = scene_cube(d)
    n, p, q = cube.shape
    scm = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    if "scm" in d.files:
        s = scm.matrix
        assert np.array_equal(s, s.conj().T)
        # FP64 DMMA engine: rounding only; int8-slice engine: slice truncation
        # bound ~(slices+1) 2^(-7 slices) (gram_ozaki.cu); CRT engine: rounding
        # x to beta bits, 64 2^-beta (gram_crt.cu)
        mode, slices = kst.lrkron.get_gram_engine()
        if mode == "dmma":
            tol = 1e-13
        elif mode == "int8":
            tol = 64 * (slices + 1) * 2.0 ** (-7 * slices)
        else:
            tol = 64 * 2.0 ** (-crt_beta(slices, n))
        assert np.linalg.norm(s - d["scm"]) <= tol * np.linalg.norm(d["scm"])
    est = kst.lr_kron_estimate(scm, int(d["ra"]), int(d["rb"]), tol=float(d["tol"]),
                               max_iter=int(d["max_iter"]))
    assert est.iterations == int(d["iterations"])
    assert est.converged == bool(d["converged"])
    np.testing.assert_allclose(est.residuals, d["residuals"], rtol=1e-9)
    sp = d["spatial"]
    assert np.linalg.norm(est.spatial - sp) <= 1e-9 * np.linalg.norm(sp)
    if "temporal" in d.files:
        t = d["temporal"]
        assert np.linalg.norm(est.temporal - t) <= 1e-9 * np.linalg.norm(t)
    filt = kst.build_filter(str(d["kind"]), estimate=est, drop_temporal=bool(d["drop_temporal"]))
    for got, key in ((filt.spatial_basis, "ua"), (filt.temporal_basis, "ub")):
        want = basis_of(d, key)
        assert (got is None) == (want is None), key
        if got is not None:
            assert got.shape == want.shape, key
            assert np.abs(_proj(got) - _proj(want)).max() < 1e-8, key
    img = kst.detection_image(filt, cube, kst.make_doppler_grid(int(d["D"])),
                              kst.make_spatial_grid(p, int(d["G"])))
    ref, m0 = d["values"], float(d["m0"])
    err = np.abs(img.values - ref)
    assert img.values.dtype == np.float64 and img.values.shape == ref.shape
    assert np.all(err <= map_tolerance(ref, m0)), err.max()
    if _well_conditioned(name):
        assert np.all(err <= tight_tolerance(ref, m0, precision)), err.max() / m0


@pytest.mark.parametrize("name", ["readme_q16", "sweep_q64_ra1_rb3", "cfg1_q256"])
def test_fused_pipeline_matches_reference(name, precision):
    d = golden(name)
    cube = scene_cube(d)
    n, p, q = cube.shape
    vals, info = kst.process_frame(cube, int(d["ra"]), int(d["rb"]),
                                   dopplers=kst.make_doppler_grid(int(d["D"])),
                                   spatial_grid=kst.make_spatial_grid(p, int(d["G"])))
    assert info["iterations"] == int(d["iterations"])
    ref, m0 = d["values"], float(d["m0"])
    assert np.all(np.abs(vals - ref) <= tight_tolerance(ref, m0, precision))


def test_estimator_edge_cases_match_reference():
    g = golden("estimator_cases")
    for key in g["keys"]:
        key = str(key)
        c = {k.split("__", 1)[1]: g[k] for k in g.files if k.startswith(key + "__")}
        p, q = int(c["p"]), int(c["q"])
        scm = kst.SampleCovariance(np.array(c["s"]), 1, p, q)
        args = (int(c["ra"]), int(c["rb"]))
        kw = dict(tol=float(c["tol"]), max_iter=int(c["max_iter"]))
        if str(c["error"]):
            with pytest.raises(getattr(kst, str(c["error"]))):
                kst.lr_kron_estimate(scm, *args, **kw)
            continue
        est = kst.lr_kron_estimate(scm, *args, **kw)
        assert est.iterations == int(c["iterations"]), key
        assert est.converged == bool(c["converged"]), key
        # the expanded-norm residual has an absolute rounding floor ~sqrt(eps)
        # (src/lrkron.py:129-133): exact-fit cases agree only to that floor
        np.testing.assert_allclose(est.residuals, c["residuals"], rtol=1e-7, atol=1e-7, err_msg=key)
        for got, want in ((est.spatial, c["spatial"]), (est.temporal, c["temporal"])):
            scale = max(np.linalg.norm(want), 1e-300)
            assert np.linalg.norm(got - want) <= 1e-8 * scale, key


def test_eig_conventions_match_reference():
    g = golden("eig_cases")
    for i in range(int(g["count"])):
        m = g[f"m{i}"]
        n = m.shape[0]
        lam, vec = kst.hermitian_eig(m)
        np.testing.assert_allclose(lam, g[f"lam{i}"], rtol=1e-11, atol=1e-12)
        if n < 2 or np.min(np.abs(np.diff(g[f"lam{i}"]))) > 1e-6:
            np.testing.assert_allclose(vec, g[f"vec{i}"], atol=1e-9)
        for r in sorted({1, max(1, n // 2), n}):
            np.testing.assert_allclose(kst.eig_truncate(m, r), g[f"trunc{i}_{r}"], atol=1e-10)
            b = kst.subspace_basis(m, r)
            want = g[f"basis{i}_{r}"]
            if b is None:
                assert want.size == 0
            else:
                assert b.shape == want.shape
                np.testing.assert_allclose(_proj(b), _proj(want), atol=1e-9)


def test_detection_argument_space_matches_reference(precision):
    g = golden("detect_cases")
    cube = g["cube"]
    n, p, q = cube.shape
    for i in range(int(g["count"])):
        filt = kst.projection_filter(str(g[f"kind{i}"]), basis_of(g, f"ua{i}"), basis_of(g, f"ub{i}"),
                                     p, q, spatial_only=bool(g[f"so{i}"]))
        img = kst.detection_image(filt, cube, g[f"dop{i}"], g[f"grid{i}"])
        want = g[f"values{i}"]
        scale = max(np.abs(want).max(), 1.0)
        assert np.abs(img.values - want).max() <= (1e-11 if precision == "f64" else 1e-6) * scale, i
        # the same filter applied in the time domain (kst_filter)
        fo = filt.apply_cube(cube)
        ref = np.stack([orc.apply_filter(str(g[f"kind{i}"]), basis_of(g, f"ua{i}"),
                                         basis_of(g, f"ub{i}"), cube[m], bool(g[f"so{i}"]))
                        for m in range(n)])
        assert np.abs(fo - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0), i


def test_multipass_matches_reference():
    g = golden("multipass_cases")
    for name in g["names"]:
        name = str(name)
        data = g[f"{name}__data"]
        k, n, p, q = data.shape
        hist = kst.PhaseHistory(p, q, k, data)
        st = kst.stack_passes(hist)
        est = kst.multipass_estimate(st, int(g[f"{name}__rb"]))
        assert est.iterations == int(g[f"{name}__iterations"])
        # identical noiseless passes fit exactly: residuals sit on the sqrt(eps) floor
        np.testing.assert_allclose(est.residuals, g[f"{name}__residuals"], rtol=1e-9, atol=1e-7)
        filt = kst.build_filter("kron", estimate=est)
        imgs = kst.pass_images(filt, st, kst.make_doppler_grid(int(g[f"{name}__D"])),
                               spatial_count=int(g[f"{name}__G"]))
        want = g[f"{name}__maps"]
        # M0 floor: identical-pass scenes give maps of pure rounding noise
        m0 = orc.detect("kron", None, None, st.data, orc.doppler_grid(int(g[f"{name}__D"])),
                        orc.spatial_grid(k * p, 4)).max()
        scale = max(np.abs(want).max(), m0)
        got = np.stack([im.values for im in imgs])
        assert np.abs(got - want).max() <= 1e-8 * scale
        ch = kst.change_detect(imgs[0], imgs[1])
        assert np.abs(ch.values - g[f"{name}__change01"]).max() <= 1e-8 * scale
        sg = kst.change_detect(imgs[0], imgs[1], signed=True)
        assert np.abs(sg.values - g[f"{name}__signed01"]).max() <= 1e-8 * scale


def test_results_are_bitwise_deterministic():
    d = golden("sweep_q64_ra1_rb1")
    cube = scene_cube(d)
    outs = [kst.process_frame(cube, 1, 3)[0] for _ in range(3)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    n, p, q = cube.shape
    s1 = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q).matrix
    s2 = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q).matrix
    assert np.array_equal(s1, s2)


def test_device_tensors_stay_on_device(precision):
    d = golden("readme_q16")
    cube = torch.from_numpy(scene_cube(d)).cuda()
    n, p, q = cube.shape
    scm = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    assert scm.matrix.is_cuda
    est = kst.lr_kron_estimate(scm, 1, 3)
    assert est.spatial.is_cuda and est.temporal.is_cuda
    filt = kst.build_filter("kron", estimate=est)
    img = kst.detection_image(filt, cube, kst.make_doppler_grid(64), kst.make_spatial_grid(p))
    assert img.values.is_cuda
    ref, m0 = d["values"], float(d["m0"])
    assert np.all(np.abs(img.values.cpu().numpy() - ref) <= tight_tolerance(ref, m0, precision))


@pytest.mark.parametrize("slices", [5, 6, 7, 8])
def test_int8_gram_engine_error_bound(slices):
    """The int8 tensor-core Gram against the FP64 DMMA Gram on a cfg-1 scene:
    exactly Hermitian, real diagonal, relative error within the slice bound."""
    from paper_1604_03622_b200 import lrkron, scenes
    cube = scenes.bench_scene(3, 256, 256, seed=17).data[0]
    snaps = kst.cube_to_snapshots(cube)
    before = lrkron.get_gram_engine()
    try:
        lrkron.set_gram_engine("dmma")
        ref = kst.sample_covariance(snaps, 3, 256).matrix
        lrkron.set_gram_engine("int8", slices)
        s = kst.sample_covariance(snaps, 3, 256).matrix
    finally:
        lrkron.set_gram_engine(*before)
    assert np.array_equal(s, s.conj().T)
    assert not np.any(np.diagonal(s).imag)
    dg = np.sqrt(np.outer(ref.diagonal().real, ref.diagonal().real))
    bound = 64 * (slices + 1) * 2.0 ** (-7 * slices)
    assert (np.abs(s - ref) / dg).max() <= bound
    assert np.linalg.norm(s - ref) <= bound * np.linalg.norm(ref)


@pytest.mark.parametrize("nmod", [8, 9, 10, 11, 12, 13, 14])
def test_crt_gram_engine_error_bound(nmod):
    """The modular (CRT) int8 Gram against the FP64 DMMA Gram: exactly
    Hermitian, real diagonal, error of rounding x to beta bits, where beta is
    the largest value with 2n 2^(2 beta) <= P/4 (gram_crt.cu)."""
    from paper_1604_03622_b200 import lrkron, scenes
    n = 256
    cube = scenes.bench_scene(3, 256, n, seed=17).data[0]
    snaps = kst.cube_to_snapshots(cube)
    before = lrkron.get_gram_engine()
    try:
        lrkron.set_gram_engine("dmma")
        ref = kst.sample_covariance(snaps, 3, 256).matrix
        lrkron.set_gram_engine("crt", nmod)
        assert lrkron.get_gram_engine() == ("crt", nmod)
        s = kst.sample_covariance(snaps, 3, 256).matrix
    finally:
        lrkron.set_gram_engine(*before)
    beta = crt_beta(nmod, n)
    assert np.array_equal(s, s.conj().T)
    assert not np.any(np.diagonal(s).imag)
    dg = np.sqrt(np.outer(ref.diagonal().real, ref.diagonal().real))
    bound = 64 * 2.0 ** (-beta)
    assert (np.abs(s - ref) / dg).max() <= bound
    assert np.linalg.norm(s - ref) <= bound * np.linalg.norm(ref)


@pytest.mark.parametrize("shape", [(3, 256, 256), (3, 100, 77), (2, 300, 1000), (1, 40, 3),
                                   (2, 1700, 300)])
@pytest.mark.parametrize("nmod", [9, 10, 13])
def test_crt_tcgen05_kernel_matches_library_gemm_path(shape, nmod):
    """The hand-written tcgen05 CRT Gram (mode "crt") against the same CRT
    numerics on cuBLAS int8 GEMMs (mode "crt-cublas"): both recover the same
    exact integer products, so S agrees to the last rounding of the
    reconstruction; ragged shapes exercise the TMA out-of-bounds fill."""
    from paper_1604_03622_b200 import lrkron
    p, q, n = shape
    rng = np.random.default_rng(7 + n)
    snaps = rng.standard_normal((n, p * q)) + 1j * rng.standard_normal((n, p * q))
    snaps[:, 0] *= 1e3  # column scales differ
    before = lrkron.get_gram_engine()
    try:
        lrkron.set_gram_engine("crt-cublas", nmod)
        ref = kst.sample_covariance(snaps, p, q).matrix
        lrkron.set_gram_engine("crt", nmod)
        s = kst.sample_covariance(snaps, p, q).matrix
    finally:
        lrkron.set_gram_engine(*before)
    assert np.array_equal(s, s.conj().T)
    assert not np.any(np.diagonal(s).imag)
    dg = np.sqrt(np.outer(ref.diagonal().real, ref.diagonal().real))
    assert (np.abs(s - ref) / dg).max() <= 1e-14


@pytest.mark.parametrize("shape", [(3, 256, 256), (3, 100, 77), (2, 300, 1000), (3, 672, 2016)])
def test_crt_pair_kernel_bit_identical(shape, monkeypatch):
    """The two-SM cta_group::2 kernel (KST_TC2=1) and the single-CTA kernel
    produce the same exact residue products, so S is bit-identical."""
    from paper_1604_03622_b200 import lrkron
    p, q, n = shape
    rng = np.random.default_rng(11 + n)
    snaps = rng.standard_normal((n, p * q)) + 1j * rng.standard_normal((n, p * q))
    before = lrkron.get_gram_engine()
    try:
        lrkron.set_gram_engine("crt", 10)
        monkeypatch.setenv("KST_TC2", "0")
        ref = kst.sample_covariance(snaps, p, q).matrix
        monkeypatch.setenv("KST_TC2", "1")
        s = kst.sample_covariance(snaps, p, q).matrix
    finally:
        lrkron.set_gram_engine(*before)
    np.testing.assert_array_equal(s, ref)


@pytest.mark.parametrize("engine", [("int8", 6), ("crt", 10), ("crt-cublas", 10)])
def test_int8_gram_propagates_non_finite_inputs(engine):
    from paper_1604_03622_b200 import lrkron
    before = lrkron.get_gram_engine()
    try:
        lrkron.set_gram_engine(*engine)
        x = np.ones((8, 6), complex)
        x[3, 2] = np.nan
        scm = kst.sample_covariance(x, 2, 3)
        with pytest.raises(kst.DataError):
            kst.lr_kron_estimate(scm, 1, 1)
    finally:
        lrkron.set_gram_engine(*before)


def test_frame_stream_overlap_matches_single_frames():
    from paper_1604_03622_b200 import scenes
    from paper_1604_03622_b200.pipeline import FrameStream
    cubes = [scenes.bench_scene(3, 64, 80, seed=200 + i, movers=2).data[0] for i in range(4)]
    pinned = [torch.from_numpy(c).pin_memory() for c in cubes]
    fs = FrameStream(cubes[0].shape, 0, 1, 3)
    got = []
    for c in pinned:
        r = fs.submit(c)
        if r is not None:
            r[1].synchronize()
            got.append(r[0].numpy().copy())
    r = fs.flush()
    r[1].synchronize()
    got.append(r[0].numpy().copy())
    for c, g in zip(cubes, got):
        want, _ = kst.process_frame(c, 1, 3)
        assert np.array_equal(g, want)


@pytest.mark.parametrize("p,G", [(3, 16), (2, 8), (4, 12), (3, 6), (1, 4)])
def test_uniform_spatial_grid_fast_path(p, G, precision):
    """make_spatial_grid(p, G) with G % 4 == 0 takes the radix-4 candidate
    split in the fused kernels; a grid differing from it by 1e-9 (or G % 4 != 0)
    takes the generic candidate loop. Both equal the oracle to 1e-11 of M0
    (FP64 detection) / 1e-6 of M0 (FP32)."""
    from paper_1604_03622_b200 import scenes
    q, nb, D = 48, 30, 48
    cube = scenes.bench_scene(p, q, nb, seed=5, movers=2, rank_temporal=2).data[0]
    dop = kst.make_doppler_grid(D)
    grid = kst.make_spatial_grid(p, G)
    off = grid.copy()
    off[1, -1] += 1e-9  # no longer the uniform grid: generic loop
    s = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    filt = kst.build_filter("kron", estimate=kst.lr_kron_estimate(s, 1, 2))
    ua, ub = filt.spatial_basis, filt.temporal_basis
    m0 = orc.detect("kron", None, None, cube, dop, grid).max()
    for gr in (grid, off):
        got = kst.detection_image(filt, cube, dop, gr).values
        want = orc.detect("kron", ua, ub, cube, dop, gr)
        assert np.abs(got - want).max() <= (1e-11 if precision == "f64" else 1e-6) * m0


def test_frame_stream_multipass_groups():
    """FrameStream with groups = K (pass-stacked cubes, K maps per stack)
    returns exactly the single-stack pipeline's maps."""
    from paper_1604_03622_b200 import scenes
    from paper_1604_03622_b200.pipeline import FrameStream, process_frame_device
    K, p, q, n = 3, 2, 24, 40
    stacks = [np.ascontiguousarray(kst.stack_passes(
        scenes.bench_scene(p, q, n, seed=300 + i, movers=2, n_passes=K)).data) for i in range(3)]
    dop, grid = kst.make_doppler_grid(q), kst.make_stacked_spatial_grid(p, K, 8)
    fs = FrameStream(stacks[0].shape, 0, K, 2, dop, grid, groups=K)
    got = []
    for s_ in stacks:
        r = fs.submit(torch.from_numpy(s_).pin_memory())
        if r is not None:
            r[1].synchronize()
            got.append(r[0].numpy().copy())
    r = fs.flush()
    r[1].synchronize()
    got.append(r[0].numpy().copy())
    for s_, g in zip(stacks, got):
        want, _ = process_frame_device(torch.from_numpy(s_).cuda(), K, 2, dop, grid, groups=K)
        assert g.shape == (K, n, q) and np.array_equal(g, want.cpu().numpy())


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_detection_maps_identical_off_threshold(name, precision):
    """Thresholded detection maps (v >= tau, tau at the 50/90/99/99.9 %
    quantiles of the reference map and at 0.5 M0) equal the reference's
    except at pixels within the §8c tolerance of tau."""
    from conftest import binary_map_mismatch
    d = golden(name)
    cube = scene_cube(d)
    n, p, q = cube.shape
    D, G = int(d["D"]), int(d["G"])
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    scm = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    est = kst.lr_kron_estimate(scm, int(d["ra"]), int(d["rb"]), tol=float(d["tol"]),
                               max_iter=int(d["max_iter"]))
    filt = kst.build_filter(str(d["kind"]), estimate=est, drop_temporal=bool(d["drop_temporal"]))
    vals = kst.detection_image(filt, cube, dop, grid).values
    ref = d["values"]
    m0 = float(d["m0"])
    taus = list(np.quantile(ref, [0.5, 0.9, 0.99, 0.999])) + [0.5 * m0]
    bad, near = binary_map_mismatch(vals, ref, m0, taus)
    assert bad == 0, (bad, near)


@pytest.mark.parametrize("n,rb", [(1, 2), (1, 3), (2, 3)])
def test_rank_deficient_temporal_basis_matches_oracle(n, rb, precision):
    """b of rank n r_a < r_b: the kept temporal rank kb < r_b (src/filters.py:70
    keep rule), and the fused pipeline / step API hand detect a q x kb basis
    (regression: the q x r_b eigenvector block was passed with a kb pitch)."""
    from paper_1604_03622_b200 import scenes
    p, q, D, G = 3, 32, 32, 16
    cube = scenes.bench_scene(p, q, 24, seed=9, movers=1).data[0][:n]
    fit, ua, ub, ref = orc.pipeline(cube, 1, rb, D, G)
    assert ub.shape[1] < rb
    m0 = orc.detect("kron", None, None, cube, orc.doppler_grid(D), orc.spatial_grid(p, G)).max()
    vals, info = kst.process_frame(cube, 1, rb, dopplers=kst.make_doppler_grid(D),
                                   spatial_grid=kst.make_spatial_grid(p, G))
    assert info["kb"] == ub.shape[1] and info["iterations"] == fit.iterations
    assert np.all(np.abs(vals - ref) <= tight_tolerance(ref, m0, precision))
    s = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    filt = kst.build_filter("kron", estimate=kst.lr_kron_estimate(s, 1, rb))
    img = kst.detection_image(filt, cube, kst.make_doppler_grid(D), kst.make_spatial_grid(p, G))
    assert np.all(np.abs(img.values - ref) <= tight_tolerance(ref, m0, precision))


def test_pipeline_optimistic_path_falls_back_exactly():
    """kst_pipeline's host-sync-free form (q > 64) validates its assumptions on
    the device and recomputes on the synchronous path when one fails: a
    rank-deficient b (k_B < r_B), an all-zero frame, a non-finite frame. Each
    outcome equals the step API / the oracle."""
    from paper_1604_03622_b200 import scenes
    p, q, D, G = 3, 96, 96, 16
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    base = scenes.bench_scene(p, q, 40, seed=5, movers=2).data[0]
    m0 = orc.detect("kron", None, None, base, orc.doppler_grid(D), orc.spatial_grid(p, G)).max()
    # common case (no fallback) and k_B < r_B (one bin: b of rank 1)
    for cube, rb in ((base, 3), (base[:1], 3), (base[:2], 3)):
        fit, ua, ub, ref = orc.pipeline(cube, 1, rb, D, G)
        vals, info = kst.process_frame(cube, 1, rb, dopplers=dop, spatial_grid=grid)
        assert info["iterations"] == fit.iterations and info["kb"] == ub.shape[1]
        assert np.all(np.abs(vals - ref) <= 1e-5 * np.abs(ref) + 1e-6 * m0)
    # all-zero frame: zero estimate, identity filter (src/lrkron.py:152-160)
    z = np.zeros_like(base)
    vals, info = kst.process_frame(z, 1, 3, dopplers=dop, spatial_grid=grid)
    assert info["iterations"] == 0 and info["kb"] == 0 and not np.any(vals)
    # non-finite frame: DataError as the reference's covariance validation
    bad = base.copy()
    bad[3, 1, 7] = np.nan
    with pytest.raises(kst.DataError):
        kst.process_frame(bad, 1, 3, dopplers=dop, spatial_grid=grid)
    # and the context is usable afterwards
    vals, info = kst.process_frame(base, 1, 3, dopplers=dop, spatial_grid=grid)
    assert info["iterations"] >= 1
