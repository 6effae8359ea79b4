"""GPU parity of the "optimal" (covariance-whitening) filter kind and the SINR
helpers (src/filters.py:27-55, 98-100, 144-198) against
the reference's outputs (tests/golden/optimal_cases.npz, written by the
unmodified reference) and the oracle; mirrors the reference's own tests
(tests/test_filters.py TestSinr / TestBuildFilter / TestFilterOutput,
tests/test_acceptance.py criterion 6)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "optimal_cases.npz")


def _cg(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def _psd(rng, n):
    a = _cg(rng, (n, n))
    return a @ a.conj().T


def test_optimal_matches_reference_golden():
    g = np.load(GOLD)
    sigma, cube = g["sigma"], g["cube"]
    filt = kst.build_filter("optimal", sigma=sigma, p=3, q=32)
    wh = filt.apply_cube(cube)
    scale = np.abs(g["whitened"]).max()
    assert np.abs(wh - g["whitened"]).max() <= 1e-10 * scale
    for m in (0, 9, 47):
        assert np.abs(filt.apply_matrix(cube[m]) - g["whitened"][m]).max() <= 1e-10 * scale
    img = kst.detection_image(filt, cube, kst.make_doppler_grid(32), kst.make_spatial_grid(3, 8))
    assert np.abs(img.values - g["map"]).max() <= 1e-10 * np.abs(g["map"]).max()
    b, d = np.unravel_index(int(np.argmax(img.values)), img.values.shape)
    assert (b, d / 32) == (9, 0.25)
    # SINR / filter_output of the kron, classical and optimal weights
    sv = kst.make_steering(0.25, 3, 32, kappa=2.0)
    assert np.abs(sv.vector - g["steering"]).max() <= 1e-15
    est = kst.lr_kron_estimate(kst.sample_covariance(kst.cube_to_snapshots(cube[:5]), 3, 32), 1, 4)
    filts = [kst.build_filter("kron", estimate=est), kst.build_filter("classical", estimate=est), filt]
    for f, want, out in zip(filts, g["sinr"], g["filter_output"]):
        got = kst.sinr(f.apply(sv.vector), sv, 2.0, sigma)
        assert abs(got - want) <= 1e-8 * want
        y = kst.filter_output(f, sv, cube[9].ravel())
        assert abs(y - out) <= 1e-8 * max(abs(out), 1.0)


def test_optimal_whitens_against_the_covariance():
    rng = np.random.default_rng(25)
    p, q = 2, 4
    cov = _psd(rng, p * q) + 0.2 * np.eye(p * q)
    filt = kst.build_filter("optimal", sigma=cov, p=p, q=q)
    x = _cg(rng, p * q)
    assert np.allclose(filt.apply(x), np.linalg.solve(cov, x), atol=1e-10)
    # device tensors in -> device tensors out
    xd = torch.from_numpy(x).cuda()
    yd = filt.apply(xd)
    assert yd.is_cuda and np.allclose(yd.cpu().numpy(), np.linalg.solve(cov, x), atol=1e-10)


def test_optimal_reads_only_the_lower_triangle():
    """cho_factor(lower=True) ignores sigma's strict upper triangle."""
    rng = np.random.default_rng(3)
    d = 12
    cov = _psd(rng, d) + np.eye(d)
    junk = cov.copy()
    junk[np.triu_indices(d, 1)] = 7.0 + 3.0j
    x = _cg(rng, (5, 3, 4))
    a = kst.build_filter("optimal", sigma=cov, p=3, q=4).apply_cube(x)
    b = kst.build_filter("optimal", sigma=junk, p=3, q=4).apply_cube(x)
    assert np.array_equal(a, b)
    assert np.abs(a - orc.optimal_whiten(cov, x)).max() <= 1e-12 * np.abs(a).max()


def test_optimal_errors():
    with pytest.raises(kst.DataError):
        kst.build_filter("optimal", sigma=np.diag([1.0, -1.0]), p=1, q=2)
    bad = np.eye(4, dtype=complex)
    bad[3, 0] = np.nan
    with pytest.raises(kst.DataError):
        kst.build_filter("optimal", sigma=bad, p=2, q=2)
    filt = kst.build_filter("optimal", sigma=np.eye(4), p=2, q=2)
    x = np.ones((3, 2, 2), complex)
    x[1, 0, 1] = np.inf
    with pytest.raises(kst.DataError):
        filt.apply_cube(x)
    with pytest.raises(kst.DimensionError):
        filt.apply_matrix(np.zeros((2, 3), complex))
    with pytest.raises(kst.DimensionError):
        kst.projection_filter("optimal", None, None, 2, 2)


def test_optimal_at_cfg1_size():
    """configs[0] shape (p=3, q=256: a 768 x 768 sigma), 64 bins: whitened map
    against the oracle (scipy cho_solve)."""
    cfg = kst.SceneConfig(p=3, q=256, n_bins=64, rank_temporal=3, noise_power=1e-2, seed=17)
    sigma = kst.total_covariance(cfg)
    cube = kst.inject_target(kst.gen_clutter(cfg), 20, 0.25, 2.0).data[0]
    dop, grid = kst.make_doppler_grid(256), kst.make_spatial_grid(3, 16)
    filt = kst.build_filter("optimal", sigma=sigma, p=3, q=256)
    got = kst.detection_image(filt, cube, dop, grid).values
    want = orc.detect("kron", None, None, orc.optimal_whiten(sigma, cube), dop, grid)
    assert np.abs(got - want).max() <= 1e-9 * np.abs(want).max()
    b, d = np.unravel_index(int(np.argmax(got)), got.shape)
    assert (b, d / 256) == (20, 0.25)


class TestSinr:
    def test_white_noise_matched_filter(self):
        sv = kst.make_steering(0.2, 2, 5)
        value = kst.sinr(sv.vector, sv, 1.5, 0.3 * np.eye(10))
        assert abs(value - (1.5 ** 2) / 0.3) < 1e-10

    def test_whitened_steering_maximizes_sinr(self):
        rng = np.random.default_rng(23)
        n = 8
        cov = _psd(rng, n) + 0.1 * np.eye(n)
        d = _cg(rng, n)
        d /= np.linalg.norm(d)
        filt = kst.build_filter("optimal", sigma=cov, p=2, q=4)
        best = kst.sinr(filt.apply(d), d, 1.0, cov)
        for _ in range(200):
            w = _cg(rng, n)
            assert best >= kst.sinr(w, d, 1.0, cov) * (1.0 - 1e-12)

    def test_scale_invariance_is_exact(self):
        rng = np.random.default_rng(24)
        cov = _psd(rng, 6) + 0.5 * np.eye(6)
        d, w = _cg(rng, 6), _cg(rng, 6)
        assert kst.sinr(2.0 * w, d, 0.7, cov) == kst.sinr(w, d, 0.7, cov)

    def test_degenerate_denominator_is_rejected(self):
        with pytest.raises(kst.DataError):
            kst.sinr(np.zeros(4), np.ones(4) / 2.0, 1.0, np.eye(4))


class TestFilterOutput:
    def test_identity_filter_reduces_to_matched_filter(self):
        rng = np.random.default_rng(20)
        sv = kst.make_steering(0.3, 3, 7)
        x = _cg(rng, 21)
        filt = kst.projection_filter("kron", None, None, 3, 7)
        assert abs(kst.filter_output(filt, sv, x) - complex(np.vdot(sv.vector, x))) < 1e-14

    def test_clutter_snapshot_is_annihilated(self):
        rng = np.random.default_rng(21)
        u_a = np.linalg.qr(_cg(rng, (3, 1)))[0]
        u_b = np.linalg.qr(_cg(rng, (9, 4)))[0]
        filt = kst.projection_filter("kron", u_a, u_b, 3, 9)
        sv = kst.make_steering(0.4, 3, 9)
        for _ in range(10):
            x = np.kron(u_a @ _cg(rng, 1), u_b @ _cg(rng, 4))
            assert abs(kst.filter_output(filt, sv, x)) <= 1e-10 * np.linalg.norm(x)


def test_criterion_06_small_sample_advantage_over_classical():
    """Acceptance criterion 6 shape (tests/test_acceptance.py:181-203) on 20
    trials: kron beats classical in median SINR from n = 5 training bins, and
    every SINR equals the oracle's (reference algorithm) to 1e-8."""
    p, q, rank, amp = 3, 32, 4, 2.0
    sv = kst.make_steering(0.25, p, q, kappa=2.0)
    ks, cs = [], []
    for t in range(20):
        cfg = kst.SceneConfig(p=p, q=q, n_bins=5, rank_temporal=rank, noise_power=1e-2, seed=1000 + t)
        cov = kst.total_covariance(cfg)
        cube = kst.gen_clutter(cfg).data[0]
        est = kst.lr_kron_estimate(kst.sample_covariance(kst.cube_to_snapshots(cube), p, q), 1, rank)
        fit = orc.lrkron(orc.scm(cube.reshape(5, -1), p, q), p, q, 1, rank)
        ua, ub = orc.filter_bases(fit)
        for kind, acc in (("kron", ks), ("classical", cs)):
            got = kst.sinr(kst.build_filter(kind, estimate=est).apply(sv.vector), sv, amp, cov)
            w = orc.apply_filter(kind, ua, ub, sv.vector.reshape(p, q)).ravel()
            want = orc.sinr(w, sv.vector, amp, cov)
            assert abs(got - want) <= 1e-8 * want
            acc.append(got)
    assert np.median(ks) > np.median(cs)
