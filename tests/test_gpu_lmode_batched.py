"""The batched L-mode path (kst_lmode, csrc/lmode.cu: banded snapshot Gram,
one CTA per window, spectral detection) against the oracle's per-window
loop over the reference functions (SURVEY.md §8 "L-mode definition") and
against the per-window step path it replaces (KST_LMODE=serial).

Comparators: per window identical iterations and convergence; maps within
the §8c rule |v - v_ref| <= 1e-4 |v_ref| + 1e-5 M0 everywhere, and within
1e-9 |v_ref| + 1e-10 M0 at r_a = 1 (well-conditioned: SURVEY.md App. B
flags r_a = 2 on single-pass scenes, and r_a = p gives a zero map)."""

import os

import numpy as np
import pytest

from conftest import map_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes, windowed  # noqa: E402


def _m0(cube, D, G):
    return float(np.max(orc.detect("kron", None, None, cube, orc.doppler_grid(D),
                                   orc.spatial_grid(cube.shape[1], G))))


def _serial(fn):
    old = os.environ.get("KST_LMODE")
    os.environ["KST_LMODE"] = "serial"
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["KST_LMODE"]
        else:
            os.environ["KST_LMODE"] = old


@pytest.mark.parametrize("n_w", [9, 25, 49, 81])
@pytest.mark.parametrize("ra,rb", [(1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (3, 3)])
def test_batched_sweep_matches_oracle(n_w, ra, rb):
    """configs[3]'s window x rank sweep (3x3 .. 9x9 training windows) on a
    q = 64 frame: every window's fit and every map row against the oracle."""
    p, q, nb, D, G = 3, 64, 96, 64, 16
    cube = scenes.bench_scene(p, q, nb, seed=17, movers=4).data[0]
    ref, fits = orc.windowed(cube, n_w, ra, rb, D, G)
    dmap = kst.windowed_detection_image(cube, n_w, ra, rb, kst.make_doppler_grid(D),
                                        kst.make_spatial_grid(p, G))
    info = windowed.last_window_info()
    assert info.shape == (nb - n_w + 1, 8)
    assert np.all(info[:, 0] == 0), info[info[:, 0] != 0]  # no window fell back
    for s in range(nb - n_w + 1):
        assert info[s, 1] == fits[s].iterations and bool(info[s, 2]) == fits[s].converged
    m0 = _m0(cube, D, G)
    err = np.abs(dmap.values - ref)
    assert np.all(err <= map_tolerance(ref, m0)), (err / map_tolerance(ref, m0)).max()
    if ra == 1:
        assert np.all(err <= 1e-9 * np.abs(ref) + 1e-10 * m0), \
            (err / (1e-9 * np.abs(ref) + 1e-10 * m0)).max()


def test_batched_cfg3_frame_matches_oracle_and_serial():
    """configs[3] size (p=3, q=n_bins=D=256, G=16, n_w=81, ranks (1, 3)): the
    whole map against the serial per-window path, a seeded bin sample
    against the oracle."""
    p, q, nb, D, G, n_w = 3, 256, 256, 256, 16, 81
    cube = scenes.bench_scene(p, q, nb, seed=17, movers=8).data[0]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    got = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid).values
    info = windowed.last_window_info()
    assert np.all(info[:, 0] == 0) and np.all(info[:, 4] == 3)
    ser = _serial(lambda: kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid).values)
    m0 = _m0(cube, D, G)
    assert np.all(np.abs(got - ser) <= 1e-9 * np.abs(ser) + 1e-10 * m0)
    bins = [0, 40, 41, 100, 173, 214, 215, 255]
    ref, _ = orc.windowed(cube, n_w, 1, 3, D, G, bins=bins)
    assert np.all(np.abs(got[bins] - ref[bins]) <= 1e-9 * np.abs(ref[bins]) + 1e-10 * m0)


@pytest.mark.parametrize("kind,drop", [("kron", False), ("classical", False), ("kron", True),
                                       ("classical", True)])
def test_batched_kinds_match_serial_path(kind, drop):
    p, q, nb, D, G, n_w = 3, 64, 40, 48, 8, 9
    cube = scenes.bench_scene(p, q, nb, seed=41, movers=3).data[0]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    kw = dict(kind=kind, drop_temporal=drop)
    got = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, **kw).values
    ser = _serial(lambda: kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, **kw).values)
    m0 = _m0(cube, D, G)
    assert np.all(np.abs(got - ser) <= 1e-9 * np.abs(ser) + 1e-10 * m0)
    # tiles with halo are bitwise the full-frame rows
    tile = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, bins=(7, 30), **kw).values
    assert np.array_equal(tile, got[7:30])


def test_batched_non_uniform_doppler_and_arbitrary_grid():
    p, q, nb, n_w = 3, 48, 30, 9
    cube = scenes.bench_scene(p, q, nb, seed=3, movers=2).data[0]
    rng = np.random.default_rng(0)
    dop = np.sort(rng.uniform(-0.5, 0.5, 37))
    grid = (rng.standard_normal((5, p)) + 1j * rng.standard_normal((5, p))) / 2
    got = kst.windowed_detection_image(cube, n_w, 1, 2, dop, grid).values
    ser = _serial(lambda: kst.windowed_detection_image(cube, n_w, 1, 2, dop, grid).values)
    scale = float(np.abs(ser).max())
    assert np.all(np.abs(got - ser) <= 1e-9 * np.abs(ser) + 1e-11 * scale)


def test_batched_edge_cases():
    p, q, nb, D, G, n_w = 3, 32, 24, 32, 16, 5
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    cube = scenes.bench_scene(p, q, nb, seed=9, movers=1).data[0]
    # all-zero training window -> zero estimate, identity filter (src/lrkron.py:152-160)
    z = cube.copy()
    z[:n_w + 2] = 0.0
    got = kst.windowed_detection_image(z, n_w, 1, 3, dop, grid).values
    ser = _serial(lambda: kst.windowed_detection_image(z, n_w, 1, 3, dop, grid).values)
    assert np.allclose(got, ser, rtol=1e-9, atol=1e-12)
    assert windowed.last_window_info()[0, 1] == 0  # no iterations on the zero window
    # non-finite data -> DataError (the reference's covariance validation)
    bad = cube.copy()
    bad[12, 1, 5] = np.inf
    with pytest.raises(kst.DataError):
        kst.windowed_detection_image(bad, n_w, 1, 3, dop, grid)
    # n_w = n_bins (one window for every bin) and n_w = 1
    for nw in (nb, 1):
        got = kst.windowed_detection_image(cube, nw, 1, 2, dop, grid).values
        ser = _serial(lambda: kst.windowed_detection_image(cube, nw, 1, 2, dop, grid).values)
        assert np.allclose(got, ser, rtol=1e-9, atol=1e-10 * float(np.abs(ser).max()))


def test_batched_is_deterministic():
    p, q, nb, D, n_w = 3, 64, 64, 64, 25
    cube = torch.from_numpy(scenes.bench_scene(p, q, nb, seed=77, movers=3).data[0]).cuda()
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, 16)
    a = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid).values
    b = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid).values
    assert a.is_cuda and torch.equal(a, b)
