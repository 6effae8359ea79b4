"""GPU parity of the L-mode windowed estimator (BASELINE.json configs[3],
SURVEY.md §8 "L-mode definition") against the oracle's loop over the
reference functions: per window identical iterations / convergence, maps
within the §8c rule |v - v_ref| <= 1e-4 |v_ref| + 1e-5 M0."""

import numpy as np
import pytest

from conftest import map_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402


def _m0(cube, D, G):
    p = cube.shape[1]
    return float(np.max(orc.detect("kron", None, None, cube, orc.doppler_grid(D),
                                   orc.spatial_grid(p, G))))


@pytest.mark.parametrize("n_w,ra,rb", [(9, 1, 3), (25, 1, 3), (9, 1, 1), (25, 2, 3)])
def test_windowed_matches_oracle(n_w, ra, rb):
    p, q, nb, D, G = 3, 64, 40, 64, 16
    cube = scenes.bench_scene(p, q, nb, seed=17, movers=4).data[0]
    ref, fits = orc.windowed(cube, n_w, ra, rb, D, G)
    dmap, ests = kst.windowed_detection_image(cube, n_w, ra, rb, kst.make_doppler_grid(D),
                                              kst.make_spatial_grid(p, G), return_estimates=True)
    assert len(ests) == nb - n_w + 1 == len(fits)
    for s, est in ests:
        assert est.iterations == fits[s].iterations and est.converged == fits[s].converged
        np.testing.assert_allclose(est.residuals, fits[s].residuals, rtol=1e-8, atol=1e-9)
    m0 = _m0(cube, D, G)
    err = np.abs(dmap.values - ref)
    assert np.all(err <= map_tolerance(ref, m0)), (err / map_tolerance(ref, m0)).max()


def test_windowed_cfg1_sampled_bins():
    """configs[3] size (p=3, q=n_bins=D=256, G=16, n_w=81, ranks (1, 3)): full
    GPU map, oracle on a seeded sample of bins (edges and interior)."""
    p, q, nb, D, G, n_w = 3, 256, 256, 256, 16, 81
    cube = scenes.bench_scene(p, q, nb, seed=17, movers=8).data[0]
    bins = [0, 40, 41, 100, 173, 215, 216, 255]
    ref, _ = orc.windowed(cube, n_w, 1, 3, D, G, bins=bins)
    dmap = kst.windowed_detection_image(cube, n_w, 1, 3, kst.make_doppler_grid(D),
                                        kst.make_spatial_grid(p, G))
    m0 = _m0(cube, D, G)
    got, want = dmap.values[bins], ref[bins]
    assert np.all(np.abs(got - want) <= map_tolerance(want, m0))
    assert np.all(np.isfinite(dmap.values)) and dmap.values.shape == (nb, D)


def test_windowed_device_tensors_stay_on_device():
    p, q, nb, D = 3, 32, 20, 32
    cube = torch.from_numpy(scenes.bench_scene(p, q, nb, seed=5, movers=2).data[0]).cuda()
    dmap = kst.windowed_detection_image(cube, 9, 1, 2, kst.make_doppler_grid(D),
                                        kst.make_spatial_grid(p, 16))
    assert dmap.values.is_cuda and tuple(dmap.values.shape) == (nb, D)


@pytest.mark.parametrize("world,n_w", [(2, 9), (3, 25), (8, 9)])
def test_bin_tiles_with_halo_equal_the_full_frame(world, n_w):
    """SURVEY.md §8e windowed L-mode sharding: each tile (tile_bounds) reads
    only its halo range; the tiles, concatenated, equal the one-GPU map
    bitwise (host cube: only the halo range is uploaded; device cube: views)."""
    from paper_1604_03622_b200 import parallel
    from paper_1604_03622_b200.windowed import halo_range
    p, q, nb, D, G = 3, 64, 40, 64, 16
    cube = scenes.bench_scene(p, q, nb, seed=23, movers=4).data[0]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    full = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid).values
    tiles = []
    for lo, hi in parallel.tile_bounds(nb, world):
        a, b = halo_range(lo, hi, n_w, nb)
        seen = np.full_like(cube, np.nan)  # bins outside the halo are never read
        seen[a:b] = cube[a:b]
        tiles.append(kst.windowed_detection_image(seen, n_w, 1, 3, dop, grid, bins=(lo, hi)).values)
    assert np.array_equal(np.concatenate(tiles), full)
    dev = torch.from_numpy(cube).cuda()
    t1 = kst.windowed_detection_image(dev, n_w, 1, 3, dop, grid, bins=(5, 17)).values
    assert t1.is_cuda and np.array_equal(t1.cpu().numpy(), full[5:17])


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_concurrent_windows_are_bitwise_serial(workers):
    """Windows estimated on concurrent host threads / streams give exactly the
    serial loop's map and estimates."""
    p, q, nb, D, G, n_w = 3, 64, 48, 64, 16, 9
    cube = scenes.bench_scene(p, q, nb, seed=31, movers=4).data[0]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    ref, ref_est = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, workers=1,
                                                return_estimates=True)
    for _ in range(2):
        got, est = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, workers=workers,
                                                return_estimates=True)
        assert np.array_equal(got.values, ref.values)
        assert [s for s, _ in est] == [s for s, _ in ref_est]
        for (_, e1), (_, e2) in zip(est, ref_est):
            assert e1.iterations == e2.iterations and e1.residuals == e2.residuals
            h = [e.spatial.cpu().numpy() if torch.is_tensor(e.spatial) else e.spatial
                 for e in (e1, e2)]
            assert np.array_equal(h[0], h[1])


@pytest.mark.parametrize("workers", [1, 4])
@pytest.mark.parametrize("kind,drop", [("kron", False), ("classical", False), ("kron", True)])
def test_fused_windows_equal_the_step_api_loop(workers, kind, drop, monkeypatch):
    """kst_windowed (one C call per worker, no per-window Python; the serial
    per-window path the batched kst_lmode falls back to) gives the step-API
    loop's map bitwise, also for a tile with halo."""
    monkeypatch.setenv("KST_LMODE", "serial")
    p, q, nb, D, G, n_w = 3, 64, 40, 48, 8, 9
    cube = scenes.bench_scene(p, q, nb, seed=41, movers=3).data[0]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    kw = dict(kind=kind, drop_temporal=drop)
    ref = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, return_estimates=True, workers=1,
                                       **kw)[0].values
    got = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, workers=workers, **kw).values
    assert np.array_equal(got, ref)
    tile = kst.windowed_detection_image(cube, n_w, 1, 3, dop, grid, bins=(7, 30), workers=workers,
                                        **kw).values
    assert np.array_equal(tile, ref[7:30])
    bad = cube.copy()
    bad[12, 1, 5] = np.nan
    with pytest.raises(kst.DataError):
        kst.windowed_detection_image(bad, n_w, 1, 3, dop, grid, workers=workers, **kw)
