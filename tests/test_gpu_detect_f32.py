"""The default FP32 detection kernel (csrc/detect_f32.cu: FP64 load pass,
Good-Thomas prime-factor DFT in FP32) against the oracle's restatement of
detection_image (src/filters.py:243-275) and against the FP64 kernels.

Comparators: SURVEY.md §8c |v - v_ref| <= 1e-4 |v_ref| + 1e-5 M0 everywhere,
and the FP32 regression bound conftest.tight_tolerance(.., "f32") =
1e-5 |v_ref| + 1e-6 M0 (measured max |err| <= 5e-8 M0)."""

import numpy as np
import pytest

from conftest import map_tolerance, tight_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402


def _filter(cube, ra, rb, kind="kron", drop=False):
    n, p, q = cube.shape
    s = kst.sample_covariance(kst.cube_to_snapshots(cube), p, q)
    return kst.build_filter(kind, estimate=kst.lr_kron_estimate(s, ra, rb), drop_temporal=drop)


def _check(cube, filt, D, grid, kind="kron"):
    dop = kst.make_doppler_grid(D)
    kst.set_detect_precision("f32")
    got = kst.detection_image(filt, cube, dop, grid).values
    want = orc.detect(kind, filt.spatial_basis, filt.temporal_basis, cube, dop, grid,
                      spatial_only=filt.spatial_only)
    m0 = orc.detect("kron", None, None, cube, dop, grid).max()
    err = np.abs(got - want)
    assert np.all(err <= map_tolerance(want, m0))
    assert np.all(err <= tight_tolerance(want, m0, "f32")), (err / m0).max()
    return got


# D: prime-power factors <= 32 (Good-Thomas), factors above 32 split a x b
# (Cooley-Tukey inside the factor: 64 = 8 x 8, 256 = 16 x 16, 125 = 25 x 5),
# a prime pencil (29), q < D (zero padding), q == D
@pytest.mark.parametrize("q,D", [(48, 48), (40, 64), (60, 60), (29, 29), (100, 256), (120, 125),
                                 (90, 2 * 3 * 5 * 7), (64, 1000), (200, 2001)])
def test_plans_match_oracle(q, D):
    cube = scenes.bench_scene(3, q, 24, seed=7, movers=3).data[0]
    _check(cube, _filter(cube, 1, 3), D, kst.make_spatial_grid(3, 16))


@pytest.mark.parametrize("p,ra,rb,kind,drop,G", [
    (3, 2, 2, "kron", False, 16),       # one reduced row (NR = 1)
    (3, 1, 1, "kron", False, 8),
    (2, 1, 2, "kron", False, 16),
    (4, 1, 3, "kron", False, 12),       # NR = 3
    (3, 1, 3, "classical", False, 16),  # joint coefficient transform, NR = P
    (3, 1, 3, "kron", True, 16),        # spatial only (no temporal coefficients)
])
def test_filter_kinds_match_oracle(p, ra, rb, kind, drop, G):
    cube = scenes.bench_scene(p, 64, 40, seed=11, movers=3).data[0]
    _check(cube, _filter(cube, ra, rb, kind, drop), 64, kst.make_spatial_grid(p, G), kind)


def test_arbitrary_spatial_grid_and_identity_filter():
    cube = scenes.bench_scene(3, 64, 32, seed=3, movers=2).data[0]
    rng = np.random.default_rng(5)
    grid = (rng.standard_normal((7, 3)) + 1j * rng.standard_normal((7, 3))) / np.sqrt(6)
    _check(cube, _filter(cube, 1, 3), 64, grid)
    # no bases: the identity filter (temporal coefficients off, Q = I)
    _check(cube, kst.projection_filter("kron", None, None, 3, 64), 64, kst.make_spatial_grid(3, 16))


def test_f32_against_f64_and_deterministic():
    cube = torch.from_numpy(scenes.bench_scene(3, 256, 256, seed=17, movers=8).data[0]).cuda()
    filt = _filter(cube, 1, 3)
    dop, grid = kst.make_doppler_grid(256), kst.make_spatial_grid(3, 16)
    kst.set_detect_precision("f64")
    ref = kst.detection_image(filt, cube, dop, grid).values.cpu().numpy()
    kst.set_detect_precision("f32")
    a = kst.detection_image(filt, cube, dop, grid).values.cpu().numpy()
    b = kst.detection_image(filt, cube, dop, grid).values.cpu().numpy()
    assert np.array_equal(a, b)  # fixed-order reductions
    m0 = float(kst.detection_image(kst.projection_filter("kron", None, None, 3, 256), cube, dop,
                                   grid).values.max())
    assert np.all(np.abs(a - ref) <= tight_tolerance(ref, m0, "f32"))
    assert kst.get_detect_precision() == "f32"


def test_non_finite_bin_raises_data_error():
    cube = scenes.bench_scene(3, 64, 20, seed=2, movers=1).data[0]
    filt = _filter(cube, 1, 3)
    for v in (np.nan, np.inf):
        bad = cube.copy()
        bad[13, 2, 7] = v
        with pytest.raises(kst.DataError):
            kst.detection_image(filt, bad, kst.make_doppler_grid(64), kst.make_spatial_grid(3))


def test_unsupported_plan_runs_the_fp64_kernels():
    """D with a prime factor above 32 (37) has no FP32 plan: the FP64 kernels
    run, bitwise equal to precision f64."""
    cube = scenes.bench_scene(3, 37, 16, seed=4, movers=1).data[0]
    filt = _filter(cube, 1, 3)
    dop, grid = kst.make_doppler_grid(74), kst.make_spatial_grid(3)
    a = kst.detection_image(filt, cube, dop, grid).values
    kst.set_detect_precision("f64")
    b = kst.detection_image(filt, cube, dop, grid).values
    assert np.array_equal(a, b)
