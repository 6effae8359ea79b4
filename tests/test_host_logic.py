"""CPU: host-side logic of the package -- argument validation raised before
any device work (mirroring the reference's DimensionError paths), grids,
layout helpers, scene generation, and the bench reference arm's JSON line."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1604_03622_b200 as kst
from conftest import ROOT
from oracle import kron_oracle as orc


def test_grids_match_the_reference_definitions():
    for count in (1, 7, 64, 2001):
        assert np.array_equal(kst.make_doppler_grid(count), orc.doppler_grid(count))
    for p, g in ((3, 16), (4, 8), (12, 16)):
        np.testing.assert_array_equal(kst.make_spatial_grid(p, g), orc.spatial_grid(p, g))
    np.testing.assert_array_equal(kst.make_stacked_spatial_grid(3, 4, 16), orc.stacked_grid(3, 4, 16))
    with pytest.raises(kst.DimensionError):
        kst.make_doppler_grid(0)
    with pytest.raises(kst.DimensionError):
        kst.make_spatial_grid(3, 0)


def test_layout_helpers():
    cube = np.arange(2 * 3 * 4, dtype=complex).reshape(2, 3, 4)
    snaps = kst.cube_to_snapshots(cube)
    assert snaps.shape == (2, 12) and snaps[1, 5] == cube[1, 1, 1]
    assert np.array_equal(kst.from_snapshot(kst.to_snapshot(cube[0]), 3, 4), cube[0])
    with pytest.raises(kst.DimensionError):
        kst.cube_to_snapshots(np.zeros((2, 3)))
    with pytest.raises(kst.DimensionError):
        kst.from_snapshot(np.zeros(5), 2, 3)


def test_sample_covariance_validation_happens_on_the_host():
    # tests/test_lrkron.py:70-76 of the reference
    with pytest.raises(kst.DimensionError):
        kst.sample_covariance(np.zeros(6), 2, 3)
    with pytest.raises(kst.DimensionError):
        kst.sample_covariance(np.zeros((0, 6)), 2, 3)
    with pytest.raises(kst.DimensionError):
        kst.sample_covariance(np.zeros((4, 5)), 2, 3)


def test_estimator_rejects_non_covariance_and_bad_shape():
    with pytest.raises(kst.DimensionError):
        kst.lr_kron_estimate(np.eye(6), 1, 1)
    with pytest.raises(kst.DimensionError):
        kst.lr_kron_estimate(kst.SampleCovariance(np.eye(5), 1, 2, 3), 1, 1)


def test_filter_and_detection_validation():
    ua = np.eye(3)[:, :1]
    with pytest.raises(kst.DimensionError):
        kst.projection_filter("optimal", ua, None, 3, 4)
    with pytest.raises(kst.DimensionError):
        kst.projection_filter("kron", ua, None, 4, 4)
    filt = kst.projection_filter("kron", None, None, 2, 4)
    with pytest.raises(kst.DimensionError):
        kst.detection_image(filt, np.zeros((3, 4, 2), complex), kst.make_doppler_grid(4),
                            kst.make_spatial_grid(2, 4))
    with pytest.raises(kst.DimensionError):
        kst.detection_image(filt, np.zeros((3, 2, 4), complex), kst.make_doppler_grid(4),
                            kst.make_spatial_grid(3, 4))
    with pytest.raises(kst.DimensionError):
        filt.apply_matrix(np.zeros((4, 2), complex))
    # optimal kind: argument / shape errors before any device work
    # (src/filters.py:144-153; as_matrix's finite check precedes the shape check)
    with pytest.raises(kst.DimensionError):
        kst.build_filter("optimal", sigma=np.eye(2), p=1)
    with pytest.raises(kst.DimensionError):
        kst.build_filter("optimal", sigma=np.eye(3), p=1, q=2)
    with pytest.raises(kst.DimensionError):
        kst.build_filter("optimal", sigma=np.ones(4), p=1, q=2)
    with pytest.raises(kst.DataError):
        kst.build_filter("optimal", sigma=np.full((3, 3), np.nan), p=1, q=2)
    with pytest.raises(kst.DimensionError):
        kst.make_steering(0.1, 0, 4)
    sv = kst.make_steering(0.0, 4, 8)
    assert np.array_equal(sv.spatial, np.ones(4))
    assert abs(np.linalg.norm(sv.vector) - 1.0) < 1e-12
    with pytest.raises(kst.DimensionError):
        kst.build_filter("bogus")


def test_multipass_validation():
    with pytest.raises(kst.DimensionError):
        kst.stack_passes(np.zeros((2, 3, 4)))
    with pytest.raises(kst.DimensionError):
        kst.unstack_passes(np.zeros((3, 4)))
    with pytest.raises(kst.DimensionError):
        kst.multipass_estimate(np.zeros((4, 4)), 2)
    d = kst.make_doppler_grid(4)
    a = kst.DetectionMap(np.zeros((2, 4)), d, None)
    with pytest.raises(kst.DimensionError):
        kst.change_detect(a, np.zeros((2, 4)))
    with pytest.raises(kst.DimensionError):
        kst.change_detect(a, kst.DetectionMap(np.zeros((3, 4)), d, None))
    with pytest.raises(kst.DimensionError):
        kst.change_detect(a, kst.DetectionMap(np.zeros((2, 4)), d + 0.5, None))


def test_stack_round_trip_host():
    cfg = kst.SceneConfig(p=2, q=8, n_bins=10, rank_temporal=2, noise_power=0.02, seed=3)
    hist = kst.gen_multipass(cfg, 3)
    back = kst.unstack_passes(kst.stack_passes(hist))
    assert np.array_equal(back.data, hist.data)
    assert np.array_equal(kst.stack_passes(hist).data, orc.stack(hist.data))


def test_bench_scene_is_deterministic():
    from paper_1604_03622_b200 import scenes
    a = scenes.bench_scene(3, 32, 40, seed=5).data
    b = scenes.bench_scene(3, 32, 40, seed=5).data
    assert np.array_equal(a, b)
    assert not np.array_equal(a, scenes.bench_scene(3, 32, 40, seed=6).data)


def test_bench_reference_arm_prints_one_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="2", OPENBLAS_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "pixels/s" and d["value"] > 0
    # the unmodified reference when baseline/_ref is installed, else the port
    has_ref = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "kronstap"))
    assert d["cpu_baseline"]["kind"] == ("reference" if has_ref else "port")
    if has_ref:
        assert set(d["cpu_baseline"]["modes"]) == {"blas", "pool"}
        assert d["cpu_baseline"]["host"]["blas"] is not None
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_window_partition_covers_every_bin_once():
    """L-mode windows: window_bins(s) are exactly the bins whose
    window_start is s, and they partition [0, n_bins)."""
    from paper_1604_03622_b200.windowed import window_bins, window_start
    for n_bins, n_w in [(40, 9), (40, 25), (256, 81), (10, 10), (7, 1)]:
        seen = []
        for s in range(n_bins - n_w + 1):
            lo, hi = window_bins(s, n_w, n_bins)
            seen.extend(range(lo, hi))
            assert all(window_start(m, n_w, n_bins) == s for m in range(lo, hi))
        assert seen == list(range(n_bins))


def test_frame_graph_rejects_host_cubes():
    """FrameGraph captures a device buffer: host tensors and wrong ranks are
    refused before anything touches the library (no CPU fallback)."""
    import torch
    with pytest.raises(kst.DimensionError):
        kst.FrameGraph(torch.zeros((4, 3, 96), dtype=torch.complex128))
    with pytest.raises(kst.DimensionError):
        kst.FrameGraph(torch.zeros((4, 96), dtype=torch.complex128))
