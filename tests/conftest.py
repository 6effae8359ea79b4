"""Shared pytest wiring: the `gpu` marker and golden-fixture loaders."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libkst_b200.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def basis_of(d, key):
    return None if bool(d[key + "_none"]) else d[key]


def cfg_of(d):
    import ast
    return ast.literal_eval(str(d["cfg"]))


def scene_cube(d, store_key="cube"):
    """Cube of a pipeline golden case: stored, or regenerated and hash-checked."""
    import hashlib
    from paper_1604_03622_b200 import scenes
    if store_key in d.files:
        return np.array(d[store_key])
    cfg = scenes.SceneConfig(**cfg_of(d))
    hist = scenes.gen_clutter(cfg)
    for b, f, a in d["targets"]:
        hist = scenes.inject_target(hist, int(b), float(f), complex(a))
    cube = hist.data[0]
    assert hashlib.sha256(np.ascontiguousarray(cube).tobytes()).hexdigest() == str(d["cube_sha"])
    return cube


PIPELINE_CASES = ["readme_q16"] + [f"sweep_q64_ra{a}_rb{b}" for a in (1, 2, 3) for b in (1, 2, 3)] + [
    "classical_q64", "droptemporal_q64", "cfg1_q256"]


@pytest.fixture(autouse=True)
def _detection_precision_default():
    """Every test starts from the library default K5 precision (f32) on this
    thread's context and leaves it there, whatever it selected."""
    yield
    if "paper_1604_03622_b200" in sys.modules:
        try:
            import torch
            if torch.cuda.is_available():
                sys.modules["paper_1604_03622_b200"].set_detect_precision("f32")
        except Exception:  # pragma: no cover - no GPU / library
            pass


@pytest.fixture
def f64_detection():
    """Run the test with the FP64 detection kernels (tight parity)."""
    import paper_1604_03622_b200 as kst
    kst.set_detect_precision("f64")
    yield
    kst.set_detect_precision("f32")


@pytest.fixture(params=["f64", "f32"])
def precision(request):
    """Parametrise a test over the two K5 precisions; yields the name."""
    import paper_1604_03622_b200 as kst
    kst.set_detect_precision(request.param)
    yield request.param
    kst.set_detect_precision("f32")


def tight_tolerance(ref, m0, precision):
    """Per-precision regression bound, far inside the SURVEY.md §8c rule:
    FP64 detection 1e-9 |v_ref| + 1e-10 M0; FP32 detection (FP32 transform
    of the spectra, measured max |err| <= 5e-8 M0) 1e-5 |v_ref| + 1e-6 M0."""
    if precision == "f64":
        return map_tolerance(ref, m0, 1e-9, 1e-10)
    return map_tolerance(ref, m0, 1e-5, 1e-6)


def map_tolerance(ref, m0, rel=1e-4, floor=1e-5):
    """SURVEY.md §8c map rule: |v - v_ref| <= rel*|v_ref| + floor*M0."""
    return rel * np.abs(ref) + floor * m0


def binary_map_mismatch(vals, ref, m0, taus):
    """north_star / SURVEY.md §8c detection-map rule: the thresholded maps
    (v >= tau) must be identical except at pixels whose reference statistic
    lies within the map tolerance of tau. Returns (disallowed mismatches,
    allowed near-threshold mismatches) summed over the thresholds."""
    tol = map_tolerance(ref, m0)
    bad = near = 0
    for tau in taus:
        diff = (vals >= tau) != (ref >= tau)
        band = np.abs(ref - tau) <= tol
        bad += int(np.count_nonzero(diff & ~band))
        near += int(np.count_nonzero(diff & band))
    return bad, near
