"""CPU: pin the oracle (oracle/kron_oracle.py) and the scene generator
(paper_1604_03622_b200/scenes.py) against outputs of the unmodified
reference (tests/golden, made by oracle/gen_golden.py)."""

import ast
import hashlib

import numpy as np
import pytest

from conftest import PIPELINE_CASES, basis_of, cfg_of, golden, scene_cube
from oracle import kron_oracle as orc
from paper_1604_03622_b200 import scenes


def _proj(u):
    return np.zeros((0, 0)) if u is None else u @ u.conj().T


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_oracle_pipeline_matches_reference(name):
    d = golden(name)
    cube = scene_cube(d)
    n, p, q = cube.shape
    s = orc.scm(cube.reshape(n, p * q), p, q)
    assert np.isclose(np.linalg.norm(s), float(d["scm_fro"]), rtol=1e-13)
    if "scm" in d.files:
        assert np.linalg.norm(s - d["scm"]) <= 1e-14 * np.linalg.norm(s)
    fit = orc.lrkron(s, p, q, int(d["ra"]), int(d["rb"]), float(d["tol"]), int(d["max_iter"]))
    assert fit.iterations == int(d["iterations"])
    assert fit.converged == bool(d["converged"])
    np.testing.assert_allclose(fit.residuals, d["residuals"], rtol=1e-9)
    assert np.linalg.norm(fit.spatial - d["spatial"]) <= 1e-10 * np.linalg.norm(d["spatial"])
    ua, ub = orc.filter_bases(fit)
    for got, key in ((ua, "ua"), (ub, "ub")):
        want = basis_of(d, key)
        assert (got is None) == (want is None)
        if got is not None:
            assert got.shape == want.shape
            assert np.abs(_proj(got) - _proj(want)).max() < 1e-8
    vals = orc.detect(str(d["kind"]), ua, ub, cube, orc.doppler_grid(int(d["D"])),
                      orc.spatial_grid(p, int(d["G"])), bool(d["drop_temporal"]))
    tol = 1e-9 * np.abs(d["values"]) + 1e-10 * float(d["m0"])
    assert np.all(np.abs(vals - d["values"]) <= tol)


def test_oracle_estimator_edge_cases():
    g = golden("estimator_cases")
    for key in g["keys"]:
        key = str(key)
        c = {k.split("__", 1)[1]: g[k] for k in g.files if k.startswith(key + "__")}
        args = (c["s"], int(c["p"]), int(c["q"]), int(c["ra"]), int(c["rb"]),
                float(c["tol"]), int(c["max_iter"]))
        if str(c["error"]):
            with pytest.raises(orc.OracleError) as ei:
                orc.lrkron(*args)
            assert ei.value.kind == str(c["error"]), key
            continue
        fit = orc.lrkron(*args)
        assert fit.iterations == int(c["iterations"]), key
        assert fit.converged == bool(c["converged"]), key
        np.testing.assert_allclose(fit.residuals, c["residuals"], rtol=1e-7, atol=1e-12, err_msg=key)
        sc = max(np.linalg.norm(c["spatial"]), 1e-300)
        assert np.linalg.norm(fit.spatial - c["spatial"]) <= 1e-9 * sc, key
        tc = max(np.linalg.norm(c["temporal"]), 1e-300)
        assert np.linalg.norm(fit.temporal - c["temporal"]) <= 1e-9 * tc, key


def test_oracle_eig_conventions():
    g = golden("eig_cases")
    for i in range(int(g["count"])):
        m = g[f"m{i}"]
        lam, vec = orc.heig(m)
        np.testing.assert_allclose(lam, g[f"lam{i}"], rtol=1e-12, atol=1e-12)
        # with distinct eigenvalues the pivot-phase rule fixes vectors uniquely
        gaps = np.diff(lam)
        if lam.size < 2 or np.min(np.abs(gaps)) > 1e-6:
            np.testing.assert_allclose(vec, g[f"vec{i}"], atol=1e-10)
        n = m.shape[0]
        for r in sorted({1, max(1, n // 2), n}):
            np.testing.assert_allclose(orc.truncate(m, r), g[f"trunc{i}_{r}"], atol=1e-11)
            b = orc.basis(m, r)
            want = g[f"basis{i}_{r}"]
            if b is None:
                assert want.size == 0
            else:
                assert b.shape == want.shape
                np.testing.assert_allclose(b @ b.conj().T, want @ want.conj().T, atol=1e-10)


def test_oracle_detection_argument_space():
    g = golden("detect_cases")
    cube = g["cube"]
    for i in range(int(g["count"])):
        v = orc.detect(str(g[f"kind{i}"]), basis_of(g, f"ua{i}"), basis_of(g, f"ub{i}"), cube,
                       g[f"dop{i}"], g[f"grid{i}"], bool(g[f"so{i}"]))
        np.testing.assert_allclose(v, g[f"values{i}"], rtol=1e-12, atol=1e-13)


def test_oracle_multipass():
    g = golden("multipass_cases")
    for name in g["names"]:
        name = str(name)
        data = g[f"{name}__data"]
        k, n, p, q = data.shape
        st = orc.stack(data)
        s = orc.scm(st.reshape(n, -1), k * p, q)
        fit = orc.lrkron(s, k * p, q, k, int(g[f"{name}__rb"]))
        assert fit.iterations == int(g[f"{name}__iterations"])
        ua, ub = orc.filter_bases(fit)
        maps = orc.pass_maps("kron", ua, ub, st, k, p, orc.doppler_grid(int(g[f"{name}__D"])),
                             int(g[f"{name}__G"]))
        want = g[f"{name}__maps"]
        scale = np.abs(want).max()
        assert np.abs(np.stack(maps) - want).max() <= 1e-9 * scale
        ch = orc.change(maps[0], maps[1])
        assert np.abs(ch - g[f"{name}__change01"]).max() <= 1e-9 * scale


def test_scenes_are_bit_exact_with_reference_simulator():
    g = golden("scene_hashes")
    for cfg_s, k, gen_s, want in zip(g["cfg"], g["k"], g["gen"], g["sha"]):
        cfg = scenes.SceneConfig(**ast.literal_eval(str(cfg_s)))
        gkw = ast.literal_eval(str(gen_s))
        k = int(k)
        hist = scenes.gen_clutter(cfg) if k == 1 and not gkw else scenes.gen_multipass(cfg, k, **gkw)
        hist = scenes.inject_target(hist, 3, 0.25, 2.0 - 1.0j, pass_index=k - 1)
        assert hashlib.sha256(np.ascontiguousarray(hist.data).tobytes()).hexdigest() == str(want)


def test_oracle_optimal_and_sinr():
    """oracle.optimal_whiten / steering / sinr against the reference's
    build_filter("optimal"), detection_image, make_steering and sinr outputs
    (oracle/gen_golden.py optimal_cases)."""
    g = golden("optimal_cases")
    sigma, cube = g["sigma"], g["cube"]
    wh = orc.optimal_whiten(sigma, cube)
    assert np.abs(wh - g["whitened"]).max() <= 1e-12 * np.abs(g["whitened"]).max()
    m = orc.detect("kron", None, None, wh, orc.doppler_grid(32), orc.spatial_grid(3, 8))
    assert np.abs(m - g["map"]).max() <= 1e-12 * np.abs(g["map"]).max()
    sv = orc.steering(0.25, 3, 32, kappa=2.0)
    assert np.abs(sv - g["steering"]).max() <= 1e-15
    w_opt = orc.optimal_whiten(sigma, sv.reshape(1, 3, 32)).ravel()
    assert abs(orc.sinr(w_opt, sv, 2.0, sigma) - g["sinr"][2]) <= 1e-10 * g["sinr"][2]
