"""GPU subcommands of the CLI (`estimate`, `filter`, `detect`, `bench`)
against the outputs of the UNMODIFIED reference CLI on the same files
(tests/golden/io/, oracle/gen_golden_io.py), plus the behavioural checks
of the reference's tests/test_cli.py."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1604_03622_b200 import cli, formats  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")


def gold(name):
    return os.path.join(GOLD, name)


def run(*args):
    return cli.main([str(a) for a in args])


def _projector(u_mat, rank, ref):
    """Rank-`rank` spectral projector, truncated to the eigenvalues of `ref`
    that clear 1e-6 of its largest (degenerate directions are arbitrary)."""
    lam = np.linalg.eigvalsh(ref)
    rank = min(rank, int(np.sum(lam > 1e-6 * lam.max())))
    w, v = np.linalg.eigh(u_mat)
    v = v[:, ::-1][:, :rank]
    return v @ v.conj().T


@pytest.mark.parametrize("cube,name,ra,rb,extra,code", [
    ("scene.kph", "fit.kes", 1, 3, [], 0),
    ("scene.kph", "cap.kes", 1, 3, ["--eps", "1e-14", "--max-iter", 1], 3),
    ("passes.kph", "joint.kes", 2, 2, [], 0),
    ("changed.kph", "changed.kes", 2, 2, [], 0)])
def test_estimate_matches_reference(cube, name, ra, rb, extra, code, tmp_path):
    out = tmp_path / name
    assert run("estimate", "--input", gold(cube), "--output", out, "--ra", ra, "--rb", rb,
               *extra) == code
    got, ref = formats.read_estimate(out), formats.read_estimate(gold(name))
    assert (got.rank_spatial, got.rank_temporal, got.iterations, got.converged) == \
        (ref.rank_spatial, ref.rank_temporal, ref.iterations, ref.converged)
    for a, b in ((got.spatial, ref.spatial), (got.temporal, ref.temporal)):
        assert a.shape == b.shape
        assert np.linalg.norm(a - b) <= 1e-9 * max(np.linalg.norm(b), 1e-300)
    assert np.linalg.norm(_projector(got.spatial, ra, ref.spatial)
                          - _projector(ref.spatial, ra, ref.spatial)) <= 1e-8
    res = formats.read_residuals_csv(str(out) + ".residuals.csv")
    ref_res = formats.read_residuals_csv(gold(name + ".residuals.csv"))
    np.testing.assert_allclose(res, ref_res, rtol=1e-9, atol=1e-12)


def test_estimate_bytes_are_thread_invariant(tmp_path):
    a, b = tmp_path / "a.kes", tmp_path / "b.kes"
    assert run("estimate", "--input", gold("scene.kph"), "--output", a, "--ra", 1, "--rb", 3,
               "--threads", 1) == 0
    assert run("estimate", "--input", gold("scene.kph"), "--output", b, "--ra", 1, "--rb", 3,
               "--threads", 8) == 0
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.parametrize("cube,est,name,extra", [
    ("scene.kph", "fit.kes", "filtered.kph", []),
    ("scene.kph", "fit.kes", "classical.kph", ["--kind", "classical"]),
    ("passes.kph", "joint.kes", "pfilt.kph", [])])
def test_filter_matches_reference(cube, est, name, extra, tmp_path):
    out = tmp_path / name
    assert run("filter", "--input", gold(cube), "--estimate", gold(est), "--output", out,
               *extra) == 0
    got, ref = formats.read_phase_history(out), formats.read_phase_history(gold(name))
    src = formats.read_phase_history(gold(cube))
    assert got.data.shape == ref.data.shape and got.truth == ref.truth
    assert np.abs(got.data - ref.data).max() <= 1e-12 * np.abs(src.data).max()
    if name == "filtered.kph":  # reference test: most clutter energy removed
        assert np.linalg.norm(got.data) <= 0.2 * np.linalg.norm(src.data)


@pytest.mark.parametrize("cube,est,name,extra", [
    ("target.kph", "fit.kes", "map.csv", []),
    ("target.kph", "fit.kes", "map_sp.csv",
     ["--grid-doppler", 40, "--grid-spatial", 8, "--no-temporal-projection"]),
    ("passes.kph", "joint.kes", "change.csv", ["--multipass"]),
    ("changed.kph", "changed.kes", "change_signed.csv",
     ["--multipass", "--signed", "--grid-doppler", 16])])
def test_detect_matches_reference(cube, est, name, extra, tmp_path):
    out = tmp_path / name
    assert run("detect", "--input", gold(cube), "--estimate", gold(est), "--output", out,
               *extra) == 0
    got, ref = formats.read_detection_csv(out), formats.read_detection_csv(gold(name))
    assert np.array_equal(got.dopplers, ref.dopplers) and got.values.shape == ref.values.shape
    scale = np.abs(formats.read_phase_history(gold(cube)).data).max()
    assert np.abs(got.values - ref.values).max() <= 1e-10 * scale
    if name == "change.csv":  # identical passes cancel (reference test)
        assert got.values.max() <= 1e-12
    if name == "change_signed.csv":
        assert (got.values < 0).any()


def test_detect_pgm_matches_reference(tmp_path):
    assert run("detect", "--input", gold("target.kph"), "--estimate", gold("fit.kes"),
               "--output", tmp_path / "m.csv", "--pgm", tmp_path / "m.pgm") == 0
    got = np.frombuffer((tmp_path / "m.pgm").read_bytes()[-40 * 64 * 2:], ">u2").astype(int)
    ref = np.frombuffer(open(gold("map.pgm"), "rb").read()[-40 * 64 * 2:], ">u2").astype(int)
    assert (tmp_path / "m.pgm").read_bytes().startswith(b"P5\n64 40\n65535\n")
    assert np.abs(got - ref).max() <= 1  # rounding of peak-scaled pixels


def test_planted_target_end_to_end(tmp_path):
    """simulate -> estimate -> detect through the CLI alone (reference
    tests/test_cli.py:155-183)."""
    fit, clean, dirty = tmp_path / "fit.kes", tmp_path / "clean.csv", tmp_path / "dirty.csv"
    assert run("estimate", "--input", gold("scene.kph"), "--output", fit, "--ra", 1,
               "--rb", 3) == 0
    assert run("detect", "--input", gold("target.kph"), "--estimate", fit, "--output", dirty) == 0
    assert run("detect", "--input", gold("scene.kph"), "--estimate", fit, "--output", clean) == 0
    img = formats.read_detection_csv(dirty)
    b, d = np.unravel_index(int(np.argmax(img.values)), img.values.shape)
    assert b == 11 and img.dopplers[d] == 0.25
    assert img.values.max() >= 10.0 * formats.read_detection_csv(clean).values.max()


def test_detect_errors(tmp_path):
    # spatial dim mismatch, single-pass estimate on a stack, change map on one pass
    assert run("detect", "--input", gold("changed.kph"), "--estimate", gold("fit.kes"),
               "--output", tmp_path / "a.csv") == cli.DATA_ERROR
    assert run("detect", "--input", gold("passes.kph"), "--estimate", gold("joint.kes"),
               "--output", tmp_path / "b.csv") == cli.DATA_ERROR
    assert run("detect", "--input", gold("scene.kph"), "--estimate", gold("fit.kes"),
               "--output", tmp_path / "c.csv", "--multipass") == cli.DATA_ERROR


def test_bench_sweep_runs(tmp_path, capsys):
    sweep = tmp_path / "sweep.cfg"
    sweep.write_text("# tiny sweep\nrow = 2 16 1 1e-4\nrow = 2 16 1 1e-6\n")
    out = tmp_path / "bench.csv"
    assert run("bench", "--sweep", sweep, "--output", out, "--trials", 2) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "p,q,n,eps,threads,trial,iterations,seconds,eta_final"
    assert len(lines) == 1 + 2 * 2
    rows = [ln.split(",") for ln in lines[1:]]
    assert all(int(r[6]) >= 1 and float(r[7]) > 0 for r in rows)
    # the tighter tolerance never iterates less on the same data
    assert int(rows[1][6]) >= int(rows[0][6]) and int(rows[3][6]) >= int(rows[2][6])
    assert "mean" in capsys.readouterr().out
