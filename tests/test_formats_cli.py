"""KPH1 / KES1 / CSV / PGM formats and the CLI's host-side behaviour against
files written by the UNMODIFIED reference CLI (tests/golden/io/, made by
oracle/gen_golden_io.py). Mirrors the reference's tests/test_formats.py and
the non-GPU half of tests/test_cli.py; the GPU subcommands are covered in
tests/test_gpu_cli.py."""

import os
import shutil

import numpy as np
import pytest

from paper_1604_03622_b200 import cli, formats
from paper_1604_03622_b200.errors import ConfigError, DataError
from paper_1604_03622_b200.filters import DetectionMap
from paper_1604_03622_b200.lrkron import KronCovEstimate
from paper_1604_03622_b200.scenes import PhaseHistory, TargetTruth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")


def gold(name):
    return os.path.join(GOLD, name)


def read_bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


def run(*args):
    return cli.main([str(a) for a in args])


# ---------------------------------------------------------------- KPH1
@pytest.mark.parametrize("name", ["scene.kph", "target.kph", "passes.kph", "changed.kph",
                                  "filtered.kph", "pfilt.kph"])
def test_kph1_read_write_reproduces_reference_bytes(name, tmp_path):
    hist = formats.read_phase_history(gold(name))
    out = tmp_path / name
    formats.write_phase_history(out, hist)
    assert read_bytes(out) == read_bytes(gold(name))


def test_kph1_fields_and_truth():
    hist = formats.read_phase_history(gold("target.kph"))
    assert (hist.p, hist.q, hist.n_passes, hist.n_bins) == (3, 16, 1, 40)
    assert hist.data.dtype == np.complex128 and hist.data.shape == (1, 40, 3, 16)
    assert [t.bin_index for t in hist.truth] == [11, 30]
    assert hist.truth[1].doppler == 0.5 and hist.truth[1].amplitude == complex(4, -2)


def test_kph1_minimal_byte_count(tmp_path):
    hist = PhaseHistory(1, 1, 1, np.zeros((1, 1, 1, 1), complex), [])
    formats.write_phase_history(tmp_path / "m.kph", hist)
    assert len(read_bytes(tmp_path / "m.kph")) == 24 + 16 + 4
    hist.truth = [TargetTruth(0, 0.25, 1 + 2j)]
    formats.write_phase_history(tmp_path / "t.kph", hist)
    assert len(read_bytes(tmp_path / "t.kph")) == 24 + 16 + 4 + 28


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XPH1" + b[4:], "bad magic"),
    (lambda b: b[:4] + b"\x02\x00" + b[6:], "unsupported format version"),
    (lambda b: b[:6] + b"\x04\x00" + b[8:], "unsupported entry encoding"),
    (lambda b: b[:8] + b"\x00\x00\x00\x00" + b[12:], "dimension fields must be positive"),
    (lambda b: b[:100], "truncated payload"),
    (lambda b: b[:10], "too short"),
    (lambda b: b + b"\x00", "trailing bytes"),
    (lambda b: b[:-1], "truncated target records"),
])
def test_kph1_malformed_files_are_data_errors(mutate, msg, tmp_path):
    bad = tmp_path / "bad.kph"
    bad.write_bytes(mutate(read_bytes(gold("target.kph"))))
    with pytest.raises(DataError, match=msg):
        formats.read_phase_history(bad)


def test_kph1_target_bin_out_of_range(tmp_path):
    b = bytearray(read_bytes(gold("target.kph")))
    tail = 24 + 40 * 3 * 16 * 16 + 4
    b[tail:tail + 4] = (40).to_bytes(4, "little")
    (tmp_path / "bad.kph").write_bytes(bytes(b))
    with pytest.raises(DataError, match="out of range"):
        formats.read_phase_history(tmp_path / "bad.kph")


# ---------------------------------------------------------------- KES1
@pytest.mark.parametrize("name", ["fit.kes", "cap.kes", "joint.kes", "changed.kes"])
def test_kes1_read_write_reproduces_reference_bytes(name, tmp_path):
    est = formats.read_estimate(gold(name))
    assert est.residuals == []
    formats.write_estimate(tmp_path / name, est)
    assert read_bytes(tmp_path / name) == read_bytes(gold(name))


def test_kes1_header_fields():
    est = formats.read_estimate(gold("cap.kes"))
    assert (est.rank_spatial, est.rank_temporal, est.iterations, est.converged) == (1, 3, 1, False)
    assert est.spatial.shape == (3, 3) and est.temporal.shape == (16, 16)
    joint = formats.read_estimate(gold("joint.kes"))
    assert joint.spatial.shape == (6, 6) and joint.temporal.shape == (8, 8)


def test_kes1_malformed(tmp_path):
    b = read_bytes(gold("fit.kes"))
    for blob, msg in [(b[:20], "too short"), (b"KXS1" + b[4:], "bad magic"),
                      (b + b"\0", "size mismatch"), (b[:-16], "size mismatch")]:
        (tmp_path / "x.kes").write_bytes(blob)
        with pytest.raises(DataError, match=msg):
            formats.read_estimate(tmp_path / "x.kes")


def test_kes1_from_estimate_object(tmp_path):
    est = KronCovEstimate(np.eye(2, dtype=complex), np.diag([1.0, 2.0, 3.0]).astype(complex),
                          1, 2, 4, [0.5], True)
    formats.write_estimate(tmp_path / "e.kes", est)
    back = formats.read_estimate(tmp_path / "e.kes")
    assert np.array_equal(back.temporal, est.temporal) and back.iterations == 4
    assert len(read_bytes(tmp_path / "e.kes")) == 32 + (4 + 9) * 16


# ---------------------------------------------------------------- CSV / PGM
@pytest.mark.parametrize("name", ["fit.kes.residuals.csv", "cap.kes.residuals.csv",
                                  "changed.kes.residuals.csv"])
def test_residual_csv_round_trip(name, tmp_path):
    res = formats.read_residuals_csv(gold(name))
    formats.write_residuals_csv(tmp_path / name, res)
    assert read_bytes(tmp_path / name) == read_bytes(gold(name))


def test_residual_csv_header_required(tmp_path):
    (tmp_path / "r.csv").write_text("1,0.5\n")
    with pytest.raises(DataError):
        formats.read_residuals_csv(tmp_path / "r.csv")


@pytest.mark.parametrize("name", ["map.csv", "map_sp.csv", "change.csv", "change_signed.csv"])
def test_detection_csv_round_trip(name, tmp_path):
    img = formats.read_detection_csv(gold(name))
    formats.write_detection_csv(tmp_path / name, img)
    assert read_bytes(tmp_path / name) == read_bytes(gold(name))


def test_detection_csv_validation(tmp_path):
    (tmp_path / "a.csv").write_text("row,f=0.0\n0,1.0\n")
    (tmp_path / "b.csv").write_text("bin,g=0.0\n0,1.0\n")
    (tmp_path / "c.csv").write_text("bin,f=0.0,f=0.5\n0,1.0\n")
    for f in ("a.csv", "b.csv", "c.csv"):
        with pytest.raises(DataError):
            formats.read_detection_csv(tmp_path / f)


def test_pgm_matches_reference_bytes(tmp_path):
    img = formats.read_detection_csv(gold("map.csv"))
    formats.write_pgm(tmp_path / "m.pgm", np.abs(img.values))
    assert read_bytes(tmp_path / "m.pgm") == read_bytes(gold("map.pgm"))


def test_pgm_zero_and_shape(tmp_path):
    formats.write_pgm(tmp_path / "z.pgm", np.zeros((2, 3)))
    b = read_bytes(tmp_path / "z.pgm")
    assert b.startswith(b"P5\n3 2\n65535\n") and b.endswith(b"\0" * 12)
    with pytest.raises(DataError):
        formats.write_pgm(tmp_path / "x.pgm", np.zeros(4))


def test_bench_csv_header(tmp_path):
    from paper_1604_03622_b200.estbench import BenchRow
    formats.write_bench_csv(tmp_path / "b.csv", [BenchRow(3, 64, 5, 1e-4, 1, 0, 7, 0.25, 0.125)])
    assert (tmp_path / "b.csv").read_text().splitlines() == [
        "p,q,n,eps,threads,trial,iterations,seconds,eta_final", "3,64,5,0.0001,1,0,7,0.25,0.125"]


# ---------------------------------------------------------------- scene configs
def test_full_config_parses():
    job = formats.parse_scene_config(
        "p = 4\nq = 32  # pulses\nn_bins = 10\nr_b = 2\nsigma2 = 0.5\ntexture = inverse_gamma\n"
        "texture_shape = 5\nkappa = 0.25\nseed = 9\nK = 3\nchange_fraction = 0.1\n"
        "shared_calibration = YES\nunit_pass_gains = 0\npass_gain_spread = 0.2\n"
        "target = 3 0.125 1.5 -2\n")
    s = job.scene
    assert (s.p, s.q, s.n_bins, s.rank_temporal, s.noise_power, s.texture) == \
        (4, 32, 10, 2, 0.5, "inverse_gamma")
    assert (s.texture_shape, s.kappa, s.seed) == (5.0, 0.25, 9)
    assert (job.n_passes, job.change_fraction, job.shared_calibration, job.unit_pass_gains,
            job.pass_gain_spread) == (3, 0.1, True, False, 0.2)
    assert job.targets == [(3, 0.125, complex(1.5, -2))]


def test_config_defaults():
    job = formats.parse_scene_config("p = 2\nq = 8\nn_bins = 4\nr_b = 1\n")
    assert (job.scene.noise_power, job.scene.texture, job.scene.seed, job.n_passes) == \
        (1e-2, "constant", 0, 1)
    assert (job.shared_calibration, job.unit_pass_gains, job.pass_gain_spread) == (False, False, 0.5)


@pytest.mark.parametrize("text,line", [
    ("p = 2\nwhat\n", 2), ("p = 2\nq =\n", 2), ("p = x\n", 1), ("sigma2 = abc\n", 1),
    ("\n\nshared_calibration = maybe\n", 3), ("target = 1 2 3\n", 1),
    ("target = a 0.1 1 1\n", 1), ("colour = red\n", 1)])
def test_config_errors_carry_line_numbers(text, line):
    with pytest.raises(ConfigError) as e:
        formats.parse_scene_config(text)
    assert e.value.line == line and str(e.value).startswith(f"line {line}:")


def test_config_semantic_errors():
    with pytest.raises(DataError, match="required key 'n_bins'"):
        formats.parse_scene_config("p = 2\nq = 8\nr_b = 1\n")
    for extra in ("K = 0\n", "target = 4 0.1 1 1\n", "texture = weird\n"):
        with pytest.raises(DataError):
            formats.parse_scene_config("p = 2\nq = 8\nn_bins = 4\nr_b = 1\n" + extra)


# ---------------------------------------------------------------- CLI (host side)
@pytest.mark.parametrize("cfg,out,extra", [
    ("scene.cfg", "scene.kph", []), ("target.cfg", "target.kph", []),
    ("passes.cfg", "passes.kph", []), ("changed.cfg", "changed.kph", []),
    ("scene.cfg", "seed99.kph", ["--seed", 99])])
def test_simulate_matches_reference_cli_bytes(cfg, out, extra, tmp_path):
    assert run("simulate", "--config", gold(cfg), "--output", tmp_path / out, *extra) == 0
    assert read_bytes(tmp_path / out) == read_bytes(gold(out))


def test_simulate_bad_config_is_data_error(tmp_path):
    (tmp_path / "c.cfg").write_text("p = 2\nwhat\n")
    assert run("simulate", "--config", tmp_path / "c.cfg", "--output", tmp_path / "x") == \
        cli.DATA_ERROR


def test_usage_errors(tmp_path):
    assert run() == cli.USAGE_ERROR
    assert run("estimate", "--input", "x") == cli.USAGE_ERROR
    assert run("simulate", "--config", tmp_path / "c", "--output", tmp_path / "o",
               "--threads", 0) == cli.USAGE_ERROR
    assert run("detect", "--input", "a", "--estimate", "b", "--output", "c",
               "--kind", "optimal") == cli.USAGE_ERROR


def test_thread_env_fallback(tmp_path, monkeypatch):
    shutil.copy(gold("scene.cfg"), tmp_path / "s.cfg")
    monkeypatch.setenv("KRONSTAP_THREADS", "3")
    assert run("simulate", "--config", tmp_path / "s.cfg", "--output", tmp_path / "a.kph") == 0
    monkeypatch.setenv("KRONSTAP_THREADS", "lots")
    assert run("simulate", "--config", tmp_path / "s.cfg", "--output", tmp_path / "b.kph") == \
        cli.USAGE_ERROR
    assert run("simulate", "--config", tmp_path / "s.cfg", "--output", tmp_path / "c.kph",
               "--threads", 2) == 0


def test_missing_files_are_data_errors(tmp_path):
    assert run("estimate", "--input", tmp_path / "nope.kph", "--output", tmp_path / "f.kes",
               "--ra", 1, "--rb", 2) == cli.DATA_ERROR
    assert run("filter", "--input", tmp_path / "nope.kph", "--estimate", gold("fit.kes"),
               "--output", tmp_path / "o.kph") == cli.DATA_ERROR


def test_bench_sweep_validation(tmp_path):
    out = tmp_path / "b.csv"
    sweep = tmp_path / "s.cfg"
    sweep.write_text("row = 2 16 1 1e-4\n")
    assert run("bench", "--output", out) == cli.DATA_ERROR
    assert run("bench", "--output", out, "--sweep", sweep, "--default-sweep") == cli.DATA_ERROR
    for text in ("row = 2 16 1\n", "# nothing\n", "col = 1 2 3 4\n", "row 1 2 3 4\n",
                 "row = a 16 1 1e-4\n"):
        sweep.write_text(text)
        assert run("bench", "--sweep", sweep, "--output", out) == cli.DATA_ERROR


def test_default_sweep_grid():
    from paper_1604_03622_b200 import estbench
    sw = estbench.default_sweep()
    assert len(sw) == 2 * 5 * 2 + 1 and sw[-1] == (3, 1024, 4, 1e-4)


def test_training_data_matches_reference_generator():
    """The estimator-bench snapshots equal the reference's (`src/bench.py:61-72`)
    bit for bit: pinned by a fixture hash."""
    import hashlib
    from paper_1604_03622_b200 import estbench
    x = estbench.training_snapshots(3, 16, 5, (0, 3, 16, 1))
    want = open(gold("bench_snapshots.sha256")).read().split()[0]
    assert hashlib.sha256(x.tobytes()).hexdigest() == want
