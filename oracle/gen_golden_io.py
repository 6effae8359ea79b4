"""Generate tests/golden/io/ by running the UNMODIFIED reference CLI here.

TEST INFRASTRUCTURE (build container only; /root/reference is absent on the
GPU box):

    python oracle/gen_golden_io.py

Runs `kronstap.cli.main` (imported from /root/reference/pkg/src, nothing
copied) on small scene configs and keeps every file it writes: KPH1 cubes
(simulate, filter), KES1 estimates + residual CSVs (estimate), detection /
change CSVs and a PGM (detect). The tests check that this package's readers
and writers reproduce these bytes and that its GPU subcommands reproduce
their values.
"""

import os
import shutil
import sys
import tempfile

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "io")

CONFIGS = {
    "scene.cfg": "p = 3\nq = 16\nn_bins = 40\nr_b = 3\nsigma2 = 0.01\nseed = 17\n",
    "target.cfg": "p = 3\nq = 16\nn_bins = 40\nr_b = 3\nsigma2 = 0.01\nseed = 17\n"
                  "target = 11 0.25 10 0\ntarget = 30 0.5 4 -2\n",
    "passes.cfg": "p = 3\nq = 8\nn_bins = 24\nr_b = 2\nsigma2 = 0.0\nseed = 18\nK = 2\n"
                  "shared_calibration = yes\nunit_pass_gains = yes\n",
    "changed.cfg": "p = 2\nq = 8\nn_bins = 30\nr_b = 2\nsigma2 = 0.01\nseed = 5\nK = 2\n"
                   "change_fraction = 0.2\ntexture = inverse_gamma\ntexture_shape = 4\n",
}

RUNS = [
    ["simulate", "--config", "scene.cfg", "--output", "scene.kph"],
    ["simulate", "--config", "target.cfg", "--output", "target.kph"],
    ["simulate", "--config", "passes.cfg", "--output", "passes.kph"],
    ["simulate", "--config", "changed.cfg", "--output", "changed.kph"],
    ["simulate", "--config", "scene.cfg", "--output", "seed99.kph", "--seed", "99"],
    ["estimate", "--input", "scene.kph", "--output", "fit.kes", "--ra", "1", "--rb", "3"],
    ["estimate", "--input", "scene.kph", "--output", "cap.kes", "--ra", "1", "--rb", "3",
     "--eps", "1e-14", "--max-iter", "1"],
    ["estimate", "--input", "passes.kph", "--output", "joint.kes", "--ra", "2", "--rb", "2"],
    ["estimate", "--input", "changed.kph", "--output", "changed.kes", "--ra", "2", "--rb", "2"],
    ["filter", "--input", "scene.kph", "--estimate", "fit.kes", "--output", "filtered.kph"],
    ["filter", "--input", "scene.kph", "--estimate", "fit.kes", "--output", "classical.kph",
     "--kind", "classical"],
    ["filter", "--input", "passes.kph", "--estimate", "joint.kes", "--output", "pfilt.kph"],
    ["detect", "--input", "target.kph", "--estimate", "fit.kes", "--output", "map.csv",
     "--pgm", "map.pgm"],
    ["detect", "--input", "target.kph", "--estimate", "fit.kes", "--output", "map_sp.csv",
     "--grid-doppler", "40", "--grid-spatial", "8", "--no-temporal-projection"],
    ["detect", "--input", "passes.kph", "--estimate", "joint.kes", "--output", "change.csv",
     "--multipass"],
    ["detect", "--input", "changed.kph", "--estimate", "changed.kes", "--output",
     "change_signed.csv", "--multipass", "--signed", "--grid-doppler", "16"],
]


def main():
    sys.path.insert(0, REF)
    from kronstap.cli import main as ref_main
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in CONFIGS.items():
            with open(os.path.join(tmp, name), "w") as fh:
                fh.write(text)
        cwd = os.getcwd()
        os.chdir(tmp)
        try:
            codes = [ref_main(list(r)) for r in RUNS]
        finally:
            os.chdir(cwd)
        print("exit codes", codes)
        for f in sorted(os.listdir(tmp)):
            shutil.copy(os.path.join(tmp, f), os.path.join(OUT, f))
    # estimator-bench training snapshots: capture the argument the reference
    # passes to sample_covariance (`src/bench.py:61-72`) and store its hash
    import hashlib
    from kronstap import bench as ref_bench
    seen = []
    real = ref_bench.sample_covariance
    ref_bench.sample_covariance = lambda x, p, q: seen.append(x) or real(x, p, q)
    try:
        ref_bench._training_covariance(3, 16, 5, (0, 3, 16, 1))
    finally:
        ref_bench.sample_covariance = real
    with open(os.path.join(OUT, "bench_snapshots.sha256"), "w") as fh:
        fh.write(hashlib.sha256(seen[0].tobytes()).hexdigest() + "  p=3 q=16 n=5 key=(0,3,16,1)\n")
    with open(os.path.join(OUT, "exit_codes.txt"), "w") as fh:
        for r, c in zip(RUNS, codes):
            fh.write(f"{c} {' '.join(r)}\n")


if __name__ == "__main__":
    main()
