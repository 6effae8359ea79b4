"""Command-line driver on the B200 path.

Same subcommands, options, outputs and exit codes as the reference
`kronstap` CLI (`src/cli.py:1-317`): 0 success, 1 usage, 2 malformed or
mismatched data (any KronStapError or OSError), 3 estimator hit max-iter.

    python -m paper_1604_03622_b200.cli estimate --input s.kph --output f.kes --ra 1 --rb 3

Data flow: a KPH1 payload is read once into pinned host memory and copied
to HBM in one transfer (`formats.load_cube`); the covariance, the
estimator, the filter and the detection map stay on the device; only the
outputs (factors, filtered cube, map) come back for writing. `simulate`
runs the host scene generator (`scenes.py`, bit-exact with the reference).
`--threads` / KRONSTAP_THREADS are validated like the reference's and
otherwise ignored: the reference guarantees thread-count-invariant output,
and the GPU path has no host worker pool.
"""

from __future__ import annotations

import argparse
import os
import sys
from dataclasses import replace

import numpy as np

from . import formats
from .errors import DataError, KronStapError

USAGE_ERROR = 1
DATA_ERROR = 2
NO_CONVERGENCE = 3


class _Parser(argparse.ArgumentParser):
    """Usage problems exit with status 1 (`src/cli.py:34-40`)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(USAGE_ERROR)


def build_parser():
    """Subcommands and options of `src/cli.py:48-110`."""
    parser = _Parser(prog="kronstap", description="Kronecker-structured STAP toolkit (B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    spec = {
        "simulate": ("generate a clutter cube", cmd_simulate, [
            ("--config", dict(required=True, help="scene config file")),
            ("--output", dict(required=True, help="output .kph file")),
            ("--seed", dict(type=int, default=None, help="override the config seed"))]),
        "estimate": ("fit the Kronecker covariance", cmd_estimate, [
            ("--input", dict(required=True, help="input .kph file")),
            ("--output", dict(required=True, help="output estimate file")),
            ("--ra", dict(type=int, required=True, help="spatial rank")),
            ("--rb", dict(type=int, required=True, help="temporal rank")),
            ("--eps", dict(type=float, default=1e-4, help="residual stall tolerance")),
            ("--max-iter", dict(type=int, default=100))]),
        "filter": ("apply a clutter filter to a cube", cmd_filter, [
            ("--input", dict(required=True)), ("--estimate", dict(required=True)),
            ("--output", dict(required=True)),
            ("--kind", dict(choices=("kron", "classical"), default="kron")),
            ("--no-temporal-projection", dict(action="store_true",
                                              help="spatial-only cancelation"))]),
        "detect": ("form a detection or change map", cmd_detect, [
            ("--input", dict(required=True)), ("--estimate", dict(required=True)),
            ("--output", dict(required=True, help="output CSV path")),
            ("--kind", dict(choices=("kron", "classical"), default="kron")),
            ("--grid-doppler", dict(type=int, default=64)),
            ("--grid-spatial", dict(type=int, default=16)),
            ("--multipass", dict(action="store_true",
                                 help="two-pass change map instead of a detection map")),
            ("--signed", dict(action="store_true", help="keep the sign of the change map")),
            ("--no-temporal-projection", dict(action="store_true")),
            ("--pgm", dict(default=None, help="also write a PGM image"))]),
        "bench": ("time the estimator over a sweep", cmd_bench, [
            ("--output", dict(required=True, help="output CSV path")),
            ("--sweep", dict(default=None, help="sweep file with 'row = p q threads eps' lines")),
            ("--default-sweep", dict(action="store_true", help="run the built-in grid")),
            ("--trials", dict(type=int, default=10)),
            ("--n", dict(type=int, default=5, dest="n_train", help="training snapshots per trial")),
            ("--seed", dict(type=int, default=0))]),
    }
    for name, (helptext, func, opts) in spec.items():
        sp = sub.add_parser(name, help=helptext)
        for flag, kw in opts:
            sp.add_argument(flag, **kw)
        sp.add_argument("--threads", type=int, default=None,
                        help="accepted for compatibility (default: KRONSTAP_THREADS or 1)")
        sp.set_defaults(func=func)
    return parser


# ---------------------------------------------------------------- subcommands
def cmd_simulate(args):
    """`src/cli.py:113-134` over the host scene generator."""
    from .scenes import gen_clutter, gen_multipass, inject_target
    job = formats.load_scene_config(args.config)
    scene = job.scene if args.seed is None else replace(job.scene, seed=args.seed)
    if job.n_passes == 1:
        hist = gen_clutter(scene)
    else:
        hist = gen_multipass(scene, job.n_passes, change_fraction=job.change_fraction,
                             shared_calibration=job.shared_calibration,
                             unit_gains=job.unit_pass_gains, gain_spread=job.pass_gain_spread)
    for b, f, amp in job.targets:
        hist = inject_target(hist, b, f, amp, kappa=scene.kappa)
    formats.write_phase_history(args.output, hist)
    print(f"wrote {args.output}: {hist.n_passes} pass(es), {hist.n_bins} bins of "
          f"{hist.p}x{hist.q}, {len(hist.truth)} target(s)")
    return 0


def _snapshots(hist):
    """(n, sdim * q) snapshot matrix on the device; passes stacked first
    (`src/cli.py:137-143`)."""
    from .layout import cube_to_snapshots
    from .multipass import stack_passes
    if hist.n_passes == 1:
        return cube_to_snapshots(hist.data[0]), hist.p, hist.q
    st = stack_passes(hist)
    return st.data.reshape(st.n_bins, -1), st.stacked_channels, st.q


def cmd_estimate(args):
    """`src/cli.py:146-157`."""
    from .lrkron import lr_kron_estimate, sample_covariance
    hist, _ = formats.load_cube(args.input)
    snaps, sdim, q = _snapshots(hist)
    est = lr_kron_estimate(sample_covariance(snaps, sdim, q), args.ra, args.rb, tol=args.eps,
                           max_iter=args.max_iter)
    formats.write_estimate(args.output, est)
    formats.write_residuals_csv(args.output + ".residuals.csv", est.residuals)
    state = "converged" if est.converged else "hit max-iter"
    print(f"wrote {args.output}: {est.iterations} iteration(s), "
          f"final residual {est.residuals[-1]:.3e}, {state}")
    return 0 if est.converged else NO_CONVERGENCE


def _filter_for(hist, est, kind, drop_temporal):
    """Projection filter matching the cube; stacked when the estimate spans
    all passes (`src/cli.py:160-174`)."""
    from .filters import build_filter
    sdim = est.spatial.shape[0]
    stacked = hist.n_passes > 1 and sdim == hist.n_passes * hist.p
    if not stacked and sdim != hist.p:
        raise DataError(f"estimate spatial dim {sdim} matches neither p={hist.p} "
                        f"nor stacked {hist.n_passes * hist.p}")
    if est.temporal.shape[0] != hist.q:
        raise DataError(f"estimate temporal dim {est.temporal.shape[0]} "
                        f"does not match q={hist.q}")
    return build_filter(kind, estimate=est, drop_temporal=drop_temporal), stacked


def cmd_filter(args):
    """`src/cli.py:177-206`: every bin of every pass through kst_filter."""
    import torch
    from .multipass import stack_passes, unstack_passes
    from .scenes import PhaseHistory
    hist, _ = formats.load_cube(args.input)
    est = formats.read_estimate(args.estimate)
    filt, stacked = _filter_for(hist, est, args.kind, args.no_temporal_projection)
    if stacked:
        st = stack_passes(hist)
        st.data = filt.apply_cube(st.data)
        out = unstack_passes(st).data
    else:
        out = torch.stack([filt.apply_cube(hist.data[k]) for k in range(hist.n_passes)])
    formats.write_phase_history(args.output,
                                PhaseHistory(hist.p, hist.q, hist.n_passes, out, list(hist.truth)))
    print(f"wrote {args.output}: filtered with {args.kind}")
    return 0


def cmd_detect(args):
    """`src/cli.py:209-240`: detection map, or the two-pass change map."""
    from .filters import detection_image, make_doppler_grid, make_spatial_grid, set_detect_precision
    from .multipass import change_detect, pass_images, stack_passes
    # the CLI writes the reference's map files: FP64 detection, so the CSV
    # matches what the reference CLI writes to ~1e-12 (the library default,
    # FP32 detection, holds the SURVEY.md §8c comparator)
    set_detect_precision("f64")
    hist, _ = formats.load_cube(args.input)
    est = formats.read_estimate(args.estimate)
    dopplers = make_doppler_grid(args.grid_doppler)
    if args.multipass:
        if hist.n_passes != 2:
            raise DataError(f"change detection needs exactly 2 passes, got {hist.n_passes}")
        filt, stacked = _filter_for(hist, est, args.kind, args.no_temporal_projection)
        if not stacked:
            raise DataError("change detection needs a stacked estimate")
        a, b = pass_images(filt, stack_passes(hist), dopplers, args.grid_spatial)
        image, label = change_detect(a, b, signed=args.signed), "change map"
    else:
        if hist.n_passes != 1:
            raise DataError("multipass input needs --multipass")
        filt, _ = _filter_for(hist, est, args.kind, args.no_temporal_projection)
        grid = make_spatial_grid(hist.p, args.grid_spatial)
        image = detection_image(filt, hist.data[0], dopplers, grid)
        label = "detection map"
    values = formats._host_array(image.values)
    image.values = values
    formats.write_detection_csv(args.output, image)
    if args.pgm is not None:
        formats.write_pgm(args.pgm, np.abs(values))
    peak = float(np.max(np.abs(values))) if values.size else 0.0
    print(f"wrote {args.output}: {label}, peak magnitude {peak:.4e}")
    return 0


def cmd_bench(args):
    """`src/cli.py:243-285` over `estbench` (the estimator on the device)."""
    from . import estbench
    if args.default_sweep == (args.sweep is not None):
        raise DataError("pass exactly one of --sweep or --default-sweep")
    sweep = estbench.default_sweep() if args.default_sweep else estbench.load_sweep(args.sweep)

    def progress(trial, trials):
        print(f"completed trial {trial + 1}/{trials} across {len(sweep)} rows")

    rows = estbench.run_bench(sweep, trials=args.trials, n=args.n_train, seed=args.seed,
                              progress=progress)
    formats.write_bench_csv(args.output, rows)
    for p, q, threads, eps in sweep:
        mean = estbench.mean_seconds(rows, p, q, threads, eps)
        print(f"p={p} q={q} threads={threads} eps={eps:g}: "
              f"mean {mean:.4f} s over {args.trials} trial(s)")
    print(f"wrote {args.output}")
    return 0


def _threads(args):
    """--threads, else KRONSTAP_THREADS, else 1; None when invalid."""
    if args.threads is not None:
        n = args.threads
    else:
        env = os.environ.get("KRONSTAP_THREADS", "1")
        try:
            n = int(env)
        except ValueError:
            sys.stderr.write(f"kronstap: bad KRONSTAP_THREADS value {env!r}\n")
            return None
    if n < 1:
        sys.stderr.write(f"kronstap: thread count must be >= 1, got {n}\n")
        return None
    return n


def main(argv=None):
    """Exit status as `src/cli.py:288-313`."""
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    if _threads(args) is None:
        return USAGE_ERROR
    try:
        return args.func(args)
    except (KronStapError, OSError) as exc:
        sys.stderr.write(f"kronstap: error: {exc}\n")
        return DATA_ERROR


def entry():
    sys.exit(main(sys.argv[1:]))


if __name__ == "__main__":
    entry()
