"""Estimator wall-clock sweep behind `kronstap bench` (`src/bench.py:1-137`).

Same sweep grid, seeded training data and row records as the reference; the
timed call is `lr_kron_estimate(scm, 1, q)` on the device (the covariance is
formed outside the timed region and kept in HBM), bracketed by device
synchronisation, best of a size-dependent number of repeats. `threads` is
recorded as given (no host pool on this path).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DataError

DEFAULT_P = (3, 6)
DEFAULT_Q = (64, 128, 256, 512, 1024)
DEFAULT_EPS = (1e-4, 1e-6)
SPEEDUP_CONFIG = (3, 1024, 4, 1e-4)
NOISE_POWER = 1.0  # 0 dB against unit clutter (`src/bench.py:55-58`)


@dataclass
class BenchRow:
    p: int
    q: int
    n: int
    eps: float
    threads: int
    trial: int
    iterations: int
    seconds: float
    eta_final: float


def default_sweep():
    """(p, q, 1, eps) over the default grid plus the thread-comparison row."""
    rows = [(p, q, 1, eps) for p in DEFAULT_P for q in DEFAULT_Q for eps in DEFAULT_EPS]
    return rows + [SPEEDUP_CONFIG]


def load_sweep(path):
    """`row = p q threads eps` lines, `#` comments (`src/cli.py:243-265`)."""
    rows = []
    with open(path) as fh:
        text = fh.read()
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, eq, value = line.partition("=")
        if not eq:
            raise ConfigError(lineno, f"expected 'row = p q threads eps', got {raw.strip()!r}")
        if key.strip() != "row":
            raise ConfigError(lineno, f"unknown key {key.strip()!r}")
        f = value.split()
        if len(f) != 4:
            raise ConfigError(lineno, "row takes exactly: p q threads eps")
        try:
            rows.append((int(f[0]), int(f[1]), int(f[2]), float(f[3])))
        except ValueError:
            raise ConfigError(lineno, f"bad row fields {value.strip()!r}") from None
    if not rows:
        raise DataError("sweep file lists no rows")
    return rows


def training_snapshots(p, q, n, key):
    """Rank-one spatial x white temporal + unit noise, keyed substream
    (seed, p, q, trial) (`src/bench.py:61-72`)."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=key[0], spawn_key=key[1:]))
    g = rng.standard_normal(2 * p)
    direction = (g[0::2] + 1j * g[1::2]) / np.sqrt(2.0)
    g = rng.standard_normal((n, 2 * q))
    pulses = (g[:, 0::2] + 1j * g[:, 1::2]) / np.sqrt(2.0)
    # einsum, not broadcasting: its complex product rounds like the reference's
    snaps = np.einsum("i,mj->mij", direction, pulses).reshape(n, p * q)
    g = rng.standard_normal((n, 2 * p * q))
    return snaps + (g[:, 0::2] + 1j * g[:, 1::2]) * np.sqrt(NOISE_POWER / 2.0)


def repeats_for(q):
    return 6 if q <= 128 else 4 if q <= 256 else 3 if q <= 512 else 2


def run_bench(sweep, trials=10, n=5, seed=0, max_iter=100, repeats=None, progress=None):
    """One BenchRow per (row, trial); trials outermost (`src/bench.py:89-127`)."""
    import torch
    from . import _native as nat
    from .lrkron import lr_kron_estimate, sample_covariance
    rows = []
    for trial in range(trials):
        cache = {}
        for p, q, threads, eps in sweep:
            if (p, q) not in cache:
                x = nat.to_device(training_snapshots(p, q, n, (seed, p, q, trial)))
                cache[p, q] = sample_covariance(x, p, q)
            scm = cache[p, q]
            best, est = math.inf, None
            for _ in range(max(repeats or repeats_for(q), 1)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                est = lr_kron_estimate(scm, 1, q, tol=eps, max_iter=max_iter)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            rows.append(BenchRow(p, q, n, eps, threads, trial, est.iterations, best,
                                 est.residuals[-1]))
        if progress is not None:
            progress(trial, trials)
    return rows


def mean_seconds(rows, p, q, threads, eps):
    ts = [r.seconds for r in rows if (r.p, r.q, r.threads, r.eps) == (p, q, threads, eps)]
    if not ts:
        raise ValueError(f"no rows for p={p} q={q} threads={threads} eps={eps}")
    return sum(ts) / len(ts)
