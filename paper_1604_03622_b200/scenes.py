"""Seeded synthetic phase-history scenes (host-side input generator).

Restates the reference simulator (`src/simulate.py`, kronstap) so the
bench and the parity tests can build the SAME cubes the reference would,
byte for byte, without the reference being present on the GPU box.
This is input generation on the CPU, not part of the measured path
(SURVEY.md §2 marks the simulator out of scope for the GPU).

Randomness uses keyed numpy SeedSequence substreams exactly as the
reference does (`src/simulate.py:115-116`): stream (0,) scene profile,
(1, m) bin m's shared speckle/texture, (2, m, k) pass k of bin m,
(3, k) per-pass calibration, (4,) changed-bin picks.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import DataError, DimensionError


@dataclass(frozen=True)
class SceneConfig:
    """Field-for-field mirror of `src/simulate.py:30-57`."""

    p: int
    q: int
    n_bins: int
    rank_temporal: int
    noise_power: float = 1e-2
    texture: str = "constant"
    texture_shape: float = 3.0
    calibration_phase: float = 0.1
    kappa: float = 0.5
    seed: int = 0

    def validate(self):
        if min(self.p, self.q, self.n_bins) < 1:
            raise DataError("scene dimensions must be positive")
        if not 1 <= self.rank_temporal <= self.q:
            raise DataError("temporal rank out of range")
        if self.noise_power < 0:
            raise DataError("noise power must be non-negative")
        if self.texture not in ("constant", "inverse_gamma"):
            raise DataError(f"unknown texture law {self.texture!r}")
        if self.texture == "inverse_gamma" and self.texture_shape <= 1.0:
            raise DataError("inverse_gamma texture needs shape > 1")


@dataclass(frozen=True)
class TargetTruth:
    bin_index: int
    doppler: float
    amplitude: complex


@dataclass(eq=False)
class PhaseHistory:
    """(passes, bins, channels, pulses) cube -- `src/simulate.py:69-81`."""

    p: int
    q: int
    n_passes: int
    data: np.ndarray
    truth: list = field(default_factory=list)

    @property
    def n_bins(self):
        return self.data.shape[1]


def _rng(seed, *key):
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=key))


def _cn(rng, count):
    # interleaved draws: even -> real, odd -> imaginary (src/simulate.py:119-121)
    z = rng.standard_normal(2 * count)
    return (z[0::2] + 1j * z[1::2]) / math.sqrt(2.0)


def _model(cfg):
    """Calibration, orthonormal temporal profiles, geometric weights
    normalised to trace q (`src/simulate.py:124-144`)."""
    cfg.validate()
    rng = _rng(cfg.seed, 0)
    r = cfg.rank_temporal
    jitter = rng.uniform(0.0, 1.0, r)
    cal = np.exp(1j * rng.uniform(-cfg.calibration_phase, cfg.calibration_phase, cfg.p))
    freqs = (np.arange(r) + 0.3 * jitter) / (2.0 * cfg.q)
    ramps = np.exp(2j * np.pi * np.outer(np.arange(cfg.q), freqs))
    prof, _ = np.linalg.qr(ramps / math.sqrt(cfg.q))
    w = 0.5 ** np.arange(r)
    w *= cfg.q / w.sum()
    return cal, prof, w


def total_covariance(cfg):
    """Exact snapshot covariance of a scene config: (h h^H) kron B + noise I
    (SceneModel.total_covariance, src/simulate.py:93-105), the sigma that the
    SINR acceptance criteria evaluate against (host ground truth, like the
    simulator itself)."""
    cal, prof, w = _model(cfg)
    b = (prof * w) @ prof.conj().T
    b = (b + b.conj().T) / 2.0
    full = np.kron(np.outer(cal, cal.conj()), b)
    full += cfg.noise_power * np.eye(full.shape[0])
    return full


def _texture(rng, cfg):
    if cfg.texture == "constant":
        return 1.0
    g = rng.gamma(cfg.texture_shape, 1.0 / (cfg.texture_shape - 1.0))
    return 1.0 / math.sqrt(g)


def _pass_cal(cfg, k):
    rng = _rng(cfg.seed, 3, k)
    return np.exp(1j * rng.uniform(-cfg.calibration_phase, cfg.calibration_phase, cfg.p))


def generate(cfg, n_passes=1, change_fraction=0.0, shared_calibration=True,
             unit_gains=True, gain_spread=0.0):
    """Texture x speckle x calibration + noise (`src/simulate.py:155-197`).

    Defaults give `gen_clutter`; `gen_multipass` passes its own flags.
    """
    if n_passes < 1:
        raise DimensionError("need at least one pass")
    if not 0.0 <= change_fraction <= 1.0:
        raise DataError("change fraction must be in [0, 1]")
    cal, prof, w = _model(cfg)
    p, q, n = cfg.p, cfg.q, cfg.n_bins
    r = cfg.rank_temporal
    sw = np.sqrt(w)
    namp = math.sqrt(cfg.noise_power)
    cals = [cal] * n_passes if shared_calibration else [_pass_cal(cfg, k) for k in range(n_passes)]
    changed = np.zeros(n, dtype=bool)
    n_changed = int(round(change_fraction * n))
    if n_changed > 0:
        changed[_rng(cfg.seed, 4).choice(n, size=n_changed, replace=False)] = True
    out = np.empty((n_passes, n, p, q), dtype=np.complex128)
    for m in range(n):
        brng = _rng(cfg.seed, 1, m)
        z = _cn(brng, r)
        tau = _texture(brng, cfg)
        speck = prof @ (sw * z)
        for k in range(n_passes):
            prng = _rng(cfg.seed, 2, m, k)
            zeta = _cn(prng, 1)[0]
            gain = 1.0 if unit_gains else 1.0 + gain_spread * zeta
            sk = prof @ (sw * _cn(prng, r)) if changed[m] else speck
            noise = _cn(prng, p * q).reshape(p, q)
            out[k, m] = (tau * gain) * np.outer(cals[k], sk)
            out[k, m] += namp * noise
    return PhaseHistory(p, q, n_passes, out)


def gen_clutter(cfg):
    return generate(cfg, 1)


def gen_multipass(cfg, n_passes, change_fraction=0.0, shared_calibration=False,
                  unit_gains=False, gain_spread=0.5):
    return generate(cfg, n_passes, change_fraction, shared_calibration,
                    unit_gains, gain_spread)


def inject_target(history, bin_index, doppler, amplitude, pass_index=0, kappa=None):
    """Additive unit-norm mover (`src/simulate.py:229-250`, steering from
    `src/filters.py:44-55`)."""
    if not 0 <= bin_index < history.n_bins:
        raise DimensionError(f"bin {bin_index} out of range")
    if not 0 <= pass_index < history.n_passes:
        raise DimensionError(f"pass {pass_index} out of range")
    kap = 0.5 if kappa is None else kappa
    sp = np.exp(2j * np.pi * kap * doppler * np.arange(history.p))
    tp = np.exp(2j * np.pi * doppler * np.arange(history.q)) / np.sqrt(history.q)
    sig = np.outer(sp, tp)
    sig /= np.linalg.norm(sp) * np.linalg.norm(tp)
    data = history.data.copy()
    data[pass_index, bin_index] += amplitude * sig
    truth = list(history.truth) + [TargetTruth(int(bin_index), float(doppler), complex(amplitude))]
    return PhaseHistory(history.p, history.q, history.n_passes, data, truth)


def bench_scene(p, q, n_bins, seed=17, movers=8, n_passes=1, rank_temporal=3,
                noise_power=1e-2, amplitude=10.0):
    """The SURVEY.md §8d bench scene: reference SceneConfig defaults,
    `movers` targets at seeded bins with on-grid Dopplers d/q."""
    cfg = SceneConfig(p=p, q=q, n_bins=n_bins, rank_temporal=rank_temporal,
                      noise_power=noise_power, seed=seed)
    hist = generate(cfg, 1) if n_passes == 1 else gen_multipass(cfg, n_passes)
    rng = np.random.default_rng(seed + 1000)
    for _ in range(movers):
        b = int(rng.integers(0, n_bins))
        d = int(rng.integers(0, q)) / q
        k = int(rng.integers(0, n_passes))
        hist = inject_target(hist, b, d, amplitude, pass_index=k)
    return hist
