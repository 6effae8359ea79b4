"""On-disk formats either side of the hot path.

Byte-compatible with the reference's `src/formats.py`:

* KPH1 phase-history cubes (`src/formats.py:3-13,39-92`): a 24-byte
  little-endian header (magic, version u16, flags u16 = 8 for complex128,
  p, q, K, n_bins u32), the (K, n_bins, p, q) `<c16` payload, then
  n_targets u32 and 28-byte target records (bin u32, doppler, re, im f64).
* KES1 estimates (`src/formats.py:95-135`): 32-byte header (magic, version,
  flags, sdim, q, rank_spatial, rank_temporal, iterations, converged u32),
  then the spatial (sdim x sdim) and temporal (q x q) factors as `<c16`.
* Residual / detection CSVs with exact float reprs, 16-bit PGM
  (`src/formats.py:138-208`), and the `key = value` scene configs
  (`src/formats.py:214-330`).

B200 side: the payload is exactly the layout the kernels consume
((K, n_bins, p, q) complex128, C order), so `load_cube` streams it from the
file straight into pinned host memory (one `readinto`, no intermediate
bytes object) and issues a single host->device copy; `write_phase_history`
accepts device tensors (one device->host copy into pinned memory).
Headers are numpy structured dtypes; every validation of the reference
reader is kept, with the same exception classes and messages.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import ConfigError, DataError
from .scenes import PhaseHistory, SceneConfig, TargetTruth

PH_MAGIC = b"KPH1"
EST_MAGIC = b"KES1"
FORMAT_VERSION = 1
FLAG_COMPLEX128 = 8

PH_HEADER = np.dtype([("magic", "S4"), ("version", "<u2"), ("flags", "<u2"), ("p", "<u4"),
                      ("q", "<u4"), ("K", "<u4"), ("n_bins", "<u4")])
TARGET_RECORD = np.dtype([("bin", "<u4"), ("doppler", "<f8"), ("re", "<f8"), ("im", "<f8")])
EST_HEADER = np.dtype([("magic", "S4"), ("version", "<u2"), ("flags", "<u2"), ("sdim", "<u4"),
                       ("q", "<u4"), ("rank_spatial", "<u4"), ("rank_temporal", "<u4"),
                       ("iterations", "<u4"), ("converged", "<u4")])
_ENTRY = np.dtype("<c16")
_COUNT = np.dtype("<u4")
assert PH_HEADER.itemsize == 24 and TARGET_RECORD.itemsize == 28 and EST_HEADER.itemsize == 32


def _host_array(data):
    """numpy view of array-likes and (device) torch tensors."""
    if hasattr(data, "detach") and hasattr(data, "is_cuda"):
        t = data.detach()
        if t.is_cuda:
            import torch
            host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            host.copy_(t)
            t = host
        return t.numpy()
    return np.asarray(data)


def _check_format(magic, version, flags, want):
    if magic != want:
        raise DataError(f"bad magic {magic!r}, expected {want!r}")
    if version != FORMAT_VERSION:
        raise DataError(f"unsupported format version {version}")
    if flags != FLAG_COMPLEX128:
        raise DataError(f"unsupported entry encoding flags {flags}")


# ---------------------------------------------------------------- KPH1
def write_phase_history(path, history):
    """Serialise a PhaseHistory (host or device data); the bytes depend only
    on the content (`src/formats.py:39-52`)."""
    data = np.ascontiguousarray(_host_array(history.data), dtype=_ENTRY)
    if data.ndim != 4:
        raise DataError(f"phase history must be (K, n_bins, p, q), got {data.shape}")
    k, n_bins, p, q = data.shape
    hdr = np.array([(PH_MAGIC, FORMAT_VERSION, FLAG_COMPLEX128, p, q, k, n_bins)],
                   dtype=PH_HEADER)
    recs = np.array([(t.bin_index, t.doppler, complex(t.amplitude).real,
                      complex(t.amplitude).imag) for t in history.truth], dtype=TARGET_RECORD)
    with open(path, "wb") as fh:
        fh.write(hdr.tobytes())
        fh.write(memoryview(data).cast("B"))
        fh.write(np.array([len(recs)], dtype=_COUNT).tobytes())
        fh.write(recs.tobytes())


def _ph_layout(fh, size):
    """Validate a KPH1 file's framing; returns (header record, payload
    offset, entry count, target records)."""
    if size < PH_HEADER.itemsize:
        raise DataError("file too short for a phase-history header")
    hdr = np.frombuffer(fh.read(PH_HEADER.itemsize), dtype=PH_HEADER)[0]
    _check_format(bytes(hdr["magic"]), int(hdr["version"]), int(hdr["flags"]), PH_MAGIC)
    p, q, k, n_bins = (int(hdr[f]) for f in ("p", "q", "K", "n_bins"))
    if min(p, q, k, n_bins) < 1:
        raise DataError("dimension fields must be positive")
    count = k * n_bins * p * q
    off = PH_HEADER.itemsize
    tail = off + count * _ENTRY.itemsize
    if size < tail + _COUNT.itemsize:
        raise DataError("truncated payload")
    fh.seek(tail)
    n_targets = int(np.frombuffer(fh.read(_COUNT.itemsize), dtype=_COUNT)[0])
    end = tail + _COUNT.itemsize + n_targets * TARGET_RECORD.itemsize
    if size < end:
        raise DataError("truncated target records")
    if size > end:
        raise DataError("trailing bytes after target records")
    recs = np.frombuffer(fh.read(n_targets * TARGET_RECORD.itemsize), dtype=TARGET_RECORD)
    truth = []
    for r in recs:
        if int(r["bin"]) >= n_bins:
            raise DataError(f"target bin {int(r['bin'])} out of range")
        truth.append(TargetTruth(int(r["bin"]), float(r["doppler"]),
                                 complex(float(r["re"]), float(r["im"]))))
    return (p, q, k, n_bins), off, count, truth


def read_phase_history(path):
    """KPH1 file -> PhaseHistory with host complex128 data, every framing
    byte verified (`src/formats.py:55-92`)."""
    with open(path, "rb") as fh:
        size = os.fstat(fh.fileno()).st_size
        (p, q, k, n_bins), off, count, truth = _ph_layout(fh, size)
        fh.seek(off)
        data = np.empty((k, n_bins, p, q), dtype=np.complex128)
        if fh.readinto(memoryview(data).cast("B")) != count * _ENTRY.itemsize:
            raise DataError("truncated payload")
    return PhaseHistory(p, q, k, data, truth)


def load_cube(path, device=None):
    """KPH1 file -> (PhaseHistory whose `data` is a device tensor, pinned
    host staging tensor). The payload goes file -> pinned memory (one
    readinto) -> HBM (one async copy on the current stream)."""
    with open(path, "rb") as fh:
        size = os.fstat(fh.fileno()).st_size
        (p, q, k, n_bins), off, count, truth = _ph_layout(fh, size)
        import torch
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        fh.seek(off)
        host = torch.empty((k, n_bins, p, q), dtype=torch.complex128, pin_memory=True)
        if fh.readinto(memoryview(host.numpy()).cast("B")) != count * _ENTRY.itemsize:
            raise DataError("truncated payload")
    data = host.to(dev, non_blocking=True)
    return PhaseHistory(p, q, k, data, truth), host


# ---------------------------------------------------------------- KES1
def write_estimate(path, estimate):
    """Spatial and temporal factors of a KronCovEstimate (`src/formats.py:95-107`)."""
    spatial = np.ascontiguousarray(_host_array(estimate.spatial), dtype=_ENTRY)
    temporal = np.ascontiguousarray(_host_array(estimate.temporal), dtype=_ENTRY)
    hdr = np.array([(EST_MAGIC, FORMAT_VERSION, FLAG_COMPLEX128, spatial.shape[0],
                     temporal.shape[0], estimate.rank_spatial, estimate.rank_temporal,
                     estimate.iterations, 1 if estimate.converged else 0)], dtype=EST_HEADER)
    with open(path, "wb") as fh:
        fh.write(hdr.tobytes())
        fh.write(memoryview(spatial).cast("B"))
        fh.write(memoryview(temporal).cast("B"))


def read_estimate(path):
    """KES1 file -> KronCovEstimate with an empty residual list
    (`src/formats.py:110-135`)."""
    from .lrkron import KronCovEstimate
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < EST_HEADER.itemsize:
        raise DataError("file too short for an estimate header")
    h = np.frombuffer(blob, dtype=EST_HEADER, count=1)[0]
    _check_format(bytes(h["magic"]), int(h["version"]), int(h["flags"]), EST_MAGIC)
    sdim, q = int(h["sdim"]), int(h["q"])
    if len(blob) != EST_HEADER.itemsize + (sdim * sdim + q * q) * _ENTRY.itemsize:
        raise DataError("estimate payload size mismatch")
    body = np.frombuffer(blob, dtype=_ENTRY, offset=EST_HEADER.itemsize)
    spatial = body[:sdim * sdim].reshape(sdim, sdim).astype(np.complex128)
    temporal = body[sdim * sdim:].reshape(q, q).astype(np.complex128)
    return KronCovEstimate(spatial, temporal, int(h["rank_spatial"]), int(h["rank_temporal"]),
                           int(h["iterations"]), [], bool(h["converged"]))


# ---------------------------------------------------------------- CSV / PGM
def write_residuals_csv(path, residuals):
    lines = ["iteration,residual"]
    lines += [f"{i},{float(eta)!r}" for i, eta in enumerate(residuals, start=1)]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def read_residuals_csv(path):
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0] != "iteration,residual":
        raise DataError("missing residual CSV header")
    return [float(line.split(",")[1]) for line in lines[1:]]


def write_detection_csv(path, image):
    """One row per range bin, one column per Doppler; shortest round-trip
    float reprs (`src/formats.py:153-161`)."""
    values = _host_array(image.values)
    dop = _host_array(image.dopplers)
    with open(path, "w") as fh:
        fh.write("bin," + ",".join("f=" + repr(f) for f in np.asarray(dop, float).tolist()) + "\n")
        for m, row in enumerate(np.asarray(values, np.float64).tolist()):
            fh.write(f"{m}," + ",".join(map(repr, row)) + "\n")


def read_detection_csv(path):
    from .filters import DetectionMap
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or not lines[0].startswith("bin,"):
        raise DataError("missing detection CSV header")
    dopplers = []
    for cell in lines[0].split(",")[1:]:
        if not cell.startswith("f="):
            raise DataError(f"bad Doppler column label {cell!r}")
        dopplers.append(float(cell[2:]))
    values = np.asarray([[float(c) for c in ln.split(",")[1:]] for ln in lines[1:]],
                        dtype=np.float64)
    if values.ndim != 2 or values.shape[1] != len(dopplers):
        raise DataError("detection CSV rows do not match header")
    return DetectionMap(values, np.asarray(dopplers), None)


def write_bench_csv(path, rows):
    with open(path, "w") as fh:
        fh.write("p,q,n,eps,threads,trial,iterations,seconds,eta_final\n")
        for r in rows:
            fh.write(f"{r.p},{r.q},{r.n},{float(r.eps)!r},{r.threads},{r.trial},"
                     f"{r.iterations},{float(r.seconds)!r},{float(r.eta_final)!r}\n")


def write_pgm(path, values):
    """Binary 16-bit PGM, peak scaled to 65535 (`src/formats.py:195-208`)."""
    v = np.asarray(_host_array(values), dtype=np.float64)
    if v.ndim != 2:
        raise DataError(f"image must be 2-D, got shape {v.shape}")
    peak = v.max() if v.size else 0.0
    px = np.round(v / peak * 65535.0) if peak > 0 else np.zeros_like(v)
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n65535\n" % (v.shape[1], v.shape[0]))
        fh.write(px.astype(">u2").tobytes())


# ---------------------------------------------------------------- scene configs
class SimJob:
    """Parsed `simulate` request (`src/formats.py:222-233`)."""

    def __init__(self, scene, n_passes, change_fraction, shared_calibration, unit_pass_gains,
                 pass_gain_spread, targets):
        self.scene = scene
        self.n_passes = n_passes
        self.change_fraction = change_fraction
        self.shared_calibration = shared_calibration
        self.unit_pass_gains = unit_pass_gains
        self.pass_gain_spread = pass_gain_spread
        self.targets = targets


def _as_bool(text, lineno):
    t = text.lower()
    if t in ("1", "true", "yes"):
        return True
    if t in ("0", "false", "no"):
        return False
    raise ConfigError(lineno, f"expected a boolean, got {text!r}")


def _as_int(key, text, lineno):
    try:
        return int(text)
    except ValueError:
        raise ConfigError(lineno, f"{key} expects an integer, got {text!r}") from None


def _as_float(key, text, lineno):
    try:
        return float(text)
    except ValueError:
        raise ConfigError(lineno, f"{key} expects a number, got {text!r}") from None


# key -> value parser (`src/formats.py:214-219`)
_KEYS = {
    **{k: _as_int for k in ("p", "q", "n_bins", "r_b", "seed", "K")},
    **{k: _as_float for k in ("sigma2", "texture_shape", "kappa", "change_fraction",
                              "pass_gain_spread")},
    **{k: (lambda key, text, lineno: _as_bool(text, lineno))
       for k in ("shared_calibration", "unit_pass_gains")},
    "texture": lambda key, text, lineno: text,
}
_REQUIRED = ("p", "q", "n_bins", "r_b")


def _parse_target(value, lineno):
    parts = value.split()
    if len(parts) != 4:
        raise ConfigError(lineno, "target takes exactly: bin doppler amp_re amp_im")
    try:
        return int(parts[0]), float(parts[1]), complex(float(parts[2]), float(parts[3]))
    except ValueError:
        raise ConfigError(lineno, f"bad target fields {value!r}") from None


def parse_scene_config(text):
    """`key = value` lines (`#` comments), movers as `target = BIN DOPPLER RE IM`
    (`src/formats.py:245-325`)."""
    vals, targets = {}, []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, eq, value = line.partition("=")
        if not eq:
            raise ConfigError(lineno, f"expected 'key = value', got {raw.strip()!r}")
        key, value = key.strip(), value.strip()
        if not value:
            raise ConfigError(lineno, f"missing value for {key!r}")
        if key == "target":
            targets.append(_parse_target(value, lineno))
        elif key in _KEYS:
            vals[key] = _KEYS[key](key, value, lineno)
        else:
            raise ConfigError(lineno, f"unknown key {key!r}")
    missing = [k for k in _REQUIRED if k not in vals]
    if missing:
        raise DataError(f"config missing required key {missing[0]!r}")
    scene = SceneConfig(p=vals["p"], q=vals["q"], n_bins=vals["n_bins"],
                        rank_temporal=vals["r_b"], noise_power=vals.get("sigma2", 1e-2),
                        texture=vals.get("texture", "constant"),
                        texture_shape=vals.get("texture_shape", 3.0),
                        kappa=vals.get("kappa", 0.5), seed=vals.get("seed", 0))
    scene.validate()
    n_passes = vals.get("K", 1)
    if n_passes < 1:
        raise DataError(f"K must be >= 1, got {n_passes}")
    for b, _, _ in targets:
        if not 0 <= b < scene.n_bins:
            raise DataError(f"target bin {b} out of range")
    return SimJob(scene, n_passes, vals.get("change_fraction", 0.0),
                  vals.get("shared_calibration", False), vals.get("unit_pass_gains", False),
                  vals.get("pass_gain_spread", 0.5), targets)


def load_scene_config(path):
    with open(path) as fh:
        return parse_scene_config(fh.read())
