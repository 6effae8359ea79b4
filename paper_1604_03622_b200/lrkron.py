"""Sample covariance and LR-Kron estimation on the GPU.

Mirrors `kronstap.lrkron` (src/lrkron.py): same function names, argument
meaning, dataclass fields and exceptions. The arithmetic runs in
libkst_b200 (K1 Gram, K2 sweeps, K3 Jacobi, K4 top-r eigensolver):

    sample_covariance -> kst_scm     (src/lrkron.py:53-78)
    lr_kron_estimate  -> kst_lrkron  (src/lrkron.py:118-230)

`pool` arguments are accepted and ignored (results are deterministic by
construction, like the reference's pool invariance, src/parallel.py:1-8).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from ._dual import Dual
from .errors import DimensionError


class SampleCovariance:
    """Mean of snapshot outer products, tagged with the bin shape
    (src/lrkron.py:26-33). `matrix` is numpy or a CUDA tensor, matching
    what the caller passed in."""

    def __init__(self, matrix, n_samples, p, q, _trusted=False):
        self._m = matrix if isinstance(matrix, Dual) else Dual(matrix)
        self.n_samples = n_samples
        self.p = p
        self.q = q
        self._trusted = _trusted  # produced by kst_scm: finite-checked, exactly Hermitian

    @property
    def matrix(self):
        return self._m.value()

    @matrix.setter
    def matrix(self, value):
        self._m = Dual(value)
        self._trusted = False

    def device_matrix(self):
        return self._m.dev()

    def __repr__(self):
        return f"SampleCovariance(p={self.p}, q={self.q}, n_samples={self.n_samples})"


class KronCovEstimate:
    """Kronecker-factored covariance estimate and its fit history
    (src/lrkron.py:36-50)."""

    def __init__(self, spatial, temporal, rank_spatial, rank_temporal, iterations,
                 residuals=None, converged=True):
        self._sp = spatial if isinstance(spatial, Dual) else Dual(spatial)
        self._tp = temporal if isinstance(temporal, Dual) else Dual(temporal)
        self.rank_spatial = rank_spatial
        self.rank_temporal = rank_temporal
        self.iterations = iterations
        self.residuals = [] if residuals is None else residuals
        self.converged = converged
        self._tb = None  # (device vectors (q, rb), host values (rb,)) of the final b

    @property
    def spatial(self):
        return self._sp.value()

    @spatial.setter
    def spatial(self, v):
        self._sp = Dual(v)
        self._tb = None

    @property
    def temporal(self):
        return self._tp.value()

    @temporal.setter
    def temporal(self, v):
        self._tp = Dual(v)
        self._tb = None

    def product(self):
        """Materialise kron(spatial, temporal). Small sizes only."""
        a, b = self.spatial, self.temporal
        if nat.is_device(a):
            import torch
            return torch.kron(a, b)
        return np.kron(np.asarray(a, dtype=np.complex128), np.asarray(b, dtype=np.complex128))

    def __repr__(self):
        return (f"KronCovEstimate(rank_spatial={self.rank_spatial}, rank_temporal={self.rank_temporal}, "
                f"iterations={self.iterations}, converged={self.converged})")


def set_gram_engine(mode="dmma", slices=7, device=None):
    """Select the sample-covariance engine (K1) for this thread's context:
    "dmma" (FP64 tensor-core tiles), "int8" (exact int8 slices on the int8
    tensor cores, `slices` 7-bit slices per operand), "crt" (int8 modular
    residues recombined by the Chinese remainder theorem, `slices` moduli, on
    the hand-written tcgen05 kernel) or "crt-cublas" (same numerics, cuBLAS
    int8 GEMMs)."""
    c = nat.ctx(device)
    code = {"dmma": 0, "int8": 1, "crt": 2, "crt-cublas": 3}[mode]
    nat.check(nat.lib().kst_set_gram(c, code, int(slices)), c)


def get_gram_engine(device=None):
    c = nat.ctx(device)
    m, s = C.c_int(0), C.c_int(0)
    nat.check(nat.lib().kst_get_gram(c, C.byref(m), C.byref(s)), c)
    return ("dmma", "int8", "crt", "crt-cublas")[m.value], s.value


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


def sample_covariance(snapshots, p, q, pool=None):
    """S = (1/n) X^T conj(X), exactly Hermitian (src/lrkron.py:53-78)."""
    import torch
    device_mode = nat.is_device(snapshots)
    shp = _shape(snapshots)
    if len(shp) != 2:
        raise DimensionError(f"snapshots must be 2-D, got shape {shp}")
    n, d = shp
    if n < 1:
        raise DimensionError("need at least one snapshot")
    if d != p * q:
        raise DimensionError(f"snapshot length {d} does not match p*q = {p * q}")
    x = nat.to_device(snapshots)
    c = nat.ctx(x.device)
    s = torch.empty((d, d), dtype=torch.complex128, device=x.device)
    nat.check(nat.lib().kst_scm(c, nat.ptr(x), n, d, nat.ptr(s), nat.stream_of(x.device)), c)
    return SampleCovariance(Dual.from_device(s, device_mode), n, p, q, _trusted=True)


def lr_kron_estimate(scm, rank_spatial, rank_temporal, tol=1e-4, max_iter=100, pool=None,
                     keep_iterates=False):
    """Alternating Kronecker-factor fit (src/lrkron.py:118-230)."""
    import torch
    if not all(hasattr(scm, a) for a in ("matrix", "p", "q")) or isinstance(scm, np.ndarray):
        raise DimensionError("estimator expects a SampleCovariance")
    p, q = int(scm.p), int(scm.q)
    dual = scm._m if isinstance(scm, SampleCovariance) else Dual(scm.matrix)
    device_mode = dual.device_mode
    shp = _shape(scm.matrix) if not isinstance(scm, SampleCovariance) else (
        _shape(dual._dev) if dual._dev is not None else _shape(dual._host))
    if len(shp) != 2:
        raise DimensionError(f"covariance must be 2-D, got shape {shp}")
    if shp != (p * q, p * q):
        raise DimensionError(f"covariance shape {shp} does not match p*q = {p * q}")
    s = dual.dev()
    dev = s.device
    c = nat.ctx(dev)
    validate = 0 if getattr(scm, "_trusted", False) else 1
    spatial = torch.empty((p, p), dtype=torch.complex128, device=dev)
    temporal = torch.empty((q, q), dtype=torch.complex128, device=dev)
    rb_ok = 1 <= rank_temporal <= q
    tbv = torch.empty((q, max(rank_temporal, 1) if rb_ok else 1), dtype=torch.complex128, device=dev)
    tbval = np.zeros(max(rank_temporal, 1) if rb_ok else 1)
    mi = max(int(max_iter), 1)
    res = np.zeros(mi)
    nres, iters, conv = C.c_int(0), C.c_int(0), C.c_int(0)
    it_sp = it_b = None
    if keep_iterates:
        it_sp = torch.empty((mi, p, p), dtype=torch.complex128, device=dev)
        it_b = torch.empty((mi, q, q), dtype=torch.complex128, device=dev)
    rc = nat.lib().kst_lrkron(
        c, nat.ptr(s), p, q, int(rank_spatial), int(rank_temporal), float(tol), int(max_iter),
        validate, nat.ptr(spatial), nat.ptr(temporal), nat.ptr(tbv) if rb_ok else None,
        tbval.ctypes.data_as(C.c_void_p) if rb_ok else None, res.ctypes.data_as(C.c_void_p),
        C.byref(nres), C.byref(iters), C.byref(conv), nat.ptr(it_sp), nat.ptr(it_b),
        nat.stream_of(dev))
    nat.check(rc, c)
    est = KronCovEstimate(Dual.from_device(spatial, device_mode), Dual.from_device(temporal, device_mode),
                          rank_spatial, rank_temporal, iters.value,
                          [float(v) for v in res[:nres.value]], bool(conv.value))
    if rb_ok and rank_temporal < q and iters.value > 0:
        est._tb = (tbv, tbval.copy())
    if keep_iterates:
        k = iters.value
        if device_mode:
            est.iterates = [(it_sp[i].clone(), it_b[i].clone()) for i in range(k)]
        else:
            hs, hb = nat.to_host(it_sp[:k]), nat.to_host(it_b[:k])
            est.iterates = [(hs[i], hb[i]) for i in range(k)]
    return est
