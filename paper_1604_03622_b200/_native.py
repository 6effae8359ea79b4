"""ctypes binding of libkst_b200.so (include/kst_b200.h).

There is no CPU fallback: if the library (or a CUDA device) is missing,
every product entry point raises. PyTorch is used only for device memory
and the current CUDA stream; the C ABI sees plain pointers and sizes.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import CudaError, DataError, DegenerateInputError, DimensionError, KronStapError

LIB_PATH = os.environ.get("KST_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libkst_b200.so")  # override: A/B builds

_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_ip = C.POINTER(C.c_int)

_SIGS = {
    "kst_version": (_i, []),
    "kst_copy_staged": (_i, [_vp, _vp, _vp, C.c_size_t, _i, _i, _vp]),
    "kst_ctx_create": (_i, [_i, C.POINTER(_vp)]),
    "kst_ctx_destroy": (_i, [_vp]),
    "kst_last_error": (C.c_char_p, [_vp]),
    "kst_launch_count": (C.c_longlong, [_vp]),
    "kst_set_gram": (_i, [_vp, _i, _i]),
    "kst_get_gram": (_i, [_vp, _ip, _ip]),
    "kst_gram_int8_ops": (_d, [_vp]),
    "kst_set_detect": (_i, [_vp, _i]),
    "kst_get_detect": (_i, [_vp, _ip]),
    "kst_set_profiling": (_i, [_vp, _i]),
    "kst_stage_times": (_i, [_vp, _vp, _i]),
    "kst_scm": (_i, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "kst_lrkron": (_i, [_vp, _vp, _i, _i, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp, _vp, _ip, _ip,
                        _ip, _vp, _vp, _vp]),
    "kst_heig_top": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp]),
    "kst_eig_truncate": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "kst_subspace_basis": (_i, [_vp, _vp, _i, _i, _d, _vp, _ip, _vp]),
    "kst_detect": (_i, [_vp, _vp, _i64, _i, _i, _vp, _i, _vp, _i, _i, _i, _vp, _i, _vp, _i, _i,
                        _vp, _vp]),
    "kst_filter": (_i, [_vp, _vp, _i64, _i, _i, _vp, _i, _vp, _i, _i, _i, _vp, _vp]),
    "kst_change": (_i, [_vp, _vp, _vp, _i64, _i, _vp, _vp]),
    "kst_chol": (_i, [_vp, _vp, _i, _vp, _vp]),
    "kst_windowed": (_i, [_vp, _vp, _i64, _i64, _i, _i, _i, _i64, _i64, _i64, _i64, _i64, _i, _i,
                          _d, _i, _i, _i, _vp, _i, _vp, _i, _vp, _vp]),
    "kst_lmode": (_i, [_vp, _vp, _i64, _i64, _i, _i, _i, _i64, _i64, _i, _i, _d, _i, _i, _i, _vp,
                       _i, _vp, _i, _vp, _vp, _vp]),
    "kst_chol_solve": (_i, [_vp, _vp, _i, _vp, _i64, _vp, _vp]),
    "kst_pipeline": (_i, [_vp, _vp, _i64, _i, _i, _i, _i, _d, _i, _i, _vp, _i, _vp, _i, _i, _vp,
                          _vp, _vp]),
    "kst_pipeline_async": (_i, [_vp, _vp, _i64, _i, _i, _i, _i, _d, _i, _i, _vp, _i, _vp, _i, _i,
                                _vp, _vp, _vp]),
    "kst_state_epoch": (C.c_longlong, []),
}

KIND = {"kron": 0, "classical": 1}

_lib = None
_lock = threading.Lock()
_ctxs = {}


def lib():
    """Load libkst_b200.so; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"libkst_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def _torch():
    import torch
    return torch


def device_index(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the Kron-STAP path runs only on the GPU (no CPU fallback)")
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index if not isinstance(device, int) else device


def ctx(device=None):
    """Per-(device, thread) kst_ctx."""
    dev = device_index(device)
    key = (dev, threading.get_ident())
    c = _ctxs.get(key)
    if c is None:
        handle = _vp()
        rc = lib().kst_ctx_create(dev, C.byref(handle))
        if rc != 0:
            raise CudaError(f"kst_ctx_create({dev}) failed with status {rc}")
        c = handle
        _ctxs[key] = c
    return c


def stream_of(device=None):
    torch = _torch()
    return _vp(torch.cuda.current_stream(device).cuda_stream)


def check(rc, c):
    if rc == 0:
        return
    msg = lib().kst_last_error(c)
    msg = msg.decode() if msg else f"status {rc}"
    if rc == 1:
        raise DimensionError(msg)
    if rc == 2:
        raise DataError(msg)
    if rc == 3:
        raise DegenerateInputError(msg)
    if rc >= 100:
        raise CudaError(msg)
    raise KronStapError(msg)


def ptr(t):
    return None if t is None else _vp(t.data_ptr())


# ------------------------------------------------------------------ array plumbing

def is_device(x):
    torch = _torch()
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, dtype="complex128", device=None):
    """numpy / array-like / tensor -> contiguous CUDA tensor of `dtype`."""
    torch = _torch()
    tdt = getattr(torch, dtype)
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(device=f"cuda:{device_index(device)}")
        if t.dtype != tdt:
            t = t.to(tdt)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.dtype(dtype)))
    dev = f"cuda:{device_index(device)}"
    if arr.nbytes >= STAGED_MIN_BYTES:
        # pageable numpy memory: staged through pinned chunks on several host
        # threads (kst_copy_staged), ~3x a pageable cudaMemcpy
        t = torch.empty(arr.shape, dtype=tdt, device=dev)
        c = ctx(t.device)
        check(lib().kst_copy_staged(c, ptr(t), arr.ctypes.data_as(C.c_void_p), arr.nbytes, 0,
                                    staged_threads(), stream_of(t.device)), c)
        return t
    return torch.from_numpy(arr).to(device=dev, non_blocking=False)


STAGED_MIN_BYTES = 8 << 20


def staged_threads():
    """Host threads of a staged copy: half the cores, 2..8."""
    return max(2, min(8, (os.cpu_count() or 4) // 2))


def to_host(t):
    if t is None:
        return None
    t = t.detach()
    if t.is_cuda and t.is_contiguous() and t.numel() * t.element_size() >= STAGED_MIN_BYTES:
        out = np.empty(tuple(t.shape), dtype=_torch().empty(0, dtype=t.dtype).numpy().dtype)
        c = ctx(t.device)
        check(lib().kst_copy_staged(c, out.ctypes.data_as(C.c_void_p), ptr(t), out.nbytes, 1,
                                    staged_threads(), stream_of(t.device)), c)
        return out
    return t.cpu().numpy()
