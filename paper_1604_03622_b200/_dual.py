"""Host/device dual storage for API results.

The reference returns numpy arrays; this package keeps results on the GPU
and hands numpy to callers that passed numpy (materialised lazily, once),
or CUDA tensors to callers that passed CUDA tensors. Chained calls
(`sample_covariance -> lr_kron_estimate -> build_filter -> detection_image`)
therefore never copy the large intermediates (S is 577 MB at Gotcha scale)
back to the host.
"""

from __future__ import annotations

from . import _native as nat


class Dual:
    """One API value held on the host, the device, or both.

    Ownership rules (the reference's dataclasses hold plain numpy arrays, so
    in-place edits there are honoured, src/lrkron.py:26-50):

    * host-origin (the caller handed us numpy): the caller's array stays the
      source of truth; every device use uploads it afresh, so in-place edits
      made between calls are seen (and re-validated by the consumer);
    * device-origin (a kernel produced it): the host copy is materialised
      once and handed out READ-ONLY, so an in-place edit raises instead of
      silently diverging from the device copy the next call would read.
      Callers that want to edit assign a new array to the field.
    """

    __slots__ = ("_host", "_dev", "device_mode", "_host_origin")

    def __init__(self, value=None, device_mode=None):
        self._host = None
        self._dev = None
        self._host_origin = False
        if value is not None:
            if nat.is_device(value):
                self._dev = value
            else:
                self._host = value
                self._host_origin = True
        self.device_mode = nat.is_device(value) if device_mode is None else device_mode

    @classmethod
    def from_device(cls, tensor, device_mode):
        d = cls(None, device_mode)
        d._dev = tensor
        return d

    def is_none(self):
        return self._host is None and self._dev is None

    def host(self):
        if self._host is None and self._dev is not None:
            h = nat.to_host(self._dev)
            if hasattr(h, "setflags"):
                h.setflags(write=False)
            self._host = h
        return self._host

    def dev(self, dtype="complex128"):
        if self._host_origin:
            # the caller's array is the truth: no cached device copy
            return nat.to_device(self._host, dtype)
        if self._dev is None and self._host is not None:
            self._dev = nat.to_device(self._host, dtype)
        return self._dev

    def value(self):
        """What the caller sees: tensor in device mode, numpy otherwise."""
        if self.is_none():
            return None
        return self.dev() if self.device_mode else self.host()
