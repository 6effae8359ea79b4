"""Staged pageable host <-> device copies (kst_copy_staged, csrc/hostio.cu):
byte-exact round trips over chunk-boundary sizes, thread counts and a
non-default stream, and the numpy drop-in path (to_device / to_host) that
uses them for large arrays."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1604_03622_b200 import _native as nat  # noqa: E402

CH = 4 << 20


@pytest.mark.parametrize("nbytes", [1, CH - 1, CH, CH + 1, 7 * CH + 12345, 50 * CH + 3])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_round_trip_is_byte_exact(nbytes, threads):
    rng = np.random.default_rng(nbytes + threads)
    host = rng.integers(0, 256, nbytes, dtype=np.uint8)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    c = nat.ctx()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        nat.check(nat.lib().kst_copy_staged(c, nat.ptr(dev), host.ctypes.data_as(C.c_void_p), nbytes,
                                            0, threads, nat.stream_of()), c)
        host[:] = 0  # the source may be reused as soon as the call returns
        back = np.empty(nbytes, dtype=np.uint8)
        nat.check(nat.lib().kst_copy_staged(c, back.ctypes.data_as(C.c_void_p), nat.ptr(dev), nbytes,
                                            1, threads, nat.stream_of()), c)
    want = np.random.default_rng(nbytes + threads).integers(0, 256, nbytes, dtype=np.uint8)
    assert np.array_equal(back, want)
    st.synchronize()
    assert torch.equal(dev.cpu(), torch.from_numpy(want))


def test_numpy_path_uses_staged_copies_and_is_exact():
    rng = np.random.default_rng(5)
    cube = rng.standard_normal((300, 3, 2001)) + 1j * rng.standard_normal((300, 3, 2001))
    assert cube.nbytes >= nat.STAGED_MIN_BYTES
    t = nat.to_device(cube)
    assert t.is_cuda and t.dtype == torch.complex128
    assert torch.equal(t.cpu(), torch.from_numpy(cube))
    back = nat.to_host(t)
    assert back.dtype == np.complex128 and np.array_equal(back, cube)
    # back-to-back calls reuse the pinned ring (slot events guard reuse)
    for k in range(3):
        x = cube * (k + 2)
        assert np.array_equal(nat.to_host(nat.to_device(x)), x)


def test_bad_arguments():
    c = nat.ctx()
    buf = np.zeros(16, dtype=np.uint8)
    assert nat.lib().kst_copy_staged(c, None, buf.ctypes.data_as(C.c_void_p), 16, 0, 2, None) == 1
    assert nat.lib().kst_copy_staged(c, buf.ctypes.data_as(C.c_void_p), buf.ctypes.data_as(C.c_void_p),
                                     16, 2, 2, None) == 1
