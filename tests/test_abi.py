"""CPU: libkst_b200.so loads without a GPU and exports every entry point
declared in include/kst_b200.h; the ctypes binding covers all of them; the
error-code mapping matches the reference exception classes."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1604_03622_b200 import _native as nat
from paper_1604_03622_b200.errors import (CudaError, DataError, DegenerateInputError,
                                          DimensionError)

HEADER = os.path.join(ROOT, "include", "kst_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kst_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    return ctypes.CDLL(nat.LIB_PATH)


def test_header_declares_the_expected_surface():
    names = header_functions()
    for want in ("kst_scm", "kst_lrkron", "kst_detect", "kst_filter", "kst_change",
                 "kst_pipeline", "kst_heig_top", "kst_eig_truncate", "kst_subspace_basis"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_binding_covers_every_declared_symbol():
    assert set(header_functions()) == set(nat.exported_symbols())


def test_exports_are_c_abi_and_sm100a_only():
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True)
    exported = {ln.split()[-1] for ln in out.stdout.splitlines() if " T " in ln}
    assert {n for n in exported if n.startswith("kst_")} == set(header_functions())
    sass = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True)
    if sass.returncode == 0 and sass.stdout.strip():
        assert "sm_100a" in sass.stdout


def test_status_codes_map_to_reference_exceptions(lib):
    lib_ = nat.lib()
    assert lib_.kst_version() == 1
    assert lib_.kst_last_error(None) == b"null context"
    for code, exc in ((1, DimensionError), (2, DataError), (3, DegenerateInputError),
                      (100, CudaError), (101, CudaError)):
        with pytest.raises(exc):
            nat.check(code, None)
    nat.check(0, None)


def test_no_context_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(CudaError):
        nat.ctx(0)
