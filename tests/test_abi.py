"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; validation paths answer without touching a GPU.  CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tsnmf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tsnmf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1402_6964_b200 import _native

    return _native.load()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("tsnmf_tsqr", "tsnmf_r_combine", "tsnmf_gram", "tsnmf_sketch", "tsnmf_normal_block",
                 "tsnmf_uniform_block", "tsnmf_workspace_bytes", "tsnmf_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_1402_6964_b200", "libtsnmf_b200.so"))
    for name in declared_symbols():
        assert hasattr(raw, name), name


def test_binding_table_matches_header(lib):
    from paper_1402_6964_b200 import _native

    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1402_6964_b200", "libtsnmf_b200.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_callable_pieces(lib, oracle):
    from paper_1402_6964_b200 import _native

    assert lib.tsnmf_abi_version() == _native.ABI_VERSION
    for seed, tag in [(0, 0), (7, 3), (2**64 - 1, 5)]:
        assert lib.tsnmf_derive_stream(seed, tag) == oracle.derive_stream(seed, tag)
    assert lib.tsnmf_max_cols() >= 256
    for op, m, n, k in [(1, 1 << 26, 200, 0), (2, 16, 200, 0), (3, 1 << 26, 200, 0), (4, 1 << 26, 200, 400),
                        (5, 1000, 25, 0), (1, 10, 1, 0), (1, 10, 512, 0)]:
        assert lib.tsnmf_workspace_bytes(op, m, n, k) > 0
    assert lib.tsnmf_workspace_bytes(1, 10, 100000, 0) == 0
    assert lib.tsnmf_workspace_bytes(99, 10, 10, 0) == 0


def test_validation_errors_without_gpu(lib):
    """Argument checks run before any device work and map to the reference's
    exit codes (usage = 1, data = 2)."""
    assert lib.tsnmf_tsqr(None, 10, 4, 4, None, 4, None, None, None, 0, None) == 1
    assert b"null" in lib.tsnmf_last_error()
    assert lib.tsnmf_tsqr(ctypes.c_void_p(8), 0, 4, 4, ctypes.c_void_p(8), 4, None, None, None, 0, None) == 2
    assert lib.tsnmf_tsqr(ctypes.c_void_p(8), 10, 4, 3, ctypes.c_void_p(8), 4, None, None, None, 0, None) == 1
    assert lib.tsnmf_sketch(ctypes.c_void_p(8), 10, 4, 4, 0, 0, 0, None, 0, ctypes.c_void_p(8), 4, None, 0,
                            None) == 1
    assert lib.tsnmf_r_combine(ctypes.c_void_p(8), 0, 4, ctypes.c_void_p(8), 4, None, 0, None) == 2


def test_status_maps_to_reference_errors(lib):
    from paper_1402_6964_b200 import _native
    from paper_1402_6964_b200.errors import DataError, UsageError

    lib.tsnmf_tsqr(None, 10, 4, 4, None, 4, None, None, None, 0, None)
    with pytest.raises(UsageError):
        _native.check(1)
    with pytest.raises(DataError):
        _native.check(2)
    assert DataError.exit_code == 2 and UsageError.exit_code == 1


def test_no_cpu_fallback():
    """Without a GPU the product path raises instead of computing on the CPU."""
    import torch

    import paper_1402_6964_b200 as tb

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tb.TsnmfError):
        tb.factor_chunk(np.eye(3))
    with pytest.raises(tb.TsnmfError):
        tb.stream_pass([tb.RowChunk(0, np.ones((5, 2)))])


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1402_6964_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "tsnmf_oracle" not in src and "liboracle" not in src, f
