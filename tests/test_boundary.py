"""The C-ABI boundary on a CPU-only box: liblopc.so (built for sm_100a) loads
and exports every function include/lopc.h declares; the product path refuses
to run without a GPU (no CPU fallback); nothing in the product package
imports the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def so():
    from paper_2603_26968_b200 import build

    return build.build()


def test_exports_every_declared_symbol(so):
    from paper_2603_26968_b200 import lopc

    L = ctypes.CDLL(so)
    names = lopc.declared_symbols()
    assert "lopc_compress" in names and "lopc_decompress" in names and len(names) >= 12
    for n in names:
        assert hasattr(L, n), n


def test_host_only_calls(so):
    from paper_2603_26968_b200 import lopc

    L = lopc.load(require_gpu=False)
    assert L.lopc_abi_version() == 1
    d = lopc._dims((100, 500, 500))
    assert L.lopc_compress_bound(3, d, 0) == 64 + 8 * 6104 + 2 * 16384 * 6104
    assert L.lopc_compress_workspace_bytes(3, d, 0, 0) > 25_000_000 * 6
    assert L.lopc_compress_bound(4, d, 0) == 0
    assert L.lopc_strerror(-4) == b"corrupt stream"


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_26968_b200 as lopc

    with pytest.raises(RuntimeError):
        lopc.compress(torch.zeros(4, 4), 0.1)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2603_26968_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b|lopc_ref", src), f


def test_header_documents_every_entry_point():
    src = open(os.path.join(ROOT, "include", "lopc.h")).read()
    for kw in ("owned by the caller", "LOPC_E_CORRUPT", "P:109-116", "P:314", "DESIGN.md"):
        assert kw in src
