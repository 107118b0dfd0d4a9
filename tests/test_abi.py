"""C-ABI boundary checks that need no GPU: the in-tree library loads, exports
exactly the entry points include/terralio_gpu.h declares, the ctypes binding
covers them, and without a B200 the product path fails loudly (no CPU
fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2509_26222_b200 import _abi

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "terralio_gpu.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tlg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 30
    for must in ("tlg_eval", "tlg_manifold_rows", "tlg_recursive_update", "tlg_select_centers",
                 "tlg_fit_batch_ridge", "tlg_scan_manifold_rows", "tlg_model_save"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(_abi.lib_path()))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(_abi.exported_symbols()) == set(declared())


def test_abi_version_and_errors():
    lib = _abi.load()
    assert lib.tlg_abi_version() == 1
    # invalid parameters are rejected before any device work
    k = _abi.KernelParamsC(0.0, 0.1, 1e-3, 0.0)
    with pytest.raises(_abi.InvalidArgument):
        _abi.check(lib.tlg_kernel_finalize(C.byref(k)))
    k = _abi.KernelParamsC(0.04, 0.1, 1e-3, 0.0)
    _abi.check(lib.tlg_kernel_finalize(C.byref(k)))
    assert abs(k.cutoff_radius - 3 * (0.04 ** 2 + 0.1 ** 2) ** 0.5) < 1e-15


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _abi.load()
    h = C.c_void_p()
    st = lib.tlg_ctx_create(0, None, C.byref(h))
    assert st == _abi.TLG_CUDA_ERROR
    with pytest.raises(_abi.CudaError):
        _abi.check(st)


def test_diag_library_exports_its_header():
    """include/terralio_diag.h (diagnostics, not the product ABI) is served by
    libterralio_diag.so."""
    text = (ROOT / "include" / "terralio_diag.h").read_text()
    names = sorted(set(re.findall(r"\b(tlg_diag_[a-z0-9_]+)\s*\(", text)))
    assert len(names) >= 5
    lib = C.CDLL(str(_abi.lib_path().parent / "libterralio_diag.so"))
    assert not [n for n in names if not hasattr(lib, n)]
