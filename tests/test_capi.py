"""The C ABI library loads and exports every entry point include/ffdp.h declares (CPU)."""
import ctypes
import os

import pytest

from paper_2509_25044_b200 import _lib


def test_header_declares_the_boundary():
    syms = _lib.header_symbols()
    for s in ("ffdp_sampler_fwd", "ffdp_sampler_bwd", "ffdp_lncc_fwd", "ffdp_mi_hist", "ffdp_step_lncc",
              "ffdp_step_mi_hist", "ffdp_step_mi_grad", "ffdp_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "libffdp.so not built (run __graft_entry__.build())"
    so = ctypes.CDLL(_lib.LIB_PATH)
    for s in _lib.header_symbols():
        assert hasattr(so, s), s
    assert set(_lib.header_symbols()) == set(_lib._SIGS), "ctypes signatures must cover the header exactly"


def test_abi_version_and_no_cpu_fallback():
    so = _lib.lib.load()
    assert so.ffdp_abi_version() == 2
    import torch
    if not torch.cuda.is_available():
        # no device: the library refuses instead of falling back to the CPU
        assert so.ffdp_device_check() == _lib.CUDA
        assert b"CUDA" in so.ffdp_last_error() or so.ffdp_last_error()


def test_parzen_make_is_host_only_and_checks_normalisation():
    k = _lib.ParzenC()
    _lib.lib.ffdp_parzen_make(_lib.PARZEN_BSPLINE3, 32, 0.5, ctypes.byref(k))
    assert k.bins == 32 and k.radius == pytest.approx(2.0 / 32)
    with pytest.raises(_lib.InvalidArgument):
        _lib.lib.ffdp_parzen_make(_lib.PARZEN_GAUSSIAN, 0, 0.5, ctypes.byref(k))
    with pytest.raises(_lib.InvalidArgument):
        _lib.lib.ffdp_parzen_make(7, 32, 0.5, ctypes.byref(k))
