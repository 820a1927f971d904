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


def test_plan_params_layout_matches_the_header(tmp_path):
    """ctypes' ffdp_plan_params / ffdp_parzen layouts equal the C compiler's (offsetof)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    src = tmp_path / "layout.c"
    fields = [f for f, _ in _lib.PlanParamsC._fields_]
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "ffdp.h"\nint main(void) {\n'
                   '  printf("%zu\\n", sizeof(ffdp_plan_params));\n' +
                   "".join(f'  printf("%zu\\n", offsetof(ffdp_plan_params, {f}));\n' for f in fields) + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_lib.PlanParamsC)
    assert vals[1:] == [getattr(_lib.PlanParamsC, f).offset for f in fields]


def test_plan_entry_points_reject_null_arguments():
    """The sharded plan's argument checks run on the host (no device needed)."""
    L = _lib.lib
    with pytest.raises(_lib.InvalidArgument):
        L.ffdp_plan_create(None, _lib.Dims(8, 8, 8), None, None)
    with pytest.raises(_lib.InvalidArgument):
        L.ffdp_plan_step(None, 1, None)
    with pytest.raises(_lib.InvalidArgument):
        L.ffdp_group_nccl(None, 2, 0, 0, None)
    with pytest.raises(_lib.InvalidArgument):
        L.ffdp_group_local(0, None, None)
    assert L.ffdp_plan_u(None) is None and L.ffdp_plan_stream(None) is None


def test_nccl_is_loaded_at_run_time():
    """NCCL comes in by dlopen (no link-time dependency of libffdp.so): the version call
    either reports it or fails with FFDP_RUNTIME naming the reason."""
    import subprocess
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in out
    v = ctypes.c_int(0)
    try:
        _lib.lib.ffdp_nccl_version(ctypes.byref(v))
        assert v.value >= 21800
    except _lib.FabricError as e:
        assert "NCCL unavailable" in str(e)
