"""ctypes binding of libffdp.so (the C ABI declared in include/ffdp.h).

The library is built in-tree (``paper_2509_25044_b200/libffdp.so``) by
``paper_2509_25044_b200.build`` / ``__graft_entry__.build()``. There is no fallback:
if the library is missing or no sm_100 device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFDP_LIB") or os.path.join(HERE, "libffdp.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ffdp.h")

OK, INVALID_ARGUMENT, RUNTIME, LOGIC, CUDA = 0, 1, 2, 3, 4
WANT_IMAGE, WANT_WARP, WANT_AFFINE, WANT_TRANSLATION = 1, 2, 4, 8
PARZEN_GAUSSIAN, PARZEN_BSPLINE3, PARZEN_DELTA = 0, 1, 2


class FfdpError(RuntimeError):
    """Base class of errors raised by libffdp."""


class InvalidArgument(FfdpError, ValueError):
    """std::invalid_argument in the reference (shape / argument errors)."""


class FabricError(FfdpError):
    """std::runtime_error in the reference (transport / size mismatch)."""


class LogicError(FfdpError):
    """std::logic_error in the reference (ParzenKernel normalisation, mi.hpp:132)."""


class CudaError(FfdpError):
    """Device failure (no sm_100 device, launch error, out of memory)."""


_EXC = {INVALID_ARGUMENT: InvalidArgument, RUNTIME: FabricError, LOGIC: LogicError, CUDA: CudaError}


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64)]


class SamplerArgsC(C.Structure):
    _fields_ = [("A", C.c_double * 9), ("t", C.c_double * 3), ("S", C.c_double * 3), ("x_min", C.c_double * 3),
                ("x_max", C.c_double * 3)]


class ImageWindow(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dims", Dims), ("z_begin", C.c_int64), ("z_end", C.c_int64),
                ("pad", C.c_int64)]


class Slab(C.Structure):
    _fields_ = [("buf_z0", C.c_int64), ("buf_nz", C.c_int64), ("z_begin", C.c_int64), ("z_end", C.c_int64),
                ("nz_global", C.c_int64)]


class ParzenC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("bins", C.c_int32), ("sigma", C.c_double), ("radius", C.c_double),
                ("norm", C.c_double)]


class PlanParamsC(C.Structure):
    """ffdp_plan_params (include/ffdp.h)."""
    _fields_ = [("loss_kind", C.c_int32), ("window", C.c_int32), ("eps", C.c_double), ("kernel", ParzenC),
                ("A", C.c_double * 9), ("t", C.c_double * 3), ("margin_planes", C.c_int32),
                ("records", C.c_int32), ("overlap", C.c_int32), ("warp_halo", C.c_int32)]


NCCL_ID_BYTES = 128

_vp, _dp = C.c_void_p, C.POINTER(C.c_double)
_vpp = C.POINTER(C.c_void_p)
_SIGS = {
    "ffdp_last_error": (C.c_char_p, []),
    "ffdp_abi_version": (C.c_int, []),
    "ffdp_device_check": (C.c_int, []),
    "ffdp_scratch_trim": (C.c_int, [C.c_int64]),
    "ffdp_sampler_fwd": (C.c_int, [ImageWindow, _vp, Dims, C.POINTER(SamplerArgsC), _vp, C.c_int, _vp, _vp, _vp]),
    "ffdp_sampler_bwd": (C.c_int, [_vp, ImageWindow, _vp, Dims, C.POINTER(SamplerArgsC), C.c_int, _vp, _vp, _vp, _vp,
                                   _vp]),
    "ffdp_convolve_axis": (C.c_int, [_vp, _vp, Dims, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                     _vp]),
    "ffdp_lncc_fwd": (C.c_int, [_vp, _vp, Dims, Slab, C.c_int, C.c_double, _vp, _vp, _vp, _vp]),
    "ffdp_lncc_gamma": (C.c_int, [_vp, C.c_int64, C.c_double, C.c_double, _vp]),
    "ffdp_lncc_bwd": (C.c_int, [C.c_double, _vp, _vp, _vp, Dims, C.c_int, C.c_double, C.c_int, _vp, _vp, _vp]),
    "ffdp_lncc_fwdbwd": (C.c_int, [_vp, _vp, Dims, C.c_int, C.c_double, C.c_int, C.c_double, _vp, _vp, _vp, _vp,
                                   _vp]),
    "ffdp_lncc_combine": (C.c_int, [_vp, Dims, Slab, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "ffdp_parzen_make": (C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(ParzenC)]),
    "ffdp_mi_hist": (C.c_int, [_vp, _vp, C.c_int64, C.POINTER(ParzenC), C.c_int, _vp, _vp,
                               C.POINTER(C.c_uint64), _vp]),
    "ffdp_mi_finalize": (C.c_int, [_vp, C.c_int, C.c_double, _vp, _vp]),
    "ffdp_mi_bwd": (C.c_int, [_vp, _vp, C.c_int64, C.POINTER(ParzenC), _vp, _vp, _vp, _vp]),
    "ffdp_step_lncc": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC), C.c_int, C.c_double,
                                 C.c_double, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ffdp_step_lncc_workspace_bytes": (C.c_int64, [Dims, Slab]),
    "ffdp_step_lncc_passes": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC), C.c_int,
                                        C.c_double, C.c_double, C.c_float, C.c_float, _vp, _vp, _vp, _vp, C.c_int,
                                        _vp]),
    "ffdp_step_lncc_passes_workspace_bytes": (C.c_int64, [Dims, Slab]),
    "ffdp_step_mi_hist": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC), C.POINTER(ParzenC),
                                    _vp, _vp, _vp, _vp]),
    "ffdp_step_mi_workspace_bytes": (C.c_int64, [C.c_int]),
    "ffdp_step_mi": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC), C.POINTER(ParzenC),
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ffdp_step_mi_record_bytes": (C.c_int64, [Dims, Slab]),
    "ffdp_step_mi_hist_rec": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC),
                                        C.POINTER(ParzenC), _vp, _vp, _vp, _vp, _vp]),
    "ffdp_step_mi_hist_final": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC),
                                          C.POINTER(ParzenC), _vp, C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "ffdp_step_mi_grad_rec": (C.c_int, [_vp, Dims, Slab, C.POINTER(ParzenC), _vp, _vp, _vp, _vp]),
    "ffdp_step_mi_grad": (C.c_int, [_vp, _vp, Dims, Slab, ImageWindow, C.POINTER(SamplerArgsC), C.POINTER(ParzenC),
                                    _vp, _vp, _vp, _vp]),
    "ffdp_gp_convolve": (C.c_int, [_vp, _vp, Dims, Slab, C.c_int, _vp, C.c_int, C.c_int, _vp]),
    "ffdp_sobolev_adam": (C.c_int, [_vp, _vp, _vp, _vp, Dims, Slab, _vp, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_int64, _vp]),
    "ffdp_resample_dims": (C.c_int, [Dims, C.c_double, C.POINTER(Dims)]),
    "ffdp_resample_scale": (C.c_int, [_vp, Dims, C.c_double, _vp, _vp, _vp]),
    "ffdp_resample_warp": (C.c_int, [_vp, Dims, _vp, Dims, _vp]),
    "ffdp_normalize": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "ffdp_jacobian_positive": (C.c_int, [_vp, Dims, C.POINTER(C.c_double), _vp]),
    "ffdp_mse": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp, _vp, _vp]),
    "ffdp_reduce_sum_f64": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "ffdp_minmax": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "ffdp_pad_window": (C.c_int, [_vp, Dims, C.c_int64, C.c_int64, _vp, _vp]),
    "ffdp_sampler_z_extent": (C.c_int, [_vp, Dims, Dims, C.POINTER(SamplerArgsC), _vp, _vp]),
    # the sharded context: per-rank arguments are arrays of device pointers
    "ffdp_comm_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "ffdp_comm_destroy": (C.c_int, [_vp]),
    "ffdp_comm_world": (C.c_int, [_vp]),
    "ffdp_comm_device": (C.c_int, [_vp, C.c_int]),
    "ffdp_shard_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ffdp_halo_exchange": (C.c_int, [_vp, _vpp, Dims, C.c_int, C.c_int, _vpp, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]),
    "ffdp_dist_gp_convolve": (C.c_int, [_vp, _vpp, Dims, C.c_int, _dp, C.c_int, C.c_int, C.c_int, _vpp]),
    "ffdp_ring_sample": (C.c_int, [_vp, _vpp, Dims, _vpp, Dims, _dp, _dp, _vpp]),
    "ffdp_ring_sample_bwd": (C.c_int, [_vp, _vpp, _vpp, Dims, _vpp, Dims, _dp, _dp, C.c_int, _vpp, _vpp, _dp]),
    "ffdp_dist_mse": (C.c_int, [_vp, _vpp, _vpp, Dims, C.c_int64, _dp, _vpp]),
    "ffdp_dist_mi": (C.c_int, [_vp, _vpp, _vpp, Dims, C.POINTER(ParzenC), C.c_int, C.c_int64, _dp, _vpp,
                               C.POINTER(C.c_int64)]),
    "ffdp_dist_lncc": (C.c_int, [_vp, _vpp, _vpp, Dims, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int64, _dp,
                                 _vpp]),
    "ffdp_dist_step": (C.c_int, [_vp, C.c_int, _vpp, _vpp, _vpp, Dims, _dp, _dp, C.c_int, C.c_double,
                                 C.POINTER(ParzenC), _dp, _vpp]),
    # the native sharded step plan (plan.cu)
    "ffdp_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "ffdp_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ffdp_group_nccl": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ffdp_group_local": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "ffdp_group_destroy": (C.c_int, [_vp]),
    "ffdp_group_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ffdp_plan_create": (C.c_int, [_vp, Dims, C.POINTER(PlanParamsC), C.POINTER(C.c_void_p)]),
    "ffdp_plan_destroy": (C.c_int, [_vp]),
    "ffdp_plan_slab": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ffdp_plan_stream": (C.c_void_p, [_vp]),
    "ffdp_plan_u": (C.c_void_p, [_vp]),
    "ffdp_plan_g_u": (C.c_void_p, [_vp]),
    "ffdp_plan_window": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ffdp_plan_load": (C.c_int, [_vp, _vp, _vp]),
    "ffdp_plan_step": (C.c_int, [_vp, C.c_int, _dp]),
    "ffdp_plan_result": (C.c_int, [_vp, _dp, _dp]),
    "ffdp_plan_warp_update": (C.c_int, [_vp, C.c_double, _dp, C.c_int, _dp, C.c_int]),
}


def header_symbols(path: str = HEADER):
    """Every entry point declared by include/ffdp.h."""
    with open(path) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^FFDP_API\s+[\w\s\*]+?\b(ffdp_\w+)\(", text, flags=re.M)))


class _Lib:
    def __init__(self):
        self._lib = None

    def load(self):
        if self._lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaError(f"libffdp.so is not built ({LIB_PATH}); run __graft_entry__.build()")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            self._lib = lib
        return self._lib

    def __getattr__(self, name):
        lib = self.load()
        fn = getattr(lib, name)
        if name in ("ffdp_last_error", "ffdp_abi_version", "ffdp_device_check", "ffdp_step_mi_workspace_bytes",
                    "ffdp_step_mi_record_bytes", "ffdp_step_lncc_workspace_bytes",
                    "ffdp_step_lncc_passes_workspace_bytes", "ffdp_comm_world",
                    "ffdp_comm_device", "ffdp_plan_stream", "ffdp_plan_u", "ffdp_plan_g_u"):
            return fn

        def call(*args):
            rc = fn(*args)
            if rc != OK:
                msg = lib.ffdp_last_error().decode(errors="replace")
                raise _EXC.get(rc, FfdpError)(f"{name}: {msg}")
            return rc

        return call


lib = _Lib()
