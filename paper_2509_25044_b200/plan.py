"""Python face of the native sharded step plan (include/ffdp.h ``ffdp_plan_*``, csrc/plan.cu).

One ``ShardPlan`` per rank: the reference's per-iteration sequence under WorkerGroup(H)
(registration.hpp:266-312 -- ring_sample, dist_lncc / dist_mi, ring_sample_backward)
runs inside the library over NCCL (one process per GPU: ``nccl_group``) or over peer
copies between the host threads of one process (``local_group``). The host code here only
creates the objects and moves the caller's slabs in; the data path has no PyTorch in it.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from ._lib import NCCL_ID_BYTES, Dims, InvalidArgument, PlanParamsC, lib


class _DeviceArray:
    """__cuda_array_interface__ over a plan-owned device buffer (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}
        self._owner = owner


def nccl_version() -> int:
    v = C.c_int(0)
    lib.ffdp_nccl_version(C.byref(v))
    return v.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    lib.ffdp_nccl_unique_id(buf)
    return buf.raw


class Group:
    """One rank's transport handle (ffdp_group)."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)
        w, r, d = C.c_int(0), C.c_int(0), C.c_int(0)
        lib.ffdp_group_info(self.h, C.byref(w), C.byref(r), C.byref(d))
        self.world, self.rank, self.device = w.value, r.value, d.value

    def close(self):
        if self.h:
            lib.ffdp_group_destroy(self.h)
            self.h = None


def nccl_group(unique_id: bytes, world: int, rank: int, device: int) -> Group:
    """Rank `rank` of an NCCL communicator (every rank passes the same unique id)."""
    out = C.c_void_p()
    lib.ffdp_group_nccl(C.c_char_p(bytes(unique_id)), world, rank, device, C.byref(out))
    return Group(out.value)


def local_group(world: int, devices: Optional[Sequence[int]] = None) -> List[Group]:
    """`world` ranks inside this process (devices may repeat); drive each from its own thread."""
    dev = (C.c_int * world)(*devices) if devices is not None else None
    out = (C.c_void_p * world)()
    lib.ffdp_group_local(world, dev, out)
    return [Group(out[r]) for r in range(world)]


class ShardPlan:
    """A rank's plan for the deformable step of a `global_shape` (nz, ny, nx) lattice.

    params: voxreg.LossParams (LNCC window 7 ANTs, or MI with the B-spline Parzen kernel);
    A, t: the stage's affine. ``load(f_slab, m_slab)`` once per scale, then per iteration
    write ``u`` (a torch view of the plan's interior displacement planes) and ``step()``."""

    def __init__(self, group: Group, global_shape, params, A=None, t=None, margin_planes: int = 8,
                 records: bool = True, overlap: bool = True, warp_halo: int = 0):
        from .voxreg import ParzenKernel
        self.group = group
        self.global_shape = tuple(int(s) for s in global_shape)
        nz, ny, nx = self.global_shape
        p = PlanParamsC()
        if params.kind == "lncc":
            p.loss_kind, p.window, p.eps = 0, int(params.window), float(params.epsilon)
        elif params.kind == "mi":
            if not params.mi_bspline_kernel:
                raise InvalidArgument("ShardPlan: the MI plan takes the B-spline Parzen kernel")
            p.loss_kind = 1
            p.kernel = ParzenKernel.bspline3(params.bins).c
        else:
            raise InvalidArgument(f"ShardPlan: loss {params.kind!r} is not a fused step")
        A = np.eye(3) if A is None else np.asarray(A, dtype=np.float64).reshape(3, 3)
        t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64)
        p.A[:] = [float(x) for x in A.ravel()]
        p.t[:] = [float(x) for x in t]
        p.margin_planes, p.records, p.overlap = int(margin_planes), int(records), int(overlap)
        p.warp_halo = int(warp_halo)
        self.params = params
        self.h = C.c_void_p()
        lib.ffdp_plan_create(group.h, Dims(nx, ny, nz), C.byref(p), C.byref(self.h))
        lo, hi = C.c_int64(0), C.c_int64(0)
        lib.ffdp_plan_slab(self.h, C.byref(lo), C.byref(hi))
        self.lo, self.hi = lo.value, hi.value
        self._dev = torch.device("cuda", group.device)
        self._shape = (self.hi - self.lo, ny, nx, 3)
        self.g_u = torch.as_tensor(_DeviceArray(lib.ffdp_plan_g_u(self.h), self._shape, self), device=self._dev)
        self.stream = torch.cuda.ExternalStream(lib.ffdp_plan_stream(self.h), device=self._dev)

    @property
    def u(self) -> torch.Tensor:
        """The slab's displacement planes (a view of the plan's buffer; the warp update moves
        it to the other buffer of its ping-pong pair, so take the view after each update)."""
        return torch.as_tensor(_DeviceArray(lib.ffdp_plan_u(self.h), self._shape, self), device=self._dev)

    def load(self, f_slab: torch.Tensor, m_slab: torch.Tensor):
        """Once per scale: this rank's F and M slabs (planes [lo, hi))."""
        f_slab = f_slab.to(torch.float32).contiguous()
        m_slab = m_slab.to(torch.float32).contiguous()
        torch.cuda.current_stream(f_slab.device).synchronize()
        lib.ffdp_plan_load(self.h, C.c_void_p(f_slab.data_ptr()), C.c_void_p(m_slab.data_ptr()))

    def set_u(self, u_slab: torch.Tensor):
        """Copies this rank's displacement slab into the plan (on the plan's stream)."""
        with torch.cuda.stream(self.stream):
            self.stream.wait_stream(torch.cuda.current_stream(u_slab.device))
            self.u.copy_(u_slab, non_blocking=True)

    def step(self, sync: bool = True):
        """One collective step. sync: the global loss (window misses repaired); else None."""
        loss = C.c_double(0.0)
        lib.ffdp_plan_step(self.h, 1 if sync else 0, C.byref(loss))
        return loss.value if sync else None

    def warp_update(self, lr_norm: float, sigma_grad: float = 1.0, sigma_warp: float = 0.5):
        """The iteration's warp update on the slab (registration.hpp:313-317), collective:
        needs a plan created with warp_halo >= the taps' radius (3 for the default sigmas)."""
        from .voxreg import gaussian_taps
        g = np.ascontiguousarray(gaussian_taps(sigma_grad), dtype=np.float64)
        w = np.ascontiguousarray(gaussian_taps(sigma_warp), dtype=np.float64)
        dp = C.POINTER(C.c_double)
        lib.ffdp_plan_warp_update(self.h, float(lr_norm), g.ctypes.data_as(dp), int(g.size), w.ctypes.data_as(dp),
                                  int(w.size))

    def result(self):
        """(loss, summed window misses) of the last step (waits for it)."""
        loss, miss = C.c_double(0.0), C.c_double(0.0)
        lib.ffdp_plan_result(self.h, C.byref(loss), C.byref(miss))
        return loss.value, miss.value

    def window(self):
        z0, z1, n = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        lib.ffdp_plan_window(self.h, C.byref(z0), C.byref(z1), C.byref(n))
        return z0.value, z1.value, n.value

    def close(self):
        if self.h:
            lib.ffdp_plan_destroy(self.h)
            self.h = None
