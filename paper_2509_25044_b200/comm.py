"""Python face of the C ABI's sharded context (`ffdp_comm`, include/ffdp.h): one process
drives H ranks, rank r a z slab on devices[r] (WorkerGroup(H) and the collective
operators of fabric.hpp / distops.hpp:54-396). Per-rank arguments are lists of CUDA
tensors, rank r's on devices[r]; every call runs all ranks in lock step.

This is the single-process multi-GPU form of the sharded path (peer copies over NVLink);
dist.py is the one-process-per-GPU form over torch.distributed. Both split z by
shard_ranges (fabric.hpp:44-70) and compose the same kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from ._lib import Dims, InvalidArgument, lib


def _ptrs(ts: Sequence[torch.Tensor]):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def _dims(shape) -> Dims:
    nz, ny, nx = (int(s) for s in shape[:3])
    return Dims(nx, ny, nz)


def _mat(A, n):
    if A is None:
        return None
    a = np.ascontiguousarray(np.asarray(A, dtype=np.float64).reshape(n))
    return a


class Comm:
    """ffdp_comm_create(world, devices) ... ffdp_comm_destroy."""

    def __init__(self, world: int, devices: Optional[Sequence[int]] = None):
        h = C.c_void_p()
        devs = None if devices is None else (C.c_int * world)(*devices)
        lib.ffdp_comm_create(world, devs, C.byref(h))
        self.h = h
        self.world = world
        self.devices = [lib.ffdp_comm_device(h, r) for r in range(world)]

    def close(self):
        if self.h:
            lib.ffdp_comm_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    # ------------------------------------------------------------ layout
    def shard_range(self, n: int, rank: int) -> Tuple[int, int]:
        lo, hi = C.c_int64(), C.c_int64()
        lib.ffdp_shard_range(n, self.world, rank, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def scatter(self, v: torch.Tensor) -> List[torch.Tensor]:
        """Rank r's z slab of a global volume / warp, on devices[r]."""
        out = []
        for r in range(self.world):
            lo, hi = self.shard_range(v.shape[0], r)
            out.append(v[lo:hi].to(torch.device("cuda", self.devices[r])).contiguous())
        return out

    def _empty(self, global_shape, tail=(), like=None) -> List[torch.Tensor]:
        out = []
        for r in range(self.world):
            lo, hi = self.shard_range(global_shape[0], r)
            out.append(torch.empty((hi - lo,) + tuple(global_shape[1:3]) + tuple(tail), dtype=torch.float32,
                                   device=torch.device("cuda", self.devices[r])))
        return out

    def _check(self, ts, what):
        if len(ts) != self.world:
            raise InvalidArgument(f"{what}: {len(ts)} tensors for {self.world} ranks")
        for r, t in enumerate(ts):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
                raise InvalidArgument(f"{what}: rank {r} needs a contiguous float32 CUDA tensor")
            if t.device.index != self.devices[r]:
                raise InvalidArgument(f"{what}: rank {r}'s tensor is not on device {self.devices[r]}")

    # ------------------------------------------------------------ collectives
    def halo_exchange(self, slabs, global_shape, pad: int):
        """halo_exchange (fabric.hpp:315-370) -> (padded slabs, halo_lo, halo_hi)."""
        self._check(slabs, "halo_exchange")
        ch = 1 if slabs[0].dim() == 3 else slabs[0].shape[3]
        lo = (C.c_int64 * self.world)()
        hi = (C.c_int64 * self.world)()
        out = []
        for r, s in enumerate(slabs):
            a = pad if r > 0 else 0
            b = pad if r < self.world - 1 else 0
            out.append(torch.empty((s.shape[0] + a + b,) + tuple(s.shape[1:]), dtype=torch.float32, device=s.device))
        lib.ffdp_halo_exchange(self.h, _ptrs(slabs), _dims(global_shape), ch, pad, _ptrs(out), lo, hi)
        return out, list(lo), list(hi)

    def gp_convolve(self, slabs, taps, global_shape, mode: str = "zero_pad", sync: bool = True):
        self._check(slabs, "gp_convolve")
        taps = np.ascontiguousarray(taps, dtype=np.float64)
        ch = 1 if slabs[0].dim() == 3 else slabs[0].shape[3]
        out = [torch.empty_like(s) for s in slabs]
        lib.ffdp_dist_gp_convolve(self.h, _ptrs(slabs), _dims(global_shape), ch,
                                  taps.ctypes.data_as(C.POINTER(C.c_double)), taps.size,
                                  1 if mode == "renormalize" else 0, int(sync), _ptrs(out))
        return out

    def ring_sample(self, m_shards, m_global, u_shards, out_global, A=None, t=None):
        self._check(m_shards, "ring_sample")
        self._check(u_shards, "ring_sample")
        out = self._empty(out_global)
        A9, t3 = _mat(A, 9), _mat(t, 3)
        lib.ffdp_ring_sample(self.h, _ptrs(m_shards), _dims(m_global), _ptrs(u_shards), _dims(out_global),
                             None if A9 is None else A9.ctypes.data_as(C.POINTER(C.c_double)),
                             None if t3 is None else t3.ctypes.data_as(C.POINTER(C.c_double)), _ptrs(out))
        return out

    def ring_sample_backward(self, upstream, m_shards, m_global, u_shards, out_global, A=None, t=None,
                             want=("warp",)):
        """-> (g_img shards or None, g_u slabs or None, dA (3, 3) or None, dt (3,) or None)."""
        for x, n in ((upstream, "upstream"), (m_shards, "m"), (u_shards, "u")):
            self._check(x, f"ring_sample_backward ({n})")
        mask = sum(b for k, b in (("image", 1), ("warp", 2), ("affine", 4), ("translation", 8)) if k in want)
        g_img = self._empty(m_global) if "image" in want else None
        g_u = self._empty(out_global, (3,)) if "warp" in want else None
        gat = np.zeros(12)
        A9, t3 = _mat(A, 9), _mat(t, 3)
        lib.ffdp_ring_sample_bwd(self.h, _ptrs(upstream), _ptrs(m_shards), _dims(m_global), _ptrs(u_shards),
                                 _dims(out_global),
                                 None if A9 is None else A9.ctypes.data_as(C.POINTER(C.c_double)),
                                 None if t3 is None else t3.ctypes.data_as(C.POINTER(C.c_double)), mask,
                                 _ptrs(g_img) if g_img else None, _ptrs(g_u) if g_u else None,
                                 gat.ctypes.data_as(C.POINTER(C.c_double)))
        return (g_img, g_u, gat[:9].reshape(3, 3) if "affine" in want else None,
                gat[9:].copy() if "translation" in want else None)

    def dist_mse(self, f, moved, global_shape, n_total: Optional[int] = None):
        self._check(f, "dist_mse")
        self._check(moved, "dist_mse")
        g = [torch.empty_like(m) for m in moved]
        loss = C.c_double()
        n = n_total or int(np.prod(global_shape[:3]))
        lib.ffdp_dist_mse(self.h, _ptrs(f), _ptrs(moved), _dims(global_shape), n, C.byref(loss), _ptrs(g))
        return loss.value, g

    def dist_mi(self, f, moved, global_shape, kernel, approx_forward: bool = False, n_total: Optional[int] = None):
        """-> (loss = -MI, grads, payload elements)."""
        self._check(f, "dist_mi")
        self._check(moved, "dist_mi")
        g = [torch.empty_like(m) for m in moved]
        loss, payload = C.c_double(), C.c_int64()
        n = n_total or int(np.prod(global_shape[:3]))
        lib.ffdp_dist_mi(self.h, _ptrs(f), _ptrs(moved), _dims(global_shape), C.byref(kernel.c), int(approx_forward),
                         n, C.byref(loss), _ptrs(g), C.byref(payload))
        return loss.value, g, payload.value

    def dist_lncc(self, f, moved, global_shape, window: int = 7, eps: float = 1e-5, ants_approx: bool = True,
                  gp_sync: bool = True, n_total: Optional[int] = None):
        self._check(f, "dist_lncc")
        self._check(moved, "dist_lncc")
        g = [torch.empty_like(m) for m in moved]
        loss = C.c_double()
        lib.ffdp_dist_lncc(self.h, _ptrs(f), _ptrs(moved), _dims(global_shape), window, eps, int(ants_approx),
                           int(gp_sync), n_total or 0, C.byref(loss), _ptrs(g))
        return loss.value, g

    def step(self, f, m, u, global_shape, A=None, t=None, params=None):
        """ffdp_dist_step: the fused deformable step over the ranks -> (loss, g_u slabs)."""
        from . import voxreg as V
        p = params or V.LossParams()
        p.validate()
        for x, n in ((f, "f"), (m, "m"), (u, "u")):
            self._check(x, f"dist_step ({n})")
        if not V.fused_step_covers(p):
            # MSE, exact-mode LNCC, other windows, approximate MI: the reference's own
            # composition over the collectives (registration.hpp:277-312)
            gshape = tuple(global_shape)
            moved = self.ring_sample(m, gshape, u, gshape, A, t)
            if p.kind == "mse":
                loss, gm = self.dist_mse(f, moved, gshape)
            elif p.kind == "lncc":
                loss, gm = self.dist_lncc(f, moved, gshape, p.window, p.epsilon, p.ants_approx)
            else:
                loss, gm, _ = self.dist_mi(f, moved, gshape, p.make_kernel(), p.mi_approx_forward)
            _, g_u, _, _ = self.ring_sample_backward(gm, m, gshape, u, gshape, A, t, want=("warp",))
            return loss, g_u
        g = [torch.empty_like(x) for x in u]
        loss = C.c_double()
        A9, t3 = _mat(A, 9), _mat(t, 3)
        k = p.make_kernel() if p.kind == "mi" else None
        lib.ffdp_dist_step(self.h, 0 if p.kind == "lncc" else 1, _ptrs(f), _ptrs(m), _ptrs(u), _dims(global_shape),
                           None if A9 is None else A9.ctypes.data_as(C.POINTER(C.c_double)),
                           None if t3 is None else t3.ctypes.data_as(C.POINTER(C.c_double)), p.window, p.epsilon,
                           None if k is None else C.byref(k.c), C.byref(loss), _ptrs(g))
        return loss.value, g

    def warp_update(self, u, g_u, states, lr_norm: float, global_shape, sigma_grad: float = 1.0,
                    sigma_warp: float = 0.5):
        """The warp update of one iteration on the ranks' slabs (registration.hpp:313-317):
        g_u halo exchange, ffdp_sobolev_adam per rank (u, m1, m2 in place), then the
        halo'd warp smoothing (ffdp_dist_gp_convolve). Bit-identical to one GPU."""
        from . import voxreg as V
        from ._lib import Slab
        for x, n in ((u, "u"), (g_u, "g_u")):
            self._check(x, f"warp_update ({n})")
        tg, tw = V.gaussian_taps(sigma_grad), V.gaussian_taps(sigma_warp)
        g_h, lo, hi = self.halo_exchange(g_u, global_shape, len(tg) // 2)
        nz = int(global_shape[0])
        for r in range(self.world):
            a, b = self.shard_range(nz, r)
            st = states[r]
            st.step += 1
            with torch.cuda.device(self.devices[r]):
                lib.ffdp_sobolev_adam(V._ptr(g_h[r]), V._ptr(u[r]), V._ptr(st.m1), V._ptr(st.m2),
                                      V._dims(g_h[r].shape), Slab(a - lo[r], g_h[r].shape[0], a, b, nz),
                                      V._taps_ptr(tg), len(tg), lr_norm, st.beta1, st.beta2, st.eps, st.step,
                                      V._stream())
        return self.gp_convolve(u, tw, global_shape, "renormalize")

    def gather(self, slabs, device=None) -> torch.Tensor:
        """gather_volume / gather_warp (fabric.hpp:102-132) onto one device."""
        dev = device if device is not None else slabs[0].device
        return torch.cat([s.to(dev) for s in slabs], 0)


def comm_deformable_stage(fixed: torch.Tensor, moving: torch.Tensor, affine, schedule, devices: Sequence[int],
                          trace=None, scale_index_base: int = 0) -> torch.Tensor:
    """deformable_stage (registration.hpp:230-331) with shards = len(devices), all ranks in
    this process (the reference's own WorkerGroup model): per scale the resampled F, M and
    warp are scattered to the ranks, each iteration runs ffdp_dist_step and the sharded
    warp update, and the slabs are gathered at the end of the scale."""
    from . import registration as R
    from . import voxreg as V
    schedule.validate()
    A, t = (np.eye(3), np.zeros(3)) if affine is None else (np.asarray(affine[0]), np.asarray(affine[1]))
    world = len(devices)
    warp = None
    with Comm(world, list(devices)) as c:
        for s, step in enumerate(schedule.steps):
            factor = 1.0 / step.downsample
            f_s = fixed if factor == 1.0 else R.resample_scale(fixed, factor)
            m_s = moving if factor == 1.0 else R.resample_scale(moving, factor)
            shape = tuple(f_s.shape)
            if shape[0] < world:
                raise InvalidArgument(f"deformable_stage: {shape[0]} planes for {world} shards")
            warp = R.resample_warp(warp, shape) if warp is not None else torch.zeros(shape + (3,), device=fixed.device)
            fs, ms, us = c.scatter(f_s), c.scatter(m_s), c.scatter(warp)
            states = [V.AdamState.zeros(x) for x in us]
            lr_norm = V.deformable_lr_norm(shape, schedule.lr)
            scale_trace = []
            for it in range(step.iterations):
                loss, g = c.step(fs, ms, us, shape, A, t, schedule.loss)
                if not np.isfinite(loss):
                    # the finished scales' trace only (registration.hpp:318-325)
                    raise R.NumericalError("deformable stage diverged (non-finite loss)",
                                           list(trace) if trace else [])
                scale_trace.append(R.TraceEntry(scale_index_base + s, it, loss))
                us = c.warp_update(us, g, states, lr_norm, shape, schedule.sigma_grad, schedule.sigma_warp)
            if trace is not None:
                trace.extend(scale_trace)
            warp = c.gather(us, fixed.device)
    if tuple(warp.shape[:3]) != tuple(fixed.shape):
        warp = R.resample_warp(warp, fixed.shape)
    return warp
