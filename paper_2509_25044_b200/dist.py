"""Z-slab sharding of the fused warp + loss step over GPUs of one node
(fabric.hpp:31-132, distops.hpp:36-396), one process per GPU over torch.distributed
(NCCL on B200s, gloo on CPU for the host-logic tests).

The reference rotates every moving-image shard around the ring twice per iteration
(ring_sample / ring_sample_backward, distops.hpp:144-248) and sums zero-padded partial
interpolations. The interpolation those partials add up to is the global one, so here
each rank keeps a *window* of moving-image planes -- its own slab plus the planes its
warped samples reach -- fetched once per scale (the moving image is static within a
scale, registration.hpp:249,270) and widened only when the kernels report a window
miss, after which the step is simply re-run (exact). Per iteration the only traffic is
the displacement halo the LNCC window needs (r planes of u from each neighbour; F's halo
is static) and the reductions: one double for LNCC (distops.hpp:309-318) or the B*B
joint histogram for MI (distops.hpp:365-373, the marginals are not consumed).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from ._lib import InvalidArgument, Slab


# ------------------------------------------------------------------ sharding rules
def shard_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """shard_ranges (fabric.hpp:44-57): contiguous z ranges, the first n % world shards
    one plane longer."""
    if world < 1 or n < world:
        raise InvalidArgument("shard_ranges: need 1 <= world <= axis size")
    base, extra = divmod(n, world)
    out, lo = [], 0
    for h in range(world):
        size = base + (1 if h < extra else 0)
        out.append((lo, lo + size))
        lo += size
    return out


def axis_coord(i: int, n: int) -> float:
    """axis_coord (geometry.hpp:106-109)."""
    if n <= 1:
        return -1.0
    return -1.0 + 2.0 * (float(i) / float(n - 1))


@dataclass
class ShardSpec:
    """ShardSpec (fabric.hpp:31-42); dims are (nz, ny, nx) like the tensors."""
    rank: int = 0
    world: int = 1
    lo: int = 0
    hi: int = 0
    global_shape: Tuple[int, int, int] = (0, 0, 0)
    x_min: Tuple[float, float, float] = (-1.0, -1.0, -1.0)
    x_max: Tuple[float, float, float] = (1.0, 1.0, 1.0)

    @property
    def thickness(self) -> int:
        return self.hi - self.lo

    @property
    def local_shape(self) -> Tuple[int, int, int]:
        return (self.hi - self.lo, self.global_shape[1], self.global_shape[2])


def make_shard_spec(global_shape: Sequence[int], world: int, rank: int) -> ShardSpec:
    """make_shard_spec (fabric.hpp:59-70): bounds in the global normalized frame."""
    nz = int(global_shape[0])
    lo, hi = shard_ranges(nz, world)[rank]
    return ShardSpec(rank, world, lo, hi, tuple(int(s) for s in global_shape), (-1.0, -1.0, axis_coord(lo, nz)),
                     (1.0, 1.0, axis_coord(hi - 1, nz)))


@dataclass
class ShardRescale:
    """ShardRescale (distops.hpp:36-39)."""
    S: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    t: Tuple[float, float, float] = (0.0, 0.0, 0.0)


def compute_shard_rescale(x_min, x_max, g_min=(-1.0, -1.0, -1.0), g_max=(1.0, 1.0, 1.0)) -> ShardRescale:
    """compute_shard_rescale (distops.hpp:41-49): S*x_min + t = g_min, S*x_max + t = g_max."""
    S = tuple((g_max[c] - g_min[c]) / (x_max[c] - x_min[c]) for c in range(3))
    t = tuple(g_min[c] - S[c] * x_min[c] for c in range(3))
    return ShardRescale(S, t)


# ------------------------------------------------------------------ collectives
def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def _staged() -> bool:
    """gloo moves CPU tensors only: CUDA tensors are staged through host memory (used to
    run the sharded path with several ranks on one GPU; NCCL moves device memory)."""
    return dist.is_initialized() and dist.get_backend() == "gloo"


def _p2p(ops_spec):
    """ops_spec: list of (kind, tensor, peer), kind 'send'|'recv'. Runs them as one batch,
    staging CUDA tensors through the host under gloo."""
    staged = _staged()
    ops, back = [], []
    for kind, t, peer in ops_spec:
        buf = t
        if staged and t.is_cuda:
            buf = t.detach().cpu() if kind == "send" else torch.empty(t.shape, dtype=t.dtype)
            if kind == "recv":
                back.append((t, buf))
        elif kind == "send":
            buf = t.contiguous()
        ops.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, buf, peer))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for t, buf in back:
        t.copy_(buf)


def _collective(fn, t: torch.Tensor, *a, **kw):
    if _staged() and t.is_cuda:
        h = t.detach().cpu()
        fn(h, *a, **kw)
        t.copy_(h)
        return t
    fn(t, *a, **kw)
    return t


def all_reduce(t: torch.Tensor, op=None) -> torch.Tensor:
    """dist.all_reduce that also runs under gloo on CUDA tensors (host staging)."""
    return _collective(dist.all_reduce, t, op=op if op is not None else dist.ReduceOp.SUM)


def halo_exchange(slab: torch.Tensor, spec: ShardSpec, pad: int) -> Tuple[torch.Tensor, int, int]:
    """halo_exchange (fabric.hpp:315-370): the slab with up to `pad` planes from each
    neighbour along z (dim 0); rank 0 has no left halo, the last rank no right halo.
    Returns (padded, halo_lo, halo_hi). Raises like the reference when pad exceeds a
    neighbour's thickness."""
    if pad < 0:
        raise InvalidArgument("halo_exchange: pad must be >= 0")
    w, r = spec.world, spec.rank
    if pad == 0 or w == 1:
        return slab, 0, 0
    ranges = shard_ranges(spec.global_shape[0], w)
    if r > 0 and pad > ranges[r - 1][1] - ranges[r - 1][0]:
        raise InvalidArgument("halo_exchange: pad exceeds left neighbor thickness")
    if r < w - 1 and pad > ranges[r + 1][1] - ranges[r + 1][0]:
        raise InvalidArgument("halo_exchange: pad exceeds right neighbor thickness")
    lo = pad if r > 0 else 0
    hi = pad if r < w - 1 else 0
    out = torch.empty((slab.shape[0] + lo + hi,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
    out[lo:lo + slab.shape[0]].copy_(slab)
    ops = []
    if r > 0:  # my first planes become the left neighbour's right halo, and vice versa
        ops.append(("send", slab[:pad], r - 1))
        ops.append(("recv", out[:lo], r - 1))
    if r < w - 1:
        ops.append(("send", slab[slab.shape[0] - pad:], r + 1))
        ops.append(("recv", out[lo + slab.shape[0]:], r + 1))
    _p2p(ops)
    return out, lo, hi


def allreduce_sum(t: torch.Tensor, ordered: bool = False) -> torch.Tensor:
    """allreduce_sum (fabric.hpp:246-263). ordered=True reproduces the reference's
    rank-ordered summation bit for bit (all-gather, then sum in rank order); the default
    is the collective's own reduction (payloads here are <= 8.7 KB)."""
    _, w = _world()
    if w == 1:
        return t
    if not ordered:
        return all_reduce(t)
    src = t.detach().cpu() if (_staged() and t.is_cuda) else t
    parts = [torch.empty_like(src) for _ in range(w)]
    dist.all_gather(parts, src)
    acc = torch.zeros_like(src)
    for p in parts:
        acc += p
    t.copy_(acc)
    return t


def fetch_planes(slab: torch.Tensor, spec: ShardSpec, z0: int, z1: int) -> torch.Tensor:
    """Global planes [z0, z1) of a z-sharded volume, gathered from their owners (every
    rank calls collectively with its own request). Used to build the moving-image window;
    the reference's equivalent is the ring rotation of whole shards (distops.hpp:154-166)."""
    r, w = spec.rank, spec.world
    nz = spec.global_shape[0]
    z0, z1 = max(0, int(z0)), min(nz, int(z1))
    out = torch.zeros((max(0, z1 - z0),) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
    if w == 1:
        out.copy_(slab[z0 - spec.lo:z1 - spec.lo])
        return out
    req = torch.tensor([z0, z1], dtype=torch.int64, device="cpu" if (_staged() or not slab.is_cuda) else slab.device)
    reqs = [torch.empty_like(req) for _ in range(w)]
    dist.all_gather(reqs, req)
    reqs = [tuple(int(v) for v in q.tolist()) for q in reqs]
    ranges = shard_ranges(nz, w)
    ops = []
    for peer in range(w):
        # what I send to peer: my planes inside peer's request
        a, b = max(reqs[peer][0], spec.lo), min(reqs[peer][1], spec.hi)
        if peer != r and a < b:
            ops.append(("send", slab[a - spec.lo:b - spec.lo], peer))
        # what I receive from peer: peer's planes inside my request
        plo, phi = ranges[peer]
        a2, b2 = max(z0, plo), min(z1, phi)
        if peer != r and a2 < b2:
            ops.append(("recv", out[a2 - z0:b2 - z0], peer))
    a, b = max(z0, spec.lo), min(z1, spec.hi)
    if a < b:
        out[a - z0:b - z0].copy_(slab[a - spec.lo:b - spec.lo])
    _p2p(ops)
    return out


# ------------------------------------------------------------------ the sharded step
class ShardedStep:
    """The deformable step (registration.hpp:277-312) on one rank's z slab.

    Constructed once per scale with the rank's F and M slabs; `step(u_slab)` returns
    (loss, g_u_slab) with the loss reduced over all ranks. The per-GPU compute is the
    same fused kernel as the single-GPU path, run on the slab with its halo planes."""

    R = 3  # LNCC window radius (window 7)

    def __init__(self, f_slab: torch.Tensor, m_slab: torch.Tensor, spec: ShardSpec, A=None, t=None,
                 params=None, margin_planes: int = 8):
        from . import voxreg
        self.V = voxreg
        self.params = params or voxreg.LossParams()
        self.params.validate()
        self.fused = voxreg.fused_step_covers(self.params)
        self.spec = spec
        self.A = np.eye(3) if A is None else np.asarray(A, dtype=np.float64).reshape(3, 3)
        self.t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64)
        self.f = f_slab.to(torch.float32).contiguous()
        self.m = m_slab.to(torch.float32).contiguous()
        self.pad = self.R if self.params.kind == "lncc" else 0
        self.f_halo, self.hlo, self.hhi = halo_exchange(self.f, spec, self.pad)
        self.ws = voxreg.StepWorkspace(self.f.device, self.params.bins)
        self.margin = int(margin_planes)
        self.m_z0 = self.m_z1 = None
        self.window_fetches = 0
        self.ranges = None

    def reload(self, f_slab: torch.Tensor = None, m_slab: torch.Tensor = None):
        """New image contents of the same geometry (a new pair, or a new scale's resampled
        images): refreshes the F halo planes, drops the moving window and the intensity ranges."""
        if f_slab is not None:
            self.f.copy_(f_slab)
            self.f_halo, self.hlo, self.hhi = halo_exchange(self.f, self.spec, self.pad)
        if m_slab is not None:
            self.m.copy_(m_slab)
        self.m_z0 = self.m_z1 = None
        self.ranges = None

    # -- moving window ------------------------------------------------------------------
    def _ensure_window(self, z0: int, z1: int):
        nz = self.spec.global_shape[0]
        z0, z1 = max(0, z0), min(nz, z1)
        if self.m_z0 is not None and self.m_z0 <= z0 and self.m_z1 >= z1:
            return
        # the window request is collective: agree on widening across ranks
        lohi = torch.tensor([z0, z1], dtype=torch.int64, device=self.f.device)
        planes = fetch_planes(self.m, self.spec, int(lohi[0]), int(lohi[1]))
        nzw = planes.shape[0]
        pad = torch.zeros((nzw + 4, planes.shape[1] + 4, planes.shape[2] + 4), dtype=torch.float32,
                          device=self.f.device)
        pad[2:-2, 2:-2, 2:-2].copy_(planes)
        self.m_pad, self.m_z0, self.m_z1 = pad, z0, z1
        self.window_fetches += 1

    def _affine_z_range(self, z0: int, z1: int) -> Tuple[int, int]:
        """Moving planes [a, b) the affine part of the warp maps lattice planes [z0, z1)
        into (z_src = A[2] . x + t[2] is linear, so the slab's corners bound it); the
        displacement's reach is covered by the margin and, past it, by the miss retry."""
        nz = self.spec.global_shape[0]
        zs = []
        for zz in (axis_coord(z0, nz), axis_coord(z1 - 1, nz)):
            for xx in (-1.0, 1.0):
                for yy in (-1.0, 1.0):
                    zn = self.A[2, 0] * xx + self.A[2, 1] * yy + self.A[2, 2] * zz + self.t[2]
                    zs.append((zn + 1.0) * 0.5 * (nz - 1))
        return int(math.floor(min(zs))) - 1, int(math.ceil(max(zs))) + 2

    def _window(self):
        from ._lib import Dims, ImageWindow
        nz, ny, nx = self.spec.global_shape
        return ImageWindow(self.m_pad.data_ptr(), Dims(nx, ny, nz), self.m_z0, self.m_z1, 2)

    # -- the step -------------------------------------------------------------------------
    def step(self, u_slab: torch.Tensor, max_retries: int = 4, check_miss: bool = True, sync: bool = True):
        """One sharded step: (loss, g_u_slab). check_miss=False skips the per-step window
        agreement (one MAX-allreduce + host read): misses then accumulate on the device
        and verify_no_miss() must be called before the results are trusted (the bench's
        timed loop does this after the loop). sync=False returns the loss as a device
        tensor (no host read)."""
        V, p, spec = self.V, self.params, self.spec
        u_slab = u_slab.to(torch.float32).contiguous()
        if not self.fused:
            return self._composite(u_slab, sync)
        u_h, lo, hi = halo_exchange(u_slab, spec, self.pad)
        nzl = spec.thickness
        ny, nx = spec.global_shape[1], spec.global_shape[2]
        slab = Slab(spec.lo - lo, nzl + lo + hi, spec.lo, spec.hi, spec.global_shape[0])
        dims = V._dims((nzl + lo + hi, ny, nx))
        args = V.SamplerArgs(A=self.A, t=self.t).to_c()
        n_total = spec.global_shape[0] * ny * nx
        g_u = torch.empty_like(u_slab)
        if self.m_z0 is None:
            a, b = self._affine_z_range(spec.lo - lo, spec.hi + hi)
            self._ensure_window(a - self.margin, b + self.margin)
        if p.kind == "lncc" and self.ranges is None:
            # one intensity frame on every rank (it fixes the fixed-point moment arithmetic)
            mm = torch.stack([self.f.min(), -self.f.max(), self.m.min(), -self.m.max()]).to(torch.float32)
            if spec.world > 1:
                all_reduce(mm, op=dist.ReduceOp.MIN)
            self.ranges = mm * torch.tensor([1.0, -1.0, 1.0, -1.0], device=mm.device)
        from ._lib import lib
        for attempt in range(max_retries + 1):
            if check_miss:
                self.ws.miss.zero_()
            win = self._window()
            stream = V._stream()
            if p.kind == "lncc":
                self.ws.sum_n.zero_()
                lib.ffdp_step_lncc(V._ptr(self.f_halo), V._ptr(u_h), dims, slab, win, C.byref(args), p.window,
                                   p.epsilon, -1.0 / n_total, V._ptr(self.ranges), V._ptr(g_u),
                                   V._ptr(self.ws.sum_n), V._ptr(self.ws.miss),
                                   V._ptr(self.ws.lncc_workspace(dims, slab)), stream)
            else:
                k = p.make_kernel()
                self.ws.raw.zero_()
                if k.kind == V.PARZEN_BSPLINE3:
                    rec = self.ws.records(dims, slab)
                    lib.ffdp_step_mi_hist_rec(V._ptr(self.f_halo), V._ptr(u_h), dims, slab, win, C.byref(args),
                                              C.byref(k.c), V._ptr(self.ws.raw), V._ptr(self.ws.scratch), V._ptr(rec),
                                              V._ptr(self.ws.miss), stream)
                else:
                    lib.ffdp_step_mi_hist(V._ptr(self.f_halo), V._ptr(u_h), dims, slab, win, C.byref(args),
                                          C.byref(k.c), V._ptr(self.ws.raw), V._ptr(self.ws.scratch),
                                          V._ptr(self.ws.miss), stream)
            if not check_miss:
                break
            # a miss on any rank means the step has to be redone everywhere (collective agreement)
            miss = self.ws.miss.to(torch.int64)
            if spec.world > 1:
                all_reduce(miss, op=dist.ReduceOp.MAX)
            if int(miss.item()) == 0:
                break
            ext = torch.empty(2, dtype=torch.int64, device=self.f.device)
            lib.ffdp_sampler_z_extent(V._ptr(u_h), dims, V._dims(spec.global_shape), C.byref(
                V.SamplerArgs(A=self.A, t=self.t, bounds=V.DomainBounds(
                    (-1.0, -1.0, axis_coord(spec.lo - lo, spec.global_shape[0])),
                    (1.0, 1.0, axis_coord(spec.hi + hi - 1, spec.global_shape[0])))).to_c()), V._ptr(ext), stream)
            e = ext.tolist()
            self.m_z0 = None
            self._ensure_window(min(e[0], spec.lo) - 1, max(e[1], spec.hi) + 2)
        else:
            raise RuntimeError("ShardedStep: moving window kept missing")
        if p.kind == "lncc":
            s = allreduce_sum(self.ws.sum_n)
            return (1.0 - float(s.item()) / n_total if sync else 1.0 - s / n_total), g_u
        b = p.bins
        allreduce_sum(self.ws.raw[:b * b])
        lib.ffdp_mi_finalize(V._ptr(self.ws.raw), b, -1.0, V._ptr(self.ws.table), V._stream())
        k = p.make_kernel()
        if k.kind == V.PARZEN_BSPLINE3:
            lib.ffdp_step_mi_grad_rec(V._ptr(self.f_halo), dims, slab, C.byref(k.c), V._ptr(self.ws.table),
                                      V._ptr(self.ws.records(dims, slab)), V._ptr(g_u), V._stream())
        else:
            lib.ffdp_step_mi_grad(V._ptr(self.f_halo), V._ptr(u_h), dims, slab, self._window(), C.byref(args),
                                  C.byref(k.c), V._ptr(self.ws.table), V._ptr(g_u), V._ptr(self.ws.miss), V._stream())
        lv = -self.ws.table[2 * b * b + 2 * b + 1:2 * b * b + 2 * b + 2]
        return (float(lv.item()) if sync else lv), g_u

    def _composite(self, u_slab: torch.Tensor, sync: bool):
        """The losses the fused kernels do not cover (MSE, exact-mode LNCC, windows other
        than 7, approximate MI), composed from the collective operators exactly as the
        reference's step does (registration.hpp:277-312): ring_sample -> dist_mse |
        dist_lncc | dist_mi -> ring_sample_backward(want warp)."""
        p, spec = self.params, self.spec
        gshape = spec.global_shape
        n_total = gshape[0] * gshape[1] * gshape[2]
        moved = ring_sample(self.m, u_slab, self.A, self.t, gshape, spec)
        if p.kind == "mse":
            dl = dist_mse(self.f, moved, n_total)
        elif p.kind == "lncc":
            dl = dist_lncc(spec, self.f, moved, p.window, p.epsilon, p.ants_approx, True, n_total)
        else:
            dl = dist_mi(self.f, moved, p.bins, p.make_kernel(), p.mi_approx_forward, n_total)
        g = ring_sample_backward(dl.grad_moved, self.m, u_slab, self.A, self.t, gshape, spec,
                                 self.V.SamplerGradWant(warp=True))
        loss = dl.loss if sync else torch.tensor([dl.loss], dtype=torch.float64, device=u_slab.device)
        return loss, g.warp

    def verify_no_miss(self):
        """After steps run with check_miss=False: raise unless no rank saw a window miss
        since the last checked step (then every such step was exact)."""
        miss = self.ws.miss.to(torch.int64)
        if self.spec.world > 1:
            all_reduce(miss, op=dist.ReduceOp.MAX)
        if int(miss.item()) != 0:
            raise RuntimeError("ShardedStep: a window miss occurred in an unchecked step")
        self.ws.miss.zero_()


# ------------------------------------------------------------------ warp update
def sharded_warp_update(u_slab: torch.Tensor, g_u_slab: torch.Tensor, state, spec: ShardSpec, lr_norm: float,
                        sigma_grad: float = 1.0, sigma_warp: float = 0.5) -> torch.Tensor:
    """The warp update of one deformable iteration on a z-slab (registration.hpp:313-317):
    halo_exchange of g_u (the gaussian radius, fabric.hpp:315-370), ffdp_sobolev_adam
    (gp_convolve(g_u, renormalize) fused with adam_step, distops.hpp:54-101 /
    adam.hpp:30-50) on the slab, halo_exchange of the updated u and ffdp_gp_convolve of
    it. The taps depend only on global planes, so the result equals the unsharded update.
    u_slab, state.m1 and state.m2 are updated in place; returns the smoothed u slab."""
    from . import voxreg as V
    from ._lib import lib
    u_slab = V._warp(u_slab, "warp_update")
    g_u_slab = V._warp(g_u_slab, "warp_update")
    nz_g, ny, nx = spec.global_shape
    tg, tw = V.gaussian_taps(sigma_grad), V.gaussian_taps(sigma_warp)
    g_h, lo, hi = halo_exchange(g_u_slab, spec, len(tg) // 2)
    slab = Slab(spec.lo - lo, spec.thickness + lo + hi, spec.lo, spec.hi, nz_g)
    state.step += 1
    lib.ffdp_sobolev_adam(V._ptr(g_h), V._ptr(u_slab), V._ptr(state.m1), V._ptr(state.m2),
                          V._dims(g_h.shape), slab, V._taps_ptr(tg), len(tg), lr_norm, state.beta1, state.beta2,
                          state.eps, state.step, V._stream())
    u_h, lo, hi = halo_exchange(u_slab, spec, len(tw) // 2)
    slab = Slab(spec.lo - lo, spec.thickness + lo + hi, spec.lo, spec.hi, nz_g)
    out = torch.empty_like(u_slab)
    lib.ffdp_gp_convolve(V._ptr(u_h), V._ptr(out), V._dims(u_h.shape), slab, 3, V._taps_ptr(tw), len(tw), 1,
                         V._stream())
    return out


def _gather_slabs(slab: torch.Tensor, spec: ShardSpec) -> torch.Tensor:
    """gather_warp / gather_volume (fabric.hpp:108-132): the full field on every rank
    (slabs padded to the thickest one for the equal-size all_gather, then trimmed)."""
    if spec.world == 1:
        return slab
    ranges = shard_ranges(spec.global_shape[0], spec.world)
    tmax = max(hi - lo for lo, hi in ranges)
    src = torch.zeros((tmax,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
    src[:slab.shape[0]].copy_(slab)
    if _staged():
        parts = [torch.empty_like(src, device="cpu") for _ in ranges]
        dist.all_gather(parts, src.cpu())
        parts = [p.to(slab.device) for p in parts]
    else:
        parts = [torch.empty_like(src) for _ in ranges]
        dist.all_gather(parts, src)
    return torch.cat([p[:hi - lo] for p, (lo, hi) in zip(parts, ranges)], 0)


def sharded_deformable_stage(fixed: torch.Tensor, moving: torch.Tensor, affine, schedule, trace=None,
                             scale_index_base: int = 0, margin_planes: int = 8) -> torch.Tensor:
    """deformable_stage (registration.hpp:230-331) with shards = world size, one rank per
    GPU: every rank resamples the scale's F and M (the reference's workers do the same
    from the shared volumes, 247-249) and keeps its z slab (make_shard_spec, 266-270);
    per iteration ShardedStep (ring window, halo, allreduced loss / histogram) and
    sharded_warp_update (halo-exchanged Sobolev + Adam + smoothing); the slabs are
    gathered at the end of each scale (gather_warp, 323). Returns the full warp on every
    rank; `trace` (rank-identical losses) gets one TraceEntry per iteration."""
    from . import registration as R
    from . import voxreg as V
    schedule.validate()
    rank, world = _world()
    A, t = (np.eye(3), np.zeros(3)) if affine is None else (np.asarray(affine[0]), np.asarray(affine[1]))
    warp = None
    for s, step in enumerate(schedule.steps):
        factor = 1.0 / step.downsample
        f_s = fixed if factor == 1.0 else R.resample_scale(fixed, factor)
        m_s = moving if factor == 1.0 else R.resample_scale(moving, factor)
        shape = tuple(f_s.shape)
        warp = R.resample_warp(warp, shape) if warp is not None else torch.zeros(shape + (3,), device=fixed.device)
        spec = make_shard_spec(shape, world, rank)
        sl = slice(spec.lo, spec.hi)
        st = ShardedStep(f_s[sl], m_s[sl], spec, A, t, schedule.loss, margin_planes=margin_planes)
        u = warp[sl].contiguous()
        adam = V.AdamState.zeros(u)
        lr_norm = V.deformable_lr_norm(shape, schedule.lr)
        scale_trace = []
        for it in range(step.iterations):
            loss, g_u = st.step(u)
            if not np.isfinite(loss):
                # the finished scales' trace only (registration.hpp:318-325)
                raise R.NumericalError("deformable stage diverged (non-finite loss)", list(trace) if trace else [])
            scale_trace.append(R.TraceEntry(scale_index_base + s, it, loss))
            u = sharded_warp_update(u, g_u, adam, spec, lr_norm, schedule.sigma_grad, schedule.sigma_warp)
        if trace is not None:
            trace.extend(scale_trace)
        warp = _gather_slabs(u, spec)
    if tuple(warp.shape[:3]) != tuple(fixed.shape):
        warp = R.resample_warp(warp, fixed.shape)
    return warp


# ------------------------------------------------------------------ standalone sharded operators
# The reference's collective operator API (distops.hpp:54-396) one call at a time: every
# rank calls in the same order. They compose the operator kernels with the exchanges; the
# fused ShardedStep is the fast path for the deformable step itself.
@dataclass
class DistLoss:
    """DistLoss (distops.hpp:251-257)."""
    loss: float
    grad_moved: torch.Tensor
    mi_payload_elements: int = 0


@dataclass
class RingSampleGrads:
    """RingSampleGrads (distops.hpp:170-176): gradients for the rank's own shards."""
    image: Optional[torch.Tensor] = None
    warp: Optional[torch.Tensor] = None
    affine: Optional[np.ndarray] = None
    translation: Optional[np.ndarray] = None


def _args_for(out_spec: ShardSpec, A, t):
    from . import voxreg as V
    nz = out_spec.global_shape[0]
    lo = (-1.0, -1.0, axis_coord(out_spec.lo, nz))
    hi = (1.0, 1.0, axis_coord(out_spec.hi - 1, nz))
    return V.SamplerArgs(A=np.eye(3) if A is None else A, t=np.zeros(3) if t is None else t,
                         bounds=V.DomainBounds(lo, hi))


def _moving_window(m_shard: torch.Tensor, u_shard: torch.Tensor, args, m_global_dims, out_spec: ShardSpec):
    """The moving planes the rank's samples touch (ffdp_sampler_z_extent over its u slab,
    exact), gathered from their owners: (planes, zero-bordered copy, z0, z1, m_spec)."""
    from . import voxreg as V
    from ._lib import lib
    m_spec = make_shard_spec(m_global_dims, out_spec.world, out_spec.rank)
    ext = torch.empty(2, dtype=torch.int64, device=u_shard.device)
    lib.ffdp_sampler_z_extent(V._ptr(u_shard), V._dims(u_shard.shape), V._dims(m_global_dims),
                              C.byref(args.to_c()), V._ptr(ext), V._stream())
    lo, hi = ext.tolist()
    z0, z1 = (lo, hi + 1) if lo <= hi else (0, 0)
    planes = fetch_planes(m_shard, m_spec, z0, z1)
    z0, z1 = max(0, z0), max(0, z0) + planes.shape[0]
    pad = torch.zeros((planes.shape[0] + 4, planes.shape[1] + 4, planes.shape[2] + 4), dtype=torch.float32,
                      device=m_shard.device)
    pad[2:-2, 2:-2, 2:-2].copy_(planes)
    return planes, pad, z0, z1, m_spec


def ring_sample(m_shard: torch.Tensor, u_shard: torch.Tensor, A, t, m_global_dims, out_spec: ShardSpec) -> torch.Tensor:
    """ring_sample (distops.hpp:144-168): the moved image on the rank's output slab. The
    reference rotates every moving shard around the ring and sums zero-padded partial
    interpolations; their sum is the global interpolation, computed here from the moving
    planes the slab's samples actually touch (fetched once, exact)."""
    from . import voxreg as V
    from ._lib import Dims, ImageWindow, lib
    u_shard = V._warp(u_shard, "ring_sample")
    m_shard = V._vol(m_shard, "ring_sample")
    args = _args_for(out_spec, A, t)
    args.validate()
    _, pad, z0, z1, _ = _moving_window(m_shard, u_shard, args, m_global_dims, out_spec)
    nz, ny, nx = m_global_dims
    win = ImageWindow(pad.data_ptr(), Dims(nx, ny, nz), z0, z1, 2)
    out = torch.empty(tuple(u_shard.shape[:3]), dtype=torch.float32, device=u_shard.device)
    lib.ffdp_sampler_fwd(win, V._ptr(u_shard), V._dims(u_shard.shape), C.byref(args.to_c()), V._ptr(out), 0, None,
                         None, V._stream())
    return out


def ring_sample_backward(upstream: torch.Tensor, m_shard: torch.Tensor, u_shard: torch.Tensor, A, t, m_global_dims,
                         out_spec: ShardSpec, want) -> RingSampleGrads:
    """ring_sample_backward (distops.hpp:179-248): gradients w.r.t. the rank's u slab, its
    moving shard (image contributions routed back to the owning ranks, 230-239) and the
    affine / translation (allreduced, 241-246)."""
    from . import voxreg as V
    from ._lib import Dims, ImageWindow, lib
    u_shard = V._warp(u_shard, "ring_sample_backward")
    m_shard = V._vol(m_shard, "ring_sample_backward")
    upstream = V._vol(upstream, "ring_sample_backward")
    args = _args_for(out_spec, A, t)
    args.validate()
    planes, pad, z0, z1, m_spec = _moving_window(m_shard, u_shard, args, m_global_dims, out_spec)
    nz, ny, nx = m_global_dims
    win = ImageWindow(pad.data_ptr(), Dims(nx, ny, nz), z0, z1, 2)
    g = RingSampleGrads()
    dev = u_shard.device
    g_img = torch.zeros((nz, ny, nx), dtype=torch.float32, device=dev) if want.image else None
    g_win = torch.zeros((z1 - z0, ny, nx), dtype=torch.float32, device=dev) if want.image else None
    if want.warp:
        g.warp = torch.empty(tuple(u_shard.shape), dtype=torch.float32, device=dev)
    gat = torch.zeros(12, dtype=torch.float64, device=dev) if (want.affine or want.translation) else None
    if want.image and z1 > z0:
        # the image gradient lands on the window's planes: sample through the unpadded
        # window so g_img shares its dense layout
        wimg = ImageWindow(planes.data_ptr(), Dims(nx, ny, nz), z0, z1, 0)
        lib.ffdp_sampler_bwd(V._ptr(upstream), wimg, V._ptr(u_shard), V._dims(u_shard.shape), C.byref(args.to_c()),
                             V.WANT_IMAGE, V._ptr(g_win), None, None, None, V._stream())
        g_img[z0:z1] += g_win
    if want.warp or gat is not None:
        mask = (V.WANT_WARP if want.warp else 0) | (V.WANT_AFFINE if want.affine else 0) | \
               (V.WANT_TRANSLATION if want.translation else 0)
        lib.ffdp_sampler_bwd(V._ptr(upstream), win, V._ptr(u_shard), V._dims(u_shard.shape), C.byref(args.to_c()),
                             mask, None, V._ptr(g.warp), V._ptr(gat), None, V._stream())
    if want.image:
        all_reduce(g_img)  # every rank's window contributions, summed at the owners' planes
        g.image = g_img[m_spec.lo:m_spec.hi].contiguous()
    if gat is not None:
        all_reduce(gat)
        h = gat.cpu().numpy()
        if want.affine:
            g.affine = h[:9].reshape(3, 3).copy()
        if want.translation:
            g.translation = h[9:].copy()
    return g


def gp_convolve(slab: torch.Tensor, taps, spec: ShardSpec, mode: str = "zero_pad", sync: bool = True) -> torch.Tensor:
    """gp_convolve (distops.hpp:84-101): the separable convolution of a z-sharded volume or
    warp with the neighbours' halo planes (sync), or of the shard treated as a standalone
    volume along z (sync = False, the ablation)."""
    from . import voxreg as V
    from ._lib import Slab
    taps = np.ascontiguousarray(taps, dtype=np.float64)
    if taps.size % 2 == 0:
        raise InvalidArgument("gp_convolve: kernel must be odd")
    slab = slab.to(torch.float32).contiguous()
    r = taps.size // 2
    if not sync or spec.world == 1 or r == 0:
        return V.gp_convolve(slab, taps, mode)
    h, lo, hi = halo_exchange(slab, spec, r)
    return V.gp_convolve(h, taps, mode, slab=Slab(spec.lo - lo, slab.shape[0] + lo + hi, spec.lo, spec.hi,
                                                  spec.global_shape[0]))


def dist_mse(f_shard: torch.Tensor, moved_shard: torch.Tensor, n_total: int) -> DistLoss:
    """dist_mse (distops.hpp:260-282): allreduced sum of squares over N_total, grad 2 d / N."""
    from . import voxreg as V
    from ._lib import lib
    f, m = V._vol(f_shard, "dist_mse"), V._vol(moved_shard, "dist_mse")
    if tuple(f.shape) != tuple(m.shape):
        raise InvalidArgument("dist_mse: shard lattices differ")
    s = torch.zeros(1, dtype=torch.float64, device=f.device)
    g = torch.empty_like(m)
    lib.ffdp_mse(V._ptr(f), V._ptr(m), f.numel(), n_total, V._ptr(g), V._ptr(s), V._stream())
    s = allreduce_sum(s)
    return DistLoss(float(s.item()) / n_total, g)


def dist_mi(f_shard: torch.Tensor, moved_shard: torch.Tensor, bins: int, kernel, approx_forward: bool,
            n_total: int) -> DistLoss:
    """dist_mi (distops.hpp:355-396): local raw histograms, allreduced (B*B + 2B payload,
    365-373), finalize, loss = -MI, mi_backward_impl on the local shard with upstream -1."""
    from . import voxreg as V
    from ._lib import lib
    f, m = V._vol(f_shard, "dist_mi"), V._vol(moved_shard, "dist_mi")
    if tuple(f.shape) != tuple(m.shape):
        raise InvalidArgument("dist_mi: shard lattices differ")
    b = bins
    raw = torch.zeros(b * b + 2 * b, dtype=torch.float64, device=f.device)
    lib.ffdp_mi_hist(V._ptr(f), V._ptr(m), f.numel(), C.byref(kernel.c), int(approx_forward), V._ptr(raw), None,
                     None, V._stream())
    raw = allreduce_sum(raw)
    table = torch.empty(2 * b * b + 2 * b + 4, dtype=torch.float64, device=f.device)
    lib.ffdp_mi_finalize(V._ptr(raw), b, -1.0, V._ptr(table), V._stream())
    g = torch.empty_like(m)
    lib.ffdp_mi_bwd(V._ptr(f), V._ptr(m), f.numel(), C.byref(kernel.c), V._ptr(table), None, V._ptr(g), V._stream())
    return DistLoss(-float(table[2 * b * b + 2 * b + 1].item()), g, b * b + 2 * b)


def dist_lncc(spec: ShardSpec, f_shard: torch.Tensor, moved_shard: torch.Tensor, window: int = 7, eps: float = 1e-5,
              ants_approx: bool = True, gp_sync: bool = True, n_total: Optional[int] = None) -> DistLoss:
    """dist_lncc (distops.hpp:285-352): the five window moments over the slab with the
    neighbours' halo planes (r = window // 2; 2r for the exact backward, whose gamma family
    is box-filtered again), sum_n allreduced, loss = 1 - sum_n / N_total, dL/dn_i = -1/N."""
    from . import voxreg as V
    from ._lib import Slab, lib
    f, m = V._vol(f_shard, "dist_lncc"), V._vol(moved_shard, "dist_lncc")
    if tuple(f.shape) != tuple(m.shape):
        raise InvalidArgument("dist_lncc: shard lattices differ")
    if window < 1 or window % 2 == 0:
        raise InvalidArgument("lncc: window must be odd and >= 1")
    n_total = n_total or spec.global_shape[0] * f.shape[1] * f.shape[2]
    r = window // 2
    sync = gp_sync and spec.world > 1
    nz_g = spec.global_shape[0] if sync else f.shape[0]
    g_lo = spec.lo if sync else 0
    pad = (r if ants_approx else 2 * r) if sync else 0
    fh, lo, hi = halo_exchange(f, spec, pad) if sync else (f, 0, 0)
    mh, _, _ = halo_exchange(m, spec, pad) if sync else (m, 0, 0)
    dims = V._dims(fh.shape)
    nint = f.numel()
    plane = f.shape[1] * f.shape[2]
    s = torch.zeros(1, dtype=torch.float64, device=f.device)
    state = torch.empty((5,) + tuple(f.shape), dtype=torch.float64, device=f.device)
    interior = Slab(g_lo - lo, fh.shape[0], g_lo, g_lo + f.shape[0], nz_g)
    lib.ffdp_lncc_fwd(V._ptr(fh), V._ptr(mh), dims, interior, window, eps, V._ptr(state), None, V._ptr(s),
                      V._stream())
    s = allreduce_sum(s)
    loss = 1.0 - float(s.item()) / n_total
    g = torch.empty_like(m)
    gi = -1.0 / n_total
    if ants_approx:
        lib.ffdp_lncc_gamma(V._ptr(state), nint, eps, gi, V._stream())
        lib.ffdp_lncc_combine(V._ptr(state), V._dims(f.shape), V._full_slab(f.shape[0]), window, 1,
                              V._ptr(f), V._ptr(m), None, V._ptr(g), V._stream())
        return DistLoss(loss, g)
    # exact: the gamma family on the slab +- r planes (inside the lattice; the 2r halo holds
    # their windows), box-filtered again (lncc.hpp:249-263). One exchange of 2r planes where
    # the reference exchanges r planes twice (neighbours must be >= 2r planes thick).
    e0 = max(0, g_lo - r)
    e1 = min(nz_g, g_lo + f.shape[0] + r)
    ext = Slab(g_lo - lo, fh.shape[0], e0, e1, nz_g)
    next_ = (e1 - e0) * plane
    st_ext = torch.empty((5, e1 - e0) + tuple(f.shape[1:]), dtype=torch.float64, device=f.device)
    lib.ffdp_lncc_fwd(V._ptr(fh), V._ptr(mh), dims, ext, window, eps, V._ptr(st_ext), None, None, V._stream())
    lib.ffdp_lncc_gamma(V._ptr(st_ext), next_, eps, gi, V._stream())
    gslab = Slab(e0, e1 - e0, g_lo, g_lo + f.shape[0], nz_g)
    lib.ffdp_lncc_combine(V._ptr(st_ext), V._dims((e1 - e0,) + tuple(f.shape[1:])), gslab, window, 0, V._ptr(f),
                          V._ptr(m), None, V._ptr(g), V._stream())
    return DistLoss(loss, g)
