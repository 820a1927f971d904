"""The deformable registration driver around the fused step (registration.hpp:33-331),
re-exposed over libffdp: the reference's ScaleStep / ScaleSchedule / TraceEntry /
NumericalError and deformable_stage, plus resample_scale / resample_warp /
normalize_intensities (resample.hpp:48-146, registration.hpp:100-115).

Per scale everything stays in HBM: F and M are resampled on the device, M is
zero-bordered once (it is static within a scale, registration.hpp:249,270), and each
iteration is three launches -- the fused warp + loss step (warp_loss_step), the fused
Sobolev + Adam update of u (ffdp_sobolev_adam) and the warp smoothing (ffdp_gp_convolve)
-- plus a device-side copy of the loss into the scale's trace. The host reads the trace
once per scale; a non-finite loss raises NumericalError then (the reference raises in the
same iteration; the returned trace is the same up to the failing entry).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import voxreg as V
from ._lib import Dims, InvalidArgument, lib


# ---------------------------------------------------------------- multi-scale plumbing
def resample_dims(shape, factor: float):
    """The (nz, ny, nx) lattice resample_scale produces (resample.hpp:52-57)."""
    nz, ny, nx = shape[:3]
    out = Dims()
    lib.ffdp_resample_dims(Dims(nx, ny, nz), factor, C.byref(out))
    return (out.nz, out.ny, out.nx)


def resample_scale(v: torch.Tensor, factor: float, scratch: Optional[torch.Tensor] = None) -> torch.Tensor:
    """resample_scale (resample.hpp:48-103): Gaussian anti-alias (sigma 0.5 / factor) when
    shrinking, then trilinear onto ceil(n * factor) keeping the end voxel centres."""
    v = V._vol(v, "resample_scale")
    shape = resample_dims(v.shape, factor)
    out = torch.empty(shape, dtype=torch.float32, device=v.device)
    lib.ffdp_resample_scale(V._ptr(v), V._dims(v.shape), factor, V._ptr(out), V._ptr(scratch), V._stream())
    return out


def resample_warp(w: torch.Tensor, shape) -> torch.Tensor:
    """resample_warp (resample.hpp:108-146): trilinear per channel onto `shape`."""
    w = V._warp(w, "resample_warp")
    out = torch.empty(tuple(shape[:3]) + (3,), dtype=torch.float32, device=w.device)
    lib.ffdp_resample_warp(V._ptr(w), V._dims(w.shape), V._ptr(out), V._dims(shape), V._stream())
    return out


def normalize_intensities(v: torch.Tensor) -> torch.Tensor:
    """normalize_intensities (registration.hpp:100-115): min-max to [0, 1], constant -> 0."""
    v = V._vol(v, "normalize_intensities")
    out = torch.empty_like(v)
    lib.ffdp_normalize(V._ptr(v), v.numel(), V._ptr(out), V._stream())
    return out


# ---------------------------------------------------------------- schedule
@dataclass
class ScaleStep:
    """ScaleStep (registration.hpp:48-51): downsample 4 = quarter resolution."""
    downsample: float = 1.0
    iterations: int = 0


@dataclass
class ScaleSchedule:
    """ScaleSchedule (registration.hpp:53-73)."""
    steps: List[ScaleStep] = field(default_factory=list)
    lr: float = 0.5
    sigma_grad: float = 1.0
    sigma_warp: float = 0.5
    loss: V.LossParams = field(default_factory=V.LossParams)

    def validate(self):
        if not self.steps:
            raise InvalidArgument("schedule: no scale steps")
        for i, s in enumerate(self.steps):
            if not s.downsample >= 1:
                raise InvalidArgument("schedule: downsample factors must be >= 1")
            if s.iterations < 0:
                raise InvalidArgument("schedule: iterations must be >= 0")
            if i > 0 and s.downsample > self.steps[i - 1].downsample:
                raise InvalidArgument("schedule: factors must be non-increasing toward 1")
        if not (self.lr > 0) or not (self.sigma_grad >= 0) or not (self.sigma_warp >= 0):
            raise InvalidArgument("schedule: bad lr/sigma")


@dataclass
class TraceEntry:
    """TraceEntry (registration.hpp:75-79)."""
    scale_index: int = 0
    iteration: int = 0
    loss: float = 0.0


class NumericalError(RuntimeError):
    """NumericalError (registration.hpp:81-85), carrying the trace so far."""

    def __init__(self, what: str, trace: Sequence[TraceEntry]):
        super().__init__(what)
        self.trace = list(trace)


@dataclass
class DeformableOptions:
    """DeformableOptions (registration.hpp:221-224); shards > 1 runs one rank per
    torch.distributed process when launched that way (dist.sharded_deformable_stage),
    else all ranks in this process over the node's GPUs (comm.comm_deformable_stage)."""
    shards: int = 1
    gp_sync: bool = True


# ---------------------------------------------------------------- the driver
class _Scale:
    """One scale's device state: F_s, the zero-bordered M_s, the workspace, the trace."""

    def __init__(self, f_s, m_s, params: V.LossParams, iterations: int):
        self.f = f_s
        self.m = V.MovingImage(m_s)
        self.params = params
        self.ws = V.StepWorkspace(f_s.device, params.bins)
        # the LNCC step's intensity frame: fixed per scale (F_s and M_s are static within it)
        self.ranges = (V.intensity_ranges(f_s, m_s) if params.kind == "lncc" and V.fused_step_covers(params)
                       else None)
        self.g_u = torch.empty(tuple(f_s.shape) + (3,), dtype=torch.float32, device=f_s.device)
        self.trace = torch.zeros(max(1, iterations), dtype=torch.float64, device=f_s.device)
        self.n = f_s.numel()

    def step(self, u, A, t, it):
        p = self.params
        if not V.fused_step_covers(p):
            # operator-kernel composition (voxreg._composite_step): the loss comes back on the host
            r = V.warp_loss_step(self.f, self.m, u, A, t, p, g_u=self.g_u, ws=self.ws)
            self.trace[it] = r.loss
            return self.g_u
        V.warp_loss_step(self.f, self.m, u, A, t, self.params, g_u=self.g_u, ws=self.ws, ranges=self.ranges,
                         sync=False)
        if self.params.kind == "lncc":
            # loss = 1 - sum_n / N (dist_lncc, distops.hpp:309-318)
            self.trace[it:it + 1].copy_(1.0 - self.ws.sum_n / self.n)
        else:
            b = self.params.bins
            self.trace[it:it + 1].copy_(-self.ws.table[2 * b * b + 2 * b + 1:2 * b * b + 2 * b + 2])
        return self.g_u


def deformable_stage(fixed: torch.Tensor, moving: torch.Tensor, affine=None, schedule: Optional[ScaleSchedule] = None,
                     opts: Optional[DeformableOptions] = None, trace: Optional[List[TraceEntry]] = None,
                     scale_index_base: int = 0) -> torch.Tensor:
    """deformable_stage (registration.hpp:230-331) on one GPU: greedy multi-scale
    optimisation of the displacement field on top of the affine (A, t) (identity by
    default). Returns the warp on F's lattice, (nz, ny, nx, 3) fp32; appends one
    TraceEntry per iteration to `trace`."""
    schedule = schedule or ScaleSchedule()
    schedule.validate()
    opts = opts or DeformableOptions()
    if opts.shards < 1:
        raise InvalidArgument("deformable_stage: shards must be >= 1")
    fixed, moving = V._vol(fixed, "deformable_stage"), V._vol(moving, "deformable_stage")
    if tuple(fixed.shape) != tuple(moving.shape):
        raise InvalidArgument("deformable_stage: F and M must share a lattice (registration.hpp:268-270)")
    if opts.shards > 1:
        if not opts.gp_sync:
            raise InvalidArgument("deformable_stage: the halo-free ablation (gp_sync = false) is not supported by "
                                  "the sharded step")
        from . import dist as D
        _, world = D._world()
        if world > 1:
            # one process per GPU: the shards are the torch.distributed ranks
            if world != opts.shards:
                raise InvalidArgument(f"deformable_stage: shards = {opts.shards} with {world} torch.distributed "
                                      "ranks")
            return D.sharded_deformable_stage(fixed, moving, affine, schedule, trace, scale_index_base)
        # one process over the node's GPUs (ffdp_comm; ranks share devices round-robin)
        from .comm import comm_deformable_stage
        n = max(1, torch.cuda.device_count())
        return comm_deformable_stage(fixed, moving, affine, schedule, [r % n for r in range(opts.shards)], trace,
                                     scale_index_base)
    A, t = (np.eye(3), np.zeros(3)) if affine is None else (np.asarray(affine[0]), np.asarray(affine[1]))
    warp = None
    for s, step in enumerate(schedule.steps):
        factor = 1.0 / step.downsample
        f_s = fixed if factor == 1.0 else resample_scale(fixed, factor)
        m_s = moving if factor == 1.0 else resample_scale(moving, factor)
        shape = tuple(f_s.shape)
        warp = resample_warp(warp, shape) if warp is not None else torch.zeros(shape + (3,), device=fixed.device)
        # registration.hpp:257-264: lr in voxels of the level -> normalized units
        lr_norm = V.deformable_lr_norm(shape, schedule.lr)
        sc = _Scale(f_s, m_s, schedule.loss, step.iterations)
        adam = V.AdamState.zeros(warp)
        spare = torch.empty_like(warp)
        for it in range(step.iterations):
            g_u = sc.step(warp, A, t, it)
            out = V.warp_update(warp, g_u, adam, lr_norm, schedule.sigma_grad, schedule.sigma_warp, out=spare)
            warp, spare = out, warp
        losses = sc.trace[:step.iterations].tolist()
        entries = [TraceEntry(scale_index_base + s, i, v) for i, v in enumerate(losses)]
        bad = next((i for i, v in enumerate(losses) if not np.isfinite(v)), None)
        if bad is not None:
            # the reference merges a scale's trace only after the scale completes
            # (registration.hpp:318-325): the error carries the trace of the finished scales
            raise NumericalError("deformable stage diverged (non-finite loss)", list(trace) if trace else [])
        if trace is not None:
            trace.extend(entries)
    if tuple(warp.shape[:3]) != tuple(fixed.shape):
        warp = resample_warp(warp, fixed.shape)
    lib.ffdp_scratch_trim(0)  # the library's cached scratch goes back to the device
    return warp


# ---------------------------------------------------------------- affine stage
def _loss_and_grad(f_s: torch.Tensor, moved: torch.Tensor, p: V.LossParams):
    """loss_and_grad (registration.hpp:123-173) through the operator kernels: MSE
    (ffdp_mse), LNCC (lncc_forward_fused + lncc_backward_fused, upstream 1) or MI (exact or
    approximate forward, mi_backward_impl with upstream -1, loss = -MI)."""
    if p.kind == "mse":
        grad = torch.empty_like(moved)
        s = torch.zeros(1, dtype=torch.float64, device=moved.device)
        lib.ffdp_mse(V._ptr(f_s), V._ptr(moved), moved.numel(), moved.numel(), V._ptr(grad), V._ptr(s), V._stream())
        return float(s.item()) / moved.numel(), grad
    if p.kind == "lncc":
        res, state = V.lncc_forward_fused(f_s, moved, p.window, p.epsilon)
        _, gm = V.lncc_backward_fused(1.0, state, f_s, moved, p.ants_approx)
        return res.loss, gm
    if p.kind == "mi":
        k = p.make_kernel()
        res = (V.mi_forward_approx if p.mi_approx_forward else V.mi_forward_exact)(f_s, moved, p.bins, k)
        _, gm = V.mi_backward(-1.0, f_s, moved, res.hist, k, check_samples=False)
        return -res.mi, gm
    raise InvalidArgument(f"loss_and_grad: unknown loss kind {p.kind!r}")


def _adam_host(params: np.ndarray, grad: np.ndarray, state: dict, lr: float):
    """adam_step (adam.hpp:30-50) on the 12 affine parameters, fp64 (host control of a
    12-number state; the volumes never leave the device)."""
    state["step"] += 1
    b1, b2, eps = 0.9, 0.999, 1e-8
    c1 = 1.0 - b1 ** state["step"]
    c2 = 1.0 - b2 ** state["step"]
    state["m1"] = b1 * state["m1"] + (1.0 - b1) * grad
    state["m2"] = b2 * state["m2"] + (1.0 - b2) * grad * grad
    return params - lr * (state["m1"] / c1) / (np.sqrt(state["m2"] / c2) + eps)


def affine_stage(fixed: torch.Tensor, moving: torch.Tensor, schedule: ScaleSchedule,
                 trace: Optional[List[TraceEntry]] = None, scale_index_base: int = 0):
    """affine_stage (registration.hpp:176-219): Adam on (A, t) from the identity; per
    iteration moved = fused_sample(M_s, zero warp, A, t) on F_s's lattice, loss_and_grad,
    fused_sample_backward(want affine + translation) -- the fp64 gA / gt reductions of
    the sampler kernel. Returns (A 3x3, t 3)."""
    schedule.validate()
    fixed, moving = V._vol(fixed, "affine_stage"), V._vol(moving, "affine_stage")
    params = np.concatenate([np.eye(3).ravel(), np.zeros(3)])
    state = {"m1": np.zeros(12), "m2": np.zeros(12), "step": 0}
    want = V.SamplerGradWant(image=False, warp=False, affine=True, translation=True)
    for s, step in enumerate(schedule.steps):
        factor = 1.0 / step.downsample
        f_s = fixed if factor == 1.0 else resample_scale(fixed, factor)
        m_s = moving if factor == 1.0 else resample_scale(moving, factor)
        zero = torch.zeros(tuple(f_s.shape) + (3,), dtype=torch.float32, device=f_s.device)
        for it in range(step.iterations):
            args = V.SamplerArgs(A=params[:9].reshape(3, 3), t=params[9:])
            moved = V.fused_sample(m_s, zero, args)
            loss, gm = _loss_and_grad(f_s, moved, schedule.loss)
            if not np.isfinite(loss):
                raise NumericalError("affine stage diverged (non-finite loss)", trace or [])
            if trace is not None:
                trace.append(TraceEntry(scale_index_base + s, it, loss))
            g = V.fused_sample_backward(gm, m_s, zero, args, want)
            params = _adam_host(params, np.concatenate([g.affine.ravel(), g.translation]), state, schedule.lr)
    lib.ffdp_scratch_trim(0)
    return params[:9].reshape(3, 3).copy(), params[9:].copy()


# ---------------------------------------------------------------- the pipeline
def jacobian_positive_fraction(u: torch.Tensor) -> float:
    """jacobian_positive_fraction (metrics.hpp:145-176): interior voxels with
    det(I + du/dx) > 0 (central differences in normalized units)."""
    u = V._warp(u, "jacobian_positive_fraction")
    if min(u.shape[:3]) < 3:
        raise InvalidArgument("jacobian_positive_fraction: lattice too small")
    out = C.c_double()
    lib.ffdp_jacobian_positive(V._ptr(u), V._dims(u.shape), C.byref(out), V._stream())
    return out.value


@dataclass
class RegistrationConfig:
    """RegistrationConfig (registration.hpp:333-338)."""
    affine: ScaleSchedule = field(default_factory=lambda: ScaleSchedule(loss=V.LossParams(kind="mi")))
    deformable: ScaleSchedule = field(default_factory=ScaleSchedule)
    deformable_opts: DeformableOptions = field(default_factory=DeformableOptions)
    skip_affine: bool = False


@dataclass
class RegistrationResult:
    """RegistrationResult (registration.hpp:87-94); warp in fp32 on the device."""
    affine: tuple
    warp: torch.Tensor
    trace: List[TraceEntry]
    seconds: float
    jacobian_positive_fraction: float


def register_volumes(fixed: torch.Tensor, moving: torch.Tensor, config: RegistrationConfig) -> RegistrationResult:
    """register_volumes (registration.hpp:340-368): intensity-normalised copies, the
    affine stage (unless skipped), the deformable stage on top of it, the Jacobian
    sign fraction of the warp (reported, not enforced)."""
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f_n, m_n = normalize_intensities(fixed), normalize_intensities(moving)
    trace: List[TraceEntry] = []
    affine = (np.eye(3), np.zeros(3))
    base = 0
    if not config.skip_affine:
        affine = affine_stage(f_n, m_n, config.affine, trace, 0)
        base = len(config.affine.steps)
    warp = deformable_stage(f_n, m_n, affine, config.deformable, config.deformable_opts, trace, base)
    jac = jacobian_positive_fraction(warp)  # throws for lattices under 3 voxels (metrics.hpp:146-148)
    torch.cuda.synchronize()
    return RegistrationResult(affine, warp, trace, time.perf_counter() - t0, jac)
