"""The reference's single-host operator API (voxreg, /root/reference/proj/include/voxreg)
re-exposed over libffdp's sm_100a kernels.

Same names, argument meanings and error behaviour as the C++ templates, on CUDA
tensors: volumes are float32 ``(nz, ny, nx)`` (x fastest, volume.hpp:3-7), warp fields
float32 ``(nz, ny, nx, 3)`` (interleaved, volume.hpp:57). Results are fresh tensors
(the reference returns owning containers). Errors raise ``InvalidArgument`` (a
``ValueError``) where the reference throws ``std::invalid_argument``,
``LogicError`` for ``std::logic_error``.

The deformable step's hot path is :func:`warp_loss_step` (one fused pass for LNCC,
two passes for MI); the per-operator functions exist for drop-in use and parity.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np
import torch

from ._lib import (PARZEN_BSPLINE3, PARZEN_DELTA, PARZEN_GAUSSIAN, WANT_AFFINE, WANT_IMAGE, WANT_TRANSLATION,
                   WANT_WARP, Dims, ImageWindow, InvalidArgument, ParzenC, SamplerArgsC, Slab, lib)

__all__ = [
    "DomainBounds", "SamplerArgs", "SamplerGradWant", "SamplerGrads", "fused_sample", "fused_sample_accumulate",
    "fused_sample_backward", "LnccState", "LnccResult", "lncc_forward_fused", "lncc_backward_fused",
    "ParzenKernel", "JointHistogram", "MiStats", "MiResult", "mi_forward_exact", "mi_forward_approx", "mi_backward",
    "LossParams", "StepResult", "warp_loss_step", "convolve_axis", "box_taps", "gaussian_taps",
    "gp_convolve", "AdamState", "adam_step", "warp_update", "deformable_lr_norm",
]


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _vol(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dim() != 3:
        raise InvalidArgument(f"{what}: expected a (nz, ny, nx) tensor")
    if not t.is_cuda:
        raise InvalidArgument(f"{what}: expected a CUDA tensor")
    if any(s < 1 for s in t.shape):
        raise InvalidArgument("Volume3: dims must be positive")
    return t.to(torch.float32).contiguous()


def _warp(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dim() != 4 or t.shape[3] != 3:
        raise InvalidArgument(f"{what}: expected a (nz, ny, nx, 3) tensor")
    if not t.is_cuda:
        raise InvalidArgument(f"{what}: expected a CUDA tensor")
    return t.to(torch.float32).contiguous()


def _dims(shape) -> Dims:
    nz, ny, nx = shape[:3]
    return Dims(nx, ny, nz)


def _window(img: torch.Tensor) -> ImageWindow:
    nz = img.shape[0]
    return ImageWindow(img.data_ptr(), _dims(img.shape), 0, nz, 0)


class MovingImage:
    """A moving image in the zero-bordered layout (2 voxels of zeros on every side) that
    the fused step kernels gather from without bounds checks (ffdp_pad_window). The
    border realises the reference's zero padding (sampler.hpp:106-110). The moving image
    is static within a scale (registration.hpp:249,270), so the padded copy is made once
    per scale and reused by every iteration."""

    def __init__(self, m: torch.Tensor):
        m = _vol(m, "MovingImage")
        self.shape = tuple(m.shape)
        nz, ny, nx = self.shape
        self.padded = torch.empty((nz + 4, ny + 4, nx + 4), dtype=torch.float32, device=m.device)
        lib.ffdp_pad_window(_ptr(m), _dims(m.shape), 0, nz, _ptr(self.padded), _stream())

    @property
    def interior(self) -> torch.Tensor:
        """View of the volume inside the border (copy new data into it in place)."""
        return self.padded[2:-2, 2:-2, 2:-2]

    def window(self) -> ImageWindow:
        return ImageWindow(self.padded.data_ptr(), _dims(self.shape), 0, self.shape[0], 2)


def _full_slab(nz: int) -> Slab:
    return Slab(0, nz, 0, nz, nz)


# ---------------------------------------------------------------- geometry / sampler
@dataclass
class DomainBounds:
    """DomainBounds (geometry.hpp:74-86): normalized coords of the first/last voxel centres."""
    x_min: Tuple[float, float, float] = (-1.0, -1.0, -1.0)
    x_max: Tuple[float, float, float] = (1.0, 1.0, 1.0)

    @staticmethod
    def full() -> "DomainBounds":
        return DomainBounds()

    def valid(self) -> bool:
        return all(a < b for a, b in zip(self.x_min, self.x_max))


@dataclass
class SamplerArgs:
    """SamplerArgs (sampler.hpp:25-37): A (row-major 3x3), t, S (displacement rescale), bounds."""
    A: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))
    S: np.ndarray = field(default_factory=lambda: np.ones(3))
    bounds: DomainBounds = field(default_factory=DomainBounds)

    def validate(self):
        """sampler.hpp:31-36 (the C ABI re-checks)."""
        if not np.all(np.isfinite(np.asarray(self.A, dtype=np.float64))):
            raise InvalidArgument("SamplerArgs: non-finite affine")
        if not np.all(np.asarray(self.S, dtype=np.float64) > 0):
            raise InvalidArgument("SamplerArgs: S must be positive")
        if not self.bounds.valid():
            raise InvalidArgument("SamplerArgs: invalid bounds")

    def to_c(self) -> SamplerArgsC:
        a = SamplerArgsC()
        A = np.asarray(self.A, dtype=np.float64).reshape(9)
        for i in range(9):
            a.A[i] = float(A[i])
        for i in range(3):
            a.t[i] = float(np.asarray(self.t, dtype=np.float64).reshape(3)[i])
            a.S[i] = float(np.asarray(self.S, dtype=np.float64).reshape(3)[i])
            a.x_min[i] = float(self.bounds.x_min[i])
            a.x_max[i] = float(self.bounds.x_max[i])
        return a


@dataclass
class SamplerGradWant:
    """SamplerGradWant (sampler.hpp:39-44)."""
    image: bool = False
    warp: bool = False
    affine: bool = False
    translation: bool = False

    def mask(self) -> int:
        return ((WANT_IMAGE if self.image else 0) | (WANT_WARP if self.warp else 0) |
                (WANT_AFFINE if self.affine else 0) | (WANT_TRANSLATION if self.translation else 0))


@dataclass
class SamplerGrads:
    """SamplerGrads (sampler.hpp:46-52); absent gradients are None."""
    image: Optional[torch.Tensor] = None
    warp: Optional[torch.Tensor] = None
    affine: Optional[np.ndarray] = None
    translation: Optional[np.ndarray] = None


def sampler_output_shape(img: torch.Tensor, u: Optional[torch.Tensor]):
    """sampler_output_dims (sampler.hpp:248-251): u's lattice when given, else I's."""
    return tuple(u.shape[:3]) if u is not None else tuple(img.shape)


def fused_sample(img: torch.Tensor, u: Optional[torch.Tensor], args: SamplerArgs) -> torch.Tensor:
    """fused_sample (sampler.hpp:254-263): I(A X + t + S u(X)), trilinear, zero padding."""
    img = _vol(img, "fused_sample")
    u = None if u is None else _warp(u, "fused_sample")
    args.validate()
    out = torch.empty(sampler_output_shape(img, u), dtype=torch.float32, device=img.device)
    ca = args.to_c()
    lib.ffdp_sampler_fwd(_window(img), _ptr(u), _dims(out.shape), C.byref(ca), _ptr(out), 0, None, None, _stream())
    return out


def fused_sample_accumulate(img: torch.Tensor, u: Optional[torch.Tensor], args: SamplerArgs, out: torch.Tensor,
                            abs_contribution: bool = False) -> Optional[float]:
    """fused_sample_accumulate (sampler.hpp:268-276): out += sample; optionally returns the
    L1 mass of this call's contribution (RingSampleStats, distops.hpp:137-139)."""
    img = _vol(img, "fused_sample_accumulate")
    u = None if u is None else _warp(u, "fused_sample_accumulate")
    if tuple(out.shape) != sampler_output_shape(img, u):
        raise InvalidArgument("fused_sample_accumulate: output lattice mismatch")
    if out.dtype != torch.float32 or not out.is_contiguous():
        raise InvalidArgument("fused_sample_accumulate: output must be contiguous float32")
    args.validate()
    acc = torch.zeros(1, dtype=torch.float64, device=img.device) if abs_contribution else None
    ca = args.to_c()
    lib.ffdp_sampler_fwd(_window(img), _ptr(u), _dims(out.shape), C.byref(ca), _ptr(out), 1, _ptr(acc), None,
                         _stream())
    return float(acc.item()) if acc is not None else None


def fused_sample_backward(upstream: torch.Tensor, img: torch.Tensor, u: Optional[torch.Tensor], args: SamplerArgs,
                          want: SamplerGradWant) -> SamplerGrads:
    """fused_sample_backward (sampler.hpp:279-300)."""
    img = _vol(img, "fused_sample_backward")
    u = None if u is None else _warp(u, "fused_sample_backward")
    upstream = _vol(upstream, "fused_sample_backward")
    od = sampler_output_shape(img, u)
    if tuple(upstream.shape) != od:
        raise InvalidArgument("fused_sample_backward: upstream lattice mismatch")
    args.validate()
    g = SamplerGrads()
    dev = img.device
    if want.image:
        g.image = torch.zeros(img.shape, dtype=torch.float32, device=dev)
    if want.warp:
        g.warp = torch.empty(od + (3,), dtype=torch.float32, device=dev)
    gat = torch.zeros(12, dtype=torch.float64, device=dev) if (want.affine or want.translation) else None
    ca = args.to_c()
    lib.ffdp_sampler_bwd(_ptr(upstream), _window(img), _ptr(u), _dims(od), C.byref(ca), want.mask(), _ptr(g.image),
                         _ptr(g.warp), _ptr(gat), None, _stream())
    if gat is not None:
        h = gat.cpu().numpy()
        if want.affine:
            g.affine = h[:9].reshape(3, 3).copy()
        if want.translation:
            g.translation = h[9:].copy()
    return g


# ---------------------------------------------------------------- smoothing
def box_taps(window: int) -> np.ndarray:
    """box_taps (smoothing.hpp:42-46)."""
    if window < 1 or window % 2 == 0:
        raise InvalidArgument("box_taps: window must be odd and >= 1")
    return np.full(window, 1.0 / window)


def gaussian_taps(sigma: float) -> np.ndarray:
    """gaussian_taps (smoothing.hpp:25-39): truncated at ceil(3 sigma), sum 1."""
    if not np.isfinite(sigma) or sigma < 0:
        raise InvalidArgument("gaussian_taps: sigma must be finite and >= 0")
    if sigma == 0:
        return np.ones(1)
    r = int(np.ceil(3.0 * sigma))
    k = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (k / sigma) * (k / sigma))
    return w / w.sum()


def convolve_axis(x: torch.Tensor, axis: int, taps, renormalize: bool = False, lo_global: int = 0,
                  n_global: Optional[int] = None) -> torch.Tensor:
    """convolve_axis (smoothing.hpp:52-94) for a volume (nz,ny,nx) or warp (nz,ny,nx,3)."""
    x = x.to(torch.float32).contiguous()
    ch = 3 if x.dim() == 4 else 1
    taps = np.ascontiguousarray(taps, dtype=np.float64)
    if n_global is None:
        n_global = x.shape[2 - axis]
    out = torch.empty_like(x)
    lib.ffdp_convolve_axis(_ptr(x), _ptr(out), _dims(x.shape), ch, axis, taps.ctypes.data_as(C.POINTER(C.c_double)),
                           len(taps), 1 if renormalize else 0, lo_global, n_global, _stream())
    return out


def _taps_ptr(taps: np.ndarray):
    return taps.ctypes.data_as(C.POINTER(C.c_double))


def gp_convolve(x: torch.Tensor, taps, mode: str = "zero_pad", slab: Optional[Slab] = None) -> torch.Tensor:
    """gp_convolve / separable_convolve (distops.hpp:84-101, smoothing.hpp:98-105): x, y, z
    passes of `taps` over a volume (nz,ny,nx) or warp (nz,ny,nx,3), EdgeMode "zero_pad" or
    "renormalize". One z-marching kernel (ffdp_gp_convolve). With a slab, x holds the
    buffer planes (incl. the halo) and the result the slab's interior planes."""
    if mode not in ("zero_pad", "renormalize"):
        raise InvalidArgument(f"gp_convolve: unknown edge mode {mode!r}")
    x = x.to(torch.float32).contiguous()
    ch = 3 if x.dim() == 4 else 1
    taps = np.ascontiguousarray(taps, dtype=np.float64)
    if taps.size % 2 == 0:
        raise InvalidArgument("gp_convolve: kernel must be odd")
    slab = slab or _full_slab(x.shape[0])
    out = torch.empty((slab.z_end - slab.z_begin,) + tuple(x.shape[1:]), dtype=torch.float32, device=x.device)
    lib.ffdp_gp_convolve(_ptr(x), _ptr(out), _dims(x.shape), slab, ch, _taps_ptr(taps), len(taps),
                         1 if mode == "renormalize" else 0, _stream())
    return out


@dataclass
class AdamState:
    """AdamState (adam.hpp:14-28) of a warp field: first / second moments in fp32 (the
    reference's T storage), the step counter and the hyper-parameters."""
    m1: torch.Tensor
    m2: torch.Tensor
    step: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @staticmethod
    def zeros(like: torch.Tensor) -> "AdamState":
        return AdamState(torch.zeros_like(like, dtype=torch.float32), torch.zeros_like(like, dtype=torch.float32))


def adam_step(param: torch.Tensor, grad: torch.Tensor, state: AdamState, lr: float) -> None:
    """adam_step (adam.hpp:30-50) on a warp field, in place: the Adam epilogue of
    ffdp_sobolev_adam with a single unit tap (no smoothing)."""
    param, grad = _warp(param, "adam_step"), _warp(grad, "adam_step")
    if param.shape != grad.shape or param.shape != state.m1.shape or param.shape != state.m2.shape:
        raise InvalidArgument("adam_step: shape mismatch")
    state.step += 1
    one = np.ones(1)
    lib.ffdp_sobolev_adam(_ptr(grad), _ptr(param), _ptr(state.m1), _ptr(state.m2), _dims(param.shape),
                          _full_slab(param.shape[0]), _taps_ptr(one), 1, lr, state.beta1, state.beta2, state.eps,
                          state.step, _stream())


def deformable_lr_norm(shape, lr: float) -> float:
    """registration.hpp:257-264: the learning rate in voxels of the level converted to
    normalized units by the mean voxel pitch."""
    nz, ny, nx = shape[:3]
    return lr * (2.0 / (nx - 1) + 2.0 / (ny - 1) + 2.0 / (nz - 1)) / 3.0


def warp_update(u: torch.Tensor, g_u: torch.Tensor, state: AdamState, lr_norm: float, sigma_grad: float = 1.0,
                sigma_warp: float = 0.5, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The warp update of one deformable iteration (registration.hpp:313-317) at H = 1:
    g_s = gp_convolve(g_u, gaussian_taps(sigma_grad), renormalize); adam_step(u, g_s,
    state, lr_norm) -- fused in one kernel, u updated in place -- then the returned field
    gp_convolve(u, gaussian_taps(sigma_warp), renormalize) (into `out` if given)."""
    u, g_u = _warp(u, "warp_update"), _warp(g_u, "warp_update")
    if u.shape != g_u.shape or u.shape != state.m1.shape or u.shape != state.m2.shape:
        raise InvalidArgument("adam_step: shape mismatch")
    slab = _full_slab(u.shape[0])
    tg, tw = gaussian_taps(sigma_grad), gaussian_taps(sigma_warp)
    state.step += 1
    lib.ffdp_sobolev_adam(_ptr(g_u), _ptr(u), _ptr(state.m1), _ptr(state.m2), _dims(u.shape), slab, _taps_ptr(tg),
                          len(tg), lr_norm, state.beta1, state.beta2, state.eps, state.step, _stream())
    if out is None:
        out = torch.empty_like(u)
    lib.ffdp_gp_convolve(_ptr(u), _ptr(out), _dims(u.shape), slab, 3, _taps_ptr(tw), len(tw), 1, _stream())
    return out


# ---------------------------------------------------------------- LNCC
@dataclass
class LnccState:
    """LnccState (lncc.hpp:30-35): the five box-filtered channels (fp64 on the device)."""
    channels: torch.Tensor  # (5, nz, ny, nx) float64: mean_f, mean_m, mean_ff, mean_mm, mean_fm
    window: int = 7
    epsilon: float = 1e-5
    voxels: int = 0

    @property
    def mean_f(self):
        return self.channels[0]

    @property
    def mean_m(self):
        return self.channels[1]

    @property
    def mean_ff(self):
        return self.channels[2]

    @property
    def mean_mm(self):
        return self.channels[3]

    @property
    def mean_fm(self):
        return self.channels[4]


@dataclass
class LnccResult:
    """LnccResult (lncc.hpp:37-42)."""
    loss: float = 0.0
    ncc_map: Optional[torch.Tensor] = None
    has_map: bool = False


def _check_lncc(f, m, window):
    if tuple(f.shape) != tuple(m.shape):
        raise InvalidArgument("lncc: lattices differ")
    if window < 1 or window % 2 == 0:
        raise InvalidArgument("lncc: window must be odd and >= 1")


def lncc_forward_fused(f: torch.Tensor, m: torch.Tensor, window: int = 7, eps: float = 1e-5,
                       want_map: bool = False) -> Tuple[LnccResult, LnccState]:
    """lncc_forward_fused (lncc.hpp:144-205). loss = 1 - mean(A^2 / (B C + eps))."""
    f, m = _vol(f, "lncc"), _vol(m, "lncc")
    _check_lncc(f, m, window)
    n = f.numel()
    state = torch.empty((5,) + tuple(f.shape), dtype=torch.float64, device=f.device)
    mp = torch.empty(f.shape, dtype=torch.float32, device=f.device) if want_map else None
    s = torch.zeros(1, dtype=torch.float64, device=f.device)
    lib.ffdp_lncc_fwd(_ptr(f), _ptr(m), _dims(f.shape), _full_slab(f.shape[0]), window, eps, _ptr(state), _ptr(mp),
                      _ptr(s), _stream())
    res = LnccResult(loss=1.0 - float(s.item()) / n, ncc_map=mp, has_map=want_map)
    return res, LnccState(state, window, eps, n)


def lncc_backward_fused(upstream: float, state: LnccState, f: torch.Tensor, m: torch.Tensor,
                        ants_approx: bool) -> Tuple[torch.Tensor, torch.Tensor]:
    """lncc_backward_fused (lncc.hpp:226-280). The state is consumed (rewritten in place
    as the gamma family, lncc.hpp:236-247)."""
    f, m = _vol(f, "lncc"), _vol(m, "lncc")
    if tuple(state.channels.shape[1:]) != tuple(f.shape) or tuple(f.shape) != tuple(m.shape):
        raise InvalidArgument("lncc_backward_fused: lattice mismatch")
    n = state.voxels
    gi = -upstream / float(n)
    lib.ffdp_lncc_gamma(_ptr(state.channels), n, state.epsilon, gi, _stream())
    gf = torch.empty(f.shape, dtype=torch.float32, device=f.device)
    gm = torch.empty(f.shape, dtype=torch.float32, device=f.device)
    lib.ffdp_lncc_combine(_ptr(state.channels), _dims(f.shape), _full_slab(f.shape[0]), state.window,
                          1 if ants_approx else 0, _ptr(f), _ptr(m), _ptr(gf), _ptr(gm), _stream())
    return gf, gm


# ---------------------------------------------------------------- MI
class ParzenKernel:
    """ParzenKernel (mi.hpp:28-140). Constructed through the C ABI so the normalisation
    check raises LogicError exactly where the reference throws std::logic_error."""

    GAUSSIAN, BSPLINE3, DELTA = PARZEN_GAUSSIAN, PARZEN_BSPLINE3, PARZEN_DELTA

    def __init__(self, kind: int, bins: int, sigma_bins: float = 0.5):
        self.c = ParzenC()
        lib.ffdp_parzen_make(kind, bins, sigma_bins, C.byref(self.c))

    @classmethod
    def gaussian(cls, bins: int, sigma_bins: float = 0.5) -> "ParzenKernel":
        return cls(PARZEN_GAUSSIAN, bins, sigma_bins)

    @classmethod
    def bspline3(cls, bins: int) -> "ParzenKernel":
        return cls(PARZEN_BSPLINE3, bins)

    @classmethod
    def delta(cls, bins: int) -> "ParzenKernel":
        return cls(PARZEN_DELTA, bins)

    def bins(self) -> int:
        return self.c.bins

    def support(self) -> float:
        return self.c.radius

    def support_bins(self) -> float:
        return self.c.radius * self.c.bins

    @property
    def kind(self) -> int:
        return self.c.kind


@dataclass
class JointHistogram:
    """JointHistogram (mi.hpp:146-154)."""
    bins: int = 0
    samples: int = 0
    raw_joint_sum: float = 0.0
    p_i: Optional[np.ndarray] = None
    p_j: Optional[np.ndarray] = None
    p_ij: Optional[np.ndarray] = None  # row-major [m * bins + n]
    raw_joint: Optional[np.ndarray] = None
    raw_marg_i: Optional[np.ndarray] = None
    raw_marg_j: Optional[np.ndarray] = None
    table: Optional[torch.Tensor] = None  # device: p_ij, p_i, p_j, ghat, {z, mi, dot, 0}


@dataclass
class MiStats:
    """MiStats (mi.hpp:156-159): counters of the reference's exact / hard-binning formulation."""
    hist_writes: int = 0
    kernel_evals: int = 0


@dataclass
class MiResult:
    """MiResult (mi.hpp:161-165)."""
    mi: float = 0.0
    hist: JointHistogram = field(default_factory=JointHistogram)
    stats: MiStats = field(default_factory=MiStats)


def _hist_from_raw(raw: torch.Tensor, bins: int, samples: int, upstream: float = -1.0) -> Tuple[float, JointHistogram]:
    b = bins
    table = torch.empty(2 * b * b + 2 * b + 4, dtype=torch.float64, device=raw.device)
    lib.ffdp_mi_finalize(_ptr(raw), b, upstream, _ptr(table), _stream())
    h = table.cpu().numpy()
    r = raw.cpu().numpy()
    hist = JointHistogram(bins=b, samples=samples, raw_joint_sum=float(h[2 * b * b + 2 * b]), p_ij=h[:b * b].copy(),
                          p_i=h[b * b:b * b + b].copy(), p_j=h[b * b + b:b * b + 2 * b].copy(),
                          raw_joint=r[:b * b].copy(), raw_marg_i=r[b * b:b * b + b].copy(),
                          raw_marg_j=r[b * b + b:].copy(), table=table)
    return float(h[2 * b * b + 2 * b + 1]), hist


def _mi_forward(img_i, img_j, bins, kernel: ParzenKernel, approx: bool) -> MiResult:
    img_i, img_j = _vol(img_i, "mi"), _vol(img_j, "mi")
    if tuple(img_i.shape) != tuple(img_j.shape):
        raise InvalidArgument("mi: lattices differ")
    if bins < 2:
        raise InvalidArgument("mi: bins must be >= 2")
    if bins != kernel.bins():
        raise InvalidArgument("mi: kernel bin count differs from bins")
    n = img_i.numel()
    raw = torch.zeros(bins * bins + 2 * bins, dtype=torch.float64, device=img_i.device)
    bad = torch.zeros(1, dtype=torch.int32, device=img_i.device)
    stats = (C.c_uint64 * 2)(0, 0)
    lib.ffdp_mi_hist(_ptr(img_i), _ptr(img_j), n, C.byref(kernel.c), 1 if approx else 0, _ptr(raw), _ptr(bad), stats,
                     _stream())
    if int(bad.item()):
        raise InvalidArgument("mi: intensities must lie in [0,1]")
    mi, hist = _hist_from_raw(raw, bins, n)
    return MiResult(mi=mi, hist=hist, stats=MiStats(int(stats[0]), int(stats[1])))


def mi_forward_exact(img_i, img_j, bins: int, kernel: ParzenKernel) -> MiResult:
    """mi_forward_exact (mi.hpp:235-272): exact Parzen joint histogram, MI."""
    return _mi_forward(img_i, img_j, bins, kernel, False)


def mi_forward_approx(img_i, img_j, bins: int, kernel: ParzenKernel) -> MiResult:
    """mi_forward_approx (mi.hpp:285-354): hard binning + kernel tap convolution."""
    return _mi_forward(img_i, img_j, bins, kernel, True)


def mi_backward(upstream: float, img_i, img_j, hist: JointHistogram, kernel: ParzenKernel,
                check_samples: bool = True) -> Tuple[torch.Tensor, torch.Tensor]:
    """mi_backward (mi.hpp:430-437); check_samples=False is detail::mi_backward_impl
    (mi.hpp:361, global histogram against a local block)."""
    img_i, img_j = _vol(img_i, "mi_backward"), _vol(img_j, "mi_backward")
    if tuple(img_i.shape) != tuple(img_j.shape):
        raise InvalidArgument("mi_backward: lattices differ")
    if check_samples and img_i.numel() != hist.samples:
        raise InvalidArgument("mi_backward: histogram sample count mismatch")
    b = hist.bins
    raw = torch.from_numpy(np.concatenate([hist.raw_joint, hist.raw_marg_i, hist.raw_marg_j])).to(img_i.device)
    table = torch.empty(2 * b * b + 2 * b + 4, dtype=torch.float64, device=img_i.device)
    lib.ffdp_mi_finalize(_ptr(raw), b, float(upstream), _ptr(table), _stream())
    gi = torch.empty(img_i.shape, dtype=torch.float32, device=img_i.device)
    gj = torch.empty(img_i.shape, dtype=torch.float32, device=img_i.device)
    lib.ffdp_mi_bwd(_ptr(img_i), _ptr(img_j), img_i.numel(), C.byref(kernel.c), _ptr(table), _ptr(gi), _ptr(gj),
                    _stream())
    return gi, gj


# ---------------------------------------------------------------- the fused step
@dataclass
class LossParams:
    """LossParams (registration.hpp:33-46). The fused step kernels cover LNCC (ANTs) and
    exact-forward MI; MSE, exact-mode LNCC and approximate-forward MI run through the
    operator kernels (warp_loss_step composes them)."""
    kind: str = "lncc"  # "lncc" | "mi" | "mse"
    window: int = 7
    epsilon: float = 1e-5
    ants_approx: bool = True
    bins: int = 32
    mi_bspline_kernel: bool = False  # the reference default (registration.hpp:40): Gaussian Parzen
    mi_approx_forward: bool = False

    def make_kernel(self) -> ParzenKernel:
        return ParzenKernel.bspline3(self.bins) if self.mi_bspline_kernel else ParzenKernel.gaussian(self.bins)

    def validate(self):
        """The reference's checks for the loss arguments (lncc.hpp:57-61, mi.hpp:170-176)."""
        if self.kind not in ("lncc", "mi", "mse"):
            raise InvalidArgument(f"unknown loss kind {self.kind!r}")
        if self.kind == "lncc" and (self.window < 1 or self.window % 2 == 0):
            raise InvalidArgument("lncc: window must be odd and >= 1")
        if self.kind == "mi" and self.bins < 2:
            raise InvalidArgument("mi: bins must be >= 2")


def fused_step_covers(params: "LossParams") -> bool:
    """True when the fused step kernels (ffdp_step_lncc: window 7, ANTs; ffdp_step_mi:
    exact Parzen forward) compute this loss; every other loss (MSE, exact-mode LNCC, other
    windows, approximate MI) is composed from the operator kernels exactly as the
    reference composes it (sample -> loss -> sampler backward)."""
    if params.kind == "lncc":
        return params.ants_approx and params.window == 7
    if params.kind == "mi":
        return not params.mi_approx_forward
    return False


@dataclass
class StepResult:
    loss: float
    g_u: torch.Tensor
    window_misses: int = 0


class StepWorkspace:
    """Device scratch reused across steps (no allocation inside a timed step)."""

    def __init__(self, device, bins: int = 32):
        self.device = device
        self.sum_n = torch.zeros(1, dtype=torch.float64, device=device)
        self.miss = torch.zeros(1, dtype=torch.int32, device=device)
        self.raw = torch.zeros(bins * bins + 2 * bins, dtype=torch.float64, device=device)
        self.table = torch.zeros(2 * bins * bins + 2 * bins + 4, dtype=torch.float64, device=device)
        self.scratch = torch.zeros(int(lib.ffdp_step_mi_workspace_bytes(bins)), dtype=torch.uint8, device=device)
        self.bins = bins
        self._rec = None
        self._lncc = None

    def lncc_workspace(self, dims: Dims, slab: Slab) -> torch.Tensor:
        """Workspace of the fused LNCC step (value ranges, one loss partial per CTA), kept
        across steps of the same lattice."""
        n = int(lib.ffdp_step_lncc_workspace_bytes(dims, slab)) // 4
        if self._lncc is None or self._lncc.numel() < n:
            self._lncc = torch.empty(n, dtype=torch.float32, device=self.device)
        return self._lncc

    def records(self, dims: Dims, slab: Slab) -> torch.Tensor:
        """Pass-1 records of the streaming MI pass 2 (16 B per interior voxel), kept across
        steps of the same lattice."""
        n = int(lib.ffdp_step_mi_record_bytes(dims, slab)) // 4
        if self._rec is None or self._rec.numel() < n:
            self._rec = torch.empty(n, dtype=torch.float32, device=self.device)
        return self._rec


def intensity_ranges(f: torch.Tensor, m: torch.Tensor) -> torch.Tensor:
    """Device float[4] {F min, F max, M min, M max} (ffdp_minmax, no host read): the value
    ranges that fix the LNCC step's intensity frame (ffdp_step_lncc `ranges`)."""
    out = torch.empty(4, dtype=torch.float32, device=f.device)
    f = f.contiguous()
    m = m.contiguous()
    lib.ffdp_minmax(_ptr(f), f.numel(), _ptr(out), _stream())
    lib.ffdp_minmax(_ptr(m), m.numel(), _ptr(out[2:]), _stream())
    return out


def intensity_shift(v: torch.Tensor) -> float:
    """Mid-range of a volume (the most accurate moment shift for the fused LNCC step)."""
    mm = torch.empty(2, dtype=torch.float32, device=v.device)
    lib.ffdp_minmax(_ptr(v), v.numel(), _ptr(mm), _stream())
    lo, hi = mm.tolist()
    return 0.5 * (lo + hi)


def warp_loss_step(f: torch.Tensor, m: torch.Tensor, u: torch.Tensor, A=None, t=None,
                   params: Optional[LossParams] = None, g_u: Optional[torch.Tensor] = None,
                   ws: Optional[StepWorkspace] = None, ranges: Optional[torch.Tensor] = None,
                   sync: bool = True) -> StepResult:
    """One deformable-step evaluation (registration.hpp:277-312 at H = 1):
    moved = fused_sample(M, u; A, t) -> LNCC (ANTs) or Mattes MI -> g_u =
    fused_sample_backward(dL/dmoved, want warp), with dL/dn_i = -1/N (dist_lncc,
    distops.hpp:320) or upstream -1 on MI (distops.hpp:392). F and M share a lattice
    (the driver extracts both with F's ShardSpec, registration.hpp:268-270)."""
    params = params or LossParams()
    f = _vol(f, "warp_loss_step")
    mi = m if isinstance(m, MovingImage) else MovingImage(m)
    u = _warp(u, "warp_loss_step")
    if tuple(u.shape[:3]) != tuple(f.shape):
        raise InvalidArgument("sampler: warp lattice mismatch")
    args = SamplerArgs(A=np.eye(3) if A is None else A, t=np.zeros(3) if t is None else t)
    args.validate()
    ca = args.to_c()
    if g_u is None:
        g_u = torch.empty(u.shape, dtype=torch.float32, device=u.device)
    ws = ws or StepWorkspace(u.device, params.bins)
    n = f.numel()
    nz = f.shape[0]
    slab = _full_slab(nz)
    if mi.shape != tuple(f.shape):
        raise InvalidArgument("warp_loss_step: F and M must share a lattice (registration.hpp:268-270)")
    win = mi.window()
    ws.miss.zero_()
    params.validate()
    if not fused_step_covers(params):
        return _composite_step(f, win, u, ca, params, g_u, ws, sync)
    if params.kind == "lncc":
        ws.sum_n.zero_()
        lws = ws.lncc_workspace(_dims(f.shape), slab)
        # ranges None: the library derives them from F and the moving window on every call
        lib.ffdp_step_lncc(_ptr(f), _ptr(u), _dims(f.shape), slab, win, C.byref(ca), params.window, params.epsilon,
                           -1.0 / n, None if ranges is None else _ptr(ranges), _ptr(g_u), _ptr(ws.sum_n),
                           _ptr(ws.miss), _ptr(lws), _stream())
        if not sync:
            return StepResult(float("nan"), g_u)
        loss = 1.0 - float(ws.sum_n.item()) / n
    elif params.kind == "mi":
        k = params.make_kernel()
        if ws.bins != params.bins:
            raise InvalidArgument("warp_loss_step: workspace built for a different bin count")
        rec = ws.records(_dims(f.shape), slab) if k.kind == PARZEN_BSPLINE3 else None
        lib.ffdp_step_mi(_ptr(f), _ptr(u), _dims(f.shape), slab, win, C.byref(ca), C.byref(k.c), _ptr(ws.raw),
                         _ptr(ws.table), _ptr(g_u), _ptr(ws.scratch), _ptr(rec), _ptr(ws.miss), _stream())
        if not sync:
            return StepResult(float("nan"), g_u)
        b = params.bins
        loss = -float(ws.table[2 * b * b + 2 * b + 1].item())
    else:
        raise InvalidArgument(f"warp_loss_step: unknown loss kind {params.kind!r}")
    return StepResult(loss, g_u, int(ws.miss.item()))


def _composite_step(f, win, u, ca, params: LossParams, g_u, ws: StepWorkspace, sync: bool) -> StepResult:
    """The deformable step for the losses the fused kernels do not cover, composed from the
    operator kernels exactly as the reference composes it (registration.hpp:277-312 at
    H = 1): moved = fused_sample(M, u) -> dist_mse (distops.hpp:260-282) / LNCC exact
    backward (lncc.hpp:226-280, upstream 1) / MI with the approximate forward
    (mi.hpp:275-354) and mi_backward_impl (upstream -1) -> fused_sample_backward(want
    warp)."""
    n = f.numel()
    dims = _dims(f.shape)
    moved = torch.empty(f.shape, dtype=torch.float32, device=f.device)
    lib.ffdp_sampler_fwd(win, _ptr(u), dims, C.byref(ca), _ptr(moved), 0, None, _ptr(ws.miss), _stream())
    if params.kind == "mse":
        ws.sum_n.zero_()
        gm = torch.empty_like(moved)
        lib.ffdp_mse(_ptr(f), _ptr(moved), n, n, _ptr(gm), _ptr(ws.sum_n), _stream())
        loss = (ws.sum_n / n) if not sync else float(ws.sum_n.item()) / n
    elif params.kind == "lncc":
        res, state = lncc_forward_fused(f, moved, params.window, params.epsilon)
        _, gm = lncc_backward_fused(1.0, state, f, moved, params.ants_approx)
        loss = res.loss
    else:
        k = params.make_kernel()
        res = (mi_forward_approx if params.mi_approx_forward else mi_forward_exact)(f, moved, params.bins, k)
        _, gm = mi_backward(-1.0, f, moved, res.hist, k, check_samples=False)
        loss = -res.mi
    lib.ffdp_sampler_bwd(_ptr(gm), win, _ptr(u), dims, C.byref(ca), WANT_WARP, None, _ptr(g_u), None, _ptr(ws.miss),
                         _stream())
    if not sync:
        return StepResult(float("nan"), g_u)
    return StepResult(float(loss), g_u, int(ws.miss.item()))
