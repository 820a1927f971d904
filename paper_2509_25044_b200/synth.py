"""Synthetic labelled pairs with a known warp (synth.hpp:18-135, rng.hpp:10-52): the
fixture generator behind `voxreg synth`. Host fp64 numpy, reproducing the reference's
arithmetic step for step (splitmix64 stream, Box-Muller through the C library's log /
sin / cos, sequential tap and moment sums), so a seed gives the reference's volumes bit
for bit. Not on the registration path: it runs once to make test data.

Arrays are (nz, ny, nx) (x fastest, volume.hpp:41-43); warps (nz, ny, nx, 3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._lib import InvalidArgument
from .metrics import warp_labels_nn

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


class Rng:
    """Rng (rng.hpp:10-52): splitmix64, uniform in [0, 1) from the top 53 bits, Box-Muller
    normals with a spare."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK
        self.have_spare = False
        self.spare = 0.0

    def uniforms(self, n: int) -> np.ndarray:
        """The next n uniform() draws, vectorised (state_k = state + k * gamma)."""
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * int(_GAMMA)) & _MASK
        return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = float(self.uniforms(1)[0])
        return u if lo is None else lo + (hi - lo) * u

    def normals(self, n: int) -> np.ndarray:
        """The next n normal() draws (Box-Muller, rng.hpp:33-46)."""
        out = np.empty(n)
        i = 0
        if n and self.have_spare:
            out[0] = self.spare
            self.have_spare = False
            i = 1
        while i < n:
            u1 = self.uniform()
            while u1 <= 0:
                u1 = self.uniform()
            u2 = self.uniform()
            r = math.sqrt(-2.0 * math.log(u1))
            theta = 6.283185307179586476925286766559 * u2
            out[i] = r * math.cos(theta)
            i += 1
            if i < n:
                out[i] = r * math.sin(theta)
                i += 1
            else:
                self.spare, self.have_spare = r * math.sin(theta), True
        return out


def gaussian_taps(sigma: float) -> np.ndarray:
    """gaussian_taps (smoothing.hpp:25-39), with the C library's exp."""
    if not math.isfinite(sigma) or sigma < 0:
        raise InvalidArgument("gaussian_taps: sigma must be finite and >= 0")
    if sigma == 0:
        return np.ones(1)
    r = int(math.ceil(3.0 * sigma))
    w = [math.exp(-0.5 * (k / sigma) * (k / sigma)) for k in range(-r, r + 1)]
    s = 0.0
    for x in w:
        s += x
    return np.array([x / s for x in w])


def _convolve_axis(v: np.ndarray, axis: int, taps: np.ndarray) -> np.ndarray:
    """convolve_axis (smoothing.hpp:52-94), renormalize mode, whole volume (lo_global 0):
    taps added in order k = -r..r; full windows divide by the full tap sum, clipped ones
    by the sum of their in-range taps."""
    r = len(taps) // 2
    n = v.shape[axis]
    full_sum = 0.0
    for w in taps:
        full_sum += float(w)
    acc = np.zeros_like(v)
    wsum = np.zeros(n)
    shape = [1] * v.ndim
    shape[axis] = n
    pos = np.arange(n)
    for k in range(-r, r + 1):
        ok = (pos + k >= 0) & (pos + k < n)
        src = np.take(v, np.clip(pos + k, 0, n - 1), axis=axis)
        term = float(taps[k + r]) * src
        acc = acc + np.where(ok.reshape(shape), term, 0.0)
        wsum = wsum + np.where(ok, float(taps[k + r]), 0.0)
    full = (pos - r >= 0) & (pos + r < n)
    div = np.where(full, full_sum, np.where(wsum > 0, wsum, 1.0))
    return acc / div.reshape(shape)


def gaussian_smooth(v: np.ndarray, sigma: float) -> np.ndarray:
    """gaussian_smooth (smoothing.hpp:107-127): x, then y, then z, renormalized edges;
    a warp (trailing axis 3) is smoothed per component."""
    if not math.isfinite(sigma) or sigma < 0:
        raise InvalidArgument("gaussian_smooth: sigma must be finite and >= 0")
    if sigma == 0:
        return v.copy()
    taps = gaussian_taps(sigma)
    out = v
    for axis in (2, 1, 0):  # x, y, z of an (nz, ny, nx[, 3]) array
        out = _convolve_axis(out, axis, taps)
    return out


def rasterize_ellipsoids(rng: Rng, shape, k: int) -> np.ndarray:
    """rasterize_ellipsoids (synth.hpp:33-53): later labels win."""
    nz, ny, nx = shape
    lab = np.zeros(shape, np.uint16)
    z, y, x = (np.arange(nz, dtype=np.float64)[:, None, None], np.arange(ny, dtype=np.float64)[None, :, None],
               np.arange(nx, dtype=np.float64)[None, None, :])
    dims = (nx, ny, nz)
    for label in range(1, k + 1):
        c, rad = [0.0] * 3, [0.0] * 3
        for a in range(3):
            n = float(dims[a])
            c[a] = rng.uniform(0.22, 0.78) * (n - 1)
            rad[a] = rng.uniform(0.10, 0.24) * n
        dx, dy, dz = (x - c[0]) / rad[0], (y - c[1]) / rad[1], (z - c[2]) / rad[2]
        lab[dx * dx + dy * dy + dz * dz <= 1.0] = label
    return lab


def random_smooth_warp(rng: Rng, shape, max_norm: float, sigma_voxels: float, rms_fraction: float = 0.7):
    """random_smooth_warp (synth.hpp:79-114)."""
    n = int(np.prod(shape))
    w = rng.normals(3 * n).reshape(tuple(shape) + (3,))
    w = gaussian_smooth(w, sigma_voxels)
    s = w[..., 0] * w[..., 0] + w[..., 1] * w[..., 1] + w[..., 2] * w[..., 2]
    rms = math.sqrt(float(np.cumsum(s.ravel())[-1]) / n)  # sequential, as the reference sums
    if rms > 0 and max_norm > 0:
        w = w * (rms_fraction * max_norm / rms)
        s = w[..., 0] * w[..., 0] + w[..., 1] * w[..., 1] + w[..., 2] * w[..., 2]
        norm = np.sqrt(s)
        clip = np.where(norm > max_norm, max_norm / np.where(norm > 0, norm, 1.0), 1.0)
        w = np.where((norm > max_norm)[..., None], w * clip[..., None], w)
    elif max_norm == 0:
        w = np.zeros_like(w)
    return w


def sample_identity(img: np.ndarray, u: np.ndarray) -> np.ndarray:
    """fused_sample(img, &u, SamplerArgs{}) (sampler.hpp:165-263) on u's lattice, fp64:
    x_src = X + u, floor cells with the face snap of cell_assign (resample.hpp:27-43),
    the 8 in-range corners added in (z, y, x) order with weight (wz wy) wx."""
    nz, ny, nx = u.shape[:3]
    n_img = (img.shape[2], img.shape[1], img.shape[0])
    coords = [(-1.0 + 2.0 * (np.arange(m, dtype=np.float64) / float(m - 1))) if m > 1 else np.full(1, -1.0)
              for m in (nx, ny, nz)]
    X = [coords[0][None, None, :], coords[1][None, :, None], coords[2][:, None, None]]
    i0, fr = [], []
    for a in range(3):
        xs = X[a] + u[..., a]
        f = (xs + 1.0) * 0.5 * float(n_img[a] - 1)
        fl = np.floor(f)
        fa = f - fl
        lo = fa < 1e-9
        hi = ~lo & (1.0 - fa < 1e-9)
        fl = np.where(hi, fl + 1.0, fl)
        fa = np.where(lo | hi, 0.0, fa)
        i0.append(fl.astype(np.int64))
        fr.append(fa)
    acc = np.zeros((nz, ny, nx))
    for bz in (0, 1):
        iz = i0[2] + bz
        wz = fr[2] if bz else 1 - fr[2]
        for by in (0, 1):
            iy = i0[1] + by
            wy = fr[1] if by else 1 - fr[1]
            for bx in (0, 1):
                ix = i0[0] + bx
                wx = fr[0] if bx else 1 - fr[0]
                ok = (ix >= 0) & (ix < n_img[0]) & (iy >= 0) & (iy < n_img[1]) & (iz >= 0) & (iz < n_img[2])
                v = img[np.clip(iz, 0, n_img[2] - 1), np.clip(iy, 0, n_img[1] - 1), np.clip(ix, 0, n_img[0] - 1)]
                acc = acc + np.where(ok, wz * wy * wx * v, 0.0)
    return 0.0 + acc


@dataclass
class SynthPair:
    """SynthPair (synth.hpp:24-31)."""
    fixed: np.ndarray
    moving: np.ndarray
    pre_blur_fixed: np.ndarray
    labels_fixed: np.ndarray
    labels_moving: np.ndarray
    true_warp: np.ndarray
    mu: np.ndarray
    sigma: np.ndarray


def synth_pair(seed: int, shape, k: int, max_disp: float = 0.12) -> SynthPair:
    """synth_pair (synth.hpp:116-135) for a (nz, ny, nx) lattice."""
    nz, ny, nx = (int(s) for s in shape)
    if nx < 16 or ny < 16 or nz < 16:
        raise InvalidArgument("synth_pair: dims must be >= 16 per axis")
    if k < 1 or k > 16:
        raise InvalidArgument("synth_pair: 1 <= K <= 16")
    if not (max_disp >= 0) or max_disp > 0.15:
        raise InvalidArgument("synth_pair: max displacement capped at 0.15")
    rng = Rng(seed)
    labels = rasterize_ellipsoids(rng, (nz, ny, nx), k)
    mu, sigma = np.zeros(k + 1), np.zeros(k + 1)
    for label in range(1, k + 1):  # draw_label_stats (synth.hpp:55-64)
        mu[label] = rng.uniform(0.3, 1.0)
        sigma[label] = rng.uniform(0.02, 0.06)
    flat = labels.ravel()
    idx = np.nonzero(flat)[0]  # paint_labels (synth.hpp:66-75): one normal per labelled voxel, in order
    nrm = rng.normals(idx.size)
    pre = np.zeros(flat.size)
    pre[idx] = mu[flat[idx]] + sigma[flat[idx]] * nrm
    pre = pre.reshape(labels.shape)
    fixed = gaussian_smooth(pre, 0.75)
    warp = random_smooth_warp(rng, (nz, ny, nx), max_disp, nx / 8.0)
    moving = sample_identity(fixed, warp)
    lm = warp_labels_nn(labels, warp)
    return SynthPair(fixed, moving, pre, labels, lm, warp, mu, sigma)
