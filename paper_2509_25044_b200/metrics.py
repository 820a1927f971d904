"""Label-overlap evaluation of a registration (metrics.hpp:17-203, sampler.hpp:331-365):
nearest-neighbour label warping through the composite transform, Dice, inverse-volume
weighted Dice and the cumulative 90th-percentile surface distance. Host numpy: these
score a result once per run (the CLI's `--fixed-labels / --moving-labels` summary block
and the `metrics` subcommand), they are not on the per-iteration path.

Label maps are uint16 arrays (nz, ny, nx), x fastest (volume.hpp:41-43); spacing is
(x, y, z).
"""
from __future__ import annotations

from typing import Dict, Sequence, Tuple

import numpy as np

from ._lib import InvalidArgument


def _host(v) -> np.ndarray:
    if hasattr(v, "detach"):
        v = v.detach().cpu().numpy()
    return np.asarray(v)


def _coords(n: int, lo: float, hi: float) -> np.ndarray:
    """lattice_coord (geometry.hpp:99-104) for i = 0..n-1."""
    if n <= 1:
        return np.full(max(n, 0), lo, dtype=np.float64)
    return lo + (hi - lo) * (np.arange(n, dtype=np.float64) / float(n - 1))


def _llround(f: np.ndarray) -> np.ndarray:
    """std::llround: halves away from zero."""
    return np.where(f >= 0, np.floor(f + 0.5), -np.floor(0.5 - f)).astype(np.int64)


def warp_labels_nn(labels, u, A=None, t=None, S=(1.0, 1.0, 1.0),
                   bounds: Tuple[Sequence[float], Sequence[float]] = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))) -> np.ndarray:
    """warp_labels_nn (sampler.hpp:331-365): out(x) = labels[round(f(A x + t + S u(x)))],
    0 where the rounded source index leaves the label lattice; u's lattice is the output."""
    lab = _host(labels)
    w = _host(u).astype(np.float64)
    if w.ndim != 4 or w.shape[3] != 3:
        raise InvalidArgument("warp_labels_nn: a (nz, ny, nx, 3) warp is required")
    A = np.eye(3) if A is None else np.asarray(A, dtype=np.float64).reshape(3, 3)
    t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64).reshape(3)
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(t))):
        raise InvalidArgument("SamplerArgs: non-finite affine")
    nz, ny, nx = w.shape[:3]
    X = _coords(nx, bounds[0][0], bounds[1][0])[None, None, :]
    Y = _coords(ny, bounds[0][1], bounds[1][1])[None, :, None]
    Z = _coords(nz, bounds[0][2], bounds[1][2])[:, None, None]
    n_src = (lab.shape[2], lab.shape[1], lab.shape[0])  # (x, y, z)
    idx, inside = [], np.ones((nz, ny, nx), dtype=bool)
    for a in range(3):
        # Mat3::apply row a, then + t, then + S u (sampler.hpp:343-346)
        xs = A[a, 0] * X + A[a, 1] * Y + A[a, 2] * Z
        xs = xs + t[a]
        xs = xs + S[a] * w[..., a]
        i = _llround((xs + 1.0) * 0.5 * float(n_src[a] - 1))
        inside &= (i >= 0) & (i < n_src[a])
        idx.append(np.clip(i, 0, n_src[a] - 1))
    out = lab[idx[2], idx[1], idx[0]]
    return np.where(inside, out, 0).astype(lab.dtype)


def _counts(a: np.ndarray, b: np.ndarray) -> Dict[int, Tuple[int, int, int]]:
    """overlap_counts (metrics.hpp:29-41): per non-zero label |A|, |B|, |A and B|."""
    a, b = _host(a).ravel(), _host(b).ravel()
    if a.shape != b.shape:
        raise InvalidArgument("metrics: lattices differ")
    a64, b64 = a.astype(np.int64), b.astype(np.int64)
    n = int(max(a64.max(initial=0), b64.max(initial=0))) + 1
    ca = np.bincount(a64, minlength=n)
    cb = np.bincount(b64, minlength=n)
    cboth = np.bincount(a64[(a64 == b64) & (a64 != 0)], minlength=n)
    return {lab: (int(ca[lab]), int(cb[lab]), int(cboth[lab])) for lab in range(1, n) if ca[lab] or cb[lab]}


def dice(a, b) -> Tuple[Dict[int, float], float]:
    """dice (metrics.hpp:44-60): per-label 2|A and B| / (|A| + |B|) and their mean over the
    labels present in either map."""
    per = {}
    s = 0.0
    for lab, (na, nb, both) in sorted(_counts(a, b).items()):
        d = 2.0 * both / (na + nb) if na + nb > 0 else 0.0
        per[lab] = d
        s += d
    return per, (s / len(per) if per else 0.0)


def inv_dice(a, b, weighting: str = "fixed_volume") -> float:
    """inv_dice (metrics.hpp:62-87): Dice weighted by 1 / label volume (in the first map,
    or in either map for "union_volume")."""
    num = den = 0.0
    for lab, (na, nb, both) in sorted(_counts(a, b).items()):
        vol = na if weighting == "fixed_volume" else na + nb - both
        if vol <= 0:
            continue
        w = 1.0 / vol
        d = 2.0 * both / (na + nb) if na + nb > 0 else 0.0
        num += w * d
        den += w
    if den == 0:
        raise InvalidArgument("inv_dice: no weighted labels")
    return num / den


def _surface(v: np.ndarray, label: int) -> np.ndarray:
    """label_surface (metrics.hpp:91-114): (x, y, z) of the label's voxels with a
    6-neighbour of another label (outside the volume counts as background), in the
    reference's z, y, x scan order."""
    m = v == label
    p = np.pad(m, 1, constant_values=False)
    interior = (p[1:-1, 1:-1, 2:] & p[1:-1, 1:-1, :-2] & p[1:-1, 2:, 1:-1] & p[1:-1, :-2, 1:-1]
                & p[2:, 1:-1, 1:-1] & p[:-2, 1:-1, 1:-1])
    z, y, x = np.nonzero(m & ~interior)
    return np.stack([x, y, z], axis=1).astype(np.int64)


def _hd90_directed(frm: np.ndarray, to: np.ndarray, spacing) -> float:
    """cumulative_hd90_directed (metrics.hpp:116-141): mean of the smallest
    max(1, floor(0.9 n)) nearest-surface distances, physical units. The nearest voxel
    comes from an exact k-d tree search; its distance is then evaluated as the reference
    sums it, ((dx sx)^2 + (dy sy)^2 + (dz sz)^2)."""
    from scipy.spatial import cKDTree
    if len(frm) == 0:
        return float("nan")
    sp = np.asarray(spacing, dtype=np.float64)
    _, j = cKDTree(to.astype(np.float64) * sp).query(frm.astype(np.float64) * sp)
    q = to[j]
    dx = (frm[:, 0] - q[:, 0]).astype(np.float64) * sp[0]
    dy = (frm[:, 1] - q[:, 1]).astype(np.float64) * sp[1]
    dz = (frm[:, 2] - q[:, 2]).astype(np.float64) * sp[2]
    d = np.sort(np.sqrt(dx * dx + dy * dy + dz * dz))
    k = max(1, int(0.9 * len(d)))
    return float(np.cumsum(d[:k])[-1] / k)  # sequential sum, as the reference adds


def hd90_cumulative(a, b, spacing=(1.0, 1.0, 1.0)) -> float:
    """hd90_cumulative (metrics.hpp:178-201): per label the max over both directions of
    the cumulative 90th-percentile surface distance, averaged over the labels."""
    a, b = _host(a), _host(b)
    if a.shape != b.shape:
        raise InvalidArgument("hd90: lattices differ")
    labels = sorted(set(np.unique(a[a != 0]).tolist()) | set(np.unique(b[b != 0]).tolist()))
    if not labels:
        raise InvalidArgument("hd90: both masks are empty")
    s = 0.0
    for lab in labels:
        sa, sb = _surface(a, lab), _surface(b, lab)
        if len(sa) == 0 or len(sb) == 0:
            raise InvalidArgument(f"hd90: label {lab} missing in one mask")
        s += max(_hd90_directed(sa, sb, spacing), _hd90_directed(sb, sa, spacing))
    return s / len(labels)
