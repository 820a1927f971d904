"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.

Two CPU implementations of the reference's fused warp + loss step, both fp64, with
numpy front-ends:

* ``Oracle`` -- ``libffdp_oracle.so``, a plain-C restatement (``ffdp_oracle.c``;
  every function cites the reference file:line it follows).
* ``Reference`` -- ``_ref/libvoxreg_ref.so``, the unmodified reference headers
  (``/root/reference/proj/include``) behind an ``extern "C"`` shim
  (``ref_shim.cpp``), compiled by ``oracle/Makefile``. Optional: present when the
  library was built in a container that had ``/root/reference``.

Arrays are x-fastest volumes of shape ``(nz, ny, nx)`` and interleaved warp fields of
shape ``(nz, ny, nx, 3)``, matching the reference layout (volume.hpp:3-7,57).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libffdp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvoxreg_ref.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)

KERNEL_KINDS = {"gaussian": 0, "bspline3": 1, "delta": 2}


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64)]


class Parzen(C.Structure):
    _fields_ = [("kind", C.c_int), ("bins", C.c_int), ("sigma", C.c_double), ("radius", C.c_double),
                ("norm", C.c_double)]


class Rng(C.Structure):
    _fields_ = [("state", C.c_uint64), ("have_spare", C.c_int), ("spare", C.c_double)]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _dims_of(shape):
    nz, ny, nx = shape[:3]
    return Dims(nx, ny, nz)


def _arr_dims(shape):
    nz, ny, nx = shape[:3]
    return (C.c_int64 * 3)(nx, ny, nz)


def _args(A, t, S, bounds):
    A = _f64(np.eye(3) if A is None else A).reshape(9)
    t = _f64(np.zeros(3) if t is None else t).reshape(3)
    S = _f64(np.ones(3) if S is None else S).reshape(3)
    b = _f64(np.array([-1, -1, -1, 1, 1, 1.0]) if bounds is None else bounds).reshape(6)
    return A, t, S, b


def box_taps(window):
    return np.full(window, 1.0 / window)


class Oracle:
    """numpy front-end of the C restatement (ffdp_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        L = self.lib = C.CDLL(path)
        L.or_sample_core.argtypes = [_dp, Dims, _dp, Dims, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.or_gaussian_taps.argtypes = [C.c_double, _dp, C.c_int]
        L.or_convolve_axis.argtypes = [_dp, _dp, Dims, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int64, C.c_int64]
        L.or_separable_convolve.argtypes = [_dp, Dims, C.c_int, _dp, C.c_int, C.c_int]
        L.or_lncc_forward.argtypes = [_dp, _dp, Dims, C.c_int, C.c_double, _dp, _dp]
        L.or_lncc_forward.restype = C.c_double
        L.or_lncc_backward.argtypes = [C.c_double, _dp, _dp, _dp, Dims, C.c_int, C.c_double, C.c_int, _dp, _dp]
        L.or_parzen_make.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(Parzen)]
        L.or_parzen_kappa.argtypes = [C.POINTER(Parzen), C.c_double]
        L.or_parzen_kappa.restype = C.c_double
        L.or_parzen_omega.argtypes = [C.POINTER(Parzen), C.c_double]
        L.or_parzen_omega.restype = C.c_double
        for fn in (L.or_mi_forward_exact, L.or_mi_forward_approx):
            fn.argtypes = [_dp, _dp, C.c_int64, C.POINTER(Parzen), _dp, _u64p]
        L.or_mi_finalize.argtypes = [_dp, C.c_int, _dp, _dp, _dp, _dp]
        L.or_mi_finalize.restype = C.c_double
        L.or_mi_ghat.argtypes = [C.c_double, _dp, _dp, _dp, C.c_double, C.c_int, _dp]
        L.or_mi_backward.argtypes = [_dp, _dp, C.c_int64, C.POINTER(Parzen), _dp, _dp, _dp]
        L.or_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, _i64p, _i64p]
        L.or_ring_sample.argtypes = [_dp, Dims, C.c_int, _dp, Dims, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.or_synth_pair.argtypes = [C.c_uint64, Dims, C.c_int, C.c_double, _dp, _dp, _dp]
        L.or_normalize_intensities.argtypes = [_dp, C.c_int64]
        L.or_step_lncc.argtypes = [_dp, _dp, Dims, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp, _dp]
        L.or_step_lncc.restype = C.c_double
        L.or_step_mi.argtypes = [_dp, _dp, Dims, _dp, _dp, _dp, C.POINTER(Parzen), C.c_int, _dp, _dp, _dp, _dp]
        L.or_step_mi.restype = C.c_double
        L.or_rng_init.argtypes = [C.POINTER(Rng), C.c_uint64]
        L.or_rng_uniform.argtypes = [C.POINTER(Rng)]
        L.or_rng_uniform.restype = C.c_double
        L.or_rng_normal.argtypes = [C.POINTER(Rng)]
        L.or_rng_normal.restype = C.c_double
        L.or_rng_uniform_int.argtypes = [C.POINTER(Rng), C.c_int64, C.c_int64]
        L.or_rng_uniform_int.restype = C.c_int64
        L.or_random_volume.argtypes = [C.POINTER(Rng), _dp, C.c_int64, C.c_double, C.c_double]
        L.or_resample_scale.argtypes = [_dp, Dims, C.c_double, _dp, C.POINTER(Dims)]
        L.or_resample_warp.argtypes = [_dp, Dims, _dp, Dims]
        L.or_deformable_stage.argtypes = [_dp, _dp, Dims, _dp, _dp, C.c_int, _dp, C.POINTER(C.c_int), C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                          C.c_int, _dp, _dp]
        L.or_affine_stage.argtypes = [_dp, _dp, Dims, C.c_int, _dp, C.POINTER(C.c_int), C.c_double, C.c_int, C.c_int,
                                      C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.or_jacobian_positive.argtypes = [_dp, Dims]
        L.or_jacobian_positive.restype = C.c_double
        L.or_adam_step.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_int64]
        L.or_warp_update.argtypes = [_dp, _dp, _dp, _dp, Dims, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_double, C.c_int64]

    # -- sampler (sampler.hpp:165-300) -------------------------------------------------
    def sample(self, img, u=None, A=None, t=None, S=None, bounds=None, out_shape=None, upstream=None,
               want=("warp",)):
        """Returns dict(out=..., image=..., warp=..., affine=..., translation=...)."""
        img = _f64(img)
        if u is not None:
            u = _f64(u)
            oshape = u.shape[:3]
        else:
            oshape = img.shape if out_shape is None else tuple(out_shape)
        A, t, S, b = _args(A, t, S, bounds)
        res = {}
        out = None
        if upstream is None:
            out = np.zeros(oshape)
            res["out"] = out
        g_img = g_u = gA = gt = None
        if upstream is not None:
            upstream = _f64(upstream)
            if "image" in want:
                g_img = res["image"] = np.zeros(img.shape)
            if "warp" in want:
                g_u = res["warp"] = np.zeros(tuple(oshape) + (3,))
            if "affine" in want:
                gA = res["affine"] = np.zeros((3, 3))
            if "translation" in want:
                gt = res["translation"] = np.zeros(3)
        rc = self.lib.or_sample_core(_p(img), _dims_of(img.shape), _p(u), _dims_of(oshape), _p(A), _p(t), _p(S),
                                     _p(b), _p(out), _p(upstream), _p(g_img), _p(g_u), _p(gA), _p(gt), None)
        if rc:
            raise ValueError("oracle sampler: invalid arguments")
        return res

    # -- smoothing (smoothing.hpp:25-105) ----------------------------------------------
    def gaussian_taps(self, sigma):
        buf = np.zeros(8192)
        n = self.lib.or_gaussian_taps(sigma, _p(buf), 8192)
        if n < 0:
            raise ValueError("gaussian_taps")
        return buf[:n].copy()

    def convolve_axis(self, data, axis, taps, mode, lo_global=0, n_global=None, channels=1):
        data = _f64(data)
        out = np.zeros_like(data)
        shape = data.shape[:3]
        if n_global is None:
            n_global = shape[2 - axis]
        taps = _f64(taps)
        self.lib.or_convolve_axis(_p(data), _p(out), _dims_of(shape), channels, axis, _p(taps), len(taps),
                                  1 if mode == "renormalize" else 0, lo_global, n_global)
        return out

    def separable_convolve(self, data, taps, mode="zero_pad", channels=1):
        d = _f64(data).copy()
        taps = _f64(taps)
        self.lib.or_separable_convolve(_p(d), _dims_of(d.shape), channels, _p(taps), len(taps),
                                       1 if mode == "renormalize" else 0)
        return d

    # -- multi-scale (resample.hpp:48-146) ----------------------------------------------
    def resample_scale(self, v, factor):
        v = _f64(v)
        nd = Dims()
        if self.lib.or_resample_scale(_p(v), _dims_of(v.shape), factor, None, C.byref(nd)):
            raise ValueError("resample_scale: bad factor")
        out = np.zeros((nd.nz, nd.ny, nd.nx))
        self.lib.or_resample_scale(_p(v), _dims_of(v.shape), factor, _p(out), C.byref(nd))
        return out

    def resample_warp(self, w, shape):
        w = _f64(w)
        out = np.zeros(tuple(shape) + (3,))
        self.lib.or_resample_warp(_p(w), _dims_of(w.shape[:3]), _p(out), _dims_of(shape))
        return out

    def deformable_stage(self, fixed, moving, steps, A=None, t=None, lr=0.5, sigma_grad=1.0, sigma_warp=0.5,
                         loss="lncc", window=7, eps=1e-5, ants=True, bins=32, mi_kind="gaussian"):
        """deformable_stage (registration.hpp:230-331) at H = 1: (warp, trace).
        steps = [(downsample, iterations), ...]."""
        f, m = _f64(fixed), _f64(moving)
        A, t, _, _ = _args(A, t, None, None)
        ds = np.array([s[0] for s in steps], dtype=np.float64)
        its = (C.c_int * len(steps))(*[int(s[1]) for s in steps])
        warp = np.zeros(f.shape + (3,))
        trace = np.zeros(max(1, sum(int(s[1]) for s in steps)))
        rc = self.lib.or_deformable_stage(_p(f), _p(m), _dims_of(f.shape), _p(A), _p(t), len(steps), _p(ds), its, lr,
                                          sigma_grad, sigma_warp, 0 if loss == "lncc" else 1, window, eps, int(ants),
                                          bins, KERNEL_KINDS[mi_kind], _p(warp), _p(trace))
        if rc == 1:
            raise ValueError("deformable_stage: invalid schedule")
        if rc == 2:
            raise ArithmeticError("deformable stage diverged (non-finite loss)")
        return warp, trace[:sum(int(s[1]) for s in steps)]

    def affine_stage(self, fixed, moving, steps, lr=0.5, loss="mi", window=7, eps=1e-5, ants=True, bins=32,
                     mi_kind="gaussian"):
        """affine_stage (registration.hpp:176-219): (A, t, trace)."""
        f, m = _f64(fixed), _f64(moving)
        ds = np.array([s[0] for s in steps], dtype=np.float64)
        its = (C.c_int * len(steps))(*[int(s[1]) for s in steps])
        A, t = np.zeros(9), np.zeros(3)
        trace = np.zeros(max(1, sum(int(s[1]) for s in steps)))
        rc = self.lib.or_affine_stage(_p(f), _p(m), _dims_of(f.shape), len(steps), _p(ds), its, lr,
                                      {"mse": 0, "lncc": 1, "mi": 2}[loss], window, eps, int(ants), bins,
                                      KERNEL_KINDS[mi_kind], _p(A), _p(t), _p(trace))
        if rc == 1:
            raise ValueError("affine_stage: invalid schedule")
        if rc == 2:
            raise ArithmeticError("affine stage diverged (non-finite loss)")
        return A.reshape(3, 3), t, trace[:sum(int(s[1]) for s in steps)]

    def jacobian_positive(self, u):
        u = _f64(u)
        return self.lib.or_jacobian_positive(_p(u), _dims_of(u.shape[:3]))

    # -- warp update (adam.hpp:30-50, registration.hpp:313-317) ------------------------
    def adam_step(self, param, grad, m1, m2, lr, step, beta1=0.9, beta2=0.999, eps=1e-8):
        """Returns (param, m1, m2) after adam_step; step = the state counter after it."""
        p, g, a, b = (_f64(x).copy() for x in (param, grad, m1, m2))
        self.lib.or_adam_step(_p(p), _p(g), _p(a), _p(b), p.size, lr, beta1, beta2, eps, step)
        return p, a, b

    def warp_update(self, g_u, u, m1, m2, lr, step, sigma_grad=1.0, sigma_warp=0.5, beta1=0.9, beta2=0.999,
                    eps=1e-8):
        """One deformable warp update on one rank: returns (u, m1, m2)."""
        g = _f64(g_u)
        uu, a, b = (_f64(x).copy() for x in (u, m1, m2))
        if self.lib.or_warp_update(_p(g), _p(uu), _p(a), _p(b), _dims_of(uu.shape[:3]), sigma_grad, sigma_warp, lr,
                                   beta1, beta2, eps, step):
            raise ValueError("warp_update: bad sigma")
        return uu, a, b

    # -- LNCC (lncc.hpp:144-280) ---------------------------------------------------------
    def lncc_forward(self, f, m, window=7, eps=1e-5, want_map=False):
        f, m = _f64(f), _f64(m)
        state = np.zeros((5,) + f.shape)
        mp = np.zeros(f.shape) if want_map else None
        loss = self.lib.or_lncc_forward(_p(f), _p(m), _dims_of(f.shape), window, eps, _p(state), _p(mp))
        return loss, state, mp

    def lncc_backward(self, upstream, state, f, m, window=7, eps=1e-5, ants=True):
        f, m = _f64(f), _f64(m)
        st = _f64(state).copy()
        gf, gm = np.zeros(f.shape), np.zeros(f.shape)
        self.lib.or_lncc_backward(upstream, _p(st), _p(f), _p(m), _dims_of(f.shape), window, eps, int(ants),
                                  _p(gf), _p(gm))
        return gf, gm, st

    # -- MI (mi.hpp:28-437) ----------------------------------------------------------------
    def parzen(self, kind, bins, sigma_bins=0.5):
        k = Parzen()
        rc = self.lib.or_parzen_make(KERNEL_KINDS[kind], bins, sigma_bins, C.byref(k))
        if rc:
            raise RuntimeError("ParzenKernel: discrete integral deviates from 1")
        return k

    def mi_forward(self, vi, vj, kernel, approx=False):
        vi, vj = _f64(vi).ravel(), _f64(vj).ravel()
        b = kernel.bins
        raw = np.zeros(b * b + 2 * b)
        stats = (C.c_uint64 * 2)(0, 0)
        fn = self.lib.or_mi_forward_approx if approx else self.lib.or_mi_forward_exact
        if fn(_p(vi), _p(vj), vi.size, C.byref(kernel), _p(raw), stats):
            raise ValueError("mi: intensities must lie in [0,1]")
        pij = np.zeros(b * b)
        pi, pj = np.zeros(b), np.zeros(b)
        z = C.c_double(0)
        mi = self.lib.or_mi_finalize(_p(raw), b, _p(pij), _p(pi), _p(pj), C.byref(z))
        return dict(mi=mi, raw=raw, p_ij=pij.reshape(b, b), p_i=pi, p_j=pj, z=z.value,
                    stats=(stats[0], stats[1]))

    def mi_backward(self, upstream, vi, vj, kernel, hist):
        shape = np.shape(vi)
        vi, vj = _f64(vi).ravel(), _f64(vj).ravel()
        b = kernel.bins
        ghat = np.zeros(b * b)
        pij = _f64(hist["p_ij"]).ravel()
        self.lib.or_mi_ghat(upstream, _p(pij), _p(_f64(hist["p_i"])), _p(_f64(hist["p_j"])), hist["z"], b, _p(ghat))
        gi, gj = np.zeros(vi.size), np.zeros(vi.size)
        self.lib.or_mi_backward(_p(vi), _p(vj), vi.size, C.byref(kernel), _p(ghat), _p(gi), _p(gj))
        return gi.reshape(shape), gj.reshape(shape), ghat.reshape(b, b)

    # -- fabric / ring (fabric.hpp:44-70, distops.hpp:144-248) -----------------------------
    def shard_range(self, n, world, rank):
        lo, hi = C.c_int64(), C.c_int64()
        if self.lib.or_shard_range(n, world, rank, C.byref(lo), C.byref(hi)):
            raise ValueError("shard_ranges: need 1 <= world <= axis size")
        return lo.value, hi.value

    def ring_sample(self, m_full, world, u_shard, out_bounds, A=None, t=None, upstream=None):
        m_full, u_shard = _f64(m_full), _f64(u_shard)
        A, t, _, b = _args(A, t, None, out_bounds)
        oshape = u_shard.shape[:3]
        out = np.zeros(oshape) if upstream is None else None
        g_u = np.zeros(u_shard.shape) if upstream is not None else None
        gAt = np.zeros(12) if upstream is not None else None
        up = None if upstream is None else _f64(upstream)
        rc = self.lib.or_ring_sample(_p(m_full), _dims_of(m_full.shape), world, _p(u_shard), _dims_of(oshape), _p(b),
                                     _p(A), _p(t), _p(out), _p(up), _p(g_u), _p(gAt))
        if rc:
            raise ValueError("ring_sample: invalid arguments")
        return out if upstream is None else (g_u, gAt)

    # -- fixtures (synth.hpp, registration.hpp:100-115) -------------------------------------
    def synth_pair(self, seed, shape, k=5, max_disp=0.12):
        nz, ny, nx = shape
        f, m = np.zeros(shape), np.zeros(shape)
        w = np.zeros(tuple(shape) + (3,))
        if self.lib.or_synth_pair(seed, Dims(nx, ny, nz), k, max_disp, _p(f), _p(m), _p(w)):
            raise ValueError("synth_pair: invalid arguments")
        return f, m, w

    def normalize(self, v):
        v = _f64(v).copy()
        self.lib.or_normalize_intensities(_p(v), v.size)
        return v

    def rng(self, seed):
        r = Rng()
        self.lib.or_rng_init(C.byref(r), seed)
        return r

    def random_volume(self, rng, shape, lo=0.0, hi=1.0):
        v = np.zeros(shape)
        self.lib.or_random_volume(C.byref(rng), _p(v), v.size, lo, hi)
        return v

    # -- the step (registration.hpp:277-312 at H=1) ------------------------------------------
    def step_lncc(self, f, m, u, A=None, t=None, window=7, eps=1e-5, ants=True):
        f, m, u = _f64(f), _f64(m), _f64(u)
        A, t, _, _ = _args(A, t, None, None)
        g_u = np.zeros(u.shape)
        moved, gm = np.zeros(f.shape), np.zeros(f.shape)
        loss = self.lib.or_step_lncc(_p(f), _p(m), _dims_of(f.shape), _p(u), _p(A), _p(t), window, eps, int(ants),
                                     _p(g_u), _p(moved), _p(gm))
        return dict(loss=loss, g_u=g_u, moved=moved, grad_moved=gm)

    def step_mi(self, f, m, u, kernel, A=None, t=None, approx=False):
        f, m, u = _f64(f), _f64(m), _f64(u)
        A, t, _, _ = _args(A, t, None, None)
        b = kernel.bins
        g_u = np.zeros(u.shape)
        moved, gm = np.zeros(f.shape), np.zeros(f.shape)
        raw = np.zeros(b * b + 2 * b)
        loss = self.lib.or_step_mi(_p(f), _p(m), _dims_of(f.shape), _p(u), _p(A), _p(t), C.byref(kernel), int(approx),
                                   _p(g_u), _p(moved), _p(gm), _p(raw))
        if not np.isfinite(loss):
            raise ValueError("mi: intensities must lie in [0,1]")
        return dict(loss=loss, g_u=g_u, moved=moved, grad_moved=gm, raw=raw)

    # -- full-size checks (ffdp_oracle_big.c): fp32 inputs, fp64 arithmetic, OpenMP ----------
    @staticmethod
    def _f32(a):
        return np.ascontiguousarray(a, dtype=np.float32)

    def _big(self, name, argtypes, restype=None):
        fn = getattr(self.lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
        return fn

    def lncc_sum_n_f32(self, f, m, u, A=None, t=None, window=7, eps=1e-5):
        """sum_i n_i of the warped pair over the whole lattice (loss = 1 - sum / N)."""
        f, m, u = self._f32(f), self._f32(m), self._f32(u)
        A, t, _, _ = _args(A, t, None, None)
        fp = C.POINTER(C.c_float)
        fn = self._big("or_lncc_sum_n_f32", [fp, fp, fp, Dims, _dp, _dp, C.c_int, C.c_double], C.c_double)
        return fn(f.ctypes.data_as(fp), m.ctypes.data_as(fp), u.ctypes.data_as(fp), _dims_of(f.shape), _p(A), _p(t),
                  window, eps)

    def lncc_ants_voxels_f32(self, f, m, u, vox, A=None, t=None, window=7, eps=1e-5, gi=None):
        """n_i, ANTs dL/dMw and g_u at the flat voxel indices `vox` (gi defaults to -1/N)."""
        f, m, u = self._f32(f), self._f32(m), self._f32(u)
        A, t, _, _ = _args(A, t, None, None)
        vox = np.ascontiguousarray(vox, dtype=np.int64)
        gi = -1.0 / f.size if gi is None else gi
        n, gm, gu = np.zeros(vox.size), np.zeros(vox.size), np.zeros((vox.size, 3))
        fp = C.POINTER(C.c_float)
        fn = self._big("or_lncc_ants_voxels_f32", [fp, fp, fp, Dims, _dp, _dp, C.c_int, C.c_double, C.c_double,
                                                   _i64p, C.c_int64, _dp, _dp, _dp])
        fn(f.ctypes.data_as(fp), m.ctypes.data_as(fp), u.ctypes.data_as(fp), _dims_of(f.shape), _p(A), _p(t), window,
           eps, gi, vox.ctypes.data_as(_i64p), vox.size, _p(n), _p(gm), _p(gu))
        return dict(n=n, grad_moved=gm, g_u=gu)

    def mi_hist_f32(self, f, m, u, kernel, A=None, t=None):
        """Raw payload (joint B*B, marginals) of mi_forward_exact for (F, warped M)."""
        f, m, u = self._f32(f), self._f32(m), self._f32(u)
        A, t, _, _ = _args(A, t, None, None)
        b = kernel.bins
        raw = np.zeros(b * b + 2 * b)
        fp = C.POINTER(C.c_float)
        fn = self._big("or_mi_hist_f32", [fp, fp, fp, Dims, _dp, _dp, C.POINTER(Parzen), _dp])
        fn(f.ctypes.data_as(fp), m.ctypes.data_as(fp), u.ctypes.data_as(fp), _dims_of(f.shape), _p(A), _p(t),
           C.byref(kernel), _p(raw))
        return raw

    def mi_table(self, raw, bins, upstream=-1.0):
        """finalize_histogram + histogram_mi + ghat (mi.hpp:181-209, 369-390): (MI, ghat)."""
        b = bins
        raw = _f64(raw)
        pij, pi, pj, gh = np.zeros(b * b), np.zeros(b), np.zeros(b), np.zeros(b * b)
        z = C.c_double()
        mi = self.lib.or_mi_finalize(_p(raw), b, _p(pij), _p(pi), _p(pj), C.byref(z))
        self.lib.or_mi_ghat(upstream, _p(pij), _p(pi), _p(pj), z.value, b, _p(gh))
        return mi, gh

    def mi_voxels_f32(self, f, m, u, kernel, ghat, vox, A=None, t=None):
        """dL/dMw and g_u at the flat voxel indices `vox` given the ghat table."""
        f, m, u = self._f32(f), self._f32(m), self._f32(u)
        A, t, _, _ = _args(A, t, None, None)
        vox = np.ascontiguousarray(vox, dtype=np.int64)
        gm, gu = np.zeros(vox.size), np.zeros((vox.size, 3))
        fp = C.POINTER(C.c_float)
        fn = self._big("or_mi_voxels_f32", [fp, fp, fp, Dims, _dp, _dp, C.POINTER(Parzen), _dp, _i64p, C.c_int64,
                                            _dp, _dp])
        fn(f.ctypes.data_as(fp), m.ctypes.data_as(fp), u.ctypes.data_as(fp), _dims_of(f.shape), _p(A), _p(t),
           C.byref(kernel), _p(_f64(ghat)), vox.ctypes.data_as(_i64p), vox.size, _p(gm), _p(gu))
        return dict(grad_moved=gm, g_u=gu)


class ReferenceError_(RuntimeError):
    pass


class Reference:
    """numpy front-end of the reference headers behind ref_shim.cpp (optional)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference shim missing: {path} (run `make -C oracle ref` where "
                                    f"/root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_sample.argtypes = [_dp, _i64p, _dp, _i64p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_lncc.argtypes = [_dp, _dp, _i64p, C.c_int, C.c_double, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _dp]
        L.ref_mi.argtypes = [_dp, _dp, _i64p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, _dp, _dp, _dp, _u64p,
                             _dp, _dp]
        L.ref_parzen_eval.argtypes = [C.c_int, C.c_int, C.c_double, _dp, C.c_int64, _dp, _dp]
        L.ref_synth_pair.argtypes = [C.c_uint64, _i64p, C.c_int, C.c_double, _dp, _dp, _dp]
        L.ref_gp_convolve.argtypes = [_dp, _i64p, C.c_int, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_resample_scale.argtypes = [_dp, _i64p, C.c_double, _dp, _i64p]
        L.ref_resample_warp.argtypes = [_dp, _i64p, _i64p, _dp]
        L.ref_normalize.argtypes = [_dp, _i64p, _dp]
        L.ref_deformable_stage.argtypes = [_dp, _dp, _i64p, _dp, _dp, C.c_int, _dp, C.POINTER(C.c_int), C.c_double,
                                           C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                           C.c_int, C.c_int, _dp, _dp]
        L.ref_affine_stage.argtypes = [_dp, _dp, _i64p, C.c_int, _dp, C.POINTER(C.c_int), C.c_double, C.c_int,
                                       C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_jacobian_positive.argtypes = [_dp, _i64p, _dp]
        _u16p = C.POINTER(C.c_uint16)
        L.ref_label_metrics.argtypes = [_u16p, _u16p, _i64p, _dp, _dp]
        L.ref_synth_labels.argtypes = [C.c_uint64, _i64p, C.c_int, C.c_double, _u16p, _u16p, _dp]
        L.ref_warp_labels_nn.argtypes = [_u16p, _i64p, _dp, _i64p, _dp, _dp, _u16p]
        L.ref_warp_update.argtypes = [_dp, _dp, _dp, _dp, _i64p, C.c_double, C.c_double, C.c_double, C.c_int64,
                                      C.c_int]
        L.ref_step.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _i64p, _dp, _dp, C.c_int, C.c_double, C.c_int,
                               C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]

    _codes = {1: ValueError, 2: RuntimeError, 3: AssertionError}

    def _check(self, rc):
        if rc:
            raise self._codes.get(rc, RuntimeError)(self.lib.ref_last_error().decode())

    def sample(self, img, u=None, A=None, t=None, S=None, bounds=None, upstream=None, want=("warp",)):
        img = _f64(img)
        oshape = u.shape[:3] if u is not None else img.shape
        if u is not None:
            u = _f64(u)
        A, t, S, b = _args(A, t, S, bounds)
        res = {}
        out = None
        if upstream is None:
            out = res["out"] = np.zeros(oshape)
        g_img = g_u = gA = gt = None
        if upstream is not None:
            upstream = _f64(upstream)
            if "image" in want:
                g_img = res["image"] = np.zeros(img.shape)
            if "warp" in want:
                g_u = res["warp"] = np.zeros(tuple(oshape) + (3,))
            if "affine" in want:
                gA = res["affine"] = np.zeros((3, 3))
            if "translation" in want:
                gt = res["translation"] = np.zeros(3)
        self._check(self.lib.ref_sample(_p(img), _arr_dims(img.shape), _p(u), _arr_dims(oshape), _p(A), _p(t), _p(S),
                                        _p(b), _p(out), _p(upstream), _p(g_img), _p(g_u), _p(gA), _p(gt)))
        return res

    def lncc(self, f, m, window=7, eps=1e-5, ants=True, upstream=1.0, want_map=False):
        f, m = _f64(f), _f64(m)
        loss = C.c_double()
        state = np.zeros((5,) + f.shape)
        mp = np.zeros(f.shape) if want_map else None
        gf, gm = np.zeros(f.shape), np.zeros(f.shape)
        self._check(self.lib.ref_lncc(_p(f), _p(m), _arr_dims(f.shape), window, eps, int(ants), upstream,
                                      C.byref(loss), _p(state), _p(mp), _p(gf), _p(gm)))
        return dict(loss=loss.value, state=state, map=mp, grad_f=gf, grad_m=gm)

    def mi(self, vi, vj, bins=32, kind="bspline3", sigma_bins=0.5, approx=False, upstream=-1.0):
        vi, vj = _f64(vi), _f64(vj)
        mi = C.c_double()
        raw = np.zeros(bins * bins + 2 * bins)
        pij = np.zeros(bins * bins + 2 * bins)
        stats = (C.c_uint64 * 2)(0, 0)
        gi, gj = np.zeros(vi.shape), np.zeros(vi.shape)
        self._check(self.lib.ref_mi(_p(vi), _p(vj), _arr_dims(vi.shape), bins, KERNEL_KINDS[kind], sigma_bins,
                                    int(approx), upstream, C.byref(mi), _p(raw), _p(pij), stats, _p(gi), _p(gj)))
        return dict(mi=mi.value, raw=raw, pij=pij, stats=(stats[0], stats[1]), grad_i=gi, grad_j=gj)

    def parzen_eval(self, kind, bins, x, sigma_bins=0.5):
        x = _f64(x)
        k, w = np.zeros(x.size), np.zeros(x.size)
        self._check(self.lib.ref_parzen_eval(KERNEL_KINDS[kind], bins, sigma_bins, _p(x), x.size, _p(k), _p(w)))
        return k, w

    def synth_pair(self, seed, shape, k=5, max_disp=0.12):
        f, m = np.zeros(shape), np.zeros(shape)
        w = np.zeros(tuple(shape) + (3,))
        self._check(self.lib.ref_synth_pair(seed, _arr_dims(shape), k, max_disp, _p(f), _p(m), _p(w)))
        return f, m, w

    def gp_convolve(self, v, taps, world, renormalize=False, sync=True):
        v = _f64(v)
        channels = 3 if v.ndim == 4 else 1
        out = np.zeros_like(v)
        taps = _f64(taps)
        self._check(self.lib.ref_gp_convolve(_p(v), _arr_dims(v.shape), channels, _p(taps), len(taps),
                                             int(renormalize), int(sync), world, _p(out)))
        return out

    def resample_scale(self, v, factor):
        v = _f64(v)
        nd = np.zeros(3, dtype=np.int64)
        self._check(self.lib.ref_resample_scale(_p(v), _arr_dims(v.shape), factor, None,
                                                nd.ctypes.data_as(_i64p)))
        out = np.zeros((int(nd[2]), int(nd[1]), int(nd[0])))
        self._check(self.lib.ref_resample_scale(_p(v), _arr_dims(v.shape), factor, _p(out),
                                                nd.ctypes.data_as(_i64p)))
        return out

    def resample_warp(self, w, shape):
        w = _f64(w)
        out = np.zeros(tuple(shape) + (3,))
        self._check(self.lib.ref_resample_warp(_p(w), _arr_dims(w.shape[:3]), _arr_dims(shape), _p(out)))
        return out

    def normalize(self, v):
        v = _f64(v)
        out = np.zeros_like(v)
        self._check(self.lib.ref_normalize(_p(v), _arr_dims(v.shape), _p(out)))
        return out

    def deformable_stage(self, fixed, moving, steps, A=None, t=None, lr=0.5, sigma_grad=1.0, sigma_warp=0.5,
                         loss="lncc", window=7, eps=1e-5, ants=True, bins=32, mi_kind="gaussian", world=1):
        f, m = _f64(fixed), _f64(moving)
        A, t, _, _ = _args(A, t, None, None)
        ds = np.array([s[0] for s in steps], dtype=np.float64)
        its = (C.c_int * len(steps))(*[int(s[1]) for s in steps])
        warp = np.zeros(f.shape + (3,))
        trace = np.zeros(max(1, sum(int(s[1]) for s in steps)))
        self._check(self.lib.ref_deformable_stage(_p(f), _p(m), _arr_dims(f.shape), _p(A), _p(t), len(steps), _p(ds),
                                                  its, lr, sigma_grad, sigma_warp, 0 if loss == "lncc" else 1, window,
                                                  eps, int(ants), bins, KERNEL_KINDS[mi_kind], world, _p(warp),
                                                  _p(trace)))
        return warp, trace[:sum(int(s[1]) for s in steps)]

    def affine_stage(self, fixed, moving, steps, lr=0.5, loss="mi", window=7, eps=1e-5, ants=True, bins=32,
                     mi_kind="gaussian"):
        f, m = _f64(fixed), _f64(moving)
        ds = np.array([s[0] for s in steps], dtype=np.float64)
        its = (C.c_int * len(steps))(*[int(s[1]) for s in steps])
        A, t = np.zeros(9), np.zeros(3)
        trace = np.zeros(max(1, sum(int(s[1]) for s in steps)))
        self._check(self.lib.ref_affine_stage(_p(f), _p(m), _arr_dims(f.shape), len(steps), _p(ds), its, lr,
                                              {"mse": 0, "lncc": 1, "mi": 2}[loss], window, eps, int(ants), bins,
                                              KERNEL_KINDS[mi_kind], _p(A), _p(t), _p(trace)))
        return A.reshape(3, 3), t, trace[:sum(int(s[1]) for s in steps)]

    def jacobian_positive(self, u):
        u = _f64(u)
        out = C.c_double()
        self._check(self.lib.ref_jacobian_positive(_p(u), _arr_dims(u.shape[:3]), C.byref(out)))
        return out.value

    def synth_labels(self, seed, shape, k=5, max_disp=0.12):
        """(labels_fixed, labels_moving, pre_blur_fixed) of synth_pair."""
        lf, lm = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        pre = np.zeros(shape)
        u16 = C.POINTER(C.c_uint16)
        self._check(self.lib.ref_synth_labels(seed, _arr_dims(shape), k, max_disp, lf.ctypes.data_as(u16),
                                              lm.ctypes.data_as(u16), _p(pre)))
        return lf, lm, pre

    def label_metrics(self, a, b, spacing=(1.0, 1.0, 1.0)):
        """(dice mean, inv_dice, hd90_cumulative) of two uint16 label maps (nz, ny, nx)."""
        a, b = (np.ascontiguousarray(x, dtype=np.uint16) for x in (a, b))
        sp = np.asarray(spacing, dtype=np.float64)
        out = np.zeros(3)
        u16 = C.POINTER(C.c_uint16)
        self._check(self.lib.ref_label_metrics(a.ctypes.data_as(u16), b.ctypes.data_as(u16), _arr_dims(a.shape),
                                               _p(sp), _p(out)))
        return tuple(float(x) for x in out)

    def warp_labels_nn(self, labels, u, A=None, t=None):
        lab = np.ascontiguousarray(labels, dtype=np.uint16)
        u = _f64(u)
        A = _f64(np.eye(3) if A is None else A).reshape(9)
        t = _f64(np.zeros(3) if t is None else t).reshape(3)
        out = np.zeros(u.shape[:3], dtype=np.uint16)
        u16 = C.POINTER(C.c_uint16)
        self._check(self.lib.ref_warp_labels_nn(lab.ctypes.data_as(u16), _arr_dims(lab.shape), _p(u),
                                                _arr_dims(u.shape[:3]), _p(A), _p(t), out.ctypes.data_as(u16)))
        return out

    def warp_update(self, g_u, u, m1, m2, lr, step, sigma_grad=1.0, sigma_warp=0.5, world=1):
        """registration.hpp:313-317 over `world` ranks (gp_convolve halos): (u, m1, m2)."""
        g = _f64(g_u)
        uu, a, b = (_f64(x).copy() for x in (u, m1, m2))
        self._check(self.lib.ref_warp_update(_p(g), _p(uu), _p(a), _p(b), _arr_dims(uu.shape[:3]), sigma_grad,
                                             sigma_warp, lr, step, world))
        return uu, a, b

    def step(self, loss_kind, f, m, u, A=None, t=None, window=7, eps=1e-5, ants=True, bins=32, kind="bspline3",
             approx=False, world=1, fp32=False):
        f, m, u = _f64(f), _f64(m), _f64(u)
        A, t, _, _ = _args(A, t, None, None)
        loss = C.c_double()
        g_u = np.zeros(u.shape)
        moved = np.zeros(f.shape)
        self._check(self.lib.ref_step(0 if loss_kind == "lncc" else 1, int(fp32), _p(f), _p(m), _p(u),
                                      _arr_dims(f.shape), _p(A), _p(t), window, eps, int(ants), bins,
                                      KERNEL_KINDS[kind], int(approx), world, C.byref(loss), _p(g_u), _p(moved)))
        return dict(loss=loss.value, g_u=g_u, moved=moved)


@dataclass
class StepInputs:
    """The survey's synthetic step fixture."""
    f: np.ndarray
    m: np.ndarray
    u: np.ndarray
    A: np.ndarray
    t: np.ndarray


def step_inputs(orc: Oracle, shape, seed=4242, loss="lncc", jitter=0.01, affine=0.02):
    """F = normalize(synth.fixed); M = synth.moving (LNCC) or a non-monotone remap of it
    (MI); u = smooth random warp (<=0.12) + U(-jitter, jitter); A = I + U(-affine, affine),
    t = U(-affine, affine). All rounded to fp32 (the GPU's storage type)."""
    f, m, w = orc.synth_pair(seed, shape, 5, 0.12)
    f = orc.normalize(f)
    m = orc.normalize(m)
    r = orc.rng(seed + 1)
    if loss == "mi":
        # non-linear, non-monotone remap + noise: a correlated multimodal pair
        m = orc.normalize(4.0 * m * (1.0 - m) + 0.02 * orc.random_volume(r, shape, -1.0, 1.0))
    jit = orc.random_volume(r, tuple(shape) + (3,), -jitter, jitter)
    u = w + jit
    aff = orc.random_volume(r, (12,), -affine, affine)
    A = np.eye(3) + aff[:9].reshape(3, 3)
    t = aff[9:]
    r32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return StepInputs(r32(f), r32(m), r32(u), A, t)
