"""Shard invariance of the fused step on one GPU: each emulated rank runs the slab
kernels on its z slab (+ halo planes of F and u, + a moving-image window), and the
gathered g_u / reduced loss equal the single-GPU step (the reference's own invariance
tests: test_distops.cpp:161-187, 243-289, 369-423). Window misses are reported."""
import ctypes as C

import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


def global_ranges(V, si):
    """The intensity frame of the whole pair (what the sharded drivers allreduce)."""
    return V.intensity_ranges(dev(si.f), dev(si.m))


def run_slab(V, si, spec_lo, spec_hi, nz, pad, loss, window, bins=32, ranges=None, with_ws=True):
    import torch
    from paper_2509_25044_b200._lib import Dims, ImageWindow, Slab, lib
    f, m, u = dev(si.f), dev(si.m), dev(si.u)
    ny, nx = si.f.shape[1], si.f.shape[2]
    b0, b1 = max(0, spec_lo - pad), min(nz, spec_hi + pad)
    fb, ub = f[b0:b1].contiguous(), u[b0:b1].contiguous()
    z0, z1 = window
    mp = torch.zeros((z1 - z0 + 4, ny + 4, nx + 4), device="cuda")
    mp[2:-2, 2:-2, 2:-2] = m[z0:z1]
    win = ImageWindow(mp.data_ptr(), Dims(nx, ny, nz), z0, z1, 2)
    slab = Slab(b0, b1 - b0, spec_lo, spec_hi, nz)
    args = V.SamplerArgs(A=si.A, t=si.t).to_c()
    g_u = torch.empty((spec_hi - spec_lo, ny, nx, 3), device="cuda")
    miss = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = V._stream()
    if loss == "lncc":
        sn = torch.zeros(1, dtype=torch.float64, device="cuda")
        ws = None
        if with_ws:
            ws = torch.empty(int(lib.ffdp_step_lncc_workspace_bytes(V._dims(fb.shape), slab)) // 4, device="cuda")
        lib.ffdp_step_lncc(V._ptr(fb), V._ptr(ub), V._dims(fb.shape), slab, win, C.byref(args), 7, 1e-5,
                           -1.0 / si.f.size, V._ptr(global_ranges(V, si) if ranges is None else ranges), V._ptr(g_u),
                           V._ptr(sn), V._ptr(miss), V._ptr(ws),
                           s)
        return float(sn.item()), g_u, int(miss.item())
    k = V.ParzenKernel.bspline3(bins)
    raw = torch.zeros(bins * bins + 2 * bins, dtype=torch.float64, device="cuda")
    lib.ffdp_step_mi_hist(V._ptr(fb), V._ptr(ub), V._dims(fb.shape), slab, win, C.byref(args), C.byref(k.c),
                          V._ptr(raw), None, V._ptr(miss), s)
    return raw, (fb, ub, slab, win, args, k, g_u, mp), int(miss.item())


@pytest.mark.parametrize("with_ws", [True, False])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_lncc_slabs_equal_single_gpu(V, orc, world, with_ws):
    from oracle import step_inputs
    from paper_2509_25044_b200 import dist as D
    si = step_inputs(orc, (40, 36, 44), seed=4242, loss="lncc")
    nz = si.f.shape[0]
    full = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, ranges=global_ranges(V, si))
    ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
    total, parts = 0.0, []
    for r, (lo, hi) in enumerate(D.shard_ranges(nz, world)):
        sn, g, miss = run_slab(V, si, lo, hi, nz, 3, "lncc", (0, nz), with_ws=with_ws)
        assert miss == 0
        total += sn
        parts.append(host(g))
    loss = 1.0 - total / si.f.size
    gu = np.concatenate(parts, axis=0)
    # exact integer window sums in one intensity frame: every voxel's g_u is bit-identical
    # whatever the slab / chunk split; the loss differs only in the order of the CTA sums
    assert loss == pytest.approx(full.loss, rel=1e-9)  # fp32 per-thread n_i partials, other order
    assert np.array_equal(gu, host(full.g_u))
    assert loss == pytest.approx(ref["loss"], rel=1e-5)
    assert maxrel(gu, ref["g_u"]) < 1e-4


@pytest.mark.parametrize("world", [2, 4])
def test_mi_slabs_equal_single_gpu(V, orc, world):
    import torch
    from oracle import step_inputs
    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200._lib import lib
    si = step_inputs(orc, (32, 36, 40), seed=4242, loss="mi")
    nz, b = si.f.shape[0], 32
    ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", b), si.A, si.t)
    raws, ctx = [], []
    for lo, hi in D.shard_ranges(nz, world):
        raw, c_, miss = run_slab(V, si, lo, hi, nz, 0, "mi", (0, nz))
        assert miss == 0
        raws.append(raw)
        ctx.append(c_)
    raw = sum(raws)  # the allreduce of the joint payload (distops.hpp:365-373)
    table = torch.empty(2 * b * b + 2 * b + 4, dtype=torch.float64, device="cuda")
    lib.ffdp_mi_finalize(V._ptr(raw), b, -1.0, V._ptr(table), V._stream())
    parts = []
    for fb, ub, slab, win, args, k, g_u, mp in ctx:
        lib.ffdp_step_mi_grad(V._ptr(fb), V._ptr(ub), V._dims(fb.shape), slab, win, C.byref(args), C.byref(k.c),
                              V._ptr(table), V._ptr(g_u), None, V._stream())
        parts.append(host(g_u))
    loss = -float(table[2 * b * b + 2 * b + 1].item())
    assert loss == pytest.approx(ref["loss"], rel=1e-5)
    assert maxrel(np.concatenate(parts, axis=0), ref["g_u"]) < 1e-4


def test_window_miss_is_reported_and_exact_when_wide(V, orc):
    from oracle import step_inputs
    si = step_inputs(orc, (30, 24, 28), seed=11, loss="lncc")
    nz = si.f.shape[0]
    lo, hi = 10, 20
    _, g_narrow, miss = run_slab(V, si, lo, hi, nz, 3, "lncc", (lo, hi))
    assert miss > 0  # samples reach planes outside [10, 20)
    _, g_wide, miss = run_slab(V, si, lo, hi, nz, 3, "lncc", (0, nz))
    assert miss == 0
    full = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, ranges=global_ranges(V, si))
    assert maxrel(host(g_wide), host(full.g_u)[lo:hi]) < 2e-5


@pytest.mark.parametrize("world", [2, 4])
def test_mi_slabs_straddle_fixed_point_switch(V, orc, world):
    """The whole 48x64x64 volume (196608 voxels >= 2^17) runs pass 1 on the 2^-21
    fixed-point grid; its 2-rank slabs (98304 voxels) on the 2^-23 grid and its 4-rank slabs
    (49152 < 2^16) on the scalar kernels (step_mi.cu). The sharded step changes arithmetic
    with H, so it is gated against the single-GPU step and the oracle at the north-star
    tolerances instead of bit equality."""
    import torch
    from oracle import step_inputs
    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200._lib import lib
    si = step_inputs(orc, (48, 64, 64), seed=4242, loss="mi")
    nz, b = si.f.shape[0], 32
    ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", b), si.A, si.t)
    full = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t,
                            V.LossParams(kind="mi", bins=b, mi_bspline_kernel=True))
    raws, ctx = [], []
    for lo, hi in D.shard_ranges(nz, world):
        raw, c_, miss = run_slab(V, si, lo, hi, nz, 0, "mi", (0, nz))
        assert miss == 0
        raws.append(raw)
        ctx.append(c_)
    raw = sum(raws)
    table = torch.empty(2 * b * b + 2 * b + 4, dtype=torch.float64, device="cuda")
    lib.ffdp_mi_finalize(V._ptr(raw), b, -1.0, V._ptr(table), V._stream())
    parts = []
    for fb, ub, slab, win, args, k, g_u, mp in ctx:
        lib.ffdp_step_mi_grad(V._ptr(fb), V._ptr(ub), V._dims(fb.shape), slab, win, C.byref(args), C.byref(k.c),
                              V._ptr(table), V._ptr(g_u), None, V._stream())
        parts.append(host(g_u))
    loss = -float(table[2 * b * b + 2 * b + 1].item())
    gu = np.concatenate(parts, axis=0)
    print(f"mi straddle H={world}: loss vs 1 GPU {abs(loss / full.loss - 1):.2e}, vs oracle "
          f"{abs(loss / ref['loss'] - 1):.2e}; g_u vs 1 GPU {maxrel(gu, host(full.g_u)):.2e}, vs oracle "
          f"{maxrel(gu, ref['g_u']):.2e}")
    assert loss == pytest.approx(full.loss, rel=1e-5)
    assert loss == pytest.approx(ref["loss"], rel=1e-5)
    assert maxrel(gu, host(full.g_u)) < 1e-4
    assert maxrel(gu, ref["g_u"]) < 1e-4
