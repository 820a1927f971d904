"""The fused warp + loss step (the hot path) vs the oracle's step at H = 1.

Gates: |dloss|/|loss| <= 1e-5 and
max|dg_u|/max|g_u| <= 1e-4 on the survey's synthetic fixture, fp32 inputs."""
import numpy as np
import pytest

from gpu_util import dev, host, l2rel, maxrel, need_gpu

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-5
GRAD_MAXREL = 1e-4


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


@pytest.fixture(scope="module")
def lncc_case(orc):
    from oracle import step_inputs
    si = step_inputs(orc, (64, 72, 80), seed=4242, loss="lncc")
    ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
    return si, ref


@pytest.fixture(scope="module")
def mi_case(orc):
    from oracle import step_inputs
    si = step_inputs(orc, (48, 56, 64), seed=4242, loss="mi")
    ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    return si, ref


def test_step_lncc_parity(V, lncc_case):
    si, ref = lncc_case
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, V.LossParams(kind="lncc"))
    assert res.window_misses == 0
    assert res.loss == pytest.approx(ref["loss"], rel=LOSS_RTOL)
    gu = host(res.g_u)
    print("lncc step: loss rel", abs(res.loss - ref["loss"]) / abs(ref["loss"]), "g_u maxrel",
          maxrel(gu, ref["g_u"]), "l2rel", l2rel(gu, ref["g_u"]))
    assert maxrel(gu, ref["g_u"]) <= GRAD_MAXREL


def test_step_mi_records_equal_recompute(V, mi_case):
    """Pass 2 from the pass-1 records (ffdp_step_mi_grad_rec) and pass 2 re-sampling the
    warp (ffdp_step_mi_grad) compute the same arithmetic: bit-identical g_u and loss."""
    import ctypes as C

    import torch
    from paper_2509_25044_b200._lib import lib
    si, _ = mi_case
    f, u = dev(si.f), dev(si.u)
    mimg = V.MovingImage(dev(si.m))
    k = V.ParzenKernel.bspline3(32)
    ca = V.SamplerArgs(A=si.A, t=si.t).to_c()
    dims, slab = V._dims(f.shape), V._full_slab(f.shape[0])
    out = []
    for use_rec in (True, False):
        ws = V.StepWorkspace(f.device, 32)
        g = torch.empty_like(u)
        rec = ws.records(dims, slab) if use_rec else None
        lib.ffdp_step_mi(V._ptr(f), V._ptr(u), dims, slab, mimg.window(), C.byref(ca), C.byref(k.c), V._ptr(ws.raw),
                         V._ptr(ws.table), V._ptr(g), V._ptr(ws.scratch), V._ptr(rec), V._ptr(ws.miss), V._stream())
        out.append((host(g), float(ws.table[2 * 32 * 32 + 2 * 32 + 1].item())))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_step_mi_parity(V, mi_case):
    si, ref = mi_case
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True))
    assert res.window_misses == 0
    assert res.loss == pytest.approx(ref["loss"], rel=LOSS_RTOL)
    gu = host(res.g_u)
    print("mi step: loss rel", abs(res.loss - ref["loss"]) / abs(ref["loss"]), "g_u maxrel",
          maxrel(gu, ref["g_u"]), "l2rel", l2rel(gu, ref["g_u"]))
    assert maxrel(gu, ref["g_u"]) <= GRAD_MAXREL


def test_step_lncc_matches_operator_chain(V, lncc_case):
    """The fused single pass equals the operator-by-operator chain on the GPU."""
    si, _ = lncc_case
    f, m, u = dev(si.f), dev(si.m), dev(si.u)
    args = V.SamplerArgs(A=si.A, t=si.t)
    mw = V.fused_sample(m, u, args)
    res, st = V.lncc_forward_fused(f, mw, 7, 1e-5)
    _, gm = V.lncc_backward_fused(1.0, st, f, mw, True)
    gu = V.fused_sample_backward(gm, m, u, args, V.SamplerGradWant(warp=True)).warp
    step = V.warp_loss_step(f, m, u, si.A, si.t)
    assert step.loss == pytest.approx(res.loss, rel=1e-6)
    assert maxrel(host(step.g_u), host(gu)) < 1e-4


def test_step_deterministic_mi(V, mi_case):
    si, _ = mi_case
    f, m, u = dev(si.f), dev(si.m), dev(si.u)
    p = V.LossParams(kind="mi", mi_bspline_kernel=True)
    a = V.warp_loss_step(f, m, u, si.A, si.t, p)
    b = V.warp_loss_step(f, m, u, si.A, si.t, p)
    assert a.loss == b.loss  # integer fixed-point histogram: order independent
    assert np.array_equal(host(a.g_u), host(b.g_u))


@pytest.mark.parametrize("shape,seed", [((24, 28, 32), 7), ((20, 20, 20), 11)])
def test_step_mi_sparse_histogram(V, orc, shape, seed):
    """Small volumes leave many joint bins holding only B-spline tail products; ghat =
    log(p / p_i p_j) needs them to relative accuracy (fixed point with residual counter)."""
    from oracle import step_inputs
    si = step_inputs(orc, shape, seed=seed, loss="mi")
    ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True))
    assert res.loss == pytest.approx(ref["loss"], rel=LOSS_RTOL)
    assert maxrel(host(res.g_u), ref["g_u"]) <= GRAD_MAXREL


@pytest.mark.parametrize("mode", ["mse", "lncc_exact", "mi_approx", "mi_gaussian"])
def test_step_operator_composed_losses(V, orc, mode):
    """The step for the losses outside the fused kernels (registration.hpp:277-312 with
    dist_mse distops.hpp:260-282, LNCC exact backward lncc.hpp:226-280, MI approximate
    forward mi.hpp:275-354) and the Gaussian-Parzen fused MI step, against the oracle."""
    from gpu_util import dev, host, maxrel
    from oracle import step_inputs
    loss_kind = "lncc" if mode.startswith("lncc") or mode == "mse" else "mi"
    si = step_inputs(orc, (17, 19, 23), seed=4242, loss=loss_kind)
    if mode == "mse":
        moved = orc.sample(si.m, si.u, si.A, si.t)["out"]
        n = moved.size
        ref_loss = float(np.sum((moved - si.f) ** 2) / n)
        ref_gu = orc.sample(si.m, si.u, si.A, si.t, upstream=2.0 * (moved - si.f) / n)["warp"]
        p = V.LossParams(kind="mse")
    elif mode == "lncc_exact":
        r = orc.step_lncc(si.f, si.m, si.u, si.A, si.t, ants=False)
        ref_loss, ref_gu = r["loss"], r["g_u"]
        p = V.LossParams(kind="lncc", ants_approx=False)
    elif mode == "mi_approx":
        r = orc.step_mi(si.f, si.m, si.u, orc.parzen("gaussian", 32), si.A, si.t, approx=True)
        ref_loss, ref_gu = r["loss"], r["g_u"]
        p = V.LossParams(kind="mi", bins=32, mi_approx_forward=True)
    else:
        r = orc.step_mi(si.f, si.m, si.u, orc.parzen("gaussian", 32), si.A, si.t)
        ref_loss, ref_gu = r["loss"], r["g_u"]
        p = V.LossParams(kind="mi", bins=32)
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, p)
    assert res.loss == pytest.approx(ref_loss, rel=1e-5)
    assert maxrel(host(res.g_u), ref_gu) <= 1e-4


@pytest.mark.parametrize("shape", [(3, 5, 33), (8, 9, 65), (1, 6, 7), (2, 40, 31)])
@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_step_ragged_and_thin_lattices(V, orc, shape, loss):
    """Lattices thinner than the LNCC window, single planes (lattice_coord n = 1,
    geometry.hpp:101-104) and x extents off the 32-wide warp units, on random
    intensities and a random sub-voxel warp, against the oracle step."""
    from gpu_util import dev, host, maxrel
    r = orc.rng(500 + sum(shape))
    f = orc.random_volume(r, shape, 0.0, 1.0)
    m = np.clip(0.7 * f + 0.3 * orc.random_volume(r, shape, 0.0, 1.0), 0.0, 1.0)
    u = orc.random_volume(r, shape + (3,), -0.01, 0.01)
    A = np.eye(3) + orc.random_volume(r, (3, 3), -0.02, 0.02)
    t = orc.random_volume(r, (3,), -0.02, 0.02)
    f, m, u = (a.astype(np.float32).astype(np.float64) for a in (f, m, u))
    if loss == "lncc":
        ref = orc.step_lncc(f, m, u, A, t)
        p = V.LossParams(kind="lncc")
    else:
        ref = orc.step_mi(f, m, u, orc.parzen("bspline3", 32), A, t)
        p = V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True)
    res = V.warp_loss_step(dev(f), dev(m), dev(u), A, t, p)
    assert res.loss == pytest.approx(ref["loss"], rel=1e-5, abs=1e-7)
    assert maxrel(host(res.g_u), ref["g_u"]) <= 1e-4


@pytest.mark.parametrize("window", [3, 5, 9])
def test_step_lncc_other_windows(V, orc, window):
    """windows other than 7 (the fused kernel's) run the operator composition
    with the reference's semantics, at the parity gates."""
    from oracle import step_inputs
    si = step_inputs(orc, (24, 26, 28), seed=4242, loss="lncc")
    ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t, window=window)
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, V.LossParams(kind="lncc", window=window))
    assert res.loss == pytest.approx(ref["loss"], rel=LOSS_RTOL)
    assert maxrel(host(res.g_u), ref["g_u"]) <= GRAD_MAXREL
