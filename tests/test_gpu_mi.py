"""Mattes MI operator parity on the GPU vs the oracle."""
import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu, r32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


def make(V, kind, bins):
    return {"gaussian": V.ParzenKernel.gaussian, "bspline3": V.ParzenKernel.bspline3,
            "delta": V.ParzenKernel.delta}[kind](bins)


@pytest.mark.parametrize("kind", ["gaussian", "bspline3", "delta"])
@pytest.mark.parametrize("bins", [8, 32])
@pytest.mark.parametrize("approx", [False, True])
def test_mi_forward_backward(V, orc, golden, kind, bins, approx):
    vi, vj = r32(golden["mi_i"]), r32(golden["mi_j"])
    k = orc.parzen(kind, bins)
    h = orc.mi_forward(vi, vj, k, approx=approx)
    kk = make(V, kind, bins)
    res = (V.mi_forward_approx if approx else V.mi_forward_exact)(dev(vi), dev(vj), bins, kk)
    # fixed point 2^-20 per accumulated contribution
    assert res.mi == pytest.approx(h["mi"], rel=1e-6, abs=1e-9)
    raw = np.concatenate([res.hist.raw_joint, res.hist.raw_marg_i, res.hist.raw_marg_j])
    assert np.max(np.abs(raw - h["raw"])) < 1e-5 * max(1.0, np.max(h["raw"]))
    assert (res.stats.hist_writes, res.stats.kernel_evals) == tuple(int(s) for s in h["stats"])
    if not approx:
        gi, gj, _ = orc.mi_backward(-1.0, vi, vj, k, h)
        g1, g2 = V.mi_backward(-1.0, dev(vi), dev(vj), res.hist, kk)
        assert maxrel(host(g1), gi) < 1e-4
        assert maxrel(host(g2), gj) < 1e-4


def test_mi_rejects(V):
    import torch
    a = torch.full((4, 4, 4), 0.5, device="cuda")
    with pytest.raises(ValueError):
        V.mi_forward_exact(a, a, 1, V.ParzenKernel.gaussian(8))
    with pytest.raises(ValueError):
        V.mi_forward_exact(a, torch.full((4, 4, 4), 1.5, device="cuda"), 8, V.ParzenKernel.gaussian(8))
    with pytest.raises(ValueError):
        V.mi_forward_exact(a, torch.full((3, 4, 4), 0.5, device="cuda"), 8, V.ParzenKernel.gaussian(8))


def test_self_mi_is_entropy(V, orc):
    v = r32(orc.random_volume(orc.rng(163), (10, 10, 10), 0.02, 0.98))
    k = V.ParzenKernel.gaussian(8)
    res = V.mi_forward_exact(dev(v), dev(v), 8, k)
    p = res.hist.p_i
    ent = -np.sum(p[p > 0] * np.log(p[p > 0]))
    assert 0 < res.mi <= ent + 1e-9


def _margin(orc, seed, shape, bins):
    """Intensities kept half a bin inside [0, 1] (test_mi.cpp:56-69)."""
    lo = 0.5 / bins
    return r32(orc.random_volume(orc.rng(seed), shape, lo, 1.0 - lo))


def test_mi_independent_noise_small(V, orc):
    """test_mi.cpp:188-196: independent noise has MI within the finite-sample bias."""
    a, b = _margin(orc, 331, (32, 32, 32), 32), _margin(orc, 332, (32, 32, 32), 32)
    for k in (V.ParzenKernel.gaussian(32), V.ParzenKernel.bspline3(32)):
        res = V.mi_forward_exact(dev(a), dev(b), 32, k)
        assert -1e-9 <= res.mi <= 0.05


def test_mi_symmetric(V, orc):
    """test_mi.cpp:198-207."""
    a, b = _margin(orc, 337, (9, 9, 9), 12), _margin(orc, 338, (9, 9, 9), 12)
    for k in (V.ParzenKernel.gaussian(12), V.ParzenKernel.bspline3(12)):
        ab = V.mi_forward_exact(dev(a), dev(b), 12, k).mi
        ba = V.mi_forward_exact(dev(b), dev(a), 12, k).mi
        assert ab == pytest.approx(ba, abs=1e-9)


def test_mi_approx_collapses_at_bin_centres_and_for_delta(V, orc):
    """test_mi.cpp:224-238 and 259-270: at bin centres (Gaussian) and for the delta kernel
    the binned forward equals the Parzen one."""
    rng = np.random.default_rng(349)
    bins = 8
    a = ((rng.integers(0, bins, (8, 8, 8)) + 0.5) / bins).astype(np.float32)
    b = ((rng.integers(0, bins, (8, 8, 8)) + 0.5) / bins).astype(np.float32)
    k = V.ParzenKernel.gaussian(bins)
    ex, ap = V.mi_forward_exact(dev(a), dev(b), bins, k), V.mi_forward_approx(dev(a), dev(b), bins, k)
    assert np.max(np.abs(ex.hist.p_ij - ap.hist.p_ij)) <= 1e-6
    assert ex.mi == pytest.approx(ap.mi, abs=1e-6)
    a, b = _margin(orc, 359, (7, 7, 7), bins), _margin(orc, 360, (7, 7, 7), bins)
    k = V.ParzenKernel.delta(bins)
    ex, ap = V.mi_forward_exact(dev(a), dev(b), bins, k), V.mi_forward_approx(dev(a), dev(b), bins, k)
    assert np.max(np.abs(ex.hist.p_ij - ap.hist.p_ij)) <= 1e-7
    assert ex.mi == pytest.approx(ap.mi, abs=1e-7)


def test_mi_approx_close_on_random_input(V, orc):
    """test_mi.cpp:243-257: L1(p_exact, p_approx) <= 0.15, |dMI| <= 0.05 at 16^3, B = 32."""
    a, b = _margin(orc, 353, (16, 16, 16), 32), _margin(orc, 354, (16, 16, 16), 32)
    k = V.ParzenKernel.gaussian(32)
    ex, ap = V.mi_forward_exact(dev(a), dev(b), 32, k), V.mi_forward_approx(dev(a), dev(b), 32, k)
    assert np.sum(np.abs(ex.hist.p_ij - ap.hist.p_ij)) <= 0.15
    assert abs(ex.mi - ap.mi) <= 0.05
    assert np.all(ap.hist.p_ij >= 0) and abs(np.sum(ap.hist.p_ij) - 1.0) <= 1e-9


def test_mi_zero_upstream_and_constant_image(V, orc):
    """test_mi.cpp:308-334: zero upstream -> zero gradients; a constant pair -> a uniform
    gradient on the constant image."""
    bins = 8
    k = V.ParzenKernel.gaussian(bins)
    a, b = _margin(orc, 373, (5, 5, 5), bins), _margin(orc, 374, (5, 5, 5), bins)
    fwd = V.mi_forward_exact(dev(a), dev(b), bins, k)
    ga, gb = V.mi_backward(0.0, dev(a), dev(b), fwd.hist, k)
    assert not np.any(host(ga)) and not np.any(host(gb))
    ca = np.full((5, 5, 5), 0.4, np.float32)
    cb = np.full((5, 5, 5), 0.6, np.float32)
    fwd2 = V.mi_forward_exact(dev(ca), dev(cb), bins, k)
    ga2, _ = V.mi_backward(1.0, dev(ca), dev(cb), fwd2.hist, k)
    g = host(ga2).ravel()
    assert np.all(g == g[0])
