"""LNCC operator parity on the GPU vs the oracle."""
import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu, r32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


@pytest.mark.parametrize("i", [0, 1, 2])
@pytest.mark.parametrize("ants", [True, False])
def test_lncc_vs_oracle(V, orc, golden, i, ants):
    f, m, w = r32(golden[f"lncc{i}_f"]), r32(golden[f"lncc{i}_m"]), int(golden[f"lncc{i}_w"])
    loss, state, mp = orc.lncc_forward(f, m, window=w, want_map=True)
    gf, gm, _ = orc.lncc_backward(1.3, state, f, m, window=w, ants=ants)
    res, st = V.lncc_forward_fused(dev(f), dev(m), w, 1e-5, want_map=True)
    assert res.loss == pytest.approx(loss, rel=1e-9)
    assert maxrel(host(st.channels), state) < 1e-12
    assert maxrel(host(res.ncc_map), mp) < 1e-6
    g1, g2 = V.lncc_backward_fused(1.3, st, dev(f), dev(m), ants)
    assert maxrel(host(g1), gf) < 1e-6
    assert maxrel(host(g2), gm) < 1e-6


def test_lncc_self_similarity_and_constants(V, orc):
    f = r32(orc.random_volume(orc.rng(211), (12, 12, 12)))
    res, _ = V.lncc_forward_fused(dev(f), dev(f), 7, 1e-12, want_map=True)
    mp = host(res.ncc_map)[3:-3, 3:-3, 3:-3]
    assert np.allclose(mp, 1.0, atol=1e-6)  # test_lncc.cpp:27-33 (interior)
    c = np.full((10, 10, 10), 0.5)
    res, _ = V.lncc_forward_fused(dev(c), dev(c), 7, 1e-5, want_map=True)
    assert np.allclose(host(res.ncc_map)[3:-3, 3:-3, 3:-3], 0.0, atol=1e-9)


def test_lncc_rejects(V):
    import torch
    a = torch.zeros((6, 6, 6), device="cuda")
    with pytest.raises(ValueError):
        V.lncc_forward_fused(a, torch.zeros((5, 6, 6), device="cuda"), 7, 1e-5)
    with pytest.raises(ValueError):
        V.lncc_forward_fused(a, a, 4, 1e-5)


def test_convolve_axis_matches_oracle(V, orc):
    v = r32(orc.random_volume(orc.rng(9), (9, 8, 7)))
    taps = orc.gaussian_taps(1.0)
    for axis in range(3):
        for mode in ("zero_pad", "renormalize"):
            out = host(V.convolve_axis(dev(v), axis, taps, renormalize=(mode == "renormalize")))
            ref = orc.convolve_axis(v, axis, taps, mode)
            assert maxrel(out, ref) < 1e-6


def _interior(a, r):
    return a[r:-r, r:-r, r:-r]


def test_lncc_affine_intensity_invariance(V, orc):
    """test_lncc.cpp:38-53: M = 1.7 F + 0.4 correlates perfectly in full windows (eps 0)."""
    f = r32(orc.random_volume(orc.rng(223), (12, 12, 12)))
    m = r32(1.7 * f.astype(np.float64) + 0.4)
    res, _ = V.lncc_forward_fused(dev(f), dev(m), 5, 0.0, want_map=True)
    assert np.allclose(_interior(host(res.ncc_map), 2), 1.0, atol=1e-5)


def test_lncc_near_stationary_at_self_similarity(V, orc):
    """test_lncc.cpp:159-173: with F == M the exact gradient is O(eps) and far below a
    generic pair's."""
    f = r32(orc.random_volume(orc.rng(241), (12, 12, 12)))
    other = r32(orc.random_volume(orc.rng(242), (12, 12, 12)))
    _, st = V.lncc_forward_fused(dev(f), dev(f), 5, 1e-5)
    gf, gm = V.lncc_backward_fused(1.0, st, dev(f), dev(f), False)
    bound = 2e-5 * np.linalg.norm(f.astype(np.float64))
    assert np.linalg.norm(host(gf)) <= bound and np.linalg.norm(host(gm)) <= bound
    _, st2 = V.lncc_forward_fused(dev(f), dev(other), 5, 1e-5)
    gf2, _ = V.lncc_backward_fused(1.0, st2, dev(f), dev(other), False)
    assert np.linalg.norm(host(gf)) <= 0.01 * np.linalg.norm(host(gf2))


def test_lncc_swap_symmetry(V, orc):
    """test_lncc.cpp:175-185: swapping F and M swaps the gradients (bit-exact in the
    reference; here the 5 channels are formed in the same order either way)."""
    f = r32(orc.random_volume(orc.rng(251), (9, 9, 9)))
    m = r32(orc.random_volume(orc.rng(252), (9, 9, 9)))
    _, s1 = V.lncc_forward_fused(dev(f), dev(m), 5, 1e-5)
    gf1, gm1 = V.lncc_backward_fused(1.0, s1, dev(f), dev(m), False)
    _, s2 = V.lncc_forward_fused(dev(m), dev(f), 5, 1e-5)
    gm2, gf2 = V.lncc_backward_fused(1.0, s2, dev(m), dev(f), False)
    assert maxrel(host(gf1), host(gf2).astype(np.float64)) <= 1e-6
    assert maxrel(host(gm1), host(gm2).astype(np.float64)) <= 1e-6


def test_lncc_ants_equals_exact_for_window_1(V, orc):
    """test_lncc.cpp:187-199: with a 1-voxel window the gamma box filter is the identity."""
    f = r32(orc.random_volume(orc.rng(257), (7, 7, 7)))
    m = r32(orc.random_volume(orc.rng(258), (7, 7, 7)))
    _, s1 = V.lncc_forward_fused(dev(f), dev(m), 1, 1e-5)
    ge = V.lncc_backward_fused(1.0, s1, dev(f), dev(m), False)
    _, s2 = V.lncc_forward_fused(dev(f), dev(m), 1, 1e-5)
    ga = V.lncc_backward_fused(1.0, s2, dev(f), dev(m), True)
    for a, b in zip(ge, ga):
        assert maxrel(host(a), host(b).astype(np.float64)) <= 1e-6


def test_lncc_loss_non_decreasing_in_eps(V, orc):
    """test_lncc.cpp:201-211."""
    f = r32(orc.random_volume(orc.rng(263), (10, 10, 10)))
    m = r32(orc.random_volume(orc.rng(264), (10, 10, 10)))
    losses = [V.lncc_forward_fused(dev(f), dev(m), 5, eps)[0].loss for eps in (0.0, 1e-6, 1e-4, 1e-2, 1.0)]
    assert all(b >= a for a, b in zip(losses, losses[1:]))


def test_lncc_state_is_five_lattices(V, orc):
    """test_lncc.cpp:81-98: the fused forward keeps exactly the 5 channel lattices."""
    f = r32(orc.random_volume(orc.rng(81), (9, 10, 11)))
    m = r32(orc.random_volume(orc.rng(82), (9, 10, 11)))
    _, st = V.lncc_forward_fused(dev(f), dev(m), 5, 1e-5)
    assert tuple(st.channels.shape) == (5, 9, 10, 11)


@pytest.mark.parametrize("ants", [True, False])
def test_lncc_fwdbwd_one_call(V, orc, golden, ants):
    """ffdp_lncc_fwdbwd / ffdp_lncc_bwd (the one-call forward + backward of the survey's
    ABI list) equal lncc_forward_fused + lncc_backward_fused."""
    import ctypes as C
    import torch
    from paper_2509_25044_b200._lib import lib
    f, m, w = r32(golden["lncc1_f"]), r32(golden["lncc1_m"]), int(golden["lncc1_w"])
    res, st = V.lncc_forward_fused(dev(f), dev(m), w, 1e-5)
    g1, g2 = V.lncc_backward_fused(1.3, st, dev(f), dev(m), ants)
    ft, mt = dev(f), dev(m)
    state = torch.empty((5,) + ft.shape, dtype=torch.float64, device="cuda")
    sn = torch.zeros(1, dtype=torch.float64, device="cuda")
    gf, gm = torch.empty_like(ft), torch.empty_like(mt)
    lib.ffdp_lncc_fwdbwd(V._ptr(ft), V._ptr(mt), V._dims(ft.shape), w, 1e-5, int(ants), 1.3, V._ptr(state),
                         V._ptr(sn), V._ptr(gf), V._ptr(gm), V._stream())
    assert 1.0 - float(sn.item()) / ft.numel() == res.loss
    assert torch.equal(gf, g1) and torch.equal(gm, g2)
