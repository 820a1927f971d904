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
