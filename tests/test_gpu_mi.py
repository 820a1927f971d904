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
