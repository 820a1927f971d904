"""Sampler parity on the GPU vs the oracle (oracle/ffdp_oracle.c, pinned to the reference)."""
import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu, r32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


def args_of(V, A, t, S, bounds=None):
    a = V.SamplerArgs(A=np.asarray(A), t=np.asarray(t), S=np.asarray(S))
    if bounds is not None:
        a.bounds = V.DomainBounds(tuple(bounds[:3]), tuple(bounds[3:]))
    return a


@pytest.mark.parametrize("i", [0, 1, 2])
def test_margin_fixtures_fwd_bwd(V, orc, golden, i):
    g = lambda k: golden[f"smp{i}_{k}"]
    img, u, up = r32(g("img")), r32(g("u")), r32(g("up"))
    A, t, S = g("A"), g("t"), g("S")
    ref_f = orc.sample(img, u, A, t, S)["out"]
    ref_b = orc.sample(img, u, A, t, S, upstream=up, want=("image", "warp", "affine", "translation"))
    a = args_of(V, A, t, S)
    out = host(V.fused_sample(dev(img), dev(u), a))
    assert maxrel(out, ref_f) < 2e-6
    # against the reference's own golden output on the fp64 inputs: fp32 input rounding only
    assert maxrel(out, g("out")) < 1e-5
    gr = V.fused_sample_backward(dev(up), dev(img), dev(u), a, V.SamplerGradWant(True, True, True, True))
    assert maxrel(host(gr.warp), ref_b["warp"]) < 1e-5
    assert maxrel(host(gr.image), ref_b["image"]) < 1e-5
    assert maxrel(gr.affine, ref_b["affine"]) < 1e-5
    assert maxrel(gr.translation, ref_b["translation"]) < 1e-5


def test_identity_and_shift(V, orc):
    img = r32(orc.random_volume(orc.rng(101), (6, 7, 8)))
    out = host(V.fused_sample(dev(img), dev(np.zeros((6, 7, 8, 3))), V.SamplerArgs()))
    assert np.max(np.abs(out - img)) <= 1e-6
    n = 8
    ramp = np.broadcast_to(np.arange(n, dtype=np.float64), (n, n, n)).copy()
    a = V.SamplerArgs(t=np.array([2.0 / (n - 1), 0, 0]))
    out = host(V.fused_sample(dev(ramp), dev(np.zeros((n, n, n, 3))), a))
    assert np.allclose(out[:, :, :-1], ramp[:, :, 1:], atol=1e-5)
    assert np.all(out[:, :, -1] == 0.0)  # zero-padded border column (test_sampler.cpp:109-125)


def test_face_uses_floor_cell(V, golden):
    img, u, up = golden["face_img"], golden["face_u"], golden["face_up"]
    g = V.fused_sample_backward(dev(up), dev(img), dev(u), V.SamplerArgs(), V.SamplerGradWant(warp=True))
    gu = host(g.warp)
    img32 = r32(img)
    assert gu[2, 2, 2, 0] == pytest.approx((img32[2, 2, 4] - img32[2, 2, 3]) * 2.5, rel=1e-6)
    assert maxrel(gu, golden["face_gu"]) < 1e-6


def test_bounds_and_distinct_lattices(V, orc, golden):
    img, u, b = r32(golden["bnd_img"]), r32(golden["bnd_u"]), golden["bnd_bounds"]
    a = args_of(V, np.eye(3), np.zeros(3), np.ones(3), b)
    out = host(V.fused_sample(dev(img), dev(u), a))
    assert maxrel(out, orc.sample(img, u, bounds=b)["out"]) < 2e-6


def test_no_warp_uses_image_lattice(V, orc):
    img = r32(orc.random_volume(orc.rng(5), (5, 6, 7)))
    A = np.eye(3) + 0.03
    out = host(V.fused_sample(dev(img), None, V.SamplerArgs(A=A)))
    assert maxrel(out, orc.sample(img, None, A=A)["out"]) < 2e-6


def test_accumulate_and_abs_contribution(V, orc):
    img = r32(orc.random_volume(orc.rng(7), (6, 6, 6)))
    u = r32(orc.random_volume(orc.rng(8), (6, 6, 6, 3), -0.1, 0.1))
    import torch
    out = torch.ones((6, 6, 6), dtype=torch.float32, device="cuda")
    l1 = V.fused_sample_accumulate(dev(img), dev(u), V.SamplerArgs(), out, abs_contribution=True)
    ref = orc.sample(img, u)["out"]
    assert maxrel(host(out), 1.0 + ref) < 2e-6
    assert l1 == pytest.approx(np.abs(ref).sum(), rel=1e-6)


def test_rejects_bad_arguments(V):
    from paper_2509_25044_b200 import InvalidArgument
    import torch
    img = torch.zeros((6, 6, 6), device="cuda")
    w = torch.zeros((6, 6, 6, 3), device="cuda")
    with pytest.raises(InvalidArgument):
        V.fused_sample_backward(torch.zeros((5, 5, 5), device="cuda"), img, w, V.SamplerArgs(),
                                V.SamplerGradWant(image=True))
    with pytest.raises(ValueError):
        V.fused_sample(img, w, V.SamplerArgs(S=np.array([0.0, 1, 1])))
    with pytest.raises(ValueError):
        V.fused_sample(img, w, V.SamplerArgs(A=np.full((3, 3), np.nan)))


def test_zero_upstream_zero_gradients(V, orc):
    img = r32(orc.random_volume(orc.rng(113), (6, 6, 6)))
    u = r32(orc.random_volume(orc.rng(114), (6, 6, 6, 3), -0.1, 0.1))
    import torch
    g = V.fused_sample_backward(torch.zeros((6, 6, 6), device="cuda"), dev(img), dev(u), V.SamplerArgs(),
                                V.SamplerGradWant(True, True, True, True))
    assert not host(g.image).any() and not host(g.warp).any()
    assert not g.affine.any() and not g.translation.any()


def test_sampler_linearity(V, orc):
    """test_sampler.cpp:138-151: the sample is linear in the image."""
    a = orc.random_volume(orc.rng(141), (6, 7, 8))
    b = orc.random_volume(orc.rng(142), (6, 7, 8))
    u = r32(orc.random_volume(orc.rng(143), (6, 7, 8, 3), -0.05, 0.05))
    args = V.SamplerArgs()
    sa = host(V.fused_sample(dev(r32(a)), dev(u), args)).astype(np.float64)
    sb = host(V.fused_sample(dev(r32(b)), dev(u), args)).astype(np.float64)
    sab = host(V.fused_sample(dev(r32(2.0 * a - 0.5 * b)), dev(u), args)).astype(np.float64)
    assert np.max(np.abs(sab - (2.0 * sa - 0.5 * sb))) <= 1e-5


def test_sampler_allocates_only_its_output(V, orc):
    """test_sampler.cpp:89-107: fused_sample allocates exactly one output lattice."""
    import torch
    img = dev(r32(orc.random_volume(orc.rng(89), (20, 21, 22))))
    u = dev(r32(orc.random_volume(orc.rng(90), (20, 21, 22, 3), -0.05, 0.05)))
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    out = V.fused_sample(img, u, V.SamplerArgs())
    torch.cuda.synchronize()
    grown = torch.cuda.memory_allocated() - before
    assert out.numel() * 4 <= grown <= out.numel() * 4 + 511  # one block (allocator rounds to 512 B)
