"""The warp update of the deformable step on the GPU (registration.hpp:313-317):
ffdp_gp_convolve (gp_convolve / separable_convolve, distops.hpp:54-101,
smoothing.hpp:52-105) and ffdp_sobolev_adam (gp_convolve of g_u fused with adam_step,
adam.hpp:30-50) against the oracle (tests/test_oracle_golden.py pins the oracle's warp
update to the reference itself, H = 1 and 3). Tolerances: smoothing rel 1e-6 of the
field's max (fp32 sums of <= 9^3 taps), Adam rel 1e-5 (fp32 moments)."""
import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


# odd lattices spanning several 32 x 16 tiles, with a ragged last tile
SHAPES = [(11, 19, 37), (7, 33, 65), (1, 5, 6)]
TAPS = {"box7": np.full(7, 1 / 7), "g1.0": None, "g0.5": None, "g1.3": None, "unit": np.ones(1)}


def taps_of(orc, name):
    if TAPS[name] is not None:
        return TAPS[name]
    return orc.gaussian_taps(float(name[1:]))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("channels", [1, 3])
@pytest.mark.parametrize("mode", ["zero_pad", "renormalize"])
@pytest.mark.parametrize("tname", ["box7", "g1.0", "g0.5", "g1.3", "unit"])
def test_gp_convolve_matches_oracle(V, orc, shape, channels, mode, tname):
    taps = taps_of(orc, tname)
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, shape + ((3,) if channels == 3 else ()))
    x = x.astype(np.float32).astype(np.float64)
    ref = orc.separable_convolve(x, taps, mode=mode, channels=channels)
    got = host(V.gp_convolve(dev(x), taps, mode))
    assert maxrel(got, ref) <= 1e-6


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("mode", ["zero_pad", "renormalize"])
def test_gp_convolve_sharded_equals_unsharded(V, orc, world, mode):
    """distops.hpp:54-101 / smoothing.hpp:10-13: a halo-padded slab sees the same taps as
    the unsharded volume -- here bit for bit (same per-voxel arithmetic)."""
    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200._lib import Slab
    shape = (17, 21, 40)
    taps = orc.gaussian_taps(1.0)
    r = len(taps) // 2
    x = np.random.default_rng(3).uniform(-1, 1, shape + (3,))
    full = V.gp_convolve(dev(x), taps, mode)
    xt = dev(x)
    parts = []
    for lo, hi in D.shard_ranges(shape[0], world):
        b0, b1 = max(0, lo - r), min(shape[0], hi + r)
        parts.append(V.gp_convolve(xt[b0:b1].contiguous(), taps, mode, slab=Slab(b0, b1 - b0, lo, hi, shape[0])))
    import torch
    assert torch.equal(torch.cat(parts, 0), full)


def test_gp_convolve_rejects(V):
    import torch

    from paper_2509_25044_b200._lib import InvalidArgument, Slab
    x = torch.zeros((8, 8, 8), device="cuda")
    with pytest.raises(InvalidArgument):
        V.gp_convolve(x, np.ones(4) / 4)  # even kernel (distops.hpp:87,97)
    with pytest.raises(InvalidArgument):
        V.gp_convolve(x, np.ones(15) / 15)  # radius above the kernel's limit (6)
    with pytest.raises(InvalidArgument):
        # planes [2, 6) of a 12-plane lattice with only 1 halo plane for a radius-3 window
        V.gp_convolve(x[:6].contiguous(), np.full(7, 1 / 7), slab=Slab(1, 6, 2, 6, 12))


@pytest.mark.parametrize("shape", [(11, 19, 37), (6, 17, 33)])
def test_warp_update_matches_oracle(V, orc, shape):
    """Two consecutive warp updates (Adam steps 1 and 2) vs the oracle's fp64 restatement.
    Adam's step is sign-like where the smoothed gradient is small against eps-free |g|
    (d/dg of g / (|g| + eps) is 1/eps at 0), so the Adam output is compared where
    |g_s| > 1e-3 max|g_s|; the moments everywhere; the final smoothing on the GPU's own
    Adam output (its error does not depend on that conditioning)."""
    rng = np.random.default_rng(5)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    tg, tw = orc.gaussian_taps(1.0), orc.gaussian_taps(0.5)
    g = r32(rng.uniform(-1e-3, 1e-3, shape + (3,)))
    u_ref = r32(rng.uniform(-0.02, 0.02, shape + (3,)))
    a_ref, b_ref = np.zeros_like(u_ref), np.zeros_like(u_ref)
    lr = V.deformable_lr_norm(shape, 0.5)
    u = dev(u_ref)
    st = V.AdamState.zeros(u)
    for step, scale in ((1, 1.0), (2, 0.5)):
        gs = orc.separable_convolve(scale * g, tg, "renormalize", 3)
        p_ref, a_ref, b_ref = orc.adam_step(u_ref, gs, a_ref, b_ref, lr, step)
        out = V.warp_update(u, dev(scale * g), st, lr)
        assert st.step == step
        assert maxrel(host(st.m1), a_ref) <= 1e-5 and maxrel(host(st.m2), b_ref) <= 1e-5
        mask = np.abs(gs) > 1e-3 * np.max(np.abs(gs))
        assert mask.mean() > 0.95
        err = np.abs(host(u) - p_ref)[mask]
        assert np.max(err) <= 1e-5 * np.max(np.abs(p_ref))
        assert maxrel(host(out), orc.separable_convolve(host(u), tw, "renormalize", 3)) <= 1e-6
        # the next step starts from the GPU state (as the reference loop would)
        u_ref, a_ref, b_ref = host(out), host(st.m1), host(st.m2)
        u = out


def test_adam_step_matches_oracle(V, orc):
    """adam_step (adam.hpp:30-50) alone, three steps."""
    shape = (5, 9, 34)
    rng = np.random.default_rng(9)
    p = rng.uniform(-1, 1, shape + (3,)).astype(np.float32).astype(np.float64)
    pr, ar, br = p, np.zeros_like(p), np.zeros_like(p)
    pt = dev(p)
    st = V.AdamState.zeros(pt)
    for k in range(1, 4):
        gk = rng.uniform(-1, 1, shape + (3,)).astype(np.float32).astype(np.float64)
        pr, ar, br = orc.adam_step(pr, gk, ar, br, 0.01, k)
        V.adam_step(pt, dev(gk), st, 0.01)
    assert maxrel(host(pt), pr) <= 1e-6
    assert maxrel(host(st.m1), ar) <= 1e-6 and maxrel(host(st.m2), br) <= 1e-6


def test_sharded_warp_update_equals_unsharded(V, orc):
    """dist.sharded_warp_update on emulated ranks (halo slices instead of the exchange)
    equals the single-GPU update bit for bit."""
    import torch

    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200._lib import Slab
    shape = (19, 18, 35)
    rng = np.random.default_rng(21)
    g = dev(rng.uniform(-1e-3, 1e-3, shape + (3,)))
    u0 = dev(rng.uniform(-0.02, 0.02, shape + (3,)))
    lr = 0.01
    st = V.AdamState.zeros(u0)
    u_ref = u0.clone()
    full = V.warp_update(u_ref, g, st, lr)
    tg, tw = V.gaussian_taps(1.0), V.gaussian_taps(0.5)
    parts = []
    for lo, hi in D.shard_ranges(shape[0], 3):
        # rank-local emulation of sharded_warp_update with the halos sliced from the full fields
        sts = V.AdamState.zeros(u0[lo:hi])
        u_s = u0[lo:hi].clone()
        b0, b1 = max(0, lo - 3), min(shape[0], hi + 3)
        from paper_2509_25044_b200._lib import lib
        sts.step += 1
        lib.ffdp_sobolev_adam(V._ptr(g[b0:b1].contiguous()), V._ptr(u_s), V._ptr(sts.m1), V._ptr(sts.m2),
                              V._dims((b1 - b0,) + shape[1:]), Slab(b0, b1 - b0, lo, hi, shape[0]), V._taps_ptr(tg),
                              len(tg), lr, 0.9, 0.999, 1e-8, 1, V._stream())
        parts.append((lo, hi, u_s))
    # second half: smoothing of the updated u with 2 halo planes from the neighbours' slabs
    u_upd = torch.cat([p[2] for p in parts], 0)
    assert torch.equal(u_upd, u_ref)
    out = []
    for lo, hi, _ in parts:
        b0, b1 = max(0, lo - 2), min(shape[0], hi + 2)
        out.append(V.gp_convolve(u_upd[b0:b1].contiguous(), tw, "renormalize",
                                 slab=Slab(b0, b1 - b0, lo, hi, shape[0])))
    assert torch.equal(torch.cat(out, 0), full)
