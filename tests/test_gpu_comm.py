"""The C ABI's sharded context (ffdp_comm, csrc/comm.cu) at H = 2 and 3 ranks sharing
one GPU: every collective against the same operator on the whole volume (the reference's
invariance property, test_distops.cpp:47-423), and its argument errors
(fabric.hpp:315-370)."""
import numpy as np
import pytest

from gpu_util import maxrel, need_gpu

pytestmark = pytest.mark.gpu
SHAPE = (19, 22, 37)


def _inputs():
    rng = np.random.default_rng(31)
    f = rng.uniform(0, 1, SHAPE).astype(np.float32)
    m = np.clip(0.7 * f + 0.3 * rng.uniform(0, 1, SHAPE), 0, 1).astype(np.float32)
    u = rng.uniform(-0.03, 0.03, SHAPE + (3,)).astype(np.float32)
    A = np.eye(3) + rng.uniform(-0.03, 0.03, (3, 3))
    t = rng.uniform(-0.03, 0.03, 3)
    up = rng.uniform(-1, 1, SHAPE).astype(np.float32)
    return f, m, u, A, t, up


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


def cat(ts):
    return np.concatenate([t.cpu().numpy() for t in ts], axis=0)


@pytest.mark.parametrize("world", [2, 3])
def test_comm_collectives_match_single_gpu(V, world):
    import torch
    from paper_2509_25044_b200.comm import Comm
    f, m, u, A, t, up = _inputs()
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    args = V.SamplerArgs(A=A, t=t)
    with Comm(world, [0] * world) as c:
        assert c.world == world and c.devices == [0] * world
        assert [c.shard_range(SHAPE[0], r) for r in range(world)] == \
            [(r * (19 // world) + min(r, 19 % world), (r + 1) * (19 // world) + min(r + 1, 19 % world))
             for r in range(world)]
        fs, ms, us, ups = c.scatter(T(f)), c.scatter(T(m)), c.scatter(T(u)), c.scatter(T(up))
        # halo exchange: the padded slabs are the global planes
        hs, lo, hi = c.halo_exchange(us, SHAPE, 2)
        for r in range(world):
            a, b = c.shard_range(SHAPE[0], r)
            assert lo[r] == (2 if r else 0) and hi[r] == (2 if r < world - 1 else 0)
            assert np.array_equal(hs[r].cpu().numpy(), u[a - lo[r]:b + hi[r]])
        # gp_convolve with halos = the whole-volume convolution, bit for bit; the ablation
        # convolves each shard alone
        taps = V.gaussian_taps(1.0)
        assert np.array_equal(cat(c.gp_convolve(us, taps, SHAPE, "renormalize")),
                              V.gp_convolve(T(u), taps, "renormalize").cpu().numpy())
        alone = c.gp_convolve(us, taps, SHAPE, "renormalize", sync=False)
        for r in range(world):
            assert np.array_equal(alone[r].cpu().numpy(), V.gp_convolve(us[r], taps, "renormalize").cpu().numpy())
        # ring sample forward / backward
        moved = V.fused_sample(T(m), T(u), args)
        ms_moved = c.ring_sample(ms, SHAPE, us, SHAPE, A, t)
        assert maxrel(cat(ms_moved), moved.cpu().numpy()) <= 1e-6
        g = V.fused_sample_backward(T(up), T(m), T(u), args,
                                    V.SamplerGradWant(image=True, warp=True, affine=True, translation=True))
        gi, gu, gA, gt = c.ring_sample_backward(ups, ms, SHAPE, us, SHAPE, A, t,
                                                want=("image", "warp", "affine", "translation"))
        assert maxrel(cat(gu), g.warp.cpu().numpy()) <= 1e-6
        assert maxrel(cat(gi), g.image.cpu().numpy()) <= 1e-5
        assert np.max(np.abs(gA - g.affine)) <= 1e-6 * max(1.0, np.max(np.abs(g.affine)))
        assert np.max(np.abs(gt - g.translation)) <= 1e-6 * max(1.0, np.max(np.abs(g.translation)))
        # the distributed losses on the moved slabs vs the operators on the whole volume
        n = int(np.prod(SHAPE))
        fm, mm = T(f), moved
        sm = ((mm.double() - fm.double()) ** 2).sum().item() / n
        lv, gv = c.dist_mse(fs, ms_moved, SHAPE)
        assert lv == pytest.approx(sm, rel=1e-6) and maxrel(cat(gv), (2.0 * (mm - fm) / n).cpu().numpy()) <= 1e-5
        k = V.ParzenKernel.bspline3(32)
        res = V.mi_forward_exact(fm, mm, 32, k)
        lv, gv, payload = c.dist_mi(fs, ms_moved, SHAPE, k)
        assert payload == 32 * 32 + 64
        assert lv == pytest.approx(-res.mi, rel=1e-6)
        assert maxrel(cat(gv), V.mi_backward(-1.0, fm, mm, res.hist, k)[1].cpu().numpy()) <= 1e-5
        for ants in (True, False):
            lr, st = V.lncc_forward_fused(fm, mm, 7, 1e-5)
            ref_g = V.lncc_backward_fused(1.0, st, fm, mm, ants)[1].cpu().numpy()
            lv, gv = c.dist_lncc(fs, ms_moved, SHAPE, 7, 1e-5, ants)
            assert lv == pytest.approx(lr.loss, rel=1e-6), ants
            assert maxrel(cat(gv), ref_g) <= 1e-5, ants
        # determinism: rank-ordered reductions repeat bit for bit
        assert c.dist_lncc(fs, ms_moved, SHAPE)[0] == c.dist_lncc(fs, ms_moved, SHAPE)[0]


def test_comm_errors(V):
    import torch
    from paper_2509_25044_b200._lib import InvalidArgument
    from paper_2509_25044_b200.comm import Comm
    with pytest.raises(InvalidArgument):
        Comm(2, [0, 99])
    with pytest.raises(InvalidArgument):
        Comm(0)
    with Comm(3, [0, 0, 0]) as c:
        v = torch.zeros((7, 4, 5), device="cuda")
        sl = c.scatter(v)  # thicknesses 3, 2, 2
        with pytest.raises(InvalidArgument, match="pad exceeds"):
            c.halo_exchange(sl, (7, 4, 5), 3)
        with pytest.raises(InvalidArgument):
            c.dist_lncc(sl, sl, (7, 4, 5), window=4)
        with pytest.raises(InvalidArgument):
            c.halo_exchange(sl[:2], (7, 4, 5), 1)


@pytest.mark.parametrize("loss", ["lncc", "mi"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_comm_fused_step_matches_single_gpu(V, orc, loss, world):
    """ffdp_dist_step (the sharded deformable step of the C ABI) against the single-GPU
    fused step on the whole volume, at the survey's parity gates."""
    import torch
    from oracle import step_inputs
    from paper_2509_25044_b200.comm import Comm
    si = step_inputs(orc, (40, 44, 48), seed=4242, loss=loss)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    f, m, u = T(si.f), T(si.m), T(si.u)
    p = V.LossParams(kind=loss, mi_bspline_kernel=True)
    ref = V.warp_loss_step(f, m, u, si.A, si.t, p)
    with Comm(world, [0] * world) as c:
        lv, g = c.step(c.scatter(f), c.scatter(m), c.scatter(u), tuple(f.shape), si.A, si.t, p)
        lv2, g2 = c.step(c.scatter(f), c.scatter(m), c.scatter(u), tuple(f.shape), si.A, si.t, p)
    assert lv == lv2 and all(torch.equal(a, b) for a, b in zip(g, g2))  # rank-ordered: deterministic
    assert abs(lv - ref.loss) <= 1e-5 * abs(ref.loss)
    assert maxrel(cat(g), ref.g_u.cpu().numpy()) <= 1e-4
    if world == 1 and loss == "lncc":
        assert lv == ref.loss and np.array_equal(cat(g), ref.g_u.cpu().numpy())


def test_comm_step_fd_across_ranks(V, orc):
    """test_distops.cpp:314-367: the gradient through the collective (2 ranks, MI B-spline
    step) matches a directional finite difference of the reduced loss (5%: fp32)."""
    import torch
    from oracle import step_inputs
    from paper_2509_25044_b200.comm import Comm
    si = step_inputs(orc, (40, 44, 48), seed=4242, loss="mi")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    f, m, u = T(si.f), T(si.m), T(si.u)
    p = V.LossParams(kind="mi", mi_bspline_kernel=True)
    gen = torch.Generator(device="cuda").manual_seed(6)
    v = V.gp_convolve(torch.randn(u.shape, device="cuda", generator=gen).contiguous(), V.gaussian_taps(2.0),
                      "renormalize")
    with Comm(2, [0, 0]) as c:
        fs, ms = c.scatter(f), c.scatter(m)
        loss = lambda uu: c.step(fs, ms, c.scatter(uu.contiguous()), tuple(f.shape), si.A, si.t, p)
        _, g = loss(u)
        g = torch.cat([x.double() for x in g], 0)
        for vox in (0.01, 0.03):
            d = v / v.abs().max() * (vox * 2.0 / 39)
            fd = (loss(u + d)[0] - loss(u - d)[0]) / 2.0
            an = float((g * d.double()).sum())
            assert abs(fd - an) <= 5e-2 * abs(an), (vox, fd, an)


@pytest.mark.parametrize("world", [2, 3])
def test_comm_ring_sample_distinct_lattices(V, world):
    """ring_sample with a moving lattice different from the output lattice
    (distops.hpp:144-168 allows it; test_distops.cpp:139-289 pattern)."""
    import torch
    from paper_2509_25044_b200.comm import Comm
    rng = np.random.default_rng(61)
    m = rng.uniform(0, 1, (21, 23, 25)).astype(np.float32)
    u = rng.uniform(-0.04, 0.04, SHAPE + (3,)).astype(np.float32)
    up = rng.uniform(-1, 1, SHAPE).astype(np.float32)
    A = np.eye(3) + rng.uniform(-0.03, 0.03, (3, 3))
    t = rng.uniform(-0.03, 0.03, 3)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    args = V.SamplerArgs(A=A, t=t)
    ref = V.fused_sample(T(m), T(u), args).cpu().numpy()
    g = V.fused_sample_backward(T(up), T(m), T(u), args, V.SamplerGradWant(image=True, warp=True))
    with Comm(world, [0] * world) as c:
        ms, us, ups = c.scatter(T(m)), c.scatter(T(u)), c.scatter(T(up))
        out = c.ring_sample(ms, m.shape, us, SHAPE, A, t)
        assert maxrel(cat(out), ref) <= 1e-6
        gi, gu, _, _ = c.ring_sample_backward(ups, ms, m.shape, us, SHAPE, A, t, want=("image", "warp"))
        assert maxrel(cat(gu), g.warp.cpu().numpy()) <= 1e-6
        assert maxrel(cat(gi), g.image.cpu().numpy()) <= 1e-5
