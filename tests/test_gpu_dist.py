"""The sharded step (dist.ShardedStep) as real multi-process runs on ONE GPU: world 2 and 3
ranks over gloo (CUDA tensors staged through the host; on a B200 node the same code runs
over NCCL, one rank per GPU). Each rank owns a z slab of the oracle's fixture; the
concatenated g_u slabs and the (rank-identical) loss are checked against the oracle's
unsharded step (dist_lncc / dist_mi at H = 1, distops.hpp:285-396) -- the reference's
own shard-invariance property (test_distops.cpp:369-423)."""
import numpy as np
import pytest

from gpu_util import maxrel, need_gpu
from test_dist_gloo import spawn

pytestmark = pytest.mark.gpu

SHAPE = (30, 28, 32)


def _inputs(loss):
    from oracle import Oracle, step_inputs
    return step_inputs(Oracle(), SHAPE, seed=4242, loss=loss)


def w_sharded(rank, world, loss):
    import torch

    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200 import voxreg as V
    si = _inputs(loss)
    spec = D.make_shard_spec(SHAPE, world, rank)
    sl = slice(spec.lo, spec.hi)
    dev = torch.device("cuda", 0)
    f = torch.from_numpy(np.ascontiguousarray(si.f[sl])).to(dev)
    m = torch.from_numpy(np.ascontiguousarray(si.m[sl])).to(dev)
    u = torch.from_numpy(np.ascontiguousarray(si.u[sl])).to(dev)
    st = D.ShardedStep(f, m, spec, si.A, si.t, V.LossParams(kind=loss, bins=32, mi_bspline_kernel=True), margin_planes=2)
    loss_v, g_u = st.step(u)
    loss_2, g_2 = st.step(u)  # a second step reuses the window: identical
    assert loss_2 == loss_v and torch.equal(g_2, g_u)
    return loss_v, g_u.cpu().numpy(), st.window_fetches


def w_lncc(rank, world):
    return w_sharded(rank, world, "lncc")


def w_mi(rank, world):
    return w_sharded(rank, world, "mi")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_sharded_step_matches_unsharded_oracle(orc, world, loss):
    need_gpu()
    si = _inputs(loss)
    if loss == "lncc":
        ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
    else:
        ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    out = spawn(w_lncc if loss == "lncc" else w_mi, world)
    losses = [out[r][0] for r in range(world)]
    assert all(v == losses[0] for v in losses)  # the reduced loss is the same on every rank
    assert losses[0] == pytest.approx(ref["loss"], rel=1e-5)
    g = np.concatenate([out[r][1] for r in range(world)], axis=0)
    assert maxrel(g, ref["g_u"]) <= 1e-4


WU_SHAPE = (17, 20, 36)


def w_warp_update(rank, world):
    """dist.sharded_warp_update over real ranks (gloo halo exchange of g_u and of u)."""
    import torch

    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200 import voxreg as V
    rng = np.random.default_rng(77)
    g = rng.uniform(-1e-3, 1e-3, WU_SHAPE + (3,)).astype(np.float32)
    u = rng.uniform(-0.02, 0.02, WU_SHAPE + (3,)).astype(np.float32)
    spec = D.make_shard_spec(WU_SHAPE, world, rank)
    dev = torch.device("cuda", 0)
    us = torch.from_numpy(np.ascontiguousarray(u[spec.lo:spec.hi])).to(dev)
    gs = torch.from_numpy(np.ascontiguousarray(g[spec.lo:spec.hi])).to(dev)
    st = V.AdamState.zeros(us)
    out = D.sharded_warp_update(us, gs, st, spec, 0.01)
    out = D.sharded_warp_update(out, 0.5 * gs, st, spec, 0.01)
    return out.cpu().numpy(), st.m1.cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_warp_update_matches_single_gpu(world):
    """registration.hpp:313-317 on `world` ranks equals the single-GPU warp update exactly."""
    need_gpu()
    import torch

    from paper_2509_25044_b200 import voxreg as V
    rng = np.random.default_rng(77)
    g = rng.uniform(-1e-3, 1e-3, WU_SHAPE + (3,)).astype(np.float32)
    u = rng.uniform(-0.02, 0.02, WU_SHAPE + (3,)).astype(np.float32)
    ut = torch.from_numpy(u).cuda()
    gt = torch.from_numpy(g).cuda()
    st = V.AdamState.zeros(ut)
    ref = V.warp_update(ut, gt, st, 0.01)
    ref = V.warp_update(ref, 0.5 * gt, st, 0.01)
    out = spawn(w_warp_update, world)
    got = np.concatenate([out[r][0] for r in range(world)], axis=0)
    m1 = np.concatenate([out[r][1] for r in range(world)], axis=0)
    assert np.array_equal(got, ref.cpu().numpy())
    assert np.array_equal(m1, st.m1.cpu().numpy())


def w_stage(rank, world, loss):
    """dist.sharded_deformable_stage over real ranks (every rank gets the full volumes)."""
    import torch

    from oracle import Oracle, step_inputs
    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200 import registration as R
    from paper_2509_25044_b200 import voxreg as V
    si = step_inputs(Oracle(), (18, 20, 22), seed=4242, loss=loss)
    dev = torch.device("cuda", 0)
    f = torch.from_numpy(si.f.astype(np.float32)).to(dev)
    m = torch.from_numpy(si.m.astype(np.float32)).to(dev)
    sch = R.ScaleSchedule([R.ScaleStep(2, 3), R.ScaleStep(1, 3)],
                          loss=V.LossParams(kind=loss, bins=32, mi_bspline_kernel=True))
    trace = []
    w = D.sharded_deformable_stage(f, m, (si.A, si.t), sch, trace, margin_planes=2)
    return w.cpu().numpy(), [e.loss for e in trace]


def w_stage_lncc(rank, world):
    return w_stage(rank, world, "lncc")


def w_stage_mi(rank, world):
    return w_stage(rank, world, "mi")


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_sharded_deformable_stage_matches_oracle(orc, loss):
    """deformable_stage with shards = 2 (registration.hpp:230-331) against the oracle's
    single-rank stage (pinned to the reference at H = 1 and 3): same tolerances as the
    single-GPU stage (trace 1e-5; warp l2 1e-3 and a quarter of one Adam step)."""
    need_gpu()
    from gpu_util import l2rel
    from oracle import step_inputs
    from paper_2509_25044_b200 import voxreg as V
    si = step_inputs(orc, (18, 20, 22), seed=4242, loss=loss)
    w_ref, tr_ref = orc.deformable_stage(si.f, si.m, [(2, 3), (1, 3)], si.A, si.t, loss=loss, mi_kind="bspline3")
    out = spawn(w_stage_lncc if loss == "lncc" else w_stage_mi, 2)
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]
    w, tr = out[0][0], np.array(out[0][1])
    assert np.max(np.abs(tr - tr_ref) / np.abs(tr_ref)) <= 1e-5
    assert l2rel(w, w_ref) <= 1e-3
    assert np.max(np.abs(w - w_ref)) <= 0.25 * V.deformable_lr_norm(si.f.shape, 0.5)


OPS_SHAPE = (19, 22, 37)


def _ops_inputs():
    rng = np.random.default_rng(31)
    f = rng.uniform(0, 1, OPS_SHAPE).astype(np.float32)
    m = np.clip(0.7 * f + 0.3 * rng.uniform(0, 1, OPS_SHAPE), 0, 1).astype(np.float32)
    u = rng.uniform(-0.03, 0.03, OPS_SHAPE + (3,)).astype(np.float32)
    A = np.eye(3) + rng.uniform(-0.03, 0.03, (3, 3))
    t = rng.uniform(-0.03, 0.03, 3)
    up = rng.uniform(-1, 1, OPS_SHAPE).astype(np.float32)
    return f, m, u, A, t, up


def w_ops(rank, world):
    """The standalone sharded operators (distops.hpp:54-396) on real ranks."""
    import torch

    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200 import voxreg as V
    f, m, u, A, t, up = _ops_inputs()
    spec = D.make_shard_spec(OPS_SHAPE, world, rank)
    sl = slice(spec.lo, spec.hi)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a[sl])).to(dev)
    fs, ms, us, ups = T(f), T(m), T(u), T(up)
    out = {}
    moved = D.ring_sample(ms, us, A, t, OPS_SHAPE, spec)
    out["moved"] = moved.cpu().numpy()
    g = D.ring_sample_backward(ups, ms, us, A, t, OPS_SHAPE, spec,
                               V.SamplerGradWant(image=True, warp=True, affine=True, translation=True))
    out["g_img"], out["g_u"], out["gA"], out["gt"] = g.image.cpu().numpy(), g.warp.cpu().numpy(), g.affine, g.translation
    n = int(np.prod(OPS_SHAPE))
    for name, r in (("mse", D.dist_mse(fs, moved, n)),
                    ("mi", D.dist_mi(fs, moved, 32, V.ParzenKernel.bspline3(32), False, n)),
                    ("lncc_ants", D.dist_lncc(spec, fs, moved, 7, 1e-5, True, True, n)),
                    ("lncc_exact", D.dist_lncc(spec, fs, moved, 7, 1e-5, False, True, n))):
        out[name] = (r.loss, r.grad_moved.cpu().numpy())
    out["gp"] = D.gp_convolve(us, V.gaussian_taps(1.0), spec, "renormalize").cpu().numpy()
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_standalone_sharded_operators_match_single_gpu(world):
    """ring_sample / ring_sample_backward / dist_mse / dist_mi / dist_lncc (ANTs and exact)
    / gp_convolve over `world` ranks against the same operators on the whole volume on one
    GPU (the reference's invariance property, test_distops.cpp:139-423)."""
    need_gpu()
    import torch

    from gpu_util import maxrel
    from paper_2509_25044_b200 import voxreg as V
    f, m, u, A, t, up = _ops_inputs()
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    args = V.SamplerArgs(A=A, t=t)
    moved = V.fused_sample(T(m), T(u), args)
    g = V.fused_sample_backward(T(up), T(m), T(u), args,
                                V.SamplerGradWant(image=True, warp=True, affine=True, translation=True))
    out = spawn(w_ops, world)
    cat = lambda k: np.concatenate([out[r][k] for r in range(world)], axis=0)
    assert maxrel(cat("moved"), moved.cpu().numpy()) <= 1e-6
    assert maxrel(cat("g_u"), g.warp.cpu().numpy()) <= 1e-6
    assert maxrel(cat("g_img"), g.image.cpu().numpy()) <= 1e-5
    assert np.max(np.abs(out[0]["gA"] - g.affine)) <= 1e-6 * max(1.0, np.max(np.abs(g.affine)))
    assert np.max(np.abs(out[0]["gt"] - g.translation)) <= 1e-6 * max(1.0, np.max(np.abs(g.translation)))
    n = int(np.prod(f.shape))
    fm, mm = T(f), moved
    # single-GPU references of the losses on the whole moved volume
    sm = ((mm.double() - fm.double()) ** 2).sum().item() / n
    refs = {"mse": (sm, (2.0 * (mm - fm) / n).cpu().numpy())}
    k = V.ParzenKernel.bspline3(32)
    res = V.mi_forward_exact(fm, mm, 32, k)
    refs["mi"] = (-res.mi, V.mi_backward(-1.0, fm, mm, res.hist, k)[1].cpu().numpy())
    for ants in (True, False):
        lr, st = V.lncc_forward_fused(fm, mm, 7, 1e-5)
        refs["lncc_ants" if ants else "lncc_exact"] = (lr.loss, V.lncc_backward_fused(1.0, st, fm, mm, ants)[1].cpu()
                                                       .numpy())
    for name, (lv, gv) in refs.items():
        losses = [out[r][name][0] for r in range(world)]
        assert all(v == losses[0] for v in losses), name
        assert losses[0] == pytest.approx(lv, rel=1e-6), name
        assert maxrel(np.concatenate([out[r][name][1] for r in range(world)], axis=0), gv) <= 1e-5, name
    assert np.array_equal(cat("gp"), V.gp_convolve(T(u), V.gaussian_taps(1.0), "renormalize").cpu().numpy())


COMPOSED = {
    "mse": dict(kind="mse"),
    "lncc_w5": dict(kind="lncc", window=5),
    "lncc_exact": dict(kind="lncc", ants_approx=False),
    "mi_approx": dict(kind="mi", bins=32, mi_approx_forward=True),
}


def w_composed(rank, world, name):
    """ShardedStep for the losses the fused kernels do not cover: composed from
    ring_sample -> dist_mse | dist_lncc | dist_mi -> ring_sample_backward."""
    import torch

    from paper_2509_25044_b200 import dist as D
    from paper_2509_25044_b200 import voxreg as V
    si = _inputs("mi" if name.startswith("mi") else "lncc")
    spec = D.make_shard_spec(SHAPE, world, rank)
    sl = slice(spec.lo, spec.hi)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a[sl], dtype=np.float32)).to(dev)
    st = D.ShardedStep(T(si.f), T(si.m), spec, si.A, si.t, V.LossParams(**COMPOSED[name]))
    loss_v, g_u = st.step(T(si.u))
    return loss_v, g_u.cpu().numpy()


def w_composed_mse(rank, world):
    return w_composed(rank, world, "mse")


def w_composed_lncc_w5(rank, world):
    return w_composed(rank, world, "lncc_w5")


def w_composed_lncc_exact(rank, world):
    return w_composed(rank, world, "lncc_exact")


def w_composed_mi_approx(rank, world):
    return w_composed(rank, world, "mi_approx")


@pytest.mark.parametrize("name", sorted(COMPOSED))
def test_sharded_composed_losses_match_single_gpu(name):
    """every loss kind runs sharded (the reference's deformable_stage supports
    them at any shard count); the 2-rank result equals the single-GPU step."""
    need_gpu()
    import torch

    from paper_2509_25044_b200 import voxreg as V
    si = _inputs("mi" if name.startswith("mi") else "lncc")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    ref = V.warp_loss_step(T(si.f), T(si.m), T(si.u), si.A, si.t, V.LossParams(**COMPOSED[name]))
    fn = {"mse": w_composed_mse, "lncc_w5": w_composed_lncc_w5, "lncc_exact": w_composed_lncc_exact,
          "mi_approx": w_composed_mi_approx}[name]
    out = spawn(fn, 2)
    assert out[0][0] == out[1][0]
    assert out[0][0] == pytest.approx(ref.loss, rel=1e-6)
    g = np.concatenate([out[r][1] for r in range(2)], axis=0)
    assert maxrel(g, ref.g_u.cpu().numpy()) <= 1e-5
