"""The native sharded step plan (include/ffdp.h ffdp_plan_*, csrc/plan.cu) on one GPU.

Ranks of an in-process group (one host thread each, sharing cuda:0) run the whole
deformable step -- u halo exchange, fused kernels on their slabs, allreduce of sum n_i /
the integer joint histogram -- and the gathered g_u / global loss are compared with the
single-GPU step (the reference's shard-invariance tests, test_distops.cpp:161-187,
243-289, 369-423) and with the fp64 oracle. The NCCL transport runs at world 1 here (one
device) and at world 2 when the box has two devices."""
import threading

import numpy as np
import pytest

from gpu_util import dev, host, maxrel, need_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    need_gpu()
    from paper_2509_25044_b200 import voxreg
    return voxreg


@pytest.fixture(scope="module")
def PL():
    need_gpu()
    from paper_2509_25044_b200 import plan
    return plan


def params_for(V, loss):
    if loss == "lncc":
        return V.LossParams(kind="lncc")
    return V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True)


def run_ranks(groups, fn):
    """fn(group) on one thread per rank; re-raises the first failure."""
    out, err = [None] * len(groups), []

    def body(i, g):
        import torch
        try:
            torch.cuda.set_device(g.device)
            out[i] = fn(g)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(i, g)) for i, g in enumerate(groups)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def plan_step(PL, V, groups, si, loss, steps=1, records=True, overlap=True, margin=8, u=None):
    """Every rank: plan, load its slabs, set u, `steps` steps; returns [(loss, g_u, lo, hi, window)]."""
    import torch
    shape = si.f.shape
    A, t = si.A, si.t
    u = si.u if u is None else u

    def rank(g):
        p = PL.ShardPlan(g, shape, params_for(V, loss), A, t, margin_planes=margin, records=records,
                         overlap=overlap)
        try:
            p.load(dev(si.f)[p.lo:p.hi], dev(si.m)[p.lo:p.hi])
            p.set_u(dev(u)[p.lo:p.hi])
            lv = None
            for _ in range(steps):
                lv = p.step()
            torch.cuda.synchronize()
            return lv, host(p.g_u.clone()), p.lo, p.hi, p.window()
        finally:
            p.close()

    return run_ranks(groups, rank)


def single(V, si, loss, u=None):
    r = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u if u is None else u), si.A, si.t, params_for(V, loss))
    return r.loss, host(r.g_u)


@pytest.fixture(scope="module")
def cases(orc):
    from oracle import step_inputs
    # MI above 2^16 voxels: the single-GPU step then takes the same quad kernels and 2^-23
    # fixed-point grid as the plan (smaller lattices use the scalar kernels)
    return {"lncc": step_inputs(orc, (29, 26, 24), seed=515, loss="lncc"),
            "mi": step_inputs(orc, (44, 42, 40), seed=515, loss="mi")}


@pytest.mark.parametrize("loss", ["lncc", "mi"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_local_group_matches_single_gpu(V, PL, cases, loss, world):
    si = cases[loss]
    groups = PL.local_group(world, [0] * world)
    try:
        res = plan_step(PL, V, groups, si, loss)
    finally:
        for g in groups:
            g.close()
    l1, g1 = single(V, si, loss)
    gu = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
    assert all(r[0] == res[0][0] for r in res), "every rank reports the same global loss"
    lrel = abs(res[0][0] - l1) / abs(l1)
    grel = maxrel(gu, g1)
    print(f"plan {loss} H={world}: loss rel {lrel:.2e}, g_u maxrel {grel:.2e}")
    # integer window sums (LNCC) / the integer joint histogram on the single-GPU grid (MI):
    # the sharded gradient is the single-GPU gradient up to the finalize's fp64 order
    assert lrel <= 1e-9
    assert grel <= 1e-6


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_local_group_bit_identical_across_world_sizes(V, PL, cases, loss):
    si = cases[loss]
    out = {}
    for world in (1, 2, 4):
        groups = PL.local_group(world, [0] * world)
        try:
            res = plan_step(PL, V, groups, si, loss, steps=2)
        finally:
            for g in groups:
                g.close()
        out[world] = (res[0][0], np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0))
    for world in (2, 4):
        assert np.array_equal(out[world][1], out[1][1]), f"g_u at H={world} differs from H=1"
        if loss == "mi":
            assert out[world][0] == out[1][0]
        else:
            assert abs(out[world][0] - out[1][0]) <= 1e-12


def test_plan_matches_oracle(V, PL, orc, cases):
    """The plan at H = 2 against the fp64 oracle step (loss 1e-5, g_u 1e-4: north star)."""
    for loss in ("lncc", "mi"):
        si = cases[loss]
        if loss == "lncc":
            ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
        else:
            ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
        groups = PL.local_group(2, [0, 0])
        try:
            res = plan_step(PL, V, groups, si, loss)
        finally:
            for g in groups:
                g.close()
        gu = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
        lrel = abs(res[0][0] - ref["loss"]) / abs(ref["loss"])
        grel = maxrel(gu, ref["g_u"])
        print(f"plan {loss} H=2 vs oracle: loss rel {lrel:.2e}, g_u maxrel {grel:.2e}")
        assert lrel <= 1e-5 and grel <= 1e-4


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_window_miss_widens_and_stays_exact(V, PL, cases, loss):
    """No margin and a displacement of +0.3 (normalized, ~4 planes) along z: the affine
    window misses the displaced samples, the summed miss count makes the ranks widen their
    windows from the z extent of their samples and repeat the step."""
    si = cases[loss]
    u = np.array(si.u, dtype=np.float64)
    u[..., 2] += 0.3
    groups = PL.local_group(3, [0, 0, 0])
    try:
        res = plan_step(PL, V, groups, si, loss, margin=0, u=u)
    finally:
        for g in groups:
            g.close()
    gu = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
    l1, g1 = single(V, si, loss, u=u)
    fetches = [r[4][2] for r in res]
    print(f"plan {loss} margin 0: window fetches per rank {fetches}")
    assert max(fetches) > 1, "the displaced samples should have missed the affine window"
    assert abs(res[0][0] - l1) / abs(l1) <= 1e-9
    assert maxrel(gu, g1) <= 1e-6


def test_records_and_overlap_variants(V, PL, cases):
    """MI with and without pass-1 records, LNCC with and without the overlapped halo
    exchange: identical gradients (the split is a launch boundary, the sums are exact)."""
    import torch  # noqa: F401
    for loss, kw in (("mi", "records"), ("lncc", "overlap")):
        si = cases[loss]
        res = {}
        for flag in (True, False):
            groups = PL.local_group(2, [0, 0])
            try:
                r = plan_step(PL, V, groups, si, loss, **{kw: flag})
            finally:
                for g in groups:
                    g.close()
            res[flag] = np.concatenate([x[1] for x in sorted(r, key=lambda x: x[2])], axis=0)
        assert np.array_equal(res[True], res[False]), kw


def test_overlap_split_on_thick_slabs(V, PL, orc):
    """Slabs thick enough for the interior / boundary split (> 2 x 16 + 8 planes)."""
    from oracle import step_inputs
    si = step_inputs(orc, (100, 20, 24), seed=77, loss="lncc")
    out = {}
    for overlap in (True, False):
        groups = PL.local_group(2, [0, 0])
        try:
            r = plan_step(PL, V, groups, si, "lncc", overlap=overlap)
        finally:
            for g in groups:
                g.close()
        out[overlap] = (r[0][0], np.concatenate([x[1] for x in sorted(r, key=lambda x: x[2])], axis=0))
    l1, g1 = single(V, si, "lncc")
    assert np.array_equal(out[True][1], out[False][1])
    assert maxrel(out[True][1], g1) <= 1e-6
    assert abs(out[True][0] - l1) / abs(l1) <= 1e-9


def test_nccl_world1_matches_local(V, PL, cases):
    try:
        PL.nccl_version()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"NCCL not loadable: {e}")
    for loss in ("lncc", "mi"):
        si = cases[loss]
        g = PL.nccl_group(PL.nccl_unique_id(), 1, 0, 0)
        try:
            rn = plan_step(PL, V, [g], si, loss)
        finally:
            g.close()
        gl = PL.local_group(1, [0])
        try:
            rl = plan_step(PL, V, gl, si, loss)
        finally:
            gl[0].close()
        assert rn[0][0] == rl[0][0]
        assert np.array_equal(rn[0][1], rl[0][1])


def test_nccl_world2_two_devices(V, PL, cases):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two devices")
    uid = PL.nccl_unique_id()
    for loss in ("lncc", "mi"):
        si = cases[loss]
        holder = {}

        def mk(r):
            torch.cuda.set_device(r)
            holder[r] = PL.nccl_group(uid, 2, r, r)

        th = [threading.Thread(target=mk, args=(r,)) for r in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        groups = [holder[0], holder[1]]
        try:
            res = plan_step(PL, V, groups, si, loss)
        finally:
            for g in groups:
                g.close()
        l1, g1 = single(V, si, loss)
        gu = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
        assert abs(res[0][0] - l1) / abs(l1) <= 1e-9 and maxrel(gu, g1) <= 1e-6
        uid = PL.nccl_unique_id()


def test_plan_argument_errors(V, PL):
    from paper_2509_25044_b200._lib import InvalidArgument, LogicError
    g = PL.local_group(1, [0])[0]
    try:
        with pytest.raises(InvalidArgument):
            PL.ShardPlan(g, (16, 16, 16), V.LossParams(kind="lncc", window=5))
        with pytest.raises(InvalidArgument):
            PL.ShardPlan(g, (16, 16, 16), V.LossParams(kind="mi", bins=32, mi_bspline_kernel=False))
        p = PL.ShardPlan(g, (16, 16, 16), V.LossParams(kind="lncc"))
        with pytest.raises(LogicError):
            p.step()
        p.close()
    finally:
        g.close()


def test_first_use_from_many_threads_in_a_fresh_process():
    """Kernel attributes are set lazily per device on first use: 4 rank threads reaching the
    same launch sites at once in a fresh process must all launch after the setup (a race
    here failed with 'invalid argument' on the > 48 KB shared-memory kernels)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, threading, numpy as np, torch; sys.path.insert(0, %r)\n"
        "from oracle import Oracle, step_inputs\n"
        "from paper_2509_25044_b200 import plan as PL, voxreg as V\n"
        "orc = Oracle()\n"
        "for loss in ('mi', 'lncc'):\n"
        "    si = step_inputs(orc, (64, 40, 36), seed=11, loss=loss)\n"
        "    p = V.LossParams(kind=loss, bins=32, mi_bspline_kernel=True)\n"
        "    d = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).cuda()\n"
        "    gs = PL.local_group(4, [0] * 4); out = [None] * 4; err = []\n"
        "    def rank(r):\n"
        "        try:\n"
        "            torch.cuda.set_device(0)\n"
        "            pl = PL.ShardPlan(gs[r], si.f.shape, p, si.A, si.t)\n"
        "            pl.load(d(si.f)[pl.lo:pl.hi], d(si.m)[pl.lo:pl.hi]); pl.set_u(d(si.u)[pl.lo:pl.hi])\n"
        "            out[r] = pl.step(); pl.close()\n"
        "        except Exception as e:\n"
        "            err.append(repr(e)); import os; os._exit(3)\n"
        "    th = [threading.Thread(target=rank, args=(r,)) for r in range(4)]\n"
        "    [t.start() for t in th]; [t.join() for t in th]\n"
        "    assert len(set(out)) == 1, out\n"
        "print('ok')\n") % root
    for _ in range(3):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_thin_slabs_rotation_and_translation(V, PL, orc, loss):
    """Five ranks on 21 planes (slabs of 4-5 planes, halos of 3 from thin neighbours), a
    rotated / scaled affine with a z translation (every rank's moving window differs from
    its slab), ragged x / y (62 x 57): the plan equals the single-GPU step."""
    from oracle import step_inputs
    # > 2^16 voxels: the single-GPU MI step then uses the quad kernels and grid the plan uses
    si = step_inputs(orc, (21, 62, 57), seed=29, loss=loss)
    th = 0.12
    A = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.05], [0.02, -0.03, 0.97]])
    t = np.array([0.01, -0.02, 0.08])
    import copy
    si = copy.copy(si)
    si.A, si.t = A, t
    groups = PL.local_group(5, [0] * 5)
    try:
        res = plan_step(PL, V, groups, si, loss, margin=2)
    finally:
        for g in groups:
            g.close()
    gu = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
    l1, g1 = single(V, si, loss)
    print(f"plan {loss} H=5 thin slabs: windows {[r[4] for r in res]}")
    assert abs(res[0][0] - l1) / abs(l1) <= 1e-9
    assert maxrel(gu, g1) <= 1e-6


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_plan_iterations_with_warp_update(V, PL, cases, loss):
    """Three deformable iterations on the plan (step, then ffdp_plan_warp_update: halo'd
    Sobolev smoothing fused with Adam, halo'd warp smoothing; registration.hpp:277-317) at
    1-3 ranks against the single-GPU iteration (warp_loss_step + warp_update): the loss trace
    and the final warp agree bit for bit."""
    import torch
    si = cases[loss]
    shape = si.f.shape
    lr = V.deformable_lr_norm(shape, 0.5)
    # single GPU
    u = dev(si.u)
    st = V.AdamState.zeros(u)
    trace1 = []
    for _ in range(3):
        r = V.warp_loss_step(dev(si.f), dev(si.m), u, si.A, si.t, params_for(V, loss))
        trace1.append(r.loss)
        u = V.warp_update(u, r.g_u, st, lr)
    u1 = host(u)
    for world in (1, 2, 3):
        groups = PL.local_group(world, [0] * world)

        def rank(g):
            torch.cuda.set_device(0)
            p = PL.ShardPlan(g, shape, params_for(V, loss), si.A, si.t, warp_halo=3)
            try:
                p.load(dev(si.f)[p.lo:p.hi], dev(si.m)[p.lo:p.hi])
                p.set_u(dev(si.u)[p.lo:p.hi])
                tr = []
                for _ in range(3):
                    tr.append(p.step())
                    p.warp_update(lr)
                torch.cuda.synchronize()
                return tr, host(p.u.clone()), p.lo
            finally:
                p.close()

        try:
            res = run_ranks(groups, rank)
        finally:
            for g in groups:
                g.close()
        un = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[2])], axis=0)
        tr = res[0][0]
        print(f"plan {loss} H={world} 3 iterations: trace {tr} vs {trace1}; "
              f"warp maxrel {maxrel(un, u1):.2e}")
        if loss == "mi":
            assert tr == trace1
        else:
            assert max(abs(a - b) for a, b in zip(tr, trace1)) <= 1e-12
        assert np.array_equal(un, u1)
