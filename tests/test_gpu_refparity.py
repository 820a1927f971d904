"""The CUDA step against the REFERENCE ITSELF at BASELINE configs[0] (128^3).

`oracle.Reference.step` runs the reference's own deformable-step sequence
(ring_sample -> dist_lncc | dist_mi -> ring_sample_backward(want warp),
registration.hpp:277-312, distops.hpp:144-396) from the unmodified headers
(oracle/_ref/libvoxreg_ref.so, built by oracle/Makefile), in T=double on the same
fp32-rounded inputs, with one worker and with a sharded WorkerGroup. Gates (north star):
|dloss|/|loss| <= 1e-5, max|dg_u|/max|g_u| <= 1e-4."""
import os

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
def ref():
    from oracle import Reference
    try:
        return Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")


def _case(orc, loss, shape=(128, 128, 128)):
    from oracle import step_inputs
    return step_inputs(orc, shape, seed=4242, loss=loss)


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_step_matches_reference_128(V, orc, ref, loss):
    si = _case(orc, loss)
    params = V.LossParams(kind="lncc") if loss == "lncc" else V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True)
    res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, params)
    assert res.window_misses == 0
    gu = host(res.g_u)
    worlds = [1, min(8, os.cpu_count() or 1)]
    for world in worlds:
        r = ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=world)
        lrel = abs(res.loss - r["loss"]) / abs(r["loss"])
        grel = maxrel(gu, r["g_u"])
        print(f"{loss} 128^3 vs reference (T=double, H={world}): loss {res.loss:.10f} ref {r['loss']:.10f} "
              f"rel {lrel:.2e}; g_u maxrel {grel:.2e} l2rel {l2rel(gu, r['g_u']):.2e}")
        assert lrel <= LOSS_RTOL
        assert grel <= GRAD_MAXREL


def test_sharded_step_matches_reference_96(V, orc, ref):
    """The z-slab sharded step (emulated ranks on one GPU, ffdp_comm) against the
    reference's sharded WorkerGroup run of the same world size."""
    import torch
    from paper_2509_25044_b200.comm import Comm
    for loss in ("lncc", "mi"):
        si = _case(orc, loss, (96, 80, 88))
        f, m, u = dev(si.f), dev(si.m), dev(si.u)
        p = V.LossParams(kind=loss, bins=32, mi_bspline_kernel=True)
        for world in (2, 3):
            r = ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=world)
            with Comm(world, [0] * world) as c:
                lv, g = c.step(c.scatter(f), c.scatter(m), c.scatter(u), tuple(f.shape), si.A, si.t, p)
            gu = torch.cat([x.cpu() for x in g], 0).double().numpy()
            lrel = abs(lv - r["loss"]) / abs(r["loss"])
            grel = maxrel(gu, r["g_u"])
            print(f"sharded {loss} H={world} vs reference H={world}: loss rel {lrel:.2e} g_u maxrel {grel:.2e}")
            assert lrel <= LOSS_RTOL and grel <= GRAD_MAXREL
