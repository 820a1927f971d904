"""Small invocations of every step kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the fused LNCC step (ragged tile, TMA and LDG paths, z chunks),
the MI step (records, record-free pass 2, fused finalize), the native plan over an
in-process group of 2 ranks, the warp update. Run under
    compute-sanitizer --tool <tool> python tools/sanitize_run.py"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import Oracle, step_inputs  # noqa: E402
from paper_2509_25044_b200 import plan as PL  # noqa: E402
from paper_2509_25044_b200 import voxreg as V  # noqa: E402


def d(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).cuda()


def main():
    torch.cuda.set_device(0)
    orc = Oracle()
    for shape in ((21, 37, 44), (40, 36, 32)):
        for loss in ("lncc", "mi"):
            si = step_inputs(orc, shape, seed=3, loss=loss)
            p = V.LossParams(kind="lncc") if loss == "lncc" else V.LossParams(kind="mi", bins=32,
                                                                                mi_bspline_kernel=True)
            r = V.warp_loss_step(d(si.f), d(si.m), d(si.u), si.A, si.t, p)
            torch.cuda.synchronize()
            print(shape, loss, r.loss, flush=True)
    # MI quad path (>= 2^16 voxels) with and without records
    si = step_inputs(orc, (48, 44, 40), seed=5, loss="mi")
    p = V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True)
    r = V.warp_loss_step(d(si.f), d(si.m), d(si.u), si.A, si.t, p)
    torch.cuda.synchronize()
    print("mi quad", r.loss, flush=True)
    # the native plan, two ranks in one process
    for loss, p in (("lncc", V.LossParams(kind="lncc")), ("mi", V.LossParams(kind="mi", bins=32,
                                                                             mi_bspline_kernel=True))):
        si = step_inputs(orc, (44, 30, 28), seed=9, loss=loss)
        groups = PL.local_group(2, [0, 0])
        out = [None, None]

        def rank(r):
            torch.cuda.set_device(0)
            pl = PL.ShardPlan(groups[r], si.f.shape, p, si.A, si.t)
            pl.load(d(si.f)[pl.lo:pl.hi], d(si.m)[pl.lo:pl.hi])
            pl.set_u(d(si.u)[pl.lo:pl.hi])
            out[r] = pl.step()
            pl.close()

        th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for g in groups:
            g.close()
        print("plan", loss, out, flush=True)
    # warp update kernels
    g = torch.randn((20, 24, 28, 3), device="cuda") * 1e-3
    u = torch.zeros_like(g)
    st = V.AdamState.zeros(u)
    V.warp_update(u, g, st, 0.01)
    torch.cuda.synchronize()
    print("warp update ok", flush=True)


if __name__ == "__main__":
    main()
