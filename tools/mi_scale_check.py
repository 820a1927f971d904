"""MI step accuracy vs the oracle at a few lattice sizes (the library is FFDP_LIB)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from oracle import step_inputs
from paper_2509_25044_b200 import voxreg as V
orc = oracle.Oracle()
for shape in ((48, 52, 56), (64, 64, 64), (96, 96, 96)):
    si = step_inputs(orc, shape, seed=4242, loss="mi")
    ref = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    r = V.warp_loss_step(T(si.f), T(si.m), T(si.u), si.A, si.t, V.LossParams(kind="mi", mi_bspline_kernel=True))
    g = r.g_u.cpu().numpy().astype(np.float64)
    print(os.environ.get("FFDP_LIB", "in-tree").split("/")[-1], shape, "loss rel %.2e" % abs(r.loss / ref["loss"] - 1),
          "g maxrel %.2e" % (np.max(np.abs(g - ref["g_u"])) / np.max(np.abs(ref["g_u"]))), flush=True)
