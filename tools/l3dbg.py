import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import Oracle, step_inputs
from paper_2509_25044_b200 import voxreg
orc = Oracle()
si = step_inputs(orc, (24, 28, 32), seed=7, loss="lncc")
d = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).cuda()
ref = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
res = voxreg.warp_loss_step(d(si.f), d(si.m), d(si.u), si.A, si.t, voxreg.LossParams(kind="lncc"))
gu = res.g_u.double().cpu().numpy()
print("loss", res.loss, ref["loss"], "g maxrel", np.max(np.abs(gu - ref["g_u"])) / np.max(np.abs(ref["g_u"])))
