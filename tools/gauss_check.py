import sys, os; sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import Oracle, step_inputs
from gpu_util import dev, host, maxrel
from paper_2509_25044_b200 import voxreg as V
orc = Oracle()
for shape in [(18, 20, 22), (9, 10, 11), (32, 28, 24)]:
    si = step_inputs(orc, shape, seed=4242, loss="mi")
    for kind in ("gaussian", "bspline3"):
        ref = orc.step_mi(si.f, si.m, si.u, orc.parzen(kind, 32), si.A, si.t)
        res = V.warp_loss_step(dev(si.f), dev(si.m), dev(si.u), si.A, si.t, V.LossParams(kind="mi", bins=32, mi_bspline_kernel=kind == "bspline3"))
        print(shape, kind, abs(res.loss - ref["loss"]) / abs(ref["loss"]), maxrel(host(res.g_u), ref["g_u"]))
        # the operator path
        mw = dev(ref["moved"])
        k = V.ParzenKernel.bspline3(32) if kind == "bspline3" else V.ParzenKernel.gaussian(32)
        r2 = V.mi_forward_exact(dev(si.f), mw, 32, k)
        print("   op mi", r2.mi if hasattr(r2, "mi") else r2)
