"""Per-step MI (B-spline) accuracy of the quad and scalar paths on small lattices vs the oracle.
Run twice: FFDP_MI_QUAD_MIN=0 (quad everywhere) and =1000000000 (scalar everywhere)."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from oracle import Oracle
from gpu_util import dev, host, maxrel
from paper_2509_25044_b200 import voxreg as V
orc = Oracle()
worst = 0
for shape in [(9, 10, 11), (18, 20, 22), (12, 30, 17), (6, 40, 40)]:
    for seed in range(4):
        r = orc.rng(900 + seed)
        f = orc.random_volume(r, shape, 0.0, 1.0)
        m = np.clip(0.6 * f + 0.4 * orc.random_volume(r, shape, 0.0, 1.0), 0, 1)
        u = orc.random_volume(r, shape + (3,), -0.02, 0.02)
        f, m, u = (a.astype(np.float32).astype(np.float64) for a in (f, m, u))
        ref = orc.step_mi(f, m, u, orc.parzen("bspline3", 32))
        res = V.warp_loss_step(dev(f), dev(m), dev(u), None, None, V.LossParams(kind="mi", bins=32, mi_bspline_kernel=True))
        e = maxrel(host(res.g_u), ref["g_u"])
        worst = max(worst, e)
        print(shape, seed, f"{abs(res.loss - ref['loss']) / abs(ref['loss']):.2e} {e:.2e}")
print("worst", worst)
