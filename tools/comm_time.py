"""Time repeated fused sharded steps through ffdp_comm (ranks sharing GPU 0)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2509_25044_b200 import voxreg as V
from paper_2509_25044_b200.comm import Comm
for loss in ("mi", "lncc"):
    shape = (256, 256, 256) if loss == "mi" else (320, 320, 320)
    f, m, u, A, t = bench.synth_inputs(shape, loss, 1234, "cuda")
    p = V.LossParams(kind=loss, mi_bspline_kernel=True)
    for world in (1, 2):
        with Comm(world, [0] * world) as c:
            fs, ms, us = c.scatter(f), c.scatter(m), c.scatter(u)
            c.step(fs, ms, us, tuple(f.shape), A, t, p)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                c.step(fs, ms, us, tuple(f.shape), A, t, p)
            torch.cuda.synchronize()
            print(os.environ.get("FFDP_LIB", "in-tree").split("/")[-1], loss, world, round((time.perf_counter() - t0) / 5 * 1e3, 2), "ms/step", flush=True)
