"""Pass-1 time with the finalize fused into its last CTA vs pass 1 alone (256^3 MI)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2509_25044_b200 import voxreg as V
from paper_2509_25044_b200._lib import lib
f, m, u, A, t = bench.synth_inputs((256, 256, 256), "mi", 1234, "cuda")
mi = V.MovingImage(m)
k = V.ParzenKernel.bspline3(32)
ws = V.StepWorkspace(f.device, 32)
args = V.SamplerArgs(A=A, t=t).to_c()
dims, slab = V._dims(f.shape), V._full_slab(f.shape[0])
rec = ws.records(dims, slab)
s = V._stream()
def run(fused):
    ws.raw.zero_()
    if fused:
        lib.ffdp_step_mi_hist_final(V._ptr(f), V._ptr(u), dims, slab, mi.window(), C.byref(args), C.byref(k.c),
                                    V._ptr(ws.raw), -1.0, V._ptr(ws.table), V._ptr(ws.scratch), V._ptr(rec), None, s)
    else:
        lib.ffdp_step_mi_hist_rec(V._ptr(f), V._ptr(u), dims, slab, mi.window(), C.byref(args), C.byref(k.c),
                                  V._ptr(ws.raw), V._ptr(ws.scratch), V._ptr(rec), None, s)
for fused in (True, False, True, False):
    for _ in range(5): run(fused)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): run(fused)
    e1.record(); torch.cuda.synchronize()
    print("fused" if fused else "plain", round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us (incl. raw zeroing)")
