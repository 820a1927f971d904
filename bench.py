#!/usr/bin/env python
"""Benchmark of the fused warp + loss forward+backward step (the FFDP hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload auto|mi1760|lncc720|mi256|lncc128|lncc1024] [--jitter bench|survey]
                    [--no-secondary] [--no-cpu]

Metric (BASELINE.json): Gvoxel/s of the fused warp+loss fwd+bwd step, voxel = output
(fixed-lattice) voxel; one step = read F, M, u -> Mw -> loss -> dL/dMw -> g_u
(registration.hpp:277-312). The N = 1 headline (--workload auto) is the largest
single-GPU configuration: BASELINE configs[4], a 1760x1760x1200 (3.7 G-voxel) multimodal
pair, warp + Mattes MI (32 bins, B-spline Parzen), when it fits the GPU, else configs[2]
(720x640x720 LNCC, window 7, ANTs). Secondary lines: configs[2] and configs[1] (256^3 MI),
each with the bench's sub-voxel u jitter and with SURVEY 8(d)'s U(-0.01, 0.01)-normalized
jitter, each with its roofline and CPU baseline; the warp update; the configs[2]
multi-scale registration. Every input set exceeds the 126 MB L2, so no flush is needed
between steps. Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (shape (nz, ny, nx), loss, BASELINE config index)
    "mi256": ((256, 256, 256), "mi", 1),
    "lncc720": ((720, 640, 720), "lncc", 2),
    "lncc128": ((128, 128, 128), "lncc", 0),
    "lncc1024": ((1024, 1024, 1024), "lncc", 3),
    "mi1760": ((1200, 1760, 1760), "mi", 4),
}
BYTES_PER_VOXEL = {"lncc": 32, "mi": 52}
DTYPE = {"lncc": "f32 (fp64 coordinates; exact int32 box sums of 2^-21 fixed-point moments)",
         "mi": "f32 (fp64 coordinates; integer fixed-point histogram)"}  # algorithmic bytes per output voxel
METRIC = "Gvoxel/s of fused warp+loss fwd+bwd step (1–8 B200), % of HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel, nvox):
    """roofline.traffic: dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed --set full capture (profiles/traffic.json, tools/profile_summary.py),
    scaled to this launch's voxel count; None when no capture of this kernel exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)[kernel]
        return round(t["bytes_per_voxel"] * nvox), (f"{t['bytes_per_voxel']} B/voxel from profiles/"
                                                     f"{t['round']}_full_*.txt ({t['workload']})")
    except Exception:
        return None, "no ncu capture"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ synthetic inputs
def synth_inputs(shape, loss, seed, device, z0=0, z1=None, reduce_minmax=None, jitter="bench", chunk=32,
                 fine=None):
    """Synthetic pair of the survey's recipe on the GPU, analytic in the
    global normalized frame so any z slab [z0, z1) of the global `shape` is generated
    locally and consistently across ranks: smooth ellipsoidal structures with texture,
    M = F pushed through a smooth warp, u = smooth field + sub-voxel jitter,
    A = I + U(-0.02, 0.02), t = U(-0.02, 0.02). MI: M = normalize(4 m (1 - m) + noise).
    reduce_minmax(lo, hi) -> (lo, hi) makes the intensity normalisation global.
    jitter: "bench" adds U(-0.01, 0.01) voxel to u; "survey" adds SURVEY 8(d)'s
    U(-0.01, 0.01) in normalized units (+-0.5 (n-1) / 100 voxels: +-3.6 at 720).
    The outputs are allocated first and filled `chunk` planes at a time (the noise streams
    are seeded per chunk), so no volume-sized temporary fragments the device memory: at
    configs[4] (119 GB of F, M, u, g_u) the step's 16 B/voxel records must still fit.
    fine = (wavelength in voxels, amplitude, true-warp amplitude): adds a texture at the LNCC
    window's scale and sets the true deformation's amplitude (the registration demo: the
    smooth pair alone leaves every 7^3 window nearly constant, so LNCC is epsilon-dominated)."""
    import numpy as np
    import torch

    g = torch.Generator(device="cpu").manual_seed(seed)
    rnd = lambda *s: torch.rand(*s, generator=g, dtype=torch.float64)
    nz, ny, nx = shape
    z1 = nz if z1 is None else z1
    lshape = (z1 - z0, ny, nx)
    ax = lambda n: torch.linspace(-1.0, 1.0, n, device=device, dtype=torch.float32)
    zax, y, x = ax(nz), ax(ny).view(1, ny, 1), ax(nx).view(1, 1, nx)
    blobs = [((rnd(3) * 1.2 - 0.6).tolist(), (rnd(3) * 0.3 + 0.2).tolist(), float(rnd(1) * 0.7 + 0.3))
             for _ in range(6)]
    tex = [((rnd(3) * 12 + 4).tolist(), (rnd(3) * 6.28).tolist()) for _ in range(3)]

    def modes(amp):
        return [[((rnd(3) * 3 + 0.5).tolist(), (rnd(3) * 6.28).tolist(), float(rnd(1) * 2 - 1) * amp)
                 for _ in range(3)] for _ in range(3)]

    modes_true, modes_u = modes(0.04 if fine is None else fine[2]), modes(0.02)
    aff = rnd(12).numpy() * 0.04 - 0.02
    # fine texture: k_a = pi (n_a - 1) / wavelength rad per normalized unit
    kf = None if fine is None else [math.pi * (n - 1) / fine[0] for n in (nx, ny, nz)]

    def f_at(X, Y, Z):
        out = torch.zeros(torch.broadcast_shapes(X.shape, Y.shape, Z.shape), dtype=torch.float32, device=device)
        for c, r, inten in blobs:
            out += inten * torch.sigmoid((1.0 - (((X - c[0]) / r[0]) ** 2 + ((Y - c[1]) / r[1]) ** 2 +
                                                 ((Z - c[2]) / r[2]) ** 2)) * 10.0)
        for k, ph in tex:
            out += 0.04 * torch.sin(k[0] * X + ph[0]) * torch.sin(k[1] * Y + ph[1]) * torch.sin(k[2] * Z + ph[2])
        if kf is not None:
            out += fine[1] * torch.sin(kf[0] * X + 0.3) * torch.sin(kf[1] * Y + 1.1) * torch.sin(kf[2] * Z + 0.7)
        return out

    def field(md, z, out):
        for cpt in range(3):
            acc = out[..., cpt]
            acc.zero_()
            for k, ph, a in md[cpt]:
                acc += a * torch.sin(k[0] * x + ph[0]) * torch.sin(k[1] * y + ph[1]) * torch.sin(k[2] * z + ph[2])

    def normalize_(v):
        lo, hi = float(v.min()), float(v.max())
        if reduce_minmax is not None:
            lo, hi = reduce_minmax(lo, hi)
        v.sub_(lo).div_(hi - lo).clamp_(0.0, 1.0)

    if jitter == "survey":
        jit = torch.tensor([0.02, 0.02, 0.02], device=device)
    else:
        # sub-voxel jitter (+-0.01 voxel) keeps samples off cell faces; a registration warp
        # is smooth (it is Gaussian-smoothed every iteration, registration.hpp:316)
        jit = torch.tensor([0.04 / (nx - 1), 0.04 / (ny - 1), 0.04 / (nz - 1)], device=device)
    f = torch.empty(lshape, dtype=torch.float32, device=device)
    m = torch.empty(lshape, dtype=torch.float32, device=device)
    u = torch.empty(lshape + (3,), dtype=torch.float32, device=device)
    ut = torch.empty((min(chunk, lshape[0]), ny, nx, 3), dtype=torch.float32, device=device)
    for c0 in range(0, lshape[0], chunk):
        c1 = min(lshape[0], c0 + chunk)
        z = zax[z0 + c0:z0 + c1].view(-1, 1, 1)
        f[c0:c1] = f_at(x, y, z)
        t3 = ut[:c1 - c0]
        field(modes_true, z, t3)
        m[c0:c1] = f_at(x + t3[..., 0], y + t3[..., 1], z + t3[..., 2])
        field(modes_u, z, u[c0:c1])
        gj = torch.Generator(device=device).manual_seed(seed + 2 + z0 + c0)
        u[c0:c1] += (torch.rand((c1 - c0, ny, nx, 3), generator=gj, device=device) - 0.5) * jit
    del ut
    normalize_(f)
    normalize_(m)
    if loss == "mi":
        for c0 in range(0, lshape[0], chunk):
            c1 = min(lshape[0], c0 + chunk)
            gn = torch.Generator(device=device).manual_seed(seed + 1 + z0 + c0)
            mc = m[c0:c1]
            mc.copy_(4.0 * mc * (1.0 - mc) + 0.02 * torch.randn((c1 - c0, ny, nx), generator=gn, device=device))
        normalize_(m)
    A = np.eye(3) + aff[:9].reshape(3, 3)
    t = aff[9:]
    if torch.device(device).type == "cuda":
        torch.cuda.synchronize()
    return f, m, u, A, t


# ------------------------------------------------------------------ the GPU arm
class Stepper:
    """Launches one fused step through the C ABI on the current stream, recording CUDA
    events around each of our kernels so per-kernel device time is measured live."""

    def __init__(self, f, m, u, A, t, loss, bins=32):
        import ctypes as C

        import torch

        from paper_2509_25044_b200 import voxreg
        from paper_2509_25044_b200._lib import lib

        self.C, self.torch, self.V, self.lib = C, torch, voxreg, lib
        self.f, self.u, self.loss = f, u, loss
        self.n = f.numel()
        self.g_u = torch.empty_like(u)
        self.args = voxreg.SamplerArgs(A=A, t=t).to_c()
        self.ws = voxreg.StepWorkspace(f.device, bins)
        self.bins = bins
        self.slab = voxreg._full_slab(f.shape[0])
        self.mimg = voxreg.MovingImage(m)  # zero-bordered layout, made once per scale
        torch.cuda.synchronize()
        self.win = self.mimg.window()
        self.dims = voxreg._dims(f.shape)
        if loss == "lncc":
            # the one-pass fused step (default) or the round-1 two-pass form (comparison)
            self.twopass = os.environ.get("FFDP_LNCC_IMPL") == "twopass"
            if self.twopass:
                self.shifts = (voxreg.intensity_shift(f), voxreg.intensity_shift(self.mimg.interior.contiguous()))
                n = int(lib.ffdp_step_lncc_passes_workspace_bytes(self.dims, self.slab)) // 4
                self._lws_t = torch.empty(n, dtype=torch.float32, device=f.device)
                self._lws = self._p(self._lws_t)
            else:
                # the bordered copy: its zeros do not move the frame (it always spans 0, step_lncc3.cu)
                self.ranges = voxreg.intensity_ranges(f, self.mimg.padded)
                self._lws = self._p(self.ws.lncc_workspace(self.dims, self.slab))
        else:
            self.kernel = voxreg.ParzenKernel.bspline3(bins)
            self.choose_records()
        self.kernel_ms = {}
        # lncc: sample, moments, partial-sum reduction (fused: 1); mi: pass 1 (finalize fused
        # into its last CTA) and pass 2 (memsets of the histogram are not kernels of ours)
        self.launches_per_step = ((3 if self.twopass else 2) if loss == "lncc" else
                                  2 if self.use_rec else 4)

    def choose_records(self):
        """MI: the pass-1 records (16 B/voxel) when they fit next to the step's buffers
        with 4 GiB to spare; else pass 2 samples the warp again (ffdp_step_mi without
        records). Re-evaluated once the caller has released its own copy of M."""
        if self.loss != "mi":
            return
        free, _ = self.torch.cuda.mem_get_info()
        need = 16 * self.n + (4 << 30)
        # FFDP_BENCH_NOREC=1 forces the record-free pass 2 (A/B measurements)
        self.use_rec = free > need and os.environ.get("FFDP_BENCH_NOREC") != "1"
        self.launches_per_step = 2 if self.use_rec else 4
        self.records_note = {"used": self.use_rec, "device_free_bytes": int(free), "needed_bytes": int(need),
                             "torch_reserved_bytes": int(self.torch.cuda.memory_reserved())}

    def _p(self, t):
        return self.C.c_void_p(t.data_ptr())

    def step(self, record=False):
        """One step on the current stream. record=True brackets each of our kernels with
        CUDA events (per-kernel device time, live); record=False is launch-only and is
        what the CUDA graph captures."""
        torch, C, lib = self.torch, self.C, self.lib
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
        if self.loss == "lncc":
            self.ws.sum_n.zero_()
            if not self.twopass:
                if record:
                    ev[0].record()
                lib.ffdp_step_lncc(self._p(self.f), self._p(self.u), self.dims, self.slab, self.win, C.byref(self.args),
                                   7, 1e-5, -1.0 / self.n, self._p(self.ranges), self._p(self.g_u),
                                   self._p(self.ws.sum_n), None, self._lws, s)
                if not record:
                    return None
                ev[1].record()
                return [("k_lncc_fused", ev[0], ev[1])]
            a = (self._p(self.f), self._p(self.u), self.dims, self.slab, self.win, C.byref(self.args), 7, 1e-5,
                 -1.0 / self.n, self.shifts[0], self.shifts[1], self._p(self.g_u), self._p(self.ws.sum_n), None)
            if not record:
                lib.ffdp_step_lncc_passes(*a, self._lws, 3, s)
                return None
            ev[0].record()
            lib.ffdp_step_lncc_passes(*a, self._lws, 1, s)
            ev[1].record()
            lib.ffdp_step_lncc_passes(*a, self._lws, 2, s)
            ev[2].record()
            return [("k_lncc_sample", ev[0], ev[1]), ("k_lncc_moments", ev[1], ev[2])]
        rec = self.ws.records(self.dims, self.slab) if self.use_rec else None
        if rec is None and record:
            self.ws.raw.zero_()
            ev[0].record()
            lib.ffdp_step_mi_hist(self._p(self.f), self._p(self.u), self.dims, self.slab, self.win, C.byref(self.args),
                                  C.byref(self.kernel.c), self._p(self.ws.raw), self._p(self.ws.scratch), None, s)
            lib.ffdp_mi_finalize(self._p(self.ws.raw), self.bins, -1.0, self._p(self.ws.table), s)
            ev[1].record()
            lib.ffdp_step_mi_grad(self._p(self.f), self._p(self.u), self.dims, self.slab, self.win,
                                  C.byref(self.args), C.byref(self.kernel.c), self._p(self.ws.table),
                                  self._p(self.g_u), None, s)
            ev[2].record()
            return [("k_mi_hist_bs+finalize", ev[0], ev[1]), ("k_step_mi_grad", ev[1], ev[2])]
        if not record:
            lib.ffdp_step_mi(self._p(self.f), self._p(self.u), self.dims, self.slab, self.win, C.byref(self.args),
                             C.byref(self.kernel.c), self._p(self.ws.raw), self._p(self.ws.table), self._p(self.g_u),
                             self._p(self.ws.scratch), self._p(rec) if rec is not None else None, None, s)
            return None
        self.ws.raw.zero_()
        ev[0].record()
        # pass 1 with the finalize fused into its last CTA (what ffdp_step_mi launches)
        lib.ffdp_step_mi_hist_final(self._p(self.f), self._p(self.u), self.dims, self.slab, self.win,
                                    C.byref(self.args), C.byref(self.kernel.c), self._p(self.ws.raw), -1.0,
                                    self._p(self.ws.table), self._p(self.ws.scratch), self._p(rec), None, s)
        ev[1].record()
        lib.ffdp_step_mi_grad_rec(self._p(self.f), self.dims, self.slab, C.byref(self.kernel.c),
                                  self._p(self.ws.table), self._p(rec), self._p(self.g_u), s)
        ev[2].record()
        return [("k_mi_hist_bs", ev[0], ev[1]), ("k_step_mi_grad_rec", ev[1], ev[2])]

    def capture(self):
        """CUDA graph of one launch-only step: the timed loop replays it, so host launch
        overhead never gates the device."""
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                self.step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step()
        torch.cuda.synchronize()
        return g

    def new_pair(self):
        if self.loss == "lncc" and not self.twopass:
            lib, V, C = self.lib, self.V, self.C
            lib.ffdp_minmax(self._p(self.f), self.f.numel(), self._p(self.ranges), V._stream())
            pm = self.mimg.padded
            lib.ffdp_minmax(self._p(pm), pm.numel(), C.c_void_p(self.ranges.data_ptr() + 8), V._stream())

    def loss_value(self):
        if self.loss == "lncc":
            return 1.0 - float(self.ws.sum_n.item()) / self.n
        b = self.bins
        return -float(self.ws.table[2 * b * b + 2 * b + 1].item())


def run_sharded(args, rank, world, local_rank, dev):
    """N > 1: the native sharded plan (include/ffdp.h ffdp_plan_*, csrc/plan.cu), one rank
    per GPU over NCCL (the communicator is created by the library from a unique id that
    torch.distributed only broadcasts). Strong scaling (default): the N = 1 workload's
    volume split into N z slabs; weak: each GPU keeps the N = 1 voxel count of an N x taller
    volume. Per step, inside the library: the u halo exchange overlapped with the interior
    planes (LNCC), the fused kernels on the slab, one allreduce ({sum n_i, misses} or the
    integer joint histogram + misses)."""
    import torch
    import torch.distributed as dist

    from paper_2509_25044_b200 import plan as PL
    from paper_2509_25044_b200 import voxreg

    shape, loss, cfg = WORKLOADS[args.workload]
    strong = args.scaling == "strong"
    gshape = shape if strong else (shape[0] * world, shape[1], shape[2])
    lo, hi = _shard_range(gshape[0], world, rank)

    def reduce_minmax(a, b):
        t = torch.tensor([a, -b], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t[0]), -float(t[1])

    f, m, u, A, t = synth_inputs(gshape, loss, 1234, dev, lo, hi, reduce_minmax, jitter=args.jitter)
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(PL.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    group = PL.nccl_group(bytes(uid.cpu().numpy().tobytes()), world, rank, local_rank)
    params = voxreg.LossParams(kind=loss, bins=32, mi_bspline_kernel=True)
    pl = PL.ShardPlan(group, gshape, params, A, t, records=True, overlap=True)
    pl.load(f, m)
    pl.set_u(u)
    out = _time_plan(args, pl, world, lambda x, op: dist.all_reduce(x, op=op), dist.ReduceOp.MAX, dist.barrier,
                     local_rank)
    # end to end: every step the rank's slabs come from host memory (pinned), a new pair is
    # loaded (F halo planes, intensity frame, moving window), the step runs, the loss is read
    nbytes = 4 * (f.numel() + m.numel() + u.numel())
    hf, hm, hu = (x.cpu() for x in (f, m, u))
    if nbytes <= (8 << 30):
        hf, hm, hu = (x.pin_memory() for x in (hf, hm, hu))
    steps_e2e = 3
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps_e2e):
        f.copy_(hf, non_blocking=True)
        m.copy_(hm, non_blocking=True)
        u.copy_(hu, non_blocking=True)
        pl.load(f, m)
        pl.set_u(u)
        pl.step(sync=True)
    te = torch.tensor([(time.perf_counter() - t0) / steps_e2e * 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    pl.close()
    group.close()
    nvox_total = gshape[0] * gshape[1] * gshape[2]
    out.update({
        "scaling": "strong" if strong else "weak",
        "config": {"workload": f"{args.workload}: BASELINE configs[{cfg}]" + ("" if strong else " per GPU"),
                   "volume": "x".join(str(s) for s in gshape[::-1]), "loss": loss, "voxels_per_gpu": f.numel(),
                   "parallelism": f"z-slab x{world}: native plan over NCCL (halo send/recv overlapped with "
                                  f"interior planes; allreduce of the loss / integer histogram)",
                   "u_jitter": "SURVEY 8(d)" if args.jitter == "survey" else "U(-0.01, 0.01) voxel",
                   "l2": "inputs exceed the 126 MB L2; no flush between steps"},
        "e2e": {"value": round(nvox_total / (float(te.item()) * 1e-3) / 1e9, 4), "unit": "Gvoxel/s",
                "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": 16 * world,
                "ms_per_step": round(float(te.item()), 3), "steps": steps_e2e},
    })
    return out


def _shard_range(n, world, rank):
    """shard_ranges (fabric.hpp:44-57)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _time_plan(args, pl, world, allreduce, op_max, barrier, local_rank):
    """Warm-up (the first step is checked: window misses repaired), K launch-only steps
    between CUDA events on the plan's stream, misses verified after the loop, the step time
    is the max over ranks."""
    import torch
    pl.step(sync=True)
    for _ in range(args.warmup - 1):
        pl.step(sync=False)
    pl.result()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    e0.record(pl.stream)
    for _ in range(args.steps):
        pl.step(sync=False)
    e1.record(pl.stream)
    torch.cuda.synchronize()
    clocks.stop()
    loss_val, misses = pl.result()
    if misses != 0:
        raise RuntimeError(f"plan: {misses} window misses in the timed (unchecked) steps")
    tt = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=pl.u.device)
    allreduce(tt, op_max)
    ms_step = float(tt.item()) / args.steps
    shape, loss, _ = WORKLOADS[args.workload]
    gshape = pl.global_shape
    nvox_total = gshape[0] * gshape[1] * gshape[2]
    nloc = (pl.hi - pl.lo) * gshape[1] * gshape[2]
    value = nvox_total / (ms_step * 1e-3) / 1e9
    hbm, hbm_kind = peaks()
    per_gpu_gbs = BYTES_PER_VOXEL[loss] * nloc / (ms_step * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": round(value, 3), "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "vs_baseline": None, "dtype": DTYPE[loss], "data": "synthetic", "loss": loss_val,
        "roofline": {"bound": "hbm", "kernel": "step (per GPU, rank 0's slab)", "achieved": round(per_gpu_gbs, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(per_gpu_gbs / hbm, 4), "traffic": None,
                     "peak_kind": hbm_kind, "algorithmic_bytes_per_voxel": BYTES_PER_VOXEL[loss]},
        # ours per step: LNCC up to 3 fused launches + their partial sums + the miss pack; MI
        # pass 1, histogram conversion, finalize, pass 2, readback pack
        "gpu_launches": (7 if loss == "lncc" else 5) * args.steps,
        "window": pl.window(),
        "clocks": clocks.summary(),
    }


def run_local_group(args):
    """--transport local: the N ranks as host threads of ONE process over the library's
    in-process group (peer copies between the visible devices, round-robin; several ranks
    may share one device). The reference's own one-process WorkerGroup(H) model
    (fabric.hpp:266-300); on one GPU a functional run of the sharded path, not a scaling
    measurement."""
    import threading

    import torch

    from paper_2509_25044_b200 import plan as PL
    from paper_2509_25044_b200 import voxreg
    world = args.gpus
    shape, loss, cfg = WORKLOADS[args.workload]
    ndev = max(1, torch.cuda.device_count())
    devs = [r % ndev for r in range(world)]
    groups = PL.local_group(world, devs)
    f, m, u, A, t = synth_inputs(shape, loss, 1234, "cuda:0", jitter=args.jitter)
    params = voxreg.LossParams(kind=loss, bins=32, mi_bspline_kernel=True)
    plans = [None] * world
    barrier = threading.Barrier(world)
    res = [None] * world
    err = []
    times = [0.0] * world

    def rank(r):
        try:
            torch.cuda.set_device(devs[r])
            pl = PL.ShardPlan(groups[r], shape, params, A, t, records=True, overlap=True)
            plans[r] = pl
            pl.load(f[pl.lo:pl.hi].to(f"cuda:{devs[r]}"), m[pl.lo:pl.hi].to(f"cuda:{devs[r]}"))
            pl.set_u(u[pl.lo:pl.hi].to(f"cuda:{devs[r]}"))
            red = {}

            def allreduce(x, op):
                times[r] = float(x.item())
                barrier.wait()
                x.fill_(max(times))
                barrier.wait()

            res[r] = _time_plan(args, pl, world, allreduce, None, barrier.wait, devs[r])
            del red
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            barrier.abort()

    th = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(world)]
    for x in th:
        x.start()
    # a rank that fails leaves its peers inside a collective: report it instead of waiting
    while any(x.is_alive() for x in th):
        for x in th:
            x.join(timeout=0.5)
        if err:
            import traceback
            traceback.print_exception(err[0], file=sys.stderr)
            sys.stderr.flush()
            os._exit(1)
    if err:
        raise err[0]
    for pl in plans:
        pl.close()
    for g in groups:
        g.close()
    out = res[0]
    out.update({"scaling": "strong",
                "config": {"workload": f"{args.workload}: BASELINE configs[{cfg}]",
                           "volume": "x".join(str(s) for s in shape[::-1]), "loss": loss,
                           "parallelism": f"z-slab x{world}: native plan, in-process group on devices {devs}",
                           "l2": "inputs exceed the 126 MB L2; no flush between steps"}})
    return out


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    local_rank %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2509_25044_b200._lib import lib
    so = lib.load()
    if so.ffdp_device_check() != 0:
        raise RuntimeError(so.ffdp_last_error().decode())
    if world > 1 or getattr(args, "force_plan", False):
        return run_sharded(args, rank, world, local_rank, dev), None
    shape, loss, cfg = WORKLOADS[args.workload]
    jitter = getattr(args, "jitter", "bench")
    f, m, u, A, t = synth_inputs(shape, loss, 1234, dev, jitter=jitter)
    # M lives only in the step's zero-bordered layout from here on: at configs[4] the 15 GB
    # of a second copy would crowd out the 16 B/voxel pass-1 records
    st = Stepper(f, m, u, A, t, loss)
    del m
    torch.cuda.empty_cache()
    st.choose_records()
    hbm, hbm_kind = peaks()
    for _ in range(args.warmup):
        st.step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = st.capture()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    e0.record()
    for i in range(args.steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    clocks.stop()
    ms = e0.elapsed_time(e1)
    # per-kernel device time: the same K steps launched with events around each kernel
    recs = [st.step(record=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    per_kernel = {}
    for r in recs:
        for name, a, b in r:
            per_kernel.setdefault(name, []).append(a.elapsed_time(b))
    kern_ms = {k: sum(v) / len(v) for k, v in per_kernel.items()}
    nvox = f.numel()
    ms_step = ms / args.steps
    value = world * nvox / (ms_step * 1e-3) / 1e9
    loss_val = st.loss_value()

    # dominant kernel roofline (algorithmic bytes per launch / live event duration)
    if loss == "lncc" and "k_lncc_fused" in kern_ms:
        # the one-pass step: the kernel IS the step (32 algorithmic B/voxel: F, u, M, g_u)
        dom, dom_bytes = "k_lncc_fused", 32 * nvox
    elif loss == "lncc":
        # two passes: algorithmic bytes of the step (32 B/voxel: read F, u, M once, write
        # g_u) split as pass 1 reads u + M (16 B), pass 2 reads F and writes g_u (16 B)
        dom = max(kern_ms, key=kern_ms.get)
        dom_bytes = 16 * nvox
    else:
        dom = max(kern_ms, key=kern_ms.get)
        dom_bytes = (20 if "hist" in dom else 32) * nvox
    achieved = dom_bytes / (kern_ms[dom] * 1e-3) / 1e9
    traffic = ncu_traffic(dom.split("+")[0], nvox)
    step_gbs = BYTES_PER_VOXEL[loss] * nvox / (ms_step * 1e-3) / 1e9

    # end to end through the public API with host buffers (pinned), H2D + step + D2H(loss)
    e2e = run_e2e(args, st, f, u, A, t, loss, world)

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[loss], "data": "synthetic",
        "config": {"workload": f"{args.workload}: BASELINE configs[{cfg}]",
                   "volume": "x".join(str(s) for s in shape[::-1]), "loss": loss,
                   "u_jitter": ("SURVEY 8(d): U(-0.01, 0.01) normalized" if jitter == "survey" else
                                "U(-0.01, 0.01) voxel"),
                   "loss_params": "window 7, eps 1e-5, ANTs" if loss == "lncc" else "32 bins, B-spline Parzen, exact",
                   "voxels_per_gpu": nvox, "parallelism": f"z-slab x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs (F, M, u, g_u) exceed the 126 MB L2; no flush between steps"},
        "loss": loss_val,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic[0], "traffic_note": traffic[1],
                     "peak_kind": hbm_kind,
                     "algorithmic_bytes_per_voxel": dom_bytes // nvox},
        "step_roofline": {"achieved": round(step_gbs, 1), "frac": round(step_gbs / hbm, 4),
                          "bytes_per_voxel": BYTES_PER_VOXEL[loss]},
        "kernel_ms": {k: round(v, 5) for k, v in kern_ms.items()},
        "mi_records": getattr(st, "records_note", None),
        "gpu_launches": st.launches_per_step * args.steps,
        "clocks": clocks.summary(),
        "e2e": e2e,
    }
    return out, st


def run_warp_update(shape, steps, hbm, hbm_kind):
    """The warp update after the step (registration.hpp:313-317):
    ffdp_sobolev_adam (gp_convolve(g_u, gaussian 1.0) + adam_step, 84 B/voxel: reads g_u,
    u, m1, m2, writes u, m1, m2) and ffdp_gp_convolve(u, gaussian 0.5) (24 B/voxel), each
    timed with CUDA events on the launching stream."""
    import ctypes as C

    import torch

    from paper_2509_25044_b200 import voxreg as V
    from paper_2509_25044_b200._lib import lib
    nz, ny, nx = shape
    g = torch.empty((nz, ny, nx, 3), device="cuda").uniform_(-1e-6, 1e-6)
    u = torch.empty_like(g).uniform_(-0.01, 0.01)
    m1, m2, out = torch.zeros_like(g), torch.zeros_like(g), torch.empty_like(g)
    slab = V._full_slab(nz)
    dims = V._dims(g.shape)
    tg, tw = V.gaussian_taps(1.0), V.gaussian_taps(0.5)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    lr = V.deformable_lr_norm(shape, 0.5)

    def once(k, ev=None):
        if ev:
            ev[0].record()
        lib.ffdp_sobolev_adam(V._ptr(g), V._ptr(u), V._ptr(m1), V._ptr(m2), dims, slab, V._taps_ptr(tg), len(tg), lr,
                              0.9, 0.999, 1e-8, k, s)
        if ev:
            ev[1].record()
        lib.ffdp_gp_convolve(V._ptr(u), V._ptr(out), dims, slab, 3, V._taps_ptr(tw), len(tw), 1, s)
        if ev:
            ev[2].record()

    for k in range(3):
        once(k + 1)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k, ev in enumerate(evs):
        once(k + 4, ev)
    torch.cuda.synchronize()
    t_adam = sum(e[0].elapsed_time(e[1]) for e in evs) / steps
    t_conv = sum(e[1].elapsed_time(e[2]) for e in evs) / steps
    n = nz * ny * nx
    gbs = lambda b, ms: b * n / (ms * 1e-3) / 1e9
    return {"lattice": f"{nx}x{ny}x{nz}", "ms": round(t_adam + t_conv, 4),
            "kernel_ms": {"k_smooth<3,3,adam> (sobolev_adam)": round(t_adam, 4),
                          "k_smooth<2,3,store> (gp_convolve)": round(t_conv, 4)},
            "roofline": {"bound": "hbm", "achieved": round(gbs(108, t_adam + t_conv), 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(gbs(108, t_adam + t_conv) / hbm, 4), "peak_kind": hbm_kind,
                         "algorithmic_bytes_per_voxel": 108,
                         "per_kernel_frac": {"sobolev_adam": round(gbs(84, t_adam) / hbm, 4),
                                             "gp_convolve": round(gbs(24, t_conv) / hbm, 4)}},
            "gpu_launches": 2 * steps}


def run_registration(shape, schedule_spec):
    """BASELINE configs[2]: multi-scale deformable LNCC registration (registration.hpp:
    230-331) of the synthetic 720x640x720 pair on one GPU through the public driver
    (registration.deformable_stage): per scale resample F/M on the device, then per
    iteration the fused step + Sobolev/Adam update + warp smoothing. Timed with CUDA
    events around the whole call (host reads the loss trace once per scale)."""
    import torch

    from paper_2509_25044_b200 import registration as R
    from paper_2509_25044_b200 import voxreg as V
    # the pair differs by a smooth deformation of ~4 voxels and carries texture at the
    # window's scale (32-voxel wavelength), so LNCC sees structure and the registration has
    # something to recover; the deformable stage starts from the identity affine (the affine
    # stage's job is not part of this config)
    f, m, _, _, _ = synth_inputs(shape, "lncc", 1234, "cuda", fine=(32.0, 0.25, 0.012))
    sch = R.ScaleSchedule([R.ScaleStep(d, n) for d, n in schedule_spec], loss=V.LossParams(kind="lncc"))
    # warm-up: one iteration per scale (allocations, attributes)
    R.deformable_stage(f, m, None, R.ScaleSchedule([R.ScaleStep(d, 1) for d, _ in schedule_spec],
                                                   loss=V.LossParams(kind="lncc")))
    torch.cuda.synchronize()
    # three timed registrations; the median is reported (per-scale device allocations of
    # up to a few GB make single runs vary by ~0.1 s)
    runs = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        trace = []
        e0.record()
        R.deformable_stage(f, m, None, sch, trace=trace)
        e1.record()
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    ms = sorted(runs)[1]
    vox_iters = sum(int(__import__("numpy").prod(R.resample_dims(shape, 1.0 / d))) * n for d, n in schedule_spec)
    return {"workload": "lncc720 multi-scale deformable registration: BASELINE configs[2]",
            "lattice": "x".join(str(s) for s in shape[::-1]),
            "schedule": [{"downsample": d, "iterations": n} for d, n in schedule_spec],
            "seconds": round(ms / 1e3, 4), "seconds_runs": [round(x / 1e3, 4) for x in runs],
            "voxel_iterations": vox_iters,
            "gvoxel_iterations_per_s": round(vox_iters / (ms * 1e-3) / 1e9, 3),
            # per scale: the loss falls within a scale; across scales it is not comparable
            # (a 7^3 window sees less structure at full resolution than at 1/4)
            "loss_per_scale": [{"downsample": d, "first": round(min(e.loss for e in trace if e.scale_index == i and
                                                                    e.iteration == 0), 6),
                                "last": round([e.loss for e in trace if e.scale_index == i][-1], 6)}
                               for i, (d, _) in enumerate(schedule_spec)],
            "per_iteration": "the one-pass fused warp+LNCC step (k_lncc_fused + its partial-sum reduction), "
                             "ffdp_sobolev_adam, ffdp_gp_convolve"}


class HostStager:
    """Host -> device copies of inputs that live in ordinary (pageable) host memory,
    through two pinned staging buffers: the CPU fills one buffer while the DMA engine
    drains the other (cudaMemcpyAsync from pinned memory on a copy stream). Used when the
    inputs are too large to pin whole (configs[4]: 74 GB of F, M, u per step)."""

    def __init__(self, chunk_bytes=256 << 20):
        import torch
        self.torch = torch
        self.n = chunk_bytes // 4
        self.bufs = [torch.empty(self.n, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.evs = [None, None]
        self.stream = torch.cuda.Stream()
        self.k = 0

    def copy(self, dst, src):
        """dst (CUDA, any strides) <- src (host, contiguous, same shape), split along dim 0."""
        torch = self.torch
        per = max(1, src[0].numel()) if src.dim() > 0 else 1
        rows = max(1, self.n // per)
        self.stream.wait_stream(torch.cuda.current_stream())
        for z0 in range(0, src.shape[0], rows):
            z1 = min(src.shape[0], z0 + rows)
            i = self.k % 2
            self.k += 1
            if self.evs[i] is not None:
                self.evs[i].synchronize()  # the DMA out of this buffer is done
            cnt = (z1 - z0) * per
            buf = self.bufs[i][:cnt]
            buf.copy_(src[z0:z1].reshape(-1))
            with torch.cuda.stream(self.stream):
                dst[z0:z1].copy_(buf.view(src[z0:z1].shape), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self.evs[i] = ev
        torch.cuda.current_stream().wait_stream(self.stream)


def run_e2e(args, st, f, u, A, t, loss, world):
    """End to end through the public API: every step copies the step's inputs (F, M, u)
    from host memory to the device, runs the step, and reads the loss back (8 bytes).
    The host inputs are pinned whole when they take at most 60 % of the host's available
    RAM (configs[4]: 74 GB of 196 GB; the DMA then runs at the PCIe rate, ~55 GB/s on the
    B200 boxes, against ~43 GB/s through staging); otherwise they stay in pageable memory
    and go through HostStager's double-buffered pinned chunks."""
    import torch
    m = st.mimg.interior
    nbytes = 4 * (f.numel() + m.numel() + u.numel())
    steps = max(3, min(args.steps, 20 if nbytes <= (8 << 30) else 3))
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    staged = nbytes > (8 << 30) and (os.environ.get("FFDP_E2E_STAGED") == "1" or nbytes > 0.6 * avail)
    # host copies made straight from the device (M from its bordered layout a few planes at
    # a time: a strided view, and a whole-volume device temporary would not fit next to
    # configs[4]'s records)
    hf = torch.empty(tuple(f.shape), dtype=torch.float32)
    hu = torch.empty(tuple(u.shape), dtype=torch.float32)
    hm = torch.empty(tuple(m.shape), dtype=torch.float32)
    for dst, src in ((hf, f), (hu, u), (hm, m)):
        for z0 in range(0, src.shape[0], 16):
            dst[z0:z0 + 16].copy_(src[z0:z0 + 16])
    registered = []
    if not staged:
        # page-lock the buffers in place (cudaHostRegister; torch's pinned allocator would
        # round each one up to a power of two: 103 instead of 74 GB at configs[4])
        rt = torch.cuda.cudart()
        for x in (hf, hu, hm):
            if int(rt.cudaHostRegister(x.data_ptr(), x.numel() * 4, 0)) != 0:
                raise RuntimeError("cudaHostRegister failed")
            registered.append(x)

        def cp(dst, src):
            # 32 planes at a time: M's bordered destination is strided, and torch stages a
            # strided H2D through a contiguous device temporary of the chunk's size
            for z0 in range(0, src.shape[0], 32):
                dst[z0:z0 + 32].copy_(src[z0:z0 + 32], non_blocking=True)
    else:
        stager = HostStager()
        cp = stager.copy
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_loss = 0.0
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        cp(st.f, hf)
        cp(st.mimg.interior, hm)  # H2D straight into the bordered layout
        cp(st.u, hu)
        st.new_pair()  # a new (F, M) pair: the LNCC intensity frame is re-derived on the device
        st.step()
        host_loss = st.loss_value()  # D2H read of the step result (8 bytes)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    ms = max(e0.elapsed_time(e1) / steps, wall)
    for x in registered:
        torch.cuda.cudart().cudaHostUnregister(x.data_ptr())
    return {"value": round(world * f.numel() / (ms * 1e-3) / 1e9, 4), "unit": "Gvoxel/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 8, "ms_per_step": round(ms, 3), "steps": steps,
            "host_buffers": "pageable, double-buffered pinned staging (256 MB chunks)" if staged else "pinned",
            "host_available_bytes": int(avail),
            "loss": host_loss}


# ------------------------------------------------------------------ the CPU reference
def cpu_reference(loss, sample_shape, steps, threads):
    """The reference's own step (ring_sample -> dist_lncc|dist_mi -> ring_sample_backward
    under WorkerGroup(H), oracle/_ref) on a bounded sample, H = `threads` std::threads."""
    from oracle import Oracle, Reference, step_inputs
    try:
        ref = Reference()
        kind = "reference"
    except FileNotFoundError:
        ref = None
        kind = "port"
    orc = Oracle()
    si = step_inputs(orc, sample_shape, seed=4242, loss=loss)
    n = int(si.f.size)
    t0 = time.perf_counter()
    for _ in range(steps):
        if ref is not None:
            ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=threads)
        elif loss == "lncc":
            orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
        else:
            orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    dt = (time.perf_counter() - t0) / steps
    return {"value": round(n / dt / 1e9, 6), "unit": "Gvoxel/s", "cores": threads if ref is not None else 1,
            "kind": kind, "sample": f"{'x'.join(str(s) for s in sample_shape[::-1])} {loss} step x{steps} "
                                    f"({'T=double, WorkerGroup(%d)' % threads if ref is not None else 'C port, 1 thread'})",
            "s_per_step": round(dt, 4)}


def cpu_variants(loss, sample_shape, threads):
    """SURVEY.md 8(d)'s other CPU timings of the reference step on the same sample: one
    worker (H = 1) in double, and all host threads in T=float. One step each."""
    from oracle import Oracle, Reference, step_inputs
    try:
        ref = Reference()
    except FileNotFoundError:
        return []
    si = step_inputs(Oracle(), sample_shape, seed=4242, loss=loss)
    n = int(si.f.size)
    out = []
    for world, fp32 in ((1, False), (threads, True)):
        t0 = time.perf_counter()
        ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=world, fp32=fp32)
        dt = time.perf_counter() - t0
        out.append({"threads": world, "T": "float" if fp32 else "double", "value": round(n / dt / 1e9, 6),
                    "unit": "Gvoxel/s", "s_per_step": round(dt, 4)})
    return out


def cpu_sample_for(loss):
    return (96, 96, 96) if loss == "mi" else (128, 128, 128)


def default_workload():
    """SURVEY / VERDICT rule: the N = 1 headline is the largest single-GPU configuration,
    configs[4] (3.7 G-voxel MI; 119 GB of F, M, u, g_u) when it fits, else configs[2]."""
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.get_device_properties(0).total_memory >= (150 << 30):
            return "mi1760"
    except Exception:
        pass
    return "lncc720"


SECONDARY_KEYS = ("value", "unit", "ms_per_step", "config", "roofline", "step_roofline", "kernel_ms", "clocks",
                  "e2e", "loss", "gpu_launches")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto"] + sorted(WORKLOADS))
    ap.add_argument("--jitter", default="bench", choices=["bench", "survey"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: split the N = 1 volume (strong) or grow it N x along z (weak)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "local"],
                    help="N > 1: one process per GPU over NCCL (torchrun), or N ranks as threads of one process")
    ap.add_argument("--force-plan", action="store_true",
                    help="run the native sharded plan over NCCL even at one rank (a functional check of the N > 1 path)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.workload == "auto":
        args.workload = default_workload()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    shape, loss, cfg = WORKLOADS[args.workload]
    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's own step (oracle/_ref: the unmodified headers) on a bounded
        # sample of the workload, all host threads; inputs and libraries are prepared once,
        # outside the timed loop, so each timed step is exactly one ref.step call
        from oracle import Oracle, Reference, step_inputs
        threads = os.cpu_count() or 1
        samp = cpu_sample_for(loss)
        try:
            ref = Reference()
            kind = "reference"
        except FileNotFoundError:
            ref, kind = None, "port"
        orc = Oracle()
        si = step_inputs(orc, samp, seed=4242, loss=loss)
        kern = orc.parzen("bspline3", 32)

        def one():
            if ref is not None:
                ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=threads)
            elif loss == "lncc":
                orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
            else:
                orc.step_mi(si.f, si.m, si.u, kern, si.A, si.t)

        for _ in range(args.warmup):
            one()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one()
        dt = (time.perf_counter() - t0) / args.steps
        n = samp[0] * samp[1] * samp[2]
        v = n / dt / 1e9
        sample = (f"{'x'.join(str(s) for s in samp[::-1])} {loss} step x{args.steps} "
                  f"({'T=double, WorkerGroup(%d)' % threads if ref is not None else 'C port, 1 thread'})")
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gvoxel/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: BASELINE configs[{cfg}] (bounded sample "
                                   f"{'x'.join(str(s) for s in samp[::-1])} on the host cores)", "loss": loss},
            "cpu_baseline": {"value": round(v, 6), "unit": "Gvoxel/s", "cores": threads if ref is not None else 1,
                             "kind": kind, "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "Gvoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    if args.transport == "local" and args.gpus > 1:
        print(json.dumps(run_local_group(args)))
        return
    if world > 1 or args.force_plan:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    out, st = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.force_plan:
        import torch
        del st
        torch.cuda.empty_cache()
        cpu = {}

        def baseline(kind_loss):
            if args.no_cpu:
                return None
            if kind_loss not in cpu:
                try:
                    cb = cpu_reference(kind_loss, cpu_sample_for(kind_loss), 2, os.cpu_count() or 1)
                    cb["variants"] = cpu_variants(kind_loss, cpu_sample_for(kind_loss), os.cpu_count() or 1)
                except Exception as e:  # the baseline is reported, never required
                    cb = {"value": None, "unit": "Gvoxel/s", "cores": 0, "kind": "port", "sample": f"unavailable: {e}"}
                cpu[kind_loss] = cb
            return cpu[kind_loss]

        cb = baseline(loss)
        if cb is not None:
            out["cpu_baseline"] = cb
        if not args.no_secondary:
            sec = []
            for wl, jit in (("lncc720", "bench"), ("lncc720", "survey"), ("mi256", "bench"), ("mi256", "survey")):
                if wl == args.workload and jit == args.jitter:
                    continue
                a2 = argparse.Namespace(**vars(args))
                a2.workload, a2.jitter, a2.steps = wl, jit, max(5, min(args.steps, 20))
                r, s2 = run_ours(a2, rank, world, local_rank)
                del s2
                torch.cuda.empty_cache()
                line = {k: r[k] for k in SECONDARY_KEYS if k in r}
                c2 = baseline(WORKLOADS[wl][1])
                if c2 is not None:
                    line["cpu_baseline"] = c2
                sec.append(line)
            out["secondary"] = sec
            hbm, hbm_kind = peaks()
            out["warp_update"] = run_warp_update(WORKLOADS["lncc720"][0], max(5, min(args.steps, 20)), hbm, hbm_kind)
            torch.cuda.empty_cache()
            out["registration"] = run_registration(WORKLOADS["lncc720"][0], [(4, 20), (2, 20), (1, 10)])
    if world > 1 or args.force_plan:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
