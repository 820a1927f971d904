"""The `voxreg` command line over the B200 path (tools/main.cpp:1-496): the same
subcommand, flags, `--config` file rules, output files and exit codes.

    python -m paper_2509_25044_b200.cli register --fixed F.nii --moving M.nii --out run [...]
    python -m paper_2509_25044_b200.cli metrics --a A.nii --b B.nii [--spacing x,y,z] [--out m.json]
    python -m paper_2509_25044_b200.cli synth --out pair [--seed S] [--dims N|Nx,Ny,Nz] [--labels K]
    python -m paper_2509_25044_b200.cli info --in F.nii

Exit codes (main.cpp:3-4): 0 success, 1 configuration error, 2 I/O or format error,
3 numerical abort (trace flushed first).

`register` reads the NIfTI pair, runs register_volumes (registration.py: the affine
stage, then the multi-scale deformable stage on the GPU), warps the ORIGINAL moving
image with the result and writes `<out>_warp.{raw,json}`, `<out>_moved.nii` (fp64),
`<out>_trace.csv` and `<out>_summary.json` (also printed), as main.cpp:219-300 does.
`--shards H` runs the z-slab sharded deformable stage: in this process over the node's
GPUs (ffdp_comm, the reference's one-process model), or one rank per process under
`python -m torch.distributed.run --nproc-per-node H -m paper_2509_25044_b200.cli
register ... --shards H` (rank 0 writes the outputs). The GPU path computes in fp32
whatever `--float32` says (the flag is recorded in the summary); `--lncc-backend naive`
names the reference's materialised-graph ablation, whose values equal the fused
backend's (test_lncc.cpp:70-79), and runs the fused path (single worker only, as in
registration.hpp:238-239). `peak_alloc_bytes` is the device allocator's peak.
`metrics` and the label block of the summary use metrics.py and `synth` uses synth.py
(host numpy, as the reference's are host code; both bit-identical to the reference).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import dataclass
from typing import List, Optional


class ConfigError(ValueError):
    """CLI::ValidationError / std::invalid_argument: exit code 1."""


@dataclass
class _Opt:
    name: str            # long name without the leading dashes
    dest: str
    kind: type           # str, int, float, bool (flag)
    default: object
    choices: Optional[tuple] = None
    required: bool = False
    negatable: bool = False  # "--x,!--no-x"
    help: str = ""


# tools/main.cpp:38-64 (defaults) and 376-418 (names, checks)
REGISTER_OPTIONS = [
    _Opt("fixed", "fixed_path", str, "", required=True, help="fixed image (.nii)"),
    _Opt("moving", "moving_path", str, "", required=True, help="moving image (.nii)"),
    _Opt("out", "out_prefix", str, "", required=True, help="output prefix"),
    _Opt("fixed-labels", "fixed_labels_path", str, "", help="fixed label map (.nii)"),
    _Opt("moving-labels", "moving_labels_path", str, "", help="moving label map (.nii)"),
    _Opt("loss", "loss", str, "lncc", ("mse", "lncc", "mi"), help="similarity: mse|lncc|mi"),
    _Opt("window", "window", int, 7, help="LNCC window (odd)"),
    _Opt("epsilon", "epsilon", float, 1e-5, help="LNCC epsilon"),
    _Opt("ants-approx", "ants_approx", bool, True, negatable=True,
         help="skip gamma convolutions in the LNCC backward"),
    _Opt("lncc-backend", "lncc_backend", str, "fused", ("fused", "naive"),
         help="fused (5-channel state) or naive (materialized graph, single worker)"),
    _Opt("bins", "bins", int, 32, help="MI histogram bins"),
    _Opt("mi-kernel", "mi_kernel", str, "gaussian", ("gaussian", "bspline"), help="MI Parzen kernel: gaussian|bspline"),
    _Opt("mi-approx-forward", "mi_approx_forward", bool, False, help="binned-histogram MI forward"),
    _Opt("scales", "scales", str, "4,2,1", help="deformable downsample factors, e.g. 4,2,1"),
    _Opt("iters", "iters", str, "100,100,50", help="iterations per deformable scale"),
    _Opt("lr", "lr", float, 0.5, help="deformable learning rate (voxels)"),
    _Opt("sigma-grad", "sigma_grad", float, 1.0, help="gradient smoothing (voxels)"),
    _Opt("sigma-warp", "sigma_warp", float, 0.5, help="warp smoothing (voxels)"),
    _Opt("affine-scales", "affine_scales", str, "4,2", help="affine downsample factors"),
    _Opt("affine-iters", "affine_iters", str, "60,40", help="iterations per affine scale"),
    _Opt("affine-lr", "affine_lr", float, 0.01, help="affine learning rate"),
    _Opt("affine-loss", "affine_loss", str, "mi", ("mse", "lncc", "mi"), help="affine similarity: mse|lncc|mi"),
    _Opt("skip-affine", "skip_affine", bool, False, help="start deformable from identity"),
    _Opt("shards", "shards", int, 1, help="worker count H (torch.distributed ranks)"),
    _Opt("gp-sync", "gp_sync", bool, True, negatable=True, help="halo synchronization for sharded convolutions"),
    _Opt("seed", "seed", int, 0, help="seed recorded in the summary"),
    _Opt("float32", "float32", bool, False, help="optimize in single precision (the GPU path always does)"),
    _Opt("emit-timings", "emit_timings", bool, False,
         help="include wall time in the summary (breaks byte-reproducibility)"),
]


def _known_names():
    """The register option names a config file may use (get_lnames, main.cpp:85-91)."""
    known, flags = {"help"}, {"help"}
    for o in REGISTER_OPTIONS:
        known.add(o.name)
        if o.kind is bool:
            flags.add(o.name)
            if o.negatable:
                known.add("no-" + o.name)
                flags.add("no-" + o.name)
    return known, flags


def expand_register_config(args: List[str]) -> List[str]:
    """expand_register_config (main.cpp:69-147): splice a `--config FILE` of key=value
    lines in right after `register`; explicit flags win, unknown keys are rejected."""
    from .nifti import IoError
    if not args or args[0] != "register":
        return args
    args = list(args)
    path, i = "", 1
    while i < len(args):
        if args[i] == "--config" and i + 1 < len(args):
            path = args[i + 1]
            del args[i:i + 2]
        elif args[i].startswith("--config="):
            path = args[i][9:]
            del args[i]
        else:
            i += 1
    if not path:
        return args
    known, known_flags = _known_names()
    explicit = set()
    for a in args:
        if not a.startswith("--"):
            continue
        key = a[2:].split("=", 1)[0]
        explicit.add(key)
        if key.startswith("no-"):
            explicit.add(key[3:])
        explicit.add("no-" + key)
    try:
        with open(path, "rb") as fh:
            lines = fh.read().decode("utf-8", "replace").split("\n")
    except OSError:
        raise IoError(f"cannot open config file {path}") from None
    if lines and lines[-1] == "":
        lines.pop()
    expanded = []
    for lineno, line in enumerate(lines, 1):
        if "#" in line:
            line = line[:line.index("#")]
        line = line.rstrip(" \r")
        if line.strip(" ") == "":
            continue
        start = len(line) - len(line.lstrip(" "))
        if "=" not in line:
            raise ConfigError(f"config line {lineno}: expected key=value")
        eq = line.index("=")
        key = line[start:eq].rstrip(" ")
        value = line[eq + 1:].lstrip(" ")
        if key not in known:
            raise ConfigError(f"config line {lineno}: unknown key '{key}'")
        if key in explicit:
            continue
        if key in known_flags:
            if value in ("true", "1", "yes", "on", ""):
                expanded.append("--" + key)
            elif "no-" + key in known_flags:
                expanded.append("--no-" + key)
            # a false value for a plain default-false flag is a no-op
        else:
            expanded += ["--" + key, value]
    return args[:1] + expanded + args[1:]


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI::ParseError: exit code 1
        raise ConfigError(message)


def _int(s: str) -> int:
    try:
        return int(s, 10)
    except ValueError:
        raise argparse.ArgumentTypeError(f"{s!r} is not an integer") from None


def _build_parser() -> argparse.ArgumentParser:
    app = _Parser(prog="voxreg", description="voxreg: deformable 3-D image registration (B200)")
    sub = app.add_subparsers(dest="command", parser_class=_Parser)
    reg = sub.add_parser("register", help="register a moving volume onto a fixed volume")
    for o in REGISTER_OPTIONS:
        if o.kind is bool:
            reg.add_argument("--" + o.name, dest=o.dest, action="store_true", default=o.default, help=o.help)
            if o.negatable:
                reg.add_argument("--no-" + o.name, dest=o.dest, action="store_false")
        else:
            reg.add_argument("--" + o.name, dest=o.dest, type=_int if o.kind is int else o.kind, default=o.default,
                             choices=o.choices, required=o.required, help=o.help)
    met = sub.add_parser("metrics", help="dice / inv_dice / hd90 between label maps")
    met.add_argument("--a", dest="a", required=True, help="first label map (.nii)")
    met.add_argument("--b", dest="b", required=True, help="second label map (.nii)")
    met.add_argument("--spacing", dest="spacing", default="", help="override spacing x,y,z (mm)")
    met.add_argument("--out", dest="out", default="", help="also write the JSON here")
    syn = sub.add_parser("synth", help="generate a labeled synthetic pair")
    syn.add_argument("--seed", dest="seed", type=_int, default=2024, help="generator seed")
    syn.add_argument("--dims", dest="dims", default="48", help="volume size, N or Nx,Ny,Nz (>= 16)")
    syn.add_argument("--labels", dest="labels", type=_int, default=5, help="number of ellipsoidal labels (1..16)")
    syn.add_argument("--max-disp", dest="max_disp", type=float, default=0.15,
                     help="ground-truth warp cap, normalized units")
    syn.add_argument("--out", dest="out", required=True, help="output prefix")
    inf = sub.add_parser("info", help="print a NIfTI header summary")
    inf.add_argument("--in", dest="in_path", required=True, help="input volume (.nii)")
    return app


def parse_list(csv: str) -> List[float]:
    """parse_list (main.cpp:28-36): comma-separated numbers, empty items skipped."""
    out = []
    for tok in csv.split(","):
        if tok:
            try:
                out.append(float(tok))
            except ValueError:
                raise ConfigError("stod") from None
    return out


def build_schedule(scales: str, iters: str, lr: float, sg: float, sw: float, loss):
    """build_schedule (main.cpp:156-172)."""
    from .registration import ScaleSchedule, ScaleStep
    f, it = parse_list(scales), parse_list(iters)
    if len(f) != len(it):
        raise ConfigError("scales and iters must have the same length")
    s = ScaleSchedule(steps=[ScaleStep(fi, int(ii)) for fi, ii in zip(f, it)], lr=lr, sigma_grad=sg,
                      sigma_warp=sw, loss=loss)
    s.validate()
    return s


def config_json(o) -> dict:
    """config_json (main.cpp:174-205), in the reference's key order."""
    return {"fixed": o.fixed_path, "moving": o.moving_path, "out_prefix": o.out_prefix,
            "fixed_labels": o.fixed_labels_path, "moving_labels": o.moving_labels_path, "loss": o.loss,
            "window": o.window, "epsilon": o.epsilon, "ants_approx": o.ants_approx, "lncc_backend": o.lncc_backend,
            "bins": o.bins, "mi_kernel": o.mi_kernel, "mi_approx_forward": o.mi_approx_forward, "scales": o.scales,
            "iters": o.iters, "lr": o.lr, "sigma_grad": o.sigma_grad, "sigma_warp": o.sigma_warp,
            "affine_scales": o.affine_scales, "affine_iters": o.affine_iters, "affine_lr": o.affine_lr,
            "affine_loss": o.affine_loss, "skip_affine": o.skip_affine, "shards": o.shards, "gp_sync": o.gp_sync,
            "seed": o.seed, "float32": o.float32}


def write_trace_csv(path: str, trace) -> None:
    """write_trace_csv (main.cpp:207-216): `%d,%d,%.17g` rows."""
    from .nifti import IoError
    try:
        with open(path, "w") as fh:
            fh.write("scale_index,iteration,loss\n")
            for t in trace:
                fh.write("%d,%d,%.17g\n" % (t.scale_index, t.iteration, t.loss))
    except OSError:
        raise IoError(f"cannot open {path} for writing") from None


def _finite(v):
    """nlohmann writes non-finite doubles as null."""
    if isinstance(v, float) and not math.isfinite(v):
        return None
    if isinstance(v, dict):
        return {k: _finite(x) for k, x in v.items()}
    if isinstance(v, list):
        return [_finite(x) for x in v]
    return v


def dump_json(obj) -> str:
    """ordered_json::dump(2) (main.cpp:289-300): 2-space indent, one array item per line."""
    return json.dumps(_finite(obj), indent=2, ensure_ascii=False)


def _loss_params(o, kind: str):
    from . import voxreg as V
    if kind not in ("mse", "lncc", "mi"):
        raise ConfigError("loss must be one of mse|lncc|mi")
    return V.LossParams(kind=kind, window=o.window, epsilon=o.epsilon, ants_approx=o.ants_approx, bins=o.bins,
                        mi_bspline_kernel=o.mi_kernel == "bspline", mi_approx_forward=o.mi_approx_forward)


def _device():
    """The GPU the registration runs on (the product path has no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("register: the B200 path needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def run_register(o) -> int:
    """run_register_typed (main.cpp:227-300)."""
    import numpy as np
    import torch
    from . import nifti, registration as R, voxreg as V
    if o.shards < 1:
        raise ConfigError("--shards: value must be a positive number")
    from . import dist as D
    rank, world = D._world()
    fixed_file = nifti.read_nifti(o.fixed_path)
    moving_file = nifti.read_nifti(o.moving_path)
    dev = _device()
    fixed, moving = fixed_file.to_device(dev), moving_file.to_device(dev)

    deformable_loss = _loss_params(o, o.loss)
    affine_loss = _loss_params(o, o.affine_loss)
    cfg = R.RegistrationConfig(
        affine=build_schedule(o.affine_scales, o.affine_iters, o.affine_lr, o.sigma_grad, o.sigma_warp, affine_loss),
        deformable=build_schedule(o.scales, o.iters, o.lr, o.sigma_grad, o.sigma_warp, deformable_loss),
        deformable_opts=R.DeformableOptions(shards=o.shards, gp_sync=o.gp_sync), skip_affine=o.skip_affine)
    if o.lncc_backend == "naive" and o.shards > 1:
        raise ConfigError("deformable_stage: the naive LNCC backend is single-worker")
    if dev.type == "cuda":
        torch.cuda.reset_peak_memory_stats(dev)
    try:
        result = R.register_volumes(fixed, moving, cfg)
    except R.NumericalError as e:
        if rank == 0:
            write_trace_csv(o.out_prefix + "_trace.csv", e.trace)
        print(f"numerical abort: {e} (trace flushed)", file=sys.stderr)
        return 3
    if rank != 0:
        return 0

    # apply the recovered transform to the original moving image
    A, t = result.affine
    args = V.SamplerArgs(A=np.asarray(A, dtype=np.float64), t=np.asarray(t, dtype=np.float64))
    moved = V.fused_sample(moving, result.warp, args)
    nifti.write_warp(result.warp, o.out_prefix + "_warp", fixed_file.spacing, fixed_file.origin)
    nifti.write_nifti(moved.double(), o.out_prefix + "_moved.nii", fixed_file.spacing, fixed_file.origin)
    write_trace_csv(o.out_prefix + "_trace.csv", result.trace)

    summary = {"config": config_json(o),
               "affine_matrix": [float(x) for x in np.asarray(A, dtype=np.float64).reshape(9)],
               "affine_translation": [float(x) for x in np.asarray(t, dtype=np.float64).reshape(3)],
               "final_loss": float(result.trace[-1].loss) if result.trace else 0.0,
               "iterations": len(result.trace),
               "peak_alloc_bytes": int(torch.cuda.max_memory_allocated(dev)) if dev.type == "cuda" else 0,
               "jacobian_positive_fraction": float(result.jacobian_positive_fraction)}
    if o.fixed_labels_path and o.moving_labels_path:
        from . import metrics as MT
        lf_file = nifti.read_nifti(o.fixed_labels_path)
        lf, lm = nifti.nifti_to_labels(lf_file), nifti.nifti_to_labels(nifti.read_nifti(o.moving_labels_path))
        warped = MT.warp_labels_nn(lm, result.warp, A, t)
        summary["metrics"] = {"dice_before": MT.dice(lf, lm)[1], "dice_after": MT.dice(lf, warped)[1],
                              "inv_dice_before": MT.inv_dice(lf, lm), "inv_dice_after": MT.inv_dice(lf, warped),
                              "hd90_before": MT.hd90_cumulative(lf, lm, lf_file.spacing),
                              "hd90_after": MT.hd90_cumulative(lf, warped, lf_file.spacing)}
    if o.emit_timings:
        summary["seconds"] = float(result.seconds)
    text = dump_json(summary) + "\n"
    try:
        with open(o.out_prefix + "_summary.json", "w") as fh:
            fh.write(text)
    except OSError:
        raise nifti.IoError("cannot open summary for writing") from None
    sys.stdout.write(text)
    return 0


def run_metrics(a_path: str, b_path: str, spacing_csv: str, out_path: str) -> int:
    """run_metrics (main.cpp:302-324): dice / inv_dice / hd90 between two label maps."""
    from . import metrics as MT, nifti
    a_file = nifti.read_nifti(a_path)
    a, b = nifti.nifti_to_labels(a_file), nifti.nifti_to_labels(nifti.read_nifti(b_path))
    spacing = a_file.spacing
    if spacing_csv:
        s = parse_list(spacing_csv)
        if len(s) != 3:
            raise ConfigError("spacing must be x,y,z")
        spacing = tuple(s)
    text = dump_json({"dice": MT.dice(a, b)[1], "inv_dice": MT.inv_dice(a, b),
                      "hd90": MT.hd90_cumulative(a, b, spacing)}) + "\n"
    if out_path:
        try:
            with open(out_path, "w") as fh:
                fh.write(text)
        except OSError:
            raise nifti.IoError(f"cannot open {out_path} for writing") from None
    sys.stdout.write(text)
    return 0


def run_synth(seed: int, dims_csv: str, labels: int, max_disp: float, prefix: str) -> int:
    """run_synth (main.cpp:326-356): synth_pair written as NIfTI volumes, label maps and the
    true warp (synth.py reproduces the reference's generator bit for bit)."""
    from . import nifti, synth
    d = parse_list(dims_csv)
    if len(d) == 1:
        nx = ny = nz = int(d[0])
    elif len(d) == 3:
        nx, ny, nz = (int(v) for v in d)
    else:
        raise ConfigError("dims must be N or Nx,Ny,Nz")
    p = synth.synth_pair(seed, (nz, ny, nx), labels, max_disp)
    nifti.write_nifti(p.fixed, prefix + "_fixed.nii")
    nifti.write_nifti(p.moving, prefix + "_moving.nii")
    nifti.write_labels(p.labels_fixed, prefix + "_fixed_labels.nii")
    nifti.write_labels(p.labels_moving, prefix + "_moving_labels.nii")
    nifti.write_warp(p.true_warp, prefix + "_true_warp")
    sys.stdout.write(f"wrote {prefix}_{{fixed,moving,fixed_labels,moving_labels}}.nii and "
                     f"{prefix}_true_warp.{{raw,json}}\n")
    return 0


def run_info(path: str) -> int:
    """run_info (main.cpp:358-370)."""
    from .nifti import read_nifti
    nv = read_nifti(path)
    nz, ny, nx = nv.volume.shape
    h = nv.header
    g = lambda v: "%g" % v  # ostream default formatting
    sys.stdout.write(f"dims: {nx} x {ny} x {nz}\n"
                     f"spacing: {g(nv.spacing[0])} {g(nv.spacing[1])} {g(nv.spacing[2])}\n"
                     f"datatype: {h.datatype} (bitpix {h.bitpix})\n"
                     f"endianness: {'big' if h.big_endian else 'little'}\n"
                     f"scl_slope/inter: {g(h.scl_slope)} / {g(h.scl_inter)}\n")
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    """main (main.cpp:372-496), with its exit-code mapping."""
    from . import nifti
    args = list(sys.argv[1:] if argv is None else argv)
    try:
        args = expand_register_config(args)
    except (ConfigError, nifti.IoError, ValueError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 1
    parser = _build_parser()
    try:
        ns = parser.parse_args(args)
    except ConfigError as e:
        print(str(e), file=sys.stderr)
        return 1
    except SystemExit as e:  # --help
        return int(e.code or 0)
    if ns.command is None:
        print("A subcommand is required", file=sys.stderr)
        return 1
    own = []
    try:
        return _dispatch(ns, own)
    finally:
        if own:  # the process group this call created (torchrun)
            import torch.distributed as dist
            dist.destroy_process_group()


def _dispatch(ns, own: list) -> int:
    from . import nifti
    from ._lib import InvalidArgument
    try:
        if ns.command == "register":
            world = int(os.environ.get("WORLD_SIZE", "1"))
            if world > 1:
                import torch
                import torch.distributed as dist
                if not dist.is_initialized():
                    if torch.cuda.is_available():  # several ranks may share one GPU (gloo staging)
                        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
                    dist.init_process_group(os.environ.get("FFDP_DIST_BACKEND", "nccl"))
                    own.append(True)
            return run_register(ns)
        if ns.command == "metrics":
            return run_metrics(ns.a, ns.b, ns.spacing, ns.out)
        if ns.command == "synth":
            return run_synth(ns.seed, ns.dims, ns.labels, ns.max_disp, ns.out)
        return run_info(ns.in_path)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 1
    except nifti.FormatError as e:
        print(f"format error: {e}", file=sys.stderr)
        return 2
    except nifti.IoError as e:
        print(f"i/o error: {e}", file=sys.stderr)
        return 2
    except InvalidArgument as e:
        print(f"config error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # noqa: BLE001 (main.cpp:490-493)
        from .registration import NumericalError
        if isinstance(e, NumericalError):
            print(f"numerical abort: {e}", file=sys.stderr)
            return 3
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
