"""`voxreg register` end to end on the GPU (cli.py over registration.register_volumes):
the files it writes equal the library call's results, the label block is filled, and
`--shards 2` -- under torch.distributed.run (gloo staging, two ranks on one GPU) and in
one process over ffdp_comm -- reproduces the one-shard warp to the sharded-stage
tolerances."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def files(tmp_path_factory, orc):
    need_gpu()
    from oracle import step_inputs
    from paper_2509_25044_b200 import nifti
    d = tmp_path_factory.mktemp("cli")
    si = step_inputs(orc, (18, 20, 22), seed=4242, loss="lncc")
    pf, pm = str(d / "f.nii"), str(d / "m.nii")
    nifti.write_nifti(si.f, pf, spacing=(1.0, 1.0, 1.5))
    nifti.write_nifti(si.m, pm, spacing=(1.0, 1.0, 1.5))
    lf = (si.f > 0.5).astype(np.uint16) + (si.f > 0.8).astype(np.uint16)
    lm = (si.m > 0.5).astype(np.uint16) + (si.m > 0.8).astype(np.uint16)
    plf, plm = str(d / "lf.nii"), str(d / "lm.nii")
    nifti.write_labels(lf, plf, spacing=(1.0, 1.0, 1.5))
    nifti.write_labels(lm, plm)
    return d, pf, pm, plf, plm


ARGS = ["--scales", "2,1", "--iters", "3,3", "--affine-scales", "2", "--affine-iters", "3", "--seed", "7"]


def test_register_matches_library(files, capsys):
    import torch
    from paper_2509_25044_b200 import cli, nifti, registration as R, voxreg as V
    d, pf, pm, plf, plm = files
    out = str(d / "run")
    code = cli.main(["register", "--fixed", pf, "--moving", pm, "--out", out, "--fixed-labels", plf,
                     "--moving-labels", plm] + ARGS)
    text = capsys.readouterr().out
    assert code == 0
    s = json.loads(text)
    assert s["iterations"] == 9 and s["config"]["seed"] == 7 and s["peak_alloc_bytes"] > 0
    assert set(s["metrics"]) == {"dice_before", "dice_after", "inv_dice_before", "inv_dice_after", "hd90_before",
                                 "hd90_after"}
    assert 0.0 < s["metrics"]["dice_after"] <= 1.0
    # the same registration through the library
    f = nifti.read_nifti(pf).to_device("cuda")
    m = nifti.read_nifti(pm).to_device("cuda")
    cfg = R.RegistrationConfig(
        affine=cli.build_schedule("2", "3", 0.01, 1.0, 0.5, V.LossParams(kind="mi")),
        deformable=cli.build_schedule("2,1", "3,3", 0.5, 1.0, 0.5, V.LossParams(kind="lncc")))
    res = R.register_volumes(f, m, cfg)
    w = nifti.read_warp(out + "_warp")
    assert np.array_equal(w, res.warp.double().cpu().numpy())
    assert s["final_loss"] == res.trace[-1].loss
    assert s["affine_matrix"] == [float(x) for x in np.asarray(res.affine[0]).reshape(9)]
    rows = open(out + "_trace.csv").read().splitlines()
    assert rows[0] == "scale_index,iteration,loss" and len(rows) == 10
    assert rows[-1] == "%d,%d,%.17g" % (res.trace[-1].scale_index, res.trace[-1].iteration, res.trace[-1].loss)
    moved = nifti.read_nifti(out + "_moved.nii")
    args = V.SamplerArgs(A=np.asarray(res.affine[0]), t=np.asarray(res.affine[1]))
    assert np.array_equal(moved.volume, V.fused_sample(m, res.warp, args).double().cpu().numpy())
    assert moved.spacing == (1.0, 1.0, 1.5)
    torch.cuda.synchronize()


def test_register_sharded_torchrun(files):
    from paper_2509_25044_b200 import nifti, voxreg as V
    from gpu_util import l2rel
    d, pf, pm, _, _ = files
    base = ["register", "--fixed", pf, "--moving", pm, "--skip-affine"] + ARGS
    one = subprocess.run([sys.executable, "-m", "paper_2509_25044_b200.cli"] + base + ["--out", str(d / "h1")],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr
    env = dict(os.environ, FFDP_DIST_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29533", "-m", "paper_2509_25044_b200.cli"]
                         + base + ["--out", str(d / "h2"), "--shards", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert two.returncode == 0, two.stderr[-2000:]
    w1, w2 = nifti.read_warp(str(d / "h1_warp")), nifti.read_warp(str(d / "h2_warp"))
    assert l2rel(w2, w1) <= 1e-3
    assert np.max(np.abs(w2 - w1)) <= 0.25 * V.deformable_lr_norm(w1.shape[:3], 0.5)
    s1, s2 = (json.load(open(str(d / f"{h}_summary.json"))) for h in ("h1", "h2"))
    assert s2["config"]["shards"] == 2 and s1["iterations"] == s2["iterations"] == 6
    assert abs(s2["final_loss"] - s1["final_loss"]) <= 1e-5 * abs(s1["final_loss"])
    # --shards 2 in ONE process (the reference's model): both ranks over ffdp_comm, here
    # sharing the GPU
    one2 = subprocess.run([sys.executable, "-m", "paper_2509_25044_b200.cli"] + base
                          + ["--out", str(d / "h3"), "--shards", "2"], cwd=ROOT, capture_output=True, text=True,
                          timeout=600)
    assert one2.returncode == 0, one2.stderr[-2000:]
    w3 = nifti.read_warp(str(d / "h3_warp"))
    assert l2rel(w3, w1) <= 1e-3
    assert np.max(np.abs(w3 - w1)) <= 0.25 * V.deformable_lr_norm(w1.shape[:3], 0.5)
    s3 = json.load(open(str(d / "h3_summary.json")))
    assert abs(s3["final_loss"] - s1["final_loss"]) <= 1e-5 * abs(s1["final_loss"])
    # a shard count that does not match the torch.distributed ranks is a configuration error
    bad = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29534", "-m", "paper_2509_25044_b200.cli"]
                         + base + ["--out", str(d / "h4"), "--shards", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert bad.returncode != 0 and "config error" in bad.stderr
