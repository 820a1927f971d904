"""The `voxreg` command line (paper_2509_25044_b200/cli.py vs tools/main.cpp) and the label
evaluation it reports (metrics.py vs metrics.hpp / sampler.hpp:331-365, pinned by the
reference's own outputs in tests/golden). CPU only: `register` runs with the GPU pieces
replaced, the real GPU run is tests/test_gpu_cli.py."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2509_25044_b200 import cli, metrics as MT, nifti, registration as R, synth


def run(capsys, *argv):
    code = cli.main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


# ---------------------------------------------------------------- label evaluation
def test_label_metrics_match_reference(golden):
    g = golden
    w = MT.warp_labels_nn(g["lab_b"], g["lab_u"], g["lab_A"], g["lab_t"])
    assert np.array_equal(w, g["lab_warped"])
    a, b = g["lab_a"], g["lab_b"]
    assert (MT.dice(a, b)[1], MT.inv_dice(a, b), MT.hd90_cumulative(a, b)) == tuple(g["lab_metrics"])
    sp = (0.7, 1.3, 2.1)
    assert (MT.dice(a, w)[1], MT.inv_dice(a, w), MT.hd90_cumulative(a, w, sp)) == tuple(g["lab_metrics_sp"])


def test_label_metrics_rejects():
    a = np.zeros((3, 4, 5), np.uint16)
    with pytest.raises(ValueError):
        MT.hd90_cumulative(a, a)  # both masks empty (metrics.hpp:186)
    with pytest.raises(ValueError):
        MT.inv_dice(a, a)  # no weighted labels (metrics.hpp:84)
    b = a.copy()
    b[1, 1, 1] = 2
    c = a.copy()
    c[1, 1, 1] = 3
    with pytest.raises(ValueError):
        MT.hd90_cumulative(b, c)  # a label missing in one mask
    with pytest.raises(ValueError):
        MT.dice(a, np.zeros((3, 4, 6), np.uint16))
    assert MT.dice(a, a) == ({}, 0.0)
    assert MT.dice(b, b)[1] == 1.0 and MT.inv_dice(b, b) == 1.0 and MT.hd90_cumulative(b, b) == 0.0


# ---------------------------------------------------------------- config files
def test_config_expansion(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# a comment\n\n  loss = mi   # trailing\nbins=16\r\nants-approx = false\nskip-affine = no\n"
                 "emit-timings =\nlr = 0.25\ngp-sync=off\n")
    args = cli.expand_register_config(["register", "--config", str(p), "--lr", "0.75"])
    # spliced in right after the subcommand; the explicit --lr wins
    assert args == ["register", "--loss", "mi", "--bins", "16", "--no-ants-approx", "--emit-timings", "--no-gp-sync",
                    "--lr", "0.75"]
    args = cli.expand_register_config(["register", f"--config={p}", "--no-ants-approx"])
    assert "--ants-approx" not in args and args.count("--no-ants-approx") == 1
    assert cli.expand_register_config(["info", "--config", str(p)]) == ["info", "--config", str(p)]


@pytest.mark.parametrize("body, msg", [("loss mi\n", "config line 1: expected key=value"),
                                       ("# x\nlosss = mi\n", "config line 2: unknown key 'losss'"),
                                       ("config = other\n", "unknown key 'config'")])
def test_config_errors_exit_1(tmp_path, capsys, body, msg):
    p = tmp_path / "bad.cfg"
    p.write_text(body)
    code, _, err = run(capsys, "register", "--config", str(p), "--fixed", "a", "--moving", "b", "--out", "o")
    assert code == 1 and err.startswith("config error: ") and msg in err


def test_config_missing_file_exit_1(tmp_path, capsys):
    code, _, err = run(capsys, "register", "--config", str(tmp_path / "none.cfg"))
    assert code == 1 and "cannot open config file" in err  # main.cpp:425-428: config errors are code 1


# ---------------------------------------------------------------- parsing / exit codes
@pytest.mark.parametrize("argv", [[], ["register", "--fixed", "a"], ["register", "--fixed", "a", "--moving", "b",
                                                                      "--out", "o", "--loss", "ncc"],
                                  ["register", "--fixed", "a", "--moving", "b", "--out", "o", "--window", "7.5"],
                                  ["frobnicate"], ["synth", "--dims", "1,2", "--out", "x"],
                                  ["synth", "--dims", "8", "--out", "x"], ["synth", "--labels", "0", "--out", "x"],
                                  ["synth", "--max-disp", "0.2", "--out", "x"], ["synth", "--seed", "1"]])
def test_parse_errors_exit_1(capsys, argv):
    assert run(capsys, *argv)[0] == 1


def test_help_exit_0(capsys):
    code, out, _ = run(capsys, "register", "--help")
    assert code == 0 and "--sigma-grad" in out and "--no-gp-sync" in out


def test_info(capsys):
    d = os.path.join(os.path.dirname(__file__), "golden", "nifti")
    code, out, _ = run(capsys, "info", "--in", os.path.join(d, "labels.nii"))
    assert code == 0
    assert out == ("dims: 6 x 3 x 4\nspacing: 0.7 1.1 2.5\ndatatype: 4 (bitpix 16)\nendianness: little\n"
                   "scl_slope/inter: 0 / 0\n")
    code, out, _ = run(capsys, "info", "--in", os.path.join(d, "vol_be.nii"))
    assert code == 0 and "endianness: big" in out


def test_io_and_format_errors_exit_2(tmp_path, capsys):
    code, _, err = run(capsys, "info", "--in", str(tmp_path / "missing.nii"))
    assert code == 2 and err.startswith("i/o error: ")
    bad = tmp_path / "bad.nii"
    bad.write_bytes(b"\0" * 400)
    code, _, err = run(capsys, "info", "--in", str(bad))
    assert code == 2 and err.startswith("format error: ")
    code, _, err = run(capsys, "register", "--fixed", str(bad), "--moving", str(bad), "--out", str(tmp_path / "o"))
    assert code == 2


def test_metrics_subcommand(golden, tmp_path, capsys):
    a, b = golden["lab_a"], golden["lab_b"]
    pa, pb = str(tmp_path / "a.nii"), str(tmp_path / "b.nii")
    nifti.write_labels(a, pa)
    nifti.write_labels(b, pb)
    out_json = str(tmp_path / "m.json")
    code, out, _ = run(capsys, "metrics", "--a", pa, "--b", pb, "--out", out_json)
    assert code == 0
    d = json.loads(out)
    assert list(d) == ["dice", "inv_dice", "hd90"]
    assert (d["dice"], d["inv_dice"], d["hd90"]) == tuple(golden["lab_metrics"])
    assert open(out_json).read() == out
    code, out, _ = run(capsys, "metrics", "--a", pa, "--b", pb, "--spacing", "1,2")
    assert code == 1


# ---------------------------------------------------------------- register (GPU pieces replaced)
@pytest.fixture
def pair(tmp_path):
    rng = np.random.default_rng(3)
    f = rng.uniform(0, 1, (6, 7, 8))
    m = rng.uniform(0, 1, (6, 7, 8))
    pf, pm = str(tmp_path / "f.nii"), str(tmp_path / "m.nii")
    nifti.write_nifti(f, pf, spacing=(0.5, 0.75, 2.0), origin=(1.0, 2.0, 3.0))
    nifti.write_nifti(m, pm)
    return pf, pm, str(tmp_path / "run")


def test_register_numerical_abort_exit_3(pair, capsys, monkeypatch):
    pf, pm, out = pair
    monkeypatch.setattr(cli, "_device", lambda: torch.device("cpu"))

    def boom(fixed, moving, cfg):
        raise R.NumericalError("deformable stage diverged (non-finite loss)",
                               [R.TraceEntry(0, 0, 0.5), R.TraceEntry(0, 1, float("nan"))])
    monkeypatch.setattr(R, "register_volumes", boom)
    code, _, err = run(capsys, "register", "--fixed", pf, "--moving", pm, "--out", out)
    assert code == 3 and "numerical abort" in err and "(trace flushed)" in err
    assert open(out + "_trace.csv").read() == "scale_index,iteration,loss\n0,0,0.5\n0,1,nan\n"


def test_register_outputs(pair, capsys, monkeypatch):
    """Output files, summary keys in the reference's order (main.cpp:278-300) and the
    schedule / loss the options build."""
    pf, pm, out = pair
    from paper_2509_25044_b200 import voxreg as V
    monkeypatch.setattr(cli, "_device", lambda: torch.device("cpu"))
    seen = {}
    warp = torch.full((6, 7, 8, 3), 0.125)
    A, t = np.eye(3) * 1.5, np.array([0.1, 0.2, 0.3])

    def fake_register(fixed, moving, cfg):
        seen["cfg"] = cfg
        return R.RegistrationResult((A, t), warp, [R.TraceEntry(0, 0, 0.75), R.TraceEntry(2, 0, 0.1)], 1.5, 0.875)
    monkeypatch.setattr(R, "register_volumes", fake_register)
    monkeypatch.setattr(V, "fused_sample", lambda img, u, args: img * 2.0)
    code, text, _ = run(capsys, "register", "--fixed", pf, "--moving", pm, "--out", out, "--loss", "mi",
                        "--mi-kernel", "bspline", "--scales", "2,1", "--iters", "5,3", "--affine-scales", "2",
                        "--affine-iters", "4", "--seed", "9", "--emit-timings")
    assert code == 0
    cfg = seen["cfg"]
    assert [(s.downsample, s.iterations) for s in cfg.deformable.steps] == [(2.0, 5), (1.0, 3)]
    assert cfg.deformable.loss.kind == "mi" and cfg.deformable.loss.mi_bspline_kernel
    assert cfg.affine.loss.kind == "mi" and [(s.downsample, s.iterations) for s in cfg.affine.steps] == [(2.0, 4)]
    s = json.loads(open(out + "_summary.json").read())
    assert text == open(out + "_summary.json").read()
    assert list(s) == ["config", "affine_matrix", "affine_translation", "final_loss", "iterations",
                       "peak_alloc_bytes", "jacobian_positive_fraction", "seconds"]
    assert list(s["config"])[:3] == ["fixed", "moving", "out_prefix"] and s["config"]["seed"] == 9
    assert s["affine_matrix"] == list((np.eye(3) * 1.5).reshape(9)) and s["affine_translation"] == [0.1, 0.2, 0.3]
    assert s["final_loss"] == 0.1 and s["iterations"] == 2 and s["jacobian_positive_fraction"] == 0.875
    assert open(out + "_trace.csv").read() == "scale_index,iteration,loss\n0,0,0.75\n2,0,0.10000000000000001\n"
    w = nifti.read_warp(out + "_warp")
    assert w.shape == (6, 7, 8, 3) and np.all(w == 0.125)
    meta = json.load(open(out + "_warp.json"))
    assert meta["spacing"] == [0.5, 0.75, 2.0] and meta["origin"] == [1.0, 2.0, 3.0]
    moved = nifti.read_nifti(out + "_moved.nii")
    assert moved.header.datatype == 64 and moved.spacing == (0.5, 0.75, 2.0)
    m_in = nifti.read_nifti(pm).volume
    assert np.array_equal(moved.volume, (m_in.astype(np.float32) * 2.0).astype(np.float64))


def test_register_config_errors(pair, capsys, monkeypatch):
    pf, pm, out = pair
    monkeypatch.setattr(cli, "_device", lambda: torch.device("cpu"))
    base = ["register", "--fixed", pf, "--moving", pm, "--out", out]
    assert run(capsys, *base, "--scales", "4,2", "--iters", "1")[0] == 1      # lengths differ
    assert run(capsys, *base, "--scales", "1,2", "--iters", "1,1")[0] == 1    # validate(): non-increasing
    assert run(capsys, *base, "--scales", "x", "--iters", "1")[0] == 1        # stod
    assert run(capsys, *base, "--shards", "0")[0] == 1
    assert run(capsys, *base, "--shards", "2", "--lncc-backend", "naive")[0] == 1


# ---------------------------------------------------------------- synth (synth.hpp, main.cpp:326-356)
def test_synth_pair_matches_reference(golden):
    p = synth.synth_pair(4242, (16, 17, 18), 5, 0.12)
    for mine, key in ((p.fixed, "synth_f"), (p.moving, "synth_m"), (p.true_warp, "synth_w"),
                      (p.labels_fixed, "synth_lf"), (p.labels_moving, "synth_lm"), (p.pre_blur_fixed, "synth_pre")):
        assert np.array_equal(mine, golden[key]), key


def test_synth_subcommand(golden, tmp_path, capsys):
    pre = str(tmp_path / "pair")
    code, out, _ = run(capsys, "synth", "--seed", "4242", "--dims", "18,17,16", "--labels", "5", "--max-disp", "0.12",
                       "--out", pre)
    assert code == 0 and out.startswith("wrote ")
    f, m = nifti.read_nifti(pre + "_fixed.nii"), nifti.read_nifti(pre + "_moving.nii")
    assert f.header.datatype == 64 and np.array_equal(f.volume, golden["synth_f"])
    assert np.array_equal(m.volume, golden["synth_m"])
    assert np.array_equal(nifti.nifti_to_labels(nifti.read_nifti(pre + "_fixed_labels.nii")), golden["synth_lf"])
    assert np.array_equal(nifti.nifti_to_labels(nifti.read_nifti(pre + "_moving_labels.nii")), golden["synth_lm"])
    assert np.array_equal(nifti.read_warp(pre + "_true_warp"), golden["synth_w"])
