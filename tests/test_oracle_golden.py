"""Pins the C restatement (oracle/ffdp_oracle.c) against golden vectors produced by the
reference itself (tests/golden/make_golden.py over oracle/_ref). CPU only."""
import numpy as np
import pytest

from oracle import step_inputs


def close(a, b, tol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.max(np.abs(a - b), initial=0.0) <= tol * max(1.0, np.max(np.abs(b), initial=0.0))


@pytest.mark.parametrize("i", [0, 1, 2])
def test_sampler_margin_fixtures(orc, golden, i):
    g = lambda k: golden[f"smp{i}_{k}"]
    fw = orc.sample(g("img"), g("u"), g("A"), g("t"), g("S"))
    close(fw["out"], g("out"))
    bw = orc.sample(g("img"), g("u"), g("A"), g("t"), g("S"), upstream=g("up"),
                    want=("image", "warp", "affine", "translation"))
    close(bw["image"], g("gimg"))
    close(bw["warp"], g("gu"))
    close(bw["affine"], g("gA"))
    close(bw["translation"], g("gt"))


def test_sampler_face_and_bounds(orc, golden):
    bw = orc.sample(golden["face_img"], golden["face_u"], upstream=golden["face_up"], want=("warp",))
    close(bw["warp"], golden["face_gu"])
    img = golden["face_img"]
    # floor cell at a face: one-sided slope (test_sampler.cpp:225-241)
    assert bw["warp"][2, 2, 2, 0] == pytest.approx((img[2, 2, 4] - img[2, 2, 3]) * 2.5, abs=1e-12)
    fw = orc.sample(golden["bnd_img"], golden["bnd_u"], bounds=golden["bnd_bounds"])
    close(fw["out"], golden["bnd_out"])


def test_sampler_rejects_bad_args(orc):
    with pytest.raises(ValueError):
        orc.sample(np.zeros((4, 4, 4)), np.zeros((4, 4, 4, 3)), S=[0.0, 1, 1])


@pytest.mark.parametrize("i", [0, 1, 2])
def test_lncc(orc, golden, i):
    g = lambda k: golden[f"lncc{i}_{k}"]
    w = int(g("w"))
    loss, state, mp = orc.lncc_forward(g("f"), g("m"), window=w, eps=1e-5, want_map=True)
    close(state, g("state"))
    close(mp, g("map"))
    for mode in ("ants", "exact"):
        assert loss == pytest.approx(float(golden[f"lncc{i}_{mode}_loss"]), rel=1e-12)
        gf, gm, _ = orc.lncc_backward(1.3, state, g("f"), g("m"), window=w, eps=1e-5, ants=(mode == "ants"))
        close(gf, golden[f"lncc{i}_{mode}_gf"])
        close(gm, golden[f"lncc{i}_{mode}_gm"])


@pytest.mark.parametrize("kind", ["gaussian", "bspline3", "delta"])
@pytest.mark.parametrize("bins", [8, 32])
@pytest.mark.parametrize("approx", [False, True])
def test_mi(orc, golden, kind, bins, approx):
    k = orc.parzen(kind, bins)
    key = f"mi_{kind}_{bins}_{int(approx)}"
    h = orc.mi_forward(golden["mi_i"], golden["mi_j"], k, approx=approx)
    assert h["mi"] == pytest.approx(float(golden[f"{key}_mi"]), rel=1e-12, abs=1e-15)
    close(h["raw"], golden[f"{key}_raw"])
    b = bins
    close(np.concatenate([h["p_ij"].ravel(), h["p_i"], h["p_j"]]), golden[f"{key}_pij"])
    assert tuple(int(s) for s in h["stats"]) == tuple(int(s) for s in golden[f"{key}_stats"])
    if not approx:
        gi, gj, _ = orc.mi_backward(-1.0, golden["mi_i"], golden["mi_j"], k, h)
        close(gi, golden[f"{key}_gi"])
        close(gj, golden[f"{key}_gj"])
    assert b == bins


@pytest.mark.parametrize("kind", ["gaussian", "bspline3", "delta"])
def test_parzen(orc, golden, kind):
    k = orc.parzen(kind, 32)
    xs = golden["parzen_x"]
    kap = np.array([orc.lib.or_parzen_kappa(k, float(x)) for x in xs])
    om = np.array([orc.lib.or_parzen_omega(k, float(x)) for x in xs])
    close(kap, golden[f"parzen_{kind}_kappa"])
    close(om, golden[f"parzen_{kind}_omega"])


def test_synth_pair_bit_identical(orc, golden):
    f, m, w = orc.synth_pair(4242, (16, 17, 18), 5, 0.12)
    assert np.array_equal(f, golden["synth_f"])
    assert np.array_equal(m, golden["synth_m"])
    assert np.array_equal(w, golden["synth_w"])


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_step_h1_and_shard_invariance(orc, golden, loss):
    si = step_inputs(orc, (18, 17, 16), seed=4242, loss=loss)
    for k in ("f", "m", "u", "A", "t"):
        assert np.array_equal(getattr(si, k), golden[f"step_{loss}_{k}"])
    if loss == "lncc":
        res = orc.step_lncc(si.f, si.m, si.u, si.A, si.t)
    else:
        res = orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)
    for world in (1, 2, 3):
        ref_loss = float(golden[f"step_{loss}_H{world}_loss"])
        assert res["loss"] == pytest.approx(ref_loss, rel=1e-10)
        close(res["g_u"], golden[f"step_{loss}_H{world}_gu"], tol=1e-8)
        close(res["moved"], golden[f"step_{loss}_H{world}_moved"], tol=1e-9)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_ring_sample_partials_sum_to_global(orc, golden, world):
    """distops.hpp:144-248: per-shard zero-padded partial interpolations sum to the
    global interpolation (restated single-process)."""
    si = step_inputs(orc, (18, 17, 16), seed=4242, loss="lncc")
    nz = si.f.shape[0]
    out = []
    for r in range(world):
        lo, hi = orc.shard_range(nz, world, r)
        ax = lambda i: -1.0 + 2.0 * (i / (nz - 1))
        bounds = [-1, -1, ax(lo), 1, 1, ax(hi - 1)]
        out.append(orc.ring_sample(si.m, world, si.u[lo:hi], bounds, si.A, si.t))
    close(np.concatenate(out, axis=0), golden[f"step_lncc_H{world}_moved"], tol=1e-9)


def test_shard_ranges(orc):
    assert [orc.shard_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        orc.shard_range(2, 3, 0)


@pytest.mark.parametrize("world", [1, 3])
def test_warp_update(orc, golden, world):
    """registration.hpp:313-317: gp_convolve(g_u, gaussian 1.0, renormalize) -> adam_step
    (adam.hpp:30-50) -> gp_convolve(u, gaussian 0.5, renormalize), two Adam steps; the
    sharded reference (halo exchange) equals the single-rank restatement."""
    g, u = golden["wu_g"], golden["wu_u"]
    z = np.zeros_like(u)
    u1, a1, b1 = orc.warp_update(g, u, z, z, 0.01, 1)
    close(u1, golden[f"wu_H{world}_u1"], tol=1e-14)
    close(a1, golden[f"wu_H{world}_m1"], tol=1e-14)
    close(b1, golden[f"wu_H{world}_v1"], tol=1e-14)
    u2, a2, b2 = orc.warp_update(0.5 * g, u1, a1, b1, 0.01, 2)
    close(u2, golden[f"wu_H{world}_u2"], tol=1e-14)
    close(a2, golden[f"wu_H{world}_m2"], tol=1e-14)
    close(b2, golden[f"wu_H{world}_v2"], tol=1e-14)


def test_resample_and_normalize(orc, golden):
    """resample_scale (anti-alias + trilinear, resample.hpp:48-103), resample_warp
    (108-146) and normalize_intensities (registration.hpp:100-115), bit for bit."""
    v = golden["rs_v"]
    for f in (0.5, 0.25, 0.37, 2.0):
        close(orc.resample_scale(v, f), golden[f"rs_scale_{f}"], tol=0.0)
    for sh in ((13, 17, 19), (4, 5, 6), (1, 9, 11)):
        close(orc.resample_warp(golden["rs_w"], sh), golden["rs_warp_" + "x".join(map(str, sh))], tol=0.0)
    close(orc.normalize(v), golden["rs_norm"], tol=0.0)


@pytest.mark.parametrize("loss", ["mse", "lncc", "mi"])
def test_affine_stage(orc, golden, loss):
    """affine_stage (registration.hpp:176-219): 12-parameter Adam over two scales."""
    si = step_inputs(orc, (18, 20, 22), seed=4242, loss="mi")
    A, t, tr = orc.affine_stage(si.f, si.m, [(2, 3), (1, 3)], lr=0.01, loss=loss)
    close(A, golden[f"aff_{loss}_A"], tol=1e-12)
    close(t, golden[f"aff_{loss}_t"], tol=1e-12)
    close(tr, golden[f"aff_{loss}_trace"], tol=1e-12)


@pytest.mark.parametrize("loss,kind", [("lncc", "gaussian"), ("mi", "bspline3"), ("mi", "gaussian")])
def test_deformable_stage(orc, golden, loss, kind):
    """deformable_stage (registration.hpp:230-331): the single-rank restatement equals the
    reference at H = 1 and H = 3 (ring sampler + halos + allreduces)."""
    si = step_inputs(orc, (18, 20, 22), seed=4242, loss=loss)
    w, tr = orc.deformable_stage(si.f, si.m, [(2, 3), (1, 3)], si.A, si.t, loss=loss, mi_kind=kind)
    for world in (1, 3):
        close(tr, golden[f"def_{loss}_{kind}_H{world}_trace"], tol=1e-9)
        close(w, golden[f"def_{loss}_{kind}_H{world}_warp"], tol=1e-8)


def test_jacobian_positive(orc, golden):
    assert orc.jacobian_positive(golden["jac_w"]) == float(golden["jac_frac"])
    assert 0.0 < float(golden["jac_frac"]) < 1.0
