"""The full-size checkers (oracle/ffdp_oracle_big.c) against the whole-volume oracle.

The GPU tests at BASELINE configs[2] / configs[4] (tests/test_gpu_fullsize.py) compare
the CUDA step with these per-voxel / OpenMP restatements because the whole-volume oracle
is too slow there; here they are pinned to that oracle (itself pinned to the reference,
tests/test_oracle_golden.py) on small lattices."""
import numpy as np
import pytest

from oracle import step_inputs


@pytest.fixture(scope="module")
def lncc_case(orc):
    si = step_inputs(orc, (18, 21, 23), seed=4242, loss="lncc")
    return si, orc.step_lncc(si.f, si.m, si.u, si.A, si.t)


@pytest.fixture(scope="module")
def mi_case(orc):
    si = step_inputs(orc, (16, 17, 19), seed=4243, loss="mi")
    return si, orc.step_mi(si.f, si.m, si.u, orc.parzen("bspline3", 32), si.A, si.t)


def test_lncc_sum_n_matches_oracle(orc, lncc_case):
    si, ref = lncc_case
    s = orc.lncc_sum_n_f32(si.f, si.m, si.u, si.A, si.t)
    loss = 1.0 - s / si.f.size
    assert loss == pytest.approx(ref["loss"], rel=1e-12, abs=1e-14)


def test_lncc_voxels_match_oracle(orc, lncc_case):
    si, ref = lncc_case
    vox = np.arange(si.f.size)  # every voxel, borders included
    r = orc.lncc_ants_voxels_f32(si.f, si.m, si.u, vox, si.A, si.t)
    np.testing.assert_allclose(r["grad_moved"], ref["grad_moved"].ravel(), rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(r["g_u"], ref["g_u"].reshape(-1, 3), rtol=1e-10, atol=1e-15)
    assert 1.0 - r["n"].sum() / si.f.size == pytest.approx(ref["loss"], rel=1e-12)


def test_mi_hist_and_voxels_match_oracle(orc, mi_case):
    si, ref = mi_case
    k = orc.parzen("bspline3", 32)
    raw = orc.mi_hist_f32(si.f, si.m, si.u, k, si.A, si.t)
    np.testing.assert_allclose(raw, ref["raw"], rtol=1e-11, atol=1e-12)
    mi, gh = orc.mi_table(raw, 32)
    assert -mi == pytest.approx(ref["loss"], rel=1e-11)
    vox = np.arange(si.f.size)
    r = orc.mi_voxels_f32(si.f, si.m, si.u, k, gh, vox, si.A, si.t)
    scale = np.max(np.abs(ref["g_u"]))
    assert np.max(np.abs(r["g_u"] - ref["g_u"].reshape(-1, 3))) <= 1e-10 * scale
