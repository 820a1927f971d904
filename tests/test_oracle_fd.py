"""Finite-difference checks of the oracle's backward passes (CPU, fp64): the standing
B-spline MI gradient check SURVEY.md 8(c) asks for (the reference's own FD tests use
the Gaussian kernel only, test_mi.cpp:272-306), and the patterns of test_lncc.cpp:100-137
(exact LNCC backward) and test_sampler.cpp:176-221 (sampler backward w.r.t. u). The
oracle is pinned to the reference by tests/test_oracle_golden.py; these pin the
gradients to the losses themselves."""
import numpy as np
import pytest


def _fd_idx(rng, n, k=24):
    return rng.choice(n, size=min(k, n), replace=False)


@pytest.mark.parametrize("bins", [8, 32])
def test_mi_bspline_backward_fd(orc, bins):
    """d MI / d J by central differences (step 1e-6) on a 6^3 pair kept a margin inside
    [0, 1] (test_mi.cpp:56-69): max |FD - analytic| <= 1e-6 of max |g|."""
    rng = np.random.default_rng(bins)
    vi = rng.uniform(0.1, 0.9, (6, 6, 6))
    vj = np.clip(0.6 * vi + 0.4 * rng.uniform(0.1, 0.9, vi.shape), 0.05, 0.95)
    k = orc.parzen("bspline3", bins)
    fwd = orc.mi_forward(vi, vj, k)
    _, gj, _ = orc.mi_backward(1.0, vi, vj, k, fwd)
    h = 1e-6
    flat = vj.ravel()
    errs = []
    for i in _fd_idx(rng, flat.size):
        a, b = flat.copy(), flat.copy()
        a[i] += h
        b[i] -= h
        fd = (orc.mi_forward(vi, a.reshape(vj.shape), k)["mi"] - orc.mi_forward(vi, b.reshape(vj.shape), k)["mi"]) / (2 * h)
        errs.append(abs(fd - gj.ravel()[i]))
    assert max(errs) <= 1e-6 * np.max(np.abs(gj))


def test_lncc_exact_backward_fd(orc):
    """d loss / d M of the exact LNCC backward (lncc.hpp:226-280), window 3 and 7."""
    rng = np.random.default_rng(7)
    f = rng.uniform(0, 1, (7, 8, 9))
    m = np.clip(0.5 * f + 0.5 * rng.uniform(0, 1, f.shape), 0, 1)
    for window in (3, 7):
        loss, state, _ = orc.lncc_forward(f, m, window)
        _, gm, _ = orc.lncc_backward(1.0, state, f, m, window, ants=False)
        h = 1e-6
        flat = m.ravel()
        errs = []
        for i in _fd_idx(rng, flat.size):
            a, b = flat.copy(), flat.copy()
            a[i] += h
            b[i] -= h
            fd = (orc.lncc_forward(f, a.reshape(m.shape), window)[0] - orc.lncc_forward(f, b.reshape(m.shape), window)[0]) \
                / (2 * h)
            errs.append(abs(fd - gm.ravel()[i]))
        assert max(errs) <= 1e-6 * np.max(np.abs(gm)), window


def test_sampler_backward_fd(orc):
    """d (sum up * sample) / d u, dA, dt (sampler.hpp:165-243) by central differences."""
    rng = np.random.default_rng(11)
    img = rng.uniform(0, 1, (6, 7, 8))
    u = rng.uniform(-0.05, 0.05, (6, 7, 8, 3))
    A = np.eye(3) + rng.uniform(-0.03, 0.03, (3, 3))
    t = rng.uniform(-0.03, 0.03, 3)
    up = rng.uniform(-1, 1, (6, 7, 8))
    bw = orc.sample(img, u, A, t, upstream=up, want=("warp", "affine", "translation"))
    L = lambda uu, AA, tt: float(np.sum(up * orc.sample(img, uu, AA, tt)["out"]))
    h = 1e-7
    flat = u.ravel()
    for i in _fd_idx(rng, flat.size):
        a, b = flat.copy(), flat.copy()
        a[i] += h
        b[i] -= h
        fd = (L(a.reshape(u.shape), A, t) - L(b.reshape(u.shape), A, t)) / (2 * h)
        assert abs(fd - bw["warp"].ravel()[i]) <= 1e-5 * np.max(np.abs(bw["warp"])) + 1e-7
    for r in range(3):
        for c in range(3):
            a, b = A.copy(), A.copy()
            a[r, c] += h
            b[r, c] -= h
            fd = (L(u, a, t) - L(u, b, t)) / (2 * h)
            assert abs(fd - bw["affine"][r, c]) <= 1e-5 * max(1.0, np.max(np.abs(bw["affine"])))
        a, b = t.copy(), t.copy()
        a[r] += h
        b[r] -= h
        fd = (L(u, A, a) - L(u, A, b)) / (2 * h)
        assert abs(fd - bw["translation"][r]) <= 1e-5 * max(1.0, np.max(np.abs(bw["translation"])))
