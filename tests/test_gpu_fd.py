"""Directional finite differences of the GPU steps (g_u is the gradient of the loss they
report): (L(u + v) - L(u - v)) / 2 against <g_u, v> for a
smooth direction v of a few hundredths of a voxel, on the survey's synthetic pair
(SURVEY.md 8(d)); fp32 storage, so the tolerance is 5% (the trilinear
interpolant is piecewise linear: voxels whose samples cross a cell face in +-v bend the
difference). MI runs the fused B-spline step; LNCC runs the exact backward (the
operator composition): the fused LNCC step implements the ANTs backward, which by design
drops the window terms of the gradient (lncc.hpp:265-278) and is not the loss's gradient."""
import numpy as np
import pytest

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("loss", ["lncc", "mi"])
def test_fused_step_directional_fd(orc, loss):
    need_gpu()
    import torch
    from oracle import step_inputs
    from paper_2509_25044_b200 import voxreg as V
    si = step_inputs(orc, (40, 44, 48), seed=4242, loss=loss)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    f, m, u = T(si.f), T(si.m), T(si.u)
    p = V.LossParams(kind=loss, mi_bspline_kernel=True, ants_approx=False)
    step = lambda uu: V.warp_loss_step(f, m, uu, si.A, si.t, p)
    r = step(u)
    g = r.g_u.double().clone()
    gen = torch.Generator(device="cuda").manual_seed(5)
    v = torch.randn(u.shape, device="cuda", generator=gen)
    v = V.gp_convolve(v.contiguous(), V.gaussian_taps(2.0), "renormalize")
    results = []
    for vox in (0.01, 0.03):
        d = v / v.abs().max() * (vox * 2.0 / (min(u.shape[:3]) - 1))
        fd = (step((u + d).contiguous()).loss - step((u - d).contiguous()).loss) / 2.0
        an = float((g * d.double()).sum())
        results.append((vox, fd, an))
        assert an != 0.0
        assert abs(fd - an) <= 5e-2 * abs(an), results
