// step_lncc.cu -- C ABI of the fused warp + LNCC(ANTs) step (ffdp_step_lncc).
//
// Reference sequence replaced (registration.hpp:277-312): ring_sample (distops.hpp:144)
// -> dist_lncc(ants_approx) (distops.hpp:285-352) -> ring_sample_backward(want warp)
// (distops.hpp:179-248). The kernel is the one-pass k_lncc_fused (step_lncc3.cu); the
// earlier two-pass form (warp pass + moments pass through an HBM workspace,
// step_lncc2.cu) stays reachable through ffdp_step_lncc_passes for comparison.
#include <algorithm>

#include "ffdp_common.cuh"

using namespace ffdp;

namespace ffdp {
int64_t lncc2_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s);
int lncc2_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, float shift_f, float shift_m, float* g_u,
               double* sum_n, int32_t* miss, void* workspace, int passes, cudaStream_t st);
int64_t lncc3_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s);
int lncc3_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, const float* ranges, float* g_u, double* sum_n,
               int32_t* miss, void* workspace, cudaStream_t st);
}  // namespace ffdp

static constexpr int R = 3, WIN = 7;

extern "C" int64_t ffdp_step_lncc_workspace_bytes(ffdp_dims d, ffdp_slab s) { return lncc3_workspace_bytes(d, s); }
extern "C" int64_t ffdp_step_lncc_passes_workspace_bytes(ffdp_dims d, ffdp_slab s) {
    return lncc2_workspace_bytes(d, s);
}

// the argument checks of dist_lncc / lncc_forward_fused / fused_sample (lncc.hpp:57-61,
// distops.hpp:285-300, sampler.hpp:45-52) for the fused step
static int check_step_args(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                           const ffdp_sampler_args* args, int window, const float* g_u) {
    if (window != WIN) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the fused kernel is built for window %d", WIN);
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !g_u || !m.data) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: null pointer");
    if (d.nx < 1 || d.ny < 1 || d.nz < 1 || s.buf_nz != d.nz || s.z_begin < s.buf_z0 || s.z_end > s.buf_z0 + s.buf_nz ||
        s.z_begin >= s.z_end || s.buf_z0 < 0 || s.buf_z0 + s.buf_nz > s.nz_global)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: inconsistent slab");
    const int64_t need_lo = std::max<int64_t>(0, s.z_begin - R), need_hi = std::min<int64_t>(s.nz_global, s.z_end + R);
    if (s.buf_z0 > need_lo || s.buf_z0 + s.buf_nz < need_hi)
        return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: buffer lacks the %d halo planes the window needs", R);
    if (m.z_begin < 0 || m.z_end > m.dims.nz || m.z_begin >= m.z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: bad moving window");
    if (m.pad != 2)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the moving image must be zero-bordered (pad = 2, "
                                                "ffdp_pad_window)");
    // 32-bit in-plane offsets, 16-bit tile coordinates
    if (d.nx >= 32000 || d.ny >= 32000 || 3 * d.nx * d.ny >= (1LL << 31) || s.nz_global >= (1 << 30))
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: lattice too large for the fused kernel");
    return FFDP_OK;
}

extern "C" int ffdp_step_lncc(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                              const ffdp_sampler_args* args, int window, double eps, double gi, const float* ranges,
                              float* g_u, double* sum_n, int32_t* miss, void* workspace, void* stream) {
    int rc = check_step_args(f, u, d, s, m, args, window, g_u);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void* ws = workspace;
    if (!ws) {
        ws = scratch_alloc((size_t)lncc3_workspace_bytes(d, s), st);
        if (!ws) return set_error(FFDP_CUDA, "step_lncc: scratch allocation failed");
    }
    rc = lncc3_step(f, u, d, s, m, *args, eps, gi, ranges, g_u, sum_n, miss, ws, st);
    if (!workspace) scratch_free(ws, st);
    return rc;
}

extern "C" int ffdp_step_lncc_passes(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                                     const ffdp_sampler_args* args, int window, double eps, double gi, float shift_f,
                                     float shift_m, float* g_u, double* sum_n, int32_t* miss, void* workspace,
                                     int passes, void* stream) {
    int rc = check_step_args(f, u, d, s, m, args, window, g_u);
    if (rc) return rc;
    if (!workspace) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the two-pass step needs its workspace");
    if (passes < 1 || passes > 3) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: passes must be 1, 2 or 3");
    return lncc2_step(f, u, d, s, m, *args, eps, gi, shift_f, shift_m, g_u, sum_n, miss, workspace, passes,
                      (cudaStream_t)stream);
}
