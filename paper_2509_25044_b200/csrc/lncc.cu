// lncc.cu -- LNCC operator API on the GPU (lncc.hpp:144-280, distops.hpp:285-352) and the
// generic separable convolution (smoothing.hpp:52-94).
//
// These are the standalone operators behind lncc_forward_fused / lncc_backward_fused /
// dist_lncc. They keep the five window moments in fp64 (exact fp32 products, fp64
// sums), so the cancellation in mean(FM) - mean(F)mean(M) costs no accuracy. The
// performance path of the deformable step is the single-pass fused kernel in
// step_lncc.cu; these operators serve the drop-in API and the exact (non-ANTs) mode.
#include <algorithm>

#include "ffdp_common.cuh"

namespace ffdp {

constexpr int kNT = 256;
constexpr int kMaxTaps = 63;

struct Taps {
    double w[kMaxTaps];
    int n;
    double full_sum;
};

// convolve_axis (smoothing.hpp:52-94) on a channel-interleaved fp32 block, fp64 accumulation.
__global__ void __launch_bounds__(kNT) k_conv_axis_f32(const float* __restrict__ in, float* __restrict__ out,
                                                        int64_t nx, int64_t ny, int64_t nz, int ch, int axis, Taps t,
                                                        int renorm, int64_t lo_global, int64_t n_global) {
    const int64_t n = nx * ny * nz * ch;
    const int r = t.n / 2;
    const int64_t n_axis = axis == 0 ? nx : axis == 1 ? ny : nz;
    const int64_t stride = axis == 0 ? ch : axis == 1 ? nx * ch : nx * ny * ch;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const int64_t vox = i / ch;
        const int64_t x = vox % nx, y = (vox / nx) % ny, z = vox / (nx * ny);
        const int64_t p = axis == 0 ? x : axis == 1 ? y : z;
        const int64_t gpos = lo_global + p;
        const bool full = (gpos - r >= 0) && (gpos + r < n_global) && (p - r >= 0) && (p + r < n_axis);
        double acc = 0, wsum = 0;
        for (int k = -r; k <= r; ++k) {
            if (!full && (gpos + k < 0 || gpos + k >= n_global || p + k < 0 || p + k >= n_axis)) continue;
            const double w = t.w[k + r];
            acc += w * (double)in[i + k * stride];
            wsum += w;
        }
        if (renorm) {
            if (full)
                acc /= t.full_sum;
            else if (wsum > 0)
                acc /= wsum;
        }
        out[i] = (float)acc;
    }
}

// Box filter (1/w taps) along one axis of a planar 5-channel fp64 block; writes planes
// [oz0, oz0+onz) of the block's local z range (z axis only; x/y passes use oz0 = 0,
// onz = nz). Same edge semantics as convolve_axis with EdgeMode::zero_pad.
__global__ void __launch_bounds__(kNT) k_box5_f64(const double* __restrict__ in, double* __restrict__ out,
                                                   int64_t nx, int64_t ny, int64_t nz, int axis, int r,
                                                   double inv_w, int64_t lo_global, int64_t n_global, int64_t oz0,
                                                   int64_t onz) {
    const int64_t plane = nx * ny;
    const int64_t n_in = plane * nz, n_out = plane * onz;
    const int64_t n_axis = axis == 0 ? nx : axis == 1 ? ny : nz;
    const int64_t stride = axis == 0 ? 1 : axis == 1 ? nx : plane;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < 5 * n_out; i += (int64_t)gridDim.x * kNT) {
        const int c = (int)(i / n_out);
        const int64_t o = i - c * n_out;
        const int64_t x = o % nx, y = (o / nx) % ny, z = o / plane + oz0;
        const int64_t p = axis == 0 ? x : axis == 1 ? y : z;
        const int64_t gpos = lo_global + p;
        const int64_t base = c * n_in + z * plane + y * nx + x;
        double acc = 0;
        for (int k = -r; k <= r; ++k) {
            if (gpos + k < 0 || gpos + k >= n_global || p + k < 0 || p + k >= n_axis) continue;
            acc += inv_w * in[base + k * stride];
        }
        out[i] = acc;
    }
}

__global__ void __launch_bounds__(kNT) k_lncc_channels(const float* __restrict__ f, const float* __restrict__ m,
                                                        int64_t n, double* __restrict__ c5) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double fv = f[i], mv = m[i];  // products of fp32 values are exact in fp64
        c5[i] = fv;
        c5[n + i] = mv;
        c5[2 * n + i] = fv * fv;
        c5[3 * n + i] = mv * mv;
        c5[4 * n + i] = fv * mv;
    }
}

__device__ __forceinline__ double lncc_ncc(double muf, double mum, double muff, double mumm, double mufm,
                                           double eps) {  // lncc.hpp:63-69
    const double a = mufm - muf * mum;
    const double b = muff - muf * muf;
    const double c = mumm - mum * mum;
    return a * a / (b * c + eps);
}

__global__ void __launch_bounds__(kNT) k_lncc_finalize(const double* __restrict__ st, int64_t n, double eps,
                                                        float* __restrict__ map, double* __restrict__ part) {
    __shared__ double red[kNT / 32];
    double acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double ni = lncc_ncc(st[i], st[n + i], st[2 * n + i], st[3 * n + i], st[4 * n + i], eps);
        if (map) map[i] = (float)ni;
        acc += ni;
    }
    const double s = block_sum<kNT>(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_add_partials(const double* part, int nb, double* out) {
    double s = 0;
    for (int b = 0; b < nb; ++b) s += part[b];
    *out += s;
}

// lncc_gamma (lncc.hpp:77-90) in place.
__global__ void __launch_bounds__(kNT) k_lncc_gamma(double* __restrict__ st, int64_t n, double eps, double gi) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double muf = st[i], mum = st[n + i], muff = st[2 * n + i], mumm = st[3 * n + i],
                     mufm = st[4 * n + i];
        const double a = mufm - muf * mum;
        const double b = muff - muf * muf;
        const double c = mumm - mum * mum;
        const double denom = b * c + eps;
        const double gamma = 2.0 * gi * a / denom;
        st[i] = gamma;
        st[n + i] = gamma * (a * c / denom);
        st[2 * n + i] = gamma * (a * b / denom);
        st[3 * n + i] = gamma * (muf * (a * c / denom) - mum);
        st[4 * n + i] = gamma * (mum * (a * b / denom) - muf);
    }
}

// Final combination (lncc.hpp:265-278). gam: planar 5 x n interior voxels.
__global__ void __launch_bounds__(kNT) k_lncc_combine(const double* __restrict__ gam, int64_t n,
                                                       const float* __restrict__ f, const float* __restrict__ m,
                                                       float* __restrict__ gf, float* __restrict__ gm) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double fv = f[i], mv = m[i];
        if (gf) gf[i] = (float)(mv * gam[i] - fv * gam[n + i] + gam[3 * n + i]);
        gm[i] = (float)(fv * gam[i] - mv * gam[2 * n + i] + gam[4 * n + i]);
    }
}

static int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kNT - 1) / kNT, 16LL * num_sms()));
}

static int check_slab(const ffdp_dims& d, const ffdp_slab& s, int window) {
    if (d.nx < 1 || d.ny < 1 || d.nz < 1) return set_error(FFDP_INVALID_ARGUMENT, "Volume3: dims must be positive");
    if (window < 1 || window % 2 == 0)
        return set_error(FFDP_INVALID_ARGUMENT, "lncc: window must be odd and >= 1");
    if (s.buf_nz != d.nz) return set_error(FFDP_INVALID_ARGUMENT, "lncc: slab.buf_nz != buffer nz");
    if (s.buf_z0 < 0 || s.buf_z0 + s.buf_nz > s.nz_global || s.z_begin < s.buf_z0 ||
        s.z_end > s.buf_z0 + s.buf_nz || s.z_begin >= s.z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "lncc: inconsistent slab");
    const int r = window / 2;
    const int64_t need_lo = std::max<int64_t>(0, s.z_begin - r), need_hi = std::min<int64_t>(s.nz_global, s.z_end + r);
    if (s.buf_z0 > need_lo || s.buf_z0 + s.buf_nz < need_hi)
        return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: buffer lacks the %d halo planes the window needs", r);
    return FFDP_OK;
}

// The separable box over a slab: c5 (5 planar channels of the whole buffer) -> out
// (5 planar channels of the interior planes). Uses tmp as scratch of the buffer size.
static void box5_slab(double* c5, double* tmp, double* out, const ffdp_dims& d, const ffdp_slab& s, int window,
                      cudaStream_t st) {
    const int r = window / 2;
    const double inv_w = 1.0 / window;  // box_taps (smoothing.hpp:42-46)
    const int64_t nbuf = d.nx * d.ny * d.nz;
    const int64_t nint = d.nx * d.ny * (s.z_end - s.z_begin);
    k_box5_f64<<<grid_for(5 * nbuf), kNT, 0, st>>>(c5, tmp, d.nx, d.ny, d.nz, 0, r, inv_w, 0, d.nx, 0, d.nz);
    k_box5_f64<<<grid_for(5 * nbuf), kNT, 0, st>>>(tmp, c5, d.nx, d.ny, d.nz, 1, r, inv_w, 0, d.ny, 0, d.nz);
    k_box5_f64<<<grid_for(5 * nint), kNT, 0, st>>>(c5, out, d.nx, d.ny, d.nz, 2, r, inv_w, s.buf_z0, s.nz_global,
                                                   s.z_begin - s.buf_z0, s.z_end - s.z_begin);
}

}  // namespace ffdp

using namespace ffdp;

extern "C" {

int ffdp_convolve_axis(const float* in, float* out, ffdp_dims dims, int channels, int axis, const double* taps,
                       int ntaps, int mode, int64_t lo_global, int64_t n_global, void* stream) {
    if (!in || !out || !taps) return set_error(FFDP_INVALID_ARGUMENT, "convolve_axis: null pointer");
    if (ntaps < 1 || ntaps % 2 == 0 || ntaps > kMaxTaps)
        return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: kernel must be odd (and <= %d taps)", kMaxTaps);
    if (axis < 0 || axis > 2 || channels < 1 || dims.nx < 1 || dims.ny < 1 || dims.nz < 1)
        return set_error(FFDP_INVALID_ARGUMENT, "convolve_axis: bad axis/channels/dims");
    Taps t;
    t.n = ntaps;
    t.full_sum = 0;
    for (int i = 0; i < ntaps; ++i) {
        t.w[i] = taps[i];
        t.full_sum += taps[i];
    }
    const int64_t n = dims.nx * dims.ny * dims.nz * channels;
    k_conv_axis_f32<<<grid_for(n), kNT, 0, (cudaStream_t)stream>>>(in, out, dims.nx, dims.ny, dims.nz, channels,
                                                                    axis, t, mode == 1, lo_global, n_global);
    return check_launch("convolve_axis");
}

int ffdp_lncc_fwd(const float* f, const float* m, ffdp_dims d, ffdp_slab s, int window, double eps, double* state,
                  float* map, double* sum_n, void* stream) {
    if (int rc = check_slab(d, s, window)) return rc;
    if (!f || !m || !state) return set_error(FFDP_INVALID_ARGUMENT, "lncc: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nbuf = d.nx * d.ny * d.nz;
    const int64_t nint = d.nx * d.ny * (s.z_end - s.z_begin);
    double* c5 = (double*)scratch_alloc(sizeof(double) * 10 * nbuf, st);
    if (!c5) return set_error(FFDP_CUDA, "lncc: scratch allocation failed");
    k_lncc_channels<<<grid_for(nbuf), kNT, 0, st>>>(f, m, nbuf, c5);
    box5_slab(c5, c5 + 5 * nbuf, state, d, s, window, st);
    const int nb = grid_for(nint);
    double* part = (double*)scratch_alloc(sizeof(double) * nb, st);
    k_lncc_finalize<<<nb, kNT, 0, st>>>(state, nint, eps, map, part);
    if (sum_n) k_add_partials<<<1, 1, 0, st>>>(part, nb, sum_n);
    scratch_free(part, st);
    scratch_free(c5, st);
    return check_launch("lncc_fwd");
}

int ffdp_lncc_gamma(double* state, int64_t voxels, double eps, double gi, void* stream) {
    if (!state || voxels < 1) return set_error(FFDP_INVALID_ARGUMENT, "lncc_gamma: bad arguments");
    k_lncc_gamma<<<grid_for(voxels), kNT, 0, (cudaStream_t)stream>>>(state, voxels, eps, gi);
    return check_launch("lncc_gamma");
}

int ffdp_lncc_combine(const double* gamma, ffdp_dims d, ffdp_slab s, int window, int ants, const float* f,
                      const float* m, float* grad_f, float* grad_m, void* stream) {
    if (!gamma || !f || !m || !grad_m) return set_error(FFDP_INVALID_ARGUMENT, "lncc_combine: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nbuf = d.nx * d.ny * d.nz;
    const int64_t nint = d.nx * d.ny * (s.z_end - s.z_begin);
    if (ants) {
        if (s.z_end - s.z_begin != d.nz || s.z_begin != s.buf_z0)
            return set_error(FFDP_INVALID_ARGUMENT, "lncc_combine: ANTs mode takes an interior-only gamma buffer");
        k_lncc_combine<<<grid_for(nint), kNT, 0, st>>>(gamma, nint, f, m, grad_f, grad_m);
        return check_launch("lncc_combine");
    }
    if (int rc = check_slab(d, s, window)) return rc;
    double* c5 = (double*)scratch_alloc(sizeof(double) * (10 * nbuf + 5 * nint), st);
    if (!c5) return set_error(FFDP_CUDA, "lncc_combine: scratch allocation failed");
    cudaMemcpyAsync(c5, gamma, sizeof(double) * 5 * nbuf, cudaMemcpyDeviceToDevice, st);
    double* out = c5 + 10 * nbuf;
    box5_slab(c5, c5 + 5 * nbuf, out, d, s, window, st);
    k_lncc_combine<<<grid_for(nint), kNT, 0, st>>>(out, nint, f, m, grad_f, grad_m);
    scratch_free(c5, st);
    return check_launch("lncc_combine");
}


int ffdp_lncc_bwd(double upstream, double* state, const float* f, const float* m, ffdp_dims d, int window, double eps,
                  int ants, float* grad_f, float* grad_m, void* stream) {
    // lncc_backward_fused (lncc.hpp:226-280): gi = -upstream / N (lncc.hpp:234)
    if (!state || !f || !m || !grad_m) return set_error(FFDP_INVALID_ARGUMENT, "lncc_backward: null pointer");
    const int64_t n = d.nx * d.ny * d.nz;
    if (n < 1) return set_error(FFDP_INVALID_ARGUMENT, "lncc_backward: empty volume");
    const ffdp_slab full{0, d.nz, 0, d.nz, d.nz};
    if (int rc = check_slab(d, full, window)) return rc;
    if (int rc = ffdp_lncc_gamma(state, n, eps, -upstream / (double)n, stream)) return rc;
    return ffdp_lncc_combine(state, d, full, window, ants, f, m, grad_f, grad_m, stream);
}

int ffdp_lncc_fwdbwd(const float* f, const float* m, ffdp_dims d, int window, double eps, int ants, double upstream,
                     double* state, double* sum_n, float* grad_f, float* grad_m, void* stream) {
    if (!sum_n) return set_error(FFDP_INVALID_ARGUMENT, "lncc: null sum_n");
    const ffdp_slab full{0, d.nz, 0, d.nz, d.nz};
    if (int rc = ffdp_lncc_fwd(f, m, d, full, window, eps, state, nullptr, sum_n, stream)) return rc;
    return ffdp_lncc_bwd(upstream, state, f, m, d, window, eps, ants, grad_f, grad_m, stream);
}

}  // extern "C"
