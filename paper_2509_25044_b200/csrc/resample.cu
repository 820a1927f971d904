// resample.cu -- the multi-scale plumbing around the deformable loop
// (registration.hpp:230-331):
//   ffdp_resample_scale   resample_scale (resample.hpp:48-103): Gaussian anti-alias
//                         (sigma 0.5 / factor, renormalized, only when shrinking) then
//                         trilinear resampling preserving the first / last voxel centres;
//   ffdp_resample_warp    resample_warp (resample.hpp:108-146): trilinear on each channel
//                         (normalized displacements carry over unchanged);
//   ffdp_normalize        normalize_intensities (registration.hpp:100-115).
// The per-axis source coordinate f = i (n_src - 1) / (n_dst - 1) and its cell
// (resample.hpp:17-43: floor, 1e-9 face snap, upper corner clamped into the lattice) are
// fp64 per axis, computed once per output row / plane; values and weights are fp32.
#include <algorithm>
#include <cmath>

#include "ffdp_common.cuh"

namespace ffdp {
namespace rs {

struct Axis {
    int32_t i0, i1;  // lower / upper corner (clamped)
    float w1;        // weight of the upper corner
};

__device__ __forceinline__ Axis axis_sample(int64_t i, int64_t n_src, int64_t n_dst) {
    const double f = n_dst > 1 ? (double)i * (double)(n_src - 1) / (double)(n_dst - 1) : 0.0;
    double fl = floor(f);
    double a = f - fl;
    if (a < FFDP_FACE_SNAP) {
        a = 0.0;
    } else if (1.0 - a < FFDP_FACE_SNAP) {
        fl += 1.0;
        a = 0.0;
    }
    Axis r;
    r.i0 = (int32_t)min((int64_t)fl, n_src - 1);
    r.i1 = (int32_t)min((int64_t)fl + 1, n_src - 1);
    r.w1 = (float)a;
    return r;
}

template <int CH>
__global__ void __launch_bounds__(256) k_trilinear(const float* __restrict__ in, ffdp_dims sd, float* __restrict__ out,
                                                   ffdp_dims dd) {
    const int64_t n = dd.nx * dd.ny * dd.nz;
    for (int64_t v = blockIdx.x * 256LL + threadIdx.x; v < n; v += (int64_t)gridDim.x * 256) {
        const int64_t x = v % dd.nx, yz = v / dd.nx, y = yz % dd.ny, z = yz / dd.ny;
        const Axis ax = axis_sample(x, sd.nx, dd.nx), ay = axis_sample(y, sd.ny, dd.ny),
                   az = axis_sample(z, sd.nz, dd.nz);
        const int64_t r00 = ((int64_t)az.i0 * sd.ny + ay.i0) * sd.nx, r01 = ((int64_t)az.i0 * sd.ny + ay.i1) * sd.nx;
        const int64_t r10 = ((int64_t)az.i1 * sd.ny + ay.i0) * sd.nx, r11 = ((int64_t)az.i1 * sd.ny + ay.i1) * sd.nx;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            auto at = [&](int64_t row, int32_t xi) { return __ldg(in + (row + xi) * CH + c); };
            const float e00 = fmaf(ax.w1, at(r00, ax.i1) - at(r00, ax.i0), at(r00, ax.i0));
            const float e01 = fmaf(ax.w1, at(r01, ax.i1) - at(r01, ax.i0), at(r01, ax.i0));
            const float e10 = fmaf(ax.w1, at(r10, ax.i1) - at(r10, ax.i0), at(r10, ax.i0));
            const float e11 = fmaf(ax.w1, at(r11, ax.i1) - at(r11, ax.i0), at(r11, ax.i0));
            const float g0 = fmaf(ay.w1, e01 - e00, e00), g1 = fmaf(ay.w1, e11 - e10, e10);
            out[v * CH + c] = fmaf(az.w1, g1 - g0, g0);
        }
    }
}

__global__ void __launch_bounds__(256) k_normalize(const float* __restrict__ in, int64_t n, const float* mm,
                                                   float* __restrict__ out) {
    const double lo = mm[0], range = (double)mm[1] - (double)mm[0];
    for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
        out[i] = range > 0 ? (float)(((double)in[i] - lo) / range) : 0.0f;
}

// jacobian_positive_fraction (metrics.hpp:145-176): central differences over interior
// voxels (normalized steps 2 / (n - 1)), det(I + du/dx) > 0, counted per CTA and added.
__global__ void __launch_bounds__(256) k_jacobian_positive(const float* __restrict__ u, ffdp_dims d,
                                                           unsigned long long* count) {
    const int64_t ix = d.nx - 2, iy = d.ny - 2, iz = d.nz - 2, n = ix * iy * iz;
    const double h0 = 1.0 / (2.0 * (2.0 / (double)(d.nx - 1))), h1 = 1.0 / (2.0 * (2.0 / (double)(d.ny - 1))),
                 h2 = 1.0 / (2.0 * (2.0 / (double)(d.nz - 1)));
    unsigned long long pos = 0;
    for (int64_t v = blockIdx.x * 256LL + threadIdx.x; v < n; v += (int64_t)gridDim.x * 256) {
        const int64_t x = v % ix + 1, yz = v / ix, y = yz % iy + 1, z = yz / iy + 1;
        const int64_t c0 = ((z * d.ny + y) * d.nx + x) * 3, sx = 3, sy = 3 * d.nx, sz = 3 * d.nx * d.ny;
        double j[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            j[c][0] = ((double)u[c0 + sx + c] - (double)u[c0 - sx + c]) * h0;
            j[c][1] = ((double)u[c0 + sy + c] - (double)u[c0 - sy + c]) * h1;
            j[c][2] = ((double)u[c0 + sz + c] - (double)u[c0 - sz + c]) * h2;
            j[c][c] += 1.0;
        }
        const double det = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                           j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                           j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
        pos += det > 0 ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, o);
    if ((threadIdx.x & 31) == 0 && pos) atomicAdd(count, pos);
}

// dist_mse at one rank (distops.hpp:260-282, loss_and_grad mse registration.hpp:126-137):
// sum of (moved - fixed)^2 into *sum (fp64, fixed-order per CTA then atomics of partial
// sums -- reproducible to rounding), grad = 2 (moved - fixed) / n_total.
__global__ void __launch_bounds__(256) k_mse(const float* __restrict__ f, const float* __restrict__ m, int64_t n,
                                             double inv_n2, float* __restrict__ grad, double* partial) {
    double acc = 0;
    for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
        const double dd = (double)m[i] - (double)f[i];
        acc += dd * dd;
        if (grad) grad[i] = (float)(dd * inv_n2);
    }
    __shared__ double red[8];
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void k_sum_partials(const double* partial, int nb, double* out) {
    double s = 0;
    for (int i = 0; i < nb; ++i) s += partial[i];
    *out += s;
}

inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16LL * num_sms())); }

}  // namespace rs
}  // namespace ffdp

using namespace ffdp;

extern "C" {

int ffdp_resample_dims(ffdp_dims d, double factor, ffdp_dims* out) {
    if (!out) return set_error(FFDP_INVALID_ARGUMENT, "resample_scale: null output");
    if (!std::isfinite(factor) || factor <= 0)
        return set_error(FFDP_INVALID_ARGUMENT, "resample_scale: factor must be finite and > 0");
    if (factor == 1.0) {
        *out = d;
        return FFDP_OK;
    }
    ffdp_dims nd{(int64_t)std::ceil((double)d.nx * factor), (int64_t)std::ceil((double)d.ny * factor),
                 (int64_t)std::ceil((double)d.nz * factor)};
    if (nd.nx < 2 || nd.ny < 2 || nd.nz < 2) return set_error(FFDP_INVALID_ARGUMENT, "resample_scale: resulting dim < 2");
    *out = nd;
    return FFDP_OK;
}

int ffdp_resample_scale(const float* in, ffdp_dims d, double factor, float* out, float* scratch, void* stream) {
    ffdp_dims nd;
    if (int rc = ffdp_resample_dims(d, factor, &nd)) return rc;
    if (!in || !out) return set_error(FFDP_INVALID_ARGUMENT, "resample_scale: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = d.nx * d.ny * d.nz;
    if (factor == 1.0) {
        FFDP_CHECK_CUDA(cudaMemcpyAsync(out, in, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
        return FFDP_OK;
    }
    const float* src = in;
    float* own = nullptr;
    if (factor < 1.0) {
        // gaussian_smooth(v, 0.5 / factor) (smoothing.hpp:108-115): renormalized separable
        const double sigma = 0.5 / factor;
        const int64_t radius = (int64_t)std::ceil(3.0 * sigma);
        if (radius > 6) return set_error(FFDP_INVALID_ARGUMENT, "resample_scale: factor below 1/4 not supported");
        double taps[13];
        double sum = 0;
        for (int64_t k = -radius; k <= radius; ++k) {
            taps[k + radius] = std::exp(-0.5 * ((double)k / sigma) * ((double)k / sigma));
            sum += taps[k + radius];
        }
        for (int64_t k = 0; k <= 2 * radius; ++k) taps[k] /= sum;
        float* sm = scratch;
        if (!sm) sm = own = (float*)scratch_alloc(sizeof(float) * n, st);
        if (!sm) return set_error(FFDP_CUDA, "resample_scale: scratch allocation failed");
        const ffdp_slab full{0, d.nz, 0, d.nz, d.nz};
        if (int rc = ffdp_gp_convolve(in, sm, d, full, 1, taps, (int)(2 * radius + 1), 1, stream)) {
            if (own) scratch_free(own, st);
            return rc;
        }
        src = sm;
    }
    const int64_t no = nd.nx * nd.ny * nd.nz;
    rs::k_trilinear<1><<<rs::grid_for(no), 256, 0, st>>>(src, d, out, nd);
    if (own) scratch_free(own, st);
    return check_launch("resample_scale");
}

int ffdp_resample_warp(const float* in, ffdp_dims d, float* out, ffdp_dims nd, void* stream) {
    if (!in || !out) return set_error(FFDP_INVALID_ARGUMENT, "resample_warp: null pointer");
    if (nd.nx < 1 || nd.ny < 1 || nd.nz < 1 || d.nx < 1 || d.ny < 1 || d.nz < 1)
        return set_error(FFDP_INVALID_ARGUMENT, "resample_warp: dims must be positive");
    const int64_t no = nd.nx * nd.ny * nd.nz;
    rs::k_trilinear<3><<<rs::grid_for(no), 256, 0, (cudaStream_t)stream>>>(in, d, out, nd);
    return check_launch("resample_warp");
}

int ffdp_normalize(const float* in, int64_t n, float* out, void* stream) {
    if (!in || !out || n < 1) return set_error(FFDP_INVALID_ARGUMENT, "normalize_intensities: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    float* mm = (float*)scratch_alloc(2 * sizeof(float), st);
    if (!mm) return set_error(FFDP_CUDA, "normalize_intensities: scratch allocation failed");
    if (int rc = ffdp_minmax(in, n, mm, stream)) {
        scratch_free(mm, st);
        return rc;
    }
    rs::k_normalize<<<rs::grid_for(n), 256, 0, st>>>(in, n, mm, out);
    scratch_free(mm, st);
    return check_launch("normalize_intensities");
}

int ffdp_jacobian_positive(const float* u, ffdp_dims d, double* fraction, void* stream) {
    if (!u || !fraction) return set_error(FFDP_INVALID_ARGUMENT, "jacobian_positive_fraction: null pointer");
    if (d.nx < 3 || d.ny < 3 || d.nz < 3)
        return set_error(FFDP_INVALID_ARGUMENT, "jacobian_positive_fraction: lattice too small");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* cnt = (unsigned long long*)scratch_alloc(sizeof(unsigned long long), st);
    if (!cnt) return set_error(FFDP_CUDA, "jacobian_positive_fraction: scratch allocation failed");
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st);
    const int64_t n = (d.nx - 2) * (d.ny - 2) * (d.nz - 2);
    rs::k_jacobian_positive<<<rs::grid_for(n), 256, 0, st>>>(u, d, cnt);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
    scratch_free(cnt, st);
    FFDP_CHECK_CUDA(cudaStreamSynchronize(st));
    *fraction = (double)h / (double)n;
    return check_launch("jacobian_positive_fraction");
}

int ffdp_mse(const float* f, const float* m, int64_t n, int64_t n_total, float* grad, double* sum, void* stream) {
    if (!f || !m || !sum || n < 1 || n_total < 1) return set_error(FFDP_INVALID_ARGUMENT, "dist_mse: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = rs::grid_for(n);
    double* part = (double*)scratch_alloc(sizeof(double) * nb, st);
    if (!part) return set_error(FFDP_CUDA, "dist_mse: scratch allocation failed");
    rs::k_mse<<<nb, 256, 0, st>>>(f, m, n, 2.0 / (double)n_total, grad, part);
    rs::k_sum_partials<<<1, 1, 0, st>>>(part, nb, sum);
    scratch_free(part, st);
    return check_launch("dist_mse");
}

}  // extern "C"
