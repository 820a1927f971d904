// sampler.cu -- the composite implicit grid sampler I(A*X + t + S*u(X)) as standalone
// sm_100a kernels: forward (fused_sample / fused_sample_accumulate, sampler.hpp:254-276)
// and backward (fused_sample_backward, sampler.hpp:279-300). No coordinate grid is
// materialised: the output lattice is implicit in the launch, the affine/rescale chain
// is folded into Geom on the host.
#include <algorithm>

#include "ffdp_common.cuh"

namespace ffdp {

constexpr int kSampNT = 256;

__device__ __forceinline__ void lattice_xyz(int64_t v, const Geom& g, int32_t& x, int32_t& y, int32_t& z) {
    const int64_t plane = (int64_t)g.on[0] * g.on[1];
    z = (int32_t)(v / plane);
    const int32_t r = (int32_t)(v - (int64_t)z * plane);
    y = r / g.on[0];
    x = r - y * g.on[0];
}

__device__ __forceinline__ void flag_miss(int miss, int32_t* counter) {
    const unsigned any = __ballot_sync(0xffffffffu, miss);
    if (any && counter && (threadIdx.x & 31) == 0) atomicAdd(counter, __popc(any));
}

__global__ void __launch_bounds__(kSampNT) k_sampler_fwd(Geom g, const float* __restrict__ u, int64_t n_out,
                                                          float* __restrict__ out, int accumulate,
                                                          double* abs_contrib, int32_t* miss_counter) {
    __shared__ double red[kSampNT / 32];
    double abs_acc = 0;
    const int64_t stride = (int64_t)gridDim.x * kSampNT;
    const int64_t n_iter = (n_out + stride - 1) / stride;  // uniform trip count keeps the ballot converged
    for (int64_t it = 0; it < n_iter; ++it) {
        const int64_t v = it * stride + blockIdx.x * (int64_t)kSampNT + threadIdx.x;
        int miss = 0;
        if (v < n_out) {
            int32_t x, y, z;
            lattice_xyz(v, g, x, y, z);
            float u0 = 0.f, u1 = 0.f, u2 = 0.f;
            if (u) {
                u0 = u[3 * v];
                u1 = u[3 * v + 1];
                u2 = u[3 * v + 2];
            }
            const Cell c = resolve(g, x, y, z, u0, u1, u2);
            const Corners k = gather(g, c, miss);
            const float val = interp(k, c);
            out[v] = accumulate ? out[v] + val : val;
            abs_acc += fabs((double)val);
        }
        flag_miss(miss, miss_counter);
    }
    if (abs_contrib) {
        const double s = block_sum<kSampNT>(abs_acc, red);
        if (threadIdx.x == 0) atomicAdd(abs_contrib, s);
    }
}

// Backward sweep (sampler.hpp:200-239). Per-block fp64 partials of gA|gt go to part[12*block].
__global__ void __launch_bounds__(kSampNT) k_sampler_bwd(Geom g, const float* __restrict__ up,
                                                          const float* __restrict__ u, int64_t n_out, int want,
                                                          float* __restrict__ g_img, float* __restrict__ g_u,
                                                          double* __restrict__ part, int32_t* miss_counter) {
    double acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0;
    const bool want_at = (want & (FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION)) != 0;
    const int64_t stride = (int64_t)gridDim.x * kSampNT;
    const int64_t n_iter = (n_out + stride - 1) / stride;
    for (int64_t it = 0; it < n_iter; ++it) {
        const int64_t v = it * stride + blockIdx.x * (int64_t)kSampNT + threadIdx.x;
        int miss = 0;
        if (v < n_out) {
            int32_t x, y, z;
            lattice_xyz(v, g, x, y, z);
            float u0 = 0.f, u1 = 0.f, u2 = 0.f;
            if (u) {
                u0 = u[3 * v];
                u1 = u[3 * v + 1];
                u2 = u[3 * v + 2];
            }
            const float gv = up[v];
            const Cell c = resolve(g, x, y, z, u0, u1, u2);
            if (want & FFDP_WANT_IMAGE) {
                // scatter w * g into the 8 corners (sampler.hpp:204-220)
                for (int q = 0; q < 8; ++q) {
                    const int32_t ix = c.i0[0] + (q & 1), iy = c.i0[1] + ((q >> 1) & 1), iz = c.i0[2] + (q >> 2);
                    if (ix < 0 || ix >= g.n[0] || iy < 0 || iy >= g.n[1] || iz < 0 || iz >= g.n[2]) continue;
                    if (iz < g.wz0 || iz >= g.wz1) {
                        miss = 1;
                        continue;
                    }
                    const float w = ((q & 1) ? c.frac[0] : 1.f - c.frac[0]) *
                                    ((q & 2) ? c.frac[1] : 1.f - c.frac[1]) *
                                    ((q & 4) ? c.frac[2] : 1.f - c.frac[2]);
                    atomicAdd(g_img + (int64_t)(iz - g.wz0) * g.sz + (int64_t)iy * g.sy + ix, w * gv);
                }
            }
            if (want & (FFDP_WANT_WARP | FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION)) {
                const Corners k = gather(g, c, miss);
                float d[3];
                interp_grad(k, c, d);
                if (want & FFDP_WANT_WARP) {
                    g_u[3 * v] = g.dscale[0] * d[0] * gv;
                    g_u[3 * v + 1] = g.dscale[1] * d[1] * gv;
                    g_u[3 * v + 2] = g.dscale[2] * d[2] * gv;
                }
                if (want_at) {
                    const double X[3] = {g.Xlo[0] + g.Xstep[0] * x, g.Xlo[1] + g.Xstep[1] * y,
                                         g.Xlo[2] + g.Xstep[2] * z};
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        const double dg = (double)d[r] * (double)g.hn[r] * (double)gv;  // dxsrc_r * g
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) acc[3 * r + cc] = fma(dg, X[cc], acc[3 * r + cc]);
                        acc[9 + r] += dg;
                    }
                }
            }
        }
        flag_miss(miss, miss_counter);
    }
    if (want_at) {
        __shared__ double sm[kSampNT / 32][12];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
            const double s = warp_sum(acc[i]);
            if (lane == 0) sm[w][i] = s;
        }
        __syncthreads();
        if (threadIdx.x < 12) {
            double s = 0;
            for (int j = 0; j < kSampNT / 32; ++j) s += sm[j][threadIdx.x];
            part[12 * blockIdx.x + threadIdx.x] = s;
        }
    }
}

__global__ void k_sum_partials12(const double* part, int nb, double* out) {
    const int i = threadIdx.x;
    if (i < 12) {
        double s = 0;
        for (int b = 0; b < nb; ++b) s += part[12 * b + i];  // fixed order: deterministic
        out[i] = s;
    }
}

static int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kSampNT - 1) / kSampNT, 16LL * num_sms()));
}

static int check_window(const ffdp_image_window& img) {
    if (!img.data) return set_error(FFDP_INVALID_ARGUMENT, "sampler: null image");
    if (img.dims.nx < 1 || img.dims.ny < 1 || img.dims.nz < 1)
        return set_error(FFDP_INVALID_ARGUMENT, "Volume3: dims must be positive");
    if (img.pad != 0 && img.pad != 2) return set_error(FFDP_INVALID_ARGUMENT, "sampler: pad must be 0 or 2");
    if (img.z_begin < 0 || img.z_end > img.dims.nz || img.z_begin >= img.z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "sampler: bad image window [%lld,%lld) of %lld planes",
                         (long long)img.z_begin, (long long)img.z_end, (long long)img.dims.nz);
    if (img.dims.nx * img.dims.ny * img.dims.nz >= (1LL << 40) || img.dims.nx >= (1 << 30) ||
        img.dims.ny >= (1 << 30) || img.dims.nz >= (1 << 30))
        return set_error(FFDP_INVALID_ARGUMENT, "sampler: image too large");
    return FFDP_OK;
}

}  // namespace ffdp

using namespace ffdp;

extern "C" {

int ffdp_sampler_fwd(ffdp_image_window img, const float* u, ffdp_dims out_dims, const ffdp_sampler_args* args,
                     float* out, int accumulate, double* abs_contrib, int32_t* miss, void* stream) {
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (int rc = check_window(img)) return rc;
    if (out_dims.nx < 1 || out_dims.ny < 1 || out_dims.nz < 1 || !out)
        return set_error(FFDP_INVALID_ARGUMENT, "fused_sample: bad output lattice");
    const int64_t n = out_dims.nx * out_dims.ny * out_dims.nz;
    const Geom g = make_geom(img, out_dims, *args);
    k_sampler_fwd<<<grid_for(n), kSampNT, 0, (cudaStream_t)stream>>>(g, u, n, out, accumulate, abs_contrib, miss);
    return check_launch("sampler_fwd");
}

int ffdp_sampler_bwd(const float* upstream, ffdp_image_window img, const float* u, ffdp_dims out_dims,
                     const ffdp_sampler_args* args, int want, float* g_img, float* g_u, double* gAt, int32_t* miss,
                     void* stream) {
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (int rc = check_window(img)) return rc;
    if (!upstream) return set_error(FFDP_INVALID_ARGUMENT, "fused_sample_backward: null upstream");
    if ((want & FFDP_WANT_IMAGE) && !g_img) return set_error(FFDP_INVALID_ARGUMENT, "sampler_bwd: g_img missing");
    if ((want & FFDP_WANT_WARP) && !g_u) return set_error(FFDP_INVALID_ARGUMENT, "sampler_bwd: g_u missing");
    if ((want & (FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION)) && !gAt)
        return set_error(FFDP_INVALID_ARGUMENT, "sampler_bwd: gAt missing");
    const int64_t n = out_dims.nx * out_dims.ny * out_dims.nz;
    const Geom g = make_geom(img, out_dims, *args);
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = grid_for(n);
    double* part = nullptr;
    const bool want_at = (want & (FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION)) != 0;
    if (want_at) {
        part = (double*)scratch_alloc(sizeof(double) * 12 * nb, s);
        if (!part) return set_error(FFDP_CUDA, "sampler_bwd: scratch allocation failed");
    }
    k_sampler_bwd<<<nb, kSampNT, 0, s>>>(g, upstream, u, n, want, g_img, g_u, part, miss);
    if (want_at) {
        k_sum_partials12<<<1, 32, 0, s>>>(part, nb, gAt);
        scratch_free(part, s);
    }
    return check_launch("sampler_bwd");
}

}  // extern "C"
