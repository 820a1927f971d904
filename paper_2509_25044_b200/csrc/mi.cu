// mi.cu -- Mattes mutual information on the GPU: the operator API (mi.hpp:235-437,
// distops.hpp:355-396) and the two passes of the fused MI step.
//
// Histogram: each CTA owns a private joint + marginal histogram in shared memory as
// 32-bit fixed point (a 2^-20 coarse counter plus a 2^-36 residual counter per bin). A thread walks a contiguous run of voxels and
// keeps the 4x4 joint footprint of the current (m_lo, n_lo) bin cell in registers,
// flushing it with native integer shared-memory atomics only when the cell changes
// (smooth volumes change cells rarely along x). The CTA flushes once to a global
// 64-bit fixed-point histogram. Integer sums are order independent, so the histogram
// (and with it the loss and ghat) is deterministic run to run.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "ffdp_common.cuh"

namespace ffdp {

constexpr int kMiNT = 256;
constexpr double kFix = 1048576.0;  // 2^20
constexpr int kMaxBins = 64;

// Voxels a CTA may accumulate before its 32-bit counters could overflow.
static int chunk_for(const ffdp_parzen& k) {
    // max kappa: bspline 2/3, gaussian ~0.80, delta 1 (joint <= max^2, marginal <= max)
    return k.kind == FFDP_PARZEN_DELTA ? 2048 : 4096;
}

struct HistAcc {
    int32_t mi, nj;
    float j[16], ai[4], aj[4];
};

__device__ __forceinline__ void hist_reset(HistAcc& h, int32_t mi, int32_t nj) {
    h.mi = mi;
    h.nj = nj;
#pragma unroll
    for (int q = 0; q < 16; ++q) h.j[q] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) h.ai[q] = h.aj[q] = 0.f;
}

// One register-aggregated value -> shared fixed point as a coarse part (units of
// 2^-20) plus the rounding residual (units of 2^-36). Sparse bins made only of
// B-spline tail products keep their relative accuracy, which ghat = log(p / p_i p_j)
// needs (mi.hpp:375-377).
__device__ __forceinline__ void fix_add(uint32_t* coarse, uint32_t* fine, int idx, float v) {
    const float q = v * (float)kFix;
    const float qi = floorf(q);
    const uint32_t fi = __float2uint_rn((q - qi) * 65536.0f);
    if (qi != 0.f) atomicAdd(&coarse[idx], (uint32_t)qi);
    if (fi) atomicAdd(&fine[idx], fi);
}

__device__ __forceinline__ void hist_flush(const HistAcc& h, int B, uint32_t* s, bool marginals) {
    const int nh = B * B + 2 * B;
    uint32_t* fine = s + nh;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float v = h.j[4 * a + b];
            if (v != 0.f) fix_add(s, fine, (h.mi + a) * B + (h.nj + b), v);
        }
        if (marginals) {
            if (h.ai[a] != 0.f) fix_add(s, fine, B * B + h.mi + a, h.ai[a]);
            if (h.aj[a] != 0.f) fix_add(s, fine, B * B + B + h.nj + a, h.aj[a]);
        }
    }
}

__device__ __forceinline__ void hist_add(HistAcc& h, const Bins4& bi, const Bins4& bj, int B, uint32_t* s,
                                         bool marginals) {
    if (bi.m_lo != h.mi || bj.m_lo != h.nj) {
        hist_flush(h, B, s, marginals);
        hist_reset(h, bi.m_lo, bj.m_lo);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 4; ++b) h.j[4 * a + b] = fmaf(bi.k[a], bj.k[b], h.j[4 * a + b]);
        h.ai[a] += bi.k[a];
        h.aj[a] += bj.k[a];
    }
}

// CTA histogram (coarse | fine) -> global 64-bit fixed point (coarse | fine).
__device__ __forceinline__ void hist_cta_flush(int B, const uint32_t* s, unsigned long long* g, int parts = 2) {
    __syncthreads();
    const int n = parts * (B * B + 2 * B);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t v = s[i];
        if (v) atomicAdd(&g[i], (unsigned long long)v);
    }
}

__device__ __forceinline__ void hist_cta_init(int B, uint32_t* s, int parts = 2) {
    for (int i = threadIdx.x; i < parts * (B * B + 2 * B); i += blockDim.x) s[i] = 0;
    __syncthreads();
}

// ---------------------------------------------------------------- standalone hist
__global__ void __launch_bounds__(kMiNT) k_mi_hist(const float* __restrict__ vi, const float* __restrict__ vj,
                                                    int64_t n, ParzenDev p, int chunk,
                                                    unsigned long long* __restrict__ g, int32_t* bad) {
    extern __shared__ uint32_t s_hist[];
    const int B = p.bins;
    hist_cta_init(B, s_hist);
    const int per = chunk / kMiNT;
    const int64_t v0 = blockIdx.x * (int64_t)chunk + (int64_t)threadIdx.x * per;
    HistAcc h;
    hist_reset(h, -1000, -1000);
    int badv = 0;
    for (int q = 0; q < per; ++q) {
        const int64_t v = v0 + q;
        if (v >= n) break;
        const float a = vi[v], b = vj[v];
        if (!(a >= 0.f && a <= 1.f) || !(b >= 0.f && b <= 1.f)) {
            badv = 1;
            continue;
        }
        const Bins4 bi = parzen_bins<false>(p, (double)a);
        const Bins4 bj = parzen_bins<false>(p, (double)b);
        hist_add(h, bi, bj, B, s_hist, true);
    }
    hist_flush(h, B, s_hist, true);
    if (badv && bad) atomicExch(bad, 1);
    hist_cta_flush(B, s_hist, g);
}

// mi_forward_approx hard binning (mi.hpp:296-305): exact integer counts.
__global__ void __launch_bounds__(kMiNT) k_mi_count(const float* __restrict__ vi, const float* __restrict__ vj,
                                                     int64_t n, int B, unsigned long long* __restrict__ g,
                                                     int32_t* bad) {
    extern __shared__ uint32_t s_hist[];
    hist_cta_init(B, s_hist, 1);
    uint32_t *sj = s_hist, *smi = s_hist + B * B, *smj = smi + B;
    int badv = 0;
    for (int64_t v = blockIdx.x * (int64_t)kMiNT + threadIdx.x; v < n; v += (int64_t)gridDim.x * kMiNT) {
        const float a = vi[v], b = vj[v];
        if (!(a >= 0.f && a <= 1.f) || !(b >= 0.f && b <= 1.f)) {
            badv = 1;
            continue;
        }
        const int mb = min((int)((double)a * B), B - 1), nb = min((int)((double)b * B), B - 1);
        atomicAdd(&sj[mb * B + nb], 1u);
        atomicAdd(&smi[mb], 1u);
        atomicAdd(&smj[nb], 1u);
    }
    if (badv && bad) atomicExch(bad, 1);
    hist_cta_flush(B, s_hist, g, 1);
}

// Fixed-point histogram (coarse 2^-20 | fine 2^-36) -> double raw payload (accumulated).
__global__ void k_fix_to_raw(const unsigned long long* g, int n, double* raw) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
        raw[i] += (double)g[i] * (1.0 / kFix) + (double)g[n + i] * (1.0 / (kFix * 65536.0));
}

// kernel_bin_taps + separable tap convolution of the counts (mi.hpp:274-349).
__global__ void k_mi_approx_conv(const unsigned long long* cnt, int B, ParzenDev p, double* raw) {
    __shared__ double taps[2 * kMaxBins + 1];
    __shared__ double tmp[kMaxBins * kMaxBins];
    const int radius = (int)ceil(p.radius * p.bins);  // kernel_bin_taps (mi.hpp:275-282)
    if (threadIdx.x == 0) {
        for (int d = -radius; d <= radius; ++d) {
            const double x = (double)d / B;
            double k = 0;
            if (p.kind == FFDP_PARZEN_GAUSSIAN) {
                if (!(fabs(x) > p.radius)) k = p.norm * exp(-0.5 * (x / p.sigma) * (x / p.sigma));
            } else if (p.kind == FFDP_PARZEN_BSPLINE3) {
                const double a = fabs(x * B);
                k = a < 1.0 ? (4.0 - 6.0 * a * a + 3.0 * a * a * a) / 6.0 : a < 2.0 ? (2 - a) * (2 - a) * (2 - a) / 6.0 : 0;
            } else {
                k = fabs(x) < p.radius ? 1.0 : 0.0;
            }
            taps[d + radius] = k;
        }
    }
    __syncthreads();
    const unsigned long long* ci = cnt + B * B;
    const unsigned long long* cj = ci + B;
    for (int m = threadIdx.x; m < B; m += blockDim.x) {
        double ai = 0, aj = 0;
        for (int d = -radius; d <= radius; ++d) {
            const int s = m - d;
            if (s < 0 || s >= B) continue;
            ai += taps[d + radius] * (double)ci[s];
            aj += taps[d + radius] * (double)cj[s];
        }
        raw[B * B + m] += ai;
        raw[B * B + B + m] += aj;
    }
    for (int q = threadIdx.x; q < B * B; q += blockDim.x) {
        const int m = q / B, nn = q % B;
        double acc = 0;
        for (int d = -radius; d <= radius; ++d) {
            const int s = m - d;
            if (s < 0 || s >= B) continue;
            acc += taps[d + radius] * (double)cnt[s * B + nn];
        }
        tmp[q] = acc;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < B * B; q += blockDim.x) {
        const int m = q / B, nn = q % B;
        double acc = 0;
        for (int d = -radius; d <= radius; ++d) {
            const int s = nn - d;
            if (s < 0 || s >= B) continue;
            acc += taps[d + radius] * tmp[m * B + s];
        }
        raw[q] += acc;
    }
}

// finalize_histogram + histogram_mi + ghat (mi.hpp:181-209, 369-390), one CTA, fixed
// reduction order. table = p_ij[B*B], p_i[B], p_j[B], ghat[B*B], {z, mi, dot, 0}.
__global__ void __launch_bounds__(1024) k_mi_finalize(const double* __restrict__ raw, int B, double upstream,
                                                      double* __restrict__ table) {
    __shared__ double rs[kMaxBins * kMaxBins];
    __shared__ double red[mi_finalize_scratch(kMaxBins, 1024)];
    for (int q = threadIdx.x; q < B * B; q += blockDim.x) rs[q] = raw[q];
    mi_finalize_block(rs, B, upstream, table, red);
}

// d(loss)/dI and d(loss)/dJ per voxel with compact support (mi.hpp:392-421).
__device__ __forceinline__ void mi_grad_voxel(const ParzenDev& p, const float* sg /*ghat (B x (B+1))*/, int B,
                                              double a, double b, float& gi, float& gj) {
    const Bins4 bi = parzen_bins<true>(p, a);
    const Bins4 bj = parzen_bins<true>(p, b);
    const int ld = B + 1;
    float si = 0.f, sjv = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int m = bi.m_lo + q;
        if (m < 0 || m >= B || (bi.k[q] == 0.f && bi.w[q] == 0.f)) continue;
        float acc_i = 0.f, acc_j = 0.f;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int nn = bj.m_lo + r;
            if (nn < 0 || nn >= B) continue;
            const float gv = sg[m * ld + nn];
            acc_i = fmaf(gv, bj.k[r], acc_i);
            acc_j = fmaf(gv, bj.w[r], acc_j);
        }
        si = fmaf(bi.w[q], acc_i, si);
        sjv = fmaf(bi.k[q], acc_j, sjv);
    }
    gi = si;
    gj = sjv;
}

__device__ __forceinline__ void load_ghat(const double* table, int B, float* sg) {
    const double* gh = table + B * B + 2 * B;
    for (int q = threadIdx.x; q < B * B; q += blockDim.x) sg[(q / B) * (B + 1) + q % B] = (float)gh[q];
    __syncthreads();
}

__global__ void __launch_bounds__(kMiNT) k_mi_bwd(const float* __restrict__ vi, const float* __restrict__ vj,
                                                   int64_t n, ParzenDev p, const double* __restrict__ table,
                                                   float* __restrict__ gi, float* __restrict__ gj) {
    extern __shared__ float sg[];
    const int B = p.bins;
    load_ghat(table, B, sg);
    for (int64_t v = blockIdx.x * (int64_t)kMiNT + threadIdx.x; v < n; v += (int64_t)gridDim.x * kMiNT) {
        float a, b;
        mi_grad_voxel(p, sg, B, (double)vi[v], (double)vj[v], a, b);
        if (gi) gi[v] = a;
        gj[v] = b;
    }
}

// ---------------------------------------------------------------- fused MI step
// Voxel v of the slab interior: lattice (x, y, z_global); f/u index via the buffer.
struct SlabIdx {
    int32_t nx, ny;
    int64_t plane;
    int64_t z_begin, nvox;  // interior voxels
    int64_t buf_z0;
};

__device__ __forceinline__ void slab_voxel(const SlabIdx& s, int64_t v, int32_t& x, int32_t& y, int32_t& z,
                                           int64_t& bi) {
    const int64_t zz = v / s.plane;
    const int64_t r = v - zz * s.plane;
    y = (int32_t)(r / s.nx);
    x = (int32_t)(r - (int64_t)y * s.nx);
    z = (int32_t)(zz + s.z_begin);
    bi = (zz + s.z_begin - s.buf_z0) * s.plane + r;
}

template <bool F64V>
__global__ void __launch_bounds__(kMiNT) k_step_mi_hist(Geom g, SlabIdx s, const float* __restrict__ f,
                                                         const float* __restrict__ u, ParzenDev p, int chunk,
                                                         unsigned long long* __restrict__ gh, int32_t* miss_counter) {
    extern __shared__ uint32_t s_hist[];
    const int B = p.bins;
    hist_cta_init(B, s_hist);
    const int per = chunk / kMiNT;
    const int64_t v0 = blockIdx.x * (int64_t)chunk + (int64_t)threadIdx.x * per;
    HistAcc h;
    hist_reset(h, -1000, -1000);
    int miss = 0;
    for (int q = 0; q < per; ++q) {
        const int64_t v = v0 + q;
        if (v >= s.nvox) break;
        int32_t x, y, z;
        int64_t bi;
        slab_voxel(s, v, x, y, z, bi);
        const Cell c = resolve(g, x, y, z, u[3 * bi], u[3 * bi + 1], u[3 * bi + 2]);
        const Corners k = gather(g, c, miss);
        const double mw = F64V ? interp_f64(k, c) : (double)interp(k, c);
        const Bins4 b_i = parzen_bins<false>(p, (double)f[bi]);
        const Bins4 b_j = parzen_bins<false>(p, mw);
        hist_add(h, b_i, b_j, B, s_hist, true);
    }
    hist_flush(h, B, s_hist, true);
    if (miss && miss_counter) atomicAdd(miss_counter, 1);
    hist_cta_flush(B, s_hist, gh);
}

template <bool F64V>
__global__ void __launch_bounds__(kMiNT) k_step_mi_grad(Geom g, SlabIdx s, const float* __restrict__ f,
                                                         const float* __restrict__ u, ParzenDev p,
                                                         const double* __restrict__ table, float* __restrict__ g_u,
                                                         int32_t* miss_counter) {
    extern __shared__ float sg[];
    const int B = p.bins;
    load_ghat(table, B, sg);
    int miss = 0;
    for (int64_t v = blockIdx.x * (int64_t)kMiNT + threadIdx.x; v < s.nvox; v += (int64_t)gridDim.x * kMiNT) {
        int32_t x, y, z;
        int64_t bi;
        slab_voxel(s, v, x, y, z, bi);
        const Cell c = resolve(g, x, y, z, u[3 * bi], u[3 * bi + 1], u[3 * bi + 2]);
        const Corners k = gather(g, c, miss);
        float d[3];
        const float mwf = interp_grad(k, c, d);
        const double mw = F64V ? interp_f64(k, c) : (double)mwf;
        float gi_unused, gm;
        mi_grad_voxel(p, sg, B, (double)f[bi], mw, gi_unused, gm);
        const int64_t o = 3 * v;
        g_u[o] = g.dscale[0] * d[0] * gm;
        g_u[o + 1] = g.dscale[1] * d[1] * gm;
        g_u[o + 2] = g.dscale[2] * d[2] * gm;
    }
    if (miss && miss_counter) atomicAdd(miss_counter, 1);
}

static int check_parzen(const ffdp_parzen* k) {
    if (!k) return set_error(FFDP_INVALID_ARGUMENT, "mi: null kernel");
    if (k->bins < 2) return set_error(FFDP_INVALID_ARGUMENT, "mi: bins must be >= 2");
    if (k->bins > kMaxBins) return set_error(FFDP_INVALID_ARGUMENT, "mi: bins must be <= %d", kMaxBins);
    if (k->kind < 0 || k->kind > 2) return set_error(FFDP_INVALID_ARGUMENT, "mi: unknown kernel kind");
    return FFDP_OK;
}

static size_t hist_smem(int B) { return 2 * sizeof(uint32_t) * (B * B + 2 * B); }
static size_t ghat_smem(int B) { return sizeof(float) * B * (B + 1); }

static int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kMiNT - 1) / kMiNT, 16LL * num_sms()));
}

static int check_slab_mi(const ffdp_dims& d, const ffdp_slab& s) {
    if (d.nx < 1 || d.ny < 1 || d.nz < 1 || s.buf_nz != d.nz || s.z_begin < s.buf_z0 ||
        s.z_end > s.buf_z0 + s.buf_nz || s.z_begin >= s.z_end || s.buf_z0 + s.buf_nz > s.nz_global)
        return set_error(FFDP_INVALID_ARGUMENT, "dist_mi: inconsistent slab");
    return FFDP_OK;
}

static SlabIdx make_slab_idx(const ffdp_dims& d, const ffdp_slab& s) {
    SlabIdx r;
    r.nx = (int32_t)d.nx;
    r.ny = (int32_t)d.ny;
    r.plane = d.nx * d.ny;
    r.z_begin = s.z_begin;
    r.nvox = r.plane * (s.z_end - s.z_begin);
    r.buf_z0 = s.buf_z0;
    return r;
}

bool mi_quad_path_applies(const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                          const ffdp_parzen& k);
// Below this many interior voxels the fused MI step uses the scalar kernels: their 2^-36
// fixed-point residual counters keep the sparse histograms of tiny lattices exact to
// ~1e-11, where the quad path's 2^-23 grid is visible in the gradient (bins fed only by
// tail products); the quad path pays off only on large lattices anyway.
// FFDP_MI_QUAD_MIN overrides the threshold (tests exercise both paths on one lattice).
inline int64_t quad_min_voxels() {
    static const int64_t v = [] {
        const char* e = std::getenv("FFDP_MI_QUAD_MIN");
        return e ? std::atoll(e) : (int64_t)(1 << 16);
    }();
    return v;
}
inline bool mi_use_quad(const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m, const ffdp_parzen& k) {
    return d.nx * d.ny * (s.z_end - s.z_begin) >= quad_min_voxels() && mi_quad_path_applies(d, s, m, k);
}
int mi_quad_hist(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, double* raw, unsigned long long* ws,
                 int32_t* miss, cudaStream_t st, float* rec = nullptr, double* table = nullptr,
                 double upstream = -1.0, int scale_exp = 0);
int mi_grad_rec(const float* f, const ffdp_dims& d, const ffdp_slab& s, const ffdp_parzen& k, const double* table,
                const float* rec, float* g_u, cudaStream_t st);
int mi_quad_grad(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, const double* table, float* g_u, int32_t* miss,
                 cudaStream_t st);

}  // namespace ffdp

using namespace ffdp;

extern "C" {

int ffdp_mi_hist(const float* vi, const float* vj, int64_t n, const ffdp_parzen* kernel, int approx, double* raw,
                 int32_t* bad_input, uint64_t* stats, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (n < 1 || !vi || !vj || !raw) return set_error(FFDP_INVALID_ARGUMENT, "mi: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int B = kernel->bins;
    const int nh = B * B + 2 * B;
    unsigned long long* g = (unsigned long long*)scratch_alloc(sizeof(unsigned long long) * 2 * nh, st);
    if (!g) return set_error(FFDP_CUDA, "mi: scratch allocation failed");
    cudaMemsetAsync(g, 0, sizeof(unsigned long long) * 2 * nh, st);
    const ParzenDev p = make_parzen_dev(*kernel);
    if (approx) {
        k_mi_count<<<grid_for(n), kMiNT, hist_smem(B), st>>>(vi, vj, n, B, g, bad_input);
        k_mi_approx_conv<<<1, 1024, 0, st>>>(g, B, p, raw);
    } else {
        const int chunk = chunk_for(*kernel);
        const int64_t nb = (n + chunk - 1) / chunk;
        k_mi_hist<<<(unsigned)nb, kMiNT, hist_smem(B), st>>>(vi, vj, n, p, chunk, g, bad_input);
        k_fix_to_raw<<<(nh + 255) / 256, 256, 0, st>>>(g, nh, raw);
    }
    scratch_free(g, st);
    if (stats) {
        // MiStats (mi.hpp:156-159): counts of the reference's exact formulation (all B bins per
        // voxel, mi.hpp:255,265-267) and of hard binning (3 writes per voxel, mi.hpp:304).
        const uint64_t un = (uint64_t)n, ub = (uint64_t)B;
        if (approx) {
            stats[0] += 3 * un;
        } else {
            stats[0] += un * ub * ub + 2 * un * ub;
            stats[1] += 2 * un * ub;
        }
    }
    return check_launch("mi_hist");
}

int ffdp_mi_finalize(const double* raw, int bins, double upstream, double* table, void* stream) {
    if (!raw || !table || bins < 2 || bins > kMaxBins) return set_error(FFDP_INVALID_ARGUMENT, "mi_finalize: bad args");
    k_mi_finalize<<<1, 1024, 0, (cudaStream_t)stream>>>(raw, bins, upstream, table);
    return check_launch("mi_finalize");
}

int ffdp_mi_bwd(const float* vi, const float* vj, int64_t n, const ffdp_parzen* kernel, const double* table,
                float* grad_i, float* grad_j, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (n < 1 || !vi || !vj || !table || !grad_j) return set_error(FFDP_INVALID_ARGUMENT, "mi_backward: bad args");
    const int B = kernel->bins;
    k_mi_bwd<<<grid_for(n), kMiNT, ghat_smem(B), (cudaStream_t)stream>>>(vi, vj, n, make_parzen_dev(*kernel), table,
                                                                          grad_i, grad_j);
    return check_launch("mi_bwd");
}

int64_t ffdp_step_mi_workspace_bytes(int bins) {
    return (int64_t)sizeof(unsigned long long) * 2 * ((int64_t)bins * bins + 2 * bins);
}

int ffdp_step_mi_hist(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                      const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, void* workspace,
                      int32_t* miss, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (int rc = check_slab_mi(d, s)) return rc;
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !raw || !m.data) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (mi_use_quad(d, s, m, *kernel))
        return mi_quad_hist(f, u, d, s, m, *args, *kernel, raw, (unsigned long long*)workspace, miss, st);
    const int B = kernel->bins;
    const int nh = B * B + 2 * B;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    const Geom g = make_geom(m, out, *args);
    const SlabIdx si = make_slab_idx(d, s);
    const ParzenDev p = make_parzen_dev(*kernel);
    unsigned long long* gh = (unsigned long long*)workspace;
    if (!gh) gh = (unsigned long long*)scratch_alloc(sizeof(unsigned long long) * 2 * nh, st);
    if (!gh) return set_error(FFDP_CUDA, "step_mi: scratch allocation failed");
    cudaMemsetAsync(gh, 0, sizeof(unsigned long long) * 2 * nh, st);
    const int chunk = chunk_for(*kernel);
    const unsigned nb = (unsigned)((si.nvox + chunk - 1) / chunk);
    if (kernel->kind == FFDP_PARZEN_BSPLINE3)
        k_step_mi_hist<false><<<nb, kMiNT, hist_smem(B), st>>>(g, si, f, u, p, chunk, gh, miss);
    else
        k_step_mi_hist<true><<<nb, kMiNT, hist_smem(B), st>>>(g, si, f, u, p, chunk, gh, miss);
    k_fix_to_raw<<<(nh + 255) / 256, 256, 0, st>>>(gh, nh, raw);
    if (!workspace) scratch_free(gh, st);
    return check_launch("step_mi_hist");
}

int ffdp_step_mi(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                 const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, double* table, float* g_u,
                 void* workspace, float* rec, int32_t* miss, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (!raw || !table) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null raw/table");
    const int B = kernel->bins;
    cudaMemsetAsync(raw, 0, sizeof(double) * (B * B + 2 * B), (cudaStream_t)stream);
    const bool use_rec = rec && kernel->kind == FFDP_PARZEN_BSPLINE3 && mi_use_quad(d, s, m, *kernel);
    if (use_rec && workspace) {
        // one rank, caller workspace: pass 1 with the finalize fused into its last CTA
        if (int rc = ffdp_step_mi_hist_final(f, u, d, s, m, args, kernel, raw, -1.0, table, workspace, rec, miss,
                                             stream))
            return rc;
        return ffdp_step_mi_grad_rec(f, d, s, kernel, table, rec, g_u, stream);
    }
    if (use_rec) {
        if (int rc = ffdp_step_mi_hist_rec(f, u, d, s, m, args, kernel, raw, workspace, rec, miss, stream)) return rc;
        if (int rc = ffdp_mi_finalize(raw, B, -1.0, table, stream)) return rc;
        return ffdp_step_mi_grad_rec(f, d, s, kernel, table, rec, g_u, stream);
    }
    if (int rc = ffdp_step_mi_hist(f, u, d, s, m, args, kernel, raw, workspace, miss, stream)) return rc;
    if (int rc = ffdp_mi_finalize(raw, B, -1.0, table, stream)) return rc;
    return ffdp_step_mi_grad(f, u, d, s, m, args, kernel, table, g_u, miss, stream);
}

int64_t ffdp_step_mi_record_bytes(ffdp_dims d, ffdp_slab s) {
    return (int64_t)sizeof(float) * 4 * d.nx * d.ny * std::max<int64_t>(0, s.z_end - s.z_begin);
}

int ffdp_step_mi_hist_rec(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                          const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, void* workspace,
                          float* rec, int32_t* miss, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (int rc = check_slab_mi(d, s)) return rc;
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !raw || !m.data || !rec) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null pointer");
    if (kernel->kind != FFDP_PARZEN_BSPLINE3)
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need the B-spline Parzen kernel");
    if (!mi_quad_path_applies(d, s, m, *kernel))
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need a zero-bordered moving window (pad = 2)");
    return mi_quad_hist(f, u, d, s, m, *args, *kernel, raw, (unsigned long long*)workspace, miss,
                        (cudaStream_t)stream, rec);
}

int ffdp_step_mi_hist_final(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                            const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, double upstream,
                            double* table, void* workspace, float* rec, int32_t* miss, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (int rc = check_slab_mi(d, s)) return rc;
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !raw || !table || !workspace || !m.data || !rec)
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null pointer");
    if (kernel->kind != FFDP_PARZEN_BSPLINE3)
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need the B-spline Parzen kernel");
    if (!mi_quad_path_applies(d, s, m, *kernel))
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need a zero-bordered moving window (pad = 2)");
    return mi_quad_hist(f, u, d, s, m, *args, *kernel, raw, (unsigned long long*)workspace, miss,
                        (cudaStream_t)stream, rec, table, upstream);
}

int ffdp_step_mi_grad_rec(const float* f, ffdp_dims d, ffdp_slab s, const ffdp_parzen* kernel, const double* table,
                          const float* rec, float* g_u, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (int rc = check_slab_mi(d, s)) return rc;
    if (!f || !table || !rec || !g_u) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null pointer");
    return mi_grad_rec(f, d, s, *kernel, table, rec, g_u, (cudaStream_t)stream);
}

int ffdp_step_mi_grad(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                      const ffdp_sampler_args* args, const ffdp_parzen* kernel, const double* table, float* g_u,
                      int32_t* miss, void* stream) {
    if (int rc = check_parzen(kernel)) return rc;
    if (int rc = check_slab_mi(d, s)) return rc;
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !table || !g_u || !m.data) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (mi_use_quad(d, s, m, *kernel))
        return mi_quad_grad(f, u, d, s, m, *args, *kernel, table, g_u, miss, st);
    const int B = kernel->bins;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    const Geom g = make_geom(m, out, *args);
    const SlabIdx si = make_slab_idx(d, s);
    const ParzenDev p = make_parzen_dev(*kernel);
    const int nb = grid_for(si.nvox);
    if (kernel->kind == FFDP_PARZEN_BSPLINE3)
        k_step_mi_grad<false><<<nb, kMiNT, ghat_smem(B), st>>>(g, si, f, u, p, table, g_u, miss);
    else
        k_step_mi_grad<true><<<nb, kMiNT, ghat_smem(B), st>>>(g, si, f, u, p, table, g_u, miss);
    return check_launch("step_mi_grad");
}

}  // extern "C"
