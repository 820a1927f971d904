// step_mi.cu -- the fused warp + Mattes MI step (registration.hpp:277-312 with dist_mi,
// distops.hpp:355-396), two passes over HBM (the global histogram is a hard dependency
// of the gradient, mi.hpp:369-390):
//
//   pass 1  Mw = fused_sample(M, u) and the joint Parzen histogram of (F, Mw)
//           (mi_forward_exact, mi.hpp:248-268) -- reads F, u, M: 20 B/voxel;
//   finalize (ffdp_mi_finalize) -- p, MI, ghat on one CTA;
//   pass 2  Mw and dMw/du again, dL/dMw = sum_m kappa_i sum_n ghat omega_j
//           (mi.hpp:392-421), g_u = S dxsrc dL/dMw -- reads F, u, M, writes g_u: 32 B.
//
// Work unit: a quad of 4 consecutive x voxels of one row (float4 loads of F and u,
// float4 stores of g_u; needs nx % 4 == 0, other lattices use mi.cu's scalar path).
// Histogram: 16 joint products per voxel rounded to fixed point by one FFMA against
// the 1.5*2^23 magic constant and added with native shared u32 atomics; every 1024
// voxels the CTA folds the u32 counters into a u64 shared copy (no overflow), and at
// the end into the global u64 histogram. Integer sums: deterministic. The marginals
// are not accumulated here: finalize_histogram derives p_i, p_j from the joint
// (mi.hpp:181-196), so the fused step needs only the B*B joint payload.
#include <algorithm>

#include "ffdp_common.cuh"

namespace ffdp {
namespace mstep {

constexpr int NT = 256;
constexpr int CHUNK_QUADS = NT;  // one quad per thread per chunk -> 1024 voxels per fold

struct Params {
    Geom g;
    ParzenDev p;
    const float* f;
    const float* u;
    float* g_u;
    const double* table;
    unsigned long long* hist;  // global u64 [B*B]
    int32_t* miss;
    int32_t nx, ny, qpr;       // quads per row
    FastDiv div_qpr, div_ny;
    int64_t plane, z_begin, buf_z0;
    int64_t nquads;
    float fix_scale;           // 2^23 (bspline) / 2^22 (gaussian) / 2^21 (delta)
};

// B-spline weights at bins m_lo..m_lo+3 for one intensity, fp32 (the kernel is C2,
// so fp32 rounding of the bin coordinate only perturbs weights at 1e-7).
struct BS4 {
    int32_t m_lo;
    float k[4], w[4];
};

template <bool OMEGA>
__device__ __forceinline__ BS4 bspline_bins(float v, int B) {
    BS4 r;
    const float s = fmaf(v, (float)B, -0.5f);
    const float fl = floorf(s);
    const float ph = s - fl;
    // clamp keeps the 4x4 footprint inside the padded tables even for inputs outside
    // [0,1] (which the reference rejects, mi.hpp:170-179)
    r.m_lo = min(max((__float_as_int(fl + 12582912.0f) - 0x4B400000) - 1, -2), B - 2);
    const float q = 1.0f - ph;
    const float p2 = ph * ph, p3 = p2 * ph, q2 = q * q;
    const float c6 = 1.0f / 6.0f;
    r.k[0] = q2 * q * c6;
    r.k[1] = fmaf(3.0f, p3, fmaf(-6.0f, p2, 4.0f)) * c6;
    r.k[2] = fmaf(-3.0f, p3, fmaf(3.0f, p2, fmaf(3.0f, ph, 1.0f))) * c6;
    r.k[3] = p3 * c6;
    if (OMEGA) {
        const float fb = (float)B;
        r.w[0] = -0.5f * fb * q2;
        r.w[1] = -fb * fmaf(-1.5f, p2, 2.0f * ph);
        r.w[2] = -fb * fmaf(1.5f, q2, -2.0f * q);
        r.w[3] = 0.5f * fb * p2;
    }
    return r;  // out-of-range bins land in the zero / ignored pads of the bin tables
}

template <bool OMEGA>
__device__ __forceinline__ BS4 generic_bins(const ParzenDev& p, double v) {
    const Bins4 b = parzen_bins<OMEGA>(p, v);
    BS4 r;
    r.m_lo = min(max(b.m_lo, -2), p.bins - 2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r.k[i] = b.k[i];
        if (OMEGA) r.w[i] = b.w[i];
    }
    return r;
}

__device__ __forceinline__ void quad_coords(const Params& P, int64_t q, int32_t& x0, int32_t& y, int32_t& z,
                                            int64_t& bi) {
    const uint32_t row = fdiv((uint32_t)q, P.div_qpr);
    x0 = ((int32_t)q - (int32_t)row * P.qpr) * 4;
    const uint32_t zz = fdiv(row, P.div_ny);
    y = (int32_t)row - (int32_t)zz * P.ny;
    z = (int32_t)zz + (int32_t)P.z_begin;
    bi = ((int64_t)zz + P.z_begin - P.buf_z0) * P.plane + (int64_t)(y * P.nx + x0);
}

// Padded bin tables: bin m lives at row m + PAD of a (B + 2 PAD)^2 table, so the
// 4 x 4 footprint of any intensity in [0, 1] (m_lo >= -2, m_lo + 3 <= B + 1) needs no
// bounds checks; out-of-range bins have zero weight and the pad rows are never read
// back (histogram) or hold zeros (ghat).
constexpr int PAD = 2;

__device__ __forceinline__ void load_quad(const Params& P, int64_t bi, float (&ff)[4], float (&uu)[12]) {
    const float4 fv = __ldg(reinterpret_cast<const float4*>(P.f + bi));
    const float4 ua = __ldg(reinterpret_cast<const float4*>(P.u + 3 * bi));
    const float4 ub = __ldg(reinterpret_cast<const float4*>(P.u + 3 * bi + 4));
    const float4 uc = __ldg(reinterpret_cast<const float4*>(P.u + 3 * bi + 8));
    ff[0] = fv.x; ff[1] = fv.y; ff[2] = fv.z; ff[3] = fv.w;
    uu[0] = ua.x; uu[1] = ua.y; uu[2] = ua.z; uu[3] = ua.w;
    uu[4] = ub.x; uu[5] = ub.y; uu[6] = ub.z; uu[7] = ub.w;
    uu[8] = uc.x; uu[9] = uc.y; uu[10] = uc.z; uu[11] = uc.w;
}

__device__ __forceinline__ void quad_cells(const Params& P, int32_t x0, int32_t y, int32_t z, const float (&uu)[12],
                                           Cell (&c)[4]) {
    RowBase rb;
    rb.init(P.g, x0, y, z);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k) rb.step(P.g);
        c[k] = rb.cell(P.g, uu[3 * k], uu[3 * k + 1], uu[3 * k + 2]);
    }
}

// ------------------------------------------------------------------ pass 1
template <bool BSPLINE, bool FULLWIN>
__global__ void __launch_bounds__(NT) k_step_mi_hist(const Params P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = P.p.bins;
    const int LD = B + 2 * PAD;
    const int nt = LD * LD;
    unsigned long long* s64 = reinterpret_cast<unsigned long long*>(smem);
    uint32_t* s32 = reinterpret_cast<uint32_t*>(smem + sizeof(unsigned long long) * nt);
    for (int i = threadIdx.x; i < nt; i += NT) {
        s64[i] = 0ull;
        s32[i] = 0u;
    }
    __syncthreads();
    int miss = 0;
    const int64_t stride = (int64_t)gridDim.x * CHUNK_QUADS;
    for (int64_t base = (int64_t)blockIdx.x * CHUNK_QUADS; base < P.nquads; base += stride) {
        const int64_t q = base + threadIdx.x;
        if (q < P.nquads) {
            int32_t x0, y, z;
            int64_t bi;
            quad_coords(P, q, x0, y, z, bi);
            float ff[4], uu[12];
            load_quad(P, bi, ff, uu);
            Cell c[4];
            quad_cells(P, x0, y, z, uu, c);
            Corners cr[4];
            gather_n<FULLWIN, 4>(P.g, c, cr, miss);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                BS4 bi_, bj_;
                if (BSPLINE) {
                    bi_ = bspline_bins<false>(ff[k], B);
                    bj_ = bspline_bins<false>(interp(cr[k], c[k]), B);
                } else {
                    bi_ = generic_bins<false>(P.p, (double)ff[k]);
                    bj_ = generic_bins<false>(P.p, interp_f64(cr[k], c[k]));
                }
                float kj[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) kj[b] = bj_.k[b] * P.fix_scale;
                uint32_t* h = s32 + (bi_.m_lo + PAD) * LD + (bj_.m_lo + PAD);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        // round-to-nearest fixed point without a conversion instruction
                        atomicAdd(h + a * LD + b,
                                  (uint32_t)(__float_as_int(fmaf(bi_.k[a], kj[b], 12582912.0f)) - 0x4B400000));
                    }
                }
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nt; i += NT) {
            s64[i] += s32[i];
            s32[i] = 0u;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < B * B; i += NT) {
        const unsigned long long v = s64[(i / B + PAD) * LD + (i % B) + PAD];
        if (v) atomicAdd(&P.hist[i], v);
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

// ------------------------------------------------------------------ pass 2
template <bool BSPLINE, bool FULLWIN>
__global__ void __launch_bounds__(NT, 3) k_step_mi_grad(const Params P) {
    extern __shared__ __align__(16) float sg[];
    const int B = P.p.bins;
    const int LD = B + 2 * PAD;
    {
        const double* gh = P.table + B * B + 2 * B;
        for (int q = threadIdx.x; q < LD * LD; q += NT) {
            const int m = q / LD - PAD, n = q % LD - PAD;
            sg[q] = (m >= 0 && m < B && n >= 0 && n < B) ? (float)gh[m * B + n] : 0.0f;
        }
        __syncthreads();
    }
    int miss = 0;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t q = (int64_t)blockIdx.x * NT + threadIdx.x; q < P.nquads; q += stride) {
        int32_t x0, y, z;
        int64_t bi;
        quad_coords(P, q, x0, y, z, bi);
        float ff[4], uu[12];
        load_quad(P, bi, ff, uu);
        Cell c[4];
        quad_cells(P, x0, y, z, uu, c);
        Corners cr[4];
        gather_n<FULLWIN, 4>(P.g, c, cr, miss);
        float go[12];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float d[3];
            const float mw = interp_grad(cr[k], c[k], d);
            BS4 bi_, bj_;
            if (BSPLINE) {
                bi_ = bspline_bins<false>(ff[k], B);
                bj_ = bspline_bins<true>(mw, B);
            } else {
                bi_ = generic_bins<false>(P.p, (double)ff[k]);
                bj_ = generic_bins<true>(P.p, interp_f64(cr[k], c[k]));
            }
            // dL/dJ = sum_m kappa_i[m] sum_n ghat[m][n] omega_j[n]   (mi.hpp:409-418)
            const float* gr = sg + (bi_.m_lo + PAD) * LD + (bj_.m_lo + PAD);
            float gj = 0.0f;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                float acc = gr[a * LD] * bj_.w[0];
                acc = fmaf(gr[a * LD + 1], bj_.w[1], acc);
                acc = fmaf(gr[a * LD + 2], bj_.w[2], acc);
                acc = fmaf(gr[a * LD + 3], bj_.w[3], acc);
                gj = fmaf(bi_.k[a], acc, gj);
            }
            go[3 * k] = P.g.dscale[0] * d[0] * gj;
            go[3 * k + 1] = P.g.dscale[1] * d[1] * gj;
            go[3 * k + 2] = P.g.dscale[2] * d[2] * gj;
        }
        float4* out = reinterpret_cast<float4*>(P.g_u + 3 * ((bi - (P.z_begin - P.buf_z0) * P.plane)));
        out[0] = make_float4(go[0], go[1], go[2], go[3]);
        out[1] = make_float4(go[4], go[5], go[6], go[7]);
        out[2] = make_float4(go[8], go[9], go[10], go[11]);
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

__global__ void k_hist_to_raw(const unsigned long long* h, int n, double inv_scale, double* raw) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
        raw[i] += (double)h[i] * inv_scale;
}

}  // namespace mstep

// Returns FFDP_OK and launches, or a non-zero code when the quad path does not apply
// (the caller then uses the scalar kernels of mi.cu).
bool mi_quad_path_applies(const ffdp_dims& d, const ffdp_slab& s, const ffdp_parzen& k) {
    // 32-bit quad indices and in-plane offsets
    return d.nx % 4 == 0 && k.bins <= 64 && (int64_t)d.nx * d.ny < (1LL << 31) &&
           (d.nx / 4) * d.ny * (s.z_end - s.z_begin) < (1LL << 31);
}

static mstep::Params make_params(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s,
                                 const ffdp_image_window& m, const ffdp_sampler_args& args, const ffdp_parzen& k) {
    mstep::Params P;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    P.g = make_geom(m, out, args);
    P.p = make_parzen_dev(k);
    P.f = f;
    P.u = u;
    P.g_u = nullptr;
    P.table = nullptr;
    P.hist = nullptr;
    P.miss = nullptr;
    P.nx = (int32_t)d.nx;
    P.ny = (int32_t)d.ny;
    P.qpr = (int32_t)(d.nx / 4);
    P.div_qpr = make_fastdiv((uint32_t)P.qpr);
    P.div_ny = make_fastdiv((uint32_t)d.ny);
    P.plane = d.nx * d.ny;
    P.z_begin = s.z_begin;
    P.buf_z0 = s.buf_z0;
    P.nquads = (int64_t)P.qpr * d.ny * (s.z_end - s.z_begin);
    P.fix_scale = k.kind == FFDP_PARZEN_BSPLINE3 ? 8388608.0f : k.kind == FFDP_PARZEN_GAUSSIAN ? 4194304.0f
                                                                                                 : 2097152.0f;
    return P;
}

int mi_quad_hist(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, double* raw, int32_t* miss, cudaStream_t st) {
    using namespace mstep;
    Params P = make_params(f, u, d, s, m, args, k);
    const int B = k.bins;
    unsigned long long* h = (unsigned long long*)scratch_alloc(sizeof(unsigned long long) * B * B, st);
    if (!h) return set_error(FFDP_CUDA, "step_mi: scratch allocation failed");
    cudaMemsetAsync(h, 0, sizeof(unsigned long long) * B * B, st);
    P.hist = h;
    P.miss = miss;
    const size_t smem = (sizeof(unsigned long long) + sizeof(uint32_t)) * (B + 2 * PAD) * (B + 2 * PAD);
    const int64_t chunks = (P.nquads + CHUNK_QUADS - 1) / CHUNK_QUADS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, 6LL * num_sms()));
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
    const bool bs = k.kind == FFDP_PARZEN_BSPLINE3;
    if (bs && full)
        k_step_mi_hist<true, true><<<grid, NT, smem, st>>>(P);
    else if (bs)
        k_step_mi_hist<true, false><<<grid, NT, smem, st>>>(P);
    else if (full)
        k_step_mi_hist<false, true><<<grid, NT, smem, st>>>(P);
    else
        k_step_mi_hist<false, false><<<grid, NT, smem, st>>>(P);
    k_hist_to_raw<<<(B * B + 255) / 256, 256, 0, st>>>(h, B * B, 1.0 / P.fix_scale, raw);
    scratch_free(h, st);
    return check_launch("step_mi_hist");
}

int mi_quad_grad(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, const double* table, float* g_u, int32_t* miss,
                 cudaStream_t st) {
    using namespace mstep;
    Params P = make_params(f, u, d, s, m, args, k);
    P.table = table;
    P.g_u = g_u;
    P.miss = miss;
    const int B = k.bins;
    const size_t smem = sizeof(float) * (B + 2 * PAD) * (B + 2 * PAD);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P.nquads + NT - 1) / NT, 6LL * num_sms()));
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
    const bool bs = k.kind == FFDP_PARZEN_BSPLINE3;
    if (bs && full)
        k_step_mi_grad<true, true><<<grid, NT, smem, st>>>(P);
    else if (bs)
        k_step_mi_grad<true, false><<<grid, NT, smem, st>>>(P);
    else if (full)
        k_step_mi_grad<false, true><<<grid, NT, smem, st>>>(P);
    else
        k_step_mi_grad<false, false><<<grid, NT, smem, st>>>(P);
    return check_launch("step_mi_grad");
}

}  // namespace ffdp
