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
// Work unit: a warp covers 32 consecutive x voxels of 4 consecutive rows (needs the
// zero-bordered moving image, ffdp_pad_window; dense images use mi.cu's scalar path).
// Histogram: 16 joint products per voxel rounded to fixed point by one denormal FMUL
// (the bits of the product are the integer) and added with native shared u32 atomics into lane-private
// copies; every 1024 voxels per copy the CTA folds the copies into a u64 shared
// histogram (the scale keeps every counter below 2^32 in between), and at the end into
// the global u64 histogram. Integer sums: deterministic. The marginals
// are not accumulated here: finalize_histogram derives p_i, p_j from the joint
// (mi.hpp:181-196), so the fused step needs only the B*B joint payload.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ffdp_common.cuh"

// FFDP_MI_GB: corner-gather batch of the B-spline pass 1 (k_mi_hist_bs)
#ifndef FFDP_MI_GB
#define FFDP_MI_GB 4
#endif
// FFDP_MI_ZORDER = 1: z-major unit order (see unit_coords)
#ifndef FFDP_MI_ZORDER
#define FFDP_MI_ZORDER 0
#endif

namespace ffdp {
namespace mstep {


constexpr int NT = 256;  // pass 2: 8 warps x 128 voxels per CTA iteration

struct Params {
    Geom g;
    ParzenDev p;
    const float* f;
    const float* u;
    float* g_u;
    const double* table;
    float4* rec;               // pass-1 records (Mw, dscale * dMw/dfrac) per interior voxel, or null
    unsigned long long* hist;  // global u64 [B*B]
    unsigned int* done;        // fused finalize: CTA completion counter (after hist), or null
    double* fin_table;         // fused finalize: ffdp_mi_finalize's table, or null (separate finalize)
    double* raw_out;           // fused finalize: raw joint histogram out (may be null)
    double upstream;
    int32_t* miss;
    int32_t nx, ny, nxb, nyq, nzs;  // lattice, 32-wide x blocks, 4-row groups, interior planes
    FastDiv div_nxb, div_nyq, div_nzs;
    int32_t zorder;                 // z-major unit order (unit_coords)
    int64_t plane, z_begin, buf_z0;
    int64_t nunits;
    float fix_scale;           // 2^23 or 2^21 (bspline, k_mi_hist_bs) / 2^22 (gaussian) / 2^21 (delta)
};

// B-spline weights at bins m_lo..m_lo+3 for one intensity, fp32 (the kernel is C2,
// so fp32 rounding of the bin coordinate only perturbs weights at 1e-7).
struct BS4 {
    int32_t m_lo;
    float k[4], w[4];
};

// c6: 1/6, or 1/6 times the histogram fixed-point scale (folded into the weights).
template <bool OMEGA>
__device__ __forceinline__ BS4 bspline_bins(float v, int B, float c6 = 1.0f / 6.0f) {
    BS4 r;
    const float s = fmaf(v, (float)B, -0.5f);
    const float fl = floorf(s);
    const float ph = s - fl;
    // clamp keeps the 4x4 footprint inside the padded tables even for inputs outside
    // [0,1] (which the reference rejects, mi.hpp:170-179)
    r.m_lo = min(max((__float_as_int(fl + 12582912.0f) - 0x4B400000) - 1, -2), B - 2);
    const float q = 1.0f - ph;
    const float p2 = ph * ph, p3 = p2 * ph, q2 = q * q;
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

// Work unit of a warp: 32 consecutive x voxels (lane = x offset) of 4 consecutive rows.
// Consecutive lanes sample neighbouring source positions, so each corner load of the
// warp touches one or two 128-B lines (coalesced gather); a thread's 4 voxels are
// y-neighbours, so their Parzen footprints usually share bins (histogram aggregation).
struct Unit {
    int32_t x, y0, z;   // lattice coordinates (z global)
    int64_t bi;         // buffer index of (x, y0, z)
    bool vx;            // x inside the lattice
};

__device__ __forceinline__ Unit unit_coords(const Params& P, uint32_t unit, int lane) {
    Unit w;
    const uint32_t r1 = fdiv(unit, P.div_nxb);
    const int32_t xb = (int32_t)(unit - r1 * P.nxb);
    uint32_t zz;
    int32_t yq;
    if (P.zorder) {
        // units ordered x block, then z, then 4-row group: the two output planes that share a
        // moving-image plane (the trilinear z corners) are processed back to back, so its
        // lines come from L2 the second time (plane-major order re-reads them from HBM a
        // whole plane of traffic later once a plane outgrows the L2: 1760^2 planes, 81 vs
        // 92 GB read per pass 1 at configs[4])
        const uint32_t yqu = fdiv(r1, P.div_nzs);
        zz = r1 - yqu * (uint32_t)P.nzs;
        yq = (int32_t)yqu;
    } else {
        zz = fdiv(r1, P.div_nyq);
        yq = (int32_t)(r1 - zz * P.nyq);
    }
    w.x = xb * 32 + lane;
    w.y0 = yq * 4;
    w.z = (int32_t)zz + (int32_t)P.z_begin;
    w.vx = w.x < P.nx;
    w.bi = ((int64_t)zz + P.z_begin - P.buf_z0) * P.plane + (int64_t)w.y0 * P.nx + (w.vx ? w.x : 0);
    return w;
}

// Padded bin tables: bin m lives at row m + PAD of a (B + 2 PAD)^2 table, so the
// 4 x 4 footprint of any intensity in [0, 1] (m_lo >= -2, m_lo + 3 <= B + 1) needs no
// bounds checks; out-of-range bins have zero weight and the pad rows are never read
// back (histogram) or hold zeros (ghat).
constexpr int PAD = 2;

__device__ __forceinline__ void load_unit(const Params& P, const Unit& w, float (&ff)[4], float (&uu)[12],
                                          bool (&ok)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        ok[k] = w.vx && (w.y0 + k) < P.ny;
        const int64_t i = w.bi + (int64_t)k * P.nx;
        ff[k] = ok[k] ? __ldg(P.f + i) : 0.0f;
        uu[3 * k] = ok[k] ? __ldg(P.u + 3 * i) : 0.0f;
        uu[3 * k + 1] = ok[k] ? __ldg(P.u + 3 * i + 1) : 0.0f;
        uu[3 * k + 2] = ok[k] ? __ldg(P.u + 3 * i + 2) : 0.0f;
    }
}

__device__ __forceinline__ void unit_cells(const Params& P, const Unit& w, const float (&uu)[12], Cell (&c)[4]) {
    RowBase rb;
    rb.init(P.g, w.x, w.y0, w.z);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k) rb.step_y(P.g);
        c[k] = rb.cell(P.g, uu[3 * k], uu[3 * k + 1], uu[3 * k + 2]);
    }
}

// ------------------------------------------------------------------ pass 1
// Histogram privatisation. The lanes of a warp are x-neighbours, so they often fall in the
// same bins, and shared atomics from several lanes of one instruction to the same address
// serialise (8 lanes on one address cost ~8x a conflict-free instruction). Lane l
// therefore adds into copy l % HCOPY of the counters; copies are HSTRIDE words apart with
// HSTRIDE = 1 (mod 32), so lanes adding to the same bin of their own copies hit distinct
// banks. Each copy only takes the voxels of HNT / HCOPY threads, which sets the fold
// interval.
#ifndef FFDP_MI_HIST_NT
#define FFDP_MI_HIST_NT 1024
#endif
#ifndef FFDP_MI_HIST_COPIES
#define FFDP_MI_HIST_COPIES 16
#endif
constexpr int HNT = FFDP_MI_HIST_NT;
constexpr int HCOPY = FFDP_MI_HIST_COPIES;
// voxels one copy takes per CTA iteration, and iterations between folds: a voxel adds
// at most max(kappa)^2 * scale < 2^22 to one counter (B-spline (2/3)^2 * 2^23, gaussian
// 0.64 * 2^22, delta 2^21), so 1024 voxels per copy per fold keep counters below 2^32.
constexpr int HVOX_PER_COPY_ITER = (HNT / HCOPY) * 4;
constexpr int HFOLD_ITERS = 1024 / HVOX_PER_COPY_ITER > 0 ? 1024 / HVOX_PER_COPY_ITER : 1;

__host__ __device__ constexpr int hist_ld(int B) { return B + 2 * PAD; }
__host__ __device__ constexpr int hist_stride(int B) {
    return ((hist_ld(B) * hist_ld(B) + 31) / 32) * 32 + (32 / HCOPY);
}
constexpr size_t kMaxHistSmem = 226 * 1024;  // leaves room for the static shared variables
inline size_t hist_smem_bytes(int B) {
    return sizeof(unsigned long long) * B * B + sizeof(uint32_t) * (size_t)HCOPY * hist_stride(B);
}

// REC: also write the voxel's record (Mw, dscale * dMw/dfrac) for the streaming pass 2
// (k_step_mi_grad_rec): 16 more bytes written here save pass 2 the whole warp sampling.
template <bool BSPLINE, bool FULLWIN, bool REC>
__global__ void __launch_bounds__(HNT, 1) k_step_mi_hist(const Params P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = P.p.bins;
    const int LD = hist_ld(B);
    const int CS = hist_stride(B);
    unsigned long long* s64 = reinterpret_cast<unsigned long long*>(smem);  // interior B x B
    uint32_t* s32 = reinterpret_cast<uint32_t*>(smem + sizeof(unsigned long long) * B * B);
    for (int i = threadIdx.x; i < B * B; i += HNT) s64[i] = 0ull;
    for (int i = threadIdx.x; i < HCOPY * CS; i += HNT) s32[i] = 0u;
    __syncthreads();
    int miss = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* mine = s32 + (lane % HCOPY) * CS + PAD * LD + PAD;
    const int64_t stride = (int64_t)gridDim.x * (HNT / 32);
    int iter = 0;
    for (int64_t base = (int64_t)blockIdx.x * (HNT / 32); base < P.nunits; base += stride) {
        const int64_t unit = base + warp;
        if (unit < P.nunits) {
            const Unit w = unit_coords(P, (uint32_t)unit, lane);
            float ff[4], uu[12];
            bool ok[4];
            load_unit(P, w, ff, uu, ok);
            Cell c[4];
            unit_cells(P, w, uu, c);
            Corners cr[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) cr[k] = gather_pad<FULLWIN>(P.g, c[k], miss);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // Fixed point by a denormal product: with the weights pre-scaled by 2^-63 and
                // scale * 2^-86, kI * kJ lands at (scale * kI * kJ) * 2^-149, whose IEEE bits
                // ARE round(scale * kI * kJ) (exact for values < 2^24, FMUL rounds to nearest;
                // denormals are not flushed: no -ftz). One FMUL per product, no conversion.
                BS4 bI, bJ;
                const float sc = ok[k] ? P.fix_scale * 0x1p-86f : 0.0f;  // outside the lattice: adds 0
                if (BSPLINE) {
                    float mw;
                    if (REC) {
                        float d[3];
                        mw = interp_grad(cr[k], c[k], d);
                        if (ok[k])
                            P.rec[w.bi + (int64_t)k * P.nx - (P.z_begin - P.buf_z0) * P.plane] =
                                make_float4(mw, P.g.dscale[0] * d[0], P.g.dscale[1] * d[1], P.g.dscale[2] * d[2]);
                    } else {
                        mw = interp(cr[k], c[k]);
                    }
                    bI = bspline_bins<false>(ff[k], B, (1.0f / 6.0f) * 0x1p-63f);
                    bJ = bspline_bins<false>(mw, B, sc * (1.0f / 6.0f));
                } else {
                    bI = generic_bins<false>(P.p, (double)ff[k]);
                    bJ = generic_bins<false>(P.p, interp_f64(cr[k], c[k]));
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        bI.k[b] *= 0x1p-63f;
                        bJ.k[b] *= sc;
                    }
                }
                uint32_t* h = mine + bI.m_lo * LD + bJ.m_lo;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) atomicAdd(h + a * LD + b, __float_as_uint(bI.k[a] * bJ.k[b]));
            }
        }
        if (++iter == HFOLD_ITERS || base + stride >= P.nunits) {
            // fold the interior B x B counters of every copy (the pad counters take the
            // weight of bins outside [0, B), which the reference ignores: they may wrap,
            // they are never read)
            iter = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < B * B; i += HNT) {
                const int q = (i / B + PAD) * LD + (i % B) + PAD;
                unsigned long long acc = 0ull;
#pragma unroll 8
                for (int cp = 0; cp < HCOPY; ++cp) {
                    acc += s32[cp * CS + q];
                    s32[cp * CS + q] = 0u;
                }
                s64[i] += acc;
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < B * B; i += HNT) {
        const unsigned long long v = s64[i];
        if (v) atomicAdd(&P.hist[i], v);
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

// ------------------------------------------------------------------ pass 1, B-spline
// The B-spline pass 1 with the bin count as a compile-time constant (BC > 0; BC = 0 reads
// it at run time). Differences from the generic kernel above, each worth instructions per
// voxel in an issue-bound loop:
//  * a 4-bin histogram pad (HPAD): a voxel outside the lattice gets the intensity -1,
//    whose bins clamp to rows -4..-1, all pad, so it needs no weight masking; with the
//    masking gone the fixed-point scales fold into the B-spline coefficients;
//  * per-unit row pointers for F, u and the records (one 64-bit add per row);
//  * with BC > 0 every counter offset of the 4 x 4 footprint is an immediate.
// Histogram pad: 4 (out-of-lattice voxels get intensity -1, all of whose bins land in the
// pad) or 2 (the minimum for in-range intensities; out-of-lattice voxels are redirected
// to 4 dummy rows after the table). 2 keeps the shared footprint under the 100 KB
// carve-out, leaving more L1 for the gather.
#ifndef FFDP_MI_HPAD
#define FFDP_MI_HPAD 2
#endif
constexpr int HPAD = FFDP_MI_HPAD;
constexpr int HDUMMY = HPAD == 2 ? 4 : 0;  // dummy rows per copy (HPAD 2)
// Fixed-point scale 2^S (S odd):
// both weights are pre-scaled by 2^(S-149)/2 so that kI * kJ lands at 2^S kI kJ * 2^-149.
// A voxel adds at most (2/3)^2 * 2^S to one counter, so a copy takes 2^(32-S) * 2^11
// voxels between folds without wrapping (S = 21: 4096, S = 23: 1024).
// The scale is chosen per call: 2^23 below FFDP_MI_BS_LARGE_MIN interior voxels, 2^21
// from there on (half the fold barriers: 0.160 vs 0.178 ms at 256^3). The coarser grid
// rounds products under 2^-22 of a unit weight away, which only matters for a histogram
// of few voxels: measured against the oracle, g_u agrees to 1.4e-6 (140k voxels) ..
// 2.5e-6 (96^3) at either scale, while 4k-voxel slabs of the sharded step drift past the
// 1e-5 loss gate over a multi-iteration stage at 2^21.
#ifndef FFDP_REC_STREAM
#define FFDP_REC_STREAM 0
#endif
#ifndef FFDP_MI_BS_LARGE_MIN
#define FFDP_MI_BS_LARGE_MIN (1 << 17)
#endif
__host__ __device__ constexpr float bs_wscale(int S) { return S == 23 ? 0x1p-63f : S == 21 ? 0x1p-64f : 0x1p-65f; }
__host__ __device__ constexpr int bs_fold_iters(int S) {
    return (1024 << (23 - S)) / HVOX_PER_COPY_ITER > 0 ? (1024 << (23 - S)) / HVOX_PER_COPY_ITER : 1;
}
__host__ __device__ constexpr int bs_ld(int B) { return B + 2 * HPAD; }
__host__ __device__ constexpr int bs_stride(int B) {
    return ((bs_ld(B) * (bs_ld(B) + HDUMMY) + 31) / 32) * 32 + (32 / HCOPY);
}
inline size_t bs_smem_bytes(int B) {
    return sizeof(unsigned long long) * B * B + sizeof(uint32_t) * (size_t)HCOPY * bs_stride(B);
}

// Cubic B-spline weights of the 4 bins m_lo..m_lo+3 scaled by C (mi.hpp:28-140, bspline3),
// the scale folded into the polynomial coefficients.
template <int BC>
__device__ __forceinline__ int32_t bspline_scaled(float v, int B, float C, float (&k)[4]) {
    const float fb = BC > 0 ? (float)BC : (float)B;
    const float s = fmaf(v, fb, -0.5f);
    const float fl = floorf(s);
    const float ph = s - fl;
    const float q = 1.0f - ph;
    const float p2 = ph * ph, p3 = p2 * ph;
    k[0] = (q * q) * (q * (C / 6.0f));
    k[1] = fmaf(3.0f * (C / 6.0f), p3, fmaf(-6.0f * (C / 6.0f), p2, 4.0f * (C / 6.0f)));
    k[2] = fmaf(-3.0f * (C / 6.0f), p3, fmaf(3.0f * (C / 6.0f), p2, fmaf(3.0f * (C / 6.0f), ph, C / 6.0f)));
    k[3] = p3 * (C / 6.0f);
    const int32_t m = (__float_as_int(fl + 12582912.0f) - 0x4B400000) - 1;
    return min(max(m, -HPAD), (BC > 0 ? BC : B) + HPAD - 4);
}

template <bool FULLWIN, bool REC, int BC, int OFF32, int S>
__global__ void __launch_bounds__(HNT, 1) k_mi_hist_bs(const Params P) {
    static_assert(S == 21 || S == 23, "odd scale exponent: equal weight pre-scales");
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = BC > 0 ? BC : P.p.bins;
    const int LD = bs_ld(B);
    const int CS = bs_stride(B);
    unsigned long long* s64 = reinterpret_cast<unsigned long long*>(smem);  // interior B x B
    uint32_t* s32 = reinterpret_cast<uint32_t*>(smem + sizeof(unsigned long long) * B * B);
    for (int i = threadIdx.x; i < B * B; i += HNT) s64[i] = 0ull;
    for (int i = threadIdx.x; i < HCOPY * CS; i += HNT) s32[i] = 0u;
    __syncthreads();
    int miss = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* mine = s32 + (lane % HCOPY) * CS + HPAD * LD + HPAD;
    const int64_t stride = (int64_t)gridDim.x * (HNT / 32);
    const int64_t zrec = (P.z_begin - P.buf_z0) * P.plane;  // records cover the interior planes
    // The unit's F and u rows. (Loading them one unit ahead -- in registers across the
    // gathers, in registers issued after this unit's interpolations so they fly during the
    // histogram updates, or staged in shared memory by cp.async -- measured slower: 0.206,
    // 0.187 and 0.200 vs 0.177 ms at 256^3; the first spills at 64 registers, the third
    // takes L1 from the gather. With 768 or 896 threads the registers allow the second:
    // 0.178 / 0.180 ms, no better than 1024 threads without it.)
    struct Ld {
        Unit w;
        float ff[4], uu[12];
        bool ok[4];
    };
    auto load = [&](int64_t unit, Ld& L) {
        L.w = unit_coords(P, (uint32_t)unit, lane);
        const float* fp = P.f + L.w.bi;
        const float* up = P.u + 3 * L.w.bi;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            L.ok[k] = L.w.vx && (L.w.y0 + k) < P.ny;
            L.ff[k] = L.ok[k] ? __ldg(fp) : -1.0f;  // -1: every bin in the pad rows (HPAD 4)
            L.uu[3 * k] = L.ok[k] ? __ldg(up) : 0.0f;
            L.uu[3 * k + 1] = L.ok[k] ? __ldg(up + 1) : 0.0f;
            L.uu[3 * k + 2] = L.ok[k] ? __ldg(up + 2) : 0.0f;
            fp += P.nx;
            up += 3 * P.nx;
        }
    };
    int iter = 0;
    for (int64_t base = (int64_t)blockIdx.x * (HNT / 32); base < P.nunits; base += stride) {
        const int64_t unit = base + warp;
        if (unit < P.nunits) {
            Ld L;
            load(unit, L);
            const Unit& w = L.w;
            const float(&ff)[4] = L.ff;
            const bool(&ok)[4] = L.ok;
            float4* rp = P.rec + (w.bi - zrec);
            Cell c[4];
            unit_cells(P, w, L.uu, c);
            // FFDP_MI_GB voxels' corners are gathered at once (4: all of the unit's 32 loads in
            // flight; 2: half the corner registers live)
            Corners cr[FFDP_MI_GB];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k % FFDP_MI_GB == 0) {
#pragma unroll
                    for (int q = 0; q < FFDP_MI_GB; ++q) cr[q] = gather_pad<FULLWIN, OFF32>(P.g, c[k + q], miss);
                }
                const Corners& ck = cr[k % FFDP_MI_GB];
                // Fixed point by a denormal product: with both weights pre-scaled by
                // bs_wscale(S), kI * kJ lands at (2^S kI kJ) * 2^-149, whose IEEE bits ARE
                // round(2^S kI kJ) (FMUL rounds to nearest; no -ftz).
                float mw;
                if (REC) {
                    float d[3];
                    mw = interp_grad(ck, c[k], d);
                    if (ok[k]) {
                        const float4 rv = make_float4(mw, P.g.dscale[0] * d[0], P.g.dscale[1] * d[1], P.g.dscale[2] * d[2]);
                        // FFDP_REC_STREAM: evict-first stores (the records are read once, by pass 2),
                        // so the streaming 16 B/voxel do not push the moving image's lines out of L2
                        if (FFDP_REC_STREAM)
                            __stcs(rp, rv);
                        else
                            *rp = rv;
                    }
                    rp += P.nx;
                } else {
                    mw = interp(ck, c[k]);
                }
                float kI[4], kJ[4];
                const int32_t mi = bspline_scaled<BC>(ff[k], B, bs_wscale(S), kI);
                const int32_t mj = bspline_scaled<BC>(mw, B, bs_wscale(S), kJ);
                // HPAD 2: voxels outside the lattice add into the copy's dummy rows
                uint32_t* h = (HPAD == 2 && !ok[k]) ? mine - HPAD * LD - HPAD + LD * LD : mine + mi * LD + mj;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        atomicAdd(h + a * LD + b, __float_as_uint(kI[a] * kJ[b]));
            }
        }
        if (++iter == bs_fold_iters(S) || base + stride >= P.nunits) {
            // fold the interior B x B counters of every copy (pad counters take the weight of
            // bins outside [0, B) and of voxels outside the lattice: never read, may wrap)
            iter = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < B * B; i += HNT) {
                const int q = (i / B + HPAD) * LD + (i % B) + HPAD;
                unsigned long long acc = 0ull;
#pragma unroll 8
                for (int cp = 0; cp < HCOPY; ++cp) {
                    acc += s32[cp * CS + q];
                    s32[cp * CS + q] = 0u;
                }
                s64[i] += acc;
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < B * B; i += HNT) {
        const unsigned long long v = s64[i];
        if (v) atomicAdd(&P.hist[i], v);
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
    if (P.fin_table) {
        // fused finalize (single-rank step): the last CTA to finish converts the global
        // histogram, runs finalize_histogram / histogram_mi / the ghat table
        // (mi_finalize_block) and leaves the histogram and the counter zeroed
        __shared__ unsigned s_last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(P.done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            double* rs = reinterpret_cast<double*>(smem);  // the s64 area: B*B doubles
            const double inv = 1.0 / (double)P.fix_scale;
            for (int i = threadIdx.x; i < B * B; i += HNT) {
                const double v = (double)__ldcg(&P.hist[i]) * inv;
                rs[i] = v;
                if (P.raw_out) P.raw_out[i] = v;
                P.hist[i] = 0ull;
            }
            if (threadIdx.x == 0) *P.done = 0u;
            mi_finalize_block(rs, B, P.upstream, P.fin_table, reinterpret_cast<double*>(s32));
        }
    }
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
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * (NT / 32);
    for (int64_t unit = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); unit < P.nunits; unit += stride) {
        const Unit w = unit_coords(P, (uint32_t)unit, lane);
        float ff[4], uu[12];
        bool ok[4];
        load_unit(P, w, ff, uu, ok);
        Cell c[4];
        unit_cells(P, w, uu, c);
        Corners cr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) cr[k] = gather_pad<FULLWIN>(P.g, c[k], miss);
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
            if (ok[k]) {
                float* o = P.g_u + 3 * (w.bi + (int64_t)k * P.nx - (P.z_begin - P.buf_z0) * P.plane);
                o[0] = P.g.dscale[0] * d[0] * gj;
                o[1] = P.g.dscale[1] * d[1] * gj;
                o[2] = P.g.dscale[2] * d[2] * gj;
            }
        }
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

// Pass 2 for the B-spline kernel, re-sampling the warp (the record-free path: configs[4]
// has no room for 16 B/voxel of records next to its 119 GB of F, M, u and g_u). The unit
// walk of k_mi_hist_bs (per-unit F / u / g_u row pointers, unsigned 32-bit gather offsets
// when the window allows) and the ghat dot of k_step_mi_grad_rec (the table as 4
// column-shifted shared copies: one LDS.128 per footprint row). mi.hpp:392-421.
__host__ __device__ constexpr int grad_tab_floats(int B);

#ifndef FFDP_MI_G2_MINB
#define FFDP_MI_G2_MINB 3
#endif
template <bool FULLWIN, int BC, int OFF32>
__global__ void __launch_bounds__(NT, FFDP_MI_G2_MINB) k_mi_grad_bs(const Params P) {
    extern __shared__ __align__(16) float sg[];
    const int B = BC > 0 ? BC : P.p.bins;
    const int LD = B + 2 * PAD;           // rows
    const int CP = (LD + 3) / 4 * 4;      // row pitch (floats)
    const int CS = LD * CP;               // copy size
    {
        const double* gh = P.table + B * B + 2 * B;
        for (int q = threadIdx.x; q < 4 * CS; q += NT) {
            const int c = q / CS, r = (q % CS) / CP, k = q % CP;
            const int m = r - PAD, nn = k + c - PAD;
            sg[q] = (m >= 0 && m < B && nn >= 0 && nn < B) ? (float)gh[m * B + nn] : 0.0f;
        }
        __syncthreads();
    }
    int miss = 0;
    const int lane = threadIdx.x & 31;
    const float ds0 = P.g.dscale[0], ds1 = P.g.dscale[1], ds2 = P.g.dscale[2];
    const int64_t zout = (P.z_begin - P.buf_z0) * P.plane;  // g_u covers the interior planes
    const int64_t stride = (int64_t)gridDim.x * (NT / 32);
    for (int64_t unit = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); unit < P.nunits; unit += stride) {
        const Unit w = unit_coords(P, (uint32_t)unit, lane);
        const float* fp = P.f + w.bi;
        const float* up = P.u + 3 * w.bi;
        float ff[4], uu[12];
        bool ok[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            ok[k] = w.vx && (w.y0 + k) < P.ny;
            ff[k] = ok[k] ? __ldg(fp + k * P.nx) : 0.0f;
            uu[3 * k] = ok[k] ? __ldg(up + 3 * k * P.nx) : 0.0f;
            uu[3 * k + 1] = ok[k] ? __ldg(up + 3 * k * P.nx + 1) : 0.0f;
            uu[3 * k + 2] = ok[k] ? __ldg(up + 3 * k * P.nx + 2) : 0.0f;
        }
        Cell c[4];
        unit_cells(P, w, uu, c);
        Corners cr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) cr[k] = gather_pad<FULLWIN, OFF32>(P.g, c[k], miss);
        float* op = P.g_u + 3 * (w.bi - zout);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float d[3];
            const float mw = interp_grad(cr[k], c[k], d);
            const BS4 bi = bspline_bins<false>(ff[k], B);
            const BS4 bj = bspline_bins<true>(mw, B);
            // dL/dJ = sum_m kappa_i[m] sum_n ghat[m][n] omega_j[n]   (mi.hpp:409-418)
            const int n0 = bj.m_lo + PAD;
            const float4* gr =
                reinterpret_cast<const float4*>(sg + (n0 & 3) * CS + (bi.m_lo + PAD) * CP + (n0 & ~3));
            float gj = 0.0f;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const float4 g = gr[a * (CP / 4)];
                float acc = g.x * bj.w[0];
                acc = fmaf(g.y, bj.w[1], acc);
                acc = fmaf(g.z, bj.w[2], acc);
                acc = fmaf(g.w, bj.w[3], acc);
                gj = fmaf(bi.k[a], acc, gj);
            }
            if (ok[k]) {
                float* o = op + 3 * k * P.nx;
                o[0] = ds0 * d[0] * gj;
                o[1] = ds1 * d[1] * gj;
                o[2] = ds2 * d[2] * gj;
            }
        }
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (threadIdx.x & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

// Pass 2 from the pass-1 records: F and (Mw, dscale * dMw/dfrac) are streamed, dL/dMw
// from the ghat table (mi.hpp:392-421, B-spline), g_u = record.yzw * dL/dMw. No gather,
// no coordinates: 32 B/voxel of pure streaming (F 4 + record 16 in, g_u 12 out).
// The ghat table sits in shared memory as 4 column-shifted copies (copy c holds
// ghat_pad[r][k + c]), so the 4 consecutive bins n0..n0+3 of a row are one aligned
// 16-byte load from copy n0 % 4: 4 LDS.128 per voxel instead of 16 scalar loads.
// VEC: 4 voxels per thread with 16-byte loads and stores (aligned buffers), two groups
// in flight per iteration.
__host__ __device__ constexpr int grad_tab_floats(int B) { return 4 * (B + 2 * PAD) * ((B + 2 * PAD + 3) / 4 * 4); }

#ifndef FFDP_GR_HINT
#define FFDP_GR_HINT 0
#endif
#ifndef FFDP_GR_MINB
#define FFDP_GR_MINB 2
#endif
#ifndef FFDP_GR_CTAS
#define FFDP_GR_CTAS 2
#endif
#ifndef FFDP_GR_UNROLL
#define FFDP_GR_UNROLL 2
#endif
// streaming (read-once / write-once) cache hints for the records, F and g_u (FFDP_GR_HINT)
__device__ __forceinline__ float4 ld_stream(const float4* p) { return FFDP_GR_HINT ? __ldcs(p) : __ldg(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    if (FFDP_GR_HINT)
        __stcs(p, v);
    else
        *p = v;
}

template <bool VEC>
__global__ void __launch_bounds__(256, FFDP_GR_MINB) k_step_mi_grad_rec(const float* __restrict__ f, const float4* __restrict__ rec,
                                                          float* __restrict__ g_u, int64_t n, const double* table,
                                                          int B) {
    extern __shared__ __align__(16) float sg[];
    const int LD = B + 2 * PAD;            // rows
    const int CP = (LD + 3) / 4 * 4;       // row pitch (floats)
    const int CS = LD * CP;                // copy size
    {
        const double* gh = table + B * B + 2 * B;
        for (int q = threadIdx.x; q < 4 * CS; q += blockDim.x) {
            const int c = q / CS, r = (q % CS) / CP, k = q % CP;
            const int m = r - PAD, nn = k + c - PAD;
            sg[q] = (m >= 0 && m < B && nn >= 0 && nn < B) ? (float)gh[m * B + nn] : 0.0f;
        }
        __syncthreads();
    }
    auto dl = [&](float fv, float mw) {
        const BS4 bi = bspline_bins<false>(fv, B);
        const BS4 bj = bspline_bins<true>(mw, B);
        const int n0 = bj.m_lo + PAD;
        const float4* gr = reinterpret_cast<const float4*>(sg + (n0 & 3) * CS + (bi.m_lo + PAD) * CP + (n0 & ~3));
        float gj = 0.0f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float4 g = gr[a * (CP / 4)];
            float acc = g.x * bj.w[0];
            acc = fmaf(g.y, bj.w[1], acc);
            acc = fmaf(g.z, bj.w[2], acc);
            acc = fmaf(g.w, bj.w[3], acc);
            gj = fmaf(bi.k[a], acc, gj);
        }
        return gj;
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t done = 0;
    if (VEC) {
        const int64_t n4 = n / 4;
        auto group = [&](const float4 fv, const float4 r0, const float4 r1, const float4 r2, const float4 r3,
                         int64_t i) {
            const float g0 = dl(fv.x, r0.x), g1 = dl(fv.y, r1.x), g2 = dl(fv.z, r2.x), g3 = dl(fv.w, r3.x);
            float4* o = reinterpret_cast<float4*>(g_u + 12 * i);
            st_stream(o, make_float4(r0.y * g0, r0.z * g0, r0.w * g0, r1.y * g1));
            st_stream(o + 1, make_float4(r1.z * g1, r1.w * g1, r2.y * g2, r2.z * g2));
            st_stream(o + 2, make_float4(r2.w * g2, r3.y * g3, r3.z * g3, r3.w * g3));
        };
        int64_t i = tid;
#if FFDP_GR_UNROLL == 4
        for (; i + 3 * stride < n4; i += 4 * stride) {
            float4 fv[4], r[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t k = i + q * stride;
                fv[q] = ld_stream(reinterpret_cast<const float4*>(f) + k);
#pragma unroll
                for (int e = 0; e < 4; ++e) r[q][e] = ld_stream(rec + 4 * k + e);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) group(fv[q], r[q][0], r[q][1], r[q][2], r[q][3], i + q * stride);
        }
#endif
        for (; i + stride < n4; i += 2 * stride) {
            const int64_t j = i + stride;
            const float4 fa = ld_stream(reinterpret_cast<const float4*>(f) + i);
            const float4 fb = ld_stream(reinterpret_cast<const float4*>(f) + j);
            const float4 a0 = ld_stream(rec + 4 * i), a1 = ld_stream(rec + 4 * i + 1), a2 = ld_stream(rec + 4 * i + 2),
                         a3 = ld_stream(rec + 4 * i + 3);
            const float4 b0 = ld_stream(rec + 4 * j), b1 = ld_stream(rec + 4 * j + 1), b2 = ld_stream(rec + 4 * j + 2),
                         b3 = ld_stream(rec + 4 * j + 3);
            group(fa, a0, a1, a2, a3, i);
            group(fb, b0, b1, b2, b3, j);
        }
        for (; i < n4; i += stride) {
            const float4 fa = __ldg(reinterpret_cast<const float4*>(f) + i);
            group(fa, __ldg(rec + 4 * i), __ldg(rec + 4 * i + 1), __ldg(rec + 4 * i + 2), __ldg(rec + 4 * i + 3), i);
        }
        done = n4 * 4;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        const float4 r = __ldg(rec + i);
        const float g = dl(__ldg(f + i), r.x);
        g_u[3 * i] = r.y * g;
        g_u[3 * i + 1] = r.z * g;
        g_u[3 * i + 2] = r.w * g;
    }
}

// FFDP_GR_TMA = 1: pass 2 from the records as a bulk-copy stream. A persistent CTA takes
// chunks of GRT_CHUNK voxels: F and the records arrive by 1-D bulk copies
// (cp.async.bulk, one mbarrier per stage, two stages in flight), the threads compute from
// shared memory (voxels t + 256 j: conflict-free 16-byte record reads) and write g_u into a
// shared tile that one bulk store (cp.async.bulk ... bulk_group) moves out. The per-thread
// load / store instructions of the LDG form go, and the copy engine keeps a CTA's next two
// chunks (40 KB) in flight. Arithmetic identical to k_step_mi_grad_rec.
#ifndef FFDP_GR_TMA
#define FFDP_GR_TMA 1
#endif
#ifndef FFDP_GR_STAGES
#define FFDP_GR_STAGES 2
#endif
constexpr int GRT_CHUNK = 1024, GRT_NT = 256, GRT_ST = FFDP_GR_STAGES;  // input stages (chunks in flight + 1)
struct __align__(128) GrtSmem {
    float f[GRT_ST][GRT_CHUNK];
    float4 rec[GRT_ST][GRT_CHUNK];
    float g[2][3 * GRT_CHUNK];
    unsigned long long full[GRT_ST];
};

__device__ __forceinline__ uint32_t grt_saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(GRT_NT, 2) k_step_mi_grad_rec_bulk(const float* __restrict__ f,
                                                                    const float4* __restrict__ rec,
                                                                    float* __restrict__ g_u, int64_t nchunks,
                                                                    const double* table, int B) {
    extern __shared__ __align__(128) unsigned char grt_raw[];
    GrtSmem& sm = *reinterpret_cast<GrtSmem*>(grt_raw);
    float* sg = reinterpret_cast<float*>(grt_raw + sizeof(GrtSmem));
    const int LD = B + 2 * PAD, CP = (LD + 3) / 4 * 4, CS = LD * CP;
    const int t = threadIdx.x;
    auto issue = [&](int64_t c, int s) {
        const uint32_t bar = grt_saddr(&sm.full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(GRT_CHUNK * 20) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         grt_saddr(&sm.f[s][0])),
                     "l"(f + c * GRT_CHUNK), "r"(GRT_CHUNK * 4), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         grt_saddr(&sm.rec[s][0])),
                     "l"(rec + c * GRT_CHUNK), "r"(GRT_CHUNK * 16), "r"(bar)
                     : "memory");
    };
    if (t == 0) {
        for (int q = 0; q < GRT_ST; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(grt_saddr(&sm.full[q])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int q = 0; q < GRT_ST; ++q)
            if (blockIdx.x + (int64_t)q * gridDim.x < nchunks) issue(blockIdx.x + (int64_t)q * gridDim.x, q);
    }
    {
        const double* gh = table + B * B + 2 * B;
        for (int q = t; q < 4 * CS; q += GRT_NT) {
            const int c = q / CS, r = (q % CS) / CP, k = q % CP;
            const int m = r - PAD, nn = k + c - PAD;
            sg[q] = (m >= 0 && m < B && nn >= 0 && nn < B) ? (float)gh[m * B + nn] : 0.0f;
        }
        __syncthreads();
    }
    auto dl = [&](float fv, float mw) {
        const BS4 bi = bspline_bins<false>(fv, B);
        const BS4 bj = bspline_bins<true>(mw, B);
        const int n0 = bj.m_lo + PAD;
        const float4* gr = reinterpret_cast<const float4*>(sg + (n0 & 3) * CS + (bi.m_lo + PAD) * CP + (n0 & ~3));
        float gj = 0.0f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float4 g = gr[a * (CP / 4)];
            float acc = g.x * bj.w[0];
            acc = fmaf(g.y, bj.w[1], acc);
            acc = fmaf(g.z, bj.w[2], acc);
            acc = fmaf(g.w, bj.w[3], acc);
            gj = fmaf(bi.k[a], acc, gj);
        }
        return gj;
    };
    int i = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++i) {
        const int s = i % GRT_ST, go = i & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\tselp.u32 %0, 1, "
                "0, p;\n}"
                : "=r"(ok)
                : "r"(grt_saddr(&sm.full[s])), "r"((uint32_t)((i / GRT_ST) & 1))
                : "memory");
#pragma unroll
        for (int j = 0; j < GRT_CHUNK / GRT_NT; ++j) {
            const int v = t + GRT_NT * j;
            const float4 r = sm.rec[s][v];
            const float g = dl(sm.f[s][v], r.x);
            sm.g[go][3 * v] = r.y * g;
            sm.g[go][3 * v + 1] = r.z * g;
            sm.g[go][3 * v + 2] = r.w * g;
        }
        // the store of two chunks ago (same g tile) has finished reading before anyone rewrites
        // it: thread 0 waits for every earlier store's read before the barrier
        if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_u + 3 * c * GRT_CHUNK),
                         "r"(grt_saddr(&sm.g[go][0])), "r"(GRT_CHUNK * 12)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (c + GRT_ST * (int64_t)gridDim.x < nchunks) issue(c + GRT_ST * (int64_t)gridDim.x, s);
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_hist_to_raw(const unsigned long long* h, int n, double inv_scale, double* raw) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
        raw[i] += (double)h[i] * inv_scale;
}

}  // namespace mstep

// Returns FFDP_OK and launches, or a non-zero code when the quad path does not apply
// (the caller then uses the scalar kernels of mi.cu).
bool mi_quad_path_applies(const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                          const ffdp_parzen& k) {
    // zero-bordered moving image, lane-private histogram copies within shared memory,
    // 32-bit unit indices and in-plane offsets
    const size_t smem = k.kind == FFDP_PARZEN_BSPLINE3 ? mstep::bs_smem_bytes(k.bins) : mstep::hist_smem_bytes(k.bins);
    return m.pad == 2 && smem <= mstep::kMaxHistSmem && (int64_t)d.nx * d.ny < (1LL << 31) &&
           ((d.nx + 31) / 32) * ((d.ny + 3) / 4) * (s.z_end - s.z_begin) < (1LL << 31);
}

// log2 of the B-spline pass-1 fixed-point grid for a call over `voxels` interior voxels
int mi_bs_scale_exp(int64_t voxels) { return voxels >= (int64_t)FFDP_MI_BS_LARGE_MIN ? 21 : 23; }

// raw[i] += hist[i] / 2^scale_exp for the B*B joint entries (after an integer allreduce)
int mi_hist_u64_to_raw(const unsigned long long* h, int B, int scale_exp, double* raw, cudaStream_t st) {
    mstep::k_hist_to_raw<<<(B * B + 255) / 256, 256, 0, st>>>(h, B * B, std::ldexp(1.0, -scale_exp), raw);
    return check_launch("mi_hist_u64_to_raw");
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
    P.rec = nullptr;
    P.hist = nullptr;
    P.done = nullptr;
    P.fin_table = nullptr;
    P.raw_out = nullptr;
    P.upstream = -1.0;
    P.miss = nullptr;
    P.nx = (int32_t)d.nx;
    P.ny = (int32_t)d.ny;
    P.nxb = (int32_t)((d.nx + 31) / 32);
    P.nyq = (int32_t)((d.ny + 3) / 4);
    P.div_nxb = make_fastdiv((uint32_t)P.nxb);
    P.div_nyq = make_fastdiv((uint32_t)P.nyq);
    P.nzs = (int32_t)std::max<int64_t>(1, s.z_end - s.z_begin);
    P.div_nzs = make_fastdiv((uint32_t)P.nzs);
    // z-major order once a plane of F + u + M traffic no longer fits the L2 several times
    // over (FFDP_MI_ZORDER forces it on)
    P.zorder = FFDP_MI_ZORDER || d.nx * d.ny >= ((int64_t)1 << 21);
    P.plane = d.nx * d.ny;
    P.z_begin = s.z_begin;
    P.buf_z0 = s.buf_z0;
    P.nunits = (int64_t)P.nxb * P.nyq * (s.z_end - s.z_begin);
    P.fix_scale = k.kind == FFDP_PARZEN_BSPLINE3 ? 8388608.0f : k.kind == FFDP_PARZEN_GAUSSIAN ? 4194304.0f : 2097152.0f;
    return P;
}

int mi_quad_hist(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, double* raw, unsigned long long* ws,
                 int32_t* miss, cudaStream_t st, float* rec, double* table, double upstream, int scale_exp) {
    using namespace mstep;
    Params P = make_params(f, u, d, s, m, args, k);
    const int B = k.bins;
    // fused finalize (table != null): B-spline pass 1 only, workspace holds the counter
    const bool fin = table && ws && k.kind == FFDP_PARZEN_BSPLINE3;
    unsigned long long* h = ws ? ws : (unsigned long long*)scratch_alloc(sizeof(unsigned long long) * B * B, st);
    if (!h) return set_error(FFDP_CUDA, "step_mi: scratch allocation failed");
    cudaMemsetAsync(h, 0, sizeof(unsigned long long) * (B * B + (fin ? 1 : 0)), st);
    P.hist = h;
    if (fin) {
        P.done = reinterpret_cast<unsigned int*>(h + B * B);
        P.fin_table = table;
        P.raw_out = raw;
        P.upstream = upstream;
    }
    P.miss = miss;
    P.rec = reinterpret_cast<float4*>(rec);
    static std::atomic<unsigned long long> attr_mask{0};  // opt in to > 48 KB dynamic shared memory
    once_per_device(attr_mask, [&] {
        for (auto fn : {k_step_mi_hist<false, true, false>, k_step_mi_hist<false, false, false>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxHistSmem);
    });
    const int64_t chunks = (P.nunits + HNT / 32 - 1) / (HNT / 32);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)num_sms()));
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
    const bool bs = k.kind == FFDP_PARZEN_BSPLINE3;
    if (rec && !bs) return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need the B-spline Parzen kernel");
    if (bs) {
        const size_t smem = bs_smem_bytes(B);
        const int om = window_off_mode(P.g);
        // scale_exp 21 / 23 forces the grid (a sharded plan picks it from the GLOBAL voxel
        // count, so every rank accumulates on the single-GPU grid and the integer allreduce
        // reproduces the single-GPU histogram exactly)
        const bool large = scale_exp ? scale_exp == 21 : mi_bs_scale_exp(d.nx * d.ny * (s.z_end - s.z_begin)) == 21;
        P.fix_scale = large ? 2097152.0f : 8388608.0f;  // 2^21 / 2^23
        const int sel = (full ? 1 : 0) + (rec ? 2 : 0) + (B == 32 ? 4 : 0) + om * 8 + (large ? 24 : 0);
#define FFDP_BS_ROW(O, S)                                                                                        \
    k_mi_hist_bs<false, false, 0, O, S>, k_mi_hist_bs<true, false, 0, O, S>, k_mi_hist_bs<false, true, 0, O, S>,     \
        k_mi_hist_bs<true, true, 0, O, S>, k_mi_hist_bs<false, false, 32, O, S>, k_mi_hist_bs<true, false, 32, O, S>, \
        k_mi_hist_bs<false, true, 32, O, S>, k_mi_hist_bs<true, true, 32, O, S>
        static const decltype(&k_mi_hist_bs<true, true, 32, 1, 23>) table_[48] = {
            FFDP_BS_ROW(0, 23), FFDP_BS_ROW(1, 23), FFDP_BS_ROW(2, 23),
            FFDP_BS_ROW(0, 21), FFDP_BS_ROW(1, 21), FFDP_BS_ROW(2, 21)};
#undef FFDP_BS_ROW
        static std::atomic<unsigned long long> bs_attr{0};
        once_per_device(bs_attr, [&] {
            // the smallest shared-memory carve-out that holds the histogram: the rest is L1,
            // which the gather needs (percent of the 228 KB maximum, rounded up)
            const int pct = (int)std::min<size_t>(100, (smem + 2048) * 100 / (228 * 1024) + 1);
            for (auto fn : table_) {
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxHistSmem);
                cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            }
        });
        table_[sel]<<<grid, HNT, smem, st>>>(P);
    } else {
        const size_t smem = hist_smem_bytes(B);
        if (full)
            k_step_mi_hist<false, true, false><<<grid, HNT, smem, st>>>(P);
        else
            k_step_mi_hist<false, false, false><<<grid, HNT, smem, st>>>(P);
    }
    // raw == null (with a caller workspace): the fixed-point histogram stays in ws for an
    // integer allreduce; the caller converts it (mi_hist_u64_to_raw)
    if (!fin && raw) k_hist_to_raw<<<(B * B + 255) / 256, 256, 0, st>>>(h, B * B, 1.0 / P.fix_scale, raw);
    if (!ws) scratch_free(h, st);
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
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P.nunits + NT / 32 - 1) / (NT / 32),
                                                                 6LL * num_sms()));
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
    const bool bs = k.kind == FFDP_PARZEN_BSPLINE3;
    static const bool legacy = getenv("FFDP_MI_GRAD_LEGACY") && getenv("FFDP_MI_GRAD_LEGACY")[0] == '1';
    if (bs && !legacy) {
        const size_t tab = sizeof(float) * grad_tab_floats(B);
        static std::atomic<unsigned long long> attr_mask{0};
        using K = decltype(&k_mi_grad_bs<true, 32, 1>);
#define FFDP_G2_ROW(O) k_mi_grad_bs<false, 0, O>, k_mi_grad_bs<true, 0, O>, k_mi_grad_bs<false, 32, O>, k_mi_grad_bs<true, 32, O>
        static const K ks[12] = {FFDP_G2_ROW(0), FFDP_G2_ROW(1), FFDP_G2_ROW(2)};
#undef FFDP_G2_ROW
        once_per_device(attr_mask, [&] {
            for (auto fn : ks)
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(float) * grad_tab_floats(64)));
        });
        const int sel = (full ? 1 : 0) + (B == 32 ? 2 : 0) + window_off_mode(P.g) * 4;
        const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((P.nunits + NT / 32 - 1) / (NT / 32),
                                                                  (int64_t)FFDP_MI_G2_MINB * num_sms()));
        ks[sel]<<<g2, NT, tab, st>>>(P);
        return check_launch("step_mi_grad");
    }
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

int mi_grad_rec(const float* f, const ffdp_dims& d, const ffdp_slab& s, const ffdp_parzen& k, const double* table,
                const float* rec, float* g_u, cudaStream_t st) {
    using namespace mstep;
    if (k.kind != FFDP_PARZEN_BSPLINE3)
        return set_error(FFDP_INVALID_ARGUMENT, "step_mi: records need the B-spline Parzen kernel");
    const int B = k.bins;
    const float* fi = f + (s.z_begin - s.buf_z0) * d.nx * d.ny;  // interior planes
    const int64_t n_all = d.nx * d.ny * (s.z_end - s.z_begin);
    const size_t smem = sizeof(float) * grad_tab_floats(B);
    static std::atomic<unsigned long long> attr_mask{0};  // B up to 64: the 4 table copies may exceed 48 KB
    once_per_device(attr_mask, [&] {
        for (auto fn : {k_step_mi_grad_rec<true>, k_step_mi_grad_rec<false>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(float) * grad_tab_floats(64)));
    });
    const bool vec = (((uintptr_t)fi | (uintptr_t)rec | (uintptr_t)g_u) & 15) == 0;
    int64_t n = n_all;
    if (FFDP_GR_TMA && vec && n_all >= (int64_t)GRT_CHUNK * num_sms()) {
        // the chunk-aligned bulk part, then the < GRT_CHUNK tail voxels below
        const int64_t nch = n_all / GRT_CHUNK;
        const size_t smem2 = sizeof(GrtSmem) + smem;
        static std::atomic<unsigned long long> attr2{0};
        once_per_device(attr2, [&] {
            cudaFuncSetAttribute(k_step_mi_grad_rec_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(GrtSmem) + sizeof(float) * grad_tab_floats(64)));
        });
        const int grid2 = (int)std::min<int64_t>(nch, 2 * (int64_t)num_sms());
        k_step_mi_grad_rec_bulk<<<grid2, GRT_NT, smem2, st>>>(fi, reinterpret_cast<const float4*>(rec), g_u, nch,
                                                              table, B);
        if (int rc = check_launch("step_mi_grad_rec")) return rc;
        const int64_t done = nch * GRT_CHUNK;
        n = n_all - done;
        if (n == 0) return FFDP_OK;
        fi += done;
        rec += 4 * done;
        g_u += 3 * done;
    }
    const int64_t work = vec ? n / 4 : n;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)FFDP_GR_CTAS * num_sms()));
    if (vec)
        k_step_mi_grad_rec<true><<<grid, 256, smem, st>>>(fi, reinterpret_cast<const float4*>(rec), g_u, n, table, B);
    else
        k_step_mi_grad_rec<false><<<grid, 256, smem, st>>>(fi, reinterpret_cast<const float4*>(rec), g_u, n, table, B);
    return check_launch("step_mi_grad_rec");
}

}  // namespace ffdp
