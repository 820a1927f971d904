// ffdp_common.cuh -- shared device/host helpers for the sm_100a kernels of libffdp.
//
// Geometry: the composite transform x -> A*X + t + S*u(X) of the reference sampler
// (sampler.hpp:165-243) is folded on the host, in fp64, into the image's fractional
// index space:  f_a = K_a + sum_c P[a][c] * i_c + Q_a * u_a   (i = output lattice index).
// The per-voxel evaluation stays fp64 so that the floor-based cell choice and the
// 1e-9 face snap (resample.hpp:17-43) agree with the fp64 reference everywhere; the
// trilinear weights and the gather run in fp32.
#pragma once

#include <atomic>
#include <mutex>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ffdp.h"

#define FFDP_FACE_SNAP 1e-9
// gather_pad row pointers: 1 = one widened offset + 64-bit stride adds, 0 = four offsets
#ifndef FFDP_GADDR
#define FFDP_GADDR 1
#endif

namespace ffdp {

// Host-folded sampler geometry (kernel parameter, ~300 B).
struct Geom {
    double K[3];
    double P[9];  // row a = image axis, column c = output axis
    double Q[3];
    float dscale[3];  // S_a * 0.5 * (N_a - 1): dL/du_a = dscale_a * dfrac_a * g
    float hn[3];      // 0.5 * (N_a - 1): d(value)/d(xsrc_a) = dfrac_a * hn_a
    int32_t n[3];     // image lattice (global)
    int32_t wz0, wz1; // resident image planes [wz0, wz1)
    const float* img; // points at voxel (0, 0, wz0) (inside the border when padded)
    int64_t sy, sz;   // image strides in elements (of the padded layout when padded)
    int32_t pad;      // 0 or 2 (zero-bordered layout, ffdp_pad_window)
    double Xlo[3], Xstep[3];  // output lattice normalized coordinates (for gA)
    int32_t on[3];            // output lattice (global)
};

// Result of resolving one source coordinate (resolve_cell, sampler.hpp:100-113).
struct Cell {
    int32_t i0[3];
    float frac[3];
};

__device__ __forceinline__ void cell_assign(double f, int32_t n, int32_t& i0, float& frac) {
    // resample.hpp:32-43: floor, then snap fractions within 1e-9 of a face onto it.
    double fl = floor(f);
    double a = f - fl;
    if (a < FFDP_FACE_SNAP) {
        a = 0.0;
    } else if (1.0 - a < FFDP_FACE_SNAP) {
        fl += 1.0;
        a = 0.0;
    }
    // anything beyond the lattice by more than a cell is fully zero padded
    fl = fmin(fmax(fl, -2.0), (double)n + 1.0);
    i0 = (int32_t)fl;
    frac = (float)a;
}

__device__ __forceinline__ Cell resolve(const Geom& g, int32_t ix, int32_t iy, int32_t iz, float u0, float u1,
                                        float u2) {
    Cell c;
    const double x = ix, y = iy, z = iz;
    const double f0 = fma(g.Q[0], (double)u0, fma(g.P[2], z, fma(g.P[1], y, fma(g.P[0], x, g.K[0]))));
    const double f1 = fma(g.Q[1], (double)u1, fma(g.P[5], z, fma(g.P[4], y, fma(g.P[3], x, g.K[1]))));
    const double f2 = fma(g.Q[2], (double)u2, fma(g.P[8], z, fma(g.P[7], y, fma(g.P[6], x, g.K[2]))));
    cell_assign(f0, g.n[0], c.i0[0], c.frac[0]);
    cell_assign(f1, g.n[1], c.i0[1], c.frac[1]);
    cell_assign(f2, g.n[2], c.i0[2], c.frac[2]);
    return c;
}

// The 8 corner values (zero padded); counts window misses.
struct Corners {
    float v[8];  // index bx + 2*by + 4*bz
};

__device__ __forceinline__ Corners gather(const Geom& g, const Cell& c, int& miss) {
    Corners k;
    const bool vx0 = c.i0[0] >= 0 && c.i0[0] < g.n[0];
    const bool vx1 = c.i0[0] + 1 >= 0 && c.i0[0] + 1 < g.n[0];
    const bool vy0 = c.i0[1] >= 0 && c.i0[1] < g.n[1];
    const bool vy1 = c.i0[1] + 1 >= 0 && c.i0[1] + 1 < g.n[1];
#pragma unroll
    for (int bz = 0; bz < 2; ++bz) {
        const int32_t iz = c.i0[2] + bz;
        bool vz = iz >= 0 && iz < g.n[2];
        if (vz && (iz < g.wz0 || iz >= g.wz1)) {
            miss = 1;
            vz = false;
        }
        const float* plane = g.img + (int64_t)(iz - g.wz0) * g.sz;
#pragma unroll
        for (int by = 0; by < 2; ++by) {
            const bool vy = by ? vy1 : vy0;
            const float* row = plane + (int64_t)(c.i0[1] + by) * g.sy + c.i0[0];
            k.v[4 * bz + 2 * by + 0] = (vz && vy && vx0) ? __ldg(row) : 0.0f;
            k.v[4 * bz + 2 * by + 1] = (vz && vy && vx1) ? __ldg(row + 1) : 0.0f;
        }
    }
    return k;
}

// Trilinear value (sample_cell, sampler.hpp:116-134).
__device__ __forceinline__ float interp(const Corners& k, const Cell& c) {
    const float ax = c.frac[0], ay = c.frac[1], az = c.frac[2];
    const float e00 = fmaf(ax, k.v[1] - k.v[0], k.v[0]);
    const float e10 = fmaf(ax, k.v[3] - k.v[2], k.v[2]);
    const float e01 = fmaf(ax, k.v[5] - k.v[4], k.v[4]);
    const float e11 = fmaf(ax, k.v[7] - k.v[6], k.v[6]);
    const float g0 = fmaf(ay, e10 - e00, e00);
    const float g1 = fmaf(ay, e11 - e01, e01);
    return fmaf(az, g1 - g0, g0);
}

// Value and d(value)/d(fractional index) (sample_cell_dfrac, sampler.hpp:138-161).
__device__ __forceinline__ float interp_grad(const Corners& k, const Cell& c, float d[3]) {
    const float ax = c.frac[0], ay = c.frac[1], az = c.frac[2];
    const float dx00 = k.v[1] - k.v[0], dx10 = k.v[3] - k.v[2];
    const float dx01 = k.v[5] - k.v[4], dx11 = k.v[7] - k.v[6];
    const float e00 = fmaf(ax, dx00, k.v[0]);
    const float e10 = fmaf(ax, dx10, k.v[2]);
    const float e01 = fmaf(ax, dx01, k.v[4]);
    const float e11 = fmaf(ax, dx11, k.v[6]);
    const float dy0 = e10 - e00, dy1 = e11 - e01;
    const float g0 = fmaf(ay, dy0, e00);
    const float g1 = fmaf(ay, dy1, e01);
    const float h0 = fmaf(ay, dx10 - dx00, dx00);
    const float h1 = fmaf(ay, dx11 - dx01, dx01);
    d[0] = fmaf(az, h1 - h0, h0);
    d[1] = fmaf(az, dy1 - dy0, dy0);
    d[2] = g1 - g0;
    return fmaf(az, g1 - g0, g0);
}

// fp64 trilinear value, for losses whose kernels are discontinuous in the sampled value
// (Gaussian truncation, delta / hard binning): keeps bin decisions equal to fp64.
__device__ __forceinline__ double interp_f64(const Corners& k, const Cell& c) {
    const double ax = c.frac[0], ay = c.frac[1], az = c.frac[2];
    double acc = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double w = ((q & 1) ? ax : 1.0 - ax) * ((q & 2) ? ay : 1.0 - ay) * ((q & 4) ? az : 1.0 - az);
        acc = fma(w, (double)k.v[q], acc);
    }
    return acc;
}

// ------------------------------------------------------------------ fast row sampler
// Conversion-free cell assignment (the f64->int / f64->f32 conversions issue at a
// quarter of the FP64 rate on sm_100). t = f + 1.5*2^20 places floor(f) + 2^19 in
// mantissa bits 32..51 and frac(f) in units of 2^-32 in the low word (|f| < 2^19).
// The 1e-9 face snap of cell_assign (resample.hpp:32-43) is folded into the constant:
// adding 4 more units of 2^-32 carries fractions within 4 * 2^-32 (< 1e-9) of the upper
// face into the next cell with a low word < 4, and fractions within 4 units of the lower
// face leave a low word <= 8; both give frac = 0 after the 23-bit truncation below, and
// everywhere else the extra 4 units only move frac by at most one 2^-23 step.
// |f| >= 2^19 or NaN needs no test: the high word is monotone in t, so f >= 2^19 (and
// NaN) give i0 >= 2^19 and f < -2^19 gives i0 < -2^19 (a negative t's sign bit makes the
// int32 subtraction either stay far below zero or wrap above 2^30). Every caller clamps i0
// into the zero border (gather_pad), where such cells read only zeros, and frac is always
// a finite value in [0, 1).
__device__ __forceinline__ void cell_fix(double f, int32_t& i0, float& frac) {
    const double t = f + 0x1.8000000000004p+20;  // 1.5 * 2^20 + 4 * 2^-32
    const uint32_t lo = (uint32_t)__double2loint(t);
    i0 = __double2hiint(t) - 0x41380000;
    frac = __uint_as_float(0x3F800000u | (lo >> 9)) - 1.0f;
}

// Division by a runtime constant without an integer divide (round-up multiplier,
// exact for every 32-bit numerator): n / d = (hi + ((n - hi) >> 1)) >> (l - 1).
struct FastDiv {
    uint32_t d, m, s;  // s = l - 1 (0 when d == 1)
    bool one;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.one = d == 1;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    f.m = f.one ? 0u : (uint32_t)((((1ull << l) - d) << 32) / d + 1);
    f.s = f.one ? 0u : l - 1;
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    if (f.one) return n;
    const uint32_t hi = __umulhi(n, f.m);
    return (hi + ((n - hi) >> 1)) >> f.s;
}

// Row-run sampler state: the fp64 affine part of f for the current voxel, advanced by
// one DADD per axis per x step (the composite transform is affine in the lattice index).
struct RowBase {
    double b[3];
    __device__ __forceinline__ void init(const Geom& g, int32_t x, int32_t y, int32_t z) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
            b[a] = fma(g.P[3 * a + 0], (double)x, fma(g.P[3 * a + 2], (double)z, fma(g.P[3 * a + 1], (double)y, g.K[a])));
    }
    __device__ __forceinline__ void step(const Geom& g) {
#pragma unroll
        for (int a = 0; a < 3; ++a) b[a] += g.P[3 * a];
    }
    __device__ __forceinline__ void step_y(const Geom& g) {
#pragma unroll
        for (int a = 0; a < 3; ++a) b[a] += g.P[3 * a + 1];
    }
    __device__ __forceinline__ Cell cell(const Geom& g, float u0, float u1, float u2) const {
        Cell c;
        cell_fix(fma(g.Q[0], (double)u0, b[0]), c.i0[0], c.frac[0]);
        cell_fix(fma(g.Q[1], (double)u1, b[1]), c.i0[1], c.frac[1]);
        cell_fix(fma(g.Q[2], (double)u2, b[2]), c.i0[2], c.frac[2]);
        return c;
    }
};

// Gather with a branch-free interior fast path: all 8 corners inside the (resident)
// lattice -> unpredicated loads; otherwise the zero-padding path of `gather`.
template <bool FULLWIN>
__device__ __forceinline__ Corners gather_fast(const Geom& g, const Cell& c, int& miss) {
    const bool inside = (uint32_t)c.i0[0] < (uint32_t)(g.n[0] - 1) && (uint32_t)c.i0[1] < (uint32_t)(g.n[1] - 1) &&
                        (FULLWIN ? (uint32_t)c.i0[2] < (uint32_t)(g.n[2] - 1)
                                 : (c.i0[2] >= g.wz0 && c.i0[2] + 1 < g.wz1));
    if (inside) {
        Corners k;
        const float* p = g.img + (int64_t)(c.i0[2] - g.wz0) * g.sz + (int64_t)(c.i0[1] * (int32_t)g.sy + c.i0[0]);
        const int32_t sy = (int32_t)g.sy;
        k.v[0] = __ldg(p);
        k.v[1] = __ldg(p + 1);
        k.v[2] = __ldg(p + sy);
        k.v[3] = __ldg(p + sy + 1);
        p += g.sz;
        k.v[4] = __ldg(p);
        k.v[5] = __ldg(p + 1);
        k.v[6] = __ldg(p + sy);
        k.v[7] = __ldg(p + sy + 1);
        return k;
    }
    return gather(g, c, miss);
}

// Four samples at once: the corner loads of all four are issued back to back (memory
// level parallelism) when every lane's samples are interior (warp-uniform decision, no
// divergence); otherwise every sample takes the zero-padding path.
template <bool FULLWIN>
__device__ __forceinline__ bool cell_inside(const Geom& g, const Cell& c) {
    return (uint32_t)c.i0[0] < (uint32_t)(g.n[0] - 1) && (uint32_t)c.i0[1] < (uint32_t)(g.n[1] - 1) &&
           (FULLWIN ? (uint32_t)c.i0[2] < (uint32_t)(g.n[2] - 1) : (c.i0[2] >= g.wz0 && c.i0[2] + 1 < g.wz1));
}

template <bool FULLWIN, int NS>
__device__ __forceinline__ void gather_n(const Geom& g, const Cell (&c)[NS], Corners (&k)[NS], int& miss) {
    bool in = true;
#pragma unroll
    for (int q = 0; q < NS; ++q) in = in && cell_inside<FULLWIN>(g, c[q]);
    if (__all_sync(__activemask(), in)) {
        const int32_t sy = (int32_t)g.sy;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const float* p =
                g.img + (int64_t)(c[q].i0[2] - g.wz0) * g.sz + (int64_t)(c[q].i0[1] * sy + c[q].i0[0]);
            k[q].v[0] = __ldg(p);
            k[q].v[1] = __ldg(p + 1);
            k[q].v[2] = __ldg(p + sy);
            k[q].v[3] = __ldg(p + sy + 1);
            k[q].v[4] = __ldg(p + g.sz);
            k[q].v[5] = __ldg(p + g.sz + 1);
            k[q].v[6] = __ldg(p + g.sz + sy);
            k[q].v[7] = __ldg(p + g.sz + sy + 1);
        }
    } else {
#pragma unroll
        for (int q = 0; q < NS; ++q) k[q] = gather(g, c[q], miss);
    }
}

// Zero-bordered moving image (pad = 2): clamp each cell index into [-2, n] (a cell at
// -2 or n reads two border zeros, like the reference's fully zero-padded samples) and
// load the 8 corners unconditionally. With a z window, corners on non-resident planes
// inside the volume are window misses (they read the zero border).
// OFF: 0 = 64-bit addressing; 1 = signed 32-bit offsets from the window (< 2^31 elements);
// 2 = unsigned 32-bit offsets from the block origin (< 2^32 elements, window_off32).
template <bool FULLWIN, int OFF = 0>
__device__ __forceinline__ Corners gather_pad(const Geom& g, const Cell& c, int& miss) {
    const int32_t ix = min(max(c.i0[0], -2), g.n[0]);
    const int32_t iy = min(max(c.i0[1], -2), g.n[1]);
    int32_t iz;
    if (FULLWIN) {
        iz = min(max(c.i0[2], -2), g.n[2]);
    } else {
        const int32_t z0 = c.i0[2];
        const bool in0 = z0 >= 0 && z0 < g.n[2], in1 = z0 + 1 >= 0 && z0 + 1 < g.n[2];
        if ((in0 && (z0 < g.wz0 || z0 >= g.wz1)) || (in1 && (z0 + 1 < g.wz0 || z0 + 1 >= g.wz1))) miss = 1;
        iz = min(max(z0, g.wz0 - 2), g.wz1);
    }
    const int32_t sy = (int32_t)g.sy;
    Corners k;
#if FFDP_GADDR
    if (OFF == 2) {
        // one widened offset from the block origin for the first row pointer, the other three
        // by 64-bit byte-stride adds; the origin is an opaque pointer (otherwise the compiler
        // folds the border offset into every row pointer: a 64-bit subtract per pointer)
        const uint32_t o = (uint32_t)(iz - g.wz0 + 2) * (uint32_t)g.sz + (uint32_t)(iy + 2) * (uint32_t)g.sy +
                           (uint32_t)(ix + 2);
        uint64_t org;
        asm("mov.b64 %0, %1;" : "=l"(org) : "l"(g.img - (2 * g.sz + 2 * g.sy + 2)));
        const char* p0 = reinterpret_cast<const char*>(reinterpret_cast<const float*>(org) + o);
        const int64_t by = 4 * g.sy, bz = 4 * g.sz;
        const float* q0 = reinterpret_cast<const float*>(p0);
        const float* q1 = reinterpret_cast<const float*>(p0 + by);
        const float* q2 = reinterpret_cast<const float*>(p0 + bz);
        const float* q3 = reinterpret_cast<const float*>(p0 + bz + by);
        k.v[0] = __ldg(q0);
        k.v[1] = __ldg(q0 + 1);
        k.v[2] = __ldg(q1);
        k.v[3] = __ldg(q1 + 1);
        k.v[4] = __ldg(q2);
        k.v[5] = __ldg(q2 + 1);
        k.v[6] = __ldg(q3);
        k.v[7] = __ldg(q3 + 1);
        return k;
    }
#endif
    if (OFF == 1) {
        // the resident window holds < 2^31 elements: 32-bit offsets, one wide add per row
        const int32_t sz = (int32_t)g.sz;
        const int32_t o = (iz - g.wz0) * sz + iy * sy + ix;
        const float* p0 = g.img + o;
        const float* p1 = g.img + (o + sy);
        const float* p2 = g.img + (o + sz);
        const float* p3 = g.img + (o + sz + sy);
        k.v[0] = __ldg(p0);
        k.v[1] = __ldg(p0 + 1);
        k.v[2] = __ldg(p1);
        k.v[3] = __ldg(p1 + 1);
        k.v[4] = __ldg(p2);
        k.v[5] = __ldg(p2 + 1);
        k.v[6] = __ldg(p3);
        k.v[7] = __ldg(p3 + 1);
        return k;
    }
    if (OFF == 2) {
        // the zero-bordered block holds < 2^32 elements: unsigned 32-bit offsets from its
        // origin (every clamped corner index is >= -2), one IMAD.WIDE.U32 per row pointer
        const uint32_t usy = (uint32_t)g.sy, usz = (uint32_t)g.sz;
        const uint32_t o = (uint32_t)(iz - g.wz0 + 2) * usz + (uint32_t)(iy + 2) * usy + (uint32_t)(ix + 2);
        const float* org = g.img - (2 * g.sz + 2 * g.sy + 2);
        const float* p0 = org + o;
        const float* p1 = org + (o + usy);
        const float* p2 = org + (o + usz);
        const float* p3 = org + (o + usz + usy);
        k.v[0] = __ldg(p0);
        k.v[1] = __ldg(p0 + 1);
        k.v[2] = __ldg(p1);
        k.v[3] = __ldg(p1 + 1);
        k.v[4] = __ldg(p2);
        k.v[5] = __ldg(p2 + 1);
        k.v[6] = __ldg(p3);
        k.v[7] = __ldg(p3 + 1);
        return k;
    }
    const float* p = g.img + (int64_t)(iz - g.wz0) * g.sz + (int64_t)(iy * sy + ix);
    k.v[0] = __ldg(p);
    k.v[1] = __ldg(p + 1);
    k.v[2] = __ldg(p + sy);
    k.v[3] = __ldg(p + sy + 1);
    p += g.sz;
    k.v[4] = __ldg(p);
    k.v[5] = __ldg(p + 1);
    k.v[6] = __ldg(p + sy);
    k.v[7] = __ldg(p + sy + 1);
    return k;
}

// gather_pad's addressing mode for a zero-bordered window: 1 when the resident window fits
// signed 32-bit offsets (the old bound), 2 when the block fits unsigned 32-bit offsets from
// its origin ((nx+4)(ny+4)(planes+4) < 2^32), else 0 (64-bit).
inline int window_off_mode(const Geom& g) {
    const double n = (double)g.sz * (double)(g.wz1 - g.wz0 + 4);
    if (g.pad != 2) return 0;
    if (n < 2147483647.0 - 4.0 * (double)g.sz) return 1;
    return n < 4294967295.0 ? 2 : 0;
}
inline bool window_off32(const Geom& g) { return window_off_mode(g) == 1; }

// ------------------------------------------------------------------ Parzen kernels
// Up to four bins m_lo..m_lo+3 carry weight for one intensity (mi.hpp:28-140):
// bspline3 support 4 bins, gaussian 3-4 bins (radius 1.5 bins), delta 1 bin.
struct ParzenDev {
    int32_t kind, bins;
    double sigma, radius, norm;
    float inv_sigma2_f, norm_f, inv_sigma_f;
};

struct Bins4 {
    int32_t m_lo;
    float k[4];  // kappa(b_m - v)
    float w[4];  // omega(b_m - v) (only when requested)
};

__device__ __forceinline__ float bspline3(float t) {
    const float a = fabsf(t);
    if (a < 1.0f) return (4.0f - 6.0f * a * a + 3.0f * a * a * a) * (1.0f / 6.0f);
    if (a < 2.0f) {
        const float q = 2.0f - a;
        return q * q * q * (1.0f / 6.0f);
    }
    return 0.0f;
}
__device__ __forceinline__ float bspline3_deriv(float t) {
    const float a = fabsf(t);
    const float s = t < 0.0f ? -1.0f : 1.0f;
    if (a < 1.0f) return s * (-2.0f * a + 1.5f * a * a);
    if (a < 2.0f) {
        const float q = 2.0f - a;
        return s * (-0.5f * q * q);
    }
    return 0.0f;
}

// v may be supplied in fp64 (exact truncation decisions for discontinuous kernels).
template <bool WANT_OMEGA>
__device__ __forceinline__ Bins4 parzen_bins(const ParzenDev& p, double v) {
    Bins4 r;
    const int B = p.bins;
    if (p.kind == FFDP_PARZEN_BSPLINE3) {
        const double s = v * B - 0.5;
        const double fl = floor(s);
        r.m_lo = (int32_t)fl - 1;
        const float phi = (float)(s - fl);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // x*B for bin m_lo+q: (m_lo + q + 0.5) - v*B = q - 1 - phi
            const float tq = (float)(q - 1) - phi;
            const bool ok = (r.m_lo + q) >= 0 && (r.m_lo + q) < B;
            r.k[q] = ok ? bspline3(tq) : 0.0f;
            if (WANT_OMEGA) r.w[q] = ok ? -(float)B * bspline3_deriv(tq) : 0.0f;
        }
    } else if (p.kind == FFDP_PARZEN_GAUSSIAN) {
        const double s = v * B - 0.5;
        r.m_lo = (int32_t)floor(s - 1.5);  // bins with |m - s| <= 1.5 lie in m_lo .. m_lo+3
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = r.m_lo + q;
            const double x = ((double)m + 0.5) / (double)B - v;  // bin_center(m) - v, fp64 (mi.hpp:142-144)
            const bool ok = m >= 0 && m < B && !(fabs(x) > p.radius);
            const float xf = (float)x;
            const float kap = ok ? p.norm_f * expf(-0.5f * xf * xf * p.inv_sigma2_f) : 0.0f;
            r.k[q] = kap;
            if (WANT_OMEGA) r.w[q] = xf * p.inv_sigma2_f * kap;
        }
    } else {  // delta (mi.hpp:55-63): indicator |x| < radius
        r.m_lo = (int32_t)floor(v * B);
        const int m = r.m_lo;
        const double x = ((double)m + 0.5) / (double)B - v;
        const bool ok = m >= 0 && m < B && fabs(x) < p.radius;
        r.k[0] = ok ? 1.0f : 0.0f;
        r.k[1] = r.k[2] = r.k[3] = 0.0f;
        if (WANT_OMEGA) r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0.0f;
    }
    return r;
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of a double (all threads participate); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem /* NT/32 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) smem[w] = v;
    __syncthreads();
    double r = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) r += smem[i];
    return r;
}

// finalize_histogram + histogram_mi + the ghat table of mi_backward_impl
// (mi.hpp:181-209, 369-390) by one CTA (blockDim a multiple of 32, >= B) from the raw
// joint histogram in shared memory (rs[B*B], overwritten with p_ij), in a fixed reduction
// order. table = p_ij[B*B], p_i[B], p_j[B], ghat[B*B], {z, mi, dot, 0}. Marginals come
// from p_ij (mi.hpp:181-196): one warp per row / column, shuffle sums.
__device__ __forceinline__ void mi_finalize_block(double* rs, int B, double upstream, double* __restrict__ table,
                                                  double* red /* >= 34 doubles of shared scratch */) {
    const int nb2 = B * B, nt = blockDim.x, nw = nt >> 5;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* pij = table;
    double* pi = table + nb2;
    double* pj = pi + B;
    double* gh = pj + B;
    double* sc = gh + nb2;
    double acc = 0;
    for (int q = threadIdx.x; q < nb2; q += nt) acc += rs[q];
    acc = warp_sum(acc);
    __syncthreads();
    if (lane == 0) red[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double z = 0;
        for (int i = 0; i < nw; ++i) z += red[i];
        red[32] = z;
    }
    __syncthreads();
    const double z = red[32];
    for (int q = threadIdx.x; q < nb2; q += nt) {
        const double p = rs[q] / z;
        rs[q] = p;
        pij[q] = p;
    }
    __syncthreads();
    // row m / column m sums: warp m, lanes stride the B entries in a fixed order
    for (int m = w; m < B; m += nw) {
        double r = 0, c = 0;
        for (int n = lane; n < B; n += 32) {
            r += rs[m * B + n];
            c += rs[n * B + m];
        }
        r = warp_sum(r);
        c = warp_sum(c);
        if (lane == 0) {
            pi[m] = r;
            pj[m] = c;
            red[34 + m] = r;       // shared copies of the marginals for the log terms
            red[34 + B + m] = c;
        }
    }
    __syncthreads();
    double mi = 0, dot = 0;
    for (int q = threadIdx.x; q < nb2; q += nt) {
        const double p = rs[q];
        double g = 0;
        if (p > 0) {
            const double l = log(p / (red[34 + q / B] * red[34 + B + q % B]));
            mi += p * l;
            g = l - 1.0;
            dot += g * p;
        }
        rs[q] = g;
    }
    mi = warp_sum(mi);
    dot = warp_sum(dot);
    __syncthreads();
    if (lane == 0) {
        red[w] = mi;
        red[32 + 2 * B + 34 + w] = dot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0, d = 0;
        for (int i = 0; i < nw; ++i) {
            s += red[i];
            d += red[32 + 2 * B + 34 + i];
        }
        sc[0] = z;
        sc[1] = s;
        sc[2] = d;
        sc[3] = 0;
        red[33] = d;
    }
    __syncthreads();
    const double dt = red[33];
    for (int q = threadIdx.x; q < nb2; q += nt) gh[q] = pij[q] > 0 ? upstream * (rs[q] - dt) / z : 0.0;
}
// shared scratch doubles mi_finalize_block needs for B bins and nt threads
__host__ __device__ constexpr int mi_finalize_scratch(int B, int nt) { return 34 + 2 * B + 32 + nt / 32; }

}  // namespace ffdp

// ------------------------------------------------------------------ host helpers
namespace ffdp {

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
Geom make_geom(const ffdp_image_window& img, const ffdp_dims& out_dims, const ffdp_sampler_args& a);
bool valid_args(const ffdp_sampler_args& a, const char** why);
ParzenDev make_parzen_dev(const ffdp_parzen& k);
int num_sms();
// Stream-ordered scratch from the library's own per-device pool (cudaMallocFromPoolAsync);
// freed with scratch_free on the same stream.
cudaMemPool_t device_pool(int dev);
void* scratch_alloc(size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);
// Runs setup() once per device per call site (per-device kernel attributes), thread-safe:
// a second host thread driving the same device (a sharded plan's ranks) waits until the
// first has set the attributes instead of launching before them.
std::mutex& once_mutex();
template <class F>
void once_per_device(std::atomic<unsigned long long>& mask, F&& setup) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    std::lock_guard<std::mutex> lock(once_mutex());
    if (mask.load(std::memory_order_relaxed) & bit) return;
    setup();
    mask.fetch_or(bit, std::memory_order_release);
}

}  // namespace ffdp

#define FFDP_CHECK_CUDA(expr)                                                                         \
    do {                                                                                              \
        cudaError_t e_ = (expr);                                                                      \
        if (e_ != cudaSuccess) return ffdp::set_error(FFDP_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)
