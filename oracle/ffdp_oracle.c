/*
 * ffdp_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped or measured
 * as the product). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library.
 *
 * A plain-C, fp64 restatement of the reference's fused warp + loss step (voxreg, the
 * CPU engine under /root/reference/proj). Every function cites the reference
 * file:line it follows. Layouts follow the reference: volumes x-fastest
 * ((z*ny+y)*nx+x), warp fields interleaved xyz per voxel (volume.hpp:3-7,57,69-71).
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against golden vectors
 * produced by the reference itself (oracle/_ref, built from the reference headers by
 * oracle/Makefile; vectors in tests/golden/ made by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_API __attribute__((visibility("default")))

typedef struct {
    int64_t nx, ny, nz;
} or_dims;

static inline int64_t dims_voxels(or_dims d) { return d.nx * d.ny * d.nz; }
static inline int64_t dims_axis(or_dims d, int a) { return a == 0 ? d.nx : a == 1 ? d.ny : d.nz; }

/* ---------------------------------------------------------------- rng.hpp:11-52 */
typedef struct {
    uint64_t state;
    int have_spare;
    double spare;
} or_rng;

OR_API void or_rng_init(or_rng* r, uint64_t seed) {
    r->state = seed;
    r->have_spare = 0;
    r->spare = 0;
}

OR_API uint64_t or_rng_next_u64(or_rng* r) { /* splitmix64, rng.hpp:15-21 */
    r->state += 0x9E3779B97F4A7C15ull;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

OR_API double or_rng_uniform(or_rng* r) { /* rng.hpp:24 */
    return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

OR_API double or_rng_uniform_range(or_rng* r, double lo, double hi) { /* rng.hpp:26 */
    return lo + (hi - lo) * or_rng_uniform(r);
}

OR_API int64_t or_rng_uniform_int(or_rng* r, int64_t lo, int64_t hi) { /* rng.hpp:28-30 */
    return lo + (int64_t)(or_rng_uniform(r) * (double)(hi - lo + 1));
}

OR_API double or_rng_normal(or_rng* r) { /* Box-Muller, rng.hpp:33-46 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = or_rng_uniform(r);
    while (u1 <= 0) u1 = or_rng_uniform(r);
    const double u2 = or_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(theta);
    r->have_spare = 1;
    return rad * cos(theta);
}

/* ------------------------------------------------------- geometry.hpp:99-109 */
static inline double lattice_coord(double lo, double hi, int64_t i, int64_t n) {
    if (n <= 1) return lo;
    return lo + (hi - lo) * ((double)i / (double)(n - 1));
}

/* ---------------------------------------------- resample.hpp:17-43 cell_assign */
#define OR_FACE_SNAP 1e-9
static inline void cell_assign(double f, int64_t* i0, double* frac) {
    double fl = floor(f);
    double a = f - fl;
    if (a < OR_FACE_SNAP) {
        a = 0.0;
    } else if (1.0 - a < OR_FACE_SNAP) {
        fl += 1.0;
        a = 0.0;
    }
    *i0 = (int64_t)fl;
    *frac = a;
}

/* -------------------------------------------- sampler.hpp:92-161 cell helpers */
typedef struct {
    int64_t i0[3];
    double frac[3];
    int in[3][2];
    int64_t idx[3][2];
} cell_t;

static inline void resolve_cell(const double xsrc[3], or_dims d, cell_t* c) { /* sampler.hpp:100-113 */
    for (int a = 0; a < 3; ++a) {
        const int64_t n = dims_axis(d, a);
        const double f = (xsrc[a] + 1.0) * 0.5 * (double)(n - 1);
        cell_assign(f, &c->i0[a], &c->frac[a]);
        for (int s = 0; s < 2; ++s) {
            const int64_t i = c->i0[a] + s;
            c->in[a][s] = i >= 0 && i < n;
            c->idx[a][s] = i;
        }
    }
}

static inline int64_t vidx(or_dims d, int64_t x, int64_t y, int64_t z) { return (z * d.ny + y) * d.nx + x; }

static double sample_cell(const double* img, or_dims d, const cell_t* c) { /* sampler.hpp:116-134 */
    double acc = 0;
    for (int bz = 0; bz < 2; ++bz) {
        if (!c->in[2][bz]) continue;
        const double wz = bz ? c->frac[2] : 1 - c->frac[2];
        for (int by = 0; by < 2; ++by) {
            if (!c->in[1][by]) continue;
            const double wy = by ? c->frac[1] : 1 - c->frac[1];
            for (int bx = 0; bx < 2; ++bx) {
                if (!c->in[0][bx]) continue;
                const double wx = bx ? c->frac[0] : 1 - c->frac[0];
                acc += wz * wy * wx * img[vidx(d, c->idx[0][bx], c->idx[1][by], c->idx[2][bz])];
            }
        }
    }
    return acc;
}

static void sample_cell_dfrac(const double* img, or_dims d, const cell_t* c, double out[3]) { /* sampler.hpp:138-161 */
    out[0] = out[1] = out[2] = 0;
    for (int bz = 0; bz < 2; ++bz) {
        if (!c->in[2][bz]) continue;
        const double wz = bz ? c->frac[2] : 1 - c->frac[2];
        const double dz = bz ? 1.0 : -1.0;
        for (int by = 0; by < 2; ++by) {
            if (!c->in[1][by]) continue;
            const double wy = by ? c->frac[1] : 1 - c->frac[1];
            const double dy = by ? 1.0 : -1.0;
            for (int bx = 0; bx < 2; ++bx) {
                if (!c->in[0][bx]) continue;
                const double wx = bx ? c->frac[0] : 1 - c->frac[0];
                const double dx = bx ? 1.0 : -1.0;
                const double v = img[vidx(d, c->idx[0][bx], c->idx[1][by], c->idx[2][bz])];
                out[0] += dx * wy * wz * v;
                out[1] += wx * dy * wz * v;
                out[2] += wx * wy * dz * v;
            }
        }
    }
}

/*
 * composite_sample_core (sampler.hpp:165-243). A: row-major 3x3, t, S: 3,
 * bounds: {x_min[3], x_max[3]} of the implicit output lattice. u may be NULL
 * (then the output lattice is out_dims anyway). Any output may be NULL.
 * Returns 0, or 1 on invalid arguments (SamplerArgs::validate, sampler.hpp:31-36).
 */
OR_API int or_sample_core(const double* img, or_dims idims, const double* u, or_dims odims,
                          const double* A, const double* t, const double* S, const double* bounds,
                          double* out, const double* upstream, double* g_img, double* g_u,
                          double* gA, double* gt, double* abs_accum) {
    for (int i = 0; i < 9; ++i)
        if (!isfinite(A[i])) return 1;
    for (int c = 0; c < 3; ++c)
        if (!(S[c] > 0)) return 1;
    for (int c = 0; c < 3; ++c)
        if (!(bounds[c] < bounds[3 + c])) return 1;
    const double half_nm1[3] = {0.5 * (double)(idims.nx - 1), 0.5 * (double)(idims.ny - 1),
                                0.5 * (double)(idims.nz - 1)};
    for (int64_t z = 0; z < odims.nz; ++z) {
        const double Xz = lattice_coord(bounds[2], bounds[5], z, odims.nz);
        for (int64_t y = 0; y < odims.ny; ++y) {
            const double Xy = lattice_coord(bounds[1], bounds[4], y, odims.ny);
            for (int64_t x = 0; x < odims.nx; ++x) {
                const double X[3] = {lattice_coord(bounds[0], bounds[3], x, odims.nx), Xy, Xz};
                double xsrc[3];
                for (int r = 0; r < 3; ++r)
                    xsrc[r] = A[3 * r + 0] * X[0] + A[3 * r + 1] * X[1] + A[3 * r + 2] * X[2] + t[r];
                const int64_t o = vidx(odims, x, y, z);
                if (u)
                    for (int c = 0; c < 3; ++c) xsrc[c] += S[c] * u[3 * o + c];
                cell_t cell;
                resolve_cell(xsrc, idims, &cell);
                if (out) {
                    const double v = sample_cell(img, idims, &cell);
                    out[o] += v;
                    if (abs_accum) *abs_accum += fabs(v);
                }
                if (!upstream) continue;
                const double g = upstream[o];
                if (g_img) {
                    for (int bz = 0; bz < 2; ++bz) {
                        if (!cell.in[2][bz]) continue;
                        const double wz = bz ? cell.frac[2] : 1 - cell.frac[2];
                        for (int by = 0; by < 2; ++by) {
                            if (!cell.in[1][by]) continue;
                            const double wy = by ? cell.frac[1] : 1 - cell.frac[1];
                            for (int bx = 0; bx < 2; ++bx) {
                                if (!cell.in[0][bx]) continue;
                                const double wx = bx ? cell.frac[0] : 1 - cell.frac[0];
                                g_img[vidx(idims, cell.idx[0][bx], cell.idx[1][by], cell.idx[2][bz])] +=
                                    wx * wy * wz * g;
                            }
                        }
                    }
                }
                if (g_u || gA || gt) {
                    double dfrac[3];
                    sample_cell_dfrac(img, idims, &cell, dfrac);
                    const double dx[3] = {dfrac[0] * half_nm1[0], dfrac[1] * half_nm1[1],
                                          dfrac[2] * half_nm1[2]};
                    if (g_u)
                        for (int c = 0; c < 3; ++c) g_u[3 * o + c] += S[c] * dx[c] * g;
                    if (gA)
                        for (int r = 0; r < 3; ++r)
                            for (int c = 0; c < 3; ++c) gA[3 * r + c] += dx[r] * g * X[c];
                    if (gt)
                        for (int r = 0; r < 3; ++r) gt[r] += dx[r] * g;
                }
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------- smoothing.hpp:25-105 */
/* gaussian_taps (smoothing.hpp:25-39). Writes up to cap taps; returns the count (or -1). */
OR_API int or_gaussian_taps(double sigma, double* taps, int cap) {
    if (!isfinite(sigma) || sigma < 0) return -1;
    if (sigma == 0) {
        if (cap < 1) return -1;
        taps[0] = 1.0;
        return 1;
    }
    const int64_t radius = (int64_t)ceil(3.0 * sigma);
    const int n = (int)(2 * radius + 1);
    if (n > cap) return -1;
    double sum = 0;
    for (int64_t k = -radius; k <= radius; ++k) {
        const double w = exp(-0.5 * ((double)k / sigma) * ((double)k / sigma));
        taps[k + radius] = w;
        sum += w;
    }
    for (int i = 0; i < n; ++i) taps[i] /= sum;
    return n;
}

/* convolve_axis (smoothing.hpp:52-94); mode 0 = zero_pad, 1 = renormalize. */
OR_API void or_convolve_axis(const double* in, double* out, or_dims dims, int channels, int axis,
                             const double* taps, int ntaps, int mode, int64_t lo_global,
                             int64_t n_global) {
    const int64_t r = ntaps / 2;
    const int64_t n_axis = dims_axis(dims, axis);
    const int64_t sx = channels, sy = dims.nx * channels, sz = dims.nx * dims.ny * channels;
    const int64_t stride = axis == 0 ? sx : axis == 1 ? sy : sz;
    double full_sum = 0;
    for (int i = 0; i < ntaps; ++i) full_sum += taps[i];
    for (int64_t z = 0; z < dims.nz; ++z)
        for (int64_t y = 0; y < dims.ny; ++y)
            for (int64_t x = 0; x < dims.nx; ++x) {
                const int64_t p = axis == 0 ? x : axis == 1 ? y : z;
                const int64_t g = lo_global + p;
                const int full = (g - r >= 0) && (g + r < n_global) && (p - r >= 0) && (p + r < n_axis);
                const int64_t base = z * sz + y * sy + x * sx;
                for (int c = 0; c < channels; ++c) {
                    double acc = 0;
                    if (full) {
                        for (int64_t k = -r; k <= r; ++k) acc += taps[k + r] * in[base + c + k * stride];
                        if (mode == 1) acc /= full_sum;
                    } else {
                        double wsum = 0;
                        for (int64_t k = -r; k <= r; ++k) {
                            if (g + k < 0 || g + k >= n_global) continue;
                            if (p + k < 0 || p + k >= n_axis) continue;
                            const double w = taps[k + r];
                            acc += w * in[base + c + k * stride];
                            wsum += w;
                        }
                        if (mode == 1 && wsum > 0) acc /= wsum;
                    }
                    out[base + c] = acc;
                }
            }
}

/* separable_convolve (smoothing.hpp:98-105), in place through one scratch buffer. */
OR_API void or_separable_convolve(double* data, or_dims dims, int channels, const double* taps,
                                  int ntaps, int mode) {
    const size_t n = (size_t)dims_voxels(dims) * (size_t)channels;
    double* scratch = (double*)malloc(n * sizeof(double));
    or_convolve_axis(data, scratch, dims, channels, 0, taps, ntaps, mode, 0, dims.nx);
    or_convolve_axis(scratch, data, dims, channels, 1, taps, ntaps, mode, 0, dims.ny);
    or_convolve_axis(data, scratch, dims, channels, 2, taps, ntaps, mode, 0, dims.nz);
    memcpy(data, scratch, n * sizeof(double));
    free(scratch);
}

OR_API int or_gaussian_smooth(double* data, or_dims dims, int channels, double sigma) { /* smoothing.hpp:108-125 */
    if (!isfinite(sigma) || sigma < 0) return 1;
    if (sigma == 0) return 0;
    double taps[4096];
    const int nt = or_gaussian_taps(sigma, taps, 4096);
    if (nt < 0) return 1;
    or_separable_convolve(data, dims, channels, taps, nt, 1);
    return 0;
}

/* adam_step (adam.hpp:30-50): bias-corrected Adam over a flat buffer, fp64 arithmetic;
 * `step` is the state's step counter AFTER the increment (1 on the first call). */
OR_API void or_adam_step(double* param, const double* grad, double* m1, double* m2, int64_t n, double lr,
                         double beta1, double beta2, double eps, int64_t step) {
    const double c1 = 1.0 - pow(beta1, (double)step);
    const double c2 = 1.0 - pow(beta2, (double)step);
    for (int64_t i = 0; i < n; ++i) {
        const double g = grad[i];
        const double m = beta1 * m1[i] + (1.0 - beta1) * g;
        const double v = beta2 * m2[i] + (1.0 - beta2) * g * g;
        m1[i] = m;
        m2[i] = v;
        param[i] = param[i] - lr * (m / c1) / (sqrt(v / c2) + eps);
    }
}

/* The warp update of one deformable iteration (registration.hpp:313-317) on one rank:
 * g_s = separable renormalized Gaussian(sigma_grad) of g_u; adam_step(u, g_s);
 * u = separable renormalized Gaussian(sigma_warp) of u. g_u is not modified. */
OR_API int or_warp_update(const double* g_u, double* u, double* m1, double* m2, or_dims dims, double sigma_grad,
                          double sigma_warp, double lr, double beta1, double beta2, double eps, int64_t step) {
    double tg[4096], tw[4096];
    const int ng = or_gaussian_taps(sigma_grad, tg, 4096), nw = or_gaussian_taps(sigma_warp, tw, 4096);
    if (ng < 0 || nw < 0) return 1;
    const int64_t n = 3 * dims_voxels(dims);
    double* gs = (double*)malloc((size_t)n * sizeof(double));
    memcpy(gs, g_u, (size_t)n * sizeof(double));
    or_separable_convolve(gs, dims, 3, tg, ng, 1);
    or_adam_step(u, gs, m1, m2, n, lr, beta1, beta2, eps, step);
    or_separable_convolve(u, dims, 3, tw, nw, 1);
    free(gs);
    return 0;
}

/* resample_scale / resample_warp (resample.hpp:48-146): per-axis fractional index
 * i (n_src - 1) / (n_dst - 1), cell_assign (floor + 1e-9 face snap), upper corner clamped. */
static void rs_axis(int64_t i, int64_t ns, int64_t nd, int64_t* i0, int64_t* i1, double* w1) {
    const double f = nd > 1 ? (double)i * (double)(ns - 1) / (double)(nd - 1) : 0.0;
    double fr;
    int64_t lo;
    cell_assign(f, &lo, &fr);
    *i0 = lo < ns - 1 ? lo : ns - 1;
    *i1 = lo + 1 < ns - 1 ? lo + 1 : ns - 1;
    *w1 = fr;
}

static void rs_trilinear(const double* in, or_dims sd, int channels, double* out, or_dims dd) {
    for (int64_t z = 0; z < dd.nz; ++z) {
        int64_t z0, z1;
        double wz;
        rs_axis(z, sd.nz, dd.nz, &z0, &z1, &wz);
        for (int64_t y = 0; y < dd.ny; ++y) {
            int64_t y0, y1;
            double wy;
            rs_axis(y, sd.ny, dd.ny, &y0, &y1, &wy);
            for (int64_t x = 0; x < dd.nx; ++x) {
                int64_t x0, x1;
                double wx;
                rs_axis(x, sd.nx, dd.nx, &x0, &x1, &wx);
                const int64_t xs[2] = {x0, x1}, ys[2] = {y0, y1}, zs[2] = {z0, z1};
                for (int c = 0; c < channels; ++c) {
                    double acc = 0;
                    for (int bz = 0; bz < 2; ++bz)
                        for (int by = 0; by < 2; ++by)
                            for (int bx = 0; bx < 2; ++bx) {
                                const double w = (bx ? wx : 1 - wx) * (by ? wy : 1 - wy) * (bz ? wz : 1 - wz);
                                acc += w * in[((zs[bz] * sd.ny + ys[by]) * sd.nx + xs[bx]) * channels + c];
                            }
                    out[((z * dd.ny + y) * dd.nx + x) * channels + c] = acc;
                }
            }
        }
    }
}

/* Returns 1 on a bad factor / a resulting dim < 2 (std::invalid_argument). out_dims is
 * written first so callers can size `out`; pass out = NULL to query. */
OR_API int or_resample_scale(const double* in, or_dims d, double factor, double* out, or_dims* out_dims) {
    if (!isfinite(factor) || factor <= 0) return 1;
    or_dims nd = d;
    if (factor != 1.0) {
        nd.nx = (int64_t)ceil((double)d.nx * factor);
        nd.ny = (int64_t)ceil((double)d.ny * factor);
        nd.nz = (int64_t)ceil((double)d.nz * factor);
        if (nd.nx < 2 || nd.ny < 2 || nd.nz < 2) return 1;
    }
    *out_dims = nd;
    if (!out) return 0;
    const int64_t n = dims_voxels(d);
    if (factor == 1.0) {
        memcpy(out, in, (size_t)n * sizeof(double));
        return 0;
    }
    double* src = (double*)malloc((size_t)n * sizeof(double));
    memcpy(src, in, (size_t)n * sizeof(double));
    if (factor < 1.0) or_gaussian_smooth(src, d, 1, 0.5 / factor);
    rs_trilinear(src, d, 1, out, nd);
    free(src);
    return 0;
}

OR_API void or_resample_warp(const double* in, or_dims d, double* out, or_dims nd) {
    rs_trilinear(in, d, 3, out, nd);
}

/* ------------------------------------------------------------- lncc.hpp:63-90 */
static inline double lncc_ncc(double muf, double mum, double muff, double mumm, double mufm, double eps) {
    const double a = mufm - muf * mum;
    const double b = muff - muf * muf;
    const double c = mumm - mum * mum;
    return a * a / (b * c + eps);
}

static inline void lncc_gamma(double muf, double mum, double muff, double mumm, double mufm, double eps,
                              double gi, double g[5]) {
    const double a = mufm - muf * mum;
    const double b = muff - muf * muf;
    const double c = mumm - mum * mum;
    const double denom = b * c + eps;
    const double gamma = 2.0 * gi * a / denom;
    g[0] = gamma;
    g[1] = gamma * (a * c / denom);
    g[2] = gamma * (a * b / denom);
    g[3] = gamma * (muf * (a * c / denom) - mum);
    g[4] = gamma * (mum * (a * b / denom) - muf);
}

/*
 * lncc_forward_fused (lncc.hpp:144-205). state: 5*N doubles, channel-major
 * (mean_f, mean_m, mean_ff, mean_mm, mean_fm). map may be NULL. Returns the loss.
 * Box window zero-padded, no renormalization (lncc.hpp:16-17, 178-188).
 */
OR_API double or_lncc_forward(const double* f, const double* m, or_dims dims, int window, double eps,
                              double* state, double* map) {
    const int64_t n = dims_voxels(dims);
    double* ch[5];
    for (int c = 0; c < 5; ++c) ch[c] = state + (size_t)c * (size_t)n;
    for (int64_t i = 0; i < n; ++i) {
        ch[0][i] = f[i];
        ch[1][i] = m[i];
        ch[2][i] = f[i] * f[i];
        ch[3][i] = m[i] * m[i];
        ch[4][i] = f[i] * m[i];
    }
    double* taps = (double*)malloc((size_t)window * sizeof(double));
    for (int k = 0; k < window; ++k) taps[k] = 1.0 / window; /* box_taps, smoothing.hpp:42-46 */
    for (int c = 0; c < 5; ++c) or_separable_convolve(ch[c], dims, 1, taps, window, 0);
    free(taps);
    double sum = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double ni = lncc_ncc(ch[0][i], ch[1][i], ch[2][i], ch[3][i], ch[4][i], eps);
        if (map) map[i] = ni;
        sum += ni;
    }
    return 1.0 - sum / (double)n;
}

/*
 * lncc_backward_fused (lncc.hpp:226-280): state rewritten in place as the gamma
 * family; exact mode (ants=0) convolves it with the window before the combination.
 * grad_f may be NULL.
 */
OR_API void or_lncc_backward(double upstream, double* state, const double* f, const double* m, or_dims dims,
                             int window, double eps, int ants, double* grad_f, double* grad_m) {
    const int64_t n = dims_voxels(dims);
    double* ch[5];
    for (int c = 0; c < 5; ++c) ch[c] = state + (size_t)c * (size_t)n;
    const double gi = -upstream / (double)n;
    for (int64_t i = 0; i < n; ++i) {
        double g[5];
        lncc_gamma(ch[0][i], ch[1][i], ch[2][i], ch[3][i], ch[4][i], eps, gi, g);
        for (int c = 0; c < 5; ++c) ch[c][i] = g[c];
    }
    if (!ants) {
        double* taps = (double*)malloc((size_t)window * sizeof(double));
        for (int k = 0; k < window; ++k) taps[k] = 1.0 / window;
        for (int c = 0; c < 5; ++c) or_separable_convolve(ch[c], dims, 1, taps, window, 0);
        free(taps);
    }
    for (int64_t i = 0; i < n; ++i) {
        if (grad_f) grad_f[i] = m[i] * ch[0][i] - f[i] * ch[1][i] + ch[3][i];
        grad_m[i] = f[i] * ch[0][i] - m[i] * ch[2][i] + ch[4][i];
    }
}

/* ---------------------------------------------------------------- mi.hpp:28-144 */
typedef struct {
    int kind; /* 0 gaussian, 1 bspline3, 2 delta */
    int bins;
    double sigma, radius, norm;
} or_parzen;

static double bspline3_value(double t) { /* mi.hpp:100-108 */
    const double a = fabs(t);
    if (a < 1.0) return (4.0 - 6.0 * a * a + 3.0 * a * a * a) / 6.0;
    if (a < 2.0) {
        const double q = 2.0 - a;
        return q * q * q / 6.0;
    }
    return 0.0;
}

static double bspline3_deriv(double t) { /* mi.hpp:109-118 */
    const double a = fabs(t);
    const double s = t < 0 ? -1.0 : 1.0;
    if (a < 1.0) return s * (-2.0 * a + 1.5 * a * a);
    if (a < 2.0) {
        const double q = 2.0 - a;
        return s * (-0.5 * q * q);
    }
    return 0.0;
}

OR_API double or_parzen_kappa(const or_parzen* k, double x) { /* mi.hpp:65-78 */
    switch (k->kind) {
    case 0: {
        if (fabs(x) > k->radius) return 0.0;
        const double z = x / k->sigma;
        return k->norm * exp(-0.5 * z * z);
    }
    case 1:
        return bspline3_value(x * k->bins);
    case 2:
        return fabs(x) < k->radius ? 1.0 : 0.0;
    }
    return 0.0;
}

OR_API double or_parzen_omega(const or_parzen* k, double x) { /* mi.hpp:81-93 */
    switch (k->kind) {
    case 0:
        if (fabs(x) > k->radius) return 0.0;
        return x / (k->sigma * k->sigma) * or_parzen_kappa(k, x);
    case 1:
        return -(double)k->bins * bspline3_deriv(x * k->bins);
    case 2:
        return 0.0;
    }
    return 0.0;
}

/* Constructors (mi.hpp:33-63) with the normalization check (mi.hpp:120-133).
 * Returns 0, or 3 (logic_error) when the discrete integral deviates from 1. */
OR_API int or_parzen_make(int kind, int bins, double sigma_bins, or_parzen* k) {
    k->kind = kind;
    k->bins = bins;
    k->sigma = 0;
    k->norm = 1.0;
    if (kind == 0) {
        k->sigma = sigma_bins / bins;
        k->radius = 3.0 * k->sigma;
        const double erf_mass = erf(3.0 / sqrt(2.0));
        k->norm = 1.0 / (bins * k->sigma * sqrt(2.0 * 3.14159265358979323846) * erf_mass);
    } else if (kind == 1) {
        k->radius = 2.0 / bins;
    } else {
        k->radius = 0.5 / bins;
    }
    const int steps = 20000;
    const double h = 2.0 * k->radius / steps;
    double integral = 0;
    for (int i = 0; i <= steps; ++i) {
        const double x = -k->radius + i * h;
        const double w = (i == 0 || i == steps) ? 0.5 : 1.0;
        integral += w * or_parzen_kappa(k, x);
    }
    integral *= h * bins;
    if (fabs(integral - 1.0) > 1e-3) return 3;
    return 0;
}

static inline double bin_center(int j, int bins) { return ((double)j + 0.5) / (double)bins; } /* mi.hpp:142-144 */

static int check_unit(const double* v, int64_t n) { /* mi.hpp:170-179 */
    for (int64_t i = 0; i < n; ++i)
        if (!(v[i] >= 0.0 && v[i] <= 1.0)) return 1;
    return 0;
}

/*
 * mi_forward_exact (mi.hpp:235-272): raw payload = raw_joint (B*B), raw_marg_i (B),
 * raw_marg_j (B). stats[0] = hist_writes, stats[1] = kernel_evals (mi.hpp:156-159).
 * Returns 0 or 1 (invalid_argument: intensity outside [0,1], bins < 2).
 */
OR_API int or_mi_forward_exact(const double* vi, const double* vj, int64_t n, const or_parzen* k,
                               double* raw, uint64_t* stats) {
    const int b = k->bins;
    if (b < 2 || check_unit(vi, n) || check_unit(vj, n)) return 1;
    double* joint = raw;
    double* mi = raw + (size_t)b * b;
    double* mj = mi + b;
    memset(raw, 0, sizeof(double) * ((size_t)b * b + 2 * (size_t)b));
    double* ri = (double*)malloc(sizeof(double) * (size_t)b);
    double* rj = (double*)malloc(sizeof(double) * (size_t)b);
    for (int64_t q = 0; q < n; ++q) {
        for (int m = 0; m < b; ++m) {
            ri[m] = or_parzen_kappa(k, bin_center(m, b) - vi[q]);
            rj[m] = or_parzen_kappa(k, bin_center(m, b) - vj[q]);
        }
        for (int m = 0; m < b; ++m) {
            mi[m] += ri[m];
            mj[m] += rj[m];
        }
        for (int m = 0; m < b; ++m) {
            const double w = ri[m];
            double* row = joint + (size_t)m * b;
            for (int nn = 0; nn < b; ++nn) row[nn] += w * rj[nn];
        }
    }
    if (stats) {
        stats[0] += (uint64_t)n * ((uint64_t)b * b + 2ull * b);
        stats[1] += (uint64_t)n * 2ull * b;
    }
    free(ri);
    free(rj);
    return 0;
}

/* mi_forward_approx + kernel_bin_taps (mi.hpp:275-354). */
OR_API int or_mi_forward_approx(const double* vi, const double* vj, int64_t n, const or_parzen* k,
                                double* raw, uint64_t* stats) {
    const int b = k->bins;
    if (b < 2 || check_unit(vi, n) || check_unit(vj, n)) return 1;
    double* cij = (double*)calloc((size_t)b * b, sizeof(double));
    double* ci = (double*)calloc((size_t)b, sizeof(double));
    double* cj = (double*)calloc((size_t)b, sizeof(double));
    for (int64_t q = 0; q < n; ++q) {
        int mb = (int)(vi[q] * b);
        if (mb > b - 1) mb = b - 1;
        int nb = (int)(vj[q] * b);
        if (nb > b - 1) nb = b - 1;
        cij[(size_t)mb * b + nb] += 1.0;
        ci[mb] += 1.0;
        cj[nb] += 1.0;
    }
    if (stats) stats[0] += 3ull * (uint64_t)n;
    const int radius = (int)ceil(k->radius * k->bins);
    const int nt = 2 * radius + 1;
    double* taps = (double*)malloc(sizeof(double) * (size_t)nt);
    for (int d = -radius; d <= radius; ++d) taps[d + radius] = or_parzen_kappa(k, (double)d / b);
    double* joint = raw;
    double* mi = raw + (size_t)b * b;
    double* mj = mi + b;
    for (int m = 0; m < b; ++m) {
        double ai = 0, aj = 0;
        for (int d = -radius; d <= radius; ++d) {
            const int s = m - d;
            if (s < 0 || s >= b) continue;
            ai += taps[d + radius] * ci[s];
            aj += taps[d + radius] * cj[s];
        }
        mi[m] = ai;
        mj[m] = aj;
    }
    double* tmp = (double*)calloc((size_t)b * b, sizeof(double));
    for (int m = 0; m < b; ++m)
        for (int nn = 0; nn < b; ++nn) {
            double acc = 0;
            for (int d = -radius; d <= radius; ++d) {
                const int s = m - d;
                if (s < 0 || s >= b) continue;
                acc += taps[d + radius] * cij[(size_t)s * b + nn];
            }
            tmp[(size_t)m * b + nn] = acc;
        }
    for (int m = 0; m < b; ++m)
        for (int nn = 0; nn < b; ++nn) {
            double acc = 0;
            for (int d = -radius; d <= radius; ++d) {
                const int s = nn - d;
                if (s < 0 || s >= b) continue;
                acc += taps[d + radius] * tmp[(size_t)m * b + s];
            }
            joint[(size_t)m * b + nn] = acc;
        }
    free(tmp);
    free(taps);
    free(cij);
    free(ci);
    free(cj);
    return 0;
}

/*
 * finalize_histogram + histogram_mi (mi.hpp:181-209). p_ij: B*B, p_i, p_j: B.
 * Returns MI; *z_out = raw joint sum.
 */
OR_API double or_mi_finalize(const double* raw_joint, int b, double* p_ij, double* p_i, double* p_j,
                             double* z_out) {
    double z = 0;
    for (size_t i = 0; i < (size_t)b * b; ++i) z += raw_joint[i];
    for (size_t i = 0; i < (size_t)b * b; ++i) p_ij[i] = raw_joint[i] / z;
    for (int m = 0; m < b; ++m) p_i[m] = p_j[m] = 0;
    for (int m = 0; m < b; ++m)
        for (int nn = 0; nn < b; ++nn) {
            const double v = p_ij[(size_t)m * b + nn];
            p_i[m] += v;
            p_j[nn] += v;
        }
    double mi = 0;
    for (int m = 0; m < b; ++m)
        for (int nn = 0; nn < b; ++nn) {
            const double p = p_ij[(size_t)m * b + nn];
            if (p <= 0) continue;
            mi += p * log(p / (p_i[m] * p_j[nn]));
        }
    if (z_out) *z_out = z;
    return mi;
}

/* ghat table of mi_backward_impl (mi.hpp:369-390). */
OR_API void or_mi_ghat(double upstream, const double* p_ij, const double* p_i, const double* p_j, double z,
                       int b, double* ghat) {
    double dot = 0;
    for (int m = 0; m < b; ++m)
        for (int nn = 0; nn < b; ++nn) {
            const size_t q = (size_t)m * b + nn;
            ghat[q] = 0;
            const double p = p_ij[q];
            if (p <= 0) continue;
            const double g = log(p / (p_i[m] * p_j[nn])) - 1.0;
            ghat[q] = g;
            dot += g * p;
        }
    for (size_t q = 0; q < (size_t)b * b; ++q) {
        if (p_ij[q] <= 0) {
            ghat[q] = 0;
            continue;
        }
        ghat[q] = upstream * (ghat[q] - dot) / z;
    }
}

/* per-voxel part of mi_backward_impl (mi.hpp:392-421). grad_i may be NULL. */
OR_API void or_mi_backward(const double* vi, const double* vj, int64_t n, const or_parzen* k,
                           const double* ghat, double* grad_i, double* grad_j) {
    const int b = k->bins;
    double* ki = (double*)malloc(sizeof(double) * (size_t)b * 4);
    double* wi = ki + b;
    double* kj = wi + b;
    double* wj = kj + b;
    for (int64_t q = 0; q < n; ++q) {
        for (int m = 0; m < b; ++m) {
            const double di = bin_center(m, b) - vi[q];
            const double dj = bin_center(m, b) - vj[q];
            ki[m] = or_parzen_kappa(k, di);
            wi[m] = or_parzen_omega(k, di);
            kj[m] = or_parzen_kappa(k, dj);
            wj[m] = or_parzen_omega(k, dj);
        }
        double gi = 0, gj = 0;
        for (int m = 0; m < b; ++m) {
            const double* row = ghat + (size_t)m * b;
            double ai = 0, aj = 0;
            for (int nn = 0; nn < b; ++nn) {
                ai += row[nn] * kj[nn];
                aj += row[nn] * wj[nn];
            }
            gi += wi[m] * ai;
            gj += ki[m] * aj;
        }
        if (grad_i) grad_i[q] = gi;
        grad_j[q] = gj;
    }
    free(ki);
}

/* ------------------------------------------------------------ fabric.hpp:44-70 */
/* shard_ranges + make_shard_spec bounds along z. Returns 0 or 1 (invalid_argument). */
OR_API int or_shard_range(int64_t n, int world, int rank, int64_t* lo, int64_t* hi) {
    if (world < 1 || n < world || rank < 0 || rank >= world) return 1;
    const int64_t base = n / world, extra = n % world;
    int64_t l = 0;
    for (int h = 0; h < rank; ++h) l += base + (h < extra ? 1 : 0);
    *lo = l;
    *hi = l + base + (rank < extra ? 1 : 0);
    return 0;
}

/* compute_shard_rescale (distops.hpp:41-49) applied per ring_step_args (122-133). */
static void ring_step_args(or_dims mg, int world, int src, const double* A, const double* t, double* Ah,
                           double* th, double* Sh) {
    int64_t lo, hi;
    or_shard_range(mg.nz, world, src, &lo, &hi);
    const double smin[3] = {-1, -1, lattice_coord(-1.0, 1.0, lo, mg.nz)};
    const double smax[3] = {1, 1, lattice_coord(-1.0, 1.0, hi - 1, mg.nz)};
    for (int c = 0; c < 3; ++c) {
        const double S = (1.0 - -1.0) / (smax[c] - smin[c]);
        const double tt = -1.0 - S * smin[c];
        for (int k = 0; k < 3; ++k) Ah[3 * c + k] = S * A[3 * c + k];
        th[c] = S * t[c] + tt;
        Sh[c] = S;
    }
}

/*
 * ring_sample / ring_sample_backward (distops.hpp:144-248) restated in one process:
 * the rank `rank` output slab (out_bounds, u_shard on its lattice) accumulates the
 * zero-padded partial interpolation of every moving shard in its own frame.
 * m_full is the whole moving volume (shards are read in place).
 * Backward: g_u accumulated; gAt (12 = gA, gt) chained through S_h, NOT allreduced.
 */
OR_API int or_ring_sample(const double* m_full, or_dims mg, int world, const double* u_shard, or_dims odims,
                          const double* out_bounds, const double* A, const double* t, double* out,
                          const double* upstream, double* g_u, double* gAt) {
    for (int h = 0; h < world; ++h) {
        int64_t lo, hi;
        if (or_shard_range(mg.nz, world, h, &lo, &hi)) return 1;
        or_dims sd = {mg.nx, mg.ny, hi - lo};
        const double* shard = m_full + (size_t)(lo * mg.nx * mg.ny);
        double Ah[9], th[3], Sh[3];
        ring_step_args(mg, world, h, A, t, Ah, th, Sh);
        double gA[9] = {0}, gt[3] = {0};
        int rc = or_sample_core(shard, sd, u_shard, odims, Ah, th, Sh, out_bounds, out, upstream, NULL, g_u,
                                gAt ? gA : NULL, gAt ? gt : NULL, NULL);
        if (rc) return rc;
        if (gAt)
            for (int r = 0; r < 3; ++r) {
                for (int c = 0; c < 3; ++c) gAt[3 * r + c] += Sh[r] * gA[3 * r + c];
                gAt[9 + r] += Sh[r] * gt[r];
            }
    }
    return 0;
}

/* ----------------------------------------------------------- synth.hpp:86-135 */
OR_API void or_random_volume(or_rng* r, double* v, int64_t n, double lo, double hi) {
    /* oracles.hpp random_volume pattern: uniform per voxel */
    for (int64_t i = 0; i < n; ++i) v[i] = or_rng_uniform_range(r, lo, hi);
}

static void rasterize_ellipsoids(or_rng* r, or_dims d, int k, uint16_t* lab) { /* synth.hpp:86-106 */
    memset(lab, 0, sizeof(uint16_t) * (size_t)dims_voxels(d));
    for (int label = 1; label <= k; ++label) {
        double center[3], radius[3];
        for (int c = 0; c < 3; ++c) {
            const double n = (double)dims_axis(d, c);
            center[c] = or_rng_uniform_range(r, 0.22, 0.78) * (n - 1);
            radius[c] = or_rng_uniform_range(r, 0.10, 0.24) * n;
        }
        for (int64_t z = 0; z < d.nz; ++z)
            for (int64_t y = 0; y < d.ny; ++y)
                for (int64_t x = 0; x < d.nx; ++x) {
                    const double dx = ((double)x - center[0]) / radius[0];
                    const double dy = ((double)y - center[1]) / radius[1];
                    const double dz = ((double)z - center[2]) / radius[2];
                    if (dx * dx + dy * dy + dz * dz <= 1.0) lab[vidx(d, x, y, z)] = (uint16_t)label;
                }
    }
}

static void random_smooth_warp(or_rng* r, or_dims d, double max_norm, double sigma, double rms_fraction,
                               double* w) { /* synth.hpp:80-114 */
    const int64_t n = dims_voxels(d);
    for (int64_t i = 0; i < 3 * n; ++i) w[i] = or_rng_normal(r);
    or_gaussian_smooth(w, d, 3, sigma);
    double sq = 0;
    for (int64_t i = 0; i < n; ++i) {
        double s = 0;
        for (int c = 0; c < 3; ++c) s += w[3 * i + c] * w[3 * i + c];
        sq += s;
    }
    const double rms = sqrt(sq / (double)n);
    if (rms > 0 && max_norm > 0) {
        const double scale = rms_fraction * max_norm / rms;
        for (int64_t i = 0; i < 3 * n; ++i) w[i] *= scale;
        for (int64_t i = 0; i < n; ++i) {
            double s = 0;
            for (int c = 0; c < 3; ++c) s += w[3 * i + c] * w[3 * i + c];
            const double norm = sqrt(s);
            if (norm > max_norm) {
                const double clip = max_norm / norm;
                for (int c = 0; c < 3; ++c) w[3 * i + c] *= clip;
            }
        }
    } else if (max_norm == 0) {
        for (int64_t i = 0; i < 3 * n; ++i) w[i] = 0;
    }
}

/*
 * synth_pair (synth.hpp:116-137) without the label outputs: fixed, moving (N each),
 * true_warp (3N). Returns 0 or 1 (invalid_argument).
 */
OR_API int or_synth_pair(uint64_t seed, or_dims d, int k, double max_disp, double* fixed, double* moving,
                         double* true_warp) {
    if (d.nx < 16 || d.ny < 16 || d.nz < 16) return 1;
    if (k < 1 || k > 16) return 1;
    if (!(max_disp >= 0) || max_disp > 0.15) return 1;
    const int64_t n = dims_voxels(d);
    or_rng r;
    or_rng_init(&r, seed);
    uint16_t* lab = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
    rasterize_ellipsoids(&r, d, k, lab);
    double mu[17] = {0}, sg[17] = {0}; /* draw_label_stats, synth.hpp:108-117 */
    for (int l = 1; l <= k; ++l) {
        mu[l] = or_rng_uniform_range(&r, 0.3, 1.0);
        sg[l] = or_rng_uniform_range(&r, 0.02, 0.06);
    }
    for (int64_t i = 0; i < n; ++i) { /* paint_labels, synth.hpp:119-128 */
        const uint16_t l = lab[i];
        fixed[i] = 0;
        if (l == 0) continue;
        fixed[i] = mu[l] + sg[l] * or_rng_normal(&r);
    }
    free(lab);
    or_gaussian_smooth(fixed, d, 1, 0.75);
    random_smooth_warp(&r, d, max_disp, (double)d.nx / 8.0, 0.7, true_warp);
    memset(moving, 0, sizeof(double) * (size_t)n);
    const double A[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0}, S[3] = {1, 1, 1};
    const double bounds[6] = {-1, -1, -1, 1, 1, 1};
    or_sample_core(fixed, d, true_warp, d, A, t, S, bounds, moving, NULL, NULL, NULL, NULL, NULL, NULL);
    return 0;
}

/* normalize_intensities (registration.hpp:100-115). */
OR_API void or_normalize_intensities(double* v, int64_t n) {
    double lo = v[0], hi = v[0];
    for (int64_t i = 0; i < n; ++i) {
        if (v[i] < lo) lo = v[i];
        if (v[i] > hi) hi = v[i];
    }
    const double range = hi - lo;
    for (int64_t i = 0; i < n; ++i) v[i] = range <= 0 ? 0.0 : (v[i] - lo) / range;
}

/* ------------------------------------------------ the step (registration.hpp:277-312) */
/*
 * One deformable-step evaluation at H=1 for LNCC: moved = fused_sample(M, u; A, t),
 * dist_lncc(window, eps, ants) with gi = -1/N, g_u = fused_sample_backward(want warp).
 * moved / grad_moved may be NULL. Returns the loss.
 */
OR_API double or_step_lncc(const double* f, const double* m, or_dims d, const double* u, const double* A,
                           const double* t, int window, double eps, int ants, double* g_u, double* moved_out,
                           double* grad_moved_out) {
    const int64_t n = dims_voxels(d);
    const double S[3] = {1, 1, 1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
    double* moved = (double*)calloc((size_t)n, sizeof(double));
    or_sample_core(m, d, u, d, A, t, S, bounds, moved, NULL, NULL, NULL, NULL, NULL, NULL);
    double* state = (double*)malloc(sizeof(double) * 5 * (size_t)n);
    const double loss = or_lncc_forward(f, moved, d, window, eps, state, NULL);
    double* gm = (double*)malloc(sizeof(double) * (size_t)n);
    or_lncc_backward(1.0, state, f, moved, d, window, eps, ants, NULL, gm);
    memset(g_u, 0, sizeof(double) * 3 * (size_t)n);
    or_sample_core(m, d, u, d, A, t, S, bounds, NULL, gm, NULL, g_u, NULL, NULL, NULL);
    if (moved_out) memcpy(moved_out, moved, sizeof(double) * (size_t)n);
    if (grad_moved_out) memcpy(grad_moved_out, gm, sizeof(double) * (size_t)n);
    free(moved);
    free(state);
    free(gm);
    return loss;
}

/* Same for Mattes MI (dist_mi, distops.hpp:355-396 at H=1): loss = -MI. */
OR_API double or_step_mi(const double* f, const double* m, or_dims d, const double* u, const double* A,
                         const double* t, const or_parzen* k, int approx, double* g_u, double* moved_out,
                         double* grad_moved_out, double* raw_out) {
    const int64_t n = dims_voxels(d);
    const int b = k->bins;
    const double S[3] = {1, 1, 1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
    double* moved = (double*)calloc((size_t)n, sizeof(double));
    or_sample_core(m, d, u, d, A, t, S, bounds, moved, NULL, NULL, NULL, NULL, NULL, NULL);
    double* raw = (double*)malloc(sizeof(double) * ((size_t)b * b + 2 * (size_t)b));
    int rc = approx ? or_mi_forward_approx(f, moved, n, k, raw, NULL) : or_mi_forward_exact(f, moved, n, k, raw, NULL);
    if (rc) {
        free(moved);
        free(raw);
        return NAN;
    }
    double* p_ij = (double*)malloc(sizeof(double) * ((size_t)b * b * 2 + 2 * (size_t)b));
    double* p_i = p_ij + (size_t)b * b;
    double* p_j = p_i + b;
    double* ghat = p_j + b;
    double z;
    const double mi = or_mi_finalize(raw, b, p_ij, p_i, p_j, &z);
    or_mi_ghat(-1.0, p_ij, p_i, p_j, z, b, ghat);
    double* gm = (double*)malloc(sizeof(double) * (size_t)n);
    or_mi_backward(f, moved, n, k, ghat, NULL, gm);
    memset(g_u, 0, sizeof(double) * 3 * (size_t)n);
    or_sample_core(m, d, u, d, A, t, S, bounds, NULL, gm, NULL, g_u, NULL, NULL, NULL);
    if (moved_out) memcpy(moved_out, moved, sizeof(double) * (size_t)n);
    if (grad_moved_out) memcpy(grad_moved_out, gm, sizeof(double) * (size_t)n);
    if (raw_out) memcpy(raw_out, raw, sizeof(double) * ((size_t)b * b + 2 * (size_t)b));
    free(moved);
    free(raw);
    free(p_ij);
    free(gm);
    return -mi;
}

/*
 * deformable_stage (registration.hpp:230-331) at H = 1: per scale, resample F and M
 * (resample_scale with factor 1 / downsample), carry the warp over (resample_warp, zeros
 * at the first scale), convert lr to normalized units (257-264), then `iterations` times:
 * the step (LNCC ANTs / exact or MI) -> trace[k++] = loss -> the warp update
 * (or_warp_update, 313-317). Finally the warp is resampled onto F's lattice. Returns 0,
 * 1 (invalid argument) or 2 (non-finite loss: NumericalError, trace up to it kept).
 * loss_kind 0 = LNCC, 1 = MI (mi_kind: 0 gaussian, 1 bspline3).
 */
OR_API int or_deformable_stage(const double* fixed, const double* moving, or_dims d, const double* A,
                               const double* t, int nsteps, const double* downsample, const int* iterations,
                               double lr, double sigma_grad, double sigma_warp, int loss_kind, int window,
                               double eps, int ants, int bins, int mi_kind, double* warp_out, double* trace) {
    if (nsteps < 1 || !(lr > 0) || !(sigma_grad >= 0) || !(sigma_warp >= 0)) return 1;
    for (int s = 0; s < nsteps; ++s)
        if (!(downsample[s] >= 1) || iterations[s] < 0 || (s > 0 && downsample[s] > downsample[s - 1])) return 1;
    or_parzen k;
    if (loss_kind == 1 && or_parzen_make(mi_kind, bins, 0.5, &k)) return 1;
    double* warp = NULL;
    or_dims wd = d;
    int tk = 0;
    for (int s = 0; s < nsteps; ++s) {
        const double factor = 1.0 / downsample[s];
        or_dims sd;
        if (or_resample_scale(fixed, d, factor, NULL, &sd)) {
            free(warp);
            return 1;
        }
        const int64_t n = dims_voxels(sd);
        double* fs = (double*)malloc(sizeof(double) * (size_t)n);
        double* ms = (double*)malloc(sizeof(double) * (size_t)n);
        or_resample_scale(fixed, d, factor, fs, &sd);
        or_resample_scale(moving, d, factor, ms, &sd);
        double* u = (double*)calloc(3 * (size_t)n, sizeof(double));
        if (warp) or_resample_warp(warp, wd, u, sd);
        free(warp);
        warp = u;
        wd = sd;
        const double pitch = (2.0 / (double)(sd.nx - 1) + 2.0 / (double)(sd.ny - 1) + 2.0 / (double)(sd.nz - 1)) / 3.0;
        const double lr_norm = lr * pitch;
        double* m1 = (double*)calloc(3 * (size_t)n, sizeof(double));
        double* m2 = (double*)calloc(3 * (size_t)n, sizeof(double));
        double* g = (double*)malloc(sizeof(double) * 3 * (size_t)n);
        int bad = 0;
        for (int it = 0; it < iterations[s]; ++it) {
            const double loss = loss_kind == 0 ? or_step_lncc(fs, ms, sd, warp, A, t, window, eps, ants, g, NULL, NULL)
                                               : or_step_mi(fs, ms, sd, warp, A, t, &k, 0, g, NULL, NULL, NULL);
            trace[tk++] = loss;
            if (!isfinite(loss)) {
                bad = 1;
                break;
            }
            or_warp_update(g, warp, m1, m2, sd, sigma_grad, sigma_warp, lr_norm, 0.9, 0.999, 1e-8, it + 1);
        }
        free(fs);
        free(ms);
        free(m1);
        free(m2);
        free(g);
        if (bad) {
            free(warp);
            return 2;
        }
    }
    if (wd.nx != d.nx || wd.ny != d.ny || wd.nz != d.nz)
        or_resample_warp(warp, wd, warp_out, d);
    else
        memcpy(warp_out, warp, sizeof(double) * 3 * (size_t)dims_voxels(d));
    free(warp);
    return 0;
}

/* loss_and_grad (registration.hpp:123-173) on one host: 0 = MSE, 1 = LNCC (fused forward,
 * backward with upstream 1), 2 = MI (exact forward, mi_backward_impl with upstream -1,
 * loss = -MI). Returns the loss (NaN when the MI inputs leave [0, 1]). */
static double loss_and_grad(int kind, const double* f, const double* moved, or_dims d, int window, double eps,
                            int ants, const or_parzen* k, double* gm) {
    const int64_t n = dims_voxels(d);
    if (kind == 0) {
        double sum = 0;
        for (int64_t i = 0; i < n; ++i) {
            const double dd = moved[i] - f[i];
            sum += dd * dd;
            gm[i] = 2.0 * dd / (double)n;
        }
        return sum / (double)n;
    }
    if (kind == 1) {
        double* state = (double*)malloc(sizeof(double) * 5 * (size_t)n);
        const double loss = or_lncc_forward(f, moved, d, window, eps, state, NULL);
        or_lncc_backward(1.0, state, f, moved, d, window, eps, ants, NULL, gm);
        free(state);
        return loss;
    }
    const int b = k->bins;
    double* raw = (double*)malloc(sizeof(double) * ((size_t)b * b + 2 * (size_t)b));
    if (or_mi_forward_exact(f, moved, n, k, raw, NULL)) {
        free(raw);
        return NAN;
    }
    double* p_ij = (double*)malloc(sizeof(double) * ((size_t)b * b * 2 + 2 * (size_t)b));
    double* p_i = p_ij + (size_t)b * b;
    double* p_j = p_i + b;
    double* ghat = p_j + b;
    double z;
    const double mi = or_mi_finalize(raw, b, p_ij, p_i, p_j, &z);
    or_mi_ghat(-1.0, p_ij, p_i, p_j, z, b, ghat);
    or_mi_backward(f, moved, n, k, ghat, NULL, gm);
    free(raw);
    free(p_ij);
    return -mi;
}

/*
 * affine_stage (registration.hpp:176-219): Adam (adam.hpp, state over all scales) on the
 * 12 affine parameters (A row-major, then t) from the identity; per iteration
 * moved = fused_sample(M_s, zero warp, A, t), loss_and_grad, fused_sample_backward
 * (want affine + translation). loss_kind 0 MSE, 1 LNCC, 2 MI. Returns 0, 1 (invalid
 * schedule) or 2 (non-finite loss).
 */
OR_API int or_affine_stage(const double* fixed, const double* moving, or_dims d, int nsteps, const double* downsample,
                           const int* iterations, double lr, int loss_kind, int window, double eps, int ants,
                           int bins, int mi_kind, double* A_out, double* t_out, double* trace) {
    if (nsteps < 1 || !(lr > 0)) return 1;
    for (int s = 0; s < nsteps; ++s)
        if (!(downsample[s] >= 1) || iterations[s] < 0 || (s > 0 && downsample[s] > downsample[s - 1])) return 1;
    or_parzen k;
    if (loss_kind == 2 && or_parzen_make(mi_kind, bins, 0.5, &k)) return 1;
    double params[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0}, m1[12] = {0}, m2[12] = {0};
    int64_t step = 0;
    int tk = 0;
    const double S[3] = {1, 1, 1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
    for (int s = 0; s < nsteps; ++s) {
        const double factor = 1.0 / downsample[s];
        or_dims sd;
        if (or_resample_scale(fixed, d, factor, NULL, &sd)) return 1;
        const int64_t n = dims_voxels(sd);
        double* fs = (double*)malloc(sizeof(double) * (size_t)n);
        double* ms = (double*)malloc(sizeof(double) * (size_t)n);
        or_resample_scale(fixed, d, factor, fs, &sd);
        or_resample_scale(moving, d, factor, ms, &sd);
        double* zw = (double*)calloc(3 * (size_t)n, sizeof(double));
        double* moved = (double*)malloc(sizeof(double) * (size_t)n);
        double* gm = (double*)malloc(sizeof(double) * (size_t)n);
        int bad = 0;
        for (int it = 0; it < iterations[s] && !bad; ++it) {
            memset(moved, 0, sizeof(double) * (size_t)n);
            or_sample_core(ms, sd, zw, sd, params, params + 9, S, bounds, moved, NULL, NULL, NULL, NULL, NULL, NULL);
            const double loss = loss_and_grad(loss_kind, fs, moved, sd, window, eps, ants, &k, gm);
            trace[tk++] = loss;
            if (!isfinite(loss)) {
                bad = 1;
                break;
            }
            double grad[12] = {0};
            or_sample_core(ms, sd, zw, sd, params, params + 9, S, bounds, NULL, gm, NULL, NULL, grad, grad + 9, NULL);
            or_adam_step(params, grad, m1, m2, 12, lr, 0.9, 0.999, 1e-8, ++step);
        }
        free(fs);
        free(ms);
        free(zw);
        free(moved);
        free(gm);
        if (bad) return 2;
    }
    memcpy(A_out, params, 9 * sizeof(double));
    memcpy(t_out, params + 9, 3 * sizeof(double));
    return 0;
}

/* jacobian_positive_fraction (metrics.hpp:145-176). Returns -1 for a lattice < 3. */
OR_API double or_jacobian_positive(const double* u, or_dims d) {
    if (d.nx < 3 || d.ny < 3 || d.nz < 3) return -1.0;
    const double step[3] = {2.0 / (double)(d.nx - 1), 2.0 / (double)(d.ny - 1), 2.0 / (double)(d.nz - 1)};
    int64_t pos = 0, tot = 0;
    for (int64_t z = 1; z + 1 < d.nz; ++z)
        for (int64_t y = 1; y + 1 < d.ny; ++y)
            for (int64_t x = 1; x + 1 < d.nx; ++x) {
                double j[3][3];
                for (int c = 0; c < 3; ++c) {
                    j[c][0] = (u[3 * vidx(d, x + 1, y, z) + c] - u[3 * vidx(d, x - 1, y, z) + c]) / (2 * step[0]);
                    j[c][1] = (u[3 * vidx(d, x, y + 1, z) + c] - u[3 * vidx(d, x, y - 1, z) + c]) / (2 * step[1]);
                    j[c][2] = (u[3 * vidx(d, x, y, z + 1) + c] - u[3 * vidx(d, x, y, z - 1) + c]) / (2 * step[2]);
                    j[c][c] += 1.0;
                }
                const double det = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                                   j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                                   j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
                pos += det > 0;
                ++tot;
            }
    return (double)pos / (double)tot;
}
