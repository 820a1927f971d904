/*
 * ffdp_oracle_big.c -- TEST INFRASTRUCTURE ONLY (parity checker; linked into
 * libffdp_oracle.so beside ffdp_oracle.c, never shipped or measured as the product).
 *
 * Full-size parity checks at BASELINE configs[2] / configs[4] (331.8 M / 3.7 G voxels),
 * where the whole-volume oracle (ffdp_oracle.c, one thread, fp64 state buffers) is too
 * slow or too large. The arithmetic is the same restatement of the reference, taken at
 * fp32-stored inputs (the GPU's storage type) and evaluated in fp64:
 *
 *   - or_lncc_sum_n_f32: sum over the lattice of n_i = A^2 / (B C + eps) of
 *     lncc_forward_fused (lncc.hpp:144-205; lncc_ncc lncc.hpp:63-70) with the moving
 *     image warped by composite_sample_core (sampler.hpp:165-243): the 7^3 zero-padded
 *     box (smoothing.hpp:42-94) as fp64 sums, OpenMP over z chunks.
 *   - or_lncc_ants_voxels_f32: at listed voxels only, n_i, the ANTs dL/dMw
 *     (lncc.hpp:226-280 with ants_approx: gamma family of lncc_gamma lncc.hpp:72-90,
 *     combination grad_m = f*gamma - m*gamma_AC + gamma_MF) and
 *     g_u = S * dfrac * (n-1)/2 * dL/dMw (sampler.hpp:221-230): each needs only the
 *     voxel's 7^3 window, and gi = -1/N.
 *   - or_mi_hist_f32: the raw Parzen joint histogram of mi_forward_exact (mi.hpp:235-272)
 *     of (F, Mw), OpenMP with per-thread tables; marginals as the reference's raw sums.
 *   - or_mi_voxels_f32: at listed voxels, the per-voxel part of mi_backward_impl
 *     (mi.hpp:392-421) given the ghat table, and g_u.
 * Bounds are the default [-1, 1]^3 and S = 1, as in the deformable step at H = 1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_API __attribute__((visibility("default")))

typedef struct {
    int64_t nx, ny, nz;
} or_dims;

typedef struct {
    int kind; /* 0 gaussian, 1 bspline3, 2 delta */
    int bins;
    double sigma, radius, norm;
} or_parzen;

double or_parzen_kappa(const or_parzen* k, double x);
double or_parzen_omega(const or_parzen* k, double x);

/* geometry.hpp:99-104 with bounds [-1, 1] */
static inline double lcoord(int64_t i, int64_t n) { return n <= 1 ? -1.0 : -1.0 + 2.0 * ((double)i / (double)(n - 1)); }

/* composite_sample_core's value and d(value)/d(frac) at output voxel (x, y, z), S = 1
 * (sampler.hpp:165-243; cell_assign resample.hpp:17-43; sample_cell[_dfrac] 116-161). */
static double warp_at(const float* m, or_dims d, const float* u, const double* A, const double* t, int64_t x,
                      int64_t y, int64_t z, double dx[3]) {
    const double X[3] = {lcoord(x, d.nx), lcoord(y, d.ny), lcoord(z, d.nz)};
    const int64_t o = (z * d.ny + y) * d.nx + x;
    const int64_t n[3] = {d.nx, d.ny, d.nz};
    int64_t i0[3];
    double fr[3];
    for (int r = 0; r < 3; ++r) {
        double xs = A[3 * r + 0] * X[0] + A[3 * r + 1] * X[1] + A[3 * r + 2] * X[2] + t[r];
        xs += (double)u[3 * o + r];
        const double f = (xs + 1.0) * 0.5 * (double)(n[r] - 1);
        double fl = floor(f), a = f - fl;
        if (a < 1e-9) {
            a = 0.0;
        } else if (1.0 - a < 1e-9) {
            fl += 1.0;
            a = 0.0;
        }
        i0[r] = (int64_t)fl;
        fr[r] = a;
    }
    double v = 0, g[3] = {0, 0, 0};
    for (int bz = 0; bz < 2; ++bz) {
        const int64_t iz = i0[2] + bz;
        if (iz < 0 || iz >= d.nz) continue;
        const double wz = bz ? fr[2] : 1 - fr[2], sz = bz ? 1.0 : -1.0;
        for (int by = 0; by < 2; ++by) {
            const int64_t iy = i0[1] + by;
            if (iy < 0 || iy >= d.ny) continue;
            const double wy = by ? fr[1] : 1 - fr[1], sy = by ? 1.0 : -1.0;
            for (int bx = 0; bx < 2; ++bx) {
                const int64_t ix = i0[0] + bx;
                if (ix < 0 || ix >= d.nx) continue;
                const double wx = bx ? fr[0] : 1 - fr[0], sx = bx ? 1.0 : -1.0;
                const double mv = (double)m[(iz * d.ny + iy) * d.nx + ix];
                v += wz * wy * wx * mv;
                g[0] += sx * wy * wz * mv;
                g[1] += wx * sy * wz * mv;
                g[2] += wx * wy * sz * mv;
            }
        }
    }
    if (dx)
        for (int r = 0; r < 3; ++r) dx[r] = g[r] * 0.5 * (double)(n[r] - 1);
    return v;
}

/* x then y box sums (window w, zero pad) of the 5 channels of one plane: out[c][y*nx+x]. */
static void plane_box(const float* f, const double* mw, or_dims d, int r, double* tmp, double* out) {
    const int64_t nx = d.nx, ny = d.ny, np = nx * ny;
    for (int64_t y = 0; y < ny; ++y) {
        for (int c = 0; c < 5; ++c) {
            double* row = tmp + c * np + y * nx;
            for (int64_t x = 0; x < nx; ++x) {
                double s = 0;
                for (int64_t k = x - r; k <= x + r; ++k) {
                    if (k < 0 || k >= nx) continue;
                    const double a = f[y * nx + k], b = mw[y * nx + k];
                    s += c == 0 ? a : c == 1 ? b : c == 2 ? a * a : c == 3 ? b * b : a * b;
                }
                row[x] = s;
            }
        }
    }
    for (int c = 0; c < 5; ++c)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double s = 0;
                for (int64_t k = y - r; k <= y + r; ++k)
                    if (k >= 0 && k < ny) s += tmp[c * np + k * nx + x];
                out[c * np + y * nx + x] = s;
            }
}

static inline double ncc_from_sums(const double s[5], double inv, double eps) { /* lncc.hpp:63-70 */
    const double muf = s[0] * inv, mum = s[1] * inv, muff = s[2] * inv, mumm = s[3] * inv, mufm = s[4] * inv;
    const double a = mufm - muf * mum, b = muff - muf * muf, c = mumm - mum * mum;
    return a * a / (b * c + eps);
}

OR_API double or_lncc_sum_n_f32(const float* f, const float* m, const float* u, or_dims d, const double* A,
                                const double* t, int window, double eps) {
    const int r = window / 2;
    const int64_t nx = d.nx, ny = d.ny, nz = d.nz, np = nx * ny;
    const double inv = 1.0 / ((double)window * window * window);
    double total = 0;
#pragma omp parallel reduction(+ : total)
    {
        double* mw = (double*)malloc(sizeof(double) * (size_t)np);
        double* tmp = (double*)malloc(sizeof(double) * 5 * (size_t)np);
        double* ring = (double*)malloc(sizeof(double) * 5 * (size_t)np * (size_t)window);
#pragma omp for schedule(dynamic, 1)
        for (int64_t zc = 0; zc < nz; zc += 16) {
            const int64_t z1 = zc + 16 < nz ? zc + 16 : nz;
            /* planes zc - r .. z1 + r - 1 enter the ring; plane p's window sum is ready when p + r entered */
            for (int64_t p = zc - r; p < z1 + r; ++p) {
                double* slot = ring + (size_t)(((p % window) + window) % window) * 5 * (size_t)np;
                if (p < 0 || p >= nz) {
                    memset(slot, 0, sizeof(double) * 5 * (size_t)np);
                } else {
                    for (int64_t y = 0; y < ny; ++y)
                        for (int64_t x = 0; x < nx; ++x) mw[y * nx + x] = warp_at(m, d, u, A, t, x, y, p, NULL);
                    plane_box(f + p * np, mw, d, r, tmp, slot);
                }
                const int64_t q = p - r;
                if (q < zc) continue;
                for (int64_t i = 0; i < np; ++i) {
                    double s[5] = {0, 0, 0, 0, 0};
                    for (int k = 0; k < window; ++k)
                        for (int c = 0; c < 5; ++c) s[c] += ring[(size_t)k * 5 * np + (size_t)c * np + i];
                    total += ncc_from_sums(s, inv, eps);
                }
            }
        }
        free(mw);
        free(tmp);
        free(ring);
    }
    return total;
}

OR_API void or_lncc_ants_voxels_f32(const float* f, const float* m, const float* u, or_dims d, const double* A,
                                    const double* t, int window, double eps, double gi, const int64_t* vox, int64_t nv,
                                    double* out_n, double* out_gmw, double* out_gu) {
    const int r = window / 2;
    const double inv = 1.0 / ((double)window * window * window);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < nv; ++q) {
        const int64_t v = vox[q];
        const int64_t x = v % d.nx, y = (v / d.nx) % d.ny, z = v / (d.nx * d.ny);
        double s[5] = {0, 0, 0, 0, 0};
        for (int64_t zz = z - r; zz <= z + r; ++zz) {
            if (zz < 0 || zz >= d.nz) continue;
            for (int64_t yy = y - r; yy <= y + r; ++yy) {
                if (yy < 0 || yy >= d.ny) continue;
                for (int64_t xx = x - r; xx <= x + r; ++xx) {
                    if (xx < 0 || xx >= d.nx) continue;
                    const double a = f[(zz * d.ny + yy) * d.nx + xx];
                    const double b = warp_at(m, d, u, A, t, xx, yy, zz, NULL);
                    s[0] += a;
                    s[1] += b;
                    s[2] += a * a;
                    s[3] += b * b;
                    s[4] += a * b;
                }
            }
        }
        const double muf = s[0] * inv, mum = s[1] * inv, muff = s[2] * inv, mumm = s[3] * inv, mufm = s[4] * inv;
        const double a = mufm - muf * mum, b = muff - muf * muf, c = mumm - mum * mum;
        const double den = b * c + eps;
        const double gamma = 2.0 * gi * a / den;             /* lncc.hpp:80-90 */
        const double g_ac = gamma * (a * b / den);
        const double g_mf = gamma * (mum * (a * b / den) - muf);
        double dx[3];
        const double mv = warp_at(m, d, u, A, t, x, y, z, dx);
        const double gm = (double)f[v] * gamma - mv * g_ac + g_mf; /* ANTs combination, lncc.hpp:270-276 */
        out_n[q] = a * a / den;
        out_gmw[q] = gm;
        for (int k = 0; k < 3; ++k) out_gu[3 * q + k] = dx[k] * gm;
    }
}

/* Parzen weights of every bin for value v, as mi_forward_exact evaluates them
 * (mi.hpp:248-258). The B-spline is zero beyond two bins (mi.hpp:100-108): only the bins
 * with |b_j - v| * B < 2 are evaluated, the rest are the exact zeros the reference adds. */
static void parzen_row(const or_parzen* k, double v, double* kap, double* om) {
    int j0 = 0, j1 = k->bins;
    if (k->kind == 1) {
        const int c = (int)floor(v * k->bins - 0.5);
        j0 = c - 2 > 0 ? c - 2 : 0;
        j1 = c + 4 < k->bins ? c + 4 : k->bins;
        for (int j = 0; j < k->bins; ++j) {
            kap[j] = 0;
            if (om) om[j] = 0;
        }
    }
    for (int j = j0; j < j1; ++j) {
        const double x = ((double)j + 0.5) / (double)k->bins - v; /* bin_center(j) - v, mi.hpp:142-144 */
        kap[j] = or_parzen_kappa(k, x);
        if (om) om[j] = or_parzen_omega(k, x);
    }
}

OR_API void or_mi_hist_f32(const float* f, const float* m, const float* u, or_dims d, const double* A,
                           const double* t, const or_parzen* k, double* raw) {
    const int b = k->bins;
    const size_t nr = (size_t)b * b + 2 * (size_t)b;
    memset(raw, 0, sizeof(double) * nr);
    const int64_t np = d.nx * d.ny;
#pragma omp parallel
    {
        double* loc = (double*)calloc(nr, sizeof(double));
        double* ki = (double*)malloc(sizeof(double) * 2 * (size_t)b);
        double* kj = ki + b;
#pragma omp for schedule(dynamic, 1)
        for (int64_t z = 0; z < d.nz; ++z)
            for (int64_t y = 0; y < d.ny; ++y)
                for (int64_t x = 0; x < d.nx; ++x) {
                    const double fv = f[z * np + y * d.nx + x];
                    const double mv = warp_at(m, d, u, A, t, x, y, z, NULL);
                    parzen_row(k, fv, ki, NULL);
                    parzen_row(k, mv, kj, NULL);
                    for (int i = 0; i < b; ++i) {
                        loc[(size_t)b * b + i] += ki[i];
                        loc[(size_t)b * b + b + i] += kj[i];
                        if (ki[i] == 0) continue;
                        for (int j = 0; j < b; ++j) loc[(size_t)i * b + j] += ki[i] * kj[j];
                    }
                }
#pragma omp critical
        for (size_t i = 0; i < nr; ++i) raw[i] += loc[i];
        free(loc);
        free(ki);
    }
}

OR_API void or_mi_voxels_f32(const float* f, const float* m, const float* u, or_dims d, const double* A,
                             const double* t, const or_parzen* k, const double* ghat, const int64_t* vox, int64_t nv,
                             double* out_gmw, double* out_gu) {
    const int b = k->bins;
#pragma omp parallel
    {
        double* ki = (double*)malloc(sizeof(double) * 2 * (size_t)b);
        double* kj = ki + b;
        double* wj = (double*)malloc(sizeof(double) * (size_t)b);
#pragma omp for schedule(dynamic, 64)
        for (int64_t q = 0; q < nv; ++q) {
            const int64_t v = vox[q];
            const int64_t x = v % d.nx, y = (v / d.nx) % d.ny, z = v / (d.nx * d.ny);
            double dx[3];
            const double mv = warp_at(m, d, u, A, t, x, y, z, dx);
            parzen_row(k, (double)f[v], ki, NULL);
            parzen_row(k, mv, kj, wj);
            double gj = 0; /* mi.hpp:404-419: gJ = sum_m kappa_i[m] sum_n ghat[m,n] omega_j[n] */
            for (int i = 0; i < b; ++i) {
                double acc = 0;
                for (int j = 0; j < b; ++j) acc += ghat[(size_t)i * b + j] * wj[j];
                gj += ki[i] * acc;
            }
            out_gmw[q] = gj;
            for (int c = 0; c < 3; ++c) out_gu[3 * q + c] = dx[c] * gj;
        }
        free(ki);
        free(wj);
    }
}
