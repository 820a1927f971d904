/*
 * ffdp.h -- C ABI of the B200-native fused warp + loss step (libffdp.so, sm_100a).
 *
 * Drop-in boundary for the hot path of the voxreg reference engine
 * (/root/reference/proj/include/voxreg). Every entry point names the reference
 * interface it replaces (file:line). Conventions:
 *
 *  - all array arguments are DEVICE pointers (cudaMalloc'd, fp32 unless stated);
 *    scalars are host values; `stream` is a cudaStream_t (NULL = legacy default);
 *  - volumes are x-fastest, index (z*ny + y)*nx + x (volume.hpp:3-7,41-43);
 *    warp fields interleave xyz per voxel, index 3*voxel + c (volume.hpp:57,69-71);
 *  - outputs are caller-owned buffers; nothing is allocated on the caller's behalf
 *    except stream-ordered scratch that is released before the call returns;
 *  - every call returns an ffdp_status; on failure ffdp_last_error() (thread-local)
 *    holds the message. Status codes map onto the reference's exception types:
 *    FFDP_INVALID_ARGUMENT <-> std::invalid_argument, FFDP_RUNTIME <-> std::runtime_error,
 *    FFDP_LOGIC <-> std::logic_error (mi.hpp:132), FFDP_CUDA for device failures.
 *  - there is no CPU fallback: without a usable sm_100a device every call fails
 *    with FFDP_CUDA.
 */
#ifndef FFDP_H
#define FFDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFDP_ABI_VERSION 2

#if defined(__GNUC__)
#define FFDP_API __attribute__((visibility("default")))
#else
#define FFDP_API
#endif

typedef enum {
    FFDP_OK = 0,
    FFDP_INVALID_ARGUMENT = 1,
    FFDP_RUNTIME = 2,
    FFDP_LOGIC = 3,
    FFDP_CUDA = 4
} ffdp_status;

/* Dims3 (geometry.hpp:88-95). */
typedef struct {
    int64_t nx, ny, nz;
} ffdp_dims;

/* SamplerArgs (sampler.hpp:25-37) with DomainBounds (geometry.hpp:74-86) flattened. */
typedef struct {
    double A[9];     /* row-major affine, normalized coordinates */
    double t[3];     /* translation */
    double S[3];     /* diagonal rescale of the displacement */
    double x_min[3]; /* normalized coordinates of the first output voxel centre */
    double x_max[3]; /* ... and of the last */
} ffdp_sampler_args;

/* SamplerGradWant (sampler.hpp:39-44) as a bit mask. */
enum {
    FFDP_WANT_IMAGE = 1,
    FFDP_WANT_WARP = 2,
    FFDP_WANT_AFFINE = 4,
    FFDP_WANT_TRANSLATION = 8
};

/* ParzenKernel (mi.hpp:28-140). Build with ffdp_parzen_make. */
typedef enum { FFDP_PARZEN_GAUSSIAN = 0, FFDP_PARZEN_BSPLINE3 = 1, FFDP_PARZEN_DELTA = 2 } ffdp_parzen_kind;
typedef struct {
    int32_t kind;
    int32_t bins;
    double sigma;  /* gaussian: sigma in intensity units */
    double radius; /* support half-width in intensity units */
    double norm;   /* gaussian normaliser */
} ffdp_parzen;

/*
 * Moving-image window: planes [z_begin, z_end) of a volume whose full lattice is
 * `dims` (its own normalized frame spans [-1,1]^3). Single-GPU callers pass the whole
 * volume (z_begin 0, z_end dims.nz). Sharded callers pass the resident planes; a sample
 * whose interpolation corner falls inside the volume but outside the window increments
 * *miss (if given) and reads as zero, so the caller can widen the window and repeat
 * (exact).
 * pad = 0: `data` points at plane z_begin of a dense nx*ny*(z_end-z_begin) block.
 * pad = 2: `data` points at a zero-bordered block of (nx+4)*(ny+4)*(z_end-z_begin+4)
 *   floats (ffdp_pad_window), voxel (x,y,z) at ((z-z_begin+2)*(ny+4) + y+2)*(nx+4) + x+2.
 *   The fused step kernels then gather all eight corners without bounds checks: the
 *   border holds the reference's zero padding (sampler.hpp:106-110).
 */
typedef struct {
    const float* data;
    ffdp_dims dims;
    int64_t z_begin, z_end;
    int64_t pad;
} ffdp_image_window;

/*
 * Z-slab of a lattice that is sharded along z (fabric.hpp:31-70). A buffer described
 * by a slab holds global planes [buf_z0, buf_z0 + buf_nz) of a lattice with nz_global
 * planes; compute covers global planes [z_begin, z_end) of it. Single GPU:
 * {0, nz, 0, nz, nz}.
 */
typedef struct {
    int64_t buf_z0, buf_nz;
    int64_t z_begin, z_end;
    int64_t nz_global;
} ffdp_slab;

FFDP_API const char* ffdp_last_error(void);
FFDP_API int ffdp_abi_version(void);
/* Fails with FFDP_CUDA unless an sm_100 device is current. */
FFDP_API int ffdp_device_check(void);
/* The library's stream-ordered scratch lives in its own memory pool per device (not the
 * process's default pool), which keeps up to 4 GiB of freed scratch cached across calls.
 * ffdp_scratch_trim returns all but keep_bytes of that cache to the current device (the
 * drivers call it at the end of each scale / stage). */
FFDP_API int ffdp_scratch_trim(int64_t keep_bytes);

/* ---------------------------------------------------------------------- sampler */

/*
 * fused_sample / fused_sample_accumulate (sampler.hpp:254-276):
 * out[v] (+)= I(A*X_v + t + S*u(X_v)), trilinear, zero padding, no grid materialised.
 * u may be NULL (identity warp; the output lattice is out_dims). accumulate != 0 adds
 * into out. abs_contrib (device double, may be NULL) += sum |value| (RingSampleStats).
 */
FFDP_API int ffdp_sampler_fwd(ffdp_image_window img, const float* u, ffdp_dims out_dims, const ffdp_sampler_args* args,
                     float* out, int accumulate, double* abs_contrib, int32_t* miss, void* stream);

/*
 * fused_sample_backward (sampler.hpp:279-300) / composite_sample_core backward sweep
 * (sampler.hpp:200-239). want: FFDP_WANT_* mask. g_img (image lattice, zeroed by the
 * caller, accumulated with atomics), g_u (3 per output voxel, overwritten), gAt
 * (device double[12] = gA row-major then gt, overwritten; fp64 reduction in a fixed
 * order, deterministic). Outputs not wanted may be NULL.
 */
FFDP_API int ffdp_sampler_bwd(const float* upstream, ffdp_image_window img, const float* u, ffdp_dims out_dims,
                     const ffdp_sampler_args* args, int want, float* g_img, float* g_u, double* gAt,
                     int32_t* miss, void* stream);

/* --------------------------------------------------------------------- smoothing */

/*
 * convolve_axis (smoothing.hpp:52-94): 1-D convolution of a channel-interleaved block
 * along `axis` (0 x, 1 y, 2 z) with host taps (odd count <= 63). mode 0 = zero_pad,
 * 1 = renormalize. lo_global/n_global place the block on the global axis so sharded
 * (halo-padded) blocks match the unsharded result exactly (smoothing.hpp:10-13).
 */
FFDP_API int ffdp_convolve_axis(const float* in, float* out, ffdp_dims dims, int channels, int axis, const double* taps,
                       int ntaps, int mode, int64_t lo_global, int64_t n_global, void* stream);

/*
 * gp_convolve (distops.hpp:54-101; separable_convolve, smoothing.hpp:98-105) of a z-slab:
 * x, y and z passes of the (odd, <= 9) host taps over a 1- or 3-channel field in one
 * z-marching kernel. `in` holds buffer planes [buf_z0, buf_z0 + buf_nz) (buf_dims.nz =
 * buf_nz), which must include the ntaps/2 halo planes on each side that exist in the
 * global lattice (the halo exchange's job, fabric.hpp:315-370); `out` receives planes
 * [z_begin, z_end). mode 0 = zero_pad, 1 = renormalize (EdgeMode, smoothing.hpp:17-23).
 * Taps depend only on global coordinates, so a sharded call equals the unsharded one.
 */
FFDP_API int ffdp_gp_convolve(const float* in, float* out, ffdp_dims buf_dims, ffdp_slab slab, int channels,
                              const double* taps, int ntaps, int mode, void* stream);

/*
 * The gradient half of the warp update (registration.hpp:313-316) fused:
 * g_s = gp_convolve(g_u, taps, renormalize) (g_u buffer planes incl. halo, as `in`
 * above) and adam_step(u, g_s, {m1, m2, step}, lr) (adam.hpp:30-50) on the interior
 * planes of u, m1, m2 (updated in place; the smoothed gradient never reaches HBM).
 * step = the Adam step counter after this update (1 on the first call).
 */
FFDP_API int ffdp_sobolev_adam(const float* g_u, float* u, float* m1, float* m2, ffdp_dims buf_dims, ffdp_slab slab,
                               const double* taps, int ntaps, double lr, double beta1, double beta2, double eps,
                               int64_t step, void* stream);

/* ------------------------------------------------------------------- multi-scale */

/* The lattice resample_scale produces (resample.hpp:52-57): ceil(n * factor) per axis;
 * FFDP_INVALID_ARGUMENT for a non-finite / non-positive factor or a dimension < 2. */
FFDP_API int ffdp_resample_dims(ffdp_dims dims, double factor, ffdp_dims* out);

/*
 * resample_scale (resample.hpp:48-103): for factor < 1 gaussian_smooth(v, 0.5 / factor)
 * (renormalized, factor >= 1/4) then trilinear resampling onto ffdp_resample_dims(dims,
 * factor) keeping the first and last voxel centres. scratch: device float[voxels of
 * dims] for the smoothed volume, or NULL (stream-ordered allocation).
 */
FFDP_API int ffdp_resample_scale(const float* in, ffdp_dims dims, double factor, float* out, float* scratch,
                                 void* stream);

/* resample_warp (resample.hpp:108-146): trilinear on each channel onto out_dims. */
FFDP_API int ffdp_resample_warp(const float* in, ffdp_dims dims, float* out, ffdp_dims out_dims, void* stream);

/* normalize_intensities (registration.hpp:100-115): min-max to [0, 1] (constant -> 0). */
FFDP_API int ffdp_normalize(const float* in, int64_t n, float* out, void* stream);

/* jacobian_positive_fraction (metrics.hpp:145-176) of a warp (lattice >= 3 per axis):
 * the fraction of interior voxels with det(I + du/dx) > 0; synchronises the stream. */
FFDP_API int ffdp_jacobian_positive(const float* u, ffdp_dims dims, double* fraction, void* stream);

/* dist_mse on one slab (distops.hpp:260-282): *sum += sum (moved - fixed)^2 (fp64);
 * grad (may be NULL) = 2 (moved - fixed) / n_total. loss = allreduce(sum) / n_total. */
FFDP_API int ffdp_mse(const float* fixed, const float* moved, int64_t n, int64_t n_total, float* grad, double* sum,
                      void* stream);

/* -------------------------------------------------------------------------- LNCC */

/*
 * lncc_forward_fused (lncc.hpp:144-205) on a z-slab. f, m: buffers described by `slab`
 * (halo planes included). state: 5 channels x interior voxels, channel-major
 * (mean_f, mean_m, mean_ff, mean_mm, mean_fm -- LnccState, lncc.hpp:30-35), fp64 so the
 * cancellation in mean_fm - mean_f*mean_m stays exact-product accurate.
 * ncc_map (interior voxels, may be NULL). sum_n: device double, += sum of n_i over the
 * interior (loss = 1 - allreduce(sum_n)/N_total, distops.hpp:309-318).
 * Moments accumulate in fp64 from exact products.
 */
FFDP_API int ffdp_lncc_fwd(const float* f, const float* m, ffdp_dims buf_dims, ffdp_slab slab, int window, double eps,
                  double* state, float* ncc_map, double* sum_n, void* stream);

/*
 * First half of lncc_backward_fused (lncc.hpp:234-247): rewrites state in place as the
 * gamma family (gamma, gamma_AB, gamma_AC, gamma_FM, gamma_MF) with gi = dL/dn_i
 * (= -upstream/N, lncc.hpp:234; -1/N_total in dist_lncc, distops.hpp:320).
 */
FFDP_API int ffdp_lncc_gamma(double* state, int64_t voxels, double eps, double gi, void* stream);

/*
 * Second half (lncc.hpp:249-278): exact mode (ants == 0) box-filters the gamma family
 * (gamma buffer described by `slab`, halo planes included) before the combination;
 * ANTs mode uses it as is. grad_f may be NULL. f, m, grad_f, grad_m cover the interior.
 */
FFDP_API int ffdp_lncc_combine(const double* gamma, ffdp_dims buf_dims, ffdp_slab slab, int window, int ants,
                      const float* f, const float* m, float* grad_f, float* grad_m, void* stream);

/* lncc_backward_fused (lncc.hpp:226-280) of a whole volume in one call: the gamma family
 * (gi = -upstream / N, lncc.hpp:234) then the combination; `state` (from ffdp_lncc_fwd
 * over the whole volume) is consumed, as the reference rewrites LnccState in place. */
FFDP_API int ffdp_lncc_bwd(double upstream, double* state, const float* f, const float* m, ffdp_dims dims,
                           int window, double eps, int ants, float* grad_f, float* grad_m, void* stream);

/* lncc_forward_fused + lncc_backward_fused of a whole volume in one call (the survey's
 * ffdp_lncc_fwdbwd): *sum_n (device) += the sum of n_i (loss = 1 - sum_n / N), grad_m
 * (and grad_f if non-NULL) = d(upstream * loss) / dM; state = 5 * N doubles of workspace. */
FFDP_API int ffdp_lncc_fwdbwd(const float* f, const float* m, ffdp_dims dims, int window, double eps, int ants,
                              double upstream, double* state, double* sum_n, float* grad_f, float* grad_m,
                              void* stream);

/* ---------------------------------------------------------------------------- MI */

/* ParzenKernel::gaussian/bspline3/delta (mi.hpp:33-63) incl. the normalisation check
 * (mi.hpp:120-133, FFDP_LOGIC on failure). Host-only. */
FFDP_API int ffdp_parzen_make(int kind, int bins, double sigma_bins, ffdp_parzen* out);

/*
 * mi_forward_exact (mi.hpp:235-272) / mi_forward_approx (mi.hpp:285-354) histogram
 * accumulation. raw: device double[B*B + 2B] (raw_joint, raw_marg_i, raw_marg_j),
 * ACCUMULATED (zero it first). Accumulation is order-independent fixed point
 * (2^-24 per contribution), so results are deterministic. bad_input (device int32,
 * may be NULL) is set when an intensity lies outside [0,1] (mi.hpp:170-179).
 * stats (host uint64[2], may be NULL) += the MiStats counters (mi.hpp:156-159).
 */
FFDP_API int ffdp_mi_hist(const float* vi, const float* vj, int64_t n, const ffdp_parzen* kernel, int approx, double* raw,
                 int32_t* bad_input, uint64_t* stats, void* stream);

/*
 * finalize_histogram + histogram_mi + the ghat table of mi_backward_impl
 * (mi.hpp:181-209, 369-390). table (device double[2*B*B + 2B + 4]):
 *   p_ij[B*B], p_i[B], p_j[B], ghat[B*B], {z, mi, dot, 0}. upstream = dL/dMI.
 */
FFDP_API int ffdp_mi_finalize(const double* raw, int bins, double upstream, double* table, void* stream);

/* Per-voxel part of mi_backward_impl (mi.hpp:392-421). grad_i may be NULL. */
FFDP_API int ffdp_mi_bwd(const float* vi, const float* vj, int64_t n, const ffdp_parzen* kernel, const double* table,
                float* grad_i, float* grad_j, void* stream);

/* ------------------------------------------------------------- fused step (★) */

/*
 * The deformable step's hot path (registration.hpp:277-312) for LNCC in ANTs mode, in one
 * streaming pass: Mw = fused_sample(M, u) for the slab + 3 halo planes, the five LNCC
 * window moments (lncc_forward_fused, lncc.hpp:144-205), dL/dMw (lncc_backward_fused with
 * ants_approx, lncc.hpp:226-280) and g_u = fused_sample_backward(dL/dMw, want warp)
 * (sampler.hpp:221-230); only g_u is written.
 *   f, u: buffers described by `slab` (halo planes of radius window/2 included);
 *   g_u: interior planes only (3 floats per voxel);
 *   args: the sampler arguments of the GLOBAL output lattice (buf_dims.nx, buf_dims.ny,
 *     slab.nz_global); voxels are addressed by global lattice index, which is the
 *     ring sampler's per-shard rescale (distops.hpp:120-133) folded into one frame;
 *   gi: dL/dn_i (-1/N_total for the deformable step);
 *   ranges: device float[4] {F min, F max, M min, M max}: the value ranges of the fixed
 *     and moving volumes (ffdp_minmax; allreduced over the shards when sharded, so every
 *     rank uses the same intensity frame). They bound the exact fixed-point moment sums;
 *     values outside them are an error the kernel does not detect. NULL: computed here on
 *     every call (one extra read of F and of the moving window);
 *   sum_n: device double, += sum of n_i over the slab interior (fixed order: the loss is
 *     bit-reproducible);
 *   workspace: device buffer of ffdp_step_lncc_workspace_bytes bytes, or NULL for a
 *     stream-ordered allocation per call (pass one to capture the step in a CUDA graph).
 */
FFDP_API int ffdp_step_lncc(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab, ffdp_image_window m,
                   const ffdp_sampler_args* args, int window, double eps, double gi, const float* ranges,
                   float* g_u, double* sum_n, int32_t* miss, void* workspace, void* stream);

/* Bytes of the LNCC step workspace: 4 floats of ranges, one double per CTA. */
FFDP_API int64_t ffdp_step_lncc_workspace_bytes(ffdp_dims buf_dims, ffdp_slab slab);

/*
 * The round-1 two-pass form of the same step, kept for comparison (bench.py
 * --lncc-impl twopass): pass 1 warps every voxel once into an HBM workspace (Mw, dMw/du),
 * pass 2 runs the moments from it (moments in fp32 / fp64 around the intensity shifts
 * shift_f, shift_m). passes = 1, 2 or 3 (both). workspace:
 * ffdp_step_lncc_passes_workspace_bytes (required).
 */
FFDP_API int ffdp_step_lncc_passes(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab,
                                   ffdp_image_window m, const ffdp_sampler_args* args, int window, double eps,
                                   double gi, float shift_f, float shift_m, float* g_u, double* sum_n, int32_t* miss,
                                   void* workspace, int passes, void* stream);
FFDP_API int64_t ffdp_step_lncc_passes_workspace_bytes(ffdp_dims buf_dims, ffdp_slab slab);

/*
 * Fused MI step, pass 1 (registration.hpp:278-299 with dist_mi, distops.hpp:355-373):
 * samples Mw and accumulates the joint Parzen histogram of (f, Mw) into raw
 * (device double[B*B + 2B]). When nx % 4 == 0 only the joint is accumulated (the
 * marginal entries are left untouched): finalize_histogram derives p_i, p_j from the
 * joint (mi.hpp:181-196), so the raw marginals are payload only (distops.hpp:366-372). Then allreduce raw
 * (if sharded), ffdp_mi_finalize(raw, B, -1, table), and pass 2. f, u as for
 * ffdp_step_lncc (halo planes allowed, not needed); interior planes are processed.
 * workspace: device scratch of ffdp_step_mi_workspace_bytes(B) bytes, or NULL for a
 * stream-ordered allocation per call (pass one to capture the step in a CUDA graph).
 */
FFDP_API int ffdp_step_mi_hist(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab, ffdp_image_window m,
                      const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, void* workspace,
                      int32_t* miss, void* stream);

/* Bytes of device scratch the MI step passes need for `bins` bins. */
FFDP_API int64_t ffdp_step_mi_workspace_bytes(int bins);

/*
 * The whole single-GPU MI step in one call (pass 1, finalize with upstream -1 -- the
 * loss is -MI, distops.hpp:391-392 -- and pass 2). raw (B*B + 2B doubles) is zeroed
 * here; table as ffdp_mi_finalize (the loss is -table[2B^2 + 2B + 1]). rec: device
 * buffer of ffdp_step_mi_record_bytes, or NULL; with it (B-spline kernel, zero-bordered
 * window) pass 1 writes the per-voxel records and pass 2 streams them
 * (ffdp_step_mi_hist_rec / ffdp_step_mi_grad_rec) instead of sampling the warp again.
 * Launch-only (no host synchronisation), so it can be captured in a CUDA graph.
 */
FFDP_API int ffdp_step_mi(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab, ffdp_image_window m,
                 const ffdp_sampler_args* args, const ffdp_parzen* kernel, double* raw, double* table, float* g_u,
                 void* workspace, float* rec, int32_t* miss, void* stream);

/* Bytes of the pass-1 records of a slab interior: 4 floats per voxel. */
FFDP_API int64_t ffdp_step_mi_record_bytes(ffdp_dims buf_dims, ffdp_slab slab);

/*
 * Pass 1 as ffdp_step_mi_hist, additionally writing per interior voxel the record
 * {Mw, S_a (N_a - 1)/2 * dMw/dfrac_a (a = x, y, z)} (16 B) into rec (voxel order of the
 * interior). B-spline kernel and a zero-bordered window (pad = 2) only.
 */
FFDP_API int ffdp_step_mi_hist_rec(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab,
                                   ffdp_image_window m, const ffdp_sampler_args* args, const ffdp_parzen* kernel,
                                   double* raw, void* workspace, float* rec, int32_t* miss, void* stream);

/*
 * Single-rank pass 1 with the finalize fused in: ffdp_step_mi_hist_rec, then the last
 * CTA to finish converts the histogram into raw (joint entries overwritten; the caller
 * zeroes the marginal entries) and runs ffdp_mi_finalize(raw, B, upstream, table)
 * (mi.hpp:181-209, 369-390). workspace (ffdp_step_mi_workspace_bytes(B)) is required: it
 * holds the fixed-point histogram and the CTA completion counter. For a sharded step use
 * ffdp_step_mi_hist_rec + allreduce + ffdp_mi_finalize instead.
 */
FFDP_API int ffdp_step_mi_hist_final(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab,
                                     ffdp_image_window m, const ffdp_sampler_args* args, const ffdp_parzen* kernel,
                                     double* raw, double upstream, double* table, void* workspace, float* rec,
                                     int32_t* miss, void* stream);

/*
 * Pass 2 from the records: dL/dMw = sum_m kappa_i[m] sum_n ghat[m][n] omega_j[n]
 * (mi.hpp:392-421) with i = F, j = Mw, and g_u = record.xyz-part * dL/dMw
 * (sampler.hpp:221-230). Streams F and the records; no warp sampling.
 */
FFDP_API int ffdp_step_mi_grad_rec(const float* f, ffdp_dims buf_dims, ffdp_slab slab, const ffdp_parzen* kernel,
                                   const double* table, const float* rec, float* g_u, void* stream);

/* Pass 2: re-samples Mw, dL/dMw from the ghat table (mi.hpp:392-421), g_u (3N). */
FFDP_API int ffdp_step_mi_grad(const float* f, const float* u, ffdp_dims buf_dims, ffdp_slab slab, ffdp_image_window m,
                      const ffdp_sampler_args* args, const ffdp_parzen* kernel, const double* table, float* g_u,
                      int32_t* miss, void* stream);

/* ----------------------------------------------------------------- utilities */

/* Sum of `n` doubles into *out (device), fixed order (deterministic). */
FFDP_API int ffdp_reduce_sum_f64(const double* in, int64_t n, double* out, void* stream);

/* Copies planes [z_begin, z_end) of a dense volume (src points at plane z_begin) into
 * the zero-bordered pad = 2 layout of ffdp_image_window (dst sized
 * (nx+4)*(ny+4)*(z_end-z_begin+4), border written as zero). */
FFDP_API int ffdp_pad_window(const float* src, ffdp_dims dims, int64_t z_begin, int64_t z_end, float* dst,
                             void* stream);

/* Min and max of a float array into out[2] (device float), for intensity ranges. */
FFDP_API int ffdp_minmax(const float* in, int64_t n, float* out, void* stream);

/*
 * z-extent of the moving planes a sampler pass over `out_dims` needs
 * (ring-sampler plan, distops.hpp:144-168): out[0] = min, out[1] = max global plane
 * index of any interpolation corner that lies inside the moving volume (device int64[2];
 * out[0] > out[1] when none). Reads u once.
 */
FFDP_API int ffdp_sampler_z_extent(const float* u, ffdp_dims out_dims, ffdp_dims m_dims, const ffdp_sampler_args* args,
                          int64_t* out, void* stream);

/* ----------------------------------------------------------- sharded context */
/*
 * One process drives `world` ranks (WorkerGroup(H), fabric.hpp:266-300): rank r is a z
 * slab on devices[r] (devices may repeat; NULL = rank r on device r mod count) with its
 * own stream; exchanges are peer copies (NVLink / NVSwitch between B200s). Collectives
 * take arrays of `world` per-rank device pointers (rank r's on devices[r]) and run all
 * ranks in lock step; they return when every rank's results are complete. Slabs follow
 * shard_ranges (fabric.hpp:44-70) of the global z extent. Reductions are rank-ordered
 * (fabric.hpp:246-263): deterministic for a given world size.
 */
typedef struct ffdp_comm_s* ffdp_comm;
FFDP_API int ffdp_comm_create(int world, const int* devices, ffdp_comm* out);
FFDP_API int ffdp_comm_destroy(ffdp_comm comm);
FFDP_API int ffdp_comm_world(ffdp_comm comm);
FFDP_API int ffdp_comm_device(ffdp_comm comm, int rank);
/* shard_ranges (fabric.hpp:44-57): planes [lo, hi) of `rank` among `world` for n planes */
FFDP_API int ffdp_shard_range(int64_t n, int world, int rank, int64_t* lo, int64_t* hi);
/* halo_exchange (fabric.hpp:315-370): out[r] = [lo_r planes of rank r-1 | slab r | hi_r
 * planes of rank r+1], lo_r = pad except on rank 0, hi_r = pad except on the last rank;
 * `channels` floats per voxel. FFDP_INVALID_ARGUMENT when pad exceeds a neighbour's
 * thickness (fabric.hpp:321-326). */
FFDP_API int ffdp_halo_exchange(ffdp_comm comm, const float* const* slabs, ffdp_dims global, int channels, int pad,
                                float* const* out, int64_t* lo_out, int64_t* hi_out);
/* gp_convolve (distops.hpp:54-101): the separable convolution of a z-sharded volume /
 * warp (ffdp_gp_convolve semantics per rank) with the neighbours' halo planes (sync), or
 * of each shard as a standalone volume along z (sync = 0, the ablation). */
FFDP_API int ffdp_dist_gp_convolve(ffdp_comm comm, const float* const* slabs, ffdp_dims global, int channels,
                                   const double* taps, int ntaps, int mode, int sync, float* const* out);
/* ring_sample (distops.hpp:144-168): the moved image on each rank's output slab of
 * `out_global`, from the z-sharded moving image of `m_global` (u_shards interleaved xyz on
 * the output slabs; A row-major 9, t 3, NULL = identity). Each rank gathers exactly the
 * moving planes its samples touch (ffdp_sampler_z_extent) from their owners. */
FFDP_API int ffdp_ring_sample(ffdp_comm comm, const float* const* m_shards, ffdp_dims m_global,
                              const float* const* u_shards, ffdp_dims out_global, const double* A, const double* t,
                              float* const* out);
/* ring_sample_backward (distops.hpp:179-248): `want` as ffdp_sampler_bwd; g_img[r] is
 * rank r's moving shard (every rank's contributions routed to the owners, added in rank
 * order), g_u[r] its warp slab, gAt (host, 12 doubles: dA row-major, dt) summed over ranks. */
FFDP_API int ffdp_ring_sample_bwd(ffdp_comm comm, const float* const* upstream, const float* const* m_shards,
                                  ffdp_dims m_global, const float* const* u_shards, ffdp_dims out_global,
                                  const double* A, const double* t, int want, float* const* g_img, float* const* g_u,
                                  double* gAt);
/* dist_mse (distops.hpp:260-282): *loss = sum over ranks of (F - M)^2 / n_total; grad = 2 (M - F) / n_total. */
FFDP_API int ffdp_dist_mse(ffdp_comm comm, const float* const* f, const float* const* moved, ffdp_dims global,
                           int64_t n_total, double* loss, float* const* grad);
/* dist_mi (distops.hpp:355-396): local raw histograms, rank-ordered sum (the B*B + 2B
 * payload, reported in *payload_elements), finalize, *loss = -MI, grad = dL/dmoved per rank. */
FFDP_API int ffdp_dist_mi(ffdp_comm comm, const float* const* f, const float* const* moved, ffdp_dims global,
                          const ffdp_parzen* kernel, int approx_forward, int64_t n_total, double* loss,
                          float* const* grad, int64_t* payload_elements);
/* dist_lncc (distops.hpp:285-352): window moments with r-plane halos (2r for the exact
 * backward; none with gp_sync = 0, the ablation), sum of n allreduced, *loss = 1 - sum / N,
 * grad = dL/dmoved (upstream 1, gi = -1/N). n_total <= 0: the global voxel count. */
FFDP_API int ffdp_dist_lncc(ffdp_comm comm, const float* const* f, const float* const* moved, ffdp_dims global,
                            int window, double eps, int ants_approx, int gp_sync, int64_t n_total, double* loss,
                            float* const* grad);

/* The fused deformable step over the ranks (ring_sample -> dist_lncc (ANTs) / dist_mi ->
 * ring_sample_backward(warp), registration.hpp:277-312): per rank F and u with the
 * window radius of halo planes (LNCC), the exact moving window of its samples, the
 * single-GPU step kernels on the slab (ffdp_step_lncc / ffdp_step_mi_hist[_rec] +
 * ffdp_step_mi_grad[_rec]), rank-ordered sums of sum_n / the joint histogram.
 * loss_kind 0 = LNCC (window, eps; moment shifts = the global mid-ranges of F and M),
 * 1 = MI (kernel); *loss as the single-GPU step; g_u[r] = dL/du on rank r's slab. */
FFDP_API int ffdp_dist_step(ffdp_comm comm, int loss_kind, const float* const* f, const float* const* m,
                            const float* const* u, ffdp_dims global, const double* A, const double* t, int window,
                            double eps, const ffdp_parzen* kernel, double* loss, float* const* g_u);


/* ------------------------------------------------ native sharded step plan (plan.cu) */
/*
 * The sharded deformable step as a persistent per-rank object (one per GPU), for C / C++
 * hosts that run one process (or one thread) per rank: the reference's per-iteration
 * sequence under WorkerGroup(H) (registration.hpp:266-312: ring_sample -> dist_lncc /
 * dist_mi -> ring_sample_backward(warp), distops.hpp:144-396) over z slabs by
 * shard_ranges (fabric.hpp:44-70), with halo_exchange (fabric.hpp:315-370) and
 * allreduce_sum (fabric.hpp:246-263) as NCCL point-to-point / allreduce calls (or peer
 * copies inside one process).
 *
 * Transport ("group"): ffdp_group_nccl -- one rank of an NCCL communicator (every rank
 * passes the same FFDP_NCCL_ID_BYTES-byte id from ffdp_nccl_unique_id; NCCL is loaded at
 * run time, libnccl.so.2 or $FFDP_NCCL_LIB); ffdp_group_local -- `world` ranks inside one
 * process (out[world] handles; devices may repeat), each driven by its own host thread.
 * Every plan call below is collective over the group: all ranks call it in the same order.
 */
#define FFDP_NCCL_ID_BYTES 128
typedef struct ffdp_group_s* ffdp_group;
typedef struct ffdp_plan_s* ffdp_plan;
FFDP_API int ffdp_nccl_version(int* version);
FFDP_API int ffdp_nccl_unique_id(unsigned char* id /* FFDP_NCCL_ID_BYTES */);
FFDP_API int ffdp_group_nccl(const unsigned char* id, int world, int rank, int device, ffdp_group* out);
FFDP_API int ffdp_group_local(int world, const int* devices, ffdp_group* out /* world handles */);
FFDP_API int ffdp_group_destroy(ffdp_group g);
FFDP_API int ffdp_group_info(ffdp_group g, int* world, int* rank, int* device);

typedef struct {
    int32_t loss_kind;     /* 0 = LNCC (ANTs, window 7), 1 = Mattes MI (B-spline Parzen) */
    int32_t window;        /* LNCC window (7) */
    double eps;            /* LNCC epsilon */
    ffdp_parzen kernel;    /* MI kernel (ffdp_parzen_make) */
    double A[9], t[3];     /* affine of the stage (row-major, normalized coordinates) */
    int32_t margin_planes; /* moving-window margin beyond the affine's z reach */
    int32_t records;       /* MI: 1 = pass-1 records when they fit (+16 B/voxel), 0 = pass 2 re-samples */
    int32_t overlap;       /* LNCC: 1 = u halo exchange overlapped with the interior planes */
    int32_t warp_halo;     /* > 0: the plan also runs the warp update (ffdp_plan_warp_update) with taps of
                              radius <= warp_halo (3 for the default sigmas 1.0 / 0.5); 0: step only */
} ffdp_plan_params;

/* Creates rank g's plan for a `global` lattice (slab = shard_ranges(nz, world, rank)). */
FFDP_API int ffdp_plan_create(ffdp_group g, ffdp_dims global, const ffdp_plan_params* params, ffdp_plan* out);
FFDP_API int ffdp_plan_destroy(ffdp_plan p);
FFDP_API int ffdp_plan_slab(ffdp_plan p, int64_t* lo, int64_t* hi);
/* The plan's compute stream, and its device buffers: u (the slab's interior planes of the
 * persistent haloed displacement buffer, 3 floats per voxel -- the caller or its optimiser
 * writes it on the plan's stream; the halo planes are the plan's) and g_u (interior). */
FFDP_API void* ffdp_plan_stream(ffdp_plan p);
FFDP_API float* ffdp_plan_u(ffdp_plan p);
FFDP_API float* ffdp_plan_g_u(ffdp_plan p);
/* Moving planes [z0, z1) resident on this rank, and how many window fetches this scale. */
FFDP_API int ffdp_plan_window(ffdp_plan p, int64_t* z0, int64_t* z1, int64_t* fetches);
/* Once per scale (collective, synchronous): the rank's F and M slabs (device or host
 * pointers, slab planes only) -> F halo planes, the intensity frame (LNCC), the moving
 * window from the owners of its planes. */
FFDP_API int ffdp_plan_load(ffdp_plan p, const float* f_slab, const float* m_slab);
/* One step (collective): g_u = dL/du on the slab, loss = the global loss. sync = 1: waits,
 * repeats the step with widened windows after a window miss on any rank (exact), and
 * writes *loss. sync = 0: launch only (no host synchronisation; the misses accumulate and
 * ffdp_plan_result reports them -- a non-zero count means the unchecked steps must be
 * redone with sync = 1). */
FFDP_API int ffdp_plan_step(ffdp_plan p, int sync, double* loss);
/* The warp update of the iteration on the plan's slab (registration.hpp:313-317, collective):
 * the halo planes of g_u exchanged, gp_convolve(g_u, taps_grad, renormalize) fused with
 * adam_step on u (ffdp_sobolev_adam; beta 0.9 / 0.999, eps 1e-8, the plan holds the moments and
 * the step counter, reset by ffdp_plan_load), the halo planes of u exchanged, u =
 * gp_convolve(u, taps_warp, renormalize). Odd tap counts of radius <= warp_halo (host doubles,
 * gaussian_taps). Afterwards ffdp_plan_u points at the smoothed field (re-query it). */
FFDP_API int ffdp_plan_warp_update(ffdp_plan p, double lr_norm, const double* taps_grad, int ntaps_grad,
                                   const double* taps_warp, int ntaps_warp);
/* Waits for the last step; its loss and the summed window misses over all ranks. */
FFDP_API int ffdp_plan_result(ffdp_plan p, double* loss, double* misses);

#ifdef __cplusplus
}
#endif

#endif /* FFDP_H */
