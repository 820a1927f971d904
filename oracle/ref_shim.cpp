// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers (voxreg, included
// read-only from /root/reference/proj/include at build time; nothing is copied).
// Built by oracle/Makefile into oracle/_ref/libvoxreg_ref.so. It is used (a) to
// generate the golden vectors under tests/golden/ that pin oracle/ffdp_oracle.c and
// (b) as bench.py's CPU baseline ("kind": "reference"): the reference's own
// deformable-step sequence ring_sample -> dist_lncc|dist_mi -> ring_sample_backward
// (registration.hpp:277-312) under WorkerGroup(H).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "voxreg/distops.hpp"
#include "voxreg/fabric.hpp"
#include "voxreg/lncc.hpp"
#include "voxreg/metrics.hpp"
#include "voxreg/mi.hpp"
#include "voxreg/registration.hpp"
#include "voxreg/sampler.hpp"
#include "voxreg/synth.hpp"

using namespace voxreg;

namespace {

thread_local char g_err[512];

int fail(const std::exception& e, int code) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return code;
}

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::logic_error& e) {
        return fail(e, 3);
    } catch (const std::runtime_error& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

Dims3 D(const int64_t* d) { return Dims3{d[0], d[1], d[2]}; }

template <typename T>
Volume3<T> vol(const double* p, Dims3 d) {
    auto v = Volume3<T>::zeros(d);
    for (std::size_t i = 0; i < v.data.size(); ++i) v.data[i] = static_cast<T>(p[i]);
    return v;
}

template <typename T>
WarpField<T> warp(const double* p, Dims3 d) {
    auto w = WarpField<T>::zeros(d);
    for (std::size_t i = 0; i < w.data.size(); ++i) w.data[i] = static_cast<T>(p[i]);
    return w;
}

template <typename C>
void put(const C& src, double* dst) {
    for (std::size_t i = 0; i < src.size(); ++i) dst[i] = static_cast<double>(src[i]);
}

SamplerArgs sargs(const double* A, const double* t, const double* S, const double* bounds) {
    SamplerArgs a;
    for (int i = 0; i < 9; ++i) a.A.m[static_cast<std::size_t>(i)] = A[i];
    for (int i = 0; i < 3; ++i) {
        a.t[i] = t[i];
        a.S[i] = S[i];
        a.bounds.x_min[i] = bounds[i];
        a.bounds.x_max[i] = bounds[3 + i];
    }
    return a;
}

ParzenKernel kernel(int kind, int bins, double sigma_bins) {
    if (kind == 0) return ParzenKernel::gaussian(bins, sigma_bins);
    if (kind == 1) return ParzenKernel::bspline3(bins);
    return ParzenKernel::delta(bins);
}

// One deformable-step evaluation (registration.hpp:277-312), sharded over H
// std::thread ranks. Writes the gathered g_u (3N) and returns the loss.
template <typename T>
double step_impl(int loss_kind, const double* f, const double* m, const double* u, Dims3 d, const double* A,
                 const double* t, int window, double eps, int ants, int bins, int mi_kind, int approx,
                 int world, double* g_u_out, double* moved_out) {
    const auto fv = vol<T>(f, d), mv = vol<T>(m, d);
    const auto uv = warp<T>(u, d);
    Mat3 Am;
    for (int i = 0; i < 9; ++i) Am.m[static_cast<std::size_t>(i)] = A[i];
    const Vec3 tv{t[0], t[1], t[2]};
    std::vector<WarpField<T>> gu(static_cast<std::size_t>(world));
    std::vector<Volume3<T>> moved(static_cast<std::size_t>(world));
    double loss_out = 0;
    WorkerGroup group(world, std::chrono::milliseconds(600000));
    group.run([&](WorkerContext& ctx) {
        const auto spec = make_shard_spec(d, world, ctx.rank());
        const auto f_slab = extract_slab(fv, spec);
        const auto m_slab = extract_slab(mv, spec);
        const auto u_slab = extract_slab(uv, spec);
        auto mw = ring_sample(ctx, m_slab, u_slab, Am, tv, d, spec);
        DistLoss<T> loss;
        if (loss_kind == 0)
            loss = dist_lncc(ctx, spec, f_slab, mw, window, eps, ants != 0, true, d.voxels());
        else
            loss = dist_mi(ctx, f_slab, mw, bins, kernel(mi_kind, bins, 0.5), approx != 0, d.voxels());
        auto g = ring_sample_backward(ctx, loss.grad_moved, m_slab, u_slab, Am, tv, d, spec,
                                      SamplerGradWant{false, true, false, false});
        if (ctx.rank() == 0) loss_out = loss.loss;
        gu[static_cast<std::size_t>(ctx.rank())] = std::move(*g.warp);
        moved[static_cast<std::size_t>(ctx.rank())] = std::move(mw);
    });
    if (g_u_out) put(gather_warp(gu, d).data, g_u_out);
    if (moved_out) put(gather_volume(moved, d).data, moved_out);
    return loss_out;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

// fused_sample / fused_sample_backward (sampler.hpp:254-300); outputs may be NULL.
int ref_sample(const double* img, const int64_t* idims, const double* u, const int64_t* odims, const double* A,
               const double* t, const double* S, const double* bounds, double* out, const double* up,
               double* g_img, double* g_u, double* gA, double* gt) {
    return guarded([&] {
        const auto iv = vol<double>(img, D(idims));
        WarpField<double> w;
        if (u) w = warp<double>(u, D(odims));
        const auto a = sargs(A, t, S, bounds);
        if (out) put(fused_sample(iv, u ? &w : nullptr, a).data, out);
        if (up) {
            const auto upv = vol<double>(up, u ? D(odims) : D(idims));
            auto g = fused_sample_backward(upv, iv, u ? &w : nullptr, a,
                                           SamplerGradWant{g_img != nullptr, g_u != nullptr, gA != nullptr,
                                                           gt != nullptr});
            if (g_img) put(g.image->data, g_img);
            if (g_u) put(g.warp->data, g_u);
            if (gA) std::memcpy(gA, g.affine->m.data(), 9 * sizeof(double));
            if (gt) std::memcpy(gt, g.translation->data(), 3 * sizeof(double));
        }
    });
}

// lncc_forward_fused (lncc.hpp:144) + lncc_backward_fused (lncc.hpp:226).
int ref_lncc(const double* f, const double* m, const int64_t* dims, int window, double eps, int ants,
             double upstream, double* loss, double* state5, double* map, double* grad_f, double* grad_m) {
    return guarded([&] {
        const auto fv = vol<double>(f, D(dims)), mv = vol<double>(m, D(dims));
        auto [res, st] = lncc_forward_fused(fv, mv, window, eps, map != nullptr);
        *loss = res.loss;
        const std::size_t n = fv.data.size();
        if (state5) {
            put(st.mean_f.data, state5);
            put(st.mean_m.data, state5 + n);
            put(st.mean_ff.data, state5 + 2 * n);
            put(st.mean_mm.data, state5 + 3 * n);
            put(st.mean_fm.data, state5 + 4 * n);
        }
        if (map) put(res.ncc_map.data, map);
        if (grad_m) {
            auto [gf, gm] = lncc_backward_fused(upstream, st, fv, mv, ants != 0);
            if (grad_f) put(gf.data, grad_f);
            put(gm.data, grad_m);
        }
    });
}

// mi_forward_exact|approx (mi.hpp:235,285) + mi_backward (mi.hpp:430).
// raw: B^2 + 2B (raw_joint, raw_marg_i, raw_marg_j); pij: B^2 + 2B (p_ij, p_i, p_j).
int ref_mi(const double* vi, const double* vj, const int64_t* dims, int bins, int kind, double sigma_bins,
           int approx, double upstream, double* mi, double* raw, double* pij, uint64_t* stats, double* grad_i,
           double* grad_j) {
    return guarded([&] {
        const auto iv = vol<double>(vi, D(dims)), jv = vol<double>(vj, D(dims));
        const auto k = kernel(kind, bins, sigma_bins);
        MiResult r = approx ? mi_forward_approx(iv, jv, bins, k) : mi_forward_exact(iv, jv, bins, k);
        *mi = r.mi;
        const std::size_t b2 = static_cast<std::size_t>(bins) * static_cast<std::size_t>(bins);
        if (raw) {
            put(r.hist.raw_joint, raw);
            put(r.hist.raw_marg_i, raw + b2);
            put(r.hist.raw_marg_j, raw + b2 + static_cast<std::size_t>(bins));
        }
        if (pij) {
            put(r.hist.p_ij, pij);
            put(r.hist.p_i, pij + b2);
            put(r.hist.p_j, pij + b2 + static_cast<std::size_t>(bins));
        }
        if (stats) {
            stats[0] = r.stats.hist_writes;
            stats[1] = r.stats.kernel_evals;
        }
        if (grad_j) {
            auto [gi, gj] = mi_backward(upstream, iv, jv, r.hist, k);
            if (grad_i) put(gi.data, grad_i);
            put(gj.data, grad_j);
        }
    });
}

// Kernel evaluation and the constructor's normalisation check (mi.hpp:33-133).
int ref_parzen_eval(int kind, int bins, double sigma_bins, const double* x, int64_t n, double* kappa,
                    double* omega) {
    return guarded([&] {
        const auto k = kernel(kind, bins, sigma_bins);
        for (int64_t i = 0; i < n; ++i) {
            kappa[i] = k.kappa(x[i]);
            omega[i] = k.omega(x[i]);
        }
    });
}

// synth_pair (synth.hpp:116-137): fixed, moving (N) and the ground-truth warp (3N).
int ref_synth_pair(uint64_t seed, const int64_t* dims, int k, double max_disp, double* fixed, double* moving,
                   double* true_warp) {
    return guarded([&] {
        auto p = synth_pair(seed, D(dims), k, max_disp);
        put(p.fixed.data, fixed);
        put(p.moving.data, moving);
        put(p.true_warp.data, true_warp);
    });
}

// The label maps and the pre-blur image of synth_pair (synth.hpp:116-135).
int ref_synth_labels(uint64_t seed, const int64_t* dims, int k, double max_disp, uint16_t* labels_fixed,
                     uint16_t* labels_moving, double* pre_blur) {
    return guarded([&] {
        auto p = synth_pair(seed, D(dims), k, max_disp);
        std::memcpy(labels_fixed, p.labels_fixed.data.data(), p.labels_fixed.data.size() * sizeof(uint16_t));
        std::memcpy(labels_moving, p.labels_moving.data.data(), p.labels_moving.data.size() * sizeof(uint16_t));
        put(p.pre_blur_fixed.data, pre_blur);
    });
}

// gp_convolve (distops.hpp:84-101) of a whole volume sharded over H ranks, gathered.
int ref_gp_convolve(const double* v, const int64_t* dims, int channels, const double* taps, int ntaps,
                    int renormalize, int sync, int world, double* out) {
    return guarded([&] {
        const Dims3 d = D(dims);
        std::vector<double> tp(taps, taps + ntaps);
        const EdgeMode mode = renormalize ? EdgeMode::renormalize : EdgeMode::zero_pad;
        WorkerGroup group(world);
        if (channels == 1) {
            const auto vv = vol<double>(v, d);
            std::vector<Volume3<double>> res(static_cast<std::size_t>(world));
            group.run([&](WorkerContext& ctx) {
                const auto spec = make_shard_spec(d, world, ctx.rank());
                res[static_cast<std::size_t>(ctx.rank())] = gp_convolve(ctx, extract_slab(vv, spec), tp, spec, mode,
                                                                        sync != 0);
            });
            put(gather_volume(res, d).data, out);
        } else {
            const auto wv = warp<double>(v, d);
            std::vector<WarpField<double>> res(static_cast<std::size_t>(world));
            group.run([&](WorkerContext& ctx) {
                const auto spec = make_shard_spec(d, world, ctx.rank());
                res[static_cast<std::size_t>(ctx.rank())] = gp_convolve(ctx, extract_slab(wv, spec), tp, spec, mode,
                                                                        sync != 0);
            });
            put(gather_warp(res, d).data, out);
        }
    });
}

// The warp update of the deformable loop over H ranks (registration.hpp:313-317):
// gp_convolve(g_u, gaussian_taps(sigma_grad), renormalize) -> adam_step -> gp_convolve(u,
// gaussian_taps(sigma_warp), renormalize); `step` = the Adam step counter after this call.
int ref_warp_update(const double* g_u, double* u, double* m1, double* m2, const int64_t* dims, double sigma_grad,
                    double sigma_warp, double lr, int64_t step, int world) {
    return guarded([&] {
        const Dims3 d = D(dims);
        const auto gw = warp<double>(g_u, d);
        const auto uw = warp<double>(u, d);
        const auto w1 = warp<double>(m1, d);
        const auto w2 = warp<double>(m2, d);
        const auto taps_grad = gaussian_taps(sigma_grad);
        const auto taps_warp = gaussian_taps(sigma_warp);
        std::vector<WarpField<double>> ru(static_cast<std::size_t>(world)), r1(ru.size()), r2(ru.size());
        WorkerGroup group(world);
        group.run([&](WorkerContext& ctx) {
            const auto spec = make_shard_spec(d, world, ctx.rank());
            auto u_slab = extract_slab(uw, spec);
            auto adam = AdamState<double>::zeros(u_slab.data.size());
            const auto s1 = extract_slab(w1, spec), s2 = extract_slab(w2, spec);
            std::copy(s1.data.begin(), s1.data.end(), adam.m1.begin());
            std::copy(s2.data.begin(), s2.data.end(), adam.m2.begin());
            adam.step = step - 1;
            auto g = gp_convolve(ctx, extract_slab(gw, spec), taps_grad, spec, EdgeMode::renormalize, true);
            adam_step<double>(u_slab.data, g.data, adam, lr);
            u_slab = gp_convolve(ctx, u_slab, taps_warp, spec, EdgeMode::renormalize, true);
            const auto k = static_cast<std::size_t>(ctx.rank());
            ru[k] = std::move(u_slab);
            r1[k] = WarpField<double>::zeros(s1.dims);
            r2[k] = WarpField<double>::zeros(s2.dims);
            std::copy(adam.m1.begin(), adam.m1.end(), r1[k].data.begin());
            std::copy(adam.m2.begin(), adam.m2.end(), r2[k].data.begin());
        });
        put(gather_warp(ru, d).data, u);
        put(gather_warp(r1, d).data, m1);
        put(gather_warp(r2, d).data, m2);
    });
}

// resample_scale (resample.hpp:48-103) and resample_warp (108-146).
int ref_resample_scale(const double* v, const int64_t* dims, double factor, double* out, int64_t* out_dims) {
    return guarded([&] {
        const auto r = resample_scale(vol<double>(v, D(dims)), factor);
        out_dims[0] = r.dims.nx;
        out_dims[1] = r.dims.ny;
        out_dims[2] = r.dims.nz;
        if (out) put(r.data, out);
    });
}

int ref_resample_warp(const double* w, const int64_t* dims, const int64_t* out_dims, double* out) {
    return guarded([&] { put(resample_warp(warp<double>(w, D(dims)), D(out_dims)).data, out); });
}

// normalize_intensities (registration.hpp:100-115).
int ref_normalize(const double* v, const int64_t* dims, double* out) {
    return guarded([&] { put(detail::normalize_intensities(vol<double>(v, D(dims))).data, out); });
}

// deformable_stage (registration.hpp:230-331) on `world` ranks; trace = one loss per
// iteration. loss_kind 0 = LNCC, 1 = MI; mi_kind 0 gaussian, 1 bspline3.
int ref_deformable_stage(const double* fixed, const double* moving, const int64_t* dims, const double* A,
                         const double* t, int nsteps, const double* downsample, const int* iterations, double lr,
                         double sigma_grad, double sigma_warp, int loss_kind, int window, double eps, int ants,
                         int bins, int mi_kind, int world, double* warp_out, double* trace) {
    return guarded([&] {
        const Dims3 d = D(dims);
        ScaleSchedule sch;
        for (int s = 0; s < nsteps; ++s) sch.steps.push_back(ScaleStep{downsample[s], iterations[s]});
        sch.lr = lr;
        sch.sigma_grad = sigma_grad;
        sch.sigma_warp = sigma_warp;
        sch.loss.kind = loss_kind == 0 ? LossKind::lncc : LossKind::mi;
        sch.loss.window = window;
        sch.loss.epsilon = eps;
        sch.loss.ants_approx = ants != 0;
        sch.loss.bins = bins;
        sch.loss.mi_bspline_kernel = mi_kind == 1;
        AffineMap aff;
        for (int i = 0; i < 9; ++i) aff.matrix.m[i] = A[i];
        aff.translation = Vec3{t[0], t[1], t[2]};
        DeformableOptions opts;
        opts.shards = world;
        std::vector<TraceEntry> tr;
        const auto w = deformable_stage(vol<double>(fixed, d), vol<double>(moving, d), aff, sch, opts, &tr);
        put(w.data, warp_out);
        for (std::size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i].loss;
    });
}

// affine_stage (registration.hpp:176-219); loss_kind 0 MSE, 1 LNCC, 2 MI.
int ref_affine_stage(const double* fixed, const double* moving, const int64_t* dims, int nsteps,
                     const double* downsample, const int* iterations, double lr, int loss_kind, int window, double eps,
                     int ants, int bins, int mi_kind, double* A_out, double* t_out, double* trace) {
    return guarded([&] {
        const Dims3 d = D(dims);
        ScaleSchedule sch;
        for (int s = 0; s < nsteps; ++s) sch.steps.push_back(ScaleStep{downsample[s], iterations[s]});
        sch.lr = lr;
        sch.loss.kind = loss_kind == 0 ? LossKind::mse : loss_kind == 1 ? LossKind::lncc : LossKind::mi;
        sch.loss.window = window;
        sch.loss.epsilon = eps;
        sch.loss.ants_approx = ants != 0;
        sch.loss.bins = bins;
        sch.loss.mi_bspline_kernel = mi_kind == 1;
        std::vector<TraceEntry> tr;
        const AffineMap a = affine_stage(vol<double>(fixed, d), vol<double>(moving, d), sch, &tr);
        for (int i = 0; i < 9; ++i) A_out[i] = a.matrix.m[static_cast<std::size_t>(i)];
        for (int i = 0; i < 3; ++i) t_out[i] = a.translation[i];
        for (std::size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i].loss;
    });
}

// jacobian_positive_fraction (metrics.hpp:145-176).
int ref_jacobian_positive(const double* u, const int64_t* dims, double* out) {
    return guarded([&] { *out = jacobian_positive_fraction(warp<double>(u, D(dims))); });
}

// The deformable step over H ranks. loss_kind 0 = LNCC, 1 = MI. fp32 = 1 runs the
// reference's T=float instantiation on the same inputs.
int ref_step(int loss_kind, int fp32, const double* f, const double* m, const double* u, const int64_t* dims,
             const double* A, const double* t, int window, double eps, int ants, int bins, int mi_kind, int approx,
             int world, double* loss, double* g_u, double* moved) {
    return guarded([&] {
        const Dims3 d = D(dims);
        *loss = fp32 ? step_impl<float>(loss_kind, f, m, u, d, A, t, window, eps, ants, bins, mi_kind, approx,
                                        world, g_u, moved)
                     : step_impl<double>(loss_kind, f, m, u, d, A, t, window, eps, ants, bins, mi_kind, approx,
                                         world, g_u, moved);
    });
}

// Label evaluation (metrics.hpp:44-201, sampler.hpp:331-365): out3 = dice mean,
// inv_dice (fixed-volume weights), hd90_cumulative with `spacing` (x, y, z).
int ref_label_metrics(const uint16_t* a, const uint16_t* b, const int64_t* dims, const double* spacing,
                      double* out3) {
    return guarded([&] {
        auto la = LabelVolume::zeros(D(dims)), lb = LabelVolume::zeros(D(dims));
        std::memcpy(la.data.data(), a, la.data.size() * sizeof(uint16_t));
        std::memcpy(lb.data.data(), b, lb.data.size() * sizeof(uint16_t));
        out3[0] = dice(la, lb).mean;
        out3[1] = inv_dice(la, lb);
        out3[2] = hd90_cumulative(la, lb, Vec3{spacing[0], spacing[1], spacing[2]});
    });
}

int ref_warp_labels_nn(const uint16_t* labels, const int64_t* ldims, const double* u, const int64_t* udims,
                       const double* A, const double* t, uint16_t* out) {
    return guarded([&] {
        auto l = LabelVolume::zeros(D(ldims));
        std::memcpy(l.data.data(), labels, l.data.size() * sizeof(uint16_t));
        SamplerArgs args;
        for (int i = 0; i < 9; ++i) args.A.m[static_cast<std::size_t>(i)] = A[i];
        args.t = Vec3{t[0], t[1], t[2]};
        const auto w = warp_labels_nn(l, warp<double>(u, D(udims)), args);
        std::memcpy(out, w.data.data(), w.data.size() * sizeof(uint16_t));
    });
}

} // extern "C"
