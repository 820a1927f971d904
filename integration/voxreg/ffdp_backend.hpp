// integration/voxreg/ffdp_backend.hpp -- the reference-side binding a voxreg maintainer adds
// (INTEGRATION.md section 3). Drop it into proj/include/voxreg/ and include it after
// voxreg/registration.hpp in a translation unit built with -DVOXREG_WITH_FFDP and linked
// against libffdp.so: the UNMODIFIED reference driver (deformable_stage,
// registration.hpp:230-331) then runs its T = float hot path on the B200.
//
// How it binds: every call the driver makes on the hot path is unqualified and takes
// reference containers of T, so argument-dependent lookup at the instantiation of
// deformable_stage<float> finds the non-template overloads below, which the overload rules
// prefer over the reference's templates of the same signature:
//   ring_sample           (distops.hpp:143-168)  -> ffdp_sampler_fwd
//   dist_lncc             (distops.hpp:283-352)  -> ffdp_lncc_fwd / _gamma / _combine
//   dist_mi               (distops.hpp:354-396)  -> ffdp_mi_hist / ffdp_mi_finalize / ffdp_mi_bwd
//   dist_mse              (distops.hpp:259-282)  -> ffdp_mse
//   ring_sample_backward  (distops.hpp:178-248)  -> ffdp_sampler_bwd
//   gp_convolve (warp)    (distops.hpp:93-101)   -> ffdp_gp_convolve
// Each overload serves a single worker (WorkerGroup(1)); with more workers it defers to the
// reference template (the sharded B200 path is ffdp_plan_*).
// Every call copies its operands to the device and its results back (exact drop-in
// semantics for the reference's host containers); a driver that keeps the scale on the
// device uses ffdp::voxreg::DeformableStep instead.
#pragma once

#include <ffdp/voxreg.hpp>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "voxreg/distops.hpp"
#include "voxreg/registration.hpp"

namespace voxreg {
namespace ffdp_backend {
namespace F = ::ffdp::voxreg;

inline F::Dims3 dims(const Dims3& d) { return F::Dims3{d.nx, d.ny, d.nz}; }
inline F::Volume3 dev(const Volume3<float>& v) {
    F::Volume3 d = F::Volume3::from_host(dims(v.dims), v.data.data());
    for (int c = 0; c < 3; ++c) d.spacing[c] = v.spacing[c], d.origin[c] = v.origin[c];
    return d;
}
inline F::WarpField dev(const WarpField<float>& w) { return F::WarpField::from_host(dims(w.dims), w.data.data()); }
inline Volume3<float> host(const F::Volume3& d, const Volume3<float>& like) {
    Volume3<float> r = Volume3<float>::zeros(like.dims);
    r.spacing = like.spacing;
    r.origin = like.origin;
    const std::vector<float> h = d.to_host();
    std::copy(h.begin(), h.end(), r.data.begin());
    return r;
}
inline WarpField<float> host(const F::WarpField& d, Dims3 dd) {
    WarpField<float> r = WarpField<float>::zeros(dd);
    const std::vector<float> h = d.to_host();
    std::copy(h.begin(), h.end(), r.data.begin());
    return r;
}
// the sampler arguments ring_sample uses on a single worker (its shard is the volume, the
// per-shard rescale is the identity, distops.hpp:121-133)
inline F::SamplerArgs args(const Mat3& A, const Vec3& t) {
    F::SamplerArgs a;
    for (int i = 0; i < 9; ++i) a.A.m[i] = A.m[static_cast<std::size_t>(i)];
    for (int c = 0; c < 3; ++c) a.t[c] = t[static_cast<std::size_t>(c)];
    return a;
}
// The reference's ParzenKernel keeps its kind private: recognise it by its values.
inline F::ParzenKernel kernel_of(const ParzenKernel& k) {
    const int b = k.bins();
    const ParzenKernel bs = ParzenKernel::bspline3(b), de = ParzenKernel::delta(b);
    auto same = [&](const ParzenKernel& o) {
        for (double x : {0.0, 0.13 / b, 0.71 / b, 1.37 / b})
            if (k.kappa(x) != o.kappa(x)) return false;
        return k.support() == o.support();
    };
    if (same(bs)) return F::ParzenKernel::bspline3(b);
    if (same(de)) return F::ParzenKernel::delta(b);
    return F::ParzenKernel::gaussian(b, k.support_bins() / 3.0);  // radius = 3 sigma (mi.hpp:33-40)
}
inline bool single(const WorkerContext& ctx) { return ctx.world_size() == 1; }
}  // namespace ffdp_backend

// ring_sample (distops.hpp:143-168), T = float
inline Volume3<float> ring_sample(WorkerContext& ctx, const Volume3<float>& m_shard, const WarpField<float>& u_shard,
                                  const Mat3& A, const Vec3& t, Dims3 m_global_dims, const ShardSpec& out_spec,
                                  RingSampleStats* stats = nullptr) {
    namespace B = ffdp_backend;
    if (!B::single(ctx) || stats)
        return ring_sample<float>(ctx, m_shard, u_shard, A, t, m_global_dims, out_spec, stats);
    const B::F::Volume3 dm = B::dev(m_shard);
    const B::F::WarpField du = B::dev(u_shard);
    Volume3<float> out = B::host(B::F::fused_sample(dm, &du, B::args(A, t)), Volume3<float>::zeros(u_shard.dims));
    out.spacing = m_shard.spacing;
    out.origin = m_shard.origin;
    return out;
}

// dist_lncc (distops.hpp:283-352), T = float: forward moments, the gamma family with
// gi = -1/n_total, ANTs or exact combination
inline DistLoss<float> dist_lncc(WorkerContext& ctx, const ShardSpec& spec, const Volume3<float>& f_shard,
                                 const Volume3<float>& moved_shard, int window, double eps, bool ants_approx,
                                 bool gp_sync, std::int64_t n_total) {
    namespace B = ffdp_backend;
    if (!B::single(ctx) || n_total != f_shard.dims.voxels())
        return dist_lncc<float>(ctx, spec, f_shard, moved_shard, window, eps, ants_approx, gp_sync, n_total);
    if (!(f_shard.dims == moved_shard.dims)) throw std::invalid_argument("dist_lncc: shard misalignment");
    const B::F::Volume3 df = B::dev(f_shard), dm = B::dev(moved_shard);
    auto fw = B::F::lncc_forward_fused(df, dm, window, eps);
    auto [gf, gm] = B::F::lncc_backward_fused(1.0, fw.second, df, dm, ants_approx);
    DistLoss<float> out;
    out.loss = fw.first.loss;
    out.grad_fixed = B::host(gf, f_shard);
    out.grad_moved = B::host(gm, f_shard);
    return out;
}

// dist_mi (distops.hpp:354-396), T = float: loss = -MI, gradients of -MI
inline DistLoss<float> dist_mi(WorkerContext& ctx, const Volume3<float>& f_shard, const Volume3<float>& moved_shard,
                               int bins, const ParzenKernel& kernel, bool approx_forward, std::int64_t n_total) {
    namespace B = ffdp_backend;
    if (!B::single(ctx) || n_total != f_shard.dims.voxels())
        return dist_mi<float>(ctx, f_shard, moved_shard, bins, kernel, approx_forward, n_total);
    if (!(f_shard.dims == moved_shard.dims)) throw std::invalid_argument("dist_mi: shard misalignment");
    const B::F::Volume3 df = B::dev(f_shard), dm = B::dev(moved_shard);
    const B::F::ParzenKernel k = B::kernel_of(kernel);
    const B::F::MiResult r = approx_forward ? B::F::mi_forward_approx(df, dm, bins, k)
                                            : B::F::mi_forward_exact(df, dm, bins, k);
    auto [gi, gj] = B::F::mi_backward(-1.0, df, dm, r.hist, k);
    DistLoss<float> out;
    out.loss = -r.mi;
    out.mi_payload_elements = static_cast<std::size_t>(bins) * static_cast<std::size_t>(bins) + 2u * bins;
    out.grad_fixed = B::host(gi, f_shard);
    out.grad_moved = B::host(gj, f_shard);
    return out;
}

// dist_mse (distops.hpp:259-282), T = float
inline DistLoss<float> dist_mse(WorkerContext& ctx, const Volume3<float>& f_shard, const Volume3<float>& moved_shard,
                                std::int64_t n_total) {
    namespace B = ffdp_backend;
    if (!B::single(ctx)) return dist_mse<float>(ctx, f_shard, moved_shard, n_total);
    if (!(f_shard.dims == moved_shard.dims)) throw std::invalid_argument("dist_mse: shard misalignment");
    const B::F::Volume3 df = B::dev(f_shard), dm = B::dev(moved_shard);
    B::F::Volume3 g = B::F::Volume3::uninitialized(df.dims);
    B::F::DeviceArray<double> sum(1);
    sum.zero();
    B::F::check(ffdp_mse(df.data.data(), dm.data.data(), df.dims.voxels(), n_total, g.data.data(), sum.data(),
                         nullptr));
    DistLoss<float> out;
    out.loss = sum.download()[0] / static_cast<double>(n_total);
    out.grad_moved = B::host(g, f_shard);
    out.grad_fixed = Volume3<float>::zeros(f_shard.dims);
    for (std::size_t i = 0; i < out.grad_fixed.data.size(); ++i) out.grad_fixed.data[i] = -out.grad_moved.data[i];
    return out;
}

// ring_sample_backward (distops.hpp:178-248), T = float
inline RingSampleGrads<float> ring_sample_backward(WorkerContext& ctx, const Volume3<float>& upstream,
                                                   const Volume3<float>& m_shard, const WarpField<float>& u_shard,
                                                   const Mat3& A, const Vec3& t, Dims3 m_global_dims,
                                                   const ShardSpec& out_spec, const SamplerGradWant& want) {
    namespace B = ffdp_backend;
    if (!B::single(ctx))
        return ring_sample_backward<float>(ctx, upstream, m_shard, u_shard, A, t, m_global_dims, out_spec, want);
    if (!(upstream.dims == u_shard.dims)) throw std::invalid_argument("ring_sample_backward: upstream lattice mismatch");
    const B::F::Volume3 dup = B::dev(upstream), dm = B::dev(m_shard);
    const B::F::WarpField du = B::dev(u_shard);
    B::F::SamplerGradWant fw;
    fw.image = want.image;
    fw.warp = want.warp;
    fw.affine = want.affine;
    fw.translation = want.translation;
    B::F::SamplerGrads g = B::F::fused_sample_backward(dup, dm, &du, B::args(A, t), fw);
    RingSampleGrads<float> out;
    if (g.warp) out.warp = B::host(*g.warp, u_shard.dims);
    if (g.image) out.image = B::host(*g.image, m_shard);
    if (g.affine) {
        Mat3 a;
        for (int i = 0; i < 9; ++i) a.m[static_cast<std::size_t>(i)] = g.affine->m[i];
        out.affine = a;
    }
    if (g.translation) out.translation = Vec3{(*g.translation)[0], (*g.translation)[1], (*g.translation)[2]};
    return out;
}

// gp_convolve of a warp slab (distops.hpp:93-101), T = float
inline WarpField<float> gp_convolve(WorkerContext& ctx, const WarpField<float>& slab, const std::vector<double>& taps,
                                    const ShardSpec& spec, EdgeMode mode = EdgeMode::zero_pad, bool sync = true) {
    namespace B = ffdp_backend;
    if (!B::single(ctx)) return gp_convolve<float>(ctx, slab, taps, spec, mode, sync);
    const B::F::WarpField d = B::dev(slab);
    return B::host(B::F::gp_convolve(d, taps, mode == EdgeMode::renormalize ? B::F::EdgeMode::renormalize
                                                                               : B::F::EdgeMode::zero_pad),
                   slab.dims);
}

}  // namespace voxreg
