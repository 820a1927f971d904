// ffdp/voxreg.hpp -- C++ host mirror of the voxreg operator API over the C ABI (ffdp.h).
//
// A voxreg caller switches its hot path to the B200 by including this header instead of
// voxreg/sampler.hpp, lncc.hpp and mi.hpp: the same names, argument meaning, ownership
// (outputs are fresh owning containers; LnccState is consumed by the backward) and
// exceptions (std::invalid_argument / std::logic_error / std::runtime_error) as the
// reference, with the containers living in device memory (Volume3 / WarpField below hold
// fp32 device buffers; from_host / to_host move them). Header-only; link libffdp.so and
// libcudart. No fallback: every operation runs the sm_100a kernels or throws.
//
// Reference interfaces mirrored (file:line under proj/include/voxreg):
//   Dims3, Vec3, Mat3, DomainBounds   geometry.hpp:10-109
//   Volume3, WarpField                volume.hpp:18-84
//   SamplerArgs, SamplerGradWant,
//   SamplerGrads                      sampler.hpp:25-52
//   fused_sample[_accumulate],
//   fused_sample_backward             sampler.hpp:248-300
//   LnccState, LnccResult,
//   lncc_forward_fused,
//   lncc_backward_fused               lncc.hpp:25-42, 144-280
//   ParzenKernel, JointHistogram,
//   MiStats, MiResult, mi_forward_*,
//   mi_backward                       mi.hpp:28-165, 235-437
//   the deformable step's loss/grad   registration.hpp:277-312 (DeformableStep)
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ffdp.h"

namespace ffdp {
namespace voxreg {

// ------------------------------------------------------------------ errors
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Maps an ffdp_status onto the reference's exception types (ffdp.h header comment).
inline void check(int status) {
    if (status == FFDP_OK) return;
    const std::string msg = ffdp_last_error();
    switch (status) {
        case FFDP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case FFDP_LOGIC: throw std::logic_error(msg);
        case FFDP_RUNTIME: throw std::runtime_error(msg);
        default: throw CudaError(msg);
    }
}

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ geometry (geometry.hpp:10-109)
struct Dims3 {
    std::int64_t nx = 0, ny = 0, nz = 0;
    std::int64_t voxels() const { return nx * ny * nz; }
    bool positive() const { return nx > 0 && ny > 0 && nz > 0; }
    std::int64_t operator[](int c) const { return c == 0 ? nx : c == 1 ? ny : nz; }
    bool operator==(const Dims3& o) const { return nx == o.nx && ny == o.ny && nz == o.nz; }
    bool operator!=(const Dims3& o) const { return !(*this == o); }
    ffdp_dims c() const { return ffdp_dims{nx, ny, nz}; }
};

struct Vec3 {
    double v[3] = {0, 0, 0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};

struct Mat3 {
    double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major
    static Mat3 identity() {
        Mat3 a;
        a.m[0] = a.m[4] = a.m[8] = 1.0;
        return a;
    }
    double& operator()(int r, int c) { return m[3 * r + c]; }
    double operator()(int r, int c) const { return m[3 * r + c]; }
    bool finite() const {
        for (double x : m)
            if (!std::isfinite(x)) return false;
        return true;
    }
};

struct DomainBounds {
    Vec3 lo{{-1, -1, -1}};
    Vec3 hi{{1, 1, 1}};
    static DomainBounds full() { return DomainBounds{}; }
    bool valid() const {
        for (int c = 0; c < 3; ++c)
            if (!std::isfinite(lo[c]) || !std::isfinite(hi[c]) || !(lo[c] <= hi[c])) return false;
        return true;
    }
};

// ------------------------------------------------------------------ device containers (volume.hpp:18-84)
template <typename T>
class DeviceArray {
  public:
    DeviceArray() = default;
    explicit DeviceArray(std::size_t n) : n_(n) {
        if (n) check_cuda(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)), "cudaMalloc");
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_, n_ = o.n_;
            o.p_ = nullptr, o.n_ = 0;
        }
        return *this;
    }
    ~DeviceArray() { release(); }

    T* data() { return p_; }
    const T* data() const { return p_; }
    std::size_t size() const { return n_; }
    void zero(cudaStream_t s = nullptr) {
        if (n_) check_cuda(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s), "cudaMemsetAsync");
    }
    void upload(const T* host, cudaStream_t s = nullptr) {
        if (n_) check_cuda(cudaMemcpyAsync(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    }
    std::vector<T> download(cudaStream_t s = nullptr) const {
        std::vector<T> h(n_);
        if (n_) {
            check_cuda(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
            check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        }
        return h;
    }

  private:
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
    }
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

// Volume3<float> on the device: x-fastest, index (z*ny + y)*nx + x.
struct Volume3 {
    Dims3 dims;
    Vec3 spacing{{1, 1, 1}};
    Vec3 origin{{0, 0, 0}};
    DeviceArray<float> data;

    static Volume3 zeros(Dims3 d, cudaStream_t s = nullptr) {
        if (!d.positive()) throw std::invalid_argument("Volume3: dims must be positive");
        Volume3 v;
        v.dims = d;
        v.data = DeviceArray<float>(static_cast<std::size_t>(d.voxels()));
        v.data.zero(s);
        return v;
    }
    static Volume3 uninitialized(Dims3 d) {
        if (!d.positive()) throw std::invalid_argument("Volume3: dims must be positive");
        Volume3 v;
        v.dims = d;
        v.data = DeviceArray<float>(static_cast<std::size_t>(d.voxels()));
        return v;
    }
    static Volume3 from_host(Dims3 d, const float* host, cudaStream_t s = nullptr) {
        Volume3 v = uninitialized(d);
        v.data.upload(host, s);
        return v;
    }
    std::vector<float> to_host(cudaStream_t s = nullptr) const { return data.download(s); }
    bool same_lattice(const Volume3& o) const { return dims == o.dims; }
};

// WarpField<float> on the device: 3 interleaved components per voxel.
struct WarpField {
    Dims3 dims;
    DeviceArray<float> data;

    static WarpField zeros(Dims3 d, cudaStream_t s = nullptr) {
        WarpField w = uninitialized(d);
        w.data.zero(s);
        return w;
    }
    static WarpField uninitialized(Dims3 d) {
        if (!d.positive()) throw std::invalid_argument("WarpField: dims must be positive");
        WarpField w;
        w.dims = d;
        w.data = DeviceArray<float>(static_cast<std::size_t>(3 * d.voxels()));
        return w;
    }
    static WarpField from_host(Dims3 d, const float* host, cudaStream_t s = nullptr) {
        WarpField w = uninitialized(d);
        w.data.upload(host, s);
        return w;
    }
    std::vector<float> to_host(cudaStream_t s = nullptr) const { return data.download(s); }
};

// ------------------------------------------------------------------ sampler (sampler.hpp:25-300)
struct SamplerArgs {
    Mat3 A = Mat3::identity();
    Vec3 t{{0, 0, 0}};
    Vec3 S{{1, 1, 1}};  // diagonal rescale applied to the displacement
    DomainBounds bounds = DomainBounds::full();

    void validate() const {
        if (!A.finite()) throw std::invalid_argument("SamplerArgs: non-finite affine");
        for (int c = 0; c < 3; ++c)
            if (!(S[c] > 0)) throw std::invalid_argument("SamplerArgs: S must be positive");
        if (!bounds.valid()) throw std::invalid_argument("SamplerArgs: invalid bounds");
    }
    ffdp_sampler_args c() const {
        ffdp_sampler_args a;
        std::memcpy(a.A, A.m, sizeof(a.A));
        for (int i = 0; i < 3; ++i) {
            a.t[i] = t[i];
            a.S[i] = S[i];
            a.x_min[i] = bounds.lo[i];
            a.x_max[i] = bounds.hi[i];
        }
        return a;
    }
};

struct SamplerGradWant {
    bool image = false;
    bool warp = false;
    bool affine = false;
    bool translation = false;
    int mask() const {
        return (image ? FFDP_WANT_IMAGE : 0) | (warp ? FFDP_WANT_WARP : 0) | (affine ? FFDP_WANT_AFFINE : 0) |
               (translation ? FFDP_WANT_TRANSLATION : 0);
    }
};

struct SamplerGrads {
    std::optional<Volume3> image;
    std::optional<WarpField> warp;
    std::optional<Mat3> affine;
    std::optional<Vec3> translation;
};

inline ffdp_image_window window_of(const Volume3& img) {
    return ffdp_image_window{img.data.data(), img.dims.c(), 0, img.dims.nz, 0};
}

inline Dims3 sampler_output_dims(const Volume3& img, const WarpField* u) { return u ? u->dims : img.dims; }

// fused_sample (sampler.hpp:254-263)
inline Volume3 fused_sample(const Volume3& img, const WarpField* u, const SamplerArgs& args,
                            cudaStream_t s = nullptr) {
    args.validate();
    Volume3 out = Volume3::uninitialized(sampler_output_dims(img, u));
    out.spacing = img.spacing;
    out.origin = img.origin;
    const ffdp_sampler_args a = args.c();
    check(ffdp_sampler_fwd(window_of(img), u ? u->data.data() : nullptr, out.dims.c(), &a, out.data.data(), 0,
                           nullptr, nullptr, s));
    return out;
}

// fused_sample_accumulate (sampler.hpp:268-276); abs_contribution is a HOST double.
inline void fused_sample_accumulate(const Volume3& img, const WarpField* u, const SamplerArgs& args, Volume3& out,
                                    double* abs_contribution = nullptr, cudaStream_t s = nullptr) {
    if (out.dims != sampler_output_dims(img, u))
        throw std::invalid_argument("fused_sample_accumulate: output lattice mismatch");
    args.validate();
    const ffdp_sampler_args a = args.c();
    std::optional<DeviceArray<double>> acc;
    if (abs_contribution) {
        acc.emplace(1);
        acc->zero(s);
    }
    check(ffdp_sampler_fwd(window_of(img), u ? u->data.data() : nullptr, out.dims.c(), &a, out.data.data(), 1,
                           acc ? acc->data() : nullptr, nullptr, s));
    if (abs_contribution) *abs_contribution += acc->download(s)[0];
}

// fused_sample_backward (sampler.hpp:279-300)
inline SamplerGrads fused_sample_backward(const Volume3& upstream, const Volume3& img, const WarpField* u,
                                          const SamplerArgs& args, const SamplerGradWant& want,
                                          cudaStream_t s = nullptr) {
    const Dims3 od = sampler_output_dims(img, u);
    if (upstream.dims != od) throw std::invalid_argument("fused_sample_backward: upstream lattice mismatch");
    args.validate();
    SamplerGrads g;
    if (want.image) g.image = Volume3::zeros(img.dims, s);
    if (want.warp) g.warp = WarpField::uninitialized(od);
    std::optional<DeviceArray<double>> gat;
    if (want.affine || want.translation) gat.emplace(12);
    const ffdp_sampler_args a = args.c();
    check(ffdp_sampler_bwd(upstream.data.data(), window_of(img), u ? u->data.data() : nullptr, od.c(), &a,
                           want.mask(), want.image ? g.image->data.data() : nullptr,
                           want.warp ? g.warp->data.data() : nullptr, gat ? gat->data() : nullptr, nullptr, s));
    if (gat) {
        const std::vector<double> h = gat->download(s);
        if (want.affine) {
            Mat3 m;
            std::memcpy(m.m, h.data(), 9 * sizeof(double));
            g.affine = m;
        }
        if (want.translation) g.translation = Vec3{{h[9], h[10], h[11]}};
    }
    return g;
}

// ------------------------------------------------------------------ LNCC (lncc.hpp:25-280)
struct LnccState {
    Dims3 dims;
    DeviceArray<double> channels;  // 5 x voxels: mean_f, mean_m, mean_ff, mean_mm, mean_fm
    int window = 7;
    double epsilon = 1e-5;
    std::int64_t voxels = 0;
    const double* channel(int c) const { return channels.data() + c * voxels; }
};

struct LnccResult {
    double loss = 0;
    std::optional<Volume3> ncc_map;  // per-voxel n_i, filled only when requested
    bool has_map = false;
};

inline void check_lncc(const Volume3& f, const Volume3& m, int window) {
    if (!f.same_lattice(m)) throw std::invalid_argument("lncc: lattices differ");
    if (window < 1 || window % 2 == 0) throw std::invalid_argument("lncc: window must be odd and >= 1");
}

inline ffdp_slab full_slab(std::int64_t nz) { return ffdp_slab{0, nz, 0, nz, nz}; }

// lncc_forward_fused (lncc.hpp:144-205): loss = 1 - mean(A^2 / (B C + eps)).
inline std::pair<LnccResult, LnccState> lncc_forward_fused(const Volume3& f, const Volume3& m, int window,
                                                           double eps, bool want_map = false,
                                                           cudaStream_t s = nullptr) {
    check_lncc(f, m, window);
    LnccState st;
    st.dims = f.dims;
    st.voxels = f.dims.voxels();
    st.window = window;
    st.epsilon = eps;
    st.channels = DeviceArray<double>(static_cast<std::size_t>(5 * st.voxels));
    LnccResult res;
    if (want_map) res.ncc_map = Volume3::uninitialized(f.dims);
    res.has_map = want_map;
    DeviceArray<double> sum(1);
    sum.zero(s);
    check(ffdp_lncc_fwd(f.data.data(), m.data.data(), f.dims.c(), full_slab(f.dims.nz), window, eps,
                        st.channels.data(), want_map ? res.ncc_map->data.data() : nullptr, sum.data(), s));
    res.loss = 1.0 - sum.download(s)[0] / static_cast<double>(st.voxels);
    return {std::move(res), std::move(st)};
}

// lncc_backward_fused (lncc.hpp:226-280): consumes `state` (rewritten as the gamma family).
// Returns (dL/dF, dL/dM).
inline std::pair<Volume3, Volume3> lncc_backward_fused(double upstream, LnccState& state, const Volume3& f,
                                                       const Volume3& m, bool ants_approx,
                                                       cudaStream_t s = nullptr) {
    if (state.dims != f.dims || !f.same_lattice(m))
        throw std::invalid_argument("lncc_backward_fused: lattice mismatch");
    const double gi = -upstream / static_cast<double>(state.voxels);
    check(ffdp_lncc_gamma(state.channels.data(), state.voxels, state.epsilon, gi, s));
    Volume3 gf = Volume3::uninitialized(f.dims), gm = Volume3::uninitialized(f.dims);
    check(ffdp_lncc_combine(state.channels.data(), f.dims.c(), full_slab(f.dims.nz), state.window,
                            ants_approx ? 1 : 0, f.data.data(), m.data.data(), gf.data.data(), gm.data.data(), s));
    return {std::move(gf), std::move(gm)};
}

// ------------------------------------------------------------------ MI (mi.hpp:28-437)
class ParzenKernel {
  public:
    static ParzenKernel gaussian(int bins, double sigma_bins = 0.5) {
        return ParzenKernel(FFDP_PARZEN_GAUSSIAN, bins, sigma_bins);
    }
    static ParzenKernel bspline3(int bins) { return ParzenKernel(FFDP_PARZEN_BSPLINE3, bins, 0.5); }
    static ParzenKernel delta(int bins) { return ParzenKernel(FFDP_PARZEN_DELTA, bins, 0.5); }
    int bins() const { return c_.bins; }
    double support() const { return c_.radius; }
    double support_bins() const { return c_.radius * c_.bins; }
    const ffdp_parzen& c() const { return c_; }

  private:
    ParzenKernel(int kind, int bins, double sigma_bins) { check(ffdp_parzen_make(kind, bins, sigma_bins, &c_)); }
    ffdp_parzen c_{};
};

inline double bin_center(int j, int bins) { return (static_cast<double>(j) + 0.5) / static_cast<double>(bins); }

struct JointHistogram {
    int bins = 0;
    std::int64_t samples = 0;
    double raw_joint_sum = 0;
    std::vector<double> p_i, p_j;
    std::vector<double> p_ij;  // row-major [m * bins + n]
    std::vector<double> raw_joint;
    std::vector<double> raw_marg_i, raw_marg_j;
};

struct MiStats {
    std::uint64_t hist_writes = 0;
    std::uint64_t kernel_evals = 0;
};

struct MiResult {
    double mi = 0;
    JointHistogram hist;
    MiStats stats;
};

namespace detail {
inline std::size_t table_len(int b) { return static_cast<std::size_t>(2 * b * b + 2 * b + 4); }

// finalize_histogram + histogram_mi (mi.hpp:181-209) from the device raw accumulators.
inline double hist_from_raw(const DeviceArray<double>& raw, int b, std::int64_t samples, JointHistogram& h,
                            cudaStream_t s) {
    DeviceArray<double> table(table_len(b));
    check(ffdp_mi_finalize(raw.data(), b, -1.0, table.data(), s));
    const std::vector<double> t = table.download(s);
    const std::vector<double> r = raw.download(s);
    const std::size_t bb = static_cast<std::size_t>(b) * b;
    h.bins = b;
    h.samples = samples;
    h.p_ij.assign(t.begin(), t.begin() + bb);
    h.p_i.assign(t.begin() + bb, t.begin() + bb + b);
    h.p_j.assign(t.begin() + bb + b, t.begin() + bb + 2 * b);
    h.raw_joint_sum = t[2 * bb + 2 * b];
    h.raw_joint.assign(r.begin(), r.begin() + bb);
    h.raw_marg_i.assign(r.begin() + bb, r.begin() + bb + b);
    h.raw_marg_j.assign(r.begin() + bb + b, r.end());
    return t[2 * bb + 2 * b + 1];
}

inline MiResult mi_forward(const Volume3& i, const Volume3& j, int bins, const ParzenKernel& k, bool approx,
                           cudaStream_t s) {
    if (!i.same_lattice(j)) throw std::invalid_argument("mi: lattices differ");
    if (bins < 2) throw std::invalid_argument("mi: bins must be >= 2");
    if (bins != k.bins()) throw std::invalid_argument("mi: kernel bin count differs from bins");
    const std::int64_t n = i.dims.voxels();
    DeviceArray<double> raw(static_cast<std::size_t>(bins * bins + 2 * bins));
    raw.zero(s);
    DeviceArray<std::int32_t> bad(1);
    bad.zero(s);
    std::uint64_t stats[2] = {0, 0};
    check(ffdp_mi_hist(i.data.data(), j.data.data(), n, &k.c(), approx ? 1 : 0, raw.data(), bad.data(), stats, s));
    if (bad.download(s)[0]) throw std::invalid_argument("mi: intensities must lie in [0,1]");
    MiResult r;
    r.mi = hist_from_raw(raw, bins, n, r.hist, s);
    r.stats.hist_writes = stats[0];
    r.stats.kernel_evals = stats[1];
    return r;
}

// mi_backward_impl (mi.hpp:361-421): no sample-count check (global histograms).
inline std::pair<Volume3, Volume3> mi_backward_impl(double upstream, const Volume3& i, const Volume3& j,
                                                    const JointHistogram& h, const ParzenKernel& k,
                                                    cudaStream_t s) {
    if (!i.same_lattice(j)) throw std::invalid_argument("mi_backward: lattices differ");
    const int b = h.bins;
    std::vector<double> rawh(h.raw_joint);
    rawh.insert(rawh.end(), h.raw_marg_i.begin(), h.raw_marg_i.end());
    rawh.insert(rawh.end(), h.raw_marg_j.begin(), h.raw_marg_j.end());
    if (rawh.size() != static_cast<std::size_t>(b * b + 2 * b))
        throw std::invalid_argument("mi_backward: malformed histogram");
    DeviceArray<double> raw(rawh.size());
    raw.upload(rawh.data(), s);
    DeviceArray<double> table(table_len(b));
    check(ffdp_mi_finalize(raw.data(), b, upstream, table.data(), s));
    Volume3 gi = Volume3::uninitialized(i.dims), gj = Volume3::uninitialized(i.dims);
    check(ffdp_mi_bwd(i.data.data(), j.data.data(), i.dims.voxels(), &k.c(), table.data(), gi.data.data(),
                      gj.data.data(), s));
    check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");  // raw/table are freed on return
    return {std::move(gi), std::move(gj)};
}
}  // namespace detail

// mi_forward_exact (mi.hpp:235-272)
inline MiResult mi_forward_exact(const Volume3& i, const Volume3& j, int bins, const ParzenKernel& k,
                                 cudaStream_t s = nullptr) {
    return detail::mi_forward(i, j, bins, k, false, s);
}

// mi_forward_approx (mi.hpp:285-354)
inline MiResult mi_forward_approx(const Volume3& i, const Volume3& j, int bins, const ParzenKernel& k,
                                  cudaStream_t s = nullptr) {
    return detail::mi_forward(i, j, bins, k, true, s);
}

// mi_backward (mi.hpp:430-437): gradients w.r.t. both images given upstream = dL/dMI.
inline std::pair<Volume3, Volume3> mi_backward(double upstream, const Volume3& i, const Volume3& j,
                                               const JointHistogram& h, const ParzenKernel& k,
                                               cudaStream_t s = nullptr) {
    if (i.dims.voxels() != h.samples) throw std::invalid_argument("mi_backward: histogram sample count mismatch");
    return detail::mi_backward_impl(upstream, i, j, h, k, s);
}

// ------------------------------------------------------------------ the fused deformable step
enum class LossKind { mse, lncc, mi };

// LossParams (registration.hpp:33-46). DeformableStep fuses LNCC (ANTs) and exact-forward
// MI; the other combinations run through loss_and_grad (deformable_stage composes them).
struct LossParams {
    LossKind kind = LossKind::lncc;
    int window = 7;
    double epsilon = 1e-5;
    bool ants_approx = true;
    int bins = 32;
    bool mi_bspline_kernel = false;  // the reference default (registration.hpp:40)
    bool mi_approx_forward = false;
    bool lncc_naive_backend = false;  // registration.hpp:38: same values as the fused path here
};

struct StepResult {
    double loss = 0;
    std::int32_t window_misses = 0;
};

// One deformable-step evaluation (registration.hpp:277-312 at H = 1): moved =
// fused_sample(M, u; A, t) -> LNCC (ANTs) or Mattes MI -> g_u = fused_sample_backward(
// dL/dmoved, want warp), as one fused kernel (LNCC) or hist + finalize + grad (MI).
// Built once per scale (M is static within a scale, registration.hpp:249,270): holds the
// zero-bordered copy of M and all workspace, so step() allocates nothing and, with
// sync = false, is capturable in a CUDA graph.
class DeformableStep {
  public:
    DeformableStep(const Volume3& fixed, const Volume3& moving, const LossParams& p, cudaStream_t s = nullptr)
        : f_(fixed.data.data()), dims_(fixed.dims), p_(p), stream_(s) {
        if (!fixed.same_lattice(moving))
            throw std::invalid_argument("DeformableStep: F and M must share a lattice (registration.hpp:268-270)");
        if (p.kind == LossKind::mse) throw std::invalid_argument("DeformableStep: MSE runs through loss_and_grad");
        if (p.kind == LossKind::lncc && !p.ants_approx)
            throw std::invalid_argument("DeformableStep: the fused LNCC step implements the ANTs backward");
        if (p.kind == LossKind::lncc && p.window != 7)
            throw std::invalid_argument("DeformableStep: the fused LNCC step is built for window 7");
        if (p.kind == LossKind::mi && p.mi_approx_forward)
            throw std::invalid_argument("DeformableStep: the fused MI step uses the exact Parzen forward");
        const Dims3 d = dims_;
        m_pad_ = DeviceArray<float>(static_cast<std::size_t>((d.nx + 4) * (d.ny + 4) * (d.nz + 4)));
        check(ffdp_pad_window(moving.data.data(), d.c(), 0, d.nz, m_pad_.data(), s));
        miss_ = DeviceArray<std::int32_t>(1);
        sum_ = DeviceArray<double>(1);
        if (p.kind == LossKind::lncc) {
            // the step's intensity frame: value ranges of F and M, fixed while F and M are
            ranges_ = DeviceArray<float>(4);
            check(ffdp_minmax(fixed.data.data(), d.voxels(), ranges_.data(), s));
            check(ffdp_minmax(moving.data.data(), d.voxels(), ranges_.data() + 2, s));
            lws_ = DeviceArray<unsigned char>(
                static_cast<std::size_t>(ffdp_step_lncc_workspace_bytes(d.c(), full_slab(d.nz))));
        } else {
            kernel_.emplace(p.mi_bspline_kernel ? ParzenKernel::bspline3(p.bins) : ParzenKernel::gaussian(p.bins));
            raw_ = DeviceArray<double>(static_cast<std::size_t>(p.bins * p.bins + 2 * p.bins));
            table_ = DeviceArray<double>(detail::table_len(p.bins));
            scratch_ = DeviceArray<unsigned char>(static_cast<std::size_t>(ffdp_step_mi_workspace_bytes(p.bins)));
            // pass-1 records: pass 2 then streams them instead of sampling the warp again
            if (p.mi_bspline_kernel)
                rec_ = DeviceArray<float>(
                    static_cast<std::size_t>(ffdp_step_mi_record_bytes(d.c(), full_slab(d.nz)) / sizeof(float)));
        }
    }

    // g_u (same lattice as F) is overwritten. With sync = false nothing is read back
    // (loss() / misses() read it later).
    StepResult step(const WarpField& u, const SamplerArgs& args, WarpField& g_u, bool sync = true) {
        if (u.dims != dims_ || g_u.dims != dims_) throw std::invalid_argument("sampler: warp lattice mismatch");
        args.validate();
        const ffdp_sampler_args a = args.c();
        const ffdp_image_window w{m_pad_.data(), dims_.c(), 0, dims_.nz, 2};
        miss_.zero(stream_);
        if (p_.kind == LossKind::lncc) {
            sum_.zero(stream_);
            check(ffdp_step_lncc(f_, u.data.data(), dims_.c(), full_slab(dims_.nz), w, &a, p_.window, p_.epsilon,
                                 -1.0 / static_cast<double>(dims_.voxels()), ranges_.data(), g_u.data.data(),
                                 sum_.data(), miss_.data(), lws_.data(), stream_));
        } else {
            check(ffdp_step_mi(f_, u.data.data(), dims_.c(), full_slab(dims_.nz), w, &a, &kernel_->c(), raw_.data(),
                               table_.data(), g_u.data.data(), scratch_.data(), rec_.size() ? rec_.data() : nullptr,
                               miss_.data(), stream_));
        }
        StepResult r;
        if (sync) {
            r.loss = loss();
            r.window_misses = miss_.download(stream_)[0];
        }
        return r;
    }

    double loss() const {
        if (p_.kind == LossKind::lncc) return 1.0 - sum_.download(stream_)[0] / static_cast<double>(dims_.voxels());
        const int b = p_.bins;
        double v = 0;
        check_cuda(cudaMemcpyAsync(&v, table_.data() + 2 * b * b + 2 * b + 1, sizeof(double), cudaMemcpyDeviceToHost,
                                   stream_),
                   "D2H");
        check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
        return -v;
    }

    const Dims3& dims() const { return dims_; }

  private:
    const float* f_;
    Dims3 dims_;
    LossParams p_;
    cudaStream_t stream_;
    DeviceArray<float> m_pad_;
    DeviceArray<std::int32_t> miss_;
    DeviceArray<double> sum_, raw_, table_;
    DeviceArray<float> rec_, ranges_;
    DeviceArray<unsigned char> scratch_, lws_;
    std::optional<ParzenKernel> kernel_;
};


// ------------------------------------------------------------------ smoothing (smoothing.hpp:25-125)
enum class EdgeMode { zero_pad, renormalize };

// gaussian_taps (smoothing.hpp:25-39): truncated at ceil(3 sigma), normalized to sum 1.
inline std::vector<double> gaussian_taps(double sigma) {
    if (!std::isfinite(sigma) || sigma < 0) throw std::invalid_argument("gaussian_taps: sigma must be finite and >= 0");
    if (sigma == 0) return {1.0};
    const auto radius = static_cast<std::int64_t>(std::ceil(3.0 * sigma));
    std::vector<double> taps(static_cast<std::size_t>(2 * radius + 1));
    double sum = 0;
    for (std::int64_t k = -radius; k <= radius; ++k) {
        const double w = std::exp(-0.5 * (static_cast<double>(k) / sigma) * (static_cast<double>(k) / sigma));
        taps[static_cast<std::size_t>(k + radius)] = w;
        sum += w;
    }
    for (auto& w : taps) w /= sum;
    return taps;
}

// box_taps (smoothing.hpp:42-46).
inline std::vector<double> box_taps(int window) {
    if (window < 1 || window % 2 == 0) throw std::invalid_argument("box_taps: window must be odd and >= 1");
    return std::vector<double>(static_cast<std::size_t>(window), 1.0 / window);
}

// gp_convolve / separable_convolve (distops.hpp:84-101, smoothing.hpp:98-105) of a whole
// volume or warp field on one GPU: one z-marching kernel (ffdp_gp_convolve).
inline Volume3 gp_convolve(const Volume3& v, const std::vector<double>& taps, EdgeMode mode = EdgeMode::zero_pad,
                           cudaStream_t s = nullptr) {
    if (taps.size() % 2 == 0) throw std::invalid_argument("gp_convolve: kernel must be odd");
    Volume3 out = Volume3::uninitialized(v.dims);
    out.spacing = v.spacing;
    out.origin = v.origin;
    check(ffdp_gp_convolve(v.data.data(), out.data.data(), v.dims.c(), full_slab(v.dims.nz), 1, taps.data(),
                           static_cast<int>(taps.size()), mode == EdgeMode::renormalize ? 1 : 0, s));
    return out;
}

inline WarpField gp_convolve(const WarpField& w, const std::vector<double>& taps, EdgeMode mode = EdgeMode::zero_pad,
                             cudaStream_t s = nullptr) {
    if (taps.size() % 2 == 0) throw std::invalid_argument("gp_convolve: kernel must be odd");
    WarpField out = WarpField::uninitialized(w.dims);
    check(ffdp_gp_convolve(w.data.data(), out.data.data(), w.dims.c(), full_slab(w.dims.nz), 3, taps.data(),
                           static_cast<int>(taps.size()), mode == EdgeMode::renormalize ? 1 : 0, s));
    return out;
}

// ------------------------------------------------------------------ Adam (adam.hpp:14-50)
// AdamState of a warp field: moments on the device (fp32, the reference's T storage).
struct AdamState {
    DeviceArray<float> m1, m2;
    std::int64_t step = 0;
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;

    static AdamState zeros(std::size_t n, cudaStream_t s = nullptr) {
        AdamState a;
        a.m1 = DeviceArray<float>(n);
        a.m2 = DeviceArray<float>(n);
        a.m1.zero(s);
        a.m2.zero(s);
        return a;
    }
};

// adam_step (adam.hpp:30-50) on a warp field, in place (the Adam epilogue of
// ffdp_sobolev_adam with a single unit tap).
inline void adam_step(WarpField& param, const WarpField& grad, AdamState& st, double lr, cudaStream_t s = nullptr) {
    if (param.dims != grad.dims || param.data.size() != st.m1.size() || param.data.size() != st.m2.size())
        throw std::invalid_argument("adam_step: shape mismatch");
    st.step += 1;
    const double one = 1.0;
    check(ffdp_sobolev_adam(grad.data.data(), param.data.data(), st.m1.data(), st.m2.data(), param.dims.c(),
                            full_slab(param.dims.nz), &one, 1, lr, st.beta1, st.beta2, st.eps, st.step, s));
}

// The warp update of one deformable iteration (registration.hpp:313-317): gp_convolve(g_u,
// gaussian(sigma_grad), renormalize) fused with adam_step (u, st updated in place), then
// `out` = gp_convolve(u, gaussian(sigma_warp), renormalize).
inline void warp_update(WarpField& u, const WarpField& g_u, AdamState& st, double lr_norm, WarpField& out,
                        double sigma_grad = 1.0, double sigma_warp = 0.5, cudaStream_t s = nullptr) {
    if (u.dims != g_u.dims || u.dims != out.dims || u.data.size() != st.m1.size())
        throw std::invalid_argument("adam_step: shape mismatch");
    const auto tg = gaussian_taps(sigma_grad), tw = gaussian_taps(sigma_warp);
    st.step += 1;
    check(ffdp_sobolev_adam(g_u.data.data(), u.data.data(), st.m1.data(), st.m2.data(), u.dims.c(),
                            full_slab(u.dims.nz), tg.data(), static_cast<int>(tg.size()), lr_norm, st.beta1,
                            st.beta2, st.eps, st.step, s));
    check(ffdp_gp_convolve(u.data.data(), out.data.data(), u.dims.c(), full_slab(u.dims.nz), 3, tw.data(),
                           static_cast<int>(tw.size()), 1, s));
}

// ------------------------------------------------------------------ multi-scale (resample.hpp:48-146)
inline Dims3 resample_dims(Dims3 d, double factor) {
    ffdp_dims o;
    check(ffdp_resample_dims(d.c(), factor, &o));
    return Dims3{o.nx, o.ny, o.nz};
}

// resample_scale (resample.hpp:48-103): anti-alias (factor < 1) + trilinear onto
// ceil(n * factor), first / last voxel centres kept (spacing rescaled like the reference).
inline Volume3 resample_scale(const Volume3& v, double factor, cudaStream_t s = nullptr) {
    const Dims3 nd = resample_dims(v.dims, factor);
    Volume3 out = Volume3::uninitialized(nd);
    for (int c = 0; c < 3; ++c) {
        const double ratio = static_cast<double>(v.dims[c] - 1) / static_cast<double>(nd[c] - 1);
        out.spacing[c] = v.dims[c] > 1 ? v.spacing[c] * ratio : v.spacing[c];
    }
    out.origin = v.origin;
    check(ffdp_resample_scale(v.data.data(), v.dims.c(), factor, out.data.data(), nullptr, s));
    return out;
}

// resample_warp (resample.hpp:108-146).
inline WarpField resample_warp(const WarpField& w, Dims3 nd, cudaStream_t s = nullptr) {
    if (!nd.positive()) throw std::invalid_argument("resample_warp: dims must be positive");
    WarpField out = WarpField::uninitialized(nd);
    check(ffdp_resample_warp(w.data.data(), w.dims.c(), out.data.data(), nd.c(), s));
    return out;
}

// normalize_intensities (registration.hpp:100-115).
inline Volume3 normalize_intensities(const Volume3& v, cudaStream_t s = nullptr) {
    Volume3 out = Volume3::uninitialized(v.dims);
    out.spacing = v.spacing;
    out.origin = v.origin;
    check(ffdp_normalize(v.data.data(), v.dims.voxels(), out.data.data(), s));
    return out;
}

// jacobian_positive_fraction (metrics.hpp:145-176).
inline double jacobian_positive_fraction(const WarpField& u, cudaStream_t s = nullptr) {
    double f = 0;
    check(ffdp_jacobian_positive(u.data.data(), u.dims.c(), &f, s));
    return f;
}

// ------------------------------------------------------------------ the driver (registration.hpp:48-331)
struct AffineMap {
    Mat3 matrix = Mat3::identity();
    Vec3 translation{{0, 0, 0}};
};

struct ScaleStep {
    double downsample = 1;  // 4 means quarter resolution
    int iterations = 0;
};

struct ScaleSchedule {
    std::vector<ScaleStep> steps;
    double lr = 0.5;
    double sigma_grad = 1.0;
    double sigma_warp = 0.5;
    LossParams loss;

    void validate() const {
        if (steps.empty()) throw std::invalid_argument("schedule: no scale steps");
        for (std::size_t i = 0; i < steps.size(); ++i) {
            if (!(steps[i].downsample >= 1)) throw std::invalid_argument("schedule: downsample factors must be >= 1");
            if (steps[i].iterations < 0) throw std::invalid_argument("schedule: iterations must be >= 0");
            if (i > 0 && steps[i].downsample > steps[i - 1].downsample)
                throw std::invalid_argument("schedule: factors must be non-increasing toward 1");
        }
        if (!(lr > 0) || !(sigma_grad >= 0) || !(sigma_warp >= 0))
            throw std::invalid_argument("schedule: bad lr/sigma");
    }
};

struct TraceEntry {
    int scale_index = 0;
    int iteration = 0;
    double loss = 0;
};

struct NumericalError : std::runtime_error {
    std::vector<TraceEntry> trace;
    NumericalError(const std::string& what, std::vector<TraceEntry> t)
        : std::runtime_error(what), trace(std::move(t)) {}
};

// loss_and_grad (registration.hpp:123-173) through the operator kernels: MSE (dist_mse),
// LNCC (lncc_forward_fused + lncc_backward_fused, upstream 1) or MI (exact / approximate
// forward + mi_backward_impl, upstream -1, loss = -MI). Returns the loss and dL/dmoved.
inline std::pair<double, Volume3> loss_and_grad(const Volume3& f, const Volume3& moved, const LossParams& p,
                                                cudaStream_t s = nullptr) {
    if (!f.same_lattice(moved)) throw std::invalid_argument("loss_and_grad: lattices differ");
    if (p.kind == LossKind::mse) {
        Volume3 g = Volume3::uninitialized(f.dims);
        DeviceArray<double> sum(1);
        sum.zero(s);
        check(ffdp_mse(f.data.data(), moved.data.data(), f.dims.voxels(), f.dims.voxels(), g.data.data(),
                       sum.data(), s));
        return {sum.download(s)[0] / static_cast<double>(f.dims.voxels()), std::move(g)};
    }
    if (p.kind == LossKind::lncc) {
        auto fw = lncc_forward_fused(f, moved, p.window, p.epsilon, false, s);
        auto bw = lncc_backward_fused(1.0, fw.second, f, moved, p.ants_approx, s);
        return {fw.first.loss, std::move(bw.second)};
    }
    const ParzenKernel k = p.mi_bspline_kernel ? ParzenKernel::bspline3(p.bins) : ParzenKernel::gaussian(p.bins);
    const MiResult r = p.mi_approx_forward ? mi_forward_approx(f, moved, p.bins, k, s)
                                           : mi_forward_exact(f, moved, p.bins, k, s);
    auto bw = detail::mi_backward_impl(-1.0, f, moved, r.hist, k, s);
    return {-r.mi, std::move(bw.second)};
}

// Whether DeformableStep's fused kernels cover the loss (else deformable_stage composes
// fused_sample -> loss_and_grad -> fused_sample_backward).
inline bool fused_loss(const LossParams& p) {
    // the fused kernels: LNCC window 7 (ANTs backward), MI with the exact Parzen forward
    return (p.kind == LossKind::lncc && p.ants_approx && p.window == 7) ||
           (p.kind == LossKind::mi && !p.mi_approx_forward);
}

// deformable_stage (registration.hpp:230-331) on one GPU: per scale resample F and M on
// the device, carry the warp over (resample_warp), build the fused step once (zero-
// bordered M + workspace) and iterate step -> warp_update. The loss is read every
// iteration (the reference's non-finite check and trace, 290-296).
inline WarpField deformable_stage(const Volume3& fixed, const Volume3& moving, const AffineMap& affine,
                                  const ScaleSchedule& schedule, std::vector<TraceEntry>* trace = nullptr,
                                  int scale_index_base = 0, cudaStream_t s = nullptr) {
    schedule.validate();
    if (!fixed.same_lattice(moving))
        throw std::invalid_argument("deformable_stage: F and M must share a lattice (registration.hpp:268-270)");
    SamplerArgs args;
    args.A = affine.matrix;
    args.t = affine.translation;
    std::optional<WarpField> warp;
    for (std::size_t sc = 0; sc < schedule.steps.size(); ++sc) {
        const auto& step = schedule.steps[sc];
        const double factor = 1.0 / step.downsample;
        std::optional<Volume3> fr, mr;
        if (factor != 1.0) {
            fr.emplace(resample_scale(fixed, factor, s));
            mr.emplace(resample_scale(moving, factor, s));
        }
        const Volume3& f_s = fr ? *fr : fixed;
        const Volume3& m_s = mr ? *mr : moving;
        warp = warp ? resample_warp(*warp, f_s.dims, s) : WarpField::zeros(f_s.dims, s);
        // registration.hpp:257-264: lr in voxels of the level -> normalized units
        const Dims3 d = f_s.dims;
        const double pitch = (2.0 / static_cast<double>(d.nx - 1) + 2.0 / static_cast<double>(d.ny - 1) +
                              2.0 / static_cast<double>(d.nz - 1)) / 3.0;
        const double lr_norm = schedule.lr * pitch;
        std::optional<DeformableStep> st;
        if (fused_loss(schedule.loss)) st.emplace(f_s, m_s, schedule.loss, s);
        AdamState adam = AdamState::zeros(warp->data.size(), s);
        WarpField g = WarpField::uninitialized(d), spare = WarpField::uninitialized(d);
        for (int it = 0; it < step.iterations; ++it) {
            StepResult r;
            if (st) {
                r = st->step(*warp, args, g, true);
            } else {
                // ring_sample -> loss -> ring_sample_backward(want warp) through the operators
                const Volume3 moved = fused_sample(m_s, &*warp, args, s);
                auto lg = loss_and_grad(f_s, moved, schedule.loss, s);
                r.loss = lg.first;
                SamplerGradWant want;
                want.warp = true;
                g = std::move(*fused_sample_backward(lg.second, m_s, &*warp, args, want, s).warp);
            }
            if (!std::isfinite(r.loss))
                throw NumericalError("deformable stage diverged (non-finite loss)",
                                     trace ? *trace : std::vector<TraceEntry>{});
            if (trace) trace->push_back({scale_index_base + static_cast<int>(sc), it, r.loss});
            warp_update(*warp, g, adam, lr_norm, spare, schedule.sigma_grad, schedule.sigma_warp, s);
            std::swap(*warp, spare);
        }
    }
    if (warp->dims != fixed.dims) warp = resample_warp(*warp, fixed.dims, s);
    return std::move(*warp);
}

// affine_stage (registration.hpp:176-219): Adam on the 12 affine parameters from the
// identity (state shared by all scales); per iteration moved = fused_sample(M_s, zero warp,
// A, t) on F_s's lattice, loss_and_grad, fused_sample_backward(want affine + translation).
inline AffineMap affine_stage(const Volume3& fixed, const Volume3& moving, const ScaleSchedule& schedule,
                              std::vector<TraceEntry>* trace = nullptr, int scale_index_base = 0,
                              cudaStream_t s = nullptr) {
    schedule.validate();
    AffineMap map;
    double m1[12] = {0}, m2[12] = {0};
    std::int64_t step_count = 0;
    for (std::size_t sc = 0; sc < schedule.steps.size(); ++sc) {
        const auto& step = schedule.steps[sc];
        const double factor = 1.0 / step.downsample;
        std::optional<Volume3> fr, mr;
        if (factor != 1.0) {
            fr.emplace(resample_scale(fixed, factor, s));
            mr.emplace(resample_scale(moving, factor, s));
        }
        const Volume3& f_s = fr ? *fr : fixed;
        const Volume3& m_s = mr ? *mr : moving;
        const WarpField zero = WarpField::zeros(f_s.dims, s);  // outputs on F's lattice
        for (int it = 0; it < step.iterations; ++it) {
            SamplerArgs args;
            args.A = map.matrix;
            args.t = map.translation;
            const Volume3 moved = fused_sample(m_s, &zero, args, s);
            auto lg = loss_and_grad(f_s, moved, schedule.loss, s);
            if (!std::isfinite(lg.first))
                throw NumericalError("affine stage diverged (non-finite loss)",
                                     trace ? *trace : std::vector<TraceEntry>{});
            if (trace) trace->push_back({scale_index_base + static_cast<int>(sc), it, lg.first});
            SamplerGradWant want;
            want.affine = want.translation = true;
            const SamplerGrads gr = fused_sample_backward(lg.second, m_s, &zero, args, want, s);
            // adam_step<double> on the 12 parameters (adam.hpp:30-50)
            double params[12], grad[12];
            for (int i = 0; i < 9; ++i) params[i] = map.matrix.m[i], grad[i] = gr.affine->m[i];
            for (int i = 0; i < 3; ++i) params[9 + i] = map.translation[i], grad[9 + i] = (*gr.translation)[i];
            ++step_count;
            const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
            const double c1 = 1.0 - std::pow(b1, static_cast<double>(step_count));
            const double c2 = 1.0 - std::pow(b2, static_cast<double>(step_count));
            for (int i = 0; i < 12; ++i) {
                m1[i] = b1 * m1[i] + (1.0 - b1) * grad[i];
                m2[i] = b2 * m2[i] + (1.0 - b2) * grad[i] * grad[i];
                params[i] -= schedule.lr * (m1[i] / c1) / (std::sqrt(m2[i] / c2) + eps);
            }
            for (int i = 0; i < 9; ++i) map.matrix.m[i] = params[i];
            for (int i = 0; i < 3; ++i) map.translation[i] = params[9 + i];
        }
    }
    return map;
}

// DeformableOptions (registration.hpp:221-226): shards > 1 runs the stage z-sharded over a
// WorkerGroup (one rank per visible device, round robin); gp_sync = false is the
// reference's halo-free smoothing ablation.
struct DeformableOptions {
    int shards = 1;
    bool gp_sync = true;
};

// deformable_stage with the reference's parameter order (registration.hpp:230-234), the
// stream as a trailing extra; defined after the sharded context below.
inline WarpField deformable_stage(const Volume3& fixed, const Volume3& moving, const AffineMap& affine,
                                  const ScaleSchedule& schedule, const DeformableOptions& opts,
                                  std::vector<TraceEntry>* trace = nullptr, int scale_index_base = 0,
                                  std::vector<std::int64_t>* worker_peak_bytes = nullptr, cudaStream_t s = nullptr);

// RegistrationConfig / RegistrationResult / register_volumes (registration.hpp:333-368).
struct RegistrationConfig {
    ScaleSchedule affine;
    ScaleSchedule deformable;
    DeformableOptions deformable_opts;
    bool skip_affine = false;
};

struct RegistrationResult {
    AffineMap affine;
    WarpField warp;
    std::vector<TraceEntry> trace;
    double jacobian_positive_fraction = 1.0;
};

inline RegistrationResult register_volumes(const Volume3& fixed, const Volume3& moving,
                                           const RegistrationConfig& config, cudaStream_t s = nullptr) {
    RegistrationResult res;
    const Volume3 f_n = normalize_intensities(fixed, s), m_n = normalize_intensities(moving, s);
    int base = 0;
    if (!config.skip_affine) {
        res.affine = affine_stage(f_n, m_n, config.affine, &res.trace, 0, s);
        base = static_cast<int>(config.affine.steps.size());
    }
    res.warp = deformable_stage(f_n, m_n, res.affine, config.deformable, config.deformable_opts, &res.trace, base,
                                nullptr, s);
    const Dims3 d = res.warp.dims;
    if (d.nx >= 3 && d.ny >= 3 && d.nz >= 3) res.jacobian_positive_fraction = jacobian_positive_fraction(res.warp, s);
    return res;
}

// ------------------------------------------------------------------ sharded context
// WorkerGroup(H) (fabric.hpp:266-300) as one process over H devices (ffdp_comm, DESIGN.md
// "Sharded context"): rank r's shards live on device(r) (devices may repeat); every
// collective runs all ranks in lock step. Shards follow shard_ranges (fabric.hpp:44-70).
class DeviceScope {
  public:
    explicit DeviceScope(int d) {
        cudaGetDevice(&prev_);
        check_cuda(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceScope() { cudaSetDevice(prev_); }

  private:
    int prev_ = 0;
};

class WorkerGroup {
  public:
    explicit WorkerGroup(int world, const std::vector<int>& devices = {}) {
        if (!devices.empty() && static_cast<int>(devices.size()) != world)
            throw std::invalid_argument("WorkerGroup: one device per rank");
        check(ffdp_comm_create(world, devices.empty() ? nullptr : devices.data(), &h_));
    }
    ~WorkerGroup() {
        if (h_) ffdp_comm_destroy(h_);
    }
    WorkerGroup(const WorkerGroup&) = delete;
    WorkerGroup& operator=(const WorkerGroup&) = delete;

    int world() const { return ffdp_comm_world(h_); }
    int device(int rank) const { return ffdp_comm_device(h_, rank); }
    ffdp_comm handle() const { return h_; }
    std::pair<std::int64_t, std::int64_t> shard_range(std::int64_t nz, int rank) const {
        std::int64_t lo = 0, hi = 0;
        check(ffdp_shard_range(nz, world(), rank, &lo, &hi));
        return {lo, hi};
    }
    // rank r's z slab of v / w, allocated on device(r)
    std::vector<Volume3> scatter(const Volume3& v) const {
        std::vector<Volume3> out;
        for (int r = 0; r < world(); ++r) {
            const auto [lo, hi] = shard_range(v.dims.nz, r);
            DeviceScope ds(device(r));
            Volume3 s = Volume3::uninitialized(Dims3{v.dims.nx, v.dims.ny, hi - lo});
            check_cuda(cudaMemcpy(s.data.data(), v.data.data() + lo * v.dims.nx * v.dims.ny,
                                  sizeof(float) * s.dims.voxels(), cudaMemcpyDefault), "scatter");
            out.push_back(std::move(s));
        }
        return out;
    }
    std::vector<WarpField> scatter(const WarpField& w) const {
        std::vector<WarpField> out;
        for (int r = 0; r < world(); ++r) {
            const auto [lo, hi] = shard_range(w.dims.nz, r);
            DeviceScope ds(device(r));
            WarpField s = WarpField::uninitialized(Dims3{w.dims.nx, w.dims.ny, hi - lo});
            check_cuda(cudaMemcpy(s.data.data(), w.data.data() + 3 * lo * w.dims.nx * w.dims.ny,
                                  sizeof(float) * 3 * s.dims.voxels(), cudaMemcpyDefault), "scatter");
            out.push_back(std::move(s));
        }
        return out;
    }
    // gather_volume / gather_warp (fabric.hpp:102-132): the global field on the current device
    template <class Field>
    Field gather(const std::vector<Field>& shards, Dims3 global) const {
        Field out = Field::uninitialized(global);
        const std::size_t per = out.data.size() / static_cast<std::size_t>(global.voxels());
        for (int r = 0; r < world(); ++r) {
            const auto lo = shard_range(global.nz, r).first;
            check_cuda(cudaMemcpy(out.data.data() + per * lo * global.nx * global.ny, shards[r].data.data(),
                                  sizeof(float) * shards[r].data.size(), cudaMemcpyDefault), "gather");
        }
        return out;
    }
    template <class Field>
    std::vector<Field> empty_like(Dims3 global) const {
        std::vector<Field> out;
        for (int r = 0; r < world(); ++r) {
            const auto [lo, hi] = shard_range(global.nz, r);
            DeviceScope ds(device(r));
            out.push_back(Field::uninitialized(Dims3{global.nx, global.ny, hi - lo}));
        }
        return out;
    }

  private:
    ffdp_comm h_ = nullptr;
};

namespace detail {
template <class Field>
std::vector<const float*> cptrs(const std::vector<Field>& v) {
    std::vector<const float*> p;
    for (const auto& x : v) p.push_back(x.data.data());
    return p;
}
template <class Field>
std::vector<float*> mptrs(std::vector<Field>& v) {
    std::vector<float*> p;
    for (auto& x : v) p.push_back(x.data.data());
    return p;
}
inline void check_world(const WorkerGroup& g, std::size_t n, const char* what) {
    if (static_cast<int>(n) != g.world()) throw std::invalid_argument(std::string(what) + ": one shard per rank");
}
}  // namespace detail

struct DistLoss {
    double loss = 0;
    std::vector<Volume3> grad_moved;
    std::int64_t mi_payload_elements = 0;
};

struct RingSampleGrads {
    std::optional<std::vector<Volume3>> image;
    std::optional<std::vector<WarpField>> warp;
    std::optional<Mat3> affine;
    std::optional<Vec3> translation;
};

// halo_exchange (fabric.hpp:315-370): per rank [pad planes of r-1 | slab | pad planes of r+1]
template <class Field>
std::vector<Field> halo_exchange(const WorkerGroup& g, const std::vector<Field>& slabs, Dims3 global, int pad) {
    detail::check_world(g, slabs.size(), "halo_exchange");
    const int ch = static_cast<int>(slabs[0].data.size() / static_cast<std::size_t>(slabs[0].dims.voxels()));
    std::vector<Field> out;
    for (int r = 0; r < g.world(); ++r) {
        const auto [lo, hi] = g.shard_range(global.nz, r);
        const std::int64_t a = r > 0 ? pad : 0, b = r < g.world() - 1 ? pad : 0;
        DeviceScope ds(g.device(r));
        out.push_back(Field::uninitialized(Dims3{global.nx, global.ny, std::max<std::int64_t>(1, hi - lo + a + b)}));
    }
    auto in = detail::cptrs(slabs);
    auto o = detail::mptrs(out);
    check(ffdp_halo_exchange(g.handle(), in.data(), global.c(), ch, pad, o.data(), nullptr, nullptr));
    return out;
}

// gp_convolve (distops.hpp:54-101) over the ranks' slabs
template <class Field>
std::vector<Field> gp_convolve(const WorkerGroup& g, const std::vector<Field>& slabs, Dims3 global,
                               const std::vector<double>& taps, EdgeMode mode = EdgeMode::zero_pad, bool sync = true) {
    detail::check_world(g, slabs.size(), "gp_convolve");
    const int ch = static_cast<int>(slabs[0].data.size() / static_cast<std::size_t>(slabs[0].dims.voxels()));
    auto out = g.template empty_like<Field>(global);
    auto in = detail::cptrs(slabs);
    auto o = detail::mptrs(out);
    check(ffdp_dist_gp_convolve(g.handle(), in.data(), global.c(), ch, taps.data(), static_cast<int>(taps.size()),
                                mode == EdgeMode::renormalize ? 1 : 0, sync ? 1 : 0, o.data()));
    return out;
}

// ring_sample (distops.hpp:144-168): the moved image on every rank's output slab
inline std::vector<Volume3> ring_sample(const WorkerGroup& g, const std::vector<Volume3>& m_shards, Dims3 m_global,
                                        const std::vector<WarpField>& u_shards, Dims3 out_global, const Mat3& A,
                                        const Vec3& t) {
    detail::check_world(g, m_shards.size(), "ring_sample");
    detail::check_world(g, u_shards.size(), "ring_sample");
    auto out = g.empty_like<Volume3>(out_global);
    auto m = detail::cptrs(m_shards);
    auto u = detail::cptrs(u_shards);
    auto o = detail::mptrs(out);
    check(ffdp_ring_sample(g.handle(), m.data(), m_global.c(), u.data(), out_global.c(), A.m, t.v, o.data()));
    return out;
}

// ring_sample_backward (distops.hpp:179-248)
inline RingSampleGrads ring_sample_backward(const WorkerGroup& g, const std::vector<Volume3>& upstream,
                                            const std::vector<Volume3>& m_shards, Dims3 m_global,
                                            const std::vector<WarpField>& u_shards, Dims3 out_global, const Mat3& A,
                                            const Vec3& t, const SamplerGradWant& want) {
    detail::check_world(g, upstream.size(), "ring_sample_backward");
    RingSampleGrads r;
    std::vector<float*> gi, gu;
    if (want.image) {
        r.image = g.empty_like<Volume3>(m_global);
        gi = detail::mptrs(*r.image);
    }
    if (want.warp) {
        r.warp = g.empty_like<WarpField>(out_global);
        gu = detail::mptrs(*r.warp);
    }
    double gat[12] = {0};
    auto up = detail::cptrs(upstream);
    auto m = detail::cptrs(m_shards);
    auto u = detail::cptrs(u_shards);
    check(ffdp_ring_sample_bwd(g.handle(), up.data(), m.data(), m_global.c(), u.data(), out_global.c(), A.m, t.v,
                               want.mask(), want.image ? gi.data() : nullptr, want.warp ? gu.data() : nullptr, gat));
    if (want.affine) {
        Mat3 a;
        std::memcpy(a.m, gat, sizeof(a.m));
        r.affine = a;
    }
    if (want.translation) r.translation = Vec3{{gat[9], gat[10], gat[11]}};
    return r;
}

inline DistLoss dist_mse(const WorkerGroup& g, const std::vector<Volume3>& f, const std::vector<Volume3>& moved,
                         Dims3 global, std::int64_t n_total = 0) {
    detail::check_world(g, f.size(), "dist_mse");
    DistLoss d;
    d.grad_moved = g.empty_like<Volume3>(global);
    auto a = detail::cptrs(f), b = detail::cptrs(moved);
    auto o = detail::mptrs(d.grad_moved);
    check(ffdp_dist_mse(g.handle(), a.data(), b.data(), global.c(), n_total > 0 ? n_total : global.voxels(), &d.loss,
                        o.data()));
    return d;
}

inline DistLoss dist_mi(const WorkerGroup& g, const std::vector<Volume3>& f, const std::vector<Volume3>& moved,
                        Dims3 global, const ParzenKernel& k, bool approx_forward = false, std::int64_t n_total = 0) {
    detail::check_world(g, f.size(), "dist_mi");
    DistLoss d;
    d.grad_moved = g.empty_like<Volume3>(global);
    auto a = detail::cptrs(f), b = detail::cptrs(moved);
    auto o = detail::mptrs(d.grad_moved);
    const ffdp_parzen kc = k.c();
    check(ffdp_dist_mi(g.handle(), a.data(), b.data(), global.c(), &kc, approx_forward ? 1 : 0,
                       n_total > 0 ? n_total : global.voxels(), &d.loss, o.data(), &d.mi_payload_elements));
    return d;
}

inline DistLoss dist_lncc(const WorkerGroup& g, const std::vector<Volume3>& f, const std::vector<Volume3>& moved,
                          Dims3 global, int window = 7, double eps = 1e-5, bool ants_approx = true, bool gp_sync = true,
                          std::int64_t n_total = 0) {
    detail::check_world(g, f.size(), "dist_lncc");
    DistLoss d;
    d.grad_moved = g.empty_like<Volume3>(global);
    auto a = detail::cptrs(f), b = detail::cptrs(moved);
    auto o = detail::mptrs(d.grad_moved);
    check(ffdp_dist_lncc(g.handle(), a.data(), b.data(), global.c(), window, eps, ants_approx ? 1 : 0, gp_sync ? 1 : 0,
                         n_total, &d.loss, o.data()));
    return d;
}

// The fused deformable step over the ranks (ffdp_dist_step): (loss, g_u slabs)
inline std::pair<double, std::vector<WarpField>> dist_step(const WorkerGroup& g, const std::vector<Volume3>& f,
                                                           const std::vector<Volume3>& m,
                                                           const std::vector<WarpField>& u, Dims3 global,
                                                           const SamplerArgs& args, const LossParams& p) {
    detail::check_world(g, f.size(), "dist_step");
    if (!fused_loss(p)) throw std::invalid_argument("dist_step: the fused step runs LNCC (ANTs, window 7) and exact MI");
    auto out = g.empty_like<WarpField>(global);
    auto a = detail::cptrs(f), b = detail::cptrs(m), c = detail::cptrs(u);
    auto o = detail::mptrs(out);
    ffdp_parzen kc{};
    if (p.kind == LossKind::mi)
        kc = (p.mi_bspline_kernel ? ParzenKernel::bspline3(p.bins) : ParzenKernel::gaussian(p.bins)).c();
    double loss = 0;
    check(ffdp_dist_step(g.handle(), p.kind == LossKind::lncc ? 0 : 1, a.data(), b.data(), c.data(), global.c(),
                         args.A.m, args.t.v, p.window, p.epsilon, p.kind == LossKind::mi ? &kc : nullptr, &loss,
                         o.data()));
    return {loss, std::move(out)};
}

// deformable_stage (registration.hpp:230-331) with DeformableOptions. shards == 1: the
// single-GPU stage above. shards > 1: per scale F_s, M_s and the carried warp are scattered
// into z slabs (shard_ranges), and per iteration every rank runs the reference's sequence
// over the group: the fused step (ffdp_dist_step) for LNCC / exact MI, else ring_sample ->
// dist_mse | dist_lncc | dist_mi -> ring_sample_backward(warp); then gp_convolve(g_u) (halo'd,
// or not with gp_sync = false), adam_step per rank and gp_convolve(u). worker_peak_bytes
// receives each rank device's used memory at the end of each scale.
inline WarpField deformable_stage(const Volume3& fixed, const Volume3& moving, const AffineMap& affine,
                                  const ScaleSchedule& schedule, const DeformableOptions& opts,
                                  std::vector<TraceEntry>* trace, int scale_index_base,
                                  std::vector<std::int64_t>* worker_peak_bytes, cudaStream_t s) {
    schedule.validate();
    if (opts.shards < 1) throw std::invalid_argument("deformable_stage: shards must be >= 1");
    if (schedule.loss.lncc_naive_backend && opts.shards > 1)
        throw std::invalid_argument("deformable_stage: the naive LNCC backend is single-worker");
    if (opts.shards == 1) {
        WarpField w = deformable_stage(fixed, moving, affine, schedule, trace, scale_index_base, s);
        if (worker_peak_bytes) {
            std::size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            worker_peak_bytes->push_back(static_cast<std::int64_t>(tot - fr));
        }
        return w;
    }
    if (!fixed.same_lattice(moving))
        throw std::invalid_argument("deformable_stage: F and M must share a lattice (registration.hpp:268-270)");
    int ndev = 1;
    check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    std::vector<int> devices;
    for (int r = 0; r < opts.shards; ++r) devices.push_back(r % std::max(1, ndev));
    WorkerGroup g(opts.shards, devices);
    const SamplerArgs args = [&] {
        SamplerArgs a;
        a.A = affine.matrix;
        a.t = affine.translation;
        return a;
    }();
    const auto taps_grad = gaussian_taps(schedule.sigma_grad), taps_warp = gaussian_taps(schedule.sigma_warp);
    std::optional<WarpField> warp;
    for (std::size_t sc = 0; sc < schedule.steps.size(); ++sc) {
        const auto& step = schedule.steps[sc];
        const double factor = 1.0 / step.downsample;
        std::optional<Volume3> fr, mr;
        if (factor != 1.0) {
            fr.emplace(resample_scale(fixed, factor, s));
            mr.emplace(resample_scale(moving, factor, s));
        }
        const Volume3& f_s = fr ? *fr : fixed;
        const Volume3& m_s = mr ? *mr : moving;
        warp = warp ? resample_warp(*warp, f_s.dims, s) : WarpField::zeros(f_s.dims, s);
        check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        const Dims3 d = f_s.dims;
        if (d.nz < opts.shards) throw std::invalid_argument("deformable_stage: fewer planes than shards");
        const double pitch = (2.0 / static_cast<double>(d.nx - 1) + 2.0 / static_cast<double>(d.ny - 1) +
                              2.0 / static_cast<double>(d.nz - 1)) / 3.0;
        const double lr_norm = schedule.lr * pitch;
        const std::vector<Volume3> f_sh = g.scatter(f_s), m_sh = g.scatter(m_s);
        std::vector<WarpField> u_sh = g.scatter(*warp);
        std::vector<AdamState> adam;
        for (int r = 0; r < opts.shards; ++r) {
            DeviceScope ds(g.device(r));
            adam.push_back(AdamState::zeros(u_sh[(std::size_t)r].data.size()));
        }
        std::vector<TraceEntry> scale_trace;
        for (int it = 0; it < step.iterations; ++it) {
            double loss = 0;
            std::vector<WarpField> g_u;
            if (fused_loss(schedule.loss)) {
                auto r = dist_step(g, f_sh, m_sh, u_sh, d, args, schedule.loss);
                loss = r.first;
                g_u = std::move(r.second);
            } else {
                const auto moved = ring_sample(g, m_sh, d, u_sh, d, args.A, args.t);
                DistLoss dl;
                const LossParams& p = schedule.loss;
                if (p.kind == LossKind::mse)
                    dl = dist_mse(g, f_sh, moved, d);
                else if (p.kind == LossKind::lncc)
                    dl = dist_lncc(g, f_sh, moved, d, p.window, p.epsilon, p.ants_approx, opts.gp_sync);
                else
                    dl = dist_mi(g, f_sh, moved, d,
                                 p.mi_bspline_kernel ? ParzenKernel::bspline3(p.bins) : ParzenKernel::gaussian(p.bins),
                                 p.mi_approx_forward);
                loss = dl.loss;
                SamplerGradWant want;
                want.warp = true;
                g_u = std::move(*ring_sample_backward(g, dl.grad_moved, m_sh, d, u_sh, d, args.A, args.t, want).warp);
            }
            if (!std::isfinite(loss))
                throw NumericalError("deformable stage diverged (non-finite loss)",
                                     trace ? *trace : std::vector<TraceEntry>{});
            scale_trace.push_back({scale_index_base + static_cast<int>(sc), it, loss});
            // registration.hpp:313-317 on the slabs: smoothed gradient (halo'd), Adam, smoothed warp
            auto g_s = gp_convolve(g, g_u, d, taps_grad, EdgeMode::renormalize, opts.gp_sync);
            for (int r = 0; r < opts.shards; ++r) {
                DeviceScope ds(g.device(r));
                adam_step(u_sh[(std::size_t)r], g_s[(std::size_t)r], adam[(std::size_t)r], lr_norm);
            }
            u_sh = gp_convolve(g, u_sh, d, taps_warp, EdgeMode::renormalize, opts.gp_sync);
        }
        warp = g.gather(u_sh, d);
        if (trace) trace->insert(trace->end(), scale_trace.begin(), scale_trace.end());
        if (worker_peak_bytes)
            for (int r = 0; r < opts.shards; ++r) {
                DeviceScope ds(g.device(r));
                std::size_t fr2 = 0, tot = 0;
                cudaMemGetInfo(&fr2, &tot);
                worker_peak_bytes->push_back(static_cast<std::int64_t>(tot - fr2));
            }
    }
    if (warp->dims != fixed.dims) warp = resample_warp(*warp, fixed.dims, s);
    return std::move(*warp);
}

}  // namespace voxreg
}  // namespace ffdp
