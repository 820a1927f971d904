// C++ parity suite for include/ffdp/voxreg.hpp (the host mirror of the voxreg operator
// API over libffdp.so), written the way the reference's GTest suites are
// (proj/tests/test_sampler.cpp, test_lncc.cpp, test_mi.cpp): every GPU result is checked
// against the C oracle (oracle/ffdp_oracle.c, TEST INFRASTRUCTURE, pinned to the
// reference by tests/test_oracle_golden.py) on the same fp32-rounded inputs, and the
// reference's EXPECT_THROW cases are checked against the mirror's exceptions.
//
// Built by paper_2509_25044_b200/build.py (tests/cpp/test_voxreg_api), run by
// tests/test_cpp_api.py on a GPU. Exit code 0 = all checks passed.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "ffdp/nifti.hpp"
#include "ffdp/voxreg.hpp"

// ---------------------------------------------------------------- oracle (C, fp64)
extern "C" {
typedef struct {
    int64_t nx, ny, nz;
} or_dims;
typedef struct {
    uint64_t state;
    int have_spare;
    double spare;
} or_rng;
typedef struct {
    int kind, bins;
    double sigma, radius, norm;
} or_parzen;
void or_rng_init(or_rng* r, uint64_t seed);
double or_rng_uniform(or_rng* r);
int or_sample_core(const double* img, or_dims idims, const double* u, or_dims odims, const double* A, const double* t,
                   const double* S, const double* bounds, double* out, const double* upstream, double* g_img,
                   double* g_u, double* gA, double* gt, double* abs_accum);
double or_lncc_forward(const double* f, const double* m, or_dims dims, int window, double eps, double* state,
                       double* map);
void or_lncc_backward(double upstream, double* state, const double* f, const double* m, or_dims dims, int window,
                      double eps, int ants, double* grad_f, double* grad_m);
int or_parzen_make(int kind, int bins, double sigma_bins, or_parzen* k);
int or_mi_forward_exact(const double* vi, const double* vj, int64_t n, const or_parzen* k, double* raw,
                        uint64_t* stats);
double or_mi_finalize(const double* raw_joint, int b, double* p_ij, double* p_i, double* p_j, double* z_out);
void or_mi_ghat(double upstream, const double* p_ij, const double* p_i, const double* p_j, double z, int b,
                double* ghat);
void or_mi_backward(const double* vi, const double* vj, int64_t n, const or_parzen* k, const double* ghat,
                    double* grad_i, double* grad_j);
int or_synth_pair(uint64_t seed, or_dims d, int k, double max_disp, double* fixed, double* moving,
                  double* true_warp);
void or_normalize_intensities(double* v, int64_t n);
void or_separable_convolve(double* data, or_dims dims, int channels, const double* taps, int ntaps, int mode);
void or_adam_step(double* param, const double* grad, double* m1, double* m2, int64_t n, double lr, double beta1,
                  double beta2, double eps, int64_t step);
int or_resample_scale(const double* in, or_dims d, double factor, double* out, or_dims* out_dims);
int or_affine_stage(const double* fixed, const double* moving, or_dims d, int nsteps, const double* downsample,
                    const int* iterations, double lr, int loss_kind, int window, double eps, int ants, int bins,
                    int mi_kind, double* A_out, double* t_out, double* trace);
int or_deformable_stage(const double* fixed, const double* moving, or_dims d, const double* A, const double* t,
                        int nsteps, const double* downsample, const int* iterations, double lr, double sigma_grad,
                        double sigma_warp, int loss_kind, int window, double eps, int ants, int bins, int mi_kind,
                        double* warp_out, double* trace);
double or_step_lncc(const double* f, const double* m, or_dims d, const double* u, const double* A, const double* t,
                    int window, double eps, int ants, double* g_u, double* moved_out, double* grad_moved_out);
double or_step_mi(const double* f, const double* m, or_dims d, const double* u, const double* A, const double* t,
                  const or_parzen* k, int approx, double* g_u, double* moved_out, double* grad_moved_out,
                  double* raw_out);
}

namespace V = ffdp::voxreg;

// ---------------------------------------------------------------- a tiny test runner
static int g_failed = 0, g_checks = 0;
static std::string g_test;

#define EXPECT_TRUE(c)                                                                        \
    do {                                                                                      \
        ++g_checks;                                                                           \
        if (!(c)) {                                                                           \
            ++g_failed;                                                                       \
            std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_test.c_str(), #c); \
        }                                                                                     \
    } while (0)

#define EXPECT_THROW(stmt, ex)                                                                          \
    do {                                                                                                \
        ++g_checks;                                                                                     \
        bool caught_ = false;                                                                           \
        try {                                                                                           \
            stmt;                                                                                       \
        } catch (const ex&) {                                                                           \
            caught_ = true;                                                                             \
        } catch (...) {                                                                                 \
        }                                                                                               \
        if (!caught_) {                                                                                 \
            ++g_failed;                                                                                 \
            std::printf("  FAIL %s:%d [%s] expected %s from %s\n", __FILE__, __LINE__, g_test.c_str(), \
                        #ex, #stmt);                                                                    \
        }                                                                                               \
    } while (0)

static void run(const char* name, const std::function<void()>& fn) {
    g_test = name;
    const int before = g_failed;
    try {
        fn();
    } catch (const std::exception& e) {
        ++g_failed;
        std::printf("  FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_failed == before ? "ok  " : "FAIL", name);
}

// max|a-b| / max|b|
static double maxrel(const std::vector<float>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < b.size(); ++i) {
        num = std::max(num, std::fabs(double(a[i]) - b[i]));
        den = std::max(den, std::fabs(b[i]));
    }
    return den > 0 ? num / den : num;
}

static double rel(double a, double b) { return std::fabs(a - b) / std::max(std::fabs(b), 1e-300); }

// ---------------------------------------------------------------- fixtures
struct Pair {
    or_dims d;
    std::vector<float> f, m, u;       // fp32 inputs (what the GPU sees)
    std::vector<double> fd, md, ud;   // the same values in fp64 (what the oracle sees)
    double A[9], t[3];
};

static std::vector<double> widen(const std::vector<float>& v) { return std::vector<double>(v.begin(), v.end()); }

// synth_pair (synth.hpp) + normalize (registration.hpp:100-115); u = half the true warp +
// U(-jit, jit); A = I + U(-0.02, 0.02), t = U(-0.02, 0.02) (SURVEY.md 8(d) recipe).
static Pair make_pair(int nx, int ny, int nz, uint64_t seed, bool mi_remap, double jit = 0.01) {
    Pair p;
    p.d = {nx, ny, nz};
    const int64_t n = int64_t(nx) * ny * nz;
    std::vector<double> f(n), m(n), w(3 * n);
    if (or_synth_pair(seed, p.d, 5, 0.12, f.data(), m.data(), w.data())) throw std::runtime_error("synth_pair");
    or_normalize_intensities(f.data(), n);
    or_normalize_intensities(m.data(), n);
    or_rng r;
    or_rng_init(&r, seed + 17);
    if (mi_remap) {
        for (auto& v : m) v = 4.0 * v * (1.0 - v) + 0.02 * (2.0 * or_rng_uniform(&r) - 1.0);
        or_normalize_intensities(m.data(), n);
    }
    for (int64_t i = 0; i < 3 * n; ++i) w[i] = 0.5 * w[i] + jit * (2.0 * or_rng_uniform(&r) - 1.0);
    for (int i = 0; i < 9; ++i) p.A[i] = (i % 4 == 0 ? 1.0 : 0.0) + 0.04 * or_rng_uniform(&r) - 0.02;
    for (int i = 0; i < 3; ++i) p.t[i] = 0.04 * or_rng_uniform(&r) - 0.02;
    p.f.assign(f.begin(), f.end());
    p.m.assign(m.begin(), m.end());
    p.u.assign(w.begin(), w.end());
    p.fd = widen(p.f), p.md = widen(p.m), p.ud = widen(p.u);
    return p;
}

static V::Dims3 dims(const or_dims& d) { return V::Dims3{d.nx, d.ny, d.nz}; }

static V::SamplerArgs args_of(const Pair& p, const double S[3] = nullptr) {
    V::SamplerArgs a;
    for (int i = 0; i < 9; ++i) a.A.m[i] = p.A[i];
    for (int i = 0; i < 3; ++i) a.t[i] = p.t[i];
    if (S)
        for (int i = 0; i < 3; ++i) a.S[i] = S[i];
    return a;
}

// ---------------------------------------------------------------- sampler (test_sampler.cpp)
static void sampler_tests() {
    run("sampler: fused_sample matches the oracle (affine + S + warp)", [] {
        Pair p = make_pair(24, 20, 18, 101, false);
        const double S[3] = {1.25, 0.8, 1.1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
        auto img = V::Volume3::from_host(dims(p.d), p.m.data());
        auto u = V::WarpField::from_host(dims(p.d), p.u.data());
        auto out = V::fused_sample(img, &u, args_of(p, S));
        std::vector<double> ref(p.md.size(), 0.0);
        or_sample_core(p.md.data(), p.d, p.ud.data(), p.d, p.A, p.t, S, bounds, ref.data(), nullptr, nullptr,
                       nullptr, nullptr, nullptr, nullptr);
        EXPECT_TRUE(maxrel(out.to_host(), ref) <= 1e-5);
    });
    run("sampler: fused_sample_accumulate adds and reports the L1 contribution", [] {
        Pair p = make_pair(20, 18, 16, 102, false);
        const double S[3] = {1, 1, 1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
        auto img = V::Volume3::from_host(dims(p.d), p.m.data());
        auto u = V::WarpField::from_host(dims(p.d), p.u.data());
        auto out = V::fused_sample(img, &u, args_of(p));
        double l1 = 0;
        V::fused_sample_accumulate(img, &u, args_of(p), out, &l1);
        std::vector<double> ref(p.md.size(), 0.0);
        double l1_ref = 0;
        or_sample_core(p.md.data(), p.d, p.ud.data(), p.d, p.A, p.t, S, bounds, ref.data(), nullptr, nullptr,
                       nullptr, nullptr, nullptr, &l1_ref);
        for (auto& v : ref) v *= 2.0;
        EXPECT_TRUE(maxrel(out.to_host(), ref) <= 1e-5);
        EXPECT_TRUE(rel(l1, l1_ref) <= 1e-5);
    });
    run("sampler: fused_sample_backward (image, warp, affine, translation) matches the oracle", [] {
        Pair p = make_pair(22, 18, 16, 103, false);
        const double S[3] = {1.25, 0.8, 1.1}, bounds[6] = {-1, -1, -1, 1, 1, 1};
        const int64_t n = p.d.nx * p.d.ny * p.d.nz;
        std::vector<float> g(n);
        or_rng r;
        or_rng_init(&r, 7);
        for (auto& v : g) v = float(2.0 * or_rng_uniform(&r) - 1.0);
        auto img = V::Volume3::from_host(dims(p.d), p.m.data());
        auto u = V::WarpField::from_host(dims(p.d), p.u.data());
        auto up = V::Volume3::from_host(dims(p.d), g.data());
        V::SamplerGradWant want{true, true, true, true};
        auto gr = V::fused_sample_backward(up, img, &u, args_of(p, S), want);
        std::vector<double> gd = widen(g), gi(n, 0.0), gu(3 * n, 0.0), gA(9, 0.0), gt(3, 0.0);
        or_sample_core(p.md.data(), p.d, p.ud.data(), p.d, p.A, p.t, S, bounds, nullptr, gd.data(), gi.data(),
                       gu.data(), gA.data(), gt.data(), nullptr);
        EXPECT_TRUE(gr.image && gr.warp && gr.affine && gr.translation);
        EXPECT_TRUE(maxrel(gr.image->to_host(), gi) <= 1e-4);
        EXPECT_TRUE(maxrel(gr.warp->to_host(), gu) <= 1e-4);
        std::vector<float> a(gr.affine->m, gr.affine->m + 9), tt{float((*gr.translation)[0]),
                                                                   float((*gr.translation)[1]),
                                                                   float((*gr.translation)[2])};
        EXPECT_TRUE(maxrel(a, gA) <= 1e-4);
        EXPECT_TRUE(maxrel(tt, gt) <= 1e-4);
    });
    run("sampler: identity args reproduce the image (test_sampler.cpp:81-87)", [] {
        Pair p = make_pair(17, 19, 16, 104, false);
        auto img = V::Volume3::from_host(dims(p.d), p.m.data());
        auto out = V::fused_sample(img, nullptr, V::SamplerArgs{});
        EXPECT_TRUE(maxrel(out.to_host(), p.md) <= 1e-6);
    });
    run("sampler: rejects (test_sampler.cpp:267-277)", [] {
        Pair p = make_pair(16, 16, 16, 105, false);
        auto img = V::Volume3::from_host(dims(p.d), p.m.data());
        V::SamplerArgs bad;
        bad.S[1] = 0.0;
        EXPECT_THROW(V::fused_sample(img, nullptr, bad), std::invalid_argument);
        V::SamplerArgs nan;
        nan.A.m[4] = NAN;
        EXPECT_THROW(V::fused_sample(img, nullptr, nan), std::invalid_argument);
        auto wrong = V::Volume3::zeros(V::Dims3{8, 8, 8});
        EXPECT_THROW(V::fused_sample_accumulate(img, nullptr, V::SamplerArgs{}, wrong), std::invalid_argument);
        EXPECT_THROW(V::fused_sample_backward(wrong, img, nullptr, V::SamplerArgs{}, V::SamplerGradWant{}),
                     std::invalid_argument);
    });
}

// ---------------------------------------------------------------- LNCC (test_lncc.cpp)
static void lncc_tests() {
    for (int ants = 0; ants <= 1; ++ants) {
        run(ants ? "lncc: forward + ANTs backward match the oracle" : "lncc: forward + exact backward match the oracle",
            [ants] {
                Pair p = make_pair(20, 18, 16, 211 + ants, false);
                const int64_t n = p.d.nx * p.d.ny * p.d.nz;
                auto f = V::Volume3::from_host(dims(p.d), p.f.data());
                auto m = V::Volume3::from_host(dims(p.d), p.m.data());
                auto fr = V::lncc_forward_fused(f, m, 7, 1e-5, true);
                std::vector<double> st(5 * n), map(n), gf(n), gm(n);
                const double loss = or_lncc_forward(p.fd.data(), p.md.data(), p.d, 7, 1e-5, st.data(), map.data());
                EXPECT_TRUE(rel(fr.first.loss, loss) <= 1e-5);
                EXPECT_TRUE(fr.first.has_map && maxrel(fr.first.ncc_map->to_host(), map) <= 1e-4);
                auto g = V::lncc_backward_fused(1.0, fr.second, f, m, ants != 0);
                or_lncc_backward(1.0, st.data(), p.fd.data(), p.md.data(), p.d, 7, 1e-5, ants, gf.data(), gm.data());
                EXPECT_TRUE(maxrel(g.first.to_host(), gf) <= 1e-4);
                EXPECT_TRUE(maxrel(g.second.to_host(), gm) <= 1e-4);
            });
    }
    run("lncc: rejects (lncc.hpp:57-61)", [] {
        auto a = V::Volume3::zeros(V::Dims3{8, 8, 8}), b = V::Volume3::zeros(V::Dims3{8, 8, 9});
        EXPECT_THROW(V::lncc_forward_fused(a, b, 7, 1e-5), std::invalid_argument);
        EXPECT_THROW(V::lncc_forward_fused(a, a, 4, 1e-5), std::invalid_argument);
    });
}

// ---------------------------------------------------------------- MI (test_mi.cpp)
static void mi_tests() {
    run("mi: exact B-spline forward + backward match the oracle (32 bins)", [] {
        Pair p = make_pair(24, 20, 18, 311, true);
        const int64_t n = p.d.nx * p.d.ny * p.d.nz;
        auto i = V::Volume3::from_host(dims(p.d), p.f.data());
        auto j = V::Volume3::from_host(dims(p.d), p.m.data());
        auto k = V::ParzenKernel::bspline3(32);
        auto r = V::mi_forward_exact(i, j, 32, k);
        or_parzen ok;
        or_parzen_make(1, 32, 0.5, &ok);
        std::vector<double> raw(32 * 32 + 64), pij(32 * 32), pi(32), pj(32), gh(32 * 32), gi(n), gj(n);
        uint64_t stats[2] = {0, 0};
        or_mi_forward_exact(p.fd.data(), p.md.data(), n, &ok, raw.data(), stats);
        double z;
        const double mi = or_mi_finalize(raw.data(), 32, pij.data(), pi.data(), pj.data(), &z);
        EXPECT_TRUE(rel(r.mi, mi) <= 1e-5);
        EXPECT_TRUE(r.stats.hist_writes == stats[0] && r.stats.kernel_evals == stats[1]);
        EXPECT_TRUE(r.hist.samples == n && r.hist.bins == 32);
        auto g = V::mi_backward(-1.0, i, j, r.hist, k);
        or_mi_ghat(-1.0, pij.data(), pi.data(), pj.data(), z, 32, gh.data());
        or_mi_backward(p.fd.data(), p.md.data(), n, &ok, gh.data(), gi.data(), gj.data());
        EXPECT_TRUE(maxrel(g.first.to_host(), gi) <= 1e-4);
        EXPECT_TRUE(maxrel(g.second.to_host(), gj) <= 1e-4);
    });
    run("mi: rejects and kernel checks (mi.hpp:132,170-179,430-437)", [] {
        std::vector<float> v(512, 0.5f);
        v[3] = 1.5f;
        auto a = V::Volume3::from_host(V::Dims3{8, 8, 8}, v.data());
        auto k = V::ParzenKernel::bspline3(16);
        auto z = V::Volume3::zeros(V::Dims3{8, 8, 8});
        EXPECT_THROW(V::mi_forward_exact(a, z, 16, k), std::invalid_argument);
        EXPECT_THROW(V::mi_forward_exact(z, z, 8, k), std::invalid_argument);
        EXPECT_THROW(V::ParzenKernel::bspline3(0), std::invalid_argument);
        auto r = V::mi_forward_exact(z, z, 16, k);
        auto small = V::Volume3::zeros(V::Dims3{4, 4, 4});
        EXPECT_THROW(V::mi_backward(-1.0, small, small, r.hist, k), std::invalid_argument);
    });
}

// ---------------------------------------------------------------- the fused step
static void step_tests() {
    run("step: DeformableStep LNCC (ANTs) matches the oracle step", [] {
        Pair p = make_pair(32, 28, 24, 4242, false);
        const int64_t n = p.d.nx * p.d.ny * p.d.nz;
        auto f = V::Volume3::from_host(dims(p.d), p.f.data());
        auto m = V::Volume3::from_host(dims(p.d), p.m.data());
        auto u = V::WarpField::from_host(dims(p.d), p.u.data());
        auto g = V::WarpField::uninitialized(dims(p.d));
        V::LossParams lp;
        V::DeformableStep step(f, m, lp);
        auto r = step.step(u, args_of(p), g);
        std::vector<double> gu(3 * n);
        const double loss = or_step_lncc(p.fd.data(), p.md.data(), p.d, p.ud.data(), p.A, p.t, 7, 1e-5, 1, gu.data(),
                                         nullptr, nullptr);
        EXPECT_TRUE(rel(r.loss, loss) <= 1e-5);
        EXPECT_TRUE(maxrel(g.to_host(), gu) <= 1e-4);
        EXPECT_TRUE(r.window_misses == 0);
    });
    run("step: DeformableStep MI (B-spline, 32 bins) matches the oracle step", [] {
        Pair p = make_pair(32, 28, 24, 4243, true);
        const int64_t n = p.d.nx * p.d.ny * p.d.nz;
        auto f = V::Volume3::from_host(dims(p.d), p.f.data());
        auto m = V::Volume3::from_host(dims(p.d), p.m.data());
        auto u = V::WarpField::from_host(dims(p.d), p.u.data());
        auto g = V::WarpField::uninitialized(dims(p.d));
        V::LossParams lp;
        lp.kind = V::LossKind::mi;
        lp.mi_bspline_kernel = true;
        V::DeformableStep step(f, m, lp);
        auto r = step.step(u, args_of(p), g);
        or_parzen ok;
        or_parzen_make(1, 32, 0.5, &ok);
        std::vector<double> gu(3 * n);
        const double loss =
            or_step_mi(p.fd.data(), p.md.data(), p.d, p.ud.data(), p.A, p.t, &ok, 0, gu.data(), nullptr, nullptr, nullptr);
        EXPECT_TRUE(rel(r.loss, loss) <= 1e-5);
        EXPECT_TRUE(maxrel(g.to_host(), gu) <= 1e-4);
        // repeated steps are bit-identical (fixed-point histogram: no atomic-order dependence)
        std::vector<float> g1 = g.to_host();
        auto r2 = step.step(u, args_of(p), g);
        EXPECT_TRUE(r2.loss == r.loss && g.to_host() == g1);
    });
    run("step: rejects (registration.hpp:268-270, sampler lattice)", [] {
        auto f = V::Volume3::zeros(V::Dims3{16, 16, 16}), m = V::Volume3::zeros(V::Dims3{16, 16, 17});
        EXPECT_THROW(V::DeformableStep(f, m, V::LossParams{}), std::invalid_argument);
        V::LossParams exact;
        exact.ants_approx = false;
        EXPECT_THROW(V::DeformableStep(f, f, exact), std::invalid_argument);
        V::DeformableStep s(f, f, V::LossParams{});
        auto u = V::WarpField::zeros(V::Dims3{16, 16, 15}), g = V::WarpField::zeros(V::Dims3{16, 16, 16});
        EXPECT_THROW(s.step(u, V::SamplerArgs{}, g), std::invalid_argument);
    });
}

// ---------------------------------------------------------------- the warp update and the driver
static std::vector<float> uniform_f32(uint64_t seed, size_t n, double lo, double hi) {
    or_rng r;
    or_rng_init(&r, seed);
    std::vector<float> v(n);
    for (auto& x : v) x = float(lo + (hi - lo) * or_rng_uniform(&r));
    return v;
}

static void driver_tests() {
    run("smoothing: gp_convolve (box zero_pad, gaussian renormalize) matches the oracle", [] {
        const or_dims d{37, 19, 11};
        const size_t n = size_t(d.nx * d.ny * d.nz);
        for (int ch : {1, 3}) {
            auto h = uniform_f32(901 + ch, n * ch, -1, 1);
            for (int mode = 0; mode < 2; ++mode) {
                const auto taps = mode ? V::gaussian_taps(1.0) : V::box_taps(7);
                std::vector<double> ref = widen(h);
                or_separable_convolve(ref.data(), d, ch, taps.data(), int(taps.size()), mode);
                const auto em = mode ? V::EdgeMode::renormalize : V::EdgeMode::zero_pad;
                std::vector<float> got;
                if (ch == 1)
                    got = V::gp_convolve(V::Volume3::from_host(dims(d), h.data()), taps, em).to_host();
                else
                    got = V::gp_convolve(V::WarpField::from_host(dims(d), h.data()), taps, em).to_host();
                EXPECT_TRUE(maxrel(got, ref) <= 1e-6);
            }
        }
        EXPECT_THROW(V::box_taps(4), std::invalid_argument);
        EXPECT_THROW(V::gaussian_taps(-1.0), std::invalid_argument);
    });
    run("adam: adam_step (adam.hpp:30-50) matches the oracle over 3 steps", [] {
        const or_dims d{34, 9, 5};
        const size_t n = size_t(3 * d.nx * d.ny * d.nz);
        auto p = uniform_f32(911, n, -1, 1);
        std::vector<double> pr = widen(p), ar(n, 0.0), br(n, 0.0);
        auto param = V::WarpField::from_host(dims(d), p.data());
        auto st = V::AdamState::zeros(n);
        for (int k = 1; k <= 3; ++k) {
            auto g = uniform_f32(920 + k, n, -1, 1);
            std::vector<double> gd = widen(g);
            or_adam_step(pr.data(), gd.data(), ar.data(), br.data(), int64_t(n), 0.01, 0.9, 0.999, 1e-8, k);
            V::adam_step(param, V::WarpField::from_host(dims(d), g.data()), st, 0.01);
        }
        EXPECT_TRUE(st.step == 3);
        EXPECT_TRUE(maxrel(param.to_host(), pr) <= 1e-6);
        EXPECT_TRUE(maxrel(st.m1.download(), ar) <= 1e-6 && maxrel(st.m2.download(), br) <= 1e-6);
    });
    run("multi-scale: resample_scale (resample.hpp:48-103) matches the oracle", [] {
        const or_dims d{45, 34, 21};
        auto h = uniform_f32(931, size_t(d.nx * d.ny * d.nz), 0, 1);
        std::vector<double> hd = widen(h);
        for (double f : {0.5, 0.25, 2.0}) {
            or_dims od;
            or_resample_scale(hd.data(), d, f, nullptr, &od);
            std::vector<double> ref(size_t(od.nx * od.ny * od.nz));
            or_resample_scale(hd.data(), d, f, ref.data(), &od);
            auto got = V::resample_scale(V::Volume3::from_host(dims(d), h.data()), f);
            EXPECT_TRUE(got.dims == dims(od));
            EXPECT_TRUE(maxrel(got.to_host(), ref) <= 2e-6);
        }
        EXPECT_THROW(V::resample_scale(V::Volume3::zeros(dims(d)), 0.0), std::invalid_argument);
    });
    for (int mi = 0; mi < 2; ++mi) {
        run(mi ? "driver: deformable_stage MI (B-spline) matches the oracle stage"
               : "driver: deformable_stage LNCC matches the oracle stage",
            [mi] {
                Pair p = make_pair(22, 20, 18, 4242, mi == 1);
                const int64_t n = p.d.nx * p.d.ny * p.d.nz;
                const double ds[2] = {2, 1};
                const int its[2] = {3, 3};
                std::vector<double> wref(size_t(3 * n)), tref(6);
                // lr 0.5 voxels overshoots on this MI pair (the MI falls after the first update
                // and oscillates -- the reference does the same); 0.1 keeps the dynamics
                // non-chaotic so fp32 vs fp64 stays comparable over the iterations
                const double lr = mi ? 0.1 : 0.5;
                const int rc = or_deformable_stage(p.fd.data(), p.md.data(), p.d, p.A, p.t, 2, ds, its, lr, 1.0, 0.5,
                                                   mi, 7, 1e-5, 1, 32, 1, wref.data(), tref.data());
                EXPECT_TRUE(rc == 0);
                V::ScaleSchedule sch;
                sch.steps = {V::ScaleStep{2, 3}, V::ScaleStep{1, 3}};
                sch.loss.kind = mi ? V::LossKind::mi : V::LossKind::lncc;
                sch.loss.mi_bspline_kernel = true;
                sch.lr = lr;
                V::AffineMap aff;
                for (int i = 0; i < 9; ++i) aff.matrix.m[i] = p.A[i];
                for (int i = 0; i < 3; ++i) aff.translation[i] = p.t[i];
                std::vector<V::TraceEntry> trace;
                auto w = V::deformable_stage(V::Volume3::from_host(dims(p.d), p.f.data()),
                                             V::Volume3::from_host(dims(p.d), p.m.data()), aff, sch, &trace);
                EXPECT_TRUE(trace.size() == 6);
                double tr = 0;
                for (size_t i = 0; i < trace.size() && i < 6; ++i) tr = std::max(tr, rel(trace[i].loss, tref[i]));
                EXPECT_TRUE(tr <= 1e-5);
                // warp: l2 and per-voxel bounds in units of one Adam step (below)
                const auto wh = w.to_host();
                double num = 0, den = 0, mx = 0;
                for (size_t i = 0; i < wref.size(); ++i) {
                    const double dd = double(wh[i]) - wref[i];
                    num += dd * dd;
                    den += wref[i] * wref[i];
                    mx = std::max(mx, std::fabs(dd));
                }
                const double step = lr * (2.0 / 21 + 2.0 / 19 + 2.0 / 17) / 3.0;
                std::printf("  stage %s: trace rel %.3g, warp l2 %.3g, max/step %.3g\n", mi ? "mi" : "lncc", tr,
                            std::sqrt(num / den), mx / step);
                // Adam's step is sign-like where the smoothed gradient is near zero, so fp32 vs
                // fp64 (or one fp32 path vs another) differ there by a fraction of one step,
                // whatever the gradient accuracy: l2 1e-3, every voxel within a quarter step
                EXPECT_TRUE(std::sqrt(num / den) <= 1e-3);
                EXPECT_TRUE(mx <= 0.25 * step);
            });
    }
    for (int kind = 0; kind < 3; ++kind) {
        run(kind == 0 ? "driver: affine_stage MSE matches the oracle"
                      : kind == 1 ? "driver: affine_stage LNCC matches the oracle" : "driver: affine_stage MI matches the oracle",
            [kind] {
                Pair p = make_pair(22, 20, 18, 4242, true);
                const double ds[2] = {2, 1};
                const int its[2] = {3, 3};
                double A[9], t[3], tr[6];
                EXPECT_TRUE(or_affine_stage(p.fd.data(), p.md.data(), p.d, 2, ds, its, 0.01, kind, 7, 1e-5, 1, 32, 0, A,
                                            t, tr) == 0);
                V::ScaleSchedule sch;
                sch.steps = {V::ScaleStep{2, 3}, V::ScaleStep{1, 3}};
                sch.lr = 0.01;
                sch.loss.kind = kind == 0 ? V::LossKind::mse : kind == 1 ? V::LossKind::lncc : V::LossKind::mi;
                std::vector<V::TraceEntry> trace;
                const V::AffineMap a = V::affine_stage(V::Volume3::from_host(dims(p.d), p.f.data()),
                                                       V::Volume3::from_host(dims(p.d), p.m.data()), sch, &trace);
                EXPECT_TRUE(trace.size() == 6);
                double e = 0;
                for (size_t i = 0; i < trace.size() && i < 6; ++i) e = std::max(e, rel(trace[i].loss, tr[i]));
                EXPECT_TRUE(e <= 1e-5);
                double da = 0;
                for (int i = 0; i < 9; ++i) da = std::max(da, std::fabs(a.matrix.m[i] - A[i]));
                for (int i = 0; i < 3; ++i) da = std::max(da, std::fabs(a.translation[i] - t[i]));
                EXPECT_TRUE(da <= 1e-5);
            });
    }
    run("driver: register_volumes (affine + deformable, MSE deformable through loss_and_grad)", [] {
        Pair p = make_pair(22, 20, 18, 4243, false);
        V::RegistrationConfig cfg;
        cfg.affine.steps = {V::ScaleStep{2, 2}};
        cfg.affine.lr = 0.01;
        cfg.affine.loss.kind = V::LossKind::mi;
        cfg.deformable.steps = {V::ScaleStep{2, 2}, V::ScaleStep{1, 2}};
        cfg.deformable.loss.kind = V::LossKind::mse;
        auto f = V::Volume3::from_host(dims(p.d), p.f.data()), m = V::Volume3::from_host(dims(p.d), p.m.data());
        const auto r = V::register_volumes(f, m, cfg);
        EXPECT_TRUE(r.trace.size() == 6 && r.trace[2].scale_index == 1 && r.trace[5].scale_index == 2);
        EXPECT_TRUE(r.warp.dims == f.dims);
        EXPECT_TRUE(r.jacobian_positive_fraction > 0.5 && r.jacobian_positive_fraction <= 1.0);
        bool finite = true;
        for (const auto& e : r.trace) finite = finite && std::isfinite(e.loss);
        EXPECT_TRUE(finite);
    });
    run("driver: schedule rejects (registration.hpp:60-72)", [] {
        V::ScaleSchedule sch;
        EXPECT_THROW(sch.validate(), std::invalid_argument);
        sch.steps = {V::ScaleStep{1, 2}, V::ScaleStep{2, 2}};
        EXPECT_THROW(sch.validate(), std::invalid_argument);
        sch.steps = {V::ScaleStep{1, 2}};
        sch.lr = 0;
        EXPECT_THROW(sch.validate(), std::invalid_argument);
    });
}

// ---------------------------------------------------------------- NIfTI / warp IO
static std::string gold_dir() {
    const char* e = std::getenv("FFDP_GOLDEN_NIFTI");
    return e ? e : "tests/golden/nifti";
}

static std::vector<unsigned char> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    return std::vector<unsigned char>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

static void io_tests() {
    run("io: reference-written NIfTI read back; write_nifti byte-identical (nifti.hpp:99-239)", [] {
        const std::string d = gold_dir();
        const auto a = V::read_nifti(d + "/vol_f32.nii");
        const auto be = V::read_nifti(d + "/vol_be.nii");
        EXPECT_TRUE(!a.header.big_endian && be.header.big_endian);
        EXPECT_TRUE(a.dims == be.dims && a.data == be.data);
        EXPECT_TRUE(a.dims == (V::Dims3{7, 5, 3}) && std::fabs(a.spacing[2] - 2.5) < 1e-6);
        const auto lab = V::read_nifti(d + "/labels.nii"), sc = V::read_nifti(d + "/scaled_i16.nii");
        bool scaled = lab.data.size() == sc.data.size();
        for (size_t i = 0; scaled && i < lab.data.size(); ++i) scaled = sc.data[i] == 0.5 * lab.data[i] - 3.0;
        EXPECT_TRUE(scaled);
        // device round trip: write the fp32 volume back, byte for byte the reference's file
        auto v = a.to_device();
        V::write_nifti(v, "/tmp/ffdp_io_test.nii");
        EXPECT_TRUE(slurp("/tmp/ffdp_io_test.nii") == slurp(d + "/vol_f32.nii"));
        std::vector<unsigned char> bad = slurp(d + "/vol_f32.nii");
        bad[344] = 'x';
        EXPECT_THROW(V::read_nifti_bytes(bad), V::FormatError);
        EXPECT_THROW(V::read_nifti("/nonexistent/x.nii"), V::IoError);
    });
    run("io: raw + JSON warp (nifti.hpp:268-303) round trip", [] {
        const std::string d = gold_dir();
        auto w = V::read_warp(d + "/warp");
        EXPECT_TRUE(w.dims == (V::Dims3{5, 4, 3}));
        V::Vec3 sp{{0.7, 1.1, 2.5}}, og{{-10.0, 4.5, 0.25}};
        V::write_warp(w, "/tmp/ffdp_io_warp", sp, og);
        // the device field is fp32: the written payload is the reference's fp64 values
        // rounded to float, and nothing else
        const auto mine = slurp("/tmp/ffdp_io_warp.raw"), ref = slurp(d + "/warp.raw");
        bool same = mine.size() == ref.size();
        for (size_t i = 0; same && i + 8 <= ref.size(); i += 8) {
            double a, b;
            std::memcpy(&a, mine.data() + i, 8);
            std::memcpy(&b, ref.data() + i, 8);
            same = a == double(float(b));
        }
        EXPECT_TRUE(same);
        auto w2 = V::read_warp("/tmp/ffdp_io_warp");
        EXPECT_TRUE(w2.to_host() == w.to_host());
    });
}

// ---------------------------------------------------------------- sharded context (test_distops.cpp)
static double maxrel_f(const std::vector<float>& a, const std::vector<float>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, (double)std::fabs(a[i] - b[i]));
        den = std::max(den, (double)std::fabs(b[i]));
    }
    return den > 0 ? num / den : num;
}

static void comm_tests() {
    run("WorkerGroup collectives = single GPU (2 and 3 ranks on one device)", [] {
        const Pair p = make_pair(22, 19, 17, 611, false);
        const V::Dims3 d = dims(p.d);
        auto f = V::Volume3::from_host(d, p.f.data()), m = V::Volume3::from_host(d, p.m.data());
        auto u = V::WarpField::from_host(d, p.u.data());
        const V::SamplerArgs a = args_of(p);
        const auto moved = V::fused_sample(m, &u, a);
        for (int world : {2, 3}) {
            V::WorkerGroup g(world, std::vector<int>(world, 0));
            EXPECT_TRUE(g.world() == world && g.device(world - 1) == 0);
            auto fs = g.scatter(f), ms = g.scatter(m);
            auto us = g.scatter(u);
            auto mv = V::ring_sample(g, ms, d, us, d, a.A, a.t);
            EXPECT_TRUE(maxrel_f(g.gather(mv, d).to_host(), moved.to_host()) <= 1e-6);
            // halo'd Sobolev smoothing equals the whole-volume convolution bit for bit
            const auto taps = V::gaussian_taps(1.0);
            const auto gs = V::gp_convolve(g, us, d, taps, V::EdgeMode::renormalize);
            EXPECT_TRUE(g.gather(gs, d).to_host() == V::gp_convolve(u, taps, V::EdgeMode::renormalize).to_host());
            // distributed LNCC on the moved slabs vs the fused operator on the whole volume
            auto ref = V::lncc_forward_fused(f, moved, 7, 1e-5);
            const auto rg = V::lncc_backward_fused(1.0, ref.second, f, moved, true).second;
            const auto dl = V::dist_lncc(g, fs, mv, d);
            EXPECT_TRUE(rel(dl.loss, ref.first.loss) <= 1e-6);
            EXPECT_TRUE(maxrel_f(g.gather(dl.grad_moved, d).to_host(), rg.to_host()) <= 1e-5);
            // the fused sharded step vs the single-GPU fused step
            V::LossParams lp;
            V::DeformableStep st(f, m, lp);
            auto g1 = V::WarpField::uninitialized(d);
            const auto r1 = st.step(u, a, g1);
            const auto ds = V::dist_step(g, fs, ms, us, d, a, lp);
            EXPECT_TRUE(rel(ds.first, r1.loss) <= 1e-5);
            EXPECT_TRUE(maxrel_f(g.gather(ds.second, d).to_host(), g1.to_host()) <= 1e-4);
        }
        // deformable_stage with DeformableOptions (the reference's parameter order): shards 2 / 3
        // over a WorkerGroup sharing device 0 against the single-GPU stage, every loss kind
        for (int kind = 0; kind < 3; ++kind) {
            Pair p = make_pair(22, 20, 18, 4242, kind == 2);
            V::ScaleSchedule sch;
            sch.steps = {V::ScaleStep{2, 2}, V::ScaleStep{1, 2}};
            sch.loss.kind = kind == 0 ? V::LossKind::lncc : kind == 1 ? V::LossKind::mse : V::LossKind::mi;
            sch.loss.mi_bspline_kernel = true;
            sch.lr = 0.1;
            V::AffineMap aff;
            for (int i = 0; i < 9; ++i) aff.matrix.m[i] = p.A[i];
            for (int i = 0; i < 3; ++i) aff.translation[i] = p.t[i];
            const auto F = V::Volume3::from_host(dims(p.d), p.f.data()), M = V::Volume3::from_host(dims(p.d), p.m.data());
            std::vector<V::TraceEntry> t1;
            const auto w1 = V::deformable_stage(F, M, aff, sch, V::DeformableOptions{}, &t1).to_host();
            for (int shards : {2, 3}) {
                std::vector<V::TraceEntry> tn;
                std::vector<std::int64_t> peaks;
                V::DeformableOptions o;
                o.shards = shards;
                const auto wn = V::deformable_stage(F, M, aff, sch, o, &tn, 0, &peaks).to_host();
                double tr = 0;
                for (size_t i = 0; i < t1.size(); ++i) tr = std::max(tr, rel(tn[i].loss, t1[i].loss));
                std::printf("  sharded stage kind %d H=%d: trace rel %.3g, warp maxrel %.3g\n", kind, shards, tr,
                            maxrel_f(wn, w1));
                EXPECT_TRUE(tn.size() == t1.size() && tr <= 1e-5);
                EXPECT_TRUE(maxrel_f(wn, w1) <= 1e-3);
                EXPECT_TRUE(peaks.size() == size_t(2 * shards));
            }
        }
        {
            V::DeformableOptions bad;
            bad.shards = 0;
            V::ScaleSchedule sch;
            sch.steps = {V::ScaleStep{1, 1}};
            EXPECT_THROW(V::deformable_stage(V::Volume3::zeros(V::Dims3{8, 8, 8}), V::Volume3::zeros(V::Dims3{8, 8, 8}),
                                             V::AffineMap{}, sch, bad),
                         std::invalid_argument);
        }
        EXPECT_THROW(V::WorkerGroup(2, std::vector<int>{0}), std::invalid_argument);
        EXPECT_THROW(V::WorkerGroup(2, std::vector<int>{0, 99}), std::invalid_argument);
        V::WorkerGroup g3(3, std::vector<int>(3, 0));
        auto thin = g3.scatter(V::Volume3::zeros(V::Dims3{5, 4, 7}));  // thicknesses 3, 2, 2
        EXPECT_THROW(V::halo_exchange(g3, thin, V::Dims3{5, 4, 7}, 3), std::invalid_argument);
    });
}

int main() {
    if (ffdp_device_check() != FFDP_OK) {
        std::printf("no usable sm_100 device: %s\n", ffdp_last_error());
        return 2;
    }
    sampler_tests();
    lncc_tests();
    mi_tests();
    step_tests();
    driver_tests();
    io_tests();
    comm_tests();
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
