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
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

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

int main() {
    if (ffdp_device_check() != FFDP_OK) {
        std::printf("no usable sm_100 device: %s\n", ffdp_last_error());
        return 2;
    }
    sampler_tests();
    lncc_tests();
    mi_tests();
    step_tests();
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
