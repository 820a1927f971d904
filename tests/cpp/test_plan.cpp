// test_plan.cpp -- the native sharded plan (ffdp_plan_*) from C++, one std::thread per rank
// (the reference's WorkerGroup(H) model, fabric.hpp:266-300), against the single-GPU fused
// step (ffdp::voxreg::DeformableStep). In-process groups of 1-4 ranks share device 0; the
// NCCL group runs at world 1 here and at world 2 when two devices are visible
// (ncclCommInitRank from one unique id, one thread per device). Prints "<n> passed, <m>
// failed"; tests/test_cpp_api.py runs it on the GPU box.
#include <ffdp/voxreg.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

namespace F = ffdp::voxreg;

static int g_pass = 0, g_fail = 0;
static void expect(bool ok, const std::string& what) {
    (ok ? g_pass : g_fail)++;
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
}

// smooth synthetic pair on a (nz, ny, nx) lattice: F blobs + texture, M = F shifted, u small
struct Pair {
    F::Dims3 d;
    std::vector<float> f, m, u;
};
static Pair make_pair(int nx, int ny, int nz, bool mi) {
    Pair p;
    p.d = F::Dims3{nx, ny, nz};
    const size_t n = (size_t)nx * ny * nz;
    p.f.resize(n);
    p.m.resize(n);
    p.u.resize(3 * n);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const double X = -1 + 2.0 * x / (nx - 1), Y = -1 + 2.0 * y / (ny - 1), Z = -1 + 2.0 * z / (nz - 1);
                auto img = [](double a, double b, double c) {
                    const double r = a * a / 0.4 + b * b / 0.3 + c * c / 0.5;
                    return 1.0 / (1.0 + std::exp(8.0 * (r - 1.0))) + 0.05 * std::sin(7 * a) * std::sin(5 * b + 1) * std::sin(3 * c);
                };
                const size_t i = ((size_t)z * ny + y) * nx + x;
                const double fv = img(X, Y, Z);
                double mv = img(X + 0.05 * std::sin(2 * Y), Y + 0.04 * std::cos(3 * Z), Z - 0.03);
                if (mi) mv = 4.0 * mv * (1.0 - mv);
                p.f[i] = (float)(0.5 + 0.45 * fv);
                p.m[i] = (float)std::min(1.0, std::max(0.0, 0.5 + 0.45 * mv));
                p.u[3 * i] = (float)(0.01 * std::sin(3 * X + Y));
                p.u[3 * i + 1] = (float)(0.01 * std::cos(2 * Y - Z));
                p.u[3 * i + 2] = (float)(0.008 * std::sin(X * Z * 4));
            }
    return p;
}

static const double kA[9] = {1.01, 0.01, -0.005, -0.008, 0.995, 0.01, 0.004, -0.006, 1.003};
static const double kT[3] = {0.01, -0.008, 0.006};

struct Result {
    double loss = 0;
    std::vector<float> g_u;
};

static Result single_gpu(const Pair& p, bool mi) {
    cudaSetDevice(0);
    F::Volume3 f = F::Volume3::from_host(p.d, p.f.data()), m = F::Volume3::from_host(p.d, p.m.data());
    F::WarpField u = F::WarpField::from_host(p.d, p.u.data()), g = F::WarpField::uninitialized(p.d);
    F::LossParams lp;
    lp.kind = mi ? F::LossKind::mi : F::LossKind::lncc;
    lp.mi_bspline_kernel = true;
    F::DeformableStep step(f, m, lp);
    F::SamplerArgs a;
    std::memcpy(a.A.m, kA, sizeof(kA));
    for (int c = 0; c < 3; ++c) a.t[c] = kT[c];
    Result r;
    r.loss = step.step(u, a, g).loss;
    r.g_u = g.to_host();
    return r;
}

// every rank of `groups` on its own thread: plan, load its slabs, set u, one checked step
static Result sharded(const Pair& p, bool mi, const std::vector<ffdp_group>& groups, const std::vector<int>& dev,
                      int margin = 8) {
    const int w = (int)groups.size();
    std::vector<Result> part((size_t)w);
    std::vector<int64_t> lo((size_t)w), hi((size_t)w);
    std::vector<std::string> err((size_t)w);
    auto rank = [&](int r) {
        try {
            cudaSetDevice(dev[(size_t)r]);
            ffdp_plan_params pp;
            std::memset(&pp, 0, sizeof(pp));
            pp.loss_kind = mi ? 1 : 0;
            pp.window = 7;
            pp.eps = 1e-5;
            F::check(ffdp_parzen_make(FFDP_PARZEN_BSPLINE3, 32, 0.5, &pp.kernel));
            std::memcpy(pp.A, kA, sizeof(kA));
            std::memcpy(pp.t, kT, sizeof(kT));
            pp.margin_planes = margin;
            pp.records = 1;
            pp.overlap = 1;
            ffdp_plan pl;
            F::check(ffdp_plan_create(groups[(size_t)r], p.d.c(), &pp, &pl));
            F::check(ffdp_plan_slab(pl, &lo[(size_t)r], &hi[(size_t)r]));
            const size_t plane = (size_t)p.d.nx * p.d.ny, off = (size_t)lo[(size_t)r] * plane;
            const size_t cnt = (size_t)(hi[(size_t)r] - lo[(size_t)r]) * plane;
            F::check(ffdp_plan_load(pl, p.f.data() + off, p.m.data() + off));  // host slabs
            F::check_cuda(cudaMemcpyAsync(ffdp_plan_u(pl), p.u.data() + 3 * off, 3 * cnt * sizeof(float),
                                          cudaMemcpyHostToDevice, (cudaStream_t)ffdp_plan_stream(pl)),
                          "u H2D");
            F::check(ffdp_plan_step(pl, 1, &part[(size_t)r].loss));
            part[(size_t)r].g_u.resize(3 * cnt);
            F::check_cuda(cudaMemcpy(part[(size_t)r].g_u.data(), ffdp_plan_g_u(pl), 3 * cnt * sizeof(float),
                                     cudaMemcpyDeviceToHost),
                          "g_u D2H");
            F::check(ffdp_plan_destroy(pl));
        } catch (const std::exception& e) {
            err[(size_t)r] = e.what();
        }
    };
    std::vector<std::thread> th;
    for (int r = 0; r < w; ++r) th.emplace_back(rank, r);
    for (auto& t : th) t.join();
    for (int r = 0; r < w; ++r)
        if (!err[(size_t)r].empty()) throw std::runtime_error("rank " + std::to_string(r) + ": " + err[(size_t)r]);
    Result out;
    out.loss = part[0].loss;
    for (int r = 0; r < w; ++r) {
        if (part[(size_t)r].loss != out.loss) throw std::runtime_error("ranks disagree on the loss");
        out.g_u.insert(out.g_u.end(), part[(size_t)r].g_u.begin(), part[(size_t)r].g_u.end());
    }
    return out;
}

static double maxrel(const std::vector<float>& a, const std::vector<float>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, (double)std::fabs(a[i] - b[i]));
        den = std::max(den, (double)std::fabs(b[i]));
    }
    return den > 0 ? num / den : num;
}

int main() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        std::printf("no device\n0 passed, 1 failed\n");
        return 1;
    }
    for (int mi = 0; mi <= 1; ++mi) {
        const char* name = mi ? "mi" : "lncc";
        const Pair p = make_pair(40, 36, 64, mi);  // 92160 voxels: the MI quad path on one GPU too
        const Result ref = single_gpu(p, mi);
        std::vector<float> h1;
        for (int w : {1, 2, 3, 4}) {
            try {
                std::vector<ffdp_group> g((size_t)w);
                std::vector<int> dev((size_t)w, 0);
                F::check(ffdp_group_local(w, dev.data(), g.data()));
                const Result r = sharded(p, mi, g, dev);
                for (auto x : g) ffdp_group_destroy(x);
                const double lrel = std::fabs(r.loss - ref.loss) / std::fabs(ref.loss);
                const double grel = maxrel(r.g_u, ref.g_u);
                char buf[160];
                std::snprintf(buf, sizeof(buf), "%s local group H=%d vs single GPU: loss rel %.2e, g_u maxrel %.2e", name,
                              w, lrel, grel);
                expect(lrel <= 1e-9 && grel <= 1e-6, buf);
                if (w == 1) h1 = r.g_u;
                else expect(r.g_u == h1, std::string(name) + " local group H=" + std::to_string(w) + " bit-identical to H=1");
            } catch (const std::exception& e) {
                expect(false, std::string(name) + " local group H=" + std::to_string(w) + ": " + e.what());
            }
        }
        // NCCL: world 1 on device 0, world 2 over two devices when present
        int ver = 0;
        if (ffdp_nccl_version(&ver) != FFDP_OK) {
            std::printf("SKIP NCCL: %s\n", ffdp_last_error());
            continue;
        }
        for (int w : {1, 2}) {
            if (w > ndev) {
                std::printf("SKIP %s NCCL world %d: %d device(s)\n", name, w, ndev);
                continue;
            }
            try {
                unsigned char id[FFDP_NCCL_ID_BYTES];
                F::check(ffdp_nccl_unique_id(id));
                std::vector<ffdp_group> g((size_t)w);
                std::vector<int> dev((size_t)w);
                std::vector<std::thread> th;
                std::vector<int> rc((size_t)w, 0);
                for (int r = 0; r < w; ++r) {
                    dev[(size_t)r] = r;
                    th.emplace_back([&, r] {
                        cudaSetDevice(r);
                        rc[(size_t)r] = ffdp_group_nccl(id, w, r, r, &g[(size_t)r]);
                    });
                }
                for (auto& t : th) t.join();
                for (int r = 0; r < w; ++r) F::check(rc[(size_t)r]);
                const Result r = sharded(p, mi, g, dev);
                for (auto x : g) ffdp_group_destroy(x);
                expect(r.g_u == h1, std::string(name) + " NCCL world " + std::to_string(w) + " (v" +
                                        std::to_string(ver) + ") bit-identical to the local group");
            } catch (const std::exception& e) {
                expect(false, std::string(name) + " NCCL world " + std::to_string(w) + ": " + e.what());
            }
        }
    }
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
