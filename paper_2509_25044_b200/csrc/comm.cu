// The sharded context of the C ABI: one process drives H ranks, each a z slab on its own
// device (fabric.hpp:138-300 / distops.hpp:54-396 run H worker threads over shared
// memory; here a rank is a device and a stream, and the exchanges are peer copies over
// NVLink / NVSwitch). Several ranks may name the same device (tests on one GPU).
//
// Every collective takes arrays of `world` per-rank device pointers (rank r's on
// devices[r]) and runs all ranks in lock step, so the reference's "every rank calls in
// the same order" rule holds by construction. Shards follow shard_ranges
// (fabric.hpp:44-70): the first nz mod H ranks get one extra plane. Reductions are
// rank-ordered (fabric.hpp:246-263), so results are deterministic for a given H.
//
// The ops compose the library's operator kernels exactly as paper_2509_25044_b200/dist.py
// does over torch.distributed; DESIGN.md "Sharded context" has the mapping.
#include <algorithm>
#include <cstring>
#include <vector>

#include "ffdp_common.cuh"

struct ffdp_comm_s {
    int world = 0;
    std::vector<int> dev;
    std::vector<cudaStream_t> st;
};

namespace ffdp {
namespace comm {

// restores the caller's device on every exit path
struct DeviceGuard {
    int prev = 0;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// A device allocation of one rank, stream-ordered on the rank's stream (from the library's
// own pool of that device, device_pool, which keeps freed blocks cached: repeated
// collectives reuse memory instead of paying cudaMalloc / cudaFree), freed on scope exit. Every collective
// synchronises its ranks before returning, so the frees never overtake a reader.
struct Buf {
    void* p = nullptr;
    int dev = 0;
    cudaStream_t st = nullptr;
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p(o.p), dev(o.dev), st(o.st) { o.p = nullptr; }
    ~Buf() {
        if (p) {
            cudaSetDevice(dev);
            cudaFreeAsync(p, st);
        }
    }
    int alloc(const ffdp_comm_s* c, int rank, size_t bytes, bool zero) {
        dev = c->dev[rank];
        st = c->st[rank];
        cudaSetDevice(dev);
        const size_t n = std::max<size_t>(bytes, 16);
        cudaMemPool_t pool = device_pool(dev);
        if (!pool || cudaMallocFromPoolAsync(&p, n, pool, st) != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return set_error(FFDP_CUDA, "comm: device allocation of %zu bytes failed", bytes);
        }
        if (zero && cudaMemsetAsync(p, 0, n, st) != cudaSuccess) return set_error(FFDP_CUDA, "comm: memset failed");
        return FFDP_OK;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

#define COMM_TRY(expr)                    \
    do {                                  \
        const int rc_ = (expr);           \
        if (rc_ != FFDP_OK) return rc_;   \
    } while (0)

void range(int64_t n, int w, int r, int64_t& lo, int64_t& hi) {
    const int64_t base = n / w, rem = n % w;
    lo = r * base + std::min<int64_t>(r, rem);
    hi = lo + base + (r < rem ? 1 : 0);
}

double axis_coord(int64_t i, int64_t n) { return n <= 1 ? -1.0 : -1.0 + 2.0 * ((double)i / (double)(n - 1)); }

int check_comm(const ffdp_comm_s* c) {
    if (!c || c->world < 1) return set_error(FFDP_INVALID_ARGUMENT, "comm: null or destroyed context");
    return FFDP_OK;
}

int check_ptrs(const void* const* p, int w, const char* what) {
    if (!p) return set_error(FFDP_INVALID_ARGUMENT, "%s: null pointer array", what);
    for (int r = 0; r < w; ++r)
        if (!p[r]) return set_error(FFDP_INVALID_ARGUMENT, "%s: null pointer for rank %d", what, r);
    return FFDP_OK;
}

int check_global(ffdp_dims g, int w, const char* what) {
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) return set_error(FFDP_INVALID_ARGUMENT, "%s: dims must be positive", what);
    if (g.nz < w) return set_error(FFDP_INVALID_ARGUMENT, "%s: %lld planes for %d shards", what, (long long)g.nz, w);
    return FFDP_OK;
}

int sync_all(const ffdp_comm_s* c) {
    for (int r = 0; r < c->world; ++r) {
        cudaSetDevice(c->dev[r]);
        const cudaError_t e = cudaStreamSynchronize(c->st[r]);
        if (e != cudaSuccess) return set_error(FFDP_CUDA, "comm: rank %d: %s", r, cudaGetErrorString(e));
    }
    return FFDP_OK;
}

int copy(const ffdp_comm_s* c, int dst_rank, void* dst, int src_rank, const void* src, size_t bytes) {
    if (!bytes) return FFDP_OK;
    cudaSetDevice(c->dev[dst_rank]);
    const cudaError_t e = cudaMemcpyPeerAsync(dst, c->dev[dst_rank], src, c->dev[src_rank], bytes, c->st[dst_rank]);
    if (e != cudaSuccess) return set_error(FFDP_CUDA, "comm: peer copy: %s", cudaGetErrorString(e));
    return FFDP_OK;
}

__global__ void k_sum_rows(const double* __restrict__ rows, int nrows, int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nrows; ++r) s += rows[r * n + i];  // rank order (fabric.hpp:246-263)
        out[i] = s;
    }
}

__global__ void k_add_f32(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8LL * num_sms())); }

// In-place rank-ordered sum of `n` doubles per rank (allreduce_sum): rows staged on rank
// 0's device, summed in rank order, copied back to every rank. Inputs must be complete
// (callers synchronise the producing streams first).
int allreduce_f64(const ffdp_comm_s* c, double* const* bufs, int64_t n) {
    const int w = c->world;
    if (w == 1 || n == 0) return FFDP_OK;
    Buf rows;
    COMM_TRY(rows.alloc(c, 0, sizeof(double) * n * w, false));
    for (int r = 0; r < w; ++r) COMM_TRY(copy(c, 0, rows.as<double>() + r * n, r, bufs[r], sizeof(double) * n));
    cudaSetDevice(c->dev[0]);
    k_sum_rows<<<grid_for(n), 256, 0, c->st[0]>>>(rows.as<double>(), w, n, bufs[0]);
    COMM_TRY(check_launch("comm allreduce"));
    COMM_TRY(sync_all(c));
    for (int r = 1; r < w; ++r) COMM_TRY(copy(c, r, bufs[r], 0, bufs[0], sizeof(double) * n));
    return sync_all(c);
}

struct Shard {
    int64_t lo, hi;
    int64_t th() const { return hi - lo; }
};

std::vector<Shard> shards(int64_t nz, int w) {
    std::vector<Shard> s((size_t)w);
    for (int r = 0; r < w; ++r) range(nz, w, r, s[(size_t)r].lo, s[(size_t)r].hi);
    return s;
}

// Halo exchange into fresh buffers: out[r] = [lo_r planes of r-1 | slab r | hi_r planes of r+1].
int halo(const ffdp_comm_s* c, const float* const* slabs, ffdp_dims g, int ch, int pad, std::vector<Buf>& out,
         std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
    const int w = c->world;
    const auto sh = shards(g.nz, w);
    const int64_t plane = g.nx * g.ny * ch;
    for (int r = 0; r < w; ++r) {
        if (pad > 0 && r > 0 && pad > sh[(size_t)r - 1].th())
            return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: pad exceeds left neighbor thickness");
        if (pad > 0 && r < w - 1 && pad > sh[(size_t)r + 1].th())
            return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: pad exceeds right neighbor thickness");
    }
    out.clear();
    out.resize((size_t)w);
    lo.assign((size_t)w, 0);
    hi.assign((size_t)w, 0);
    for (int r = 0; r < w; ++r) {
        lo[(size_t)r] = r > 0 ? pad : 0;
        hi[(size_t)r] = r < w - 1 ? pad : 0;
        const int64_t th = sh[(size_t)r].th();
        COMM_TRY(out[(size_t)r].alloc(c, r, sizeof(float) * plane * (th + lo[(size_t)r] + hi[(size_t)r]), false));
        float* o = out[(size_t)r].as<float>();
        COMM_TRY(copy(c, r, o + lo[(size_t)r] * plane, r, slabs[r], sizeof(float) * plane * th));
        if (lo[(size_t)r])  // the left neighbour's last planes
            COMM_TRY(copy(c, r, o, r - 1, slabs[r - 1] + (sh[(size_t)r - 1].th() - pad) * plane,
                          sizeof(float) * plane * pad));
        if (hi[(size_t)r])  // the right neighbour's first planes
            COMM_TRY(copy(c, r, o + (lo[(size_t)r] + th) * plane, r + 1, slabs[r + 1], sizeof(float) * plane * pad));
    }
    return sync_all(c);
}

ffdp_sampler_args shard_args(const double* A, const double* t, const Shard& s, int64_t nz) {
    ffdp_sampler_args a;
    for (int i = 0; i < 9; ++i) a.A[i] = A ? A[i] : (i % 4 == 0 ? 1.0 : 0.0);
    for (int i = 0; i < 3; ++i) {
        a.t[i] = t ? t[i] : 0.0;
        a.S[i] = 1.0;
        a.x_min[i] = -1.0;
        a.x_max[i] = 1.0;
    }
    a.x_min[2] = axis_coord(s.lo, nz);
    a.x_max[2] = axis_coord(s.hi - 1, nz);
    return a;
}

// The moving planes rank r's samples touch (exact z extent of its u slab), gathered from
// their owners: the dense planes and their zero-bordered (pad = 2) copy.
struct Window {
    Buf planes, padded;
    int64_t z0 = 0, z1 = 0;
};

int moving_windows(const ffdp_comm_s* c, const float* const* m_shards, ffdp_dims mg, const float* const* u_shards,
                   ffdp_dims og, const std::vector<ffdp_sampler_args>& args, std::vector<Window>& win) {
    const int w = c->world;
    const auto msh = shards(mg.nz, w), osh = shards(og.nz, w);
    const int64_t plane = mg.nx * mg.ny;
    std::vector<Buf> ext((size_t)w);
    for (int r = 0; r < w; ++r) {
        COMM_TRY(ext[(size_t)r].alloc(c, r, 2 * sizeof(int64_t), false));
        const ffdp_dims od{og.nx, og.ny, osh[(size_t)r].th()};
        COMM_TRY(ffdp_sampler_z_extent(u_shards[r], od, mg, &args[(size_t)r], ext[(size_t)r].as<int64_t>(), c->st[r]));
    }
    COMM_TRY(sync_all(c));
    win.clear();
    win.resize((size_t)w);
    for (int r = 0; r < w; ++r) {
        int64_t e[2];
        cudaSetDevice(c->dev[r]);
        FFDP_CHECK_CUDA(cudaMemcpy(e, ext[(size_t)r].p, sizeof(e), cudaMemcpyDeviceToHost));
        Window& W = win[(size_t)r];
        W.z0 = e[0] <= e[1] ? std::max<int64_t>(0, e[0]) : 0;
        W.z1 = e[0] <= e[1] ? std::min<int64_t>(mg.nz, e[1] + 1) : 0;
        W.z1 = std::max(W.z1, W.z0);
        const int64_t nzw = W.z1 - W.z0;
        COMM_TRY(W.planes.alloc(c, r, sizeof(float) * plane * nzw, false));
        COMM_TRY(W.padded.alloc(c, r, sizeof(float) * (mg.nx + 4) * (mg.ny + 4) * (nzw + 4), nzw == 0));
        for (int s = 0; s < w; ++s) {  // the owners' planes inside the window
            const int64_t a = std::max(W.z0, msh[(size_t)s].lo), b = std::min(W.z1, msh[(size_t)s].hi);
            if (a < b)
                COMM_TRY(copy(c, r, W.planes.as<float>() + (a - W.z0) * plane, s,
                              m_shards[s] + (a - msh[(size_t)s].lo) * plane, sizeof(float) * plane * (b - a)));
        }
        if (nzw > 0)
            COMM_TRY(ffdp_pad_window(W.planes.as<float>(), mg, W.z0, W.z1, W.padded.as<float>(), c->st[r]));
    }
    return sync_all(c);
}

}  // namespace comm
}  // namespace ffdp

using namespace ffdp;
using namespace ffdp::comm;

extern "C" {

int ffdp_comm_create(int world, const int* devices, ffdp_comm* out) {
    if (!out) return set_error(FFDP_INVALID_ARGUMENT, "comm_create: null output");
    *out = nullptr;
    if (world < 1) return set_error(FFDP_INVALID_ARGUMENT, "WorkerGroup: world size must be >= 1");
    int ndev = 0;
    FFDP_CHECK_CUDA(cudaGetDeviceCount(&ndev));
    DeviceGuard guard;
    auto* c = new ffdp_comm_s;
    c->world = world;
    for (int r = 0; r < world; ++r) {
        const int d = devices ? devices[r] : r % std::max(ndev, 1);
        if (d < 0 || d >= ndev) {
            delete c;
            return set_error(FFDP_INVALID_ARGUMENT, "comm_create: rank %d names device %d of %d", r, d, ndev);
        }
        c->dev.push_back(d);
    }
    for (int r = 0; r < world; ++r) {
        cudaSetDevice(c->dev[r]);
        cudaStream_t s = nullptr;
        // blocking streams: ordered after the legacy default stream the caller produced the inputs on
        if (cudaStreamCreate(&s) != cudaSuccess) {
            for (auto x : c->st) cudaStreamDestroy(x);
            delete c;
            return set_error(FFDP_CUDA, "comm_create: stream creation failed");
        }
        c->st.push_back(s);
        for (int q = 0; q < r; ++q)  // NVLink peer access between distinct devices
            if (c->dev[q] != c->dev[r]) {
                int ok = 0;
                cudaDeviceCanAccessPeer(&ok, c->dev[r], c->dev[q]);
                if (ok && cudaDeviceEnablePeerAccess(c->dev[q], 0) != cudaSuccess) cudaGetLastError();
                cudaSetDevice(c->dev[q]);
                cudaDeviceCanAccessPeer(&ok, c->dev[q], c->dev[r]);
                if (ok && cudaDeviceEnablePeerAccess(c->dev[r], 0) != cudaSuccess) cudaGetLastError();
                cudaSetDevice(c->dev[r]);
            }
    }
    *out = c;
    return FFDP_OK;
}

int ffdp_comm_destroy(ffdp_comm c) {
    if (!c) return FFDP_OK;
    DeviceGuard guard;
    for (int r = 0; r < c->world; ++r) {
        cudaSetDevice(c->dev[r]);
        cudaStreamSynchronize(c->st[r]);
        cudaStreamDestroy(c->st[r]);
    }
    c->world = 0;
    delete c;
    return FFDP_OK;
}

int ffdp_comm_world(ffdp_comm c) { return c ? c->world : 0; }

int ffdp_comm_device(ffdp_comm c, int rank) { return c && rank >= 0 && rank < c->world ? c->dev[rank] : -1; }

int ffdp_shard_range(int64_t n, int world, int rank, int64_t* lo, int64_t* hi) {
    if (world < 1 || rank < 0 || rank >= world || n < 0 || !lo || !hi)
        return set_error(FFDP_INVALID_ARGUMENT, "shard_ranges: bad arguments");
    range(n, world, rank, *lo, *hi);
    return FFDP_OK;
}

int ffdp_halo_exchange(ffdp_comm c, const float* const* slabs, ffdp_dims global, int channels, int pad,
                       float* const* out, int64_t* lo_out, int64_t* hi_out) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)slabs, w, "halo_exchange"));
    COMM_TRY(check_ptrs((const void* const*)out, w, "halo_exchange"));
    COMM_TRY(check_global(global, w, "halo_exchange"));
    if (pad < 0) return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: pad must be >= 0");
    if (channels < 1) return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: channels must be >= 1");
    COMM_TRY(sync_all(c));
    std::vector<Buf> h;
    std::vector<int64_t> lo, hi;
    COMM_TRY(halo(c, slabs, global, channels, pad, h, lo, hi));
    const auto sh = shards(global.nz, w);
    const int64_t plane = global.nx * global.ny * channels;
    for (int r = 0; r < w; ++r) {
        COMM_TRY(copy(c, r, out[r], r, h[(size_t)r].p,
                      sizeof(float) * plane * (sh[(size_t)r].th() + lo[(size_t)r] + hi[(size_t)r])));
        if (lo_out) lo_out[r] = lo[(size_t)r];
        if (hi_out) hi_out[r] = hi[(size_t)r];
    }
    return sync_all(c);
}

int ffdp_dist_gp_convolve(ffdp_comm c, const float* const* slabs, ffdp_dims global, int channels, const double* taps,
                          int ntaps, int mode, int sync, float* const* out) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)slabs, w, "gp_convolve"));
    COMM_TRY(check_ptrs((const void* const*)out, w, "gp_convolve"));
    COMM_TRY(check_global(global, w, "gp_convolve"));
    if (!taps || ntaps < 1 || ntaps % 2 == 0) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: kernel must be odd");
    const int rad = ntaps / 2;
    const auto sh = shards(global.nz, w);
    COMM_TRY(sync_all(c));
    if (!sync || w == 1 || rad == 0) {
        // each shard a standalone volume along z (the sync = false ablation, distops.hpp:94-101)
        for (int r = 0; r < w; ++r) {
            cudaSetDevice(c->dev[r]);
            const int64_t th = sh[(size_t)r].th();
            COMM_TRY(ffdp_gp_convolve(slabs[r], out[r], ffdp_dims{global.nx, global.ny, th}, ffdp_slab{0, th, 0, th, th},
                                      channels, taps, ntaps, mode, c->st[r]));
        }
        return sync_all(c);
    }
    std::vector<Buf> h;
    std::vector<int64_t> lo, hi;
    COMM_TRY(halo(c, slabs, global, channels, rad, h, lo, hi));
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const Shard& s = sh[(size_t)r];
        const int64_t nb = s.th() + lo[(size_t)r] + hi[(size_t)r];
        COMM_TRY(ffdp_gp_convolve(h[(size_t)r].as<float>(), out[r], ffdp_dims{global.nx, global.ny, nb},
                                  ffdp_slab{s.lo - lo[(size_t)r], nb, s.lo, s.hi, global.nz}, channels, taps, ntaps,
                                  mode, c->st[r]));
    }
    return sync_all(c);
}

int ffdp_ring_sample(ffdp_comm c, const float* const* m_shards, ffdp_dims m_global, const float* const* u_shards,
                     ffdp_dims out_global, const double* A, const double* t, float* const* out) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)m_shards, w, "ring_sample"));
    COMM_TRY(check_ptrs((const void* const*)u_shards, w, "ring_sample"));
    COMM_TRY(check_ptrs((const void* const*)out, w, "ring_sample"));
    COMM_TRY(check_global(m_global, w, "ring_sample"));
    COMM_TRY(check_global(out_global, w, "ring_sample"));
    const auto osh = shards(out_global.nz, w);
    std::vector<ffdp_sampler_args> args;
    for (int r = 0; r < w; ++r) args.push_back(shard_args(A, t, osh[(size_t)r], out_global.nz));
    COMM_TRY(sync_all(c));
    std::vector<Window> win;
    COMM_TRY(moving_windows(c, m_shards, m_global, u_shards, out_global, args, win));
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const Window& W = win[(size_t)r];
        const ffdp_image_window iw{W.padded.as<float>(), m_global, W.z0, W.z1, 2};
        COMM_TRY(ffdp_sampler_fwd(iw, u_shards[r], ffdp_dims{out_global.nx, out_global.ny, osh[(size_t)r].th()},
                                  &args[(size_t)r], out[r], 0, nullptr, nullptr, c->st[r]));
    }
    return sync_all(c);
}

int ffdp_ring_sample_bwd(ffdp_comm c, const float* const* upstream, const float* const* m_shards, ffdp_dims m_global,
                         const float* const* u_shards, ffdp_dims out_global, const double* A, const double* t, int want,
                         float* const* g_img, float* const* g_u, double* gAt) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)upstream, w, "ring_sample_backward"));
    COMM_TRY(check_ptrs((const void* const*)m_shards, w, "ring_sample_backward"));
    COMM_TRY(check_ptrs((const void* const*)u_shards, w, "ring_sample_backward"));
    COMM_TRY(check_global(m_global, w, "ring_sample_backward"));
    COMM_TRY(check_global(out_global, w, "ring_sample_backward"));
    const bool wi = want & FFDP_WANT_IMAGE, ww = want & FFDP_WANT_WARP;
    const bool wat = want & (FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION);
    if (wi) COMM_TRY(check_ptrs((const void* const*)g_img, w, "ring_sample_backward (image)"));
    if (ww) COMM_TRY(check_ptrs((const void* const*)g_u, w, "ring_sample_backward (warp)"));
    if (wat && !gAt) return set_error(FFDP_INVALID_ARGUMENT, "ring_sample_backward: null affine output");
    const auto osh = shards(out_global.nz, w), msh = shards(m_global.nz, w);
    std::vector<ffdp_sampler_args> args;
    for (int r = 0; r < w; ++r) args.push_back(shard_args(A, t, osh[(size_t)r], out_global.nz));
    COMM_TRY(sync_all(c));
    std::vector<Window> win;
    COMM_TRY(moving_windows(c, m_shards, m_global, u_shards, out_global, args, win));
    const int64_t plane = m_global.nx * m_global.ny;
    std::vector<Buf> gwin((size_t)w), gat((size_t)w);
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const Window& W = win[(size_t)r];
        const ffdp_dims od{out_global.nx, out_global.ny, osh[(size_t)r].th()};
        if (wi) {
            // image gradients land on the window's planes (dense, pad = 0 window)
            COMM_TRY(gwin[(size_t)r].alloc(c, r, sizeof(float) * plane * (W.z1 - W.z0), true));
            if (W.z1 > W.z0) {
                const ffdp_image_window iw{W.planes.as<float>(), m_global, W.z0, W.z1, 0};
                COMM_TRY(ffdp_sampler_bwd(upstream[r], iw, u_shards[r], od, &args[(size_t)r], FFDP_WANT_IMAGE,
                                          gwin[(size_t)r].as<float>(), nullptr, nullptr, nullptr, c->st[r]));
            }
        }
        if (ww || wat) {
            if (wat) COMM_TRY(gat[(size_t)r].alloc(c, r, 12 * sizeof(double), true));
            const ffdp_image_window iw{W.padded.as<float>(), m_global, W.z0, W.z1, 2};
            const int mask = want & (FFDP_WANT_WARP | FFDP_WANT_AFFINE | FFDP_WANT_TRANSLATION);
            COMM_TRY(ffdp_sampler_bwd(upstream[r], iw, u_shards[r], od, &args[(size_t)r], mask, nullptr,
                                      ww ? g_u[r] : nullptr, wat ? gat[(size_t)r].as<double>() : nullptr, nullptr,
                                      c->st[r]));
        }
    }
    COMM_TRY(sync_all(c));
    if (wi) {
        // route every rank's window gradient to the owners' planes, added in rank order
        // (distops.hpp:230-239)
        for (int s = 0; s < w; ++s) {
            cudaSetDevice(c->dev[s]);
            FFDP_CHECK_CUDA(cudaMemsetAsync(g_img[s], 0, sizeof(float) * plane * msh[(size_t)s].th(), c->st[s]));
            Buf tmp;
            COMM_TRY(tmp.alloc(c, s, sizeof(float) * plane * msh[(size_t)s].th(), false));
            for (int r = 0; r < w; ++r) {
                const Window& W = win[(size_t)r];
                const int64_t a = std::max(W.z0, msh[(size_t)s].lo), b = std::min(W.z1, msh[(size_t)s].hi);
                if (a >= b) continue;
                COMM_TRY(copy(c, s, tmp.as<float>(), r, gwin[(size_t)r].as<float>() + (a - W.z0) * plane,
                              sizeof(float) * plane * (b - a)));
                cudaSetDevice(c->dev[s]);
                const int64_t n = plane * (b - a);
                k_add_f32<<<grid_for(n), 256, 0, c->st[s]>>>(g_img[s] + (a - msh[(size_t)s].lo) * plane, tmp.as<float>(),
                                                             n);
                COMM_TRY(check_launch("ring_sample_backward (image routing)"));
            }
            cudaSetDevice(c->dev[s]);
            FFDP_CHECK_CUDA(cudaStreamSynchronize(c->st[s]));  // tmp is reused / freed
        }
    }
    if (wat) {
        std::vector<double*> bufs;
        for (int r = 0; r < w; ++r) bufs.push_back(gat[(size_t)r].as<double>());
        COMM_TRY(allreduce_f64(c, bufs.data(), 12));
        cudaSetDevice(c->dev[0]);
        FFDP_CHECK_CUDA(cudaMemcpy(gAt, bufs[0], 12 * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return sync_all(c);
}

int ffdp_dist_mse(ffdp_comm c, const float* const* f, const float* const* moved, ffdp_dims global, int64_t n_total,
                  double* loss, float* const* grad) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)f, w, "dist_mse"));
    COMM_TRY(check_ptrs((const void* const*)moved, w, "dist_mse"));
    COMM_TRY(check_ptrs((const void* const*)grad, w, "dist_mse"));
    COMM_TRY(check_global(global, w, "dist_mse"));
    if (!loss || n_total < 1) return set_error(FFDP_INVALID_ARGUMENT, "dist_mse: bad arguments");
    const auto sh = shards(global.nz, w);
    COMM_TRY(sync_all(c));
    std::vector<Buf> s((size_t)w);
    std::vector<double*> bufs;
    for (int r = 0; r < w; ++r) {
        COMM_TRY(s[(size_t)r].alloc(c, r, sizeof(double), true));
        COMM_TRY(ffdp_mse(f[r], moved[r], global.nx * global.ny * sh[(size_t)r].th(), n_total, grad[r],
                          s[(size_t)r].as<double>(), c->st[r]));
        bufs.push_back(s[(size_t)r].as<double>());
    }
    COMM_TRY(sync_all(c));
    COMM_TRY(allreduce_f64(c, bufs.data(), 1));
    double v = 0;
    cudaSetDevice(c->dev[0]);
    FFDP_CHECK_CUDA(cudaMemcpy(&v, bufs[0], sizeof(double), cudaMemcpyDeviceToHost));
    *loss = v / (double)n_total;
    return FFDP_OK;
}

int ffdp_dist_mi(ffdp_comm c, const float* const* f, const float* const* moved, ffdp_dims global,
                 const ffdp_parzen* kernel, int approx_forward, int64_t n_total, double* loss, float* const* grad,
                 int64_t* payload_elements) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)f, w, "dist_mi"));
    COMM_TRY(check_ptrs((const void* const*)moved, w, "dist_mi"));
    COMM_TRY(check_ptrs((const void* const*)grad, w, "dist_mi"));
    COMM_TRY(check_global(global, w, "dist_mi"));
    if (!kernel || !loss || n_total < 1) return set_error(FFDP_INVALID_ARGUMENT, "dist_mi: bad arguments");
    const int B = kernel->bins;
    const int64_t nraw = (int64_t)B * B + 2 * B, ntab = 2LL * B * B + 2 * B + 4;
    const auto sh = shards(global.nz, w);
    COMM_TRY(sync_all(c));
    std::vector<Buf> raw((size_t)w), tab((size_t)w);
    std::vector<double*> bufs;
    for (int r = 0; r < w; ++r) {
        COMM_TRY(raw[(size_t)r].alloc(c, r, sizeof(double) * nraw, true));
        COMM_TRY(ffdp_mi_hist(f[r], moved[r], global.nx * global.ny * sh[(size_t)r].th(), kernel, approx_forward,
                              raw[(size_t)r].as<double>(), nullptr, nullptr, c->st[r]));
        bufs.push_back(raw[(size_t)r].as<double>());
    }
    COMM_TRY(sync_all(c));
    COMM_TRY(allreduce_f64(c, bufs.data(), nraw));  // the B*B + 2B payload (distops.hpp:365-373)
    for (int r = 0; r < w; ++r) {
        COMM_TRY(tab[(size_t)r].alloc(c, r, sizeof(double) * ntab, false));
        COMM_TRY(ffdp_mi_finalize(bufs[(size_t)r], B, -1.0, tab[(size_t)r].as<double>(), c->st[r]));
        COMM_TRY(ffdp_mi_bwd(f[r], moved[r], global.nx * global.ny * sh[(size_t)r].th(), kernel,
                             tab[(size_t)r].as<double>(), nullptr, grad[r], c->st[r]));
    }
    COMM_TRY(sync_all(c));
    double mi = 0;
    cudaSetDevice(c->dev[0]);
    FFDP_CHECK_CUDA(cudaMemcpy(&mi, tab[0].as<double>() + 2LL * B * B + 2 * B + 1, sizeof(double),
                               cudaMemcpyDeviceToHost));
    *loss = -mi;
    if (payload_elements) *payload_elements = nraw;
    return FFDP_OK;
}

int ffdp_dist_lncc(ffdp_comm c, const float* const* f, const float* const* moved, ffdp_dims global, int window,
                   double eps, int ants_approx, int gp_sync, int64_t n_total, double* loss, float* const* grad) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)f, w, "dist_lncc"));
    COMM_TRY(check_ptrs((const void* const*)moved, w, "dist_lncc"));
    COMM_TRY(check_ptrs((const void* const*)grad, w, "dist_lncc"));
    COMM_TRY(check_global(global, w, "dist_lncc"));
    if (window < 1 || window % 2 == 0) return set_error(FFDP_INVALID_ARGUMENT, "lncc: window must be odd and >= 1");
    if (!loss) return set_error(FFDP_INVALID_ARGUMENT, "dist_lncc: null loss");
    if (n_total < 1) n_total = global.nx * global.ny * global.nz;
    const int rad = window / 2;
    const bool sync = gp_sync && w > 1;
    const int pad = sync ? (ants_approx ? rad : 2 * rad) : 0;
    const auto sh = shards(global.nz, w);
    const int64_t plane = global.nx * global.ny;
    COMM_TRY(sync_all(c));
    std::vector<Buf> fh, mh;
    std::vector<int64_t> lo, hi;
    COMM_TRY(halo(c, f, global, 1, pad, fh, lo, hi));
    COMM_TRY(halo(c, moved, global, 1, pad, mh, lo, hi));
    std::vector<Buf> sn((size_t)w), state((size_t)w);
    std::vector<double*> bufs;
    const double gi = -1.0 / (double)n_total;
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const int64_t th = sh[(size_t)r].th();
        const int64_t nz_g = sync ? global.nz : th, g_lo = sync ? sh[(size_t)r].lo : 0;
        const int64_t nb = th + lo[(size_t)r] + hi[(size_t)r];
        const ffdp_dims bd{global.nx, global.ny, nb};
        COMM_TRY(sn[(size_t)r].alloc(c, r, sizeof(double), true));
        COMM_TRY(state[(size_t)r].alloc(c, r, sizeof(double) * 5 * plane * th, false));
        COMM_TRY(ffdp_lncc_fwd(fh[(size_t)r].as<float>(), mh[(size_t)r].as<float>(), bd,
                               ffdp_slab{g_lo - lo[(size_t)r], nb, g_lo, g_lo + th, nz_g}, window, eps,
                               state[(size_t)r].as<double>(), nullptr, sn[(size_t)r].as<double>(), c->st[r]));
        bufs.push_back(sn[(size_t)r].as<double>());
    }
    COMM_TRY(sync_all(c));
    COMM_TRY(allreduce_f64(c, bufs.data(), 1));
    double s = 0;
    cudaSetDevice(c->dev[0]);
    FFDP_CHECK_CUDA(cudaMemcpy(&s, bufs[0], sizeof(double), cudaMemcpyDeviceToHost));
    *loss = 1.0 - s / (double)n_total;
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const int64_t th = sh[(size_t)r].th();
        const ffdp_dims sd{global.nx, global.ny, th};
        if (ants_approx) {
            COMM_TRY(ffdp_lncc_gamma(state[(size_t)r].as<double>(), plane * th, eps, gi, c->st[r]));
            COMM_TRY(ffdp_lncc_combine(state[(size_t)r].as<double>(), sd, ffdp_slab{0, th, 0, th, th}, window, 1, f[r],
                                       moved[r], nullptr, grad[r], c->st[r]));
            continue;
        }
        // exact: the gamma family on the slab +- r planes (inside the lattice), box-filtered
        // again (lncc.hpp:249-263); the 2r halo holds their windows
        const int64_t nz_g = sync ? global.nz : th, g_lo = sync ? sh[(size_t)r].lo : 0;
        const int64_t nb = th + lo[(size_t)r] + hi[(size_t)r];
        const int64_t e0 = std::max<int64_t>(0, g_lo - rad), e1 = std::min<int64_t>(nz_g, g_lo + th + rad);
        Buf st_ext;
        COMM_TRY(st_ext.alloc(c, r, sizeof(double) * 5 * plane * (e1 - e0), false));
        COMM_TRY(ffdp_lncc_fwd(fh[(size_t)r].as<float>(), mh[(size_t)r].as<float>(), ffdp_dims{global.nx, global.ny, nb},
                               ffdp_slab{g_lo - lo[(size_t)r], nb, e0, e1, nz_g}, window, eps, st_ext.as<double>(),
                               nullptr, nullptr, c->st[r]));
        COMM_TRY(ffdp_lncc_gamma(st_ext.as<double>(), plane * (e1 - e0), eps, gi, c->st[r]));
        COMM_TRY(ffdp_lncc_combine(st_ext.as<double>(), ffdp_dims{global.nx, global.ny, e1 - e0},
                                   ffdp_slab{e0, e1 - e0, g_lo, g_lo + th, nz_g}, window, 0, f[r], moved[r], nullptr,
                                   grad[r], c->st[r]));
        FFDP_CHECK_CUDA(cudaStreamSynchronize(c->st[r]));  // st_ext is freed at scope exit
    }
    return sync_all(c);
}

// The fused deformable step over the ranks (ring_sample -> dist_lncc(ANTs) / dist_mi ->
// ring_sample_backward(warp), registration.hpp:277-312), as dist.ShardedStep composes it:
// F and u with r-plane halos (LNCC), the exact moving window of the halo'd slab, the
// step kernels on each slab, rank-ordered sums of sum_n / the joint histogram.
int ffdp_dist_step(ffdp_comm c, int loss_kind, const float* const* f, const float* const* m, const float* const* u,
                   ffdp_dims global, const double* A, const double* t, int window, double eps,
                   const ffdp_parzen* kernel, double* loss, float* const* g_u) {
    COMM_TRY(check_comm(c));
    DeviceGuard guard;
    const int w = c->world;
    COMM_TRY(check_ptrs((const void* const*)f, w, "dist_step"));
    COMM_TRY(check_ptrs((const void* const*)m, w, "dist_step"));
    COMM_TRY(check_ptrs((const void* const*)u, w, "dist_step"));
    COMM_TRY(check_ptrs((const void* const*)g_u, w, "dist_step"));
    COMM_TRY(check_global(global, w, "dist_step"));
    if (!loss || (loss_kind != 0 && loss_kind != 1)) return set_error(FFDP_INVALID_ARGUMENT, "dist_step: bad arguments");
    if (loss_kind == 1 && !kernel) return set_error(FFDP_INVALID_ARGUMENT, "dist_step: MI needs a Parzen kernel");
    if (loss_kind == 0 && (window < 1 || window % 2 == 0))
        return set_error(FFDP_INVALID_ARGUMENT, "lncc: window must be odd and >= 1");
    const bool lncc = loss_kind == 0;
    const int pad = (lncc && w > 1) ? window / 2 : 0;
    const auto sh = shards(global.nz, w);
    const int64_t plane = global.nx * global.ny, n_total = plane * global.nz;
    COMM_TRY(sync_all(c));
    std::vector<Buf> fh, uh;
    std::vector<int64_t> lo, hi;
    COMM_TRY(halo(c, f, global, 1, pad, fh, lo, hi));
    COMM_TRY(halo(c, u, global, 3, pad, uh, lo, hi));
    // sampler args in the global frame (the slab says which planes a buffer holds); the
    // window plan uses the halo'd slab's own bounds
    const ffdp_sampler_args ga = shard_args(A, t, Shard{0, global.nz}, global.nz);
    std::vector<ffdp_sampler_args> wargs;
    std::vector<const float*> uptr;
    for (int r = 0; r < w; ++r) {
        wargs.push_back(shard_args(A, t, Shard{sh[(size_t)r].lo - lo[(size_t)r], sh[(size_t)r].hi + hi[(size_t)r]},
                                   global.nz));
        uptr.push_back(uh[(size_t)r].as<float>());
    }
    // u buffers span the halo'd planes: plan the windows over those lattices
    std::vector<Window> win((size_t)w);
    {
        std::vector<Buf> ext((size_t)w);
        for (int r = 0; r < w; ++r) {
            COMM_TRY(ext[(size_t)r].alloc(c, r, 2 * sizeof(int64_t), false));
            const ffdp_dims bd{global.nx, global.ny, sh[(size_t)r].th() + lo[(size_t)r] + hi[(size_t)r]};
            COMM_TRY(ffdp_sampler_z_extent(uptr[(size_t)r], bd, global, &wargs[(size_t)r], ext[(size_t)r].as<int64_t>(),
                                           c->st[r]));
        }
        COMM_TRY(sync_all(c));
        for (int r = 0; r < w; ++r) {
            int64_t e[2];
            cudaSetDevice(c->dev[r]);
            FFDP_CHECK_CUDA(cudaMemcpy(e, ext[(size_t)r].p, sizeof(e), cudaMemcpyDeviceToHost));
            Window& W = win[(size_t)r];
            W.z0 = e[0] <= e[1] ? std::max<int64_t>(0, e[0]) : 0;
            W.z1 = std::max(W.z0, e[0] <= e[1] ? std::min<int64_t>(global.nz, e[1] + 1) : 0);
            const int64_t nzw = W.z1 - W.z0;
            COMM_TRY(W.planes.alloc(c, r, sizeof(float) * plane * nzw, false));
            COMM_TRY(W.padded.alloc(c, r, sizeof(float) * (global.nx + 4) * (global.ny + 4) * (nzw + 4), nzw == 0));
            for (int s2 = 0; s2 < w; ++s2) {
                const int64_t a = std::max(W.z0, sh[(size_t)s2].lo), b = std::min(W.z1, sh[(size_t)s2].hi);
                if (a < b)
                    COMM_TRY(copy(c, r, W.planes.as<float>() + (a - W.z0) * plane, s2,
                                  m[s2] + (a - sh[(size_t)s2].lo) * plane, sizeof(float) * plane * (b - a)));
            }
            if (nzw > 0)
                COMM_TRY(ffdp_pad_window(W.planes.as<float>(), global, W.z0, W.z1, W.padded.as<float>(), c->st[r]));
        }
        COMM_TRY(sync_all(c));
    }
    // LNCC intensity frame: the value ranges of F and M over all ranks (identical on every
    // rank), reduced on the device in rank order and broadcast back by peer copies
    std::vector<Buf> mm((size_t)w);
    if (lncc) {
        for (int r = 0; r < w; ++r) {
            COMM_TRY(mm[(size_t)r].alloc(c, r, 4 * sizeof(float), false));
            COMM_TRY(ffdp_minmax(f[r], plane * sh[(size_t)r].th(), mm[(size_t)r].as<float>(), c->st[r]));
            COMM_TRY(ffdp_minmax(m[r], plane * sh[(size_t)r].th(), mm[(size_t)r].as<float>() + 2, c->st[r]));
        }
        COMM_TRY(sync_all(c));
        float g4[4] = {0, 0, 0, 0};
        for (int r = 0; r < w; ++r) {
            float v[4];
            cudaSetDevice(c->dev[r]);
            FFDP_CHECK_CUDA(cudaMemcpy(v, mm[(size_t)r].p, sizeof(v), cudaMemcpyDeviceToHost));
            if (r == 0) std::copy(v, v + 4, g4);
            g4[0] = std::min(g4[0], v[0]), g4[1] = std::max(g4[1], v[1]);
            g4[2] = std::min(g4[2], v[2]), g4[3] = std::max(g4[3], v[3]);
        }
        for (int r = 0; r < w; ++r) {
            cudaSetDevice(c->dev[r]);
            FFDP_CHECK_CUDA(cudaMemcpy(mm[(size_t)r].p, g4, sizeof(g4), cudaMemcpyHostToDevice));
        }
    }
    const int B = lncc ? 0 : kernel->bins;
    const int64_t nraw = lncc ? 1 : (int64_t)B * B + 2 * B;
    std::vector<Buf> red((size_t)w), miss((size_t)w), ws((size_t)w), rec((size_t)w), tab((size_t)w);
    std::vector<double*> bufs;
    const bool bs = !lncc && kernel->kind == FFDP_PARZEN_BSPLINE3;
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const Shard& s = sh[(size_t)r];
        const int64_t nb = s.th() + lo[(size_t)r] + hi[(size_t)r];
        const ffdp_dims bd{global.nx, global.ny, nb};
        const ffdp_slab sl{s.lo - lo[(size_t)r], nb, s.lo, s.hi, global.nz};
        const Window& W = win[(size_t)r];
        const ffdp_image_window iw{W.padded.as<float>(), global, W.z0, W.z1, 2};
        COMM_TRY(red[(size_t)r].alloc(c, r, sizeof(double) * nraw, true));
        COMM_TRY(miss[(size_t)r].alloc(c, r, sizeof(int32_t), true));
        bufs.push_back(red[(size_t)r].as<double>());
        if (lncc) {
            COMM_TRY(ws[(size_t)r].alloc(c, r, (size_t)ffdp_step_lncc_workspace_bytes(bd, sl), false));
            COMM_TRY(ffdp_step_lncc(fh[(size_t)r].as<float>(), uh[(size_t)r].as<float>(), bd, sl, iw, &ga, window, eps,
                                    -1.0 / (double)n_total, mm[(size_t)r].as<float>(), g_u[r],
                                    red[(size_t)r].as<double>(),
                                    miss[(size_t)r].as<int32_t>(), ws[(size_t)r].p, c->st[r]));
        } else {
            COMM_TRY(ws[(size_t)r].alloc(c, r, (size_t)ffdp_step_mi_workspace_bytes(B), true));
            if (bs) {
                COMM_TRY(rec[(size_t)r].alloc(c, r, (size_t)ffdp_step_mi_record_bytes(bd, sl), false));
                COMM_TRY(ffdp_step_mi_hist_rec(fh[(size_t)r].as<float>(), uh[(size_t)r].as<float>(), bd, sl, iw, &ga,
                                               kernel, red[(size_t)r].as<double>(), ws[(size_t)r].p,
                                               rec[(size_t)r].as<float>(), miss[(size_t)r].as<int32_t>(), c->st[r]));
            } else {
                COMM_TRY(ffdp_step_mi_hist(fh[(size_t)r].as<float>(), uh[(size_t)r].as<float>(), bd, sl, iw, &ga,
                                           kernel, red[(size_t)r].as<double>(), ws[(size_t)r].p,
                                           miss[(size_t)r].as<int32_t>(), c->st[r]));
            }
        }
    }
    COMM_TRY(sync_all(c));
    for (int r = 0; r < w; ++r) {
        int32_t mv = 0;
        cudaSetDevice(c->dev[r]);
        FFDP_CHECK_CUDA(cudaMemcpy(&mv, miss[(size_t)r].p, sizeof(mv), cudaMemcpyDeviceToHost));
        if (mv) return set_error(FFDP_RUNTIME, "dist_step: rank %d sampled outside its moving window", r);
    }
    COMM_TRY(allreduce_f64(c, bufs.data(), nraw));
    double v = 0;
    if (lncc) {
        cudaSetDevice(c->dev[0]);
        FFDP_CHECK_CUDA(cudaMemcpy(&v, bufs[0], sizeof(double), cudaMemcpyDeviceToHost));
        *loss = 1.0 - v / (double)n_total;
        return FFDP_OK;
    }
    const int64_t ntab = 2LL * B * B + 2 * B + 4;
    for (int r = 0; r < w; ++r) {
        cudaSetDevice(c->dev[r]);
        const Shard& s = sh[(size_t)r];
        const int64_t nb = s.th() + lo[(size_t)r] + hi[(size_t)r];
        const ffdp_dims bd{global.nx, global.ny, nb};
        const ffdp_slab sl{s.lo - lo[(size_t)r], nb, s.lo, s.hi, global.nz};
        COMM_TRY(tab[(size_t)r].alloc(c, r, sizeof(double) * ntab, false));
        COMM_TRY(ffdp_mi_finalize(bufs[(size_t)r], B, -1.0, tab[(size_t)r].as<double>(), c->st[r]));
        if (bs) {
            COMM_TRY(ffdp_step_mi_grad_rec(fh[(size_t)r].as<float>(), bd, sl, kernel, tab[(size_t)r].as<double>(),
                                           rec[(size_t)r].as<float>(), g_u[r], c->st[r]));
        } else {
            const Window& W = win[(size_t)r];
            const ffdp_image_window iw{W.padded.as<float>(), global, W.z0, W.z1, 2};
            COMM_TRY(ffdp_step_mi_grad(fh[(size_t)r].as<float>(), uh[(size_t)r].as<float>(), bd, sl, iw, &ga, kernel,
                                       tab[(size_t)r].as<double>(), g_u[r], miss[(size_t)r].as<int32_t>(), c->st[r]));
        }
    }
    COMM_TRY(sync_all(c));
    cudaSetDevice(c->dev[0]);
    FFDP_CHECK_CUDA(cudaMemcpy(&v, tab[0].as<double>() + 2LL * B * B + 2 * B + 1, sizeof(double),
                               cudaMemcpyDeviceToHost));
    *loss = -v;
    return FFDP_OK;
}

}  // extern "C"
