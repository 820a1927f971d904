// plan.cu -- the sharded deformable step as a persistent per-rank plan over a native
// transport: NCCL (one process per GPU, NVLink / NVSwitch) or an in-process group (one
// host thread per rank; ranks may share a device, which is how it is tested on one GPU).
//
// Reference: the per-iteration sequence of deformable_stage under WorkerGroup(H)
// (registration.hpp:266-312): ring_sample (distops.hpp:144-168) -> dist_lncc
// (distops.hpp:285-352) or dist_mi (distops.hpp:355-396) -> ring_sample_backward with want
// warp (distops.hpp:179-248), over z slabs by shard_ranges (fabric.hpp:44-70) with
// halo_exchange (fabric.hpp:315-370) and allreduce_sum (fabric.hpp:246-263).
//
// What persists across steps (created once, loaded once per scale):
//   * u lives in a haloed buffer owned by the plan; the caller (the optimiser) updates its
//     interior in place and the halo planes are received straight into it -- no per-step
//     slab copy;
//   * F with its halo planes, the zero-bordered moving window (the planes this rank's
//     samples reach, fetched from their owners once per scale: M is static within a
//     scale, registration.hpp:249,270), the LNCC intensity frame, workspaces;
//   * the MI fixed-point grid is chosen from the GLOBAL voxel count, and the joint
//     histogram is allreduced as integers: every rank count gives the single-GPU histogram
//     bit for bit.
// Per step: LNCC -- the u halo exchange on the comm stream, overlapped with the interior
// planes of the fused kernel, then the boundary planes; one allreduce of {sum n_i,
// misses}. MI -- pass 1, one integer allreduce of {joint histogram, misses}, finalize,
// pass 2. One device->host read of {loss, misses} per step (none in the launch-only form).
// A window miss on any rank (the summed count) widens every missing rank's window from
// the z extent of its samples and repeats the step, so results are always exact.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ffdp_common.cuh"

namespace ffdp {
// internal entry points of the step kernels (step_lncc3.cu, step_mi.cu)
int lncc3_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, const float* ranges, float* g_u, double* sum_n,
               int32_t* miss, void* workspace, cudaStream_t st);
int64_t lncc3_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s);
int mi_quad_hist(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, double* raw, unsigned long long* ws,
                 int32_t* miss, cudaStream_t st, float* rec, double* table, double upstream, int scale_exp);
int mi_grad_rec(const float* f, const ffdp_dims& d, const ffdp_slab& s, const ffdp_parzen& k, const double* table,
                const float* rec, float* g_u, cudaStream_t st);
int mi_quad_grad(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
                 const ffdp_sampler_args& args, const ffdp_parzen& k, const double* table, float* g_u, int32_t* miss,
                 cudaStream_t st);
bool mi_quad_path_applies(const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m, const ffdp_parzen& k);
int mi_bs_scale_exp(int64_t voxels);
int mi_hist_u64_to_raw(const unsigned long long* h, int B, int scale_exp, double* raw, cudaStream_t st);

namespace plan {

// ------------------------------------------------------------------ NCCL (dlopen)
// Loaded at run time (libnccl.so.2, or FFDP_NCCL_LIB): single-GPU users of libffdp.so need
// no NCCL, and a process that already loaded one (PyTorch's) shares it.
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = getenv("FFDP_NCCL_LIB");
        void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = dlerror() ? dlerror() : "dlopen failed";
            return;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
#define FFDP_NCCL_SYM(F) n.F = reinterpret_cast<decltype(n.F)>(sym("nccl" #F))
        FFDP_NCCL_SYM(GetVersion);
        FFDP_NCCL_SYM(GetUniqueId);
        FFDP_NCCL_SYM(CommInitRank);
        FFDP_NCCL_SYM(CommDestroy);
        FFDP_NCCL_SYM(GroupStart);
        FFDP_NCCL_SYM(GroupEnd);
        FFDP_NCCL_SYM(Send);
        FFDP_NCCL_SYM(Recv);
        FFDP_NCCL_SYM(AllReduce);
        FFDP_NCCL_SYM(GetErrorString);
#undef FFDP_NCCL_SYM
        n.ok = n.GetVersion && n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart && n.GroupEnd &&
               n.Send && n.Recv && n.AllReduce && n.GetErrorString;
        if (!n.ok) n.why = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

#define PLAN_TRY(expr)             \
    do {                           \
        const int rc_ = (expr);    \
        if (rc_ != FFDP_OK) return rc_; \
    } while (0)
#define NCCL_TRY(expr)                                                                                            \
    do {                                                                                                          \
        const ncclResult_t r_ = (expr);                                                                           \
        if (r_ != ncclSuccess) return set_error(FFDP_RUNTIME, "%s: %s", #expr, nccl().GetErrorString(r_));       \
    } while (0)

// ------------------------------------------------------------------ transports
enum class Dt { F64, U64, I64 };
enum class Op { Sum, Min };
inline size_t dt_size(Dt) { return 8; }

struct P2P {
    bool send;
    void* buf;
    size_t bytes;
    int peer;
};

struct Transport {
    int world = 1, rank = 0, device = 0;
    virtual ~Transport() {}
    // point-to-point transfers as one group (every pair of ranks posts matching sends and
    // receives in the same order), stream-ordered on st
    virtual int p2p(const std::vector<P2P>& ops, cudaStream_t st) = 0;
    // in-place allreduce of n 8-byte elements, stream-ordered on st
    virtual int allreduce(void* buf, size_t n, Dt dt, Op op, cudaStream_t st) = 0;
};

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) nccl().CommDestroy(comm);
    }
    int p2p(const std::vector<P2P>& ops, cudaStream_t st) override {
        if (ops.empty()) return FFDP_OK;
        const Nccl& N = nccl();
        NCCL_TRY(N.GroupStart());
        for (const P2P& o : ops) {
            if (o.send)
                NCCL_TRY(N.Send(o.buf, o.bytes, ncclUint8, o.peer, comm, st));
            else
                NCCL_TRY(N.Recv(o.buf, o.bytes, ncclUint8, o.peer, comm, st));
        }
        NCCL_TRY(N.GroupEnd());
        return FFDP_OK;
    }
    int allreduce(void* buf, size_t n, Dt dt, Op op, cudaStream_t st) override {
        const ncclDataType_t t = dt == Dt::F64 ? ncclFloat64 : dt == Dt::U64 ? ncclUint64 : ncclInt64;
        NCCL_TRY(nccl().AllReduce(buf, buf, n, t, op == Op::Sum ? ncclSum : ncclMin, comm, st));
        return FFDP_OK;
    }
};

// In-process group: the ranks are host threads of one process (one per rank, as with
// ncclCommInitAll), exchanging through peer copies ordered by events; reductions sum the
// ranks' rows in rank order (fabric.hpp:246-263), identically on every rank.
struct LocalHub {
    int world;
    std::vector<int> dev;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    uint64_t gen = 0;
    struct Post {
        const std::vector<P2P>* ops = nullptr;
        void* buf = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Post> post;
    std::atomic<int> refs{0};
    void barrier() {
        std::unique_lock<std::mutex> l(mu);
        const uint64_t g = gen;
        if (++count == world) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(l, [&] { return gen != g; });
        }
    }
};

template <typename T, bool MIN>
__global__ void k_rank_reduce(const T* rows, int world, size_t n, T* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T acc = rows[i];
        for (int q = 1; q < world; ++q) {
            const T v = rows[(size_t)q * n + i];
            acc = MIN ? (v < acc ? v : acc) : acc + v;
        }
        out[i] = acc;
    }
}

struct LocalTransport : Transport {
    std::shared_ptr<LocalHub> hub;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    ~LocalTransport() override {
        cudaSetDevice(device);
        if (scratch) cudaFree(scratch);
        auto& P = hub->post[(size_t)rank];
        if (P.ready) cudaEventDestroy(P.ready);
        if (P.done) cudaEventDestroy(P.done);
    }
    LocalHub::Post& me() { return hub->post[(size_t)rank]; }
    int p2p(const std::vector<P2P>& ops, cudaStream_t st) override {
        LocalHub& H = *hub;
        me().ops = &ops;
        FFDP_CHECK_CUDA(cudaEventRecord(me().ready, st));
        H.barrier();
        // receives: the k-th receive from q matches q's k-th send to me
        std::vector<int> seen((size_t)world, 0);
        for (const P2P& o : ops) {
            if (o.send) continue;
            const int q = o.peer;
            int k = seen[(size_t)q]++;
            const P2P* src = nullptr;
            for (const P2P& so : *H.post[(size_t)q].ops)
                if (so.send && so.peer == rank && k-- == 0) {
                    src = &so;
                    break;
                }
            if (!src || src->bytes != o.bytes) {
                H.barrier();
                H.barrier();
                return set_error(FFDP_RUNTIME, "group: unmatched receive from rank %d", q);
            }
            FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, H.post[(size_t)q].ready, 0));
            FFDP_CHECK_CUDA(cudaMemcpyPeerAsync(o.buf, device, src->buf, H.dev[(size_t)q], o.bytes, st));
        }
        FFDP_CHECK_CUDA(cudaEventRecord(me().done, st));
        H.barrier();
        // a send buffer may be reused once its receiver's copies are done
        for (const P2P& o : ops)
            if (o.send) FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, H.post[(size_t)o.peer].done, 0));
        H.barrier();
        return FFDP_OK;
    }
    int allreduce(void* buf, size_t n, Dt dt, Op op, cudaStream_t st) override {
        LocalHub& H = *hub;
        const size_t bytes = n * dt_size(dt);
        if (scratch_bytes < bytes * world) {
            if (scratch) cudaFree(scratch);
            scratch = nullptr;
            scratch_bytes = 0;
            FFDP_CHECK_CUDA(cudaMalloc(&scratch, bytes * world));
            scratch_bytes = bytes * world;
        }
        me().buf = buf;
        FFDP_CHECK_CUDA(cudaEventRecord(me().ready, st));
        H.barrier();
        char* rows = static_cast<char*>(scratch);
        for (int q = 0; q < world; ++q) {
            if (q != rank) FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, H.post[(size_t)q].ready, 0));
            FFDP_CHECK_CUDA(cudaMemcpyPeerAsync(rows + bytes * q, device, H.post[(size_t)q].buf, H.dev[(size_t)q], bytes, st));
        }
        FFDP_CHECK_CUDA(cudaEventRecord(me().done, st));
        H.barrier();
        for (int q = 0; q < world; ++q)
            if (q != rank) FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, H.post[(size_t)q].done, 0));
        const int nb = (int)std::min<size_t>((n + 255) / 256, 1024);
        if (dt == Dt::F64)
            op == Op::Sum ? k_rank_reduce<double, false><<<nb, 256, 0, st>>>((const double*)rows, world, n, (double*)buf)
                          : k_rank_reduce<double, true><<<nb, 256, 0, st>>>((const double*)rows, world, n, (double*)buf);
        else if (dt == Dt::U64)
            k_rank_reduce<unsigned long long, false><<<nb, 256, 0, st>>>((const unsigned long long*)rows, world, n,
                                                                          (unsigned long long*)buf);
        else
            op == Op::Sum ? k_rank_reduce<long long, false><<<nb, 256, 0, st>>>((const long long*)rows, world, n, (long long*)buf)
                          : k_rank_reduce<long long, true><<<nb, 256, 0, st>>>((const long long*)rows, world, n, (long long*)buf);
        H.barrier();
        return check_launch("group allreduce");
    }
};

// ------------------------------------------------------------------ small kernels
// [F min, -F max, M min, -M max] in fp64 for a MIN allreduce; a NaN range (ffdp_minmax)
// becomes -inf so it survives the reduction and poisons the intensity frame.
__global__ void k_ranges_pack(const float* mm, double* d) {
    if (threadIdx.x < 4) {
        const float v = mm[threadIdx.x];
        d[threadIdx.x] = v != v ? -INFINITY : ((threadIdx.x & 1) ? -(double)v : (double)v);
    }
}
__global__ void k_ranges_unpack(const double* d, float* r) {
    if (threadIdx.x < 4) {
        const double v = d[threadIdx.x];
        r[threadIdx.x] = isinf(v) ? NAN : (float)((threadIdx.x & 1) ? -v : v);
    }
}
// LNCC payload: red[1] = the step's window misses (red[0] holds sum n_i)
__global__ void k_pack_miss(const int32_t* miss, double* red) { red[1] = (double)*miss; }
// MI readback: {loss = -MI, misses} from the finalize table and the histogram payload
__global__ void k_pack_mi(const double* table, int B, const unsigned long long* hist, double* out) {
    out[0] = -table[2 * B * B + 2 * B + 1];
    out[1] = (double)hist[B * B];
}

inline double axis_coord(int64_t i, int64_t n) { return n > 1 ? -1.0 + 2.0 * (double)i / (double)(n - 1) : 0.0; }

inline void shard_range(int64_t n, int w, int r, int64_t& lo, int64_t& hi) {
    // shard_ranges (fabric.hpp:44-57): the first n mod w ranks get one extra plane
    const int64_t base = n / w, extra = n % w;
    lo = r * base + std::min<int64_t>(r, extra);
    hi = lo + base + (r < extra ? 1 : 0);
}

// device buffer owned by a plan
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int alloc(size_t b) {
        if (b <= bytes && p) return FFDP_OK;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (b == 0) return FFDP_OK;
        FFDP_CHECK_CUDA(cudaMalloc(&p, b));
        bytes = b;
        return FFDP_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace plan
}  // namespace ffdp

using namespace ffdp;
using namespace ffdp::plan;

struct ffdp_group_s {
    std::unique_ptr<Transport> t;
};

struct ffdp_plan_s {
    Transport* tr = nullptr;
    int world = 1, rank = 0, dev = 0;
    ffdp_dims global{};
    ffdp_plan_params prm{};
    bool lncc = true;
    int B = 0, scale_exp = 21;
    int64_t lo = 0, hi = 0, hlo = 0, hhi = 0, plane = 0, n_total = 0;
    ffdp_sampler_args ga{};  // sampler args of the global output lattice
    cudaStream_t st = nullptr, cst = nullptr;
    cudaEvent_t ev_u = nullptr, ev_halo = nullptr;
    DBuf f_h, u_h, u_h2, g_h, m1, m2, m_own, stage, win, ranges, rng64, red, hist, raw, table, lws, rec, ext, req;
    int64_t adam_step = 0;  // the scale's Adam step counter (adam.hpp:30-50)
    int64_t wz0 = 0, wz1 = 0;  // resident moving planes
    bool loaded = false;
    double* host = nullptr;    // pinned {loss, misses}
    int64_t fetches = 0;
    int64_t th() const { return hi - lo; }
    int64_t nb() const { return hlo + th() + hhi; }
    ffdp_dims bd() const { return ffdp_dims{global.nx, global.ny, nb()}; }
    ffdp_slab slab(int64_t z0, int64_t z1) const { return ffdp_slab{lo - hlo, nb(), z0, z1, global.nz}; }
    // g_u lives in the interior of the haloed g buffer (the warp update smooths it in place)
    float* g_int() const { return g_h.as<float>() + 3 * hlo * plane; }
    ffdp_image_window window() const {
        return ffdp_image_window{win.as<float>(), global, wz0, wz1, 2};
    }
};

namespace {

struct DevGuard {
    int prev = 0;
    explicit DevGuard(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~DevGuard() { cudaSetDevice(prev); }
};

// exchange the w planes next to the interior of a haloed buffer (channels floats per voxel,
// the plan's hlo / hhi halo planes allocated on each side) with the z neighbours: my first /
// last w interior planes become their halo planes, theirs mine. w < 0: the whole halo.
int halo_swap(ffdp_plan_s* P, float* buf, int ch, cudaStream_t st, int64_t w = -1) {
    const int64_t pl = P->plane * ch;
    const int64_t wl = P->hlo > 0 ? (w < 0 ? P->hlo : w) : 0, wh = P->hhi > 0 ? (w < 0 ? P->hhi : w) : 0;
    std::vector<P2P> ops;
    if (wl > 0) {
        ops.push_back({true, buf + P->hlo * pl, sizeof(float) * pl * wl, P->rank - 1});
        ops.push_back({false, buf + (P->hlo - wl) * pl, sizeof(float) * pl * wl, P->rank - 1});
    }
    if (wh > 0) {
        ops.push_back({true, buf + (P->hlo + P->th() - wh) * pl, sizeof(float) * pl * wh, P->rank + 1});
        ops.push_back({false, buf + (P->hlo + P->th()) * pl, sizeof(float) * pl * wh, P->rank + 1});
    }
    return P->tr->p2p(ops, st);
}

// Moving planes [a, b) this rank needs: fetched from their owners into the zero-bordered
// window (collective: every rank calls with its own request).
int fetch_window(ffdp_plan_s* P, int64_t a, int64_t b) {
    const int64_t nz = P->global.nz;
    a = std::max<int64_t>(0, a);
    b = std::min<int64_t>(nz, std::max(a, b));
    const int w = P->world;
    PLAN_TRY(P->req.alloc(sizeof(int64_t) * 2 * w));
    std::vector<int64_t> mine((size_t)2 * w, 0);
    mine[(size_t)2 * P->rank] = a;
    mine[(size_t)2 * P->rank + 1] = b;
    FFDP_CHECK_CUDA(cudaMemcpyAsync(P->req.p, mine.data(), sizeof(int64_t) * 2 * w, cudaMemcpyHostToDevice, P->st));
    PLAN_TRY(P->tr->allreduce(P->req.p, (size_t)2 * w, Dt::I64, Op::Sum, P->st));
    std::vector<int64_t> all((size_t)2 * w);
    FFDP_CHECK_CUDA(cudaMemcpyAsync(all.data(), P->req.p, sizeof(int64_t) * 2 * w, cudaMemcpyDeviceToHost, P->st));
    FFDP_CHECK_CUDA(cudaStreamSynchronize(P->st));
    const int64_t nzw = b - a;
    PLAN_TRY(P->stage.alloc(sizeof(float) * P->plane * std::max<int64_t>(1, nzw)));
    PLAN_TRY(P->win.alloc(sizeof(float) * (P->global.nx + 4) * (P->global.ny + 4) * (nzw + 4)));
    std::vector<P2P> ops;
    for (int q = 0; q < w; ++q) {
        if (q == P->rank) continue;
        int64_t qlo, qhi;
        shard_range(nz, w, q, qlo, qhi);
        // my planes inside q's request go to q; q's planes inside mine come from q
        const int64_t s0 = std::max(all[(size_t)2 * q], P->lo), s1 = std::min(all[(size_t)2 * q + 1], P->hi);
        const int64_t r0 = std::max(a, qlo), r1 = std::min(b, qhi);
        // order per pair: the lower rank sends first (both sides list the same order)
        auto add_send = [&] {
            if (s0 < s1)
                ops.push_back({true, P->m_own.as<float>() + (s0 - P->lo) * P->plane,
                               sizeof(float) * P->plane * (s1 - s0), q});
        };
        auto add_recv = [&] {
            if (r0 < r1)
                ops.push_back({false, P->stage.as<float>() + (r0 - a) * P->plane, sizeof(float) * P->plane * (r1 - r0), q});
        };
        if (P->rank < q) {
            add_send();
            add_recv();
        } else {
            add_recv();
            add_send();
        }
    }
    const int64_t o0 = std::max(a, P->lo), o1 = std::min(b, P->hi);
    if (o0 < o1)
        FFDP_CHECK_CUDA(cudaMemcpyAsync(P->stage.as<float>() + (o0 - a) * P->plane,
                                        P->m_own.as<float>() + (o0 - P->lo) * P->plane,
                                        sizeof(float) * P->plane * (o1 - o0), cudaMemcpyDeviceToDevice, P->st));
    PLAN_TRY(P->tr->p2p(ops, P->st));
    if (nzw > 0) {
        PLAN_TRY(ffdp_pad_window(P->stage.as<float>(), P->global, a, b, P->win.as<float>(), P->st));
    } else {
        FFDP_CHECK_CUDA(cudaMemsetAsync(P->win.p, 0, P->win.bytes, P->st));
    }
    FFDP_CHECK_CUDA(cudaStreamSynchronize(P->st));
    P->wz0 = a;
    P->wz1 = b;
    ++P->fetches;
    return FFDP_OK;
}

// z range of moving planes the affine part of the warp maps the haloed slab into (the
// displacement's reach is the margin's job and, past it, the miss retry's)
void affine_z_range(const ffdp_plan_s* P, int64_t& a, int64_t& b) {
    const int64_t nz = P->global.nz;
    const double* A = P->prm.A;
    const double* t = P->prm.t;
    double zmin = 1e300, zmax = -1e300;
    for (int64_t zi : {P->lo - P->hlo, P->hi + P->hhi - 1})
        for (double xx : {-1.0, 1.0})
            for (double yy : {-1.0, 1.0}) {
                const double zn = A[6] * xx + A[7] * yy + A[8] * axis_coord(zi, nz) + t[2];
                const double f = (zn + 1.0) * 0.5 * (double)(nz - 1);
                zmin = std::min(zmin, f);
                zmax = std::max(zmax, f);
            }
    a = (int64_t)std::floor(zmin) - 1 - P->prm.margin_planes;
    b = (int64_t)std::ceil(zmax) + 2 + P->prm.margin_planes;
}

int launch_step(ffdp_plan_s* P) {
    cudaStream_t st = P->st;
    const ffdp_image_window iw = P->window();
    if (P->lncc) {
        FFDP_CHECK_CUDA(cudaMemsetAsync(P->red.p, 0, 2 * sizeof(double), st));
        FFDP_CHECK_CUDA(cudaMemsetAsync(P->hist.p, 0, sizeof(int32_t), st));  // miss counter
        int32_t* miss = P->hist.as<int32_t>();
        double* sum_n = P->red.as<double>();
        const double gi = -1.0 / (double)P->n_total;
        const bool halo = P->hlo > 0 || P->hhi > 0;
        // boundary band: outputs within c planes of a shard face wait for the u halo; the
        // interior runs meanwhile (c >= the window radius; a normal z chunk's size, so the
        // split adds no warm-up planes)
        const int64_t c = std::max<int64_t>(P->prm.window / 2, 16);
        const bool split = halo && P->prm.overlap && P->th() > 2 * c + 8;
        if (halo) {
            FFDP_CHECK_CUDA(cudaEventRecord(P->ev_u, st));
            FFDP_CHECK_CUDA(cudaStreamWaitEvent(P->cst, P->ev_u, 0));
            PLAN_TRY(halo_swap(P, P->u_h.as<float>(), 3, P->cst));
            FFDP_CHECK_CUDA(cudaEventRecord(P->ev_halo, P->cst));
        }
        const ffdp_dims bd = P->bd();
        auto run = [&](int64_t z0, int64_t z1) {
            return lncc3_step(P->f_h.as<float>(), P->u_h.as<float>(), bd, P->slab(z0, z1), iw, P->ga, P->prm.eps, gi,
                              P->ranges.as<float>(), P->g_int() + 3 * (z0 - P->lo) * P->plane, sum_n, miss,
                              P->lws.p, st);
        };
        if (split) {
            const int64_t ilo = P->hlo > 0 ? P->lo + c : P->lo, ihi = P->hhi > 0 ? P->hi - c : P->hi;
            PLAN_TRY(run(ilo, ihi));
            FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, P->ev_halo, 0));
            if (ilo > P->lo) PLAN_TRY(run(P->lo, ilo));
            if (ihi < P->hi) PLAN_TRY(run(ihi, P->hi));
        } else {
            if (halo) FFDP_CHECK_CUDA(cudaStreamWaitEvent(st, P->ev_halo, 0));
            PLAN_TRY(run(P->lo, P->hi));
        }
        k_pack_miss<<<1, 1, 0, st>>>(miss, sum_n);
        PLAN_TRY(P->tr->allreduce(P->red.p, 2, Dt::F64, Op::Sum, st));
        FFDP_CHECK_CUDA(cudaMemcpyAsync(P->host, P->red.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        return check_launch("plan step (lncc)");
    }
    const int B = P->B;
    unsigned long long* h = P->hist.as<unsigned long long>();
    FFDP_CHECK_CUDA(cudaMemsetAsync(h, 0, sizeof(unsigned long long) * (B * B + 1), st));
    FFDP_CHECK_CUDA(cudaMemsetAsync(P->raw.p, 0, sizeof(double) * (B * B + 2 * B), st));
    int32_t* miss = reinterpret_cast<int32_t*>(h + B * B);  // low word of the payload's last slot
    const ffdp_dims bd = P->bd();
    const ffdp_slab sl = P->slab(P->lo, P->hi);
    float* rec = P->rec.p ? P->rec.as<float>() : nullptr;
    PLAN_TRY(mi_quad_hist(P->f_h.as<float>(), P->u_h.as<float>(), bd, sl, iw, P->ga, P->prm.kernel, nullptr, h, miss,
                          st, rec, nullptr, -1.0, P->scale_exp));
    PLAN_TRY(P->tr->allreduce(h, (size_t)B * B + 1, Dt::U64, Op::Sum, st));
    PLAN_TRY(mi_hist_u64_to_raw(h, B, P->scale_exp, P->raw.as<double>(), st));
    PLAN_TRY(ffdp_mi_finalize(P->raw.as<double>(), B, -1.0, P->table.as<double>(), st));
    if (rec)
        PLAN_TRY(mi_grad_rec(P->f_h.as<float>(), bd, sl, P->prm.kernel, P->table.as<double>(), rec, P->g_int(), st));
    else
        PLAN_TRY(mi_quad_grad(P->f_h.as<float>(), P->u_h.as<float>(), bd, sl, iw, P->ga, P->prm.kernel,
                              P->table.as<double>(), P->g_int(), nullptr, st));
    k_pack_mi<<<1, 1, 0, st>>>(P->table.as<double>(), B, h, P->red.as<double>());
    FFDP_CHECK_CUDA(cudaMemcpyAsync(P->host, P->red.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    return check_launch("plan step (mi)");
}

double loss_of(const ffdp_plan_s* P) {
    return P->lncc ? 1.0 - P->host[0] / (double)P->n_total : P->host[0];
}

// widen this rank's window to the z extent of its samples (plus one plane each way), collective
int widen(ffdp_plan_s* P) {
    PLAN_TRY(P->ext.alloc(2 * sizeof(int64_t)));
    ffdp_sampler_args wa = P->ga;
    wa.x_min[2] = axis_coord(P->lo - P->hlo, P->global.nz);
    wa.x_max[2] = axis_coord(P->hi + P->hhi - 1, P->global.nz);
    PLAN_TRY(ffdp_sampler_z_extent(P->u_h.as<float>(), P->bd(), P->global, &wa, P->ext.as<int64_t>(), P->st));
    int64_t e[2];
    FFDP_CHECK_CUDA(cudaMemcpyAsync(e, P->ext.p, sizeof(e), cudaMemcpyDeviceToHost, P->st));
    FFDP_CHECK_CUDA(cudaStreamSynchronize(P->st));
    int64_t a = P->wz0, b = P->wz1;
    if (e[0] <= e[1]) {
        a = std::min(a, e[0] - 1);
        b = std::max(b, e[1] + 2);
    }
    return fetch_window(P, a, b);
}

int check_plan(ffdp_plan p) {
    if (!p) return set_error(FFDP_INVALID_ARGUMENT, "plan: null plan");
    if (!p->loaded) return set_error(FFDP_LOGIC, "plan: ffdp_plan_load has not been called");
    return FFDP_OK;
}

}  // namespace

extern "C" {

int ffdp_nccl_version(int* version) {
    const Nccl& N = nccl();
    if (!N.ok) return set_error(FFDP_RUNTIME, "NCCL unavailable: %s", N.why.c_str());
    int v = 0;
    NCCL_TRY(N.GetVersion(&v));
    if (version) *version = v;
    return FFDP_OK;
}

int ffdp_nccl_unique_id(unsigned char* id) {
    if (!id) return set_error(FFDP_INVALID_ARGUMENT, "nccl_unique_id: null id");
    const Nccl& N = nccl();
    if (!N.ok) return set_error(FFDP_RUNTIME, "NCCL unavailable: %s", N.why.c_str());
    ncclUniqueId u;
    NCCL_TRY(N.GetUniqueId(&u));
    static_assert(sizeof(ncclUniqueId) == FFDP_NCCL_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, &u, sizeof(u));
    return FFDP_OK;
}

int ffdp_group_nccl(const unsigned char* id, int world, int rank, int device, ffdp_group* out) {
    if (!id || !out || world < 1 || rank < 0 || rank >= world || device < 0)
        return set_error(FFDP_INVALID_ARGUMENT, "group_nccl: bad arguments");
    const Nccl& N = nccl();
    if (!N.ok) return set_error(FFDP_RUNTIME, "NCCL unavailable: %s", N.why.c_str());
    DevGuard g(device);
    auto t = std::make_unique<NcclTransport>();
    t->world = world;
    t->rank = rank;
    t->device = device;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    NCCL_TRY(N.CommInitRank(&t->comm, world, u, rank));
    *out = new ffdp_group_s{std::move(t)};
    return FFDP_OK;
}

int ffdp_group_local(int world, const int* devices, ffdp_group* out) {
    if (world < 1 || !out) return set_error(FFDP_INVALID_ARGUMENT, "group_local: bad arguments");
    int count = 0;
    FFDP_CHECK_CUDA(cudaGetDeviceCount(&count));
    if (count < 1) return set_error(FFDP_CUDA, "group_local: no device");
    auto hub = std::make_shared<LocalHub>();
    hub->world = world;
    hub->post.resize((size_t)world);
    for (int r = 0; r < world; ++r) {
        const int d = devices ? devices[r] : r % count;
        if (d < 0 || d >= count) return set_error(FFDP_INVALID_ARGUMENT, "group_local: bad device %d", d);
        hub->dev.push_back(d);
    }
    for (int r = 0; r < world; ++r)
        for (int q = 0; q < world; ++q) {
            const int a = hub->dev[(size_t)r], b = hub->dev[(size_t)q];
            int can = 0;
            if (a != b && cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
                DevGuard g(a);
                cudaDeviceEnablePeerAccess(b, 0);
                cudaGetLastError();  // already enabled is fine
            }
        }
    for (int r = 0; r < world; ++r) {
        DevGuard g(hub->dev[(size_t)r]);
        auto t = std::make_unique<LocalTransport>();
        t->world = world;
        t->rank = r;
        t->device = hub->dev[(size_t)r];
        t->hub = hub;
        FFDP_CHECK_CUDA(cudaEventCreateWithFlags(&hub->post[(size_t)r].ready, cudaEventDisableTiming));
        FFDP_CHECK_CUDA(cudaEventCreateWithFlags(&hub->post[(size_t)r].done, cudaEventDisableTiming));
        out[r] = new ffdp_group_s{std::move(t)};
    }
    return FFDP_OK;
}

int ffdp_group_destroy(ffdp_group g) {
    if (!g) return set_error(FFDP_INVALID_ARGUMENT, "group_destroy: null group");
    delete g;
    return FFDP_OK;
}

int ffdp_group_info(ffdp_group g, int* world, int* rank, int* device) {
    if (!g) return set_error(FFDP_INVALID_ARGUMENT, "group_info: null group");
    if (world) *world = g->t->world;
    if (rank) *rank = g->t->rank;
    if (device) *device = g->t->device;
    return FFDP_OK;
}

int ffdp_plan_create(ffdp_group g, ffdp_dims global, const ffdp_plan_params* prm, ffdp_plan* out) {
    if (!g || !prm || !out) return set_error(FFDP_INVALID_ARGUMENT, "plan_create: null argument");
    Transport* t = g->t.get();
    if (global.nx < 2 || global.ny < 2 || global.nz < 2)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_create: lattice must be at least 2 per axis");
    if (global.nz < t->world) return set_error(FFDP_INVALID_ARGUMENT, "plan_create: fewer planes than ranks");
    if (prm->loss_kind != 0 && prm->loss_kind != 1)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_create: loss_kind must be 0 (LNCC) or 1 (MI)");
    if (prm->loss_kind == 0 && prm->window != 7)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_create: the fused LNCC step takes window 7");
    if (prm->loss_kind == 1 && prm->kernel.kind != FFDP_PARZEN_BSPLINE3)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_create: the MI plan takes the B-spline Parzen kernel");
    if (prm->margin_planes < 0) return set_error(FFDP_INVALID_ARGUMENT, "plan_create: negative margin");
    DevGuard dg(t->device);
    auto P = std::make_unique<ffdp_plan_s>();
    P->tr = t;
    P->world = t->world;
    P->rank = t->rank;
    P->dev = t->device;
    P->global = global;
    P->prm = *prm;
    P->lncc = prm->loss_kind == 0;
    P->B = P->lncc ? 0 : prm->kernel.bins;
    shard_range(global.nz, P->world, P->rank, P->lo, P->hi);
    // halo planes of F, u and g_u: the LNCC window radius and the warp update's tap radius
    if (prm->warp_halo < 0 || prm->warp_halo > 16)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_create: warp_halo must be in [0, 16]");
    const int pad = std::max(P->lncc ? prm->window / 2 : 0, (int)prm->warp_halo);
    P->hlo = P->rank > 0 ? pad : 0;
    P->hhi = P->rank < P->world - 1 ? pad : 0;
    // halo_exchange (fabric.hpp:321-326): a neighbour thinner than the halo is an error
    for (int q : {P->rank - 1, P->rank + 1}) {
        if (q < 0 || q >= P->world) continue;
        int64_t a, b;
        shard_range(global.nz, P->world, q, a, b);
        if (b - a < pad) return set_error(FFDP_INVALID_ARGUMENT, "plan_create: halo exceeds neighbor thickness");
    }
    P->plane = global.nx * global.ny;
    P->n_total = P->plane * global.nz;
    P->scale_exp = mi_bs_scale_exp(P->n_total);
    // sampler args of the global lattice (the slab descriptors say which planes a buffer holds)
    ffdp_sampler_args& a = P->ga;
    for (int i = 0; i < 9; ++i) a.A[i] = prm->A[i];
    for (int i = 0; i < 3; ++i) {
        a.t[i] = prm->t[i];
        a.S[i] = 1.0;
        a.x_min[i] = -1.0;
        a.x_max[i] = 1.0;
    }
    const char* why = nullptr;
    if (!valid_args(a, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "bad affine");
    FFDP_CHECK_CUDA(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
    FFDP_CHECK_CUDA(cudaStreamCreateWithFlags(&P->cst, cudaStreamNonBlocking));
    FFDP_CHECK_CUDA(cudaEventCreateWithFlags(&P->ev_u, cudaEventDisableTiming));
    FFDP_CHECK_CUDA(cudaEventCreateWithFlags(&P->ev_halo, cudaEventDisableTiming));
    FFDP_CHECK_CUDA(cudaMallocHost(&P->host, 2 * sizeof(double)));
    const int64_t n_in = P->plane * P->th();
    PLAN_TRY(P->f_h.alloc(sizeof(float) * P->plane * P->nb()));
    PLAN_TRY(P->u_h.alloc(sizeof(float) * 3 * P->plane * P->nb()));
    PLAN_TRY(P->g_h.alloc(sizeof(float) * 3 * P->plane * P->nb()));
    FFDP_CHECK_CUDA(cudaMemset(P->g_h.p, 0, P->g_h.bytes));
    if (prm->warp_halo > 0) {
        // the warp update: the smoothed u (ping-pong with u_h) and the Adam moments
        PLAN_TRY(P->u_h2.alloc(sizeof(float) * 3 * P->plane * P->nb()));
        FFDP_CHECK_CUDA(cudaMemset(P->u_h2.p, 0, P->u_h2.bytes));
        PLAN_TRY(P->m1.alloc(sizeof(float) * 3 * n_in));
        PLAN_TRY(P->m2.alloc(sizeof(float) * 3 * n_in));
    }
    PLAN_TRY(P->m_own.alloc(sizeof(float) * n_in));
    FFDP_CHECK_CUDA(cudaMemset(P->u_h.p, 0, P->u_h.bytes));
    PLAN_TRY(P->ranges.alloc(4 * sizeof(float)));
    PLAN_TRY(P->rng64.alloc(4 * sizeof(double)));
    PLAN_TRY(P->red.alloc(2 * sizeof(double)));
    if (P->lncc) {
        PLAN_TRY(P->hist.alloc(sizeof(int64_t)));
        PLAN_TRY(P->lws.alloc((size_t)lncc3_workspace_bytes(P->bd(), P->slab(P->lo, P->hi))));
    } else {
        const int B = P->B;
        PLAN_TRY(P->hist.alloc(sizeof(unsigned long long) * (B * B + 1)));
        PLAN_TRY(P->raw.alloc(sizeof(double) * (B * B + 2 * B)));
        PLAN_TRY(P->table.alloc(sizeof(double) * (2 * B * B + 2 * B + 4)));
        if (prm->records) {
            // pass-1 records (16 B per interior voxel) when they fit with 4 GiB to spare
            size_t fr = 0, tot = 0;
            FFDP_CHECK_CUDA(cudaMemGetInfo(&fr, &tot));
            const size_t rb = sizeof(float) * 4 * (size_t)n_in;
            if (fr > rb + (size_t(4) << 30)) PLAN_TRY(P->rec.alloc(rb));
        }
    }
    *out = P.release();
    return FFDP_OK;
}

int ffdp_plan_destroy(ffdp_plan p) {
    if (!p) return set_error(FFDP_INVALID_ARGUMENT, "plan_destroy: null plan");
    {
        DevGuard dg(p->dev);
        cudaStreamSynchronize(p->st);
        cudaStreamSynchronize(p->cst);
        for (DBuf* b : {&p->f_h, &p->u_h, &p->u_h2, &p->g_h, &p->m1, &p->m2, &p->m_own, &p->stage, &p->win, &p->ranges, &p->rng64, &p->red,
                        &p->hist, &p->raw, &p->table, &p->lws, &p->rec, &p->ext, &p->req})
            b->release();
        if (p->host) cudaFreeHost(p->host);
        cudaEventDestroy(p->ev_u);
        cudaEventDestroy(p->ev_halo);
        cudaStreamDestroy(p->st);
        cudaStreamDestroy(p->cst);
    }
    delete p;
    return FFDP_OK;
}

int ffdp_plan_slab(ffdp_plan p, int64_t* lo, int64_t* hi) {
    if (!p) return set_error(FFDP_INVALID_ARGUMENT, "plan_slab: null plan");
    if (lo) *lo = p->lo;
    if (hi) *hi = p->hi;
    return FFDP_OK;
}

void* ffdp_plan_stream(ffdp_plan p) { return p ? (void*)p->st : nullptr; }
float* ffdp_plan_u(ffdp_plan p) { return p ? p->u_h.as<float>() + 3 * p->hlo * p->plane : nullptr; }
float* ffdp_plan_g_u(ffdp_plan p) { return p ? p->g_int() : nullptr; }

int ffdp_plan_window(ffdp_plan p, int64_t* z0, int64_t* z1, int64_t* fetches) {
    if (!p) return set_error(FFDP_INVALID_ARGUMENT, "plan_window: null plan");
    if (z0) *z0 = p->wz0;
    if (z1) *z1 = p->wz1;
    if (fetches) *fetches = p->fetches;
    return FFDP_OK;
}

int ffdp_plan_load(ffdp_plan p, const float* f_slab, const float* m_slab) {
    if (!p || !f_slab || !m_slab) return set_error(FFDP_INVALID_ARGUMENT, "plan_load: null argument");
    DevGuard dg(p->dev);
    const size_t bytes = sizeof(float) * p->plane * p->th();
    FFDP_CHECK_CUDA(cudaMemcpyAsync(p->f_h.as<float>() + p->hlo * p->plane, f_slab, bytes, cudaMemcpyDefault, p->st));
    FFDP_CHECK_CUDA(cudaMemcpyAsync(p->m_own.p, m_slab, bytes, cudaMemcpyDefault, p->st));
    PLAN_TRY(halo_swap(p, p->f_h.as<float>(), 1, p->st));
    if (p->lncc) {
        // one intensity frame on every rank: it fixes the exact fixed-point moment sums
        PLAN_TRY(ffdp_minmax(p->f_h.as<float>() + p->hlo * p->plane, p->plane * p->th(), p->ranges.as<float>(), p->st));
        PLAN_TRY(ffdp_minmax(p->m_own.as<float>(), p->plane * p->th(), p->ranges.as<float>() + 2, p->st));
        k_ranges_pack<<<1, 32, 0, p->st>>>(p->ranges.as<float>(), p->rng64.as<double>());
        PLAN_TRY(p->tr->allreduce(p->rng64.p, 4, Dt::F64, Op::Min, p->st));
        k_ranges_unpack<<<1, 32, 0, p->st>>>(p->rng64.as<double>(), p->ranges.as<float>());
    }
    // a new scale: fresh Adam moments (registration.hpp:270-273 builds AdamState per scale)
    p->adam_step = 0;
    if (p->m1.p) {
        FFDP_CHECK_CUDA(cudaMemsetAsync(p->m1.p, 0, p->m1.bytes, p->st));
        FFDP_CHECK_CUDA(cudaMemsetAsync(p->m2.p, 0, p->m2.bytes, p->st));
    }
    int64_t a, b;
    affine_z_range(p, a, b);
    p->fetches = 0;
    PLAN_TRY(fetch_window(p, a, b));
    p->loaded = true;
    return check_launch("plan_load");
}

int ffdp_plan_step(ffdp_plan p, int sync, double* loss) {
    PLAN_TRY(check_plan(p));
    DevGuard dg(p->dev);
    if (!sync) return launch_step(p);
    for (int attempt = 0; attempt < 5; ++attempt) {
        PLAN_TRY(launch_step(p));
        FFDP_CHECK_CUDA(cudaStreamSynchronize(p->st));
        if (p->host[1] == 0.0) {
            if (loss) *loss = loss_of(p);
            return FFDP_OK;
        }
        PLAN_TRY(widen(p));  // every rank sees the same summed miss count: all widen together
    }
    return set_error(FFDP_RUNTIME, "plan_step: the moving window kept missing");
}

int ffdp_plan_warp_update(ffdp_plan p, double lr_norm, const double* taps_grad, int ntaps_grad,
                          const double* taps_warp, int ntaps_warp) {
    PLAN_TRY(check_plan(p));
    if (!p->m1.p) return set_error(FFDP_LOGIC, "plan_warp_update: the plan was created with warp_halo = 0");
    if (!taps_grad || !taps_warp || ntaps_grad < 1 || ntaps_warp < 1 || ntaps_grad % 2 == 0 || ntaps_warp % 2 == 0)
        return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: kernel must be odd");
    const int rg = ntaps_grad / 2, rw = ntaps_warp / 2;
    if (rg > p->prm.warp_halo || rw > p->prm.warp_halo)
        return set_error(FFDP_INVALID_ARGUMENT, "plan_warp_update: taps wider than the plan's warp_halo");
    DevGuard dg(p->dev);
    cudaStream_t st = p->st;
    const int64_t pl3 = 3 * p->plane;
    // registration.hpp:313: g_s = gp_convolve(g_u, taps_grad, renormalize) with rg halo planes
    // (halo_exchange, fabric.hpp:315-370), fused with adam_step(u, g_s) (adam.hpp:30-50)
    PLAN_TRY(halo_swap(p, p->g_h.as<float>(), 3, st, rg));
    const int64_t glo = p->hlo > 0 ? rg : 0, ghi = p->hhi > 0 ? rg : 0;
    const ffdp_dims gd{p->global.nx, p->global.ny, glo + p->th() + ghi};
    const ffdp_slab gs{p->lo - glo, gd.nz, p->lo, p->hi, p->global.nz};
    float* u_int = p->u_h.as<float>() + p->hlo * pl3;
    ++p->adam_step;
    PLAN_TRY(ffdp_sobolev_adam(p->g_h.as<float>() + (p->hlo - glo) * pl3, u_int, p->m1.as<float>(), p->m2.as<float>(),
                               gd, gs, taps_grad, ntaps_grad, lr_norm, 0.9, 0.999, 1e-8, p->adam_step, st));
    // registration.hpp:316: u = gp_convolve(u, taps_warp, renormalize) with rw halo planes
    PLAN_TRY(halo_swap(p, p->u_h.as<float>(), 3, st, rw));
    const int64_t wlo = p->hlo > 0 ? rw : 0, whi = p->hhi > 0 ? rw : 0;
    const ffdp_dims wd{p->global.nx, p->global.ny, wlo + p->th() + whi};
    const ffdp_slab ws{p->lo - wlo, wd.nz, p->lo, p->hi, p->global.nz};
    PLAN_TRY(ffdp_gp_convolve(p->u_h.as<float>() + (p->hlo - wlo) * pl3, p->u_h2.as<float>() + p->hlo * pl3, wd, ws, 3,
                              taps_warp, ntaps_warp, 1, st));
    std::swap(p->u_h, p->u_h2);  // ffdp_plan_u now points at the smoothed field
    return check_launch("plan_warp_update");
}

int ffdp_plan_result(ffdp_plan p, double* loss, double* misses) {
    PLAN_TRY(check_plan(p));
    DevGuard dg(p->dev);
    FFDP_CHECK_CUDA(cudaStreamSynchronize(p->st));
    if (loss) *loss = loss_of(p);
    if (misses) *misses = p->host[1];
    return FFDP_OK;
}

}  // extern "C"
