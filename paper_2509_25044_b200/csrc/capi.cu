// capi.cu -- error state, host-side geometry folding, scratch memory and small utility
// kernels of the libffdp C ABI (include/ffdp.h).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <mutex>

#include "ffdp_common.cuh"

namespace ffdp {

static thread_local char g_error[1024] = "";

int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(FFDP_CUDA, "%s: launch failed: %s", what, cudaGetErrorString(e));
    return FFDP_OK;
}

bool valid_args(const ffdp_sampler_args& a, const char** why) {
    // SamplerArgs::validate (sampler.hpp:31-36)
    for (double v : a.A)
        if (!std::isfinite(v)) {
            *why = "SamplerArgs: non-finite affine";
            return false;
        }
    for (int c = 0; c < 3; ++c)
        if (!(a.S[c] > 0)) {
            *why = "SamplerArgs: S must be positive";
            return false;
        }
    for (int c = 0; c < 3; ++c)
        if (!(a.x_min[c] < a.x_max[c])) {
            *why = "SamplerArgs: invalid bounds";
            return false;
        }
    return true;
}

Geom make_geom(const ffdp_image_window& img, const ffdp_dims& out, const ffdp_sampler_args& a) {
    Geom g;
    std::memset(&g, 0, sizeof(g));
    const int64_t N[3] = {img.dims.nx, img.dims.ny, img.dims.nz};
    const int64_t on[3] = {out.nx, out.ny, out.nz};
    for (int c = 0; c < 3; ++c) {
        // lattice_coord (geometry.hpp:99-104): X_c = lo + (hi - lo) * i / (n - 1)
        g.Xlo[c] = a.x_min[c];
        g.Xstep[c] = on[c] > 1 ? (a.x_max[c] - a.x_min[c]) / (double)(on[c] - 1) : 0.0;
        g.on[c] = (int32_t)on[c];
    }
    for (int r = 0; r < 3; ++r) {
        // fractional index f = (xsrc + 1) * 0.5 * (N - 1)  (sampler.hpp:104)
        const double h = 0.5 * (double)(N[r] - 1);
        double k = a.t[r] + 1.0;
        for (int c = 0; c < 3; ++c) {
            k += a.A[3 * r + c] * g.Xlo[c];
            g.P[3 * r + c] = h * a.A[3 * r + c] * g.Xstep[c];
        }
        g.K[r] = h * k;
        g.Q[r] = h * a.S[r];
        g.dscale[r] = (float)(a.S[r] * h);
        g.hn[r] = (float)h;
        g.n[r] = (int32_t)N[r];
    }
    g.wz0 = (int32_t)img.z_begin;
    g.wz1 = (int32_t)img.z_end;
    g.pad = (int32_t)img.pad;
    if (img.pad == 2) {
        g.sy = img.dims.nx + 4;
        g.sz = (img.dims.nx + 4) * (img.dims.ny + 4);
        g.img = img.data ? img.data + 2 * g.sz + 2 * g.sy + 2 : nullptr;
    } else {
        g.sy = img.dims.nx;
        g.sz = img.dims.nx * img.dims.ny;
        g.img = img.data;
    }
    return g;
}

ParzenDev make_parzen_dev(const ffdp_parzen& k) {
    ParzenDev p;
    p.kind = k.kind;
    p.bins = k.bins;
    p.sigma = k.sigma;
    p.radius = k.radius;
    p.norm = k.norm;
    p.inv_sigma2_f = k.sigma > 0 ? (float)(1.0 / (k.sigma * k.sigma)) : 0.0f;
    p.inv_sigma_f = k.sigma > 0 ? (float)(1.0 / k.sigma) : 0.0f;
    p.norm_f = (float)k.norm;
    return p;
}

int num_sms() {
    static thread_local int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

std::mutex& once_mutex() {
    static std::mutex m;
    return m;
}

// The library's own stream-ordered pool per device (never the process's default pool, so
// PyTorch's caching allocator and other cudaMallocAsync users keep their own behaviour).
// Freed scratch stays cached up to kPoolKeep bytes: with a release threshold of 0 every
// synchronisation handed multi-GB scratch (resample_scale, workspaces) back and the next
// call paid a fresh mapping. ffdp_scratch_trim() returns the cache to the device.
static constexpr uint64_t kPoolKeep = 4ull << 30;
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64];

cudaMemPool_t device_pool(int dev) {
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t thr = kPoolKeep;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool[dev] = p;
    }
    return g_pool[dev];
}

void* scratch_alloc(size_t bytes, cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    cudaMemPool_t pool = device_pool(dev);
    if (!pool) return nullptr;
    void* p = nullptr;
    if (cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, s) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void scratch_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// ------------------------------------------------------------ utility kernels
template <int NT>
__global__ void __launch_bounds__(NT) k_reduce_sum(const double* in, int64_t n, double* out) {
    __shared__ double sm[NT / 32];
    double acc = 0;
    for (int64_t i = threadIdx.x; i < n; i += NT) acc += in[i];
    const double r = block_sum<NT>(acc, sm);
    if (threadIdx.x == 0) *out = r;
}

// Value range of a buffer. A NaN anywhere makes both bounds NaN (fminf / fmaxf would drop
// it): callers derive intensity frames from the range, and a non-finite input must reach
// the loss as NaN, as it does in the reference's arithmetic (registration.hpp:300-305).
template <int NT>
__global__ void __launch_bounds__(NT) k_minmax_partial(const float* in, int64_t n, float* part) {
    float lo = INFINITY, hi = -INFINITY;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const float v = in[i];
        bad |= v != v;
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    __shared__ float sl[NT / 32], sh[NT / 32];
    __shared__ int sb[NT / 32];
    if ((threadIdx.x & 31) == 0) {
        sl[threadIdx.x >> 5] = lo;
        sh[threadIdx.x >> 5] = hi;
        sb[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < NT / 32; ++i) {
            lo = fminf(lo, sl[i]);
            hi = fmaxf(hi, sh[i]);
            bad |= sb[i];
        }
        part[2 * blockIdx.x] = bad ? NAN : lo;
        part[2 * blockIdx.x + 1] = bad ? NAN : hi;
    }
}

__global__ void k_minmax_final(const float* part, int nb, float* out) {
    float lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    for (int i = 0; i < nb; ++i) {
        bad |= part[2 * i] != part[2 * i];
        lo = fminf(lo, part[2 * i]);
        hi = fmaxf(hi, part[2 * i + 1]);
    }
    out[0] = bad ? NAN : lo;
    out[1] = bad ? NAN : hi;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_z_extent(Geom g, const float* u, int64_t n_out, int64_t* out) {
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    const int64_t plane = (int64_t)g.on[0] * g.on[1];
    for (int64_t v = blockIdx.x * (int64_t)NT + threadIdx.x; v < n_out; v += (int64_t)gridDim.x * NT) {
        const int32_t z = (int32_t)(v / plane);
        const int64_t r = v - (int64_t)z * plane;
        const int32_t y = (int32_t)(r / g.on[0]);
        const int32_t x = (int32_t)(r - (int64_t)y * g.on[0]);
        float u0 = 0, u1 = 0, u2 = 0;
        if (u) {
            u0 = u[3 * v];
            u1 = u[3 * v + 1];
            u2 = u[3 * v + 2];
        }
        const Cell c = resolve(g, x, y, z, u0, u1, u2);
        // only corners that can carry weight inside the lattice count (sampler.hpp:106-110)
        for (int bz = 0; bz < 2; ++bz) {
            const int64_t iz = c.i0[2] + bz;
            if (iz >= 0 && iz < g.n[2]) {
                lo = iz < lo ? iz : lo;
                hi = iz > hi ? iz : hi;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long l2 = __shfl_xor_sync(0xffffffffu, (long long)lo, o);
        const long long h2 = __shfl_xor_sync(0xffffffffu, (long long)hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin((long long*)&out[0], (long long)lo);
        atomicMax((long long*)&out[1], (long long)hi);
    }
}

__global__ void k_pad_window(const float* __restrict__ src, int64_t nx, int64_t ny, int64_t nzw,
                             float* __restrict__ dst) {
    const int64_t px = nx + 4, py = ny + 4, n = px * py * (nzw + 4);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % px - 2, y = (i / px) % py - 2, z = i / (px * py) - 2;
        dst[i] = (x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nzw) ? src[(z * ny + y) * nx + x] : 0.0f;
    }
}

__global__ void k_init_extent(int64_t* out) {
    out[0] = INT64_MAX;
    out[1] = INT64_MIN;
}

}  // namespace ffdp

using namespace ffdp;

extern "C" {

const char* ffdp_last_error(void) { return g_error; }

int ffdp_abi_version(void) { return FFDP_ABI_VERSION; }

int ffdp_scratch_trim(int64_t keep_bytes) {
    int dev = 0;
    FFDP_CHECK_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool = device_pool(dev);
    if (!pool) return set_error(FFDP_CUDA, "scratch_trim: no memory pool on device %d", dev);
    FFDP_CHECK_CUDA(cudaMemPoolTrimTo(pool, keep_bytes > 0 ? (size_t)keep_bytes : 0));
    return FFDP_OK;
}

int ffdp_device_check(void) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(FFDP_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) return set_error(FFDP_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    if (p.major != 10 || p.minor != 0)
        return set_error(FFDP_CUDA, "libffdp is built for sm_100a only; device %d is sm_%d%d (%s)", dev, p.major,
                         p.minor, p.name);
    return FFDP_OK;
}

int ffdp_reduce_sum_f64(const double* in, int64_t n, double* out, void* stream) {
    if (n < 0 || !out || (n > 0 && !in)) return set_error(FFDP_INVALID_ARGUMENT, "reduce_sum: bad arguments");
    k_reduce_sum<1024><<<1, 1024, 0, (cudaStream_t)stream>>>(in, n, out);
    return check_launch("reduce_sum");
}

int ffdp_minmax(const float* in, int64_t n, float* out, void* stream) {
    if (n <= 0 || !in || !out) return set_error(FFDP_INVALID_ARGUMENT, "minmax: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = (int)std::min<int64_t>(4 * num_sms(), (n + 255) / 256);
    float* part = (float*)scratch_alloc(sizeof(float) * 2 * nb, s);
    if (!part) return set_error(FFDP_CUDA, "minmax: scratch allocation failed");
    k_minmax_partial<256><<<nb, 256, 0, s>>>(in, n, part);
    k_minmax_final<<<1, 1, 0, s>>>(part, nb, out);
    scratch_free(part, s);
    return check_launch("minmax");
}

int ffdp_sampler_z_extent(const float* u, ffdp_dims out_dims, ffdp_dims m_dims, const ffdp_sampler_args* args,
                          int64_t* out, void* stream) {
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!out) return set_error(FFDP_INVALID_ARGUMENT, "z_extent: null output");
    ffdp_image_window w{nullptr, m_dims, 0, m_dims.nz, 0};
    const Geom g = make_geom(w, out_dims, *args);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = out_dims.nx * out_dims.ny * out_dims.nz;
    k_init_extent<<<1, 1, 0, s>>>(out);
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(8 * num_sms(), (n + 255) / 256));
    k_z_extent<256><<<nb, 256, 0, s>>>(g, u, n, out);
    return check_launch("z_extent");
}

int ffdp_pad_window(const float* src, ffdp_dims d, int64_t z_begin, int64_t z_end, float* dst, void* stream) {
    if (!src || !dst || d.nx < 1 || d.ny < 1 || z_begin < 0 || z_end > d.nz || z_begin >= z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "pad_window: bad arguments");
    const int64_t n = (d.nx + 4) * (d.ny + 4) * (z_end - z_begin + 4);
    const int nb = (int)std::min<int64_t>((n + 255) / 256, 16LL * num_sms());
    k_pad_window<<<nb, 256, 0, (cudaStream_t)stream>>>(src, d.nx, d.ny, z_end - z_begin, dst);
    return check_launch("pad_window");
}

int ffdp_parzen_make(int kind, int bins, double sigma_bins, ffdp_parzen* k) {
    // ParzenKernel constructors (mi.hpp:33-63) and check_normalization (mi.hpp:120-133)
    if (!k) return set_error(FFDP_INVALID_ARGUMENT, "parzen_make: null output");
    if (bins < 1) return set_error(FFDP_INVALID_ARGUMENT, "ParzenKernel: bins must be >= 1");
    if (kind < 0 || kind > 2) return set_error(FFDP_INVALID_ARGUMENT, "ParzenKernel: unknown kind %d", kind);
    k->kind = kind;
    k->bins = bins;
    k->sigma = 0;
    k->norm = 1.0;
    if (kind == FFDP_PARZEN_GAUSSIAN) {
        k->sigma = sigma_bins / bins;
        k->radius = 3.0 * k->sigma;
        const double erf_mass = std::erf(3.0 / std::sqrt(2.0));
        k->norm = 1.0 / (bins * k->sigma * std::sqrt(2.0 * 3.14159265358979323846) * erf_mass);
    } else if (kind == FFDP_PARZEN_BSPLINE3) {
        k->radius = 2.0 / bins;
    } else {
        k->radius = 0.5 / bins;
    }
    auto kappa = [&](double x) -> double {
        if (kind == FFDP_PARZEN_GAUSSIAN) {
            if (std::abs(x) > k->radius) return 0.0;
            const double z = x / k->sigma;
            return k->norm * std::exp(-0.5 * z * z);
        }
        if (kind == FFDP_PARZEN_BSPLINE3) {
            const double a = std::abs(x * bins);
            if (a < 1.0) return (4.0 - 6.0 * a * a + 3.0 * a * a * a) / 6.0;
            if (a < 2.0) return (2.0 - a) * (2.0 - a) * (2.0 - a) / 6.0;
            return 0.0;
        }
        return std::abs(x) < k->radius ? 1.0 : 0.0;
    };
    const int steps = 20000;
    const double h = 2.0 * k->radius / steps;
    double integral = 0;
    for (int i = 0; i <= steps; ++i) {
        const double x = -k->radius + i * h;
        integral += ((i == 0 || i == steps) ? 0.5 : 1.0) * kappa(x);
    }
    integral *= h * bins;
    if (std::abs(integral - 1.0) > 1e-3)
        return set_error(FFDP_LOGIC, "ParzenKernel: discrete integral deviates from 1");
    return FFDP_OK;
}

}  // extern "C"
