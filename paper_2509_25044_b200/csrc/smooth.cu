// smooth.cu -- the warp update of the deformable step (registration.hpp:313-317):
//
//   g_s = gp_convolve(g_u, gaussian(sigma_grad), renormalize)      distops.hpp:54-101
//   adam_step(u, g_s, state, lr_norm)                               adam.hpp:30-50
//   u   = gp_convolve(u, gaussian(sigma_warp), renormalize)
//
// as two z-marching stencil kernels over a z-slab:
//   k_smooth<R, CH, ADAM>: separable (2R+1)^3 convolution of a CH-channel field whose
//   buffer holds the slab plus R halo planes (halo_exchange, fabric.hpp:315-370). A CTA
//   owns a 32 x 16 column tile and marches z: per input plane the haloed tile is loaded
//   once (coalesced rows of CH * (32 + 2R) floats) into shared memory, convolved along x
//   and y there, and pushed into a per-thread register ring of 2R+1 xy-smoothed planes;
//   the z taps then finish the output R planes behind. With ADAM the epilogue is the
//   bias-corrected Adam update of the voxel's u, m1, m2 (in place): the smoothed gradient
//   never touches HBM. Otherwise the epilogue stores the smoothed value.
//
// Boundary semantics (smoothing.hpp:52-94): zero_pad drops out-of-lattice taps;
// renormalize divides by the sum of the in-lattice taps of each axis. Both depend only on
// the global coordinate (the halo-padded z block of a shard sees the same taps as the
// unsharded volume, smoothing.hpp:10-13), and the per-axis divisors factor out of the
// separable sum, so they are applied once per output: 1 / (W_x(gx) W_y(gy) W_z(gz)).
//
// HBM traffic per voxel: ADAM reads g_u, u, m1, m2 and writes u, m1, m2 (84 B, 3
// channels); STORE reads and writes one field (24 B). The x/y halo re-reads of a plane
// come from L2 (neighbouring tiles march the same planes).
#include <algorithm>
#include <cmath>

#include "ffdp_common.cuh"

namespace ffdp {
namespace sm {

constexpr int TX = 32, TY = 16, NT = TX * TY;  // one output column per thread
constexpr int kMaxR = 4;

struct Params {
    const float* in;   // buffer planes [buf_z0, buf_z0 + buf_nz), CH per voxel
    float* out;        // interior planes [z_begin, z_end) (STORE), or null
    float* u;          // ADAM: interior planes, updated in place
    float* m1;
    float* m2;
    int32_t nx, ny;
    int64_t plane, buf_z0, buf_z1, z_begin, z_end, nz_global;
    int32_t zchunk;
    float w[2 * kMaxR + 1];
    int renorm;
    // Adam (adam.hpp:30-50): u -= lr/c1 * m / (sqrt(v / c2) + eps)
    float b1, b2, omb1, omb2, lr_c1, inv_c2, eps;
};

// In-lattice tap sum of the window of global coordinate g on an axis of n voxels.
template <int R>
__device__ __forceinline__ float wsum(const Params& P, int64_t g, int64_t n) {
    float s = 0.0f;
#pragma unroll
    for (int k = -R; k <= R; ++k) s += (g + k >= 0 && g + k < n) ? P.w[k + R] : 0.0f;
    return s;
}

template <int R, int CH>
struct Smem {
    static constexpr int HX = TX + 2 * R, HY = TY + 2 * R, ROW = CH * HX;
    float raw[2][HY][ROW];  // haloed input plane (double-buffered: the next plane loads during this one)
    float X[HY][TX * CH];   // x-convolved rows (the top barrier of the next plane protects it)
};

template <int R, int CH, bool ADAM>
__global__ void __launch_bounds__(NT, 2) k_smooth(const Params P) {
    using S = Smem<R, CH>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& sm = *reinterpret_cast<S*>(smem_raw);
    const int t = threadIdx.x;
    const int ox = t % TX, oy = t / TX;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int64_t zc0 = P.z_begin + (int64_t)blockIdx.z * P.zchunk;
    const int64_t zc1 = min(P.z_end, zc0 + P.zchunk);
    if (zc0 >= zc1) return;
    const int gx = x0 + ox, gy = y0 + oy;
    const bool own = gx < P.nx && gy < P.ny;
    // renormalize (smoothing.hpp:75-90): divide by the in-lattice tap sum of each axis
    // (the full tap sum for full windows)
    const float wxy = P.renorm ? wsum<R>(P, gx, P.nx) * wsum<R>(P, gy, P.ny) : 1.0f;
    float ring[2 * R + 1][CH];
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) ring[k][c] = 0.0f;

    // the haloed tile of plane p: rows of CH * HX consecutive floats (zero outside the
    // lattice, and for planes outside the volume)
    auto load = [&](int64_t p, int buf) {
        const bool pin = p >= 0 && p < P.nz_global;
        const float* src = P.in + (pin ? (p - P.buf_z0) * P.plane * CH : 0);
        for (int q = t; q < S::HY * S::ROW; q += NT) {
            const int r = q / S::ROW, e = q - r * S::ROW;
            const int yy = y0 - R + r;
            const int xe = (x0 - R) * CH + e;  // element index along the row
            const bool ok = pin && yy >= 0 && yy < P.ny && xe >= 0 && xe < P.nx * CH;
            sm.raw[buf][r][e] = ok ? __ldg(src + (int64_t)yy * P.nx * CH + xe) : 0.0f;
        }
    };

    const int64_t pstart = zc0 - R, pend = zc1 + R;  // input planes of this chunk
    load(pstart, 0);
    int buf = 0;
    for (int64_t p = pstart; p < pend; ++p, buf ^= 1) {
        __syncthreads();  // raw[buf] complete; X free
        if (p + 1 < pend) load(p + 1, buf ^ 1);
        // x taps: rows of the haloed tile, TX outputs each
        for (int q = t; q < S::HY * TX; q += NT) {
            const int r = q / TX, x = q - r * TX;
            float acc[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) acc[c] = 0.0f;
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k)
#pragma unroll
                for (int c = 0; c < CH; ++c) acc[c] = fmaf(P.w[k], sm.raw[buf][r][(x + k) * CH + c], acc[c]);
#pragma unroll
            for (int c = 0; c < CH; ++c) sm.X[r][x * CH + c] = acc[c];
        }
        __syncthreads();
        // y taps into the z ring
#pragma unroll
        for (int k = 0; k < 2 * R; ++k)
#pragma unroll
            for (int c = 0; c < CH; ++c) ring[k][c] = ring[k + 1][c];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            float acc = 0.0f;
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k) acc = fmaf(P.w[k], sm.X[oy + k][ox * CH + c], acc);
            ring[2 * R][c] = acc;
        }
        // z taps: output plane q = p - R
        const int64_t q = p - R;
        if (q < zc0 || !own) continue;
        const float inv = P.renorm ? 1.0f / (wxy * wsum<R>(P, q, P.nz_global)) : 1.0f;
        const int64_t o = ((q - P.z_begin) * P.plane + (int64_t)gy * P.nx + gx) * CH;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            float v = 0.0f;
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k) v = fmaf(P.w[k], ring[k][c], v);
            v *= inv;
            if (ADAM) {
                const float m = fmaf(P.b1, P.m1[o + c], P.omb1 * v);
                const float s2 = fmaf(P.b2, P.m2[o + c], P.omb2 * v * v);
                P.m1[o + c] = m;
                P.m2[o + c] = s2;
                P.u[o + c] -= P.lr_c1 * m / (sqrtf(s2 * P.inv_c2) + P.eps);
            } else {
                P.out[o + c] = v;
            }
        }
    }
}

// Planes per z chunk: the fewest (waves x planes-with-halo) over chunk counts.
inline int32_t pick_zchunk(int64_t tiles, int64_t nzs, int64_t capacity, int R) {
    int64_t best = 1, best_cost = INT64_MAX;
    for (int64_t ch = 1; ch <= std::min<int64_t>(nzs, 256); ++ch) {
        const int64_t zc = (nzs + ch - 1) / ch;
        const int64_t n = (nzs + zc - 1) / zc;
        const int64_t waves = (tiles * n + capacity - 1) / capacity;
        const int64_t cost = waves * (zc + 2 * R);
        if (cost < best_cost) best_cost = cost, best = zc;
    }
    return (int32_t)best;
}

template <int R, int CH, bool ADAM>
int launch(Params P, cudaStream_t st) {
    const size_t smem = sizeof(Smem<R, CH>);
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(k_smooth<R, CH, ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_smooth<R, CH, ADAM>, NT, smem);
        per_sm = std::max(per_sm, 1);
    }
    const int64_t tx = (P.nx + TX - 1) / TX, ty = (P.ny + TY - 1) / TY;
    const int64_t nzs = P.z_end - P.z_begin;
    P.zchunk = pick_zchunk(tx * ty, nzs, (int64_t)per_sm * num_sms(), R);
    const int64_t chunks = (nzs + P.zchunk - 1) / P.zchunk;
    if (ty > 65535 || chunks > 65535) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: grid too large");
    k_smooth<R, CH, ADAM><<<dim3((unsigned)tx, (unsigned)ty, (unsigned)chunks), NT, smem, st>>>(P);
    return check_launch(ADAM ? "sobolev_adam" : "gp_convolve");
}

template <bool ADAM>
int dispatch(const Params& P, int R, int CH, cudaStream_t st) {
    if (CH == 3) {
        switch (R) {
            case 0: return launch<0, 3, ADAM>(P, st);
            case 1: return launch<1, 3, ADAM>(P, st);
            case 2: return launch<2, 3, ADAM>(P, st);
            case 3: return launch<3, 3, ADAM>(P, st);
            case 4: return launch<4, 3, ADAM>(P, st);
        }
    } else if (!ADAM) {
        switch (R) {
            case 0: return launch<0, 1, false>(P, st);
            case 1: return launch<1, 1, false>(P, st);
            case 2: return launch<2, 1, false>(P, st);
            case 3: return launch<3, 1, false>(P, st);
            case 4: return launch<4, 1, false>(P, st);
        }
    }
    return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: radius %d / %d channels not supported (radius <= %d)", R,
                     CH, kMaxR);
}

// Common validation: odd taps, radius <= kMaxR, a slab whose buffer holds every plane the
// window needs (the halo exchange's job), compute planes inside the buffer.
int make_params(Params& P, const float* in, ffdp_dims d, ffdp_slab s, int channels, const double* taps, int ntaps,
                int mode) {
    if (!in || !taps) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: null pointer");
    if (ntaps < 1 || ntaps % 2 == 0) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: kernel must be odd");
    const int R = ntaps / 2;
    if (R > kMaxR) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: at most %d taps", 2 * kMaxR + 1);
    if (channels != 1 && channels != 3) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: 1 or 3 channels");
    if (d.nx < 1 || d.ny < 1 || s.z_begin >= s.z_end || s.z_begin < s.buf_z0 || s.z_end > s.buf_z0 + s.buf_nz ||
        s.buf_z0 < 0 || s.buf_z0 + s.buf_nz > s.nz_global || d.nz != s.buf_nz)
        return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: inconsistent slab");
    // fabric.hpp:321-326: the halo must cover the window (else the neighbour was too thin)
    if (s.buf_z0 > std::max<int64_t>(0, s.z_begin - R) || s.buf_z0 + s.buf_nz < std::min(s.nz_global, s.z_end + R))
        return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: buffer lacks the %d halo planes", R);
    if (d.nx * channels >= (1LL << 31)) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: rows too long");
    P = Params{};
    P.in = in;
    P.nx = (int32_t)d.nx;
    P.ny = (int32_t)d.ny;
    P.plane = d.nx * d.ny;
    P.buf_z0 = s.buf_z0;
    P.buf_z1 = s.buf_z0 + s.buf_nz;
    P.z_begin = s.z_begin;
    P.z_end = s.z_end;
    P.nz_global = s.nz_global;
    for (int i = 0; i < ntaps; ++i) {
        P.w[i] = (float)taps[i];

    }
    P.renorm = mode == 1;
    return FFDP_OK;
}

}  // namespace sm
}  // namespace ffdp

using namespace ffdp;

extern "C" {

int ffdp_gp_convolve(const float* in, float* out, ffdp_dims buf_dims, ffdp_slab slab, int channels, const double* taps,
                     int ntaps, int mode, void* stream) {
    sm::Params P;
    if (int rc = sm::make_params(P, in, buf_dims, slab, channels, taps, ntaps, mode)) return rc;
    if (!out) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: null pointer");
    P.out = out;
    return sm::dispatch<false>(P, ntaps / 2, channels, (cudaStream_t)stream);
}

int ffdp_sobolev_adam(const float* g_u, float* u, float* m1, float* m2, ffdp_dims buf_dims, ffdp_slab slab,
                      const double* taps, int ntaps, double lr, double beta1, double beta2, double eps, int64_t step,
                      void* stream) {
    sm::Params P;
    if (int rc = sm::make_params(P, g_u, buf_dims, slab, 3, taps, ntaps, 1)) return rc;
    if (!u || !m1 || !m2) return set_error(FFDP_INVALID_ARGUMENT, "adam_step: null pointer");
    if (step < 1 || !(lr > 0) || !(beta1 >= 0 && beta1 < 1) || !(beta2 >= 0 && beta2 < 1) || !(eps >= 0))
        return set_error(FFDP_INVALID_ARGUMENT, "adam_step: bad hyper-parameters");
    P.u = u;
    P.m1 = m1;
    P.m2 = m2;
    // adam.hpp:37-49 (bias corrections of step `step`, in fp64 on the host)
    const double c1 = 1.0 - std::pow(beta1, (double)step), c2 = 1.0 - std::pow(beta2, (double)step);
    P.b1 = (float)beta1;
    P.b2 = (float)beta2;
    P.omb1 = (float)(1.0 - beta1);
    P.omb2 = (float)(1.0 - beta2);
    P.lr_c1 = (float)(lr / c1);
    P.inv_c2 = (float)(1.0 / c2);
    P.eps = (float)eps;
    return sm::dispatch<true>(P, ntaps / 2, 3, (cudaStream_t)stream);
}

}  // extern "C"
