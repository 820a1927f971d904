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
#include <atomic>
#include <cmath>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ffdp_common.cuh"

// FFDP_SMOOTH_TMA = 1: the haloed input planes arrive by TMA (one 3-D tensor box per plane,
// OOB zero fill = the zero padding) when rows are 16-byte multiples; else per-thread cp.async
#ifndef FFDP_SMOOTH_TMA
#define FFDP_SMOOTH_TMA 1
#endif

namespace ffdp {
namespace sm {

constexpr int TX = 32, TY = 16, NT = TX * TY;  // one output column per thread
constexpr int kMaxR = 6;  // gaussian sigma <= 2 (resample_scale's anti-alias at factor 1/4)

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

constexpr int NSTAGE = 3;  // input planes in flight (cp.async ring)

template <int R, int CH>
struct __align__(128) Smem {
    // ROW: floats per row, with room for the up-to-3-float shift that 16-byte aligns the
    // row's first chunk (V16 loads); ROW is a multiple of 4 so every row starts aligned.
    // A stage is HY rows of ROW floats (the TMA box), padded to a 128-byte multiple.
    static constexpr int HX = TX + 2 * R, HY = TY + 2 * R, ROW = (CH * HX + 3 + 3) / 4 * 4;
    static constexpr int STAGE = (HY * ROW + 31) / 32 * 32;
    float raw[NSTAGE][STAGE];    // haloed input planes, filled by TMA / cp.async (zero outside)
    float X[HY][TX * CH];        // x-convolved rows (the top barrier of the next plane protects it)
    unsigned long long bar[NSTAGE];  // TMA: plane landed
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\tselp.u32 %0, 1, "
            "0, p;\n}"
            : "=r"(ok)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
}

// 4-byte asynchronous global -> shared copy; src_bytes = 0 writes a zero (no global read).
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int src_bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src, int src_bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// MODE 1 / 2 (V16): rows of CH * nx floats start 16-byte aligned, so the haloed tile row
// moves in 16-byte cp.async chunks (the row's first element sits `sh` floats into the stage
// row; chunks left of the lattice or past its end are zero-filled by src_bytes), or (MODE 2)
// the whole haloed plane is one TMA box issued by thread 0 (OOB zero fill), which leaves the
// other threads no copy instructions at all. MODE 0: 4-byte cp.async per element.
template <int R, int CH, bool ADAM, int MODE>
__global__ void __launch_bounds__(NT, 2) k_smooth(const __grid_constant__ CUtensorMap tmap, const Params P) {
    using S = Smem<R, CH>;
    constexpr bool V16 = MODE >= 1, TMA = MODE == 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
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
    float wfull = 0.0f;
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) wfull += P.w[k];
    const float inv_xy_full = 1.0f / (wxy * wfull);
    float ring[2 * R + 1][CH];
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) ring[k][c] = 0.0f;

    // The haloed tile of plane p, as rows of CH * HX consecutive floats, copied
    // asynchronously (zero outside the lattice and for planes outside the volume). A
    // thread's tile elements (or 16-byte chunks) are fixed for the whole z march: their
    // in-plane source offsets and byte counts are computed once. Each thread always
    // commits one group per plane (possibly empty) so the wait counts line up.
    const int e0 = (x0 - R) * CH;                 // the tile row's first element in the lattice row
    const int sh = V16 ? e0 - ((e0 >> 2) << 2) : 0;  // its float offset in the stage row
    constexpr int NCH = (S::ROW) / 4;              // chunks per stage row (V16)
    constexpr int NEL = V16 ? S::HY * NCH : S::HY * (CH * S::HX);
    constexpr int KL = (NEL + NT - 1) / NT;
    int32_t src_off[KL];
    int16_t dst_off[KL];  // float offset in a stage (-1: no element)
    int8_t src_bytes[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) {
        const int q = t + k * NT;
        if (V16) {
            const int r = q / NCH, c = q - r * NCH;
            dst_off[k] = (int16_t)(q < NEL ? r * S::ROW + 4 * c : -1);
            const int yy = y0 - R + r;
            const int a = ((e0 >> 2) << 2) + 4 * c;  // chunk start, a multiple of 4 (>= 0 or all left)
            const int nb = (q < NEL && yy >= 0 && yy < P.ny && a >= 0) ? min(max(P.nx * CH - a, 0), 4) * 4 : 0;
            src_off[k] = nb ? yy * P.nx * CH + a : 0;
            src_bytes[k] = (int8_t)nb;
        } else {
            const int r = q / (CH * S::HX), e = q - r * (CH * S::HX);
            dst_off[k] = (int16_t)(q < NEL ? r * S::ROW + e : -1);
            const int yy = y0 - R + r;
            const int xe = e0 + e;
            const bool ok = q < NEL && yy >= 0 && yy < P.ny && xe >= 0 && xe < P.nx * CH;
            src_off[k] = ok ? yy * P.nx * CH + xe : 0;
            src_bytes[k] = ok ? 4 : 0;
        }
    }
    if (TMA) {
        if (t == 0) {
#pragma unroll
            for (int s = 0; s < NSTAGE; ++s)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&sm.bar[s])) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    auto issue = [&](int64_t p, int stage) {
        if (TMA) {
            // planes outside the volume lie outside the buffer's z extent: zero filled
            if (t == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of the stage
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&sm.bar[stage])),
                             "r"((uint32_t)(S::HY * S::ROW * 4))
                             : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3, %4}], [%5];" ::"r"(saddr(&sm.raw[stage][0])),
                    "l"(&tmap), "r"(e0 - sh), "r"(y0 - R), "r"((int)(p - P.buf_z0)), "r"(saddr(&sm.bar[stage]))
                    : "memory");
            }
            return;
        }
        const bool pin = p >= 0 && p < P.nz_global;
        const float* src = P.in + (pin ? (p - P.buf_z0) * P.plane * CH : 0);
        asm("" : "+l"(src));  // one plane base; each copy is then one wide add of its offset
        float* dst = &sm.raw[stage][0];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            if (dst_off[k] >= 0) {
                const int nb = pin ? src_bytes[k] : 0;
                const float* sp = src + (uint32_t)src_off[k];
                if (V16)
                    cp_async16(dst + dst_off[k], sp, nb);
                else
                    cp_async4(dst + dst_off[k], sp, nb);
            }
        }
        cp_async_commit();
    };

    // x taps: a job is a run of XR outputs of one channel of one row, sliding over the
    // XR + 2R inputs in registers (runs of 8 measured no faster for R = 3); job order
    // (run, channel) inside a row keeps a row's lanes on distinct banks. A thread's jobs
    // are the same every plane: their stage / X offsets are computed once.
    constexpr int XR = 4, NJ = S::HY * CH * (TX / XR), XJ = (NJ + NT - 1) / NT;
    int32_t xj_in[XJ], xj_out[XJ];
#pragma unroll
    for (int jj = 0; jj < XJ; ++jj) {
        const int j = t + jj * NT;
        const int r = j / (CH * (TX / XR)), rc = j - r * (CH * (TX / XR));
        const int m = rc / CH, c = rc - m * CH;
        xj_in[jj] = j < NJ ? r * S::ROW + sh + XR * m * CH + c : -1;
        xj_out[jj] = r * (TX * CH) + XR * m * CH + c;
    }

    const int64_t pstart = zc0 - R, pend = zc1 + R;  // input planes of this chunk
#pragma unroll
    for (int k = 0; k < NSTAGE - 1; ++k) {
        if (pstart + k < pend) issue(pstart + k, k);
        else if (!TMA) cp_async_commit();
    }
    // Adam operands of the next output voxel, loaded one plane ahead
    float pu[CH], pm1[CH], pm2[CH];
    // element offset of the thread's output voxel in plane zc0; + plane * CH per plane
    const int64_t pstride = P.plane * CH;
    int64_t o_next = ((zc0 - P.z_begin) * P.plane + (int64_t)gy * P.nx + gx) * CH;
    auto fetch = [&](int64_t o) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            pu[c] = P.u[o + c];
            pm1[c] = P.m1[o + c];
            pm2[c] = P.m2[o + c];
        }
    };
    if (ADAM && own) fetch(o_next);
    int stage = 0;
    for (int64_t p = pstart; p < pend; ++p) {
        // plane p + NSTAGE - 1 goes into the stage read two planes ago (freed by the
        // barrier after that plane's x taps)
        const int st_next = stage == 0 ? NSTAGE - 1 : stage - 1;
        if (p + NSTAGE - 1 < pend) issue(p + NSTAGE - 1, st_next);
        else if (!TMA) cp_async_commit();
        if (TMA)
            mbar_wait(&sm.bar[stage], (uint32_t)(((p - pstart) / NSTAGE) & 1));  // plane p has landed
        else
            cp_async_wait<NSTAGE - 1>();  // this thread's copies of plane p have landed
        __syncthreads();                  // everyone's have; X is free
#pragma unroll
        for (int jj = 0; jj < XJ; ++jj) {
            if (xj_in[jj] < 0) continue;
            const float* in = &sm.raw[stage][0] + xj_in[jj];
            float w_[XR + 2 * R];
#pragma unroll
            for (int i = 0; i < XR + 2 * R; ++i) w_[i] = in[i * CH];
            float* xo = &sm.X[0][0] + xj_out[jj];
#pragma unroll
            for (int o = 0; o < XR; ++o) {
                float acc = 0.0f;
#pragma unroll
                for (int k = 0; k <= 2 * R; ++k) acc = fmaf(P.w[k], w_[o + k], acc);
                xo[o * CH] = acc;
            }
        }
        __syncthreads();
        stage = stage + 1 == NSTAGE ? 0 : stage + 1;
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
        // the z divisor only differs from the full tap sum within R planes of a face
        const float inv = !P.renorm ? 1.0f
                          : (q >= R && q + R < P.nz_global) ? inv_xy_full
                                                            : 1.0f / (wxy * wsum<R>(P, q, P.nz_global));
        const int64_t o = o_next;
        o_next += pstride;
        float v[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            float a = 0.0f;
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k) a = fmaf(P.w[k], ring[k][c], a);
            v[c] = a * inv;
        }
        if (ADAM) {
            float cu[CH], c1[CH], c2[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) cu[c] = pu[c], c1[c] = pm1[c], c2[c] = pm2[c];
            if (q + 1 < zc1) fetch(o_next);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const float m = fmaf(P.b1, c1[c], P.omb1 * v[c]);
                const float s2 = fmaf(P.b2, c2[c], P.omb2 * v[c] * v[c]);
                P.m1[o + c] = m;
                P.m2[o + c] = s2;
                // sqrt(v / c2) as v * rsqrt(v) (approximate MUFU, v = 0 -> 0) and a fast
                // division: a few ulp, well inside the fp32 budget of the update
                const float vv = s2 * P.inv_c2;
                const float sq = vv * rsqrtf(fmaxf(vv, 1e-37f));
                P.u[o + c] = cu[c] - P.lr_c1 * __fdividef(m, sq + P.eps);
            }
        } else {
#pragma unroll
            for (int c = 0; c < CH; ++c) P.out[o + c] = v[c];
        }
    }
    if (!TMA) cp_async_wait<0>();
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

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::atomic<int> state{0};
    if (state.load() == 0) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        state.store(fn ? 1 : 2);
    }
    return fn;
}

template <int R, int CH, bool ADAM>
int launch(Params P, cudaStream_t st) {
    using S = Smem<R, CH>;
    const size_t smem = sizeof(S);
    static std::atomic<unsigned long long> attr_mask{0};
    static int per_sm = 1;
    once_per_device(attr_mask, [&] {
        for (auto fn : {k_smooth<R, CH, ADAM, 0>, k_smooth<R, CH, ADAM, 1>, k_smooth<R, CH, ADAM, 2>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int p = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, k_smooth<R, CH, ADAM, 1>, NT, smem);
        per_sm = std::max(p, 1);
    });
    const bool v16 = ((uintptr_t)P.in & 15) == 0 && (P.nx * CH) % 4 == 0;
    const int64_t tx = (P.nx + TX - 1) / TX, ty = (P.ny + TY - 1) / TY;
    const int64_t nzs = P.z_end - P.z_begin;
    P.zchunk = pick_zchunk(tx * ty, nzs, (int64_t)per_sm * num_sms(), R);
    const int64_t chunks = (nzs + P.zchunk - 1) / P.zchunk;
    if (ty > 65535 || chunks > 65535) return set_error(FFDP_INVALID_ARGUMENT, "gp_convolve: grid too large");
    const dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)chunks);
    // the input field as a 3-D tensor (CH * nx floats per row, ny rows, the buffer's planes);
    // the box is one stage: HY rows of ROW floats starting at a 16-byte aligned column
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    bool tma = false;
    if (FFDP_SMOOTH_TMA && v16 && S::ROW <= 256 && S::HY <= 256) {
        if (auto enc = tensor_map_encoder()) {
            const cuuint64_t n0 = (cuuint64_t)P.nx * CH, n1 = (cuuint64_t)P.ny, n2 = (cuuint64_t)(P.buf_z1 - P.buf_z0);
            const cuuint64_t dims[3] = {n0, n1, n2};
            const cuuint64_t strides[2] = {n0 * 4, n0 * n1 * 4};
            const cuuint32_t box[3] = {(cuuint32_t)S::ROW, (cuuint32_t)S::HY, 1};
            const cuuint32_t es[3] = {1, 1, 1};
            tma = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(P.in), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
    }
    if (tma)
        k_smooth<R, CH, ADAM, 2><<<grid, NT, smem, st>>>(map, P);
    else if (v16)
        k_smooth<R, CH, ADAM, 1><<<grid, NT, smem, st>>>(map, P);
    else
        k_smooth<R, CH, ADAM, 0><<<grid, NT, smem, st>>>(map, P);
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
            case 5: return launch<5, 3, ADAM>(P, st);
            case 6: return launch<6, 3, ADAM>(P, st);
        }
    } else if (!ADAM) {
        switch (R) {
            case 0: return launch<0, 1, false>(P, st);
            case 1: return launch<1, 1, false>(P, st);
            case 2: return launch<2, 1, false>(P, st);
            case 3: return launch<3, 1, false>(P, st);
            case 4: return launch<4, 1, false>(P, st);
            case 5: return launch<5, 1, false>(P, st);
            case 6: return launch<6, 1, false>(P, st);
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
