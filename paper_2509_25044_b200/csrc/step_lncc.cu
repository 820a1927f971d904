// step_lncc.cu -- the fused warp + LNCC(ANTs) forward+backward step in ONE pass over HBM.
//
// Reference sequence replaced (registration.hpp:277-312): ring_sample (distops.hpp:144)
// -> dist_lncc(ants_approx) (distops.hpp:285-352) -> ring_sample_backward(want warp)
// (distops.hpp:179-248). In ANTs mode dL/dMw at a voxel needs only the five window
// moments at that voxel (lncc.hpp:392-405 without the gamma re-convolution), so the
// whole step streams F, u and the moving-image gathers once and writes only g_u:
// 32 algorithmic bytes per output voxel.
//
// CTA = TX x TY output columns marching along z. Per plane p:
//   S1  sample Mw (and F) on the (TX+6) x (TY+6) haloed plane into shared memory
//       (shifted by the intensity mid-range); the thread that owns an output column
//       also keeps F, Mw and dL/du-per-dL/dMw of its own voxel in a 4-plane register
//       ring (the voxel's moments are complete 3 planes later);
//   S2  x box sums of the five moment channels (runs of 4, sliding, fp32);
//   S3  y box sums -> P(p) (fp32), z box by sliding Z += P(p) - P(p-7) in fp64 (exact:
//       P(p-7) is the identical fp32 value, kept in a 7-plane shared ring); then the
//       voxel of plane p-3 is finished: A, B, C in fp64 (cancellation), gamma family,
//       dL/dMw, g_u = S * dxsrc * dL/dMw (sampler.hpp:221-230).
#include <algorithm>

#include "ffdp_common.cuh"

namespace ffdp {
namespace lstep {

constexpr int R = 3, WIN = 7;
constexpr int TX = 64, TY = 8, NT = 256;
constexpr int HX = TX + 2 * R, HY = TY + 2 * R;  // 70 x 14
constexpr int HXP = 72;                          // raw row pitch
constexpr int NOUT = TX * TY;                    // 512 outputs per plane, 2 per thread
constexpr int NHALO = HX * HY - NOUT;            // 468
constexpr int XJOBS = HY * (TX / 4);             // 224 x-pass runs of 4

struct Smem {
    float raw[2][HY][HXP];   // shifted F, Mw of the current plane
    float X[5][HY][TX];      // x box sums
    float P[WIN][5][NOUT];   // 7-plane ring of xy box sums
};

struct Params {
    Geom g;
    const float* f;
    const float* u;
    float* g_u;
    double* sum_n;
    int32_t* miss;
    int32_t nx, ny;
    int64_t plane;
    int64_t buf_z0, nz_global, z_begin, z_end;
    int32_t zchunk;
    double eps, gi;
    float sf, sm;
};

__device__ __forceinline__ void halo_pos(int h, int& hx, int& hy) {
    if (h < 6 * HX) {
        const int r6 = h / HX;
        hy = r6 < 3 ? r6 : r6 + TY;
        hx = h - r6 * HX;
    } else {
        const int k = h - 6 * HX;
        hy = R + k / 6;
        const int c = k % 6;
        hx = c < 3 ? c : TX + c;
    }
}

__device__ __forceinline__ float win_count(int64_t g, int64_t n) {
    const int64_t lo = g - R < 0 ? 0 : g - R;
    const int64_t hi = g + R >= n ? n - 1 : g + R;
    return (float)(hi - lo + 1);
}

struct Own {
    float fp, mp, gu0, gu1, gu2;  // shifted F, shifted Mw, dscale * dfrac
};

template <int SLOT>
__device__ __forceinline__ void plane_step(const Params& P, Smem& sm, Own (&ring)[4][2], double (&Z)[2][5],
                                           double& nsum, int& miss, int64_t p, int64_t pstart, int64_t pend,
                                           int x0, int y0, int64_t zc0) {
    if (p >= pend) return;  // uniform across the CTA
    const int t = threadIdx.x;
    const bool plane_in = p >= 0 && p < P.nz_global;
    const int64_t zoff = (p - P.buf_z0) * P.plane;

    // ---- S1: sampling ------------------------------------------------------------
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int o = t + NT * j;
        const int ox = o & (TX - 1), oy = o / TX;
        const int gx = x0 + ox, gy = y0 + oy;
        Own w{0.f, 0.f, 0.f, 0.f, 0.f};
        if (plane_in && gx < P.nx && gy < P.ny) {
            const int64_t bi = zoff + (int64_t)gy * P.nx + gx;
            const float fv = __ldg(P.f + bi);
            const float u0 = __ldg(P.u + 3 * bi), u1 = __ldg(P.u + 3 * bi + 1), u2 = __ldg(P.u + 3 * bi + 2);
            const Cell c = resolve(P.g, gx, gy, (int32_t)p, u0, u1, u2);
            const Corners k = gather(P.g, c, miss);
            float d[3];
            const float mw = interp_grad(k, c, d);
            w.fp = fv - P.sf;
            w.mp = mw - P.sm;
            w.gu0 = P.g.dscale[0] * d[0];
            w.gu1 = P.g.dscale[1] * d[1];
            w.gu2 = P.g.dscale[2] * d[2];
        }
        sm.raw[0][oy + R][ox + R] = w.fp;
        sm.raw[1][oy + R][ox + R] = w.mp;
        ring[SLOT][j] = w;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int h = t + NT * j;
        if (h < NHALO) {
            int hx, hy;
            halo_pos(h, hx, hy);
            const int gx = x0 + hx - R, gy = y0 + hy - R;
            float fp = 0.f, mp = 0.f;
            if (plane_in && gx >= 0 && gx < P.nx && gy >= 0 && gy < P.ny) {
                const int64_t bi = zoff + (int64_t)gy * P.nx + gx;
                const float fv = __ldg(P.f + bi);
                const float u0 = __ldg(P.u + 3 * bi), u1 = __ldg(P.u + 3 * bi + 1), u2 = __ldg(P.u + 3 * bi + 2);
                const Cell c = resolve(P.g, gx, gy, (int32_t)p, u0, u1, u2);
                const Corners k = gather(P.g, c, miss);
                fp = fv - P.sf;
                mp = interp(k, c) - P.sm;
            }
            sm.raw[0][hy][hx] = fp;
            sm.raw[1][hy][hx] = mp;
        }
    }
    __syncthreads();

    // ---- S2: x box sums, runs of 4 -------------------------------------------------
    if (t < XJOBS) {
        const int r = t >> 4, xs = (t & 15) * 4;
        float F[10], M[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            F[k] = sm.raw[0][r][xs + k];
            M[k] = sm.raw[1][r][xs + k];
        }
        float s[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < WIN; ++k) {
            s[0] += F[k];
            s[1] += M[k];
            s[2] = fmaf(F[k], F[k], s[2]);
            s[3] = fmaf(M[k], M[k], s[3]);
            s[4] = fmaf(F[k], M[k], s[4]);
        }
        float o[5][4];
#pragma unroll
        for (int c = 0; c < 5; ++c) o[c][0] = s[c];
#pragma unroll
        for (int i = 1; i < 4; ++i) {
            const float fa = F[i + 6], ma = M[i + 6], fr = F[i - 1], mr = M[i - 1];
            s[0] += fa - fr;
            s[1] += ma - mr;
            s[2] += fmaf(fa, fa, -fr * fr);
            s[3] += fmaf(ma, ma, -mr * mr);
            s[4] += fmaf(fa, ma, -fr * mr);
#pragma unroll
            for (int c = 0; c < 5; ++c) o[c][i] = s[c];
        }
#pragma unroll
        for (int c = 0; c < 5; ++c)
            *reinterpret_cast<float4*>(&sm.X[c][r][xs]) = make_float4(o[c][0], o[c][1], o[c][2], o[c][3]);
    }
    __syncthreads();

    // ---- S3: y box sums, z slide, finish plane p-3 ---------------------------------
    const int slot = (int)((p - pstart) % WIN);
    const bool emit = p >= zc0 + R;
    const int64_t q = p - R;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int o = t + NT * j;
        const int ox = o & (TX - 1), oy = o / TX;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < WIN; ++k) s += sm.X[c][oy + k][ox];
            const float old = sm.P[slot][c][o];
            sm.P[slot][c][o] = s;
            Z[j][c] += (double)s - (double)old;
        }
        const int gx = x0 + ox, gy = y0 + oy;
        if (emit && gx < P.nx && gy < P.ny) {
            const Own w = ring[(SLOT + 1) & 3][j];
            const float cw = win_count(gx, P.nx) * win_count(gy, P.ny) * win_count(q, P.nz_global);
            const double inv = 1.0 / (double)(WIN * WIN * WIN);
            const double W = (double)cw * inv;
            const double Sf = Z[j][0], Sm = Z[j][1];
            // window sums of the shifted channels; moments scaled by 343^2 (exact
            // power-free fold), cancellation-prone differences in fp64
            const double N = WIN * WIN * WIN;
            double A = N * Z[j][4] - Sf * Sm;
            double Bv = N * Z[j][2] - Sf * Sf;
            double Cv = N * Z[j][3] - Sm * Sm;
            const double sf = P.sf, smv = P.sm;
            if (cw != (float)(WIN * WIN * WIN)) {
                const double omw = 1.0 - W;
                A += N * (omw * (sf * Sm + smv * Sf) + sf * smv * N * (W - W * W));
                Bv += N * (omw * 2.0 * sf * Sf + sf * sf * N * (W - W * W));
                Cv += N * (omw * 2.0 * smv * Sm + smv * smv * N * (W - W * W));
            }
            const float a = (float)(A * (inv * inv)), b = (float)(Bv * (inv * inv)), cc = (float)(Cv * (inv * inv));
            const float D = fmaf(b, cc, (float)P.eps);
            const float invD = 1.0f / D;
            nsum += (double)(a * a * invD);
            const float gamma = 2.0f * (float)P.gi * a * invD;
            const float rab = a * b * invD;
            const float mf = (float)(Sf * inv), mm = (float)(Sm * inv);
            const float omwf = (float)(1.0 - W);
            const float df = (w.fp - mf) + P.sf * omwf;  // F - mean_F
            const float dm = (w.mp - mm) + P.sm * omwf;  // Mw - mean_M
            const float gmw = gamma * fmaf(-dm, rab, df);  // dL/dMw (lncc.hpp:404, ANTs)
            const int64_t ov = 3 * ((q - P.z_begin) * P.plane + (int64_t)gy * P.nx + gx);
            P.g_u[ov] = w.gu0 * gmw;
            P.g_u[ov + 1] = w.gu1 * gmw;
            P.g_u[ov + 2] = w.gu2 * gmw;
        }
    }
}

__global__ void __launch_bounds__(NT, 2) k_step_lncc(const Params P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int64_t zc0 = P.z_begin + (int64_t)blockIdx.z * P.zchunk;
    const int64_t zc1 = min(P.z_end, zc0 + P.zchunk);
    if (zc0 >= zc1) return;
    for (int i = threadIdx.x; i < WIN * 5 * NOUT; i += NT) (&sm.P[0][0][0])[i] = 0.f;
    __syncthreads();
    Own ring[4][2];
    double Z[2][5];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int c = 0; c < 5; ++c) Z[j][c] = 0.0;
    double nsum = 0.0;
    int miss = 0;
    const int64_t pstart = zc0 - R, pend = zc1 + R;
    for (int64_t p = pstart; p < pend; p += 4) {
        plane_step<0>(P, sm, ring, Z, nsum, miss, p, pstart, pend, x0, y0, zc0);
        plane_step<1>(P, sm, ring, Z, nsum, miss, p + 1, pstart, pend, x0, y0, zc0);
        plane_step<2>(P, sm, ring, Z, nsum, miss, p + 2, pstart, pend, x0, y0, zc0);
        plane_step<3>(P, sm, ring, Z, nsum, miss, p + 3, pstart, pend, x0, y0, zc0);
    }
    // loss partial and window misses
    nsum = warp_sum(nsum);
    const unsigned anymiss = __ballot_sync(0xffffffffu, miss);
    if ((threadIdx.x & 31) == 0) {
        if (P.sum_n) atomicAdd(P.sum_n, nsum);
        if (anymiss && P.miss) atomicAdd(P.miss, __popc(anymiss));
    }
}

}  // namespace lstep
}  // namespace ffdp

using namespace ffdp;

extern "C" int ffdp_step_lncc(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                              const ffdp_sampler_args* args, int window, double eps, double gi, float shift_f,
                              float shift_m, float* g_u, double* sum_n, int32_t* miss, void* stream) {
    using namespace ffdp::lstep;
    if (window != WIN) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the fused kernel is built for window %d", WIN);
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !g_u || !m.data) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: null pointer");
    if (d.nx < 1 || d.ny < 1 || d.nz < 1 || s.buf_nz != d.nz || s.z_begin < s.buf_z0 || s.z_end > s.buf_z0 + s.buf_nz ||
        s.z_begin >= s.z_end || s.buf_z0 < 0 || s.buf_z0 + s.buf_nz > s.nz_global)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: inconsistent slab");
    const int64_t need_lo = std::max<int64_t>(0, s.z_begin - R), need_hi = std::min<int64_t>(s.nz_global, s.z_end + R);
    if (s.buf_z0 > need_lo || s.buf_z0 + s.buf_nz < need_hi)
        return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: buffer lacks the %d halo planes the window needs", R);
    if (m.z_begin < 0 || m.z_end > m.dims.nz || m.z_begin >= m.z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: bad moving window");
    if (d.nx >= (1 << 30) || d.ny >= (1 << 30) || s.nz_global >= (1 << 30))
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: lattice too large");
    Params P;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    P.g = make_geom(m, out, *args);
    P.f = f;
    P.u = u;
    P.g_u = g_u;
    P.sum_n = sum_n;
    P.miss = miss;
    P.nx = (int32_t)d.nx;
    P.ny = (int32_t)d.ny;
    P.plane = d.nx * d.ny;
    P.buf_z0 = s.buf_z0;
    P.nz_global = s.nz_global;
    P.z_begin = s.z_begin;
    P.z_end = s.z_end;
    P.eps = eps;
    P.gi = gi;
    P.sf = shift_f;
    P.sm = shift_m;
    const int64_t tx = (d.nx + TX - 1) / TX, ty = (d.ny + TY - 1) / TY;
    const int64_t nzs = s.z_end - s.z_begin;
    // enough CTAs for ~3 waves at 2 CTAs/SM, chunks of >= 16 planes
    const int64_t target = 6LL * num_sms();
    int64_t chunks = std::max<int64_t>(1, (target + tx * ty - 1) / (tx * ty));
    chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, nzs / 16));
    P.zchunk = (int32_t)((nzs + chunks - 1) / chunks);
    chunks = (nzs + P.zchunk - 1) / P.zchunk;
    if (ty > 65535 || chunks > 65535) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: grid too large");
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_step_lncc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        attr_set = true;
    }
    const dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)chunks);
    k_step_lncc<<<grid, NT, sizeof(Smem), (cudaStream_t)stream>>>(P);
    return check_launch("step_lncc");
}
