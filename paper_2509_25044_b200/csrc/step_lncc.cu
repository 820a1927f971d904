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
//   S1  sample Mw (and F) on the (TX+6) x (TY+6) haloed plane into an 8-plane shared
//       ring of shifted (F, Mw) pairs; F and u of the next plane are already in flight
//       (register prefetch); the owner of an output column keeps S*dMw/df of its voxel
//       in a 4-plane register ring (its moments complete 3 planes later);
//   S2  x box sums of the five moment-channel DIFFERENCES v(p) - v(p-7) (runs of 4,
//       sliding, fp32), read from ring slots p and p-7;
//   S3  y box sums of the differences, Z += box in fp64 -- Z is the 7x7x7 window sum of
//       every channel by telescoping, with no ring of per-plane sums; then the voxel of
//       plane p-3 is finished: A, B, C from Z in fp64 (the cancellation-prone part),
//       gamma family, dL/dMw, g_u = S * dxsrc * dL/dMw (sampler.hpp:221-230).
// Intensities are shifted by their mid-range before the moments (exact up to rounding;
// the zero-padded border is corrected with the in-volume window weight W).
#include <algorithm>

#include "ffdp_common.cuh"

namespace ffdp {
namespace lstep {

constexpr int R = 3, WIN = 7;
constexpr int TX = 64, TY = 8, NT = 256;
constexpr int HX = TX + 2 * R, HY = TY + 2 * R;  // 70 x 14
constexpr int HXP = 72;                          // ring row pitch (float2)
constexpr int NOUT = TX * TY;                    // 512 outputs per plane, 2 per thread (a y pair)
constexpr int NHALO = HX * HY - NOUT;            // 468
constexpr int XJOBS = HY * (TX / 4);             // 224 x-pass runs of 4
constexpr int NSLOT = 8;                         // planes p-7 .. p

struct Smem {
    float2 raw[NSLOT][HY][HXP];  // shifted (F, Mw), zero outside the volume
    float X[5][HY][TX];          // x box sums of the channel differences
    int4 pos[4][NT];             // per thread and sample slot: {in-plane offset, gx | gy << 16, ring index, valid}
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

// Exact int -> double without the (quarter-rate) conversion pipe.
__device__ __forceinline__ double i2d(int32_t i) {
    return __hiloint2double(0x43300000, (int32_t)((uint32_t)i ^ 0x80000000u)) - 4503601774854144.0;
}

// Cell of the sample at lattice (x, y, plane of kz): the fp64 affine part plus Q u, then
// the conversion-free cell assignment (ffdp_common.cuh cell_fix).
__device__ __forceinline__ Cell cell_at(const Geom& g, const double (&kz)[3], int x, int y, float u0, float u1,
                                        float u2) {
    const double xd = i2d(x), yd = i2d(y);
    Cell c;
    cell_fix(fma(g.Q[0], (double)u0, fma(g.P[0], xd, fma(g.P[1], yd, kz[0]))), c.i0[0], c.frac[0]);
    cell_fix(fma(g.Q[1], (double)u1, fma(g.P[3], xd, fma(g.P[4], yd, kz[1]))), c.i0[1], c.frac[1]);
    cell_fix(fma(g.Q[2], (double)u2, fma(g.P[6], xd, fma(g.P[7], yd, kz[2]))), c.i0[2], c.frac[2]);
    return c;
}

// The thread's four sample positions, fixed for the whole z march: k = 0, 1 its owned
// outputs (a vertical pair, so the y sums share rows), k = 2, 3 halo positions
// (k = 3 exists for the first NHALO - NT threads only). Resolved once per CTA into a
// shared table (one LDS.128 per position and plane).
__device__ __forceinline__ int4 pos_record(int k, int t, int x0, int y0, const Params& P) {
    int hx, hy;
    bool slot_ok = true;
    if (k < 2) {
        hx = (t & (TX - 1)) + R;
        hy = 2 * (t / TX) + k + R;
    } else {
        const int h = t + NT * (k - 2);
        slot_ok = h < NHALO;
        halo_pos(slot_ok ? h : 0, hx, hy);
    }
    const int gx = x0 + hx - R, gy = y0 + hy - R;
    const bool in = slot_ok && gx >= 0 && gx < P.nx && gy >= 0 && gy < P.ny;
    return make_int4(in ? gy * P.nx + gx : 0, (gx & 0xFFFF) | (gy << 16), hy * HXP + hx, in ? 1 : (slot_ok ? 0 : -1));
}
__device__ __forceinline__ int pos_gx(const int4& r) { return (int)(int16_t)(r.y & 0xFFFF); }
__device__ __forceinline__ int pos_gy(const int4& r) { return r.y >> 16; }

struct Pref {
    float f[4], u[4][3];
};

__device__ __forceinline__ void prefetch(const Params& P, const Smem& sm, int t, int64_t p, Pref& pf) {
    const bool plane_in = p >= 0 && p < P.nz_global;
    const int64_t zoff = plane_in ? (p - P.buf_z0) * P.plane : 0;
    const float* fpl = P.f + zoff;
    const float* upl = P.u + 3 * zoff;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int4 r = sm.pos[k][t];
        const bool ok = plane_in && r.w > 0;
        pf.f[k] = ok ? __ldg(fpl + r.x) : 0.0f;
        pf.u[k][0] = ok ? __ldg(upl + 3 * r.x) : 0.0f;
        pf.u[k][1] = ok ? __ldg(upl + 3 * r.x + 1) : 0.0f;
        pf.u[k][2] = ok ? __ldg(upl + 3 * r.x + 2) : 0.0f;
    }
}

template <int SLOT, bool FULLWIN>
__device__ __forceinline__ void plane_step(const Params& P, Smem& sm, Pref (&pf)[2], float (&gur)[4][2][3],
                                           double (&Z)[2][5], double& nsum, int& miss, int64_t p, int64_t pstart,
                                           int64_t pend, int x0, int y0, int64_t zc0) {
    if (p >= pend) return;  // uniform across the CTA
    const int t = threadIdx.x;
    const bool plane_in = p >= 0 && p < P.nz_global;
    const int slot = (int)((p - pstart) & (NSLOT - 1));
    const int slot_old = (slot + 1) & (NSLOT - 1);  // plane p-7

    // ---- S1: sampling ------------------------------------------------------------
    // register ping-pong: this plane's F, u were loaded during the previous plane; the
    // next plane's loads are issued now and land while this plane is processed
    const Pref& cur = pf[SLOT & 1];
    if (p + 1 < pend) prefetch(P, sm, t, p + 1, pf[(SLOT + 1) & 1]);
    const double zd = i2d((int32_t)p);
    double kz[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) kz[a] = fma(P.g.P[3 * a + 2], zd, P.g.K[a]);
    // two batches (owned pair, halo pair): the 16 corner loads of a batch are in flight together
#pragma unroll
    for (int bt = 0; bt < 2; ++bt) {
        // slot 3 (second halo position) exists for the first NHALO - NT threads only
        if (bt == 1 && !__any_sync(0xffffffffu, t + NT < NHALO)) {
            const int4 q = sm.pos[2][t];
            Cell c = cell_at(P.g, kz, pos_gx(q), pos_gy(q), cur.u[2][0], cur.u[2][1], cur.u[2][2]);
            const Corners cr = gather_pad<FULLWIN>(P.g, c, miss);
            const float mw = interp(cr, c);
            (&sm.raw[slot][0][0])[q.z] =
                (plane_in && q.w > 0) ? make_float2(cur.f[2] - P.sf, mw - P.sm) : make_float2(0.f, 0.f);
            continue;
        }
        int4 q[2];
        Cell c[2];
        Corners cr[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int k = 2 * bt + i;
            q[i] = sm.pos[k][t];
            c[i] = cell_at(P.g, kz, pos_gx(q[i]), pos_gy(q[i]), cur.u[k][0], cur.u[k][1], cur.u[k][2]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) cr[i] = gather_pad<FULLWIN>(P.g, c[i], miss);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int k = 2 * bt + i;
            const bool ok = plane_in && q[i].w > 0;
            float2 v = make_float2(0.f, 0.f);
            if (bt == 0) {
                float d[3];
                const float mw = interp_grad(cr[i], c[i], d);
                if (ok) v = make_float2(cur.f[k] - P.sf, mw - P.sm);
#pragma unroll
                for (int a = 0; a < 3; ++a) gur[SLOT][i][a] = ok ? P.g.dscale[a] * d[a] : 0.0f;
            } else {
                const float mw = interp(cr[i], c[i]);
                if (ok) v = make_float2(cur.f[k] - P.sf, mw - P.sm);
            }
            if (q[i].w >= 0) (&sm.raw[slot][0][0])[q[i].z] = v;
        }
    }
    __syncthreads();

    // ---- S2: x box sums of v(p) - v(p-7), runs of 4 --------------------------------
    if (t < XJOBS) {
        const int r = t >> 4, xs = (t & 15) * 4;
        float dv[5][10];
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const float2 n = sm.raw[slot][r][xs + k], o = sm.raw[slot_old][r][xs + k];
            dv[0][k] = n.x - o.x;
            dv[1][k] = n.y - o.y;
            dv[2][k] = fmaf(n.x, n.x, -o.x * o.x);
            dv[3][k] = fmaf(n.y, n.y, -o.y * o.y);
            dv[4][k] = fmaf(n.x, n.y, -o.x * o.y);
        }
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) {
            float s = dv[ch][0] + dv[ch][1] + dv[ch][2] + dv[ch][3] + dv[ch][4] + dv[ch][5] + dv[ch][6];
            float o0 = s;
            s += dv[ch][7] - dv[ch][0];
            const float o1 = s;
            s += dv[ch][8] - dv[ch][1];
            const float o2 = s;
            s += dv[ch][9] - dv[ch][2];
            *reinterpret_cast<float4*>(&sm.X[ch][r][xs]) = make_float4(o0, o1, o2, s);
        }
    }
    __syncthreads();

    // ---- S3: y box sums, Z += box, finish plane p-3 --------------------------------
    const bool emit = p >= zc0 + R;
    const int64_t q = p - R;
    const int slot_q = (slot + NSLOT - R) & (NSLOT - 1);
    const int ox = t & (TX - 1), oy0 = 2 * (t / TX);
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
        // rows oy0 .. oy0+7 cover the windows of both owned outputs
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < WIN; ++k) s += sm.X[ch][oy0 + k][ox];
        Z[0][ch] += (double)s;
        s += sm.X[ch][oy0 + WIN][ox] - sm.X[ch][oy0][ox];
        Z[1][ch] += (double)s;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int oy = oy0 + j;
        const int gx = x0 + ox, gy = y0 + oy;
        if (emit && gx < P.nx && gy < P.ny) {
            const float2 fm = sm.raw[slot_q][oy + R][ox + R];
            const float cw = win_count(gx, P.nx) * win_count(gy, P.ny) * win_count(q, P.nz_global);
            const double inv = 1.0 / (double)(WIN * WIN * WIN);
            const double W = (double)cw * inv;
            const double Sf = Z[j][0], Sm = Z[j][1];
            // moments scaled by 343^2; the cancellation-prone differences in fp64
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
            const float df = (fm.x - mf) + P.sf * omwf;    // F - mean_F
            const float dm = (fm.y - mm) + P.sm * omwf;    // Mw - mean_M
            const float gmw = gamma * fmaf(-dm, rab, df);  // dL/dMw (lncc.hpp:404, ANTs)
            const int sq = (SLOT + 1) & 3;                 // gu of plane p-3
            const int64_t ov = 3 * ((q - P.z_begin) * P.plane + sm.pos[j][t].x);
            P.g_u[ov] = gur[sq][j][0] * gmw;
            P.g_u[ov + 1] = gur[sq][j][1] * gmw;
            P.g_u[ov + 2] = gur[sq][j][2] * gmw;
        }
    }
}

template <bool FULLWIN>
__global__ void __launch_bounds__(NT, 2) k_step_lncc(const Params P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int64_t zc0 = P.z_begin + (int64_t)blockIdx.z * P.zchunk;
    const int64_t zc1 = min(P.z_end, zc0 + P.zchunk);
    if (zc0 >= zc1) return;
    for (int i = threadIdx.x; i < NSLOT * HY * HXP; i += NT) (&sm.raw[0][0][0])[i] = make_float2(0.f, 0.f);
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) sm.pos[k][t] = pos_record(k, t, x0, y0, P);
    float gur[4][2][3];
    double Z[2][5];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) Z[j][ch] = 0.0;
    double nsum = 0.0;
    int miss = 0;
    const int64_t pstart = zc0 - R, pend = zc1 + R;
    Pref pf[2];
    __syncthreads();
    prefetch(P, sm, t, pstart, pf[0]);
    for (int64_t p = pstart; p < pend; p += 4) {
        plane_step<0, FULLWIN>(P, sm, pf, gur, Z, nsum, miss, p, pstart, pend, x0, y0, zc0);
        plane_step<1, FULLWIN>(P, sm, pf, gur, Z, nsum, miss, p + 1, pstart, pend, x0, y0, zc0);
        plane_step<2, FULLWIN>(P, sm, pf, gur, Z, nsum, miss, p + 2, pstart, pend, x0, y0, zc0);
        plane_step<3, FULLWIN>(P, sm, pf, gur, Z, nsum, miss, p + 3, pstart, pend, x0, y0, zc0);
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

namespace ffdp {
int64_t lncc2_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s);
int lncc2_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, float shift_f, float shift_m, float* g_u,
               double* sum_n, int32_t* miss, void* workspace, int passes, cudaStream_t st);
}  // namespace ffdp

extern "C" int64_t ffdp_step_lncc_workspace_bytes(ffdp_dims d, ffdp_slab s) { return lncc2_workspace_bytes(d, s); }

static int step_lncc_impl(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                          const ffdp_sampler_args* args, int window, double eps, double gi, float shift_f,
                          float shift_m, float* g_u, double* sum_n, int32_t* miss, void* workspace, int passes,
                          void* stream) {
    using namespace ffdp::lstep;
    if (window != WIN) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the fused kernel is built for window %d", WIN);
    const char* why = nullptr;
    if (!args || !valid_args(*args, &why)) return set_error(FFDP_INVALID_ARGUMENT, "%s", why ? why : "null args");
    if (!f || !u || !g_u || !m.data) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: null pointer");
    if (passes < 1 || passes > 3) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: passes must be 1, 2 or 3");
    if (d.nx < 1 || d.ny < 1 || d.nz < 1 || s.buf_nz != d.nz || s.z_begin < s.buf_z0 || s.z_end > s.buf_z0 + s.buf_nz ||
        s.z_begin >= s.z_end || s.buf_z0 < 0 || s.buf_z0 + s.buf_nz > s.nz_global)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: inconsistent slab");
    const int64_t need_lo = std::max<int64_t>(0, s.z_begin - R), need_hi = std::min<int64_t>(s.nz_global, s.z_end + R);
    if (s.buf_z0 > need_lo || s.buf_z0 + s.buf_nz < need_hi)
        return set_error(FFDP_INVALID_ARGUMENT, "halo_exchange: buffer lacks the %d halo planes the window needs", R);
    if (m.z_begin < 0 || m.z_end > m.dims.nz || m.z_begin >= m.z_end)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: bad moving window");
    if (m.pad != 2)
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the moving image must be zero-bordered (pad = 2, "
                                                "ffdp_pad_window)");
    // packed 16-bit lattice coordinates and 32-bit in-plane offsets in the position table
    if (d.nx >= 32000 || d.ny >= 32000 || 3 * d.nx * d.ny >= (1LL << 31) || s.nz_global >= (1 << 30))
        return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: lattice too large for the fused kernel");
    if (workspace)
        return lncc2_step(f, u, d, s, m, *args, eps, gi, shift_f, shift_m, g_u, sum_n, miss, workspace, passes,
                          (cudaStream_t)stream);
    if (passes != 3) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: separate passes need the workspace");
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
    static std::atomic<unsigned long long> attr_mask{0};
    if (first_on_device(attr_mask)) {
        cudaFuncSetAttribute(k_step_lncc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        cudaFuncSetAttribute(k_step_lncc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    }
    const dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)chunks);
    if (m.z_begin == 0 && m.z_end == m.dims.nz)
        k_step_lncc<true><<<grid, NT, sizeof(Smem), (cudaStream_t)stream>>>(P);
    else
        k_step_lncc<false><<<grid, NT, sizeof(Smem), (cudaStream_t)stream>>>(P);
    return check_launch("step_lncc");
}

extern "C" int ffdp_step_lncc(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                              const ffdp_sampler_args* args, int window, double eps, double gi, float shift_f,
                              float shift_m, float* g_u, double* sum_n, int32_t* miss, void* workspace,
                              void* stream) {
    return step_lncc_impl(f, u, d, s, m, args, window, eps, gi, shift_f, shift_m, g_u, sum_n, miss, workspace, 3,
                          stream);
}

extern "C" int ffdp_step_lncc_passes(const float* f, const float* u, ffdp_dims d, ffdp_slab s, ffdp_image_window m,
                                     const ffdp_sampler_args* args, int window, double eps, double gi, float shift_f,
                                     float shift_m, float* g_u, double* sum_n, int32_t* miss, void* workspace,
                                     int passes, void* stream) {
    if (!workspace) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: the two-pass step needs its workspace");
    return step_lncc_impl(f, u, d, s, m, args, window, eps, gi, shift_f, shift_m, g_u, sum_n, miss, workspace,
                          passes, stream);
}
