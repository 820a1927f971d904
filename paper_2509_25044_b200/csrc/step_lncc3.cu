// step_lncc3.cu -- the warp + LNCC(ANTs) forward+backward step as ONE streaming pass.
//
// Reference sequence (registration.hpp:277-312): ring_sample -> dist_lncc(ants) ->
// ring_sample_backward(want warp), i.e. Mw = fused_sample(M, u) (sampler.hpp:165-243),
// the five window moments of (F, Mw) (lncc_forward_fused, lncc.hpp:144-205), the ANTs
// dL/dMw (lncc_backward_fused with ants_approx, lncc.hpp:226-280) and
// g_u = S * (N-1)/2 * dMw/dfrac * dL/dMw (sampler.hpp:221-230).
//
// One CTA (512 threads, 1 per SM) owns a 32 x 32 column of output voxels and marches
// along z over a chunk of planes, warp-specialised:
//   * 8 SAMPLER warps warp the 38 x 38 haloed tile of every plane (1.41 samples per
//     output voxel): b = (Mw - shift) * scale into a 9-plane shared ring and, for the
//     1024 interior positions, G = dscale * dMw/dfrac into a 5-plane ring. They run up to
//     one plane ahead of the moment warps (mbarriers "sampled" / "consumed"), so the
//     gather latency overlaps the moment arithmetic; u is prefetched a batch ahead;
//   * F(p) of the haloed tile arrives by TMA (cp.async.bulk.tensor.3d, OOB zero fill)
//     into a 9-slot ring, one plane ahead, on per-slot mbarriers;
//   * 8 MOMENT warps: z stage -- the five channels F, M, F^2, M^2, FM of the shifted,
//     power-of-two scaled intensities are quantised to integers (2^-21 of the scaled
//     range) and the z window sums slide in registers as EXACT int32 sums (+ plane p,
//     - plane p-7): no drift over the march, no fp64 telescoping; x and y stages: exact
//     sliding integer box sums through two shared buffers; finalize plane p-3: A, B, C
//     exactly in int64 (the zero-padded border of the reference's box filter,
//     smoothing.hpp:75-90, enters as the in-lattice window count), n_i, the ANTs
//     dL/dMw = gamma [(F - muF) - (M - muM) AB/D] (lncc.hpp:80-88, 262-278), g_u = G dL/dMw.
// HBM traffic per output voxel: F 4 + u 12 (+ halo re-reads from L2) + M gathers
// (L1/L2) + g_u 12: the 32 algorithmic bytes; no intermediate tensor. Integer window
// sums make every g_u independent of the tiling, the z chunking and the z-slab sharding
// (bit-identical), given the same intensity frame.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ffdp_common.cuh"

namespace ffdp {
namespace l3 {

#ifndef FFDP_L3_ROWS
#define FFDP_L3_ROWS 1
#endif
// FFDP_L3_SPLITFIN = 1: the sampler warps finish half of every plane's outputs
#ifndef FFDP_L3_SPLITFIN
#define FFDP_L3_SPLITFIN 0
#endif
// FFDP_L3_NB: sampler passes per batch (3 or 6)
#ifndef FFDP_L3_NB
#define FFDP_L3_NB 3
#endif
// FFDP_L3_MROWS = 1: the moment warps' z stage in the row layout too (moment_rows)
#ifndef FFDP_L3_MROWS
#define FFDP_L3_MROWS 1
#endif
// L2 prefetch of the moving image (bulk tensor prefetch, one box per plane and CTA): the
// box of the zero-bordered window starting MPF_X / MPF_Y before the tile (bordered
// coordinates; the start column stays 16-byte aligned), MPF_W x MPF_H, MPF_D planes ahead
#ifndef FFDP_L3_MPF_D
#define FFDP_L3_MPF_D 2
#endif
#ifndef FFDP_L3_MPF_PAD
#define FFDP_L3_MPF_PAD 1
#endif
constexpr int MPF_D = FFDP_L3_MPF_D, MPF_X = 4 + 4 * FFDP_L3_MPF_PAD, MPF_Y = 3 + 4 * FFDP_L3_MPF_PAD;
constexpr int MPF_W = 48 + 8 * FFDP_L3_MPF_PAD, MPF_H = 32 + 10 + 8 * FFDP_L3_MPF_PAD;
constexpr int R = 3, WIN = 7, TX = 32, TY = 32, HX = TX + 2 * R, HY = TY + 2 * R;
constexpr int NT = 512;                                        // threads: moment warps + sampler warps
constexpr int NPOS = HX * HY, NIN = TX * TY;                   // 1444 haloed positions, 1024 outputs
constexpr int RING = 9;                                        // F / b ring slots (planes p-7 .. p+1)
constexpr int NG = 5;                                          // G ring slots (planes p-3 .. p+1)
constexpr int FW = 40;                                         // TMA box width: x0-4 .. x0+35
constexpr int FSLOT = 1536;                                    // floats per F slot (6144 B, 128-B aligned)
constexpr int ZP = 40;                                         // z buffer row pitch (16-B rows)
constexpr int XJOBS = 5 * HY * (TX / 4);                       // 1520 runs of 4 x sums
constexpr float QSCALE = 2097152.0f;                           // 2^21
constexpr float MAGIC = 12582912.0f;                           // 1.5 * 2^23: bits = 0x4B400000 + round(x)
constexpr double NWIN = (double)(WIN * WIN * WIN);

static_assert(FW >= HX + 1 && FW % 4 == 0 && FW * HY <= FSLOT && (FSLOT * 4) % 128 == 0, "F ring slot");
static_assert(4 * (TX / 4 - 1) + 11 < ZP, "x runs read three 16-byte words");

// The warp split: NM moment threads (warps 0 .. NM/32-1) and NS = NT - NM sampler threads,
// with their register budgets (setmaxnreg; NM * RM + NS * RS <= 64K).
template <int NM_>
struct Split {
    static constexpr int NM = NM_, NS = NT - NM_;
    static constexpr int SPOS = (NPOS + NS - 1) / NS;   // sampler positions per thread
    static constexpr int MPOS = (NPOS + NM - 1) / NM;   // z-stage positions per moment thread
    static constexpr int MJOBS = (XJOBS + NM - 1) / NM; // x-stage runs per moment thread
    static constexpr int OUTR = NIN / NM;               // output rows per moment thread (one column)
    static constexpr int DX = NS % HX, DY = NS / HX;    // sampler position step h -> h + NS
    static constexpr int RM = NM == 256 ? 128 : 168, RS = NM == 256 ? 128 : 112;
    static_assert(NM % 128 == 0 && NIN % NM == 0 && 32 % OUTR == 0 && NM * RM + NS * RS <= 65536, "split");
};

struct __align__(128) Smem {
    float fr[RING][FSLOT];     // raw F of the haloed tile (TMA destination), rows start at x0 - 4
    float br[RING][NPOS];      // b = (Mw - sm) kM of every haloed position (0 outside the lattice)
    float gr[NG][3][NIN];      // G of the interior positions
    int32_t zb[5][HY][ZP];     // z window sums of the haloed tile
    int32_t xb[5][HY][TX];     // x then z window sums
    unsigned long long fbar[RING];     // F(p) landed (TMA)
    unsigned long long sampled[RING];  // b(p), G(p) written (one arrival per sampler thread)
    unsigned long long consumed[RING]; // moment iteration p finished (one arrival per moment thread)
    unsigned long long xdone[RING];    // FFDP_L3_SPLITFIN: x stage of iteration p done (moment threads)
    unsigned long long ydone[RING];    // FFDP_L3_SPLITFIN: the samplers' outputs of iteration p done
    double red[NT / 32];
};

struct Params {
    Geom g;
    const float* f;       // buffer planes (the LDG path; the TMA path reads the tensor map)
    const float* u;       // buffer planes, 3 floats per voxel
    float* g_u;           // interior planes
    double* partial;      // one sum of n_i per CTA (summed in a fixed order afterwards)
    int32_t* miss;
    const float* ranges;  // device float[4]: F min, F max, M min, M max
    int32_t nx, ny, zchunk;
    int64_t plane, buf_z0, nz_global, z_begin, z_end;
    double eps, gi;
    // sampler position steps (+NS positions in the haloed tile): fp64 coordinate increments
    // for a step that stays in the row band (DX, DY) or wraps (DX - 38, DY + 1)
    double dstep[2][3];
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
// suspend-time hint of the mbarrier waits (ns): a waiting warp sleeps instead of spinning
// and leaves the issue slots to the other warp group
#ifndef FFDP_L3_SUSPEND_NS
#define FFDP_L3_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "n"(FFDP_L3_SUSPEND_NS)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    const uint32_t a = saddr(b);
    while (!mbar_try(a, parity)) {
    }
}
// The sampler warps' wait for a ring slot: they run ahead of the moment warps and wait there
// most of the time; a failed try_wait backs off with nanosleep so the spinning warps leave
// the issue slots to the moment warps (the spin loop was 45 of 475 instructions per voxel,
// ncu source counters, profiles/r02_full_lncc_fused.txt).
#ifndef FFDP_L3_SLEEP_NS
#define FFDP_L3_SLEEP_NS 256
#endif
__device__ __forceinline__ void mbar_wait_backoff(unsigned long long* b, uint32_t parity) {
    const uint32_t a = saddr(b);
    while (!mbar_try(a, parity)) {
        if (FFDP_L3_SLEEP_NS > 0) __nanosleep(FFDP_L3_SLEEP_NS);
    }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(saddr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void moment_sync() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

// Intensity frame from the value ranges: shift = mid-range, scale = 2^-e with
// |v - shift| < 2^e, so every scaled value lies in (-1, 1). The moving range includes 0
// (trilinear samples near the border blend in the zero padding, sampler.hpp:106-110).
__device__ __forceinline__ void frame1(float lo, float hi, float& s, float& k) {
    s = 0.5f * (lo + hi);
    const float h = fmaxf(hi - s, s - lo);
    int e = 0;
    if (h > 0.0f && h < 3.0e38f) (void)frexpf(h, &e);
    k = ldexpf(1.0f, -max(e, -100));
}

// The five quantised channels (int bits of MAGIC + round(2^21 x)): a, b, a^2, b^2, ab.
__device__ __forceinline__ void quant(float a, float b, int32_t (&q)[5]) {
    const float as = a * QSCALE, bs = b * QSCALE;
    q[0] = __float_as_int(fmaf(a, QSCALE, MAGIC));
    q[1] = __float_as_int(fmaf(b, QSCALE, MAGIC));
    q[2] = __float_as_int(fmaf(as, a, MAGIC));
    q[3] = __float_as_int(fmaf(bs, b, MAGIC));
    q[4] = __float_as_int(fmaf(as, b, MAGIC));
}

// in-lattice extent of the window of position g along an axis of n voxels
__device__ __forceinline__ int win_count(int64_t g, int64_t n) {
    return (int)(min(g + R, n - 1) - max(g - R, (int64_t)0) + 1);
}

// (only with both row-mapped sides, whose handshake it extends)
#define L3_SPLIT (FFDP_L3_SPLITFIN && FFDP_L3_ROWS && FFDP_L3_MROWS)

// The y stage and the outputs of plane q for OUTR rows oy.. of column ox (shared by the
// moment warps and, with FFDP_L3_SPLITFIN, the sampler warps, which finish the lower half
// of the tile's rows while the moment warps start the next plane's z stage).
struct FinConst {
    float sf, kF, smv, kM, ikM, cA, cB, cC, mF, mM, gi2, epsf;
    int32_t NU;
    bool poison;
    __device__ FinConst(const Params& P, float sf_, float kF_, float smv_, float kM_)
        : sf(sf_), kF(kF_), smv(smv_), kM(kM_) {
        ikM = 1.0f / kM;
        const float cAB = (float)(1.0 / (NWIN * NWIN * (double)QSCALE * (double)QSCALE));
        cA = cAB / (kF * kM);
        cB = cAB / (kF * kF);
        cC = cAB / (kM * kM);
        mF = (float)(1.0 / (NWIN * (double)QSCALE)) / kF;
        mM = (float)(1.0 / (NWIN * (double)QSCALE)) / kM;
        NU = (WIN * WIN * WIN) << 21;
        gi2 = 2.0f * (float)P.gi;
        epsf = (float)P.eps;
        poison = !(fabsf(sf) <= 3.0e38f && fabsf(smv) <= 3.0e38f);
    }
};

template <int OUTR>
__device__ __forceinline__ void finalize_rows(const Params& P, const Smem& sm, const FinConst& K, int it, int64_t q,
                                              int ox, int oy, const bool (&vout)[OUTR], const int (&cxy)[OUTR],
                                              float* go, int rs, float& nsum) {
    const int qslot = (it + RING - R) % RING, qg = (it + NG - R) % NG;
    int32_t S[OUTR][5];
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
        int32_t r[OUTR + 2 * R];
#pragma unroll
        for (int k = 0; k < OUTR + 2 * R; ++k) r[k] = sm.xb[ch][oy + k][ox];
        S[0][ch] = r[0] + r[1] + r[2] + r[3] + r[4] + r[5] + r[6];
#pragma unroll
        for (int j = 1; j < OUTR; ++j) S[j][ch] = S[j - 1][ch] + r[j + 2 * R] - r[j - 1];
    }
    const int cz = win_count(q, P.nz_global);
#pragma unroll
    for (int j = 0; j < OUTR; ++j) {
        if (!vout[j]) continue;
        const int32_t X = S[j][0], Y = S[j][1];
        // N^2 U^2 k k' {cov, var F, var M} of the quantised shifted values: exact in int64
        const int64_t TA = (int64_t)K.NU * S[j][4] - (int64_t)X * Y;
        const int64_t TB = (int64_t)K.NU * S[j][2] - (int64_t)X * X;
        const int64_t TC = (int64_t)K.NU * S[j][3] - (int64_t)Y * Y;
        const int cw = cxy[j] * cz;
        float a, b, cc, omw;
        if (cw == WIN * WIN * WIN) {
            a = (float)TA * K.cA;
            b = (float)TB * K.cB;
            cc = (float)TC * K.cC;
            omw = 0.0f;
        } else {
            // zero-padded border: the shift is missing from the N - cw outside positions
            const double U = (double)QSCALE, iUF = 1.0 / (U * (double)K.kF), iUM = 1.0 / (U * (double)K.kM);
            const double omc = NWIN - (double)cw, sfd = K.sf, smd = K.smv, cwd = cw, Xd = X, Yd = Y;
            const double invN2 = 1.0 / (NWIN * NWIN);
            a = (float)(((double)TA * (iUF * iUM) + omc * (smd * Xd * iUF + sfd * Yd * iUM + sfd * smd * cwd)) * invN2);
            b = (float)(((double)TB * (iUF * iUF) + omc * (2.0 * sfd * Xd * iUF + sfd * sfd * cwd)) * invN2);
            cc = (float)(((double)TC * (iUM * iUM) + omc * (2.0 * smd * Yd * iUM + smd * smd * cwd)) * invN2);
            omw = (float)(omc * (1.0 / NWIN));
        }
        const float D = fmaf(b, cc, K.epsf);
        const float invD = __fdividef(1.0f, D);  // D >= eps > 0
        nsum += a * a * invD;
        const float gamma = K.gi2 * a * invD;
        const float rab = a * b * invD;
        // F - muF and Mw - muM: (v - s) - (mu - s), mu - s = sum/(N U k) - s (1 - cw/N)
        const int hy = oy + j + R, hx = ox + R;
        const float fq = sm.fr[qslot][hy * FW + hx + 1];
        const float df = (fq - K.sf) - (float)X * K.mF + K.sf * omw;
        const float dm = sm.br[qslot][hy * HX + hx] * K.ikM - (float)Y * K.mM + K.smv * omw;
        // dL/dMw (lncc.hpp:262-278, ANTs)
        const float gmw = K.poison ? __int_as_float(0x7fc00000) : gamma * fmaf(-dm, rab, df);
        const int ii = (oy + j) * TX + ox;
        float* o = go + j * rs;
        o[0] = sm.gr[qg][0][ii] * gmw;
        o[1] = sm.gr[qg][1][ii] * gmw;
        o[2] = sm.gr[qg][2][ii] * gmw;
    }
}

// ------------------------------------------------------------------ sampler warps
template <int NM_, bool TMA, bool FULLWIN, bool OFF32>
__device__ __forceinline__ void sampler_warps(const CUtensorMap* umap, const CUtensorMap* mmap, const Params& P,
                                              Smem& sm, int st, int64_t pstart, int64_t pend,
                                              int64_t zc0, int64_t zc1, int x0, int y0, float kM, float nsmk) {
    using SP = Split<NM_>;
    constexpr int NS = SP::NS, SPOS = SP::SPOS;
    // positions h_i = st + NS i of the haloed tile (row-major, 38 per row)
    int32_t info[SPOS];  // h | interior index << 11 | valid << 21 | interior << 22 | wrap-step << 23
    int32_t off[SPOS];   // in-plane offset gy * nx + gx (0 outside the lattice)
    const int nx = P.nx, ny = P.ny;
#pragma unroll
    for (int i = 0; i < SPOS; ++i) {
        const int h = st + NS * i;
        const int hy = h / HX, hx = h - hy * HX;
        const int gx = x0 - R + hx, gy = y0 - R + hy;
        const bool ok = h < NPOS && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
        const bool in = hx >= R && hx < R + TX && hy >= R && hy < R + TY;
        const int ii = in ? (hy - R) * TX + (hx - R) : 0;
        // the step from h_i to h_{i+1}: (DX, DY) when hx < 38 - DX, else (DX - 38, DY + 1)
        info[i] = (h < NPOS ? h : 0) | (ii << 11) | ((int)ok << 21) | ((int)(in && ok) << 22) |
                  ((int)(hx >= HX - SP::DX) << 23);
        off[i] = ok ? gy * nx + gx : 0;
    }
    // fp64 lattice part of the coordinate of position h_0 without its z term (the z term is
    // added per plane, directly: results do not depend on where a chunk or a slab starts)
    double bxy0[3];
    {
        const int h = st, hy = h / HX, hx = h - hy * HX;
        const double gx = x0 - R + hx, gy = y0 - R + hy;
#pragma unroll
        for (int a = 0; a < 3; ++a) bxy0[a] = fma(P.g.P[3 * a + 1], gy, fma(P.g.P[3 * a + 0], gx, P.g.K[a]));
    }
    int miss = 0;
    const float dsc0 = P.g.dscale[0], dsc1 = P.g.dscale[1], dsc2 = P.g.dscale[2];
    const int64_t pl3 = 3 * P.plane;
    const float* ub = P.u + 3 * (pstart - P.buf_z0) * P.plane;  // u of plane p (uniform)
    // positions in two batches of NB0; the next batch's u is in flight during a batch
    static_assert(SPOS % 2 == 0, "sampler batches");
    constexpr int NB0 = SPOS / 2;
    float ua[NB0][3], ubb[NB0][3];
    auto load_u = [&](float (&uu)[NB0][3], const float* base, int i0, bool vz) {
#pragma unroll
        for (int k = 0; k < NB0; ++k) {
            const bool ok = vz && (info[i0 + k] >> 21 & 1);
            const float* q = base + 3 * off[i0 + k];
            uu[k][0] = ok ? __ldg(q) : 0.0f;
            uu[k][1] = ok ? __ldg(q + 1) : 0.0f;
            uu[k][2] = ok ? __ldg(q + 2) : 0.0f;
        }
    };
    load_u(ua, ub, 0, pstart >= 0 && pstart < P.nz_global);

    for (int64_t p = pstart; p < pend; ++p) {
        const int it = (int)(p - pstart);
        const int slot = it % RING, gslot = it % NG;
        // the moment warps must have finished iteration it - 2 (its b, F and G slots are reused)
        if (it >= 2) mbar_wait_backoff(&sm.consumed[(it - 2) % RING], (uint32_t)(((it - 2) / RING) & 1));
        const bool vz = p >= 0 && p < P.nz_global;
        const bool wantG = p >= zc0 && p < zc1;
        if (TMA && st == 0 && p + 2 < pend) {
            // u and the moving planes of plane p + 2 into L2 (bulk tensor prefetches): the batch
            // loads and, for moderate displacements, the corner gathers then hit L2, not HBM
            tma_prefetch_3d(umap, 3 * (x0 - R - 1), y0 - R, (int)(p + 2 - P.buf_z0));
            tma_prefetch_3d(mmap, x0 - MPF_X, y0 - MPF_Y, (int)(p + MPF_D - P.g.wz0 + 2));
        }
        const double zd = (double)p;
        double cb[3];  // coordinate base of position i (advanced per i)
#pragma unroll
        for (int a = 0; a < 3; ++a) cb[a] = fma(P.g.P[3 * a + 2], zd, bxy0[a]);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float(&uu)[NB0][3] = half ? ubb : ua;
            Cell c[NB0];
#pragma unroll
            for (int k = 0; k < NB0; ++k) {
                const int i = NB0 * half + k;
                if (i > 0) {
                    const int w = info[i - 1] >> 23 & 1;
#pragma unroll
                    for (int a = 0; a < 3; ++a) cb[a] += P.dstep[w][a];
                }
                cell_fix(fma(P.g.Q[0], (double)uu[k][0], cb[0]), c[k].i0[0], c[k].frac[0]);
                cell_fix(fma(P.g.Q[1], (double)uu[k][1], cb[1]), c[k].i0[1], c[k].frac[1]);
                cell_fix(fma(P.g.Q[2], (double)uu[k][2], cb[2]), c[k].i0[2], c[k].frac[2]);
            }
            if (half == 0) {
                load_u(ubb, ub, NB0, vz);
            } else if (p + 1 < pend) {
                ub += pl3;
                load_u(ua, ub, 0, p + 1 >= 0 && p + 1 < P.nz_global);
            }
            Corners cr[NB0];
#pragma unroll
            for (int k = 0; k < NB0; ++k) {
                int mk = 0;
                cr[k] = gather_pad<FULLWIN, OFF32>(P.g, c[k], mk);
                if (!FULLWIN) miss |= mk & (int)(vz && (info[NB0 * half + k] >> 21 & 1));
            }
#pragma unroll
            for (int k = 0; k < NB0; ++k) {
                const int i = NB0 * half + k;
                const int inf = info[i];
                const bool ok = vz && (inf >> 21 & 1);
                float v;
                if (wantG && (inf >> 22 & 1)) {
                    float d[3];
                    v = interp_grad(cr[k], c[k], d);
                    const int ii = inf >> 11 & 1023;
                    sm.gr[gslot][0][ii] = dsc0 * d[0];
                    sm.gr[gslot][1][ii] = dsc1 * d[1];
                    sm.gr[gslot][2][ii] = dsc2 * d[2];
                } else {
                    v = interp(cr[k], c[k]);
                }
                if (st + NS * i < NPOS) sm.br[slot][inf & 2047] = ok ? fmaf(v, kM, nsmk) : 0.0f;
            }
        }
        mbar_arrive(&sm.sampled[slot]);
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && (st & 31) == 0) atomicAdd(P.miss, __popc(anym));
}

// Row-mapped sampler (8 warps): a lane is an x column, so nearly every per-sample quantity
// is warp-uniform. The 32 output columns (haloed columns 3..34) of the 38 haloed rows are
// "main" passes -- warp w takes rows w, w + 8, ... (warps 0-5: 5 rows, 6-7: 4), G is wanted
// exactly on rows 3..34 (a uniform branch); the 6 halo columns x 38 rows = 228 "edge"
// positions are one pass per warp (e = 32 w + lane). Passes run in two batches of three:
// the cells of a batch, then all of its corner loads, then the interpolations, with the
// next batch's u in flight. Coordinates are evaluated directly from (gx, gy, p) -- no
// accumulated increments -- so a sample does not depend on the tiling or the chunking.
constexpr int SROWS = 5;  // main rows per warp (the last one absent on warps 6, 7)
constexpr int NEDGE = 6 * HY;
template <bool TMA, bool FULLWIN, bool OFF32>
__device__ __forceinline__ float sampler_rows(const CUtensorMap* umap, const CUtensorMap* mmap, const Params& P,
                                              Smem& sm, int st, int64_t pstart, int64_t pend, int64_t zc0,
                                              int64_t zc1, int x0, int y0, float kM, float nsmk, const FinConst& K) {
    const int lane = st & 31, w = st >> 5;
    const int nx = P.nx, ny = P.ny;
    // FFDP_L3_SPLITFIN: rows 16 + 2 w, 16 + 2 w + 1 of column lane of the moment iteration it
    // (plane pstart + it - R), after the moment warps' x stage of that iteration
    constexpr int FOUT = 2;
    float nsum_s = 0.0f;
    const int foy = TY / 2 + FOUT * w;
    bool fvout[FOUT];
    int fcxy[FOUT];
#pragma unroll
    for (int j = 0; j < FOUT; ++j) {
        fvout[j] = x0 + lane < nx && y0 + foy + j < ny;
        fcxy[j] = win_count(x0 + lane, nx) * win_count(y0 + foy + j, ny);
    }
    // the handshake barriers count output planes k = p - R - zc0 (warm-up iterations have none)
    auto fin_half = [&](int itm) {
        const int64_t pm = pstart + itm;
        const int k = (int)(pm - R - zc0);
        mbar_wait(&sm.xdone[k % RING], (uint32_t)((k / RING) & 1));
        float* go = P.g_u + 3 * ((pm - R - P.z_begin) * P.plane +
                                 (fvout[0] ? (int64_t)(y0 + foy) * nx + x0 + lane : 0));
        finalize_rows<FOUT>(P, sm, K, itm, pm - R, lane, foy, fvout, fcxy, go, 3 * nx, nsum_s);
        mbar_arrive(&sm.ydone[k % RING]);
    };
    // main column of this lane
    const int gxm = x0 + lane;
    const bool vxm = gxm < nx;
    // the lane's edge position
    const int e = 32 * w + lane;
    const int erow = e / 6, ecol = e - 6 * (e / 6);
    const int ehx = ecol < 3 ? ecol : TX + ecol;  // 0, 1, 2, 35, 36, 37
    const int gxe = x0 - R + ehx, gye = y0 - R + erow;
    const bool ve = e < NEDGE && gxe >= 0 && gxe < nx && gye >= 0 && gye < ny;
    double bxm[3], bxe[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        bxm[a] = fma(P.g.P[3 * a + 0], (double)gxm, P.g.K[a]);
        bxe[a] = fma(P.g.P[3 * a + 1], (double)gye, fma(P.g.P[3 * a + 0], (double)gxe, P.g.K[a]));
    }
    const int32_t offm = vxm ? gxm : 0;                      // + gy * nx per row
    const int32_t offe = ve ? gye * nx + gxe : 0;
    const int nrows = w < 6 ? SROWS : SROWS - 1;
    int miss = 0;
    const float dsc0 = P.g.dscale[0], dsc1 = P.g.dscale[1], dsc2 = P.g.dscale[2];
    const int64_t pl3 = 3 * P.plane;
    const float* ub = P.u + 3 * (pstart - P.buf_z0) * P.plane;  // u of plane p
    // pass j of a plane: main row hy = w + 8 j (j < nrows), then the edge pass (j = nrows)
    // NB passes per batch: 3 (two batches per plane, the second's u in flight during the
    // first's gathers) or 6 (one batch, all 48 corner loads of a lane in flight at once)
    constexpr int NB = FFDP_L3_NB, NBATCH = 6 / NB;
    float uu[NBATCH][NB][3];
    auto row_ok = [&](int j) {
        const int gy = y0 - R + w + 8 * j;
        return j < nrows && gy >= 0 && gy < ny;
    };
    auto load_u = [&](float (&u3)[NB][3], const float* base, int j0, bool vz) {
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int j = j0 + k;
            bool ok;
            int32_t o;
            if (j < SROWS) {
                ok = vz && vxm && row_ok(j);
                o = offm + (y0 - R + w + 8 * j) * nx;
            } else {
                ok = vz && ve;
                o = offe;
            }
            const float* q = base + 3 * (int64_t)(ok ? o : 0);
            u3[k][0] = ok ? __ldg(q) : 0.0f;
            u3[k][1] = ok ? __ldg(q + 1) : 0.0f;
            u3[k][2] = ok ? __ldg(q + 2) : 0.0f;
        }
    };
    load_u(uu[0], ub, 0, pstart >= 0 && pstart < P.nz_global);

    for (int64_t p = pstart; p < pend; ++p) {
        const int it = (int)(p - pstart);
        const int slot = it % RING, gslot = it % NG;
        // the moment warps must have finished iteration it - 2 (its b, F and G slots are reused)
        if (it >= 2) mbar_wait_backoff(&sm.consumed[(it - 2) % RING], (uint32_t)(((it - 2) / RING) & 1));
        const bool vz = p >= 0 && p < P.nz_global;
        const bool wantG = p >= zc0 && p < zc1;
        if (TMA && st == 0 && p + 2 < pend) {
            tma_prefetch_3d(umap, 3 * (x0 - R - 1), y0 - R, (int)(p + 2 - P.buf_z0));
            tma_prefetch_3d(mmap, x0 - MPF_X, y0 - MPF_Y, (int)(p + MPF_D - P.g.wz0 + 2));
        }
        const double zd = (double)p;
        double bzm[3], bze[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            bzm[a] = fma(P.g.P[3 * a + 2], zd, bxm[a]);
            bze[a] = fma(P.g.P[3 * a + 2], zd, bxe[a]);
        }
#pragma unroll
        for (int half = 0; half < NBATCH; ++half) {
            float(&u3)[NB][3] = uu[half];
            Cell c[NB];
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const int j = NB * half + k;
                double b0, b1, b2;
                if (j < SROWS) {
                    const double gy = (double)(y0 - R + w + 8 * j);
                    b0 = fma(P.g.P[1], gy, bzm[0]);
                    b1 = fma(P.g.P[4], gy, bzm[1]);
                    b2 = fma(P.g.P[7], gy, bzm[2]);
                } else {
                    b0 = bze[0];
                    b1 = bze[1];
                    b2 = bze[2];
                }
                cell_fix(fma(P.g.Q[0], (double)u3[k][0], b0), c[k].i0[0], c[k].frac[0]);
                cell_fix(fma(P.g.Q[1], (double)u3[k][1], b1), c[k].i0[1], c[k].frac[1]);
                cell_fix(fma(P.g.Q[2], (double)u3[k][2], b2), c[k].i0[2], c[k].frac[2]);
            }
            // the other batch's u (this plane's second batch, or the next plane's first)
            if (half == 0 && NBATCH == 2) {
                load_u(uu[NBATCH - 1], ub, NB, vz);
            } else if (p + 1 < pend) {
                ub += pl3;
                load_u(uu[0], ub, 0, p + 1 >= 0 && p + 1 < P.nz_global);
            }
            Corners cr[NB];
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                int mk = 0;
                cr[k] = gather_pad<FULLWIN, OFF32>(P.g, c[k], mk);
                const int j = NB * half + k;
                const bool ok = vz && (j < SROWS ? (vxm && row_ok(j)) : ve);
                if (!FULLWIN) miss |= mk & (int)ok;
            }
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const int j = NB * half + k;
                if (j < SROWS) {
                    if (j >= nrows) continue;  // warps 6, 7: four main rows
                    const int hy = w + 8 * j;
                    const bool ok = vz && vxm && row_ok(j);
                    float v;
                    if (wantG && hy >= R && hy < R + TY) {  // warp-uniform
                        float d[3];
                        v = interp_grad(cr[k], c[k], d);
                        const int ii = (hy - R) * TX + lane;
                        sm.gr[gslot][0][ii] = dsc0 * d[0];
                        sm.gr[gslot][1][ii] = dsc1 * d[1];
                        sm.gr[gslot][2][ii] = dsc2 * d[2];
                    } else {
                        v = interp(cr[k], c[k]);
                    }
                    sm.br[slot][hy * HX + R + lane] = ok ? fmaf(v, kM, nsmk) : 0.0f;
                } else {
                    const float v = interp(cr[k], c[k]);
                    if (e < NEDGE) sm.br[slot][erow * HX + ehx] = (vz && ve) ? fmaf(v, kM, nsmk) : 0.0f;
                }
            }
        }
        mbar_arrive(&sm.sampled[slot]);
        if (L3_SPLIT && p - 1 >= zc0 + R) fin_half(it - 1);
    }
    if (L3_SPLIT && pend - 1 >= zc0 + R) fin_half((int)(pend - 1 - pstart));
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && lane == 0) atomicAdd(P.miss, __popc(anym));
    return nsum_s;
}

// ------------------------------------------------------------------ moment warps
template <int NM_, bool TMA>
__device__ __forceinline__ float moment_warps(const CUtensorMap* fmap, const Params& P, Smem& sm, int mt,
                                              int64_t pstart, int64_t pend, int64_t zc0, int x0, int y0, float sf,
                                              float kF, float smv, float kM) {
    using SP = Split<NM_>;
    constexpr int NM = SP::NM, MPOS = SP::MPOS, MJOBS = SP::MJOBS, OUTR = SP::OUTR;
    const float nsfk = -sf * kF, ikM = 1.0f / kM;
    auto issue = [&](int64_t p, int s) {
        mbar_expect_tx(&sm.fbar[s], FW * HY * 4);
        // the innermost TMA coordinate must be 16-byte aligned (measured: x0 - 3 faults with an
        // illegal instruction, tools/probe_tma2.cu): the box starts one column early
        tma_load_3d(&sm.fr[s][0], fmap, &sm.fbar[s], x0 - R - 1, y0 - R, (int)(p - P.buf_z0));
    };
    if (TMA && mt == 0) issue(pstart, 0);

    // z-stage positions h = mt + 256 i: F ring offset | valid << 12 (h < 1444 when set)
    int32_t zpos[MPOS];
#pragma unroll
    for (int i = 0; i < MPOS; ++i) {
        const int h = mt + NM * i;
        const int hy = h / HX, hx = h - hy * HX;
        const int gx = x0 - R + hx, gy = y0 - R + hy;
        const bool ok = h < NPOS && gx >= 0 && gx < P.nx && gy >= 0 && gy < P.ny;
        zpos[i] = h < NPOS ? (hy * FW + hx + 1) | ((int)ok << 12) : -1;
    }
    const float* fsrc = P.f + (pstart - P.buf_z0) * P.plane;  // LDG path: F of plane p
    // x-stage jobs: z buffer offset | x buffer offset << 16 (-1: none)
    int32_t xjob[MJOBS];
#pragma unroll
    for (int i = 0; i < MJOBS; ++i) {
        const int j = mt + NM * i;
        const int ch = j / (HY * (TX / 4)), r = j % (HY * (TX / 4));
        const int hy = r >> 3, run = r & 7;
        xjob[i] = j < XJOBS ? ((ch * HY + hy) * ZP + 4 * run) | (((ch * HY + hy) * TX + 4 * run) << 16) : -1;
    }
    // outputs: column ox, rows oy .. oy + OUTR - 1
    const int ox = mt & 31, oy = OUTR * (mt >> 5);
    const int gx = x0 + ox;
    bool vout[OUTR];
    int cxy[OUTR];
#pragma unroll
    for (int j = 0; j < OUTR; ++j) {
        vout[j] = gx < P.nx && y0 + oy + j < P.ny;
        cxy[j] = win_count(gx, P.nx) * win_count(y0 + oy + j, P.ny);
    }
    const int64_t pl3 = 3 * P.plane;
    float* go = P.g_u + 3 * ((zc0 - P.z_begin) * P.plane + (vout[0] ? (int64_t)(y0 + oy) * P.nx + gx : 0));
    const int rs = 3 * P.nx;
    // finalize constants: 1 / (N^2 U^2 k k') and the mean scales 1 / (N U k)
    const float cAB = (float)(1.0 / (NWIN * NWIN * (double)QSCALE * (double)QSCALE));
    const float cA = cAB / (kF * kM), cB = cAB / (kF * kF), cC = cAB / (kM * kM);
    const float mF = (float)(1.0 / (NWIN * (double)QSCALE)) / kF, mM = (float)(1.0 / (NWIN * (double)QSCALE)) / kM;
    const int32_t NU = (WIN * WIN * WIN) << 21;  // N * 2^21 < 2^31
    const float gi2 = 2.0f * (float)P.gi, epsf = (float)P.eps;
    // a NaN in F or M (NaN value ranges, ffdp_minmax) poisons the loss and the gradient
    const bool poison = !(fabsf(sf) <= 3.0e38f && fabsf(smv) <= 3.0e38f);

    int32_t zs[MPOS][5];
#pragma unroll
    for (int i = 0; i < MPOS; ++i)
#pragma unroll
        for (int c = 0; c < 5; ++c) zs[i][c] = 0;
    float nsum = 0.0f;

    for (int64_t p = pstart; p < pend; ++p) {
        const int it = (int)(p - pstart);
        const int slot = it % RING;
        const uint32_t par = (uint32_t)((it / RING) & 1);
        if (TMA && mt == 0 && p + 1 < pend) issue(p + 1, (it + 1) % RING);
        const bool vz = p >= 0 && p < P.nz_global;
        const bool vzo = it >= WIN && p - WIN >= 0 && p - WIN < P.nz_global;
        const int oslot = (it + RING - WIN) % RING;  // plane p - 7
        const bool warm = p < zc0 + R;               // no output plane finishes yet

        // ---- z stage: + plane p, - plane p-7 (exact integer sums)
        if (!TMA) {
#pragma unroll
            for (int i = 0; i < MPOS; ++i) {
                const int zp = zpos[i];
                if (zp >= 0 && (zp >> 12 & 1)) {
                    const int fo = zp & 4095, hy = fo / FW, hx = fo - hy * FW - 1;
                    sm.fr[slot][fo] = vz ? __ldg(fsrc + (int64_t)(y0 - R + hy) * P.nx + (x0 - R + hx)) : 0.0f;
                }
            }
            fsrc += P.plane;
        }
        mbar_wait(&sm.sampled[slot], par);
        if (TMA) mbar_wait(&sm.fbar[slot], par);
#pragma unroll
        for (int i = 0; i < MPOS; ++i) {
            const int zp = zpos[i];
            if (zp < 0) break;
            const int fo = zp & 4095, h = mt + NM * i;
            const bool ok = zp >> 12 & 1;
            const float an = (ok && vz) ? fmaf(sm.fr[slot][fo], kF, nsfk) : 0.0f;
            const float ao = (ok && vzo) ? fmaf(sm.fr[oslot][fo], kF, nsfk) : 0.0f;
            const float bn = sm.br[slot][h];
            const float bo = it >= WIN ? sm.br[oslot][h] : 0.0f;
            int32_t qn[5], qo[5];
            quant(an, bn, qn);
            quant(ao, bo, qo);
#pragma unroll
            for (int ch = 0; ch < 5; ++ch) zs[i][ch] += qn[ch] - qo[ch];
            if (!warm) {
                const int hy = h / HX, hx = h - hy * HX;
#pragma unroll
                for (int ch = 0; ch < 5; ++ch) sm.zb[ch][hy][hx] = zs[i][ch];
            }
        }
        moment_sync<NM>();
        if (!warm) {
            // ---- x stage: runs of 4 sliding sums of the z sums (three 16-byte loads per run)
#pragma unroll
            for (int i = 0; i < MJOBS; ++i) {
                if (xjob[i] < 0) break;
                const int4* zr = reinterpret_cast<const int4*>(&sm.zb[0][0][0] + (xjob[i] & 0xFFFF));
                const int4 a = zr[0], b = zr[1], c4 = zr[2];
                const int32_t s0 = a.x + a.y + a.z + a.w + b.x + b.y + b.z;
                const int32_t s1 = s0 + b.w - a.x;
                const int32_t s2 = s1 + c4.x - a.y;
                const int32_t s3 = s2 + c4.y - a.z;
                *reinterpret_cast<int4*>(&sm.xb[0][0][0] + (xjob[i] >> 16)) = make_int4(s0, s1, s2, s3);
            }
            moment_sync<NM>();

            // ---- y stage (OUTR sliding sums down the column) and the outputs of plane q = p - 3
            const int64_t q = p - R;
            const int qslot = (it + RING - R) % RING, qg = (it + NG - R) % NG;
            int32_t S[OUTR][5];
#pragma unroll
            for (int ch = 0; ch < 5; ++ch) {
                int32_t r[OUTR + 2 * R];
#pragma unroll
                for (int k = 0; k < OUTR + 2 * R; ++k) r[k] = sm.xb[ch][oy + k][ox];
                S[0][ch] = r[0] + r[1] + r[2] + r[3] + r[4] + r[5] + r[6];
#pragma unroll
                for (int j = 1; j < OUTR; ++j) S[j][ch] = S[j - 1][ch] + r[j + 2 * R] - r[j - 1];
            }
            const int cz = win_count(q, P.nz_global);
#pragma unroll
            for (int j = 0; j < OUTR; ++j) {
                if (!vout[j]) continue;
                const int32_t X = S[j][0], Y = S[j][1];
                // N^2 U^2 k k' {cov, var F, var M} of the quantised shifted values: exact in int64
                const int64_t TA = (int64_t)NU * S[j][4] - (int64_t)X * Y;
                const int64_t TB = (int64_t)NU * S[j][2] - (int64_t)X * X;
                const int64_t TC = (int64_t)NU * S[j][3] - (int64_t)Y * Y;
                const int cw = cxy[j] * cz;
                float a, b, cc, omw;
                if (cw == WIN * WIN * WIN) {
                    a = (float)TA * cA;
                    b = (float)TB * cB;
                    cc = (float)TC * cC;
                    omw = 0.0f;
                } else {
                    // zero-padded border: the shift is missing from the N - cw outside positions
                    const double U = (double)QSCALE, iUF = 1.0 / (U * (double)kF), iUM = 1.0 / (U * (double)kM);
                    const double omc = NWIN - (double)cw, sfd = sf, smd = smv, cwd = cw, Xd = X, Yd = Y;
                    const double invN2 = 1.0 / (NWIN * NWIN);
                    a = (float)(((double)TA * (iUF * iUM) + omc * (smd * Xd * iUF + sfd * Yd * iUM + sfd * smd * cwd)) *
                                invN2);
                    b = (float)(((double)TB * (iUF * iUF) + omc * (2.0 * sfd * Xd * iUF + sfd * sfd * cwd)) * invN2);
                    cc = (float)(((double)TC * (iUM * iUM) + omc * (2.0 * smd * Yd * iUM + smd * smd * cwd)) * invN2);
                    omw = (float)(omc * (1.0 / NWIN));
                }
                const float D = fmaf(b, cc, epsf);
                const float invD = __fdividef(1.0f, D);  // D >= eps > 0
                nsum += a * a * invD;
                const float gamma = gi2 * a * invD;
                const float rab = a * b * invD;
                // F - muF and Mw - muM: (v - s) - (mu - s), mu - s = sum/(N U k) - s (1 - cw/N)
                const int hy = oy + j + R, hx = ox + R;
                const float fq = sm.fr[qslot][hy * FW + hx + 1];
                const float df = (fq - sf) - (float)X * mF + sf * omw;
                const float dm = sm.br[qslot][hy * HX + hx] * ikM - (float)Y * mM + smv * omw;
                const float gmw = poison ? __int_as_float(0x7fc00000) : gamma * fmaf(-dm, rab, df);  // dL/dMw (lncc.hpp:262-278, ANTs)
                const int ii = (oy + j) * TX + ox;
                float* o = go + j * rs;
                o[0] = sm.gr[qg][0][ii] * gmw;
                o[1] = sm.gr[qg][1][ii] * gmw;
                o[2] = sm.gr[qg][2][ii] * gmw;
            }
            go += pl3;
        }
        mbar_arrive(&sm.consumed[slot]);
    }
    return poison ? __int_as_float(0x7fc00000) : nsum;
}

// Row-mapped moment warps (FFDP_L3_MROWS): the z stage takes the positions of the row
// sampler's layout (main rows w + 8 j at column 3 + lane, edge position 32 w + lane), so
// every shared-memory offset is a row base plus the lane (no per-position decode to keep in
// registers), and x jobs decode as (row-of-channel j >> 3, run j & 7). The handshake with
// the samplers and the y stage / finalize are those of moment_warps.
template <bool TMA>
__device__ __forceinline__ float moment_rows(const CUtensorMap* fmap, const Params& P, Smem& sm, int mt,
                                             int64_t pstart, int64_t pend, int64_t zc0, int x0, int y0, float sf,
                                             float kF, float smv, float kM) {
    // FFDP_L3_SPLITFIN: the moment warps finish rows 0-15 (2 per thread), the sampler warps 16-31
    constexpr int NM = 256, OUTR = L3_SPLIT ? NIN / NM / 2 : NIN / NM, MR = SROWS, NJ = MR + 1;
    const int lane = mt & 31, w = mt >> 5;
    const float nsfk = -sf * kF, ikM = 1.0f / kM;
    auto issue = [&](int64_t p, int s) {
        mbar_expect_tx(&sm.fbar[s], FW * HY * 4);
        tma_load_3d(&sm.fr[s][0], fmap, &sm.fbar[s], x0 - R - 1, y0 - R, (int)(p - P.buf_z0));
    };
    if (TMA && mt == 0) issue(pstart, 0);
    const int nx = P.nx, ny = P.ny;
    const int nrows = w < 6 ? SROWS : SROWS - 1;
    const bool vxm = x0 + lane < nx;
    const int e = 32 * w + lane;
    const int erow = e / 6, ecol = e - 6 * (e / 6);
    const int ehx = ecol < 3 ? ecol : TX + ecol;
    const bool ehas = e < NEDGE;
    const bool ve = ehas && x0 - R + ehx >= 0 && x0 - R + ehx < nx && y0 - R + erow >= 0 && y0 - R + erow < ny;
    const float* fsrc = P.f + (pstart - P.buf_z0) * P.plane;  // LDG path: F of plane p
    const int ox = lane, oy = OUTR * w;
    const int gx = x0 + ox;
    bool vout[OUTR];
    int cxy[OUTR];
#pragma unroll
    for (int j = 0; j < OUTR; ++j) {
        vout[j] = gx < nx && y0 + oy + j < ny;
        cxy[j] = win_count(gx, nx) * win_count(y0 + oy + j, ny);
    }
    const int64_t pl3 = 3 * P.plane;
    float* go = P.g_u + 3 * ((zc0 - P.z_begin) * P.plane + (vout[0] ? (int64_t)(y0 + oy) * nx + gx : 0));
    const int rs = 3 * nx;
    const FinConst K(P, sf, kF, smv, kM);
    const bool poison = K.poison;

    int32_t zs[NJ][5];
#pragma unroll
    for (int i = 0; i < NJ; ++i)
#pragma unroll
        for (int c = 0; c < 5; ++c) zs[i][c] = 0;
    float nsum = 0.0f;

    for (int64_t p = pstart; p < pend; ++p) {
        const int it = (int)(p - pstart);
        const int slot = it % RING;
        const uint32_t par = (uint32_t)((it / RING) & 1);
        if (TMA && mt == 0 && p + 1 < pend) issue(p + 1, (it + 1) % RING);
        const bool vz = p >= 0 && p < P.nz_global;
        const bool vzo = it >= WIN && p - WIN >= 0 && p - WIN < P.nz_global;
        const int oslot = (it + RING - WIN) % RING;
        const bool warm = p < zc0 + R;
        if (!TMA) {
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const bool main = j < MR;
                if (main ? (j >= nrows) : !ve) continue;
                const int hy = main ? w + 8 * j : erow, hx = main ? R + lane : ehx;
                const int gy = y0 - R + hy, gxx = x0 - R + hx;
                if (main && !(vxm && gy >= 0 && gy < ny)) continue;
                sm.fr[slot][hy * FW + hx + 1] = vz ? __ldg(fsrc + (int64_t)gy * nx + gxx) : 0.0f;
            }
            fsrc += P.plane;
        }
        mbar_wait(&sm.sampled[slot], par);
        if (TMA) mbar_wait(&sm.fbar[slot], par);
        // ---- z stage: + plane p, - plane p-7 (exact integer sums)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const bool main = j < MR;
            if (main ? (j >= nrows) : !ehas) continue;
            const int hy = main ? w + 8 * j : erow, hx = main ? R + lane : ehx;
            const int gy = y0 - R + hy;
            const bool ok = main ? (vxm && gy >= 0 && gy < ny) : ve;
            const int fo = hy * FW + hx + 1, bo = hy * HX + hx;
            const float an = (ok && vz) ? fmaf(sm.fr[slot][fo], kF, nsfk) : 0.0f;
            const float ao = (ok && vzo) ? fmaf(sm.fr[oslot][fo], kF, nsfk) : 0.0f;
            const float bn = sm.br[slot][bo];
            const float bo_ = it >= WIN ? sm.br[oslot][bo] : 0.0f;
            int32_t qn[5], qo[5];
            quant(an, bn, qn);
            quant(ao, bo_, qo);
#pragma unroll
            for (int ch = 0; ch < 5; ++ch) zs[j][ch] += qn[ch] - qo[ch];
            if (!warm) {
                int32_t* zb = &sm.zb[0][hy][hx];
#pragma unroll
                for (int ch = 0; ch < 5; ++ch) zb[ch * HY * ZP] = zs[j][ch];
            }
        }
        moment_sync<NM>();
        if (!warm) {
            // the sampler warps' half of the previous plane's outputs must have read xb
            // (output planes k = p - R - zc0 index the handshake barriers)
            const int k = (int)(p - R - zc0);
            if (L3_SPLIT && k >= 1) mbar_wait(&sm.ydone[(k - 1) % RING], (uint32_t)(((k - 1) / RING) & 1));
#pragma unroll
            for (int i = 0; i < (XJOBS + NM - 1) / NM; ++i) {
                const int j = mt + NM * i;
                if (j >= XJOBS) break;
                const int rowch = j >> 3, run = j & 7;
                const int4* zr = reinterpret_cast<const int4*>(&sm.zb[0][0][0] + rowch * ZP + 4 * run);
                const int4 a = zr[0], b = zr[1], c4 = zr[2];
                const int32_t s0 = a.x + a.y + a.z + a.w + b.x + b.y + b.z;
                const int32_t s1 = s0 + b.w - a.x;
                const int32_t s2 = s1 + c4.x - a.y;
                const int32_t s3 = s2 + c4.y - a.z;
                *reinterpret_cast<int4*>(&sm.xb[0][0][0] + rowch * TX + 4 * run) = make_int4(s0, s1, s2, s3);
            }
            moment_sync<NM>();
            if (L3_SPLIT) mbar_arrive(&sm.xdone[k % RING]);
            finalize_rows<OUTR>(P, sm, K, it, p - R, ox, oy, vout, cxy, go, rs, nsum);
            go += pl3;
        }
        mbar_arrive(&sm.consumed[slot]);
    }
    return poison ? __int_as_float(0x7fc00000) : nsum;
}

template <int NM_, bool TMA, bool FULLWIN, bool OFF32>
__global__ void __launch_bounds__(NT, 1) k_lncc_fused(const __grid_constant__ CUtensorMap fmap,
                                                      const __grid_constant__ CUtensorMap umap,
                                                      const __grid_constant__ CUtensorMap mmap, const Params P) {
    using SP = Split<NM_>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int64_t zc0 = P.z_begin + (int64_t)blockIdx.z * P.zchunk;
    const int64_t zc1 = min(P.z_end, zc0 + P.zchunk);
    if (zc0 >= zc1) return;
    const int64_t pstart = zc0 - R, pend = zc1 + R;

    float sf, kF, smv, kM;
    frame1(P.ranges[0], P.ranges[1], sf, kF);
    frame1(fminf(P.ranges[2], 0.0f), fmaxf(P.ranges[3], 0.0f), smv, kM);
    if (P.ranges[2] != P.ranges[2]) smv = P.ranges[2];  // NaN in M: poison (fminf drops it)

    if (t == 0) {
        for (int s = 0; s < RING; ++s) {
            mbar_init(&sm.fbar[s], 1);
            mbar_init(&sm.sampled[s], SP::NS);
            mbar_init(&sm.consumed[s], SP::NM);
            mbar_init(&sm.xdone[s], SP::NM);
            mbar_init(&sm.ydone[s], SP::NS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    float nsum = 0.0f;
    if (t < SP::NM) {
        if (SP::RM != 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SP::RM));
#if FFDP_L3_ROWS && FFDP_L3_MROWS
        if (SP::NM == 256)
            nsum = moment_rows<TMA>(&fmap, P, sm, t, pstart, pend, zc0, x0, y0, sf, kF, smv, kM);
        else
#endif
            nsum = moment_warps<NM_, TMA>(&fmap, P, sm, t, pstart, pend, zc0, x0, y0, sf, kF, smv, kM);
    } else {
        if (SP::RS != 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SP::RS));
#if FFDP_L3_ROWS
        if (SP::NS == 256)
            nsum = sampler_rows<TMA, FULLWIN, OFF32>(&umap, &mmap, P, sm, t - SP::NM, pstart, pend, zc0, zc1, x0, y0,
                                                     kM, -smv * kM, FinConst(P, sf, kF, smv, kM));
        else
#endif
            sampler_warps<NM_, TMA, FULLWIN, OFF32>(&umap, &mmap, P, sm, t - SP::NM, pstart, pend, zc0, zc1, x0, y0,
                                                    kM, -smv * kM);
    }
    const double cta = block_sum<NT>((double)nsum, sm.red);
    if (t == 0) P.partial[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = cta;
}

__global__ void __launch_bounds__(256) k_add_partials3(const double* partial, int64_t n, double* sum_n) {
    __shared__ double red[8];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 256) v += partial[i];
    v = block_sum<256>(v, red);
    if (threadIdx.x == 0) *sum_n += v;
}

// Planes per z chunk: the fewest (waves x (planes + half-cost warm-up planes)).
inline int32_t pick_zchunk(int64_t tiles, int64_t nzs, int64_t capacity) {
    int64_t best = 1, best_cost = INT64_MAX;
    for (int64_t ch = 1; ch <= std::min<int64_t>(nzs, std::max<int64_t>(256, (nzs + 255) / 256)); ++ch) {
        const int64_t zc = (nzs + ch - 1) / ch;
        if (zc > 256) continue;  // measured: 1024^3 runs 2 % faster in 256-plane chunks than in one
        const int64_t n = (nzs + zc - 1) / zc;
        const int64_t waves = (tiles * n + capacity - 1) / capacity;
        const int64_t cost = waves * (2 * zc + 2 * R + 2 * R);  // warm-up planes cost about half
        if (cost < best_cost) best_cost = cost, best = zc;
    }
    return (int32_t)best;
}

}  // namespace l3

// ------------------------------------------------------------------ host side
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

template <int NM_, bool T_, bool F_, bool O_>
static void launch_fused(const CUtensorMap (&map)[3], const l3::Params& P, dim3 grid, cudaStream_t st) {
    static std::atomic<unsigned long long> attr_mask{0};
    once_per_device(attr_mask, [] {
        cudaFuncSetAttribute(l3::k_lncc_fused<NM_, T_, F_, O_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(l3::Smem));
    });
    l3::k_lncc_fused<NM_, T_, F_, O_><<<grid, l3::NT, sizeof(l3::Smem), st>>>(map[0], map[1], map[2], P);
}

static int64_t lncc3_max_ctas(const ffdp_dims& d, const ffdp_slab& s) {
    const int64_t tx = (d.nx + l3::TX - 1) / l3::TX, ty = (d.ny + l3::TY - 1) / l3::TY;
    // pick_zchunk's chunk count never exceeds this bound
    const int64_t nzs = std::max<int64_t>(1, s.z_end - s.z_begin);
    return tx * ty * std::min<int64_t>(nzs, std::max<int64_t>(256, (nzs + 255) / 256));
}

// workspace: 4 floats of value ranges (when computed here), then one double per CTA
int64_t lncc3_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s) { return 16 + 8 * lncc3_max_ctas(d, s); }

int lncc3_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, const float* ranges, float* g_u, double* sum_n,
               int32_t* miss, void* workspace, cudaStream_t st) {
    using namespace l3;
    float* rg = reinterpret_cast<float*>(workspace);
    double* partial = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 16);
    const int64_t plane = d.nx * d.ny;
    if (!ranges) {
        // the value ranges of F (buffer planes) and of the moving window (its zero border included)
        int rc = ffdp_minmax(f, plane * d.nz, rg, st);
        if (rc) return rc;
        // pad = 2: data is the zero-bordered block itself (ffdp_image_window)
        const int64_t mn = (int64_t)(m.dims.nx + 2 * m.pad) * (m.dims.ny + 2 * m.pad) *
                           (m.z_end - m.z_begin + 2 * m.pad);
        rc = ffdp_minmax(m.data, mn, rg + 2, st);
        if (rc) return rc;
        ranges = rg;
    }
    Params P;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    P.g = make_geom(m, out, args);
    // the warp split (FFDP_LNCC_NM = 128 or 256 moment threads; measured: DESIGN.md)
    static const int nm_env = getenv("FFDP_LNCC_NM") ? atoi(getenv("FFDP_LNCC_NM")) : 0;
    const int nm = nm_env == 128 ? 128 : 256;
    // sampler position step h -> h + NS in the 38-wide haloed tile (sampler_warps)
    {
        const int ns = NT - nm, dx = ns % HX, dy = ns / HX;
        for (int a = 0; a < 3; ++a) {
            P.dstep[0][a] = (double)dx * P.g.P[3 * a + 0] + (double)dy * P.g.P[3 * a + 1];
            P.dstep[1][a] = (double)(dx - HX) * P.g.P[3 * a + 0] + (double)(dy + 1) * P.g.P[3 * a + 1];
        }
    }
    P.f = f;
    P.u = u;
    P.g_u = g_u;
    P.partial = partial;
    P.miss = miss;
    P.ranges = ranges;
    P.nx = (int32_t)d.nx;
    P.ny = (int32_t)d.ny;
    P.plane = plane;
    P.buf_z0 = s.buf_z0;
    P.nz_global = s.nz_global;
    P.z_begin = s.z_begin;
    P.z_end = s.z_end;
    P.eps = eps;
    P.gi = gi;

    // tensor maps: F (TMA loads), u and the zero-bordered moving window (L2 prefetches)
    CUtensorMap map[3];
    memset(map, 0, sizeof(map));
    // TMA needs 16-byte row strides; FFDP_NO_TMA=1 forces the LDG path (diagnostics)
    static const bool no_tma = getenv("FFDP_NO_TMA") && getenv("FFDP_NO_TMA")[0] == '1';
    bool tma = !no_tma && (d.nx % 4) == 0 && ((uintptr_t)f % 16) == 0 && ((uintptr_t)u % 16) == 0 &&
               ((uintptr_t)m.data % 16) == 0;
    if (tma) {
        auto enc = tensor_map_encoder();
        tma = enc != nullptr;
        auto make = [&](CUtensorMap* mp, const float* base, cuuint64_t n0, cuuint64_t n1, cuuint64_t n2,
                        cuuint32_t b0, cuuint32_t b1) {
            const cuuint64_t dims[3] = {n0, n1, n2};
            const cuuint64_t strides[2] = {n0 * 4, n0 * n1 * 4};
            const cuuint32_t box[3] = {b0, b1, 1};
            const cuuint32_t es[3] = {1, 1, 1};
            return enc(mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        };
        const cuuint64_t mx = m.dims.nx + 4, my = m.dims.ny + 4, mz = m.z_end - m.z_begin + 4;
        tma = tma && make(&map[0], f, d.nx, d.ny, d.nz, FW, HY) && make(&map[1], u, 3 * d.nx, d.ny, d.nz, 3 * FW, HY) &&
              make(&map[2], m.data, mx, my, mz, MPF_W, MPF_H);
    }
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
    const bool o32 = window_off32(P.g);
    const int64_t tx = (d.nx + TX - 1) / TX, ty = (d.ny + TY - 1) / TY;
    const int64_t nzs = s.z_end - s.z_begin;
    // planes per CTA (FFDP_LNCC_ZCHUNK overrides the wave model, for measurements)
    static const int zc_env = getenv("FFDP_LNCC_ZCHUNK") ? atoi(getenv("FFDP_LNCC_ZCHUNK")) : 0;
    P.zchunk = pick_zchunk(tx * ty, nzs, num_sms());
    if (zc_env > 0) {
        const int64_t nzs1 = std::max<int64_t>(1, nzs);
        const int64_t max_chunks = std::min<int64_t>(nzs1, std::max<int64_t>(256, (nzs1 + 255) / 256));
        P.zchunk = (int32_t)std::max<int64_t>(std::min<int64_t>(zc_env, nzs1), (nzs1 + max_chunks - 1) / max_chunks);
    }
    const int64_t chunks = (nzs + P.zchunk - 1) / P.zchunk;
    if (ty > 65535 || chunks > 65535) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: grid too large");
    const dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)chunks);
    const int key = (nm == 128) * 8 + tma * 4 + full * 2 + o32;
    switch (key) {
#define FFDP_L3_CASE(K_)                                                                                       \
    case K_:                                                                                                   \
        launch_fused<(K_ & 8) ? 128 : 256, (K_ & 4) != 0, (K_ & 2) != 0, (K_ & 1) != 0>(map, P, grid, st); \
        break;
        FFDP_L3_CASE(0) FFDP_L3_CASE(1) FFDP_L3_CASE(2) FFDP_L3_CASE(3) FFDP_L3_CASE(4) FFDP_L3_CASE(5)
        FFDP_L3_CASE(6) FFDP_L3_CASE(7) FFDP_L3_CASE(8) FFDP_L3_CASE(9) FFDP_L3_CASE(10) FFDP_L3_CASE(11)
        FFDP_L3_CASE(12) FFDP_L3_CASE(13) FFDP_L3_CASE(14) FFDP_L3_CASE(15)
#undef FFDP_L3_CASE
    }
    if (sum_n) l3::k_add_partials3<<<1, 256, 0, st>>>(partial, tx * ty * chunks, sum_n);
    return check_launch("step_lncc (fused one pass)");
}

}  // namespace ffdp
