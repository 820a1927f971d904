// step_lncc2.cu -- the warp + LNCC(ANTs) forward+backward step as TWO streaming passes.
//
// Same reference sequence as step_lncc.cu (registration.hpp:277-312: ring_sample ->
// dist_lncc(ants) -> ring_sample_backward(want warp)), split where the halo is:
//
//   pass 1  k_lncc_sample: every voxel of the slab (+ the r = 3 halo planes the window
//           needs) is warped exactly once: Mw = fused_sample(M, u) (sampler.hpp:165-243)
//           and, for interior voxels, G = S * (N-1)/2 * dMw/dfrac (sampler.hpp:221-230).
//           Reads u 12 + M 4, writes Mw 4 + G 12 bytes per voxel.
//   pass 2  k_lncc_moments: the five window moments of (F, Mw) by separable box sums
//           (x, y running sums per plane in shared memory, z by fp64 telescoping over
//           the z march), ANTs dL/dMw (lncc.hpp:265-278) and g_u = G * dL/dMw.
//           Reads F 4 + Mw 4 + G 12, writes g_u 12 bytes per voxel; the x/y halo of F
//           and Mw comes from L2 (neighbouring tiles read the same planes).
//
// The single-pass kernel (step_lncc.cu) re-samples the warp for every halo position of a
// tile (1.9 samples per output voxel at 64 x 8 tiles) and carries the sampling latency
// and registers inside the moment pipeline; here each voxel is sampled once and both
// passes are simple streams, at 64 instead of 32 bytes per voxel of HBM traffic (the
// step is latency / instruction bound, not bandwidth bound).
#include <algorithm>

#include "ffdp_common.cuh"

#ifndef FFDP_L2_PREDLOAD
#define FFDP_L2_PREDLOAD 1
#endif

namespace ffdp {
namespace l2 {

constexpr int R = 3, WIN = 7;

// ------------------------------------------------------------------ pass 1
struct SParams {
    Geom g;
    const float* u;   // buffer planes [buf_z0, buf_z0 + buf_nz)
    float* mw;        // same planes: Mw - shift_m (0 where not sampled)
    float* gd;        // interior planes: 3 per voxel
    int32_t* miss;
    int32_t nx, ny, nxb, nyq;
    FastDiv div_nxb, div_nyq;
    int64_t plane, buf_z0, p0, z_begin, z_end, nunits;
    int64_t gd_skip;  // (z_begin - buf_z0) * plane: the halo planes G does not hold
    float sm;
};

// The unit of a warp: 32 consecutive x voxels (lane = x offset) of 4 consecutive rows of
// one plane; consecutive lanes gather neighbouring source positions (coalesced).
struct SUnit {
    int32_t x, y0, nrow;  // nrow: rows of the unit inside the lattice (0 for lanes past nx)
    int64_t p, bi;
};

__device__ __forceinline__ SUnit sunit(const SParams& P, int64_t unit, int lane) {
    SUnit w;
    const uint32_t r1 = fdiv((uint32_t)unit, P.div_nxb);
    w.x = (int32_t)((uint32_t)unit - r1 * P.nxb) * 32 + lane;
    const uint32_t zz = fdiv(r1, P.div_nyq);
    w.y0 = (int32_t)(r1 - zz * P.nyq) * 4;
    w.p = P.p0 + zz;
    const bool vx = w.x < P.nx;
    w.nrow = vx ? min(4, P.ny - w.y0) : 0;
    w.bi = (w.p - P.buf_z0) * P.plane + (int64_t)w.y0 * P.nx + (vx ? w.x : 0);
    return w;
}

// row k of the unit is 3 * nx floats of u after row k - 1: one 64-bit base per unit
__device__ __forceinline__ void sload(const SParams& P, const SUnit& w, float (&uu)[12]) {
    const float* q = P.u + 3 * w.bi;
    const int32_t rs = 3 * P.nx;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool ok = k < w.nrow;
        uu[3 * k] = ok ? __ldg(q + k * rs) : 0.0f;
        uu[3 * k + 1] = ok ? __ldg(q + k * rs + 1) : 0.0f;
        uu[3 * k + 2] = ok ? __ldg(q + k * rs + 2) : 0.0f;
    }
}

#ifndef FFDP_L2_SMINB
#define FFDP_L2_SMINB 3
#endif
#ifndef FFDP_L2_SPREF
#define FFDP_L2_SPREF 1
#endif
template <bool FULLWIN, bool OFF32>
__global__ void __launch_bounds__(256, FFDP_L2_SMINB) k_lncc_sample(const SParams P) {
    int miss = 0;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * 8;
    int64_t unit = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    SUnit w = sunit(P, unit < P.nunits ? unit : 0, lane);
    float uu[12];
    if (unit < P.nunits) sload(P, w, uu);
    for (; unit < P.nunits; unit += stride) {
        Cell c[4];
        RowBase rb;
        rb.init(P.g, w.x, w.y0, (int32_t)w.p);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k) rb.step_y(P.g);
            c[k] = rb.cell(P.g, uu[3 * k], uu[3 * k + 1], uu[3 * k + 2]);
        }
        Corners cr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) cr[k] = gather_pad<FULLWIN, OFF32>(P.g, c[k], miss);
        const SUnit cw = w;
        if (FFDP_L2_SPREF) {
            // the next unit's displacements are in flight while this unit's corners land
            const int64_t nu = unit + stride;
            if (nu < P.nunits) {
                w = sunit(P, nu, lane);
                sload(P, w, uu);
            }
        }
        const bool interior = cw.p >= P.z_begin && cw.p < P.z_end;
        float* mwp = P.mw + cw.bi;
        float* gdp = P.gd + 3 * (cw.bi - P.gd_skip);
        const int32_t rs = 3 * P.nx;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float d[3];
            const float v = interp_grad(cr[k], c[k], d);
            if (k < cw.nrow) {
                mwp[k * P.nx] = v - P.sm;
                if (interior) {
                    float* o = gdp + k * rs;
                    o[0] = P.g.dscale[0] * d[0];
                    o[1] = P.g.dscale[1] * d[1];
                    o[2] = P.g.dscale[2] * d[2];
                }
            }
        }
        if (!FFDP_L2_SPREF) {
            const int64_t nu = unit + stride;
            if (nu < P.nunits) {
                w = sunit(P, nu, lane);
                sload(P, w, uu);
            }
        }
    }
    const unsigned anym = __ballot_sync(0xffffffffu, miss);
    if (anym && P.miss && lane == 0) atomicAdd(P.miss, __popc(anym));
}

// ------------------------------------------------------------------ pass 2
struct MParams {
    const float* f;   // buffer planes
    const float* mw;  // buffer planes, shifted
    const float* gd;  // interior planes
    float* g_u;       // interior planes
    double* partial;  // one sum of n_i per CTA (summed in a fixed order afterwards)
    int32_t nx, ny;
    int64_t plane, buf_z0, nz_global, z_begin, z_end, s_lo, s_hi;  // [s_lo, s_hi): planes holding Mw
    int32_t zchunk;
    double eps, gi;
    float sf, sm;
};

template <int TX, int TY>
struct Tile {
    static constexpr int NT = TX * TY / 2;          // one vertical output pair per thread
    static constexpr int HX = TX + 2 * R, HY = TY + 2 * R;
    static constexpr int HXP = HX;                  // ring row pitch: position h = hy * HX + hx is element h
    static constexpr int NPOS = HX * HY;
    static constexpr int KPOS = (NPOS + NT - 1) / NT;  // positions per thread
    static constexpr int XJOBS = HY * (TX / 4);
    static constexpr int NSLOT = 8;
    struct Smem {
        float2 raw[NSLOT][HY][HXP];  // shifted (F, Mw), zero outside the volume
        float X[5][HY][TX];          // x box sums of the channel differences
    };
};

// in-lattice extent of the window of position g along an axis of n voxels (< 2^31)
__device__ __forceinline__ float win_count(int32_t g, int32_t n) {
    return (float)(min(g + R, n - 1) - max(g - R, 0) + 1);
}

template <int TX, int TY>
struct Pref2 {
    float2 v[Tile<TX, TY>::KPOS];  // raw (F, Mw - shift_m); F is shifted when it is stored
};

// In-plane offsets of the thread's haloed-tile positions (-1: outside the lattice or no
// position), fixed for the whole z march.
template <int TX, int TY>
__device__ __forceinline__ void plane_offsets(const MParams& P, int t, int x0, int y0,
                                              int32_t (&off)[Tile<TX, TY>::KPOS]) {
    using T = Tile<TX, TY>;
#pragma unroll
    for (int k = 0; k < T::KPOS; ++k) {
        const int h = t + T::NT * k;
        const int hy = h / T::HX, hx = h - hy * T::HX;
        const int gx = x0 + hx - R, gy = y0 + hy - R;
        off[k] = (h < T::NPOS && gx >= 0 && gx < P.nx && gy >= 0 && gy < P.ny) ? gy * P.nx + gx : -1;
    }
}

template <int TX, int TY>
__device__ __forceinline__ void load_plane(const MParams& P, const int32_t (&off)[Tile<TX, TY>::KPOS], int64_t p,
                                           Pref2<TX, TY>& pf) {
    using T = Tile<TX, TY>;
    const bool in = p >= P.s_lo && p < P.s_hi;  // planes outside [s_lo, s_hi) are outside the volume
    const int64_t zoff = in ? (p - P.buf_z0) * P.plane : 0;
    const float* fp = P.f + zoff;
    const float* mp = P.mw + zoff;
    // opaque plane bases: each load address is then one wide multiply-add of the offset
    asm("" : "+l"(fp), "+l"(mp));
#pragma unroll
    for (int k = 0; k < T::KPOS; ++k) {
        // off < 0 (outside the lattice): load a valid element and discard it, so the loads
        // need no predicate and no 64-bit select
#if FFDP_L2_PREDLOAD
        const bool ok = in && off[k] >= 0;
        const uint32_t o = (uint32_t)off[k];
        pf.v[k] = ok ? make_float2(__ldg(fp + o), __ldg(mp + o)) : make_float2(P.sf, 0.f);
#else
        const uint32_t o = (uint32_t)max(off[k], 0);
        const float a = __ldg(fp + o), b = __ldg(mp + o);
        const bool ok = in && off[k] >= 0;
        // consumed one plane later (register ping-pong): no arithmetic on the loaded values here
        pf.v[k] = ok ? make_float2(a, b) : make_float2(P.sf, 0.f);
#endif
    }
}

template <int TX, int TY, int SLOT>
__device__ __forceinline__ void mplane(const MParams& P, typename Tile<TX, TY>::Smem& sm, Pref2<TX, TY> (&pf)[2],
                                       const int32_t (&off)[Tile<TX, TY>::KPOS], const int32_t (&out_off)[2],
                                       const float (&cxy)[2], double (&Z)[2][5], float& nsum, int64_t p,
                                       int64_t pstart, int64_t pend, int64_t zc0) {
    using T = Tile<TX, TY>;
    if (p >= pend) return;  // uniform across the CTA
    const int t = threadIdx.x;
    const int slot = (int)((p - pstart) & (T::NSLOT - 1));
    const int slot_old = (slot + 1) & (T::NSLOT - 1);  // plane p-7
    // this plane's values arrived during the previous plane; start the next plane's loads
    {
        const Pref2<TX, TY>& cur = pf[SLOT & 1];
#pragma unroll
        for (int k = 0; k < T::KPOS; ++k) {
            const int h = t + T::NT * k;
            if (h < T::NPOS) (&sm.raw[slot][0][0])[h] = make_float2(cur.v[k].x - P.sf, cur.v[k].y);
        }
        if (p + 1 < pend) load_plane<TX, TY>(P, off, p + 1, pf[(SLOT + 1) & 1]);
    }
    // G of the outputs finished in this plane (plane p-3), in flight during the passes
    const bool emit = p >= zc0 + R;
    const int64_t q = p - R;
    const int ox = t % TX, oy0 = 2 * (t / TX);
    // the thread's two outputs of plane q: 3 * in-plane offset (out_off[j] < 0: outside)
    const int64_t qoff = 3 * (q - P.z_begin) * P.plane;
    float G[2][3];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const bool ok = emit && out_off[j] >= 0;
        const float* gp = P.gd + qoff + out_off[j];
#pragma unroll
        for (int a = 0; a < 3; ++a) G[j][a] = ok ? __ldg(gp + a) : 0.0f;
    }
    __syncthreads();

    // x box sums of v(p) - v(p-7), runs of 4, streamed over the 10 inputs of a run
    for (int job = t; job < T::XJOBS; job += T::NT) {
        const int r = job / (TX / 4), xs = (job % (TX / 4)) * 4;
        float acc[5], head[3][5], out[3][5];
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const float2 n = sm.raw[slot][r][xs + k], o = sm.raw[slot_old][r][xs + k];
            const float dv[5] = {n.x - o.x, n.y - o.y, fmaf(n.x, n.x, -o.x * o.x), fmaf(n.y, n.y, -o.y * o.y),
                                 fmaf(n.x, n.y, -o.x * o.y)};
#pragma unroll
            for (int ch = 0; ch < 5; ++ch) {
                if (k == 0) acc[ch] = dv[ch];
                else if (k < 7) acc[ch] += dv[ch];
                else { out[k - 7][ch] = acc[ch]; acc[ch] += dv[ch] - head[k - 7][ch]; }
                if (k < 3) head[k][ch] = dv[ch];
            }
        }
#pragma unroll
        for (int ch = 0; ch < 5; ++ch)
            *reinterpret_cast<float4*>(&sm.X[ch][r][xs]) = make_float4(out[0][ch], out[1][ch], out[2][ch], acc[ch]);
    }
    __syncthreads();

    // y box sums, Z += box (fp64 telescoping), finish plane p-3
    const int slot_q = (slot + T::NSLOT - R) & (T::NSLOT - 1);
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
        float s = sm.X[ch][oy0][ox];
#pragma unroll
        for (int k = 1; k < WIN; ++k) s += sm.X[ch][oy0 + k][ox];
        Z[0][ch] += (double)s;
        s += sm.X[ch][oy0 + WIN][ox] - sm.X[ch][oy0][ox];
        Z[1][ch] += (double)s;
    }
    const float cz = win_count((int32_t)q, (int32_t)P.nz_global);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int oy = oy0 + j;
        if (emit && out_off[j] >= 0) {
            const float2 fm = sm.raw[slot_q][oy + R][ox + R];
            const float cw = cxy[j] * cz;
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
                // zero-padded border: the shifted sums miss the shift of the (W < 1) window
                const double omw = 1.0 - W;
                A += N * (omw * (sf * Sm + smv * Sf) + sf * smv * N * (W - W * W));
                Bv += N * (omw * 2.0 * sf * Sf + sf * sf * N * (W - W * W));
                Cv += N * (omw * 2.0 * smv * Sm + smv * smv * N * (W - W * W));
            }
            const float a = (float)(A * (inv * inv)), b = (float)(Bv * (inv * inv)), cc = (float)(Cv * (inv * inv));
            const float D = fmaf(b, cc, (float)P.eps);
            const float invD = __fdividef(1.0f, D);  // D >= eps > 0; 2-ulp reciprocal
            nsum += a * a * invD;
            const float gamma = 2.0f * (float)P.gi * a * invD;
            const float rab = a * b * invD;
            const float mf = (float)(Sf * inv), mm = (float)(Sm * inv);
            const float omwf = (float)(1.0 - W);
            const float df = (fm.x - mf) + P.sf * omwf;    // F - mean_F
            const float dm = (fm.y - mm) + P.sm * omwf;    // Mw - mean_M
            const float gmw = gamma * fmaf(-dm, rab, df);  // dL/dMw (lncc.hpp:277, ANTs)
            float* o = P.g_u + qoff + out_off[j];
            o[0] = G[j][0] * gmw;
            o[1] = G[j][1] * gmw;
            o[2] = G[j][2] * gmw;
        }
    }
}

#ifndef FFDP_L2_MINB
#define FFDP_L2_MINB 2
#endif
template <int TX, int TY>
__global__ void __launch_bounds__(Tile<TX, TY>::NT, FFDP_L2_MINB) k_lncc_moments(const MParams P) {
    using T = Tile<TX, TY>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename T::Smem& sm = *reinterpret_cast<typename T::Smem*>(smem_raw);
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int64_t zc0 = P.z_begin + (int64_t)blockIdx.z * P.zchunk;
    const int64_t zc1 = min(P.z_end, zc0 + P.zchunk);
    if (zc0 >= zc1) return;
    for (int i = threadIdx.x; i < T::NSLOT * T::HY * T::HXP; i += T::NT) (&sm.raw[0][0][0])[i] = make_float2(0.f, 0.f);
    double Z[2][5];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) Z[j][ch] = 0.0;
    float nsum = 0.0f;  // this thread's sum of n_i: <= 2 zchunk terms of [0, 1]
    const int64_t pstart = zc0 - R, pend = zc1 + R;
    int32_t off[T::KPOS], out_off[2];
    float cxy[2];  // in-lattice x * y extent of the output's window (zero-padded border)
    plane_offsets<TX, TY>(P, threadIdx.x, x0, y0, off);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int gx = x0 + (int)threadIdx.x % TX, gy = y0 + 2 * ((int)threadIdx.x / TX) + j;
        out_off[j] = (gx < P.nx && gy < P.ny) ? 3 * (gy * P.nx + gx) : -1;
        cxy[j] = win_count(gx, P.nx) * win_count(gy, P.ny);
    }
    Pref2<TX, TY> pf[2];
    load_plane<TX, TY>(P, off, pstart, pf[0]);
    __syncthreads();
    for (int64_t p = pstart; p < pend; p += 2) {
        mplane<TX, TY, 0>(P, sm, pf, off, out_off, cxy, Z, nsum, p, pstart, pend, zc0);
        mplane<TX, TY, 1>(P, sm, pf, off, out_off, cxy, Z, nsum, p + 1, pstart, pend, zc0);
    }
    __shared__ double red[T::NT / 32];
    const double cta = block_sum<T::NT>((double)nsum, red);
    if (threadIdx.x == 0)
        P.partial[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = cta;
}

// *sum_n += the CTA partials, in a fixed order: the loss is bit-reproducible run to run.
__global__ void __launch_bounds__(256) k_add_partials(const double* partial, int64_t n, double* sum_n) {
    __shared__ double red[8];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 256) v += partial[i];
    v = block_sum<256>(v, red);
    if (threadIdx.x == 0) *sum_n += v;
}

// Planes per z chunk: the fewest (waves x planes-with-halo) over chunk counts.
inline int32_t pick_zchunk(int64_t tiles, int64_t nzs, int64_t capacity) {
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

}  // namespace l2

#ifndef FFDP_L2_TX
#define FFDP_L2_TX 32
#endif
#ifndef FFDP_L2_TY
#define FFDP_L2_TY 16
#endif

// CTA partial slots: at most tiles x min(planes, 256) chunks (pick_zchunk's range)
static int64_t lncc2_max_ctas(const ffdp_dims& d, const ffdp_slab& s) {
    const int64_t tx = (d.nx + FFDP_L2_TX - 1) / FFDP_L2_TX, ty = (d.ny + FFDP_L2_TY - 1) / FFDP_L2_TY;
    return tx * ty * std::min<int64_t>(std::max<int64_t>(1, s.z_end - s.z_begin), 256);
}

int64_t lncc2_workspace_bytes(const ffdp_dims& d, const ffdp_slab& s) {
    const int64_t plane = d.nx * d.ny;
    const int64_t fl = plane * d.nz + 3 * plane * (s.z_end - s.z_begin);
    return (int64_t)sizeof(float) * ((fl + 1) / 2 * 2) + (int64_t)sizeof(double) * lncc2_max_ctas(d, s);
}

// passes: 1 = warp sampling into the workspace, 2 = moments and g_u from it, 3 = both.
int lncc2_step(const float* f, const float* u, const ffdp_dims& d, const ffdp_slab& s, const ffdp_image_window& m,
               const ffdp_sampler_args& args, double eps, double gi, float shift_f, float shift_m, float* g_u,
               double* sum_n, int32_t* miss, void* workspace, int passes, cudaStream_t st) {
    using namespace l2;
    constexpr int TX = FFDP_L2_TX, TY = FFDP_L2_TY;
    using T = Tile<TX, TY>;
    const int64_t plane = d.nx * d.ny;
    float* mw = reinterpret_cast<float*>(workspace);
    float* gd = mw + plane * d.nz;
    // planes whose Mw the window needs: the interior and r halo planes inside the volume
    const int64_t s_lo = std::max<int64_t>(0, s.z_begin - R), s_hi = std::min<int64_t>(s.nz_global, s.z_end + R);

    SParams S;
    const ffdp_dims out{d.nx, d.ny, s.nz_global};
    S.g = make_geom(m, out, args);
    S.u = u;
    S.mw = mw;
    S.gd = gd;
    S.miss = miss;
    S.nx = (int32_t)d.nx;
    S.ny = (int32_t)d.ny;
    S.nxb = (int32_t)((d.nx + 31) / 32);
    S.nyq = (int32_t)((d.ny + 3) / 4);
    S.div_nxb = make_fastdiv((uint32_t)S.nxb);
    S.div_nyq = make_fastdiv((uint32_t)S.nyq);
    S.plane = plane;
    S.buf_z0 = s.buf_z0;
    S.p0 = s_lo;
    S.z_begin = s.z_begin;
    S.z_end = s.z_end;
    S.nunits = (int64_t)S.nxb * S.nyq * (s_hi - s_lo);
    S.gd_skip = (s.z_begin - s.buf_z0) * plane;
    S.sm = shift_m;
    const bool full = m.z_begin == 0 && m.z_end == m.dims.nz;
#ifndef FFDP_L2_SCTAS
#define FFDP_L2_SCTAS 3  // one wave (3 CTAs per SM): measured 2.64 -> 2.51 ms vs 16
#endif
    const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>((S.nunits + 7) / 8, (int64_t)FFDP_L2_SCTAS * num_sms()));
    if (passes & 1) {
        const bool o32 = window_off32(S.g);
        if (full && o32)
            k_lncc_sample<true, true><<<g1, 256, 0, st>>>(S);
        else if (full)
            k_lncc_sample<true, false><<<g1, 256, 0, st>>>(S);
        else if (o32)
            k_lncc_sample<false, true><<<g1, 256, 0, st>>>(S);
        else
            k_lncc_sample<false, false><<<g1, 256, 0, st>>>(S);
    }
    if (!(passes & 2)) return check_launch("step_lncc (warp sampling pass)");

    MParams M;
    M.f = f;
    M.mw = mw;
    M.gd = gd;
    M.g_u = g_u;
    const int64_t fl = plane * d.nz + 3 * plane * (s.z_end - s.z_begin);
    M.partial = reinterpret_cast<double*>(mw + (fl + 1) / 2 * 2);
    M.nx = (int32_t)d.nx;
    M.ny = (int32_t)d.ny;
    M.plane = plane;
    M.buf_z0 = s.buf_z0;
    M.nz_global = s.nz_global;
    M.z_begin = s.z_begin;
    M.z_end = s.z_end;
    M.s_lo = s_lo;
    M.s_hi = s_hi;
    M.eps = eps;
    M.gi = gi;
    M.sf = shift_f;
    M.sm = shift_m;
    static std::atomic<unsigned long long> attr_mask{0};
    static int per_sm = 1;
    once_per_device(attr_mask, [&] {
        cudaFuncSetAttribute(k_lncc_moments<TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(typename T::Smem));
        int p = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, k_lncc_moments<TX, TY>, T::NT, sizeof(typename T::Smem));
        per_sm = std::max(p, 1);
    });
    const int64_t tx = (d.nx + TX - 1) / TX, ty = (d.ny + TY - 1) / TY;
    const int64_t nzs = s.z_end - s.z_begin;
    M.zchunk = pick_zchunk(tx * ty, nzs, (int64_t)per_sm * num_sms());
    const int64_t chunks = (nzs + M.zchunk - 1) / M.zchunk;
    if (ty > 65535 || chunks > 65535) return set_error(FFDP_INVALID_ARGUMENT, "step_lncc: grid too large");
    const dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)chunks);
    k_lncc_moments<TX, TY><<<grid, T::NT, sizeof(typename T::Smem), st>>>(M);
    if (sum_n) k_add_partials<<<1, 256, 0, st>>>(M.partial, tx * ty * chunks, sum_n);
    return check_launch("step_lncc (two-pass)");
}

}  // namespace ffdp
