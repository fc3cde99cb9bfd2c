// stkde_tile_ws.cu -- the short-window FP32 engine of the PB-SYM tile kernel
// (STKDE_ENGINE_WS): for temporal windows of at most 17 layers (H_t <= 8).
//
// One work item = one 16 x 16 column x 32 layer tile (or one chunk of a hot tile's candidate
// list).  Each of the CTA's 128 threads owns two columns (x, y) and (x, y + 4) of one warp's
// 8 x 8 column patch and their 32 layers as 32 packed FP32x2 accumulators.  Per accepted point
// p (Alg. 3) a thread forms its two spatial weights
//     s_c = [c in the exact disc] a_x(x_c) a_y(y_c)      (printed kernel)
// and adds s_c K_t[p](t) to the layers of p's temporal window [T_p - H_t, T_p + H_t] only:
// the window's offset in the tile is warp-uniform (every lane works on the same point), so a
// switch on it selects a fully unrolled case whose accumulator indices are compile-time
// constants -- W = 2 H_t + 1 packed FMAs per point and column pair instead of 32, with no
// local-memory indexing.  The tcgen05 engine forms the same sums as a dense contraction whose
// k-blocks cost the same for a 15-layer window as for a 65-layer one; here the work follows
// the window.
//
// Per item: the tile's home-bucket segments (the same binning as the tcgen05 engine: 16 x 16
// x BTH buckets, records in input order per bucket from the stable radix sort), 128 candidates
// per round, one per thread: cull by window and disc-rectangle distance, order-preserving
// compaction into a batch, and the accepted thread writes its point's tables (a_x for the 16
// tile columns, a_y for the 16 rows, the exact disc chords of the 16 rows as column bit masks
// from the chord table, the K_t window, the warps whose patch the disc meets).  Every voxel
// sums its contributions in candidate order (segments in key order, points in input order),
// so results are deterministic and slabs of either kind are bitwise equal to the full grid.
// Epilogue: the 256 x 32 accumulators staged in shared memory and stored warp-coalesced
// (lane = layer, any G_t alignment), every voxel exactly once; split hot tiles add their FP32
// partials in chunk order (the last chunk to arrive stores).
#include "stkde_internal.cuh"

namespace stkde {

namespace wscfg {
constexpr int NTHR = 128;          // 4 warps, 2 columns per thread
constexpr int BT = 32;             // layers per tile (accumulators per column)
constexpr int NB = 128;            // batch: points per round (one candidate per thread)
constexpr int SROW = BT + 1;       // staging row stride (floats)
}  // namespace wscfg

template <int W>
struct WsCfg {
    static constexpr int KP = (W + 3) / 4 * 4;                    // K_t window, padded
    static constexpr size_t OFF_HDR = 0;                          // [NB] int2 {offset, warp mask}
    static constexpr size_t OFF_AX = OFF_HDR + wscfg::NB * 8;     // [NB][16] a_x
    static constexpr size_t OFF_AY = OFF_AX + wscfg::NB * 64;     // [NB][8] float2 (a_y(r), a_y(r + 4))
    static constexpr size_t OFF_MK = OFF_AY + wscfg::NB * 64;     // [NB][8] u32 chord masks of rows r, r + 4
    static constexpr size_t OFF_KV = OFF_MK + wscfg::NB * 32;     // [NB][KP] K_t window
    static constexpr size_t SZ_BATCH = OFF_KV + (size_t)wscfg::NB * KP * 4;
    static constexpr size_t SZ_STG = (size_t)256 * wscfg::SROW * 4;   // epilogue staging (aliases the batch)
    static constexpr size_t OFF_SEG = ((SZ_BATCH > SZ_STG ? SZ_BATCH : SZ_STG) + 15) / 16 * 16;
    static constexpr size_t OFF_MISC = OFF_SEG + (size_t)(2 * MAXSEG + 1) * 4;
    static constexpr size_t BYTES = OFF_MISC + 16 * 4;
};

// acc[t] += s * K[j] for the layers t = O + j of the tile, O = the window's first layer
// (a compile-time constant in each switch case)
template <int W, int O, int KP>
__device__ __forceinline__ void win_fma(float2 (&acc)[wscfg::BT], float2 s, const float (&kv)[KP]) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int t = O + j;
        if (t >= 0 && t < wscfg::BT) acc[t] = __ffma2_rn(s, make_float2(kv[j], kv[j]), acc[t]);
    }
}

template <int W, int KK>
__global__ void __launch_bounds__(wscfg::NTHR, 4)
k_tile_ws(const GridParams g, const PointRec *__restrict__ recs, const uint16_t *__restrict__ chords,
          const uint32_t *__restrict__ bucket_begin, const int4 *__restrict__ items,
          const uint64_t *__restrict__ nitems_ptr, int *__restrict__ work_counter, uint32_t *__restrict__ arrive,
          float *__restrict__ partials, const int chunk, const int c0, const float cscale,
          float *__restrict__ out, const int64_t t_begin, const int64_t t_end) {
    using namespace wscfg;
    using C = WsCfg<W>;
    constexpr int KP = C::KP;
    constexpr int HT = (W - 1) / 2;
    extern __shared__ __align__(16) unsigned char smem[];
    int2 *s_hdr = reinterpret_cast<int2 *>(smem + C::OFF_HDR);
    float *s_ax = reinterpret_cast<float *>(smem + C::OFF_AX);
    float2 *s_ay = reinterpret_cast<float2 *>(smem + C::OFF_AY);
    uint32_t *s_mk = reinterpret_cast<uint32_t *>(smem + C::OFF_MK);
    float *s_kv = reinterpret_cast<float *>(smem + C::OFF_KV);
    float *stg = reinterpret_cast<float *>(smem);
    int *seg_start = reinterpret_cast<int *>(smem + C::OFF_SEG);
    int *seg_pref = seg_start + MAXSEG;
    int *misc = reinterpret_cast<int *>(smem + C::OFF_MISC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // my columns: warp patch (px0, py0) = (8 (warp & 1), 8 (warp >> 1)); x = px0 + lane % 8,
    // rows y = py0 + lane / 8 and y + 4
    const int xl = 8 * (warp & 1) + (lane & 7);
    const int rk = 4 * (warp >> 1) + (lane >> 3);          // row-pair index: rows r, r + 4
    const uint32_t bitA = 1u << xl, bitB = 1u << (xl + 16);
    const uint32_t nitems = (uint32_t)(*nitems_ptr);
    const int Ts = (int)(t_end - t_begin);
    const int R8 = chord_rows(g.Hs);

    for (;;) {
        if (tid == 0) misc[0] = atomicAdd(work_counter, 1);
        __syncthreads();
        const uint32_t it = (uint32_t)misc[0];
        if (it >= nitems) break;
        const int4 item = items[it];
        const int ls = item.x, jchunk = item.y, nch = item.z;
        const int ta = ls % g.NXA + g.XA0, tb = (ls / g.NXA) % g.NTY, tc = ls / (g.NXA * g.NTY) + c0;
        const int tX0 = ta * BX, tY0 = tb * 16, tT0 = tc * BT;
        const int xn = min(BX, g.Gx - tX0), yn = min(16, g.Gy - tY0);
        const int gt1 = min(BT, g.Gt - tT0);                 // grid layers of the tile [0, gt1)

        // ---- home-bucket segments of this tile (key order) ----
        const int a0 = max(ta - g.Ra, 0), a1 = min(ta + g.Ra, g.NTX - 1);
        const int b0 = max(tb - g.Ray, 0), b1 = min(tb + g.Ray, g.NTY - 1);
        int cc0, cc1;
        home_t_range(g, tc, &cc0, &cc1);
        const int nbk = b1 - b0 + 1, nseg = nbk * (cc1 - cc0 + 1);
        if (warp == 0) {                                     // lengths + warp-shuffle prefix
            int carry = 0;
            for (int k0 = 0; k0 < nseg; k0 += 32) {
                const int k = k0 + lane;
                int len = 0;
                if (k < nseg) {
                    const int bb = b0 + k % nbk, cc = cc0 + k / nbk;
                    const int key = (cc * g.NTY + bb) * g.NTX;
                    const uint32_t s = bucket_begin[key + a0], e = bucket_begin[key + a1 + 1];
                    seg_start[k] = (int)s;
                    len = (int)(e - s);
                }
                int v = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                if (k < nseg) seg_pref[k + 1] = carry + v;
                carry += __shfl_sync(0xffffffffu, v, 31);
            }
            if (lane == 0) seg_pref[0] = 0;
        }
        __syncthreads();
        const int total = seg_pref[nseg];
        const int cbeg = jchunk * chunk, cend = min(total, cbeg + chunk);

        float2 acc[BT];
#pragma unroll
        for (int t = 0; t < BT; ++t) acc[t] = make_float2(0.f, 0.f);

        // tile-local column coordinates: column c's centre is at c + 0.5 from the tile origin
        const float xmax = (float)(xn - 1), ymax = (float)(yn - 1);
        const int Tlo = tT0, Thi = tT0 + gt1 - 1;
        for (int cb = cbeg; cb < cend; cb += NB) {
            // ---- (1) one candidate per thread: locate, load, cull ----
            const int i = cb + tid;
            bool ok = false;
            int wmask = 0;
            PointRec r;
            int ridx = 0;
            float px = 0.f, py = 0.f;
            if (i < cend) {
                int lo = 0, hi = nseg - 1;                   // last segment with seg_pref[k] <= i
                while (lo < hi) {
                    const int m = (lo + hi + 1) >> 1;
                    if (seg_pref[m] <= i) lo = m; else hi = m - 1;
                }
                ridx = seg_start[lo] + (i - seg_pref[lo]);
                r = recs[ridx];
                if (r.T + g.Ht >= Tlo && r.T - g.Ht <= Thi) {
                    px = (float)(r.X - tX0) + r.fx - 0.5f;
                    py = (float)(r.Y - tY0) + r.fy - 0.5f;
                    const float lim = g.rs2 * (1.0f + CULL_BAND) + 1e-6f;
#pragma unroll
                    for (int w = 0; w < 4; ++w) {            // the warp patches the disc can reach
                        const float x0 = (float)(8 * (w & 1)), y0 = (float)(8 * (w >> 1));
                        const float dx = fminf(fmaxf(px, x0), fminf(x0 + 7.f, xmax)) - px;
                        const float dy = fminf(fmaxf(py, y0), fminf(y0 + 7.f, ymax)) - py;
                        if (dx * dx + dy * dy < lim) wmask |= 1 << w;
                    }
                    ok = wmask != 0;
                }
            }
            // ---- (2) order-preserving compaction ----
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (lane == 0) misc[4 + warp] = __popc(bal);
            __syncthreads();
            int base = 0, m = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int cw = misc[4 + w];
                base += (w < warp) ? cw : 0;
                m += cw;
            }
            // ---- (3) the accepted thread writes its point's tables ----
            if (ok) {
                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                s_hdr[pos] = make_int2(r.T - HT - tT0, wmask);
                float *ax = s_ax + pos * 16;
#pragma unroll
                for (int c = 0; c < 16; c += 4) {
                    float v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float u = fabsf((float)(c + k) - px) * g.inv_rs;
                        if (KK == STKDE_KERNEL_PRINTED) { const float a = fmaxf(1.0f - u, 0.f); v[k] = a * a; }
                        else v[k] = u * u;
                    }
                    *reinterpret_cast<float4 *>(ax + c) = make_float4(v[0], v[1], v[2], v[3]);
                }
                float ayv[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float v = fabsf((float)c - py) * g.inv_rs;
                    if (KK == STKDE_KERNEL_PRINTED) { const float a = fmaxf(1.0f - v, 0.f); ayv[c] = a * a; }
                    else ayv[c] = 1.0f - v * v;
                }
                float2 *ay = s_ay + pos * 8;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int rr = 8 * (q >> 2) + (q & 3);
                    ay[q] = make_float2(ayv[rr], ayv[rr + 4]);
                }
                // exact disc chords of the tile's 16 rows -> 16-bit column masks (chord table:
                // entries for rows Y0(i) + e, Y0(i) = floor8(Y_i - H_s), int8 (lo, hi) - X_i)
                const int Y0 = (r.Y - g.Hs) & ~7;
                const int e0 = tY0 - Y0;                     // a multiple of 8
                uint32_t rm[16];
#pragma unroll
                for (int hb = 0; hb < 2; ++hb) {
                    const int eb = e0 + 8 * hb;
                    uint4 blk = make_uint4(0x0001u * 0x10001u, 0x0001u * 0x10001u, 0x0001u * 0x10001u,
                                           0x0001u * 0x10001u);   // (1, 0): empty rows
                    if (eb >= 0 && eb < R8)
                        blk = *reinterpret_cast<const uint4 *>(chords + (size_t)ridx * R8 + eb);
                    const uint32_t wds[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t ent = (wds[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
                        const int clo = r.X + (int)(int8_t)(ent & 0xFF) - tX0;
                        const int chi = r.X + (int)(int8_t)(ent >> 8) - tX0;
                        const int l = max(clo, 0), h = min(chi, 15);
                        rm[8 * hb + k] = (l <= h) ? (((2u << h) - 1u) & ~((1u << l) - 1u)) : 0u;
                    }
                }
                uint32_t *mk = s_mk + pos * 8;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int rr = 8 * (q >> 2) + (q & 3);
                    mk[q] = rm[rr] | (rm[rr + 4] << 16);
                }
                // K_t over the window layers T_i - H_t + j (inclusive gate, value 0 at |w| = 1)
                float *kv = s_kv + pos * KP;
#pragma unroll
                for (int j = 0; j < KP; ++j) {
                    float v = 0.f;
                    if (j < W) {
                        const float w = fabsf((float)(j - HT) + 0.5f - r.ft) * g.inv_rt;
                        if (KK == STKDE_KERNEL_PRINTED) { const float a = fmaxf(1.0f - w, 0.f); v = 0.75f * (a * a); }
                        else v = 0.75f * fmaxf(1.0f - w * w, 0.f);
                    }
                    kv[j] = v;
                }
            }
            __syncthreads();
            // ---- (4) accumulate: my two columns, the point's window only ----
#pragma unroll 1
            for (int p = 0; p < m; ++p) {
                const int2 h = s_hdr[p];
                if (!((h.y >> warp) & 1)) continue;          // disc misses my warp's patch
                const float ax = s_ax[p * 16 + xl];
                const float2 ay = s_ay[p * 8 + rk];
                const uint32_t mw = s_mk[p * 8 + rk];
                float2 s;
                if (KK == STKDE_KERNEL_PRINTED) {
                    s = __fmul2_rn(make_float2(ax, ax), ay);
                } else {                                     // 1 - u^2 - v^2, clamped at 0
                    s = make_float2(fmaxf(ay.x - ax, 0.f), fmaxf(ay.y - ax, 0.f));
                }
                s.x = (mw & bitA) ? s.x : 0.f;
                s.y = (mw & bitB) ? s.y : 0.f;
                float kv[KP];
#pragma unroll
                for (int q = 0; q < KP; q += 4) {
                    const float4 k4 = *reinterpret_cast<const float4 *>(s_kv + p * KP + q);
                    kv[q] = k4.x; kv[q + 1] = k4.y; kv[q + 2] = k4.z; kv[q + 3] = k4.w;
                }
                switch (h.x + (W - 1)) {                     // window start + W - 1 in [0, BT + W - 2]
#define WS_CASE(c) \
    case c:        \
        if ((c) <= BT + W - 2) win_fma<W, (c) - (W - 1), KP>(acc, s, kv); break;
                    WS_CASE(0) WS_CASE(1) WS_CASE(2) WS_CASE(3) WS_CASE(4) WS_CASE(5) WS_CASE(6) WS_CASE(7)
                    WS_CASE(8) WS_CASE(9) WS_CASE(10) WS_CASE(11) WS_CASE(12) WS_CASE(13) WS_CASE(14) WS_CASE(15)
                    WS_CASE(16) WS_CASE(17) WS_CASE(18) WS_CASE(19) WS_CASE(20) WS_CASE(21) WS_CASE(22) WS_CASE(23)
                    WS_CASE(24) WS_CASE(25) WS_CASE(26) WS_CASE(27) WS_CASE(28) WS_CASE(29) WS_CASE(30) WS_CASE(31)
                    WS_CASE(32) WS_CASE(33) WS_CASE(34) WS_CASE(35) WS_CASE(36) WS_CASE(37) WS_CASE(38) WS_CASE(39)
                    WS_CASE(40) WS_CASE(41) WS_CASE(42) WS_CASE(43) WS_CASE(44) WS_CASE(45) WS_CASE(46) WS_CASE(47)
#undef WS_CASE
                    default: break;
                }
            }
            __syncthreads();                                 // the batch is rewritten next round
        }

        // ---- epilogue: stage [column][layer], store warp-coalesced (lane = layer) ----
        // staging column sc = 64 warp + 32 half + lane (conflict-free writes)
        {
            float *sA = stg + (size_t)(64 * warp + lane) * SROW, *sB = sA + 32 * SROW;
#pragma unroll
            for (int t = 0; t < BT; ++t) {
                sA[t] = acc[t].x;
                sB[t] = acc[t].y;
            }
        }
        __syncthreads();
        // staging column sc -> tile column: warp w = sc / 64, half = (sc / 32) & 1, lane l = sc % 32:
        // x = 8 (w & 1) + l % 8, y = 8 (w >> 1) + l / 8 + 4 half
        auto col_of = [&](int sc, int &x, int &y) {
            const int w = sc >> 6, hf = (sc >> 5) & 1, l = sc & 31;
            x = 8 * (w & 1) + (l & 7);
            y = 8 * (w >> 1) + (l >> 3) + 4 * hf;
        };
        const int T = tT0 + lane;
        const bool t_ok = T >= t_begin && T < t_end && T < g.Gt;
        if (nch == 1) {
#pragma unroll 4
            for (int k = 0; k < 64; ++k) {
                const int sc = 64 * warp + k;
                int x, y;
                col_of(sc, x, y);
                if (t_ok && x < xn && y < yn)
                    out[((int64_t)(tX0 + x) * g.Gy + (tY0 + y)) * Ts + (T - t_begin)] = stg[sc * SROW + lane] * cscale;
            }
        } else {
            const int slot0 = item.w;
            float *mine = partials + (size_t)(slot0 + jchunk) * 256 * BT;
#pragma unroll 4
            for (int k = 0; k < 64; ++k) {
                const int sc = 64 * warp + k;
                mine[sc * BT + lane] = stg[sc * SROW + lane];
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const unsigned old = atomicAdd(&arrive[ls], 1u);
                misc[1] = (old == (unsigned)(nch - 1));
            }
            __syncthreads();
            if (misc[1]) {
                __threadfence();
                const float *pp = partials + (size_t)slot0 * 256 * BT + lane;
                for (int k = 0; k < 64; ++k) {
                    const int sc = 64 * warp + k;
                    const float *pk = pp + sc * BT;
                    // chunk order kept (deterministic); loads issued 8 at a time
                    float v = pk[0];
                    int j = 1;
                    for (; j + 8 <= nch; j += 8) {
                        float u[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) u[q] = pk[(size_t)(j + q) * 256 * BT];
#pragma unroll
                        for (int q = 0; q < 8; ++q) v += u[q];
                    }
                    for (; j < nch; ++j) v += pk[(size_t)j * 256 * BT];
                    int x, y;
                    col_of(sc, x, y);
                    if (t_ok && x < xn && y < yn)
                        out[((int64_t)(tX0 + x) * g.Gy + (tY0 + y)) * Ts + (T - t_begin)] = v * cscale;
                }
                if (tid == 0) arrive[ls] = 0u;
            }
        }
        __syncthreads();                                     // staging / misc reused by the next item
    }
}

// ------------------------------------------------------------ dispatch ---
typedef void (*ws_fn)(const GridParams, const PointRec *, const uint16_t *, const uint32_t *, const int4 *,
                      const uint64_t *, int *, uint32_t *, float *, int, int, float, float *, int64_t, int64_t);

// windows W = 2 H_t + 1, H_t = 1 .. 8
#define STKDE_WS_W(X) X(3) X(5) X(7) X(9) X(11) X(13) X(15) X(17)

static ws_fn ws_select(int W, int KK) {
#define STKDE_WSEL(w) \
    if (W == w) return KK ? (ws_fn)k_tile_ws<w, 1> : (ws_fn)k_tile_ws<w, 0>;
    STKDE_WS_W(STKDE_WSEL)
#undef STKDE_WSEL
    return nullptr;
}

static size_t ws_bytes(int W) {
#define STKDE_WSZ(w) \
    if (W == w) return WsCfg<w>::BYTES;
    STKDE_WS_W(STKDE_WSZ)
#undef STKDE_WSZ
    return 0;
}

size_t tile_ws_smem_bytes(int Ht) { return (Ht >= 1 && Ht <= 8) ? ws_bytes(2 * Ht + 1) : 0; }

// (every window up to the plan's gets the plan's shared-memory size: a sweep's narrower
// bandwidths launch the narrower instantiations with it)
int tile_ws_occupancy(int Ht, int KK, size_t smem, int *ctas_per_sm) {
    ws_fn f = ws_select(2 * Ht + 1, KK);
    if (!f) return STKDE_EINVAL;
    for (int h = 1; h <= Ht; ++h)
        if (cudaFuncSetAttribute(ws_select(2 * h + 1, KK), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return STKDE_ECUDA;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, wscfg::NTHR, smem) != cudaSuccess) return STKDE_ECUDA;
    *ctas_per_sm = occ;
    return STKDE_OK;
}

int launch_tile_ws(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cscale, float *out,
                   cudaStream_t st) {
    const GridParams &g = p->g;
    ws_fn f = ws_select(2 * g.Ht + 1, p->kernel);
    if (!f || g.BT != wscfg::BT || g.BY != 16) return STKDE_EINVAL;
    const int nsl = g.NXA * g.NTY * (c1 - c0);
    unsigned grid = (unsigned)std::min<int64_t>((int64_t)p->num_sms * p->ctas_per_sm, p->max_items);
    if (!p->wc_zeroed) cudaMemsetAsync(p->counters, 0, sizeof(int), st);   // (else by k_worklist_small)
    p->wc_zeroed = 0;
    const bool timed = p->timing && p->tev_used < p->tev_cap;
    if (timed) cudaEventRecord(p->tev[2 * p->tev_used], st);
    f<<<grid, wscfg::NTHR, p->smem_bytes, st>>>(g, p->rec_sorted, p->chords, p->bucket_begin, p->items,
                                                p->chunk_off + nsl, p->counters, p->arrive, p->partials, p->chunk,
                                                c0, cscale, out, t_begin, t_end);
    if (timed) {
        cudaEventRecord(p->tev[2 * p->tev_used + 1], st);
        p->tev_used += 1;
    }
    p->last_own_launches += 1;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

}  // namespace stkde
