// stkde_tile.cu -- the gather-form PB-SYM tile kernel (the hot loop).
//
// One work item = one Bx x By x Bt voxel tile (or one chunk of a hot tile's
// candidate list).  The CTA
//   1. walks the tile's home-bucket segments (candidates in a fixed order),
//      keeps the points whose cylinder can touch the tile and stages them in
//      a shared-memory ring;
//   2. per sub-batch of P points builds, in shared memory, the per-point
//      invariants of Alg. 3 restricted to the tile:
//        K_t[t]          the temporal line (Bt values, 0 outside the window),
//        a_x[x], a_y[y]  the separable factors of k_s, with the normalisation
//                        1/(n hs^2 ht) folded into a_y (as Alg. 3 folds it
//                        into K_s),
//        mask[y]         the exact disc chord of row y (16 bits);
//   3. each thread owns 4 columns (x0..x0+3 of one row y) x CT layers and
//      accumulates
//        acc[c][t] += s_c * K_t[t],   s_c = mask ? a_x * a_y : 0
//      (Alg. 3's stkde += K_s K_t) in FP32 registers with
//      packed FFMA2 (one broadcast LDS.128 of K_t feeds 8 FFMA2); a warp
//      (8 rows x 16 columns x CT layers) skips points whose window misses its
//      layers or whose disc misses its rows; after every sub-batch the
//      registers are added into a shared-memory tile accumulator (two-level
//      summation);
//   4. writes every voxel of the tile exactly once (no memset, no atomics on
//      the grid) with coalesced float4 stores; a split hot tile writes its
//      partial and the last chunk to arrive sums the partials in chunk order.
#include "stkde_internal.cuh"

namespace stkde {

template <int BT, int CT>
struct Cfg {
    // Thread tile: 4 consecutive x of one row y, CT consecutive layers.
    // Warp w: rows [8*(w&1), +8), layer group lg = w>>1 (CT layers).
    static constexpr int NTHR = 64 * (BT / CT);
    static constexpr int NWARP = NTHR / 32;
    static constexpr int P = 32;                 // points per sub-batch
    static constexpr int CAP = P + NTHR;         // staging ring (records)
    static constexpr int BT4 = BT / 4;
    static constexpr int CT4 = CT / 4;
    static constexpr int OSTR = BT4 + 1;         // padded accumulator row (float4)
    // shared-memory carve (bytes)
    static constexpr size_t OFF_OUTER = 0;
    static constexpr size_t SZ_OUTER = 256ull * OSTR * 16;
    static constexpr size_t OFF_KT = OFF_OUTER + SZ_OUTER;
    static constexpr size_t SZ_KT = (size_t)P * BT4 * 16;
    static constexpr size_t OFF_AX = OFF_KT + SZ_KT;
    static constexpr size_t SZ_AX = (size_t)P * 16 * 4;
    static constexpr size_t OFF_RING = OFF_AX + SZ_AX;
    static constexpr size_t SZ_RING = (size_t)CAP * sizeof(PointRec);
    static constexpr size_t OFF_ROW = OFF_RING + SZ_RING;
    static constexpr size_t SZ_ROW = (size_t)P * 16 * 8;
    static constexpr size_t OFF_META = OFF_ROW + SZ_ROW;
    static constexpr size_t SZ_META = (size_t)P * 4;
    static constexpr size_t OFF_SEG = OFF_META + SZ_META;
    static constexpr size_t SZ_SEG = (size_t)(2 * MAXSEG + 1) * 4;
    static constexpr size_t OFF_MISC = OFF_SEG + SZ_SEG;
    static constexpr size_t SZ_MISC = 64 * 4;
    static constexpr size_t BYTES = OFF_MISC + SZ_MISC;
};

__device__ __forceinline__ float2 ffma2(float2 a, float s, float2 c) {
    return __ffma2_rn(a, make_float2(s, s), c);
}

template <int BT, int CT, int KK>
__global__ void __launch_bounds__(Cfg<BT, CT>::NTHR, 512 / Cfg<BT, CT>::NTHR)
k_tile(const GridParams g, const PointRec *__restrict__ recs, const uint32_t *__restrict__ bucket_begin,
       const int4 *__restrict__ items, const uint64_t *__restrict__ nitems_ptr, int *__restrict__ work_counter,
       uint32_t *__restrict__ arrive, float4 *__restrict__ partials, const int chunk, const int c0,
       const float cnorm, float *__restrict__ out, const int64_t t_begin, const int64_t t_end, const int vec_ok) {
    using K = Cfg<BT, CT>;
    extern __shared__ __align__(16) unsigned char smem[];
    float4 *outer = reinterpret_cast<float4 *>(smem + K::OFF_OUTER);
    float4 *kt4 = reinterpret_cast<float4 *>(smem + K::OFF_KT);
    float4 *ax4 = reinterpret_cast<float4 *>(smem + K::OFF_AX);
    float *axt = reinterpret_cast<float *>(smem + K::OFF_AX);
    PointRec *ring = reinterpret_cast<PointRec *>(smem + K::OFF_RING);
    float2 *rowt = reinterpret_cast<float2 *>(smem + K::OFF_ROW);
    int *meta = reinterpret_cast<int *>(smem + K::OFF_META);
    int *seg_start = reinterpret_cast<int *>(smem + K::OFF_SEG);
    int *seg_pref = seg_start + MAXSEG;
    int *misc = reinterpret_cast<int *>(smem + K::OFF_MISC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int my_y = 8 * (warp & 1) + (lane & 7);   // row of the thread's 4 columns
    const int my_xg = lane >> 3;                     // x group: columns 4*my_xg .. +3
    const int my_lg = warp >> 1;                     // layer group: layers CT*my_lg .. +CT-1
    const uint32_t nitems = (uint32_t)(*nitems_ptr);
    const int Ts = (int)(t_end - t_begin);

    for (;;) {
        if (tid == 0) misc[0] = atomicAdd(work_counter, 1);
        __syncthreads();
        const uint32_t it = (uint32_t)misc[0];
        if (it >= nitems) break;
        const int4 item = items[it];
        const int ls = item.x, jchunk = item.y, nch = item.z;
        const int ta = ls % g.NTX, tb = (ls / g.NTX) % g.NTY, tc = ls / (g.NTX * g.NTY) + c0;
        const int tX0 = ta * BX, tY0 = tb * BYW, tT0 = tc * BT;
        // stored layers of this tile, tile-local [lt0, lt1)
        const int lt0 = max(0, (int)(t_begin - tT0));
        const int lt1 = min(BT, (int)min((int64_t)g.Gt, t_end) - tT0);
        const int xn = min(BX, g.Gx - tX0), yn = min(BYW, g.Gy - tY0);
        const int gt1 = min(BT, g.Gt - tT0);         // grid layers of the tile [0, gt1)

        // ---- home-bucket segments of this tile ----
        const int a0 = max(ta - g.Ra, 0), a1 = min(ta + g.Ra, g.NTX - 1);
        const int b0 = max(tb - g.Ray, 0), b1 = min(tb + g.Ray, g.NTY - 1);
        int cc0, cc1;
        home_t_range(g, tc, &cc0, &cc1);
        const int nb = b1 - b0 + 1, nseg = nb * (cc1 - cc0 + 1);
        for (int k = tid; k < nseg; k += K::NTHR) {
            int bb = b0 + k % nb, cc = cc0 + k / nb;
            int key = (cc * g.NTY + bb) * g.NTX;
            uint32_t s = bucket_begin[key + a0], e = bucket_begin[key + a1 + 1];
            seg_start[k] = (int)s;
            seg_pref[k + 1] = (int)(e - s);
        }
        for (int q = tid; q < 256 * K::OSTR; q += K::NTHR) outer[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            seg_pref[0] = 0;
            for (int k = 0; k < nseg; ++k) { acc += seg_pref[k + 1]; seg_pref[k + 1] = acc; }
        }
        __syncthreads();
        const int total = seg_pref[nseg];
        const int cbeg = jchunk * chunk, cend = min(total, cbeg + chunk);

        // Acceptance uses the tile's grid layers (not the slab), so a slab run
        // accepts exactly the points of the full run: bitwise equal layers.
        const float xmax = (float)(xn - 1), ymax = (float)(yn - 1);
        const int Tlo = tT0, Thi = tT0 + gt1 - 1;

        int head = 0, tail = 0;
        for (int cb = cbeg; cb < cend; cb += K::NTHR) {
            const int i = cb + tid;
            bool acc = false;
            PointRec r;
            if (i < cend) {
                int lo = 0, hi = nseg - 1;          // last segment with seg_pref[k] <= i
                while (lo < hi) {
                    int m = (lo + hi + 1) >> 1;
                    if (seg_pref[m] <= i) lo = m; else hi = m - 1;
                }
                r = recs[seg_start[lo] + (i - seg_pref[lo])];
                if (r.T + g.Ht >= Tlo && r.T - g.Ht <= Thi) {
                    float px = (float)(r.X - tX0) + r.fx - 0.5f;
                    float py = (float)(r.Y - tY0) + r.fy - 0.5f;
                    float dx = fminf(fmaxf(px, 0.f), xmax) - px;
                    float dy = fminf(fmaxf(py, 0.f), ymax) - py;
                    acc = dx * dx + dy * dy < g.rs2 * (1.0f + CULL_BAND) + 1e-6f;
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, acc);
            if (lane == 0) misc[8 + warp] = __popc(bal);
            __syncthreads();
            int base = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < K::NWARP; ++w) {
                int cw = misc[8 + w];
                base += (w < warp) ? cw : 0;
                tot += cw;
            }
            if (acc) {
                int pos = tail + base + __popc(bal & ((1u << lane) - 1u));
                ring[pos % K::CAP] = r;
            }
            tail += tot;
            __syncthreads();
            while (tail - head >= K::P || (cb + K::NTHR >= cend && tail > head)) {
                const int np = min(K::P, tail - head);
                // ---------------- per-point invariants (Alg. 3) ----------------
                for (int e = tid; e < np * K::BT4; e += K::NTHR) {      // K_t line
                    const int p = e / K::BT4, q = e - p * K::BT4;
                    const PointRec &pr = ring[(head + p) % K::CAP];
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float dtv = (float)(tT0 + 4 * q + j - pr.T) + 0.5f - pr.ft;
                        float w = fabsf(dtv) * g.inv_rt;
                        float kv;
                        if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - w; kv = 0.75f * (a * a); }
                        else kv = 0.75f * (1.0f - w * w);
                        v[j] = (w <= 1.0f) ? kv : 0.0f;
                    }
                    kt4[p * K::BT4 + q] = make_float4(v[0], v[1], v[2], v[3]);
                }
                for (int e = tid; e < np * 16; e += K::NTHR) {           // a_x
                    const int p = e >> 4, xx = e & 15;
                    const PointRec &pr = ring[(head + p) % K::CAP];
                    float dxv = (float)(tX0 + xx - pr.X) + 0.5f - pr.fx;
                    float u = fabsf(dxv) * g.inv_rs;
                    float av;
                    if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - u; av = a * a; }
                    else av = cnorm * (1.0f - u * u);
                    axt[e] = av;
                }
                for (int e = tid; e < np * 16; e += K::NTHR) {           // a_y and the disc chord
                    const int p = e >> 4, yy = e & 15;
                    const PointRec &pr = ring[(head + p) % K::CAP];
                    float dyv = (float)(tY0 + yy - pr.Y) + 0.5f - pr.fy;
                    float v = fabsf(dyv) * g.inv_rs;
                    float ay;
                    if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - v; ay = cnorm * (a * a); }
                    else ay = -cnorm * (v * v);
                    uint32_t m = (yy < yn) ? row_mask16(g, pr, tX0, tY0 + yy) : 0u;
                    rowt[e] = make_float2(ay, __uint_as_float(m));
                }
                for (int p = tid; p < np; p += K::NTHR) {                 // active layer groups
                    const PointRec &pr = ring[(head + p) % K::CAP];
                    float cpos = (float)(pr.T - tT0) + pr.ft - 0.5f;
                    int lo = max((int)floorf(cpos - g.rt) - 1, lt0);
                    int hi = min((int)ceilf(cpos + g.rt) + 1, lt1 - 1);
                    int m = 0;
                    if (lo <= hi) {
                        int g0 = lo / CT, g1 = hi / CT;
                        m = ((2 << g1) - 1) & ~((1 << g0) - 1);
                    }
                    meta[p] = m;
                }
                __syncthreads();
                // ---------------- accumulate: acc[c][t] += s_c * K_t[t] ----------------
                float2 acc2[4][CT / 2];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int q = 0; q < CT / 2; ++q) acc2[c][q] = make_float2(0.f, 0.f);
#pragma unroll 1
                for (int p = 0; p < np; ++p) {
                    if (!((meta[p] >> my_lg) & 1)) continue;               // window misses my layers
                    const float2 rw = rowt[p * 16 + my_y];
                    const uint32_t m4 = (__float_as_uint(rw.y) >> (4 * my_xg)) & 0xFu;
                    if (!__any_sync(0xffffffffu, m4 != 0u)) continue;      // disc misses my rows
                    const float4 a4 = ax4[p * 4 + my_xg];
                    float s[4];
                    if (KK == STKDE_KERNEL_PRINTED) {
                        s[0] = (m4 & 1u) ? a4.x * rw.x : 0.f;
                        s[1] = (m4 & 2u) ? a4.y * rw.x : 0.f;
                        s[2] = (m4 & 4u) ? a4.z * rw.x : 0.f;
                        s[3] = (m4 & 8u) ? a4.w * rw.x : 0.f;
                    } else {
                        s[0] = (m4 & 1u) ? a4.x + rw.x : 0.f;
                        s[1] = (m4 & 2u) ? a4.y + rw.x : 0.f;
                        s[2] = (m4 & 4u) ? a4.z + rw.x : 0.f;
                        s[3] = (m4 & 8u) ? a4.w + rw.x : 0.f;
                    }
                    const float4 *kp = kt4 + p * K::BT4 + my_lg * K::CT4;
#pragma unroll
                    for (int q = 0; q < K::CT4; ++q) {
                        const float4 k = kp[q];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            acc2[c][2 * q + 0] = ffma2(make_float2(k.x, k.y), s[c], acc2[c][2 * q + 0]);
                            acc2[c][2 * q + 1] = ffma2(make_float2(k.z, k.w), s[c], acc2[c][2 * q + 1]);
                        }
                    }
                }
                // two-level summation: registers -> shared tile accumulator [col][t]
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int col = (4 * my_xg + c) * 16 + my_y;
#pragma unroll
                    for (int q = 0; q < K::CT4; ++q) {
                        float4 &o = outer[col * K::OSTR + my_lg * K::CT4 + q];
                        float4 v = o;
                        v.x += acc2[c][2 * q].x;
                        v.y += acc2[c][2 * q].y;
                        v.z += acc2[c][2 * q + 1].x;
                        v.w += acc2[c][2 * q + 1].y;
                        o = v;
                    }
                }
                head += np;
                __syncthreads();
            }
        }

        // ---------------- store: every voxel exactly once ----------------
        // f enumerates the tile as [col][t4] with col = x*16 + y.
        auto store4 = [&](int col, int q, float4 v) {
            const int x = col >> 4, y = col & 15;
            if (x >= xn || y >= yn) return;
            const int T = tT0 + 4 * q;
            const int64_t rowbase = ((int64_t)(tX0 + x) * g.Gy + (tY0 + y)) * Ts - t_begin;
            if (vec_ok && T >= t_begin && T + 3 < t_end && T + 3 < g.Gt) {
                *reinterpret_cast<float4 *>(out + rowbase + T) = v;
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (T + j >= t_begin && T + j < t_end && T + j < g.Gt) out[rowbase + T + j] = vv[j];
            }
        };
        constexpr int NF = 256 * K::BT4;
        if (nch == 1) {
            for (int f = tid; f < NF; f += K::NTHR) {
                int col = f / K::BT4, q = f - col * K::BT4;
                store4(col, q, outer[col * K::OSTR + q]);
            }
        } else {
            const int slot0 = item.w;
            float4 *mine = partials + (size_t)(slot0 + jchunk) * NF;
            for (int f = tid; f < NF; f += K::NTHR) {
                int col = f / K::BT4, q = f - col * K::BT4;
                mine[f] = outer[col * K::OSTR + q];
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                unsigned old = atomicAdd(&arrive[ls], 1u);
                misc[1] = (old == (unsigned)(nch - 1));
            }
            __syncthreads();
            if (misc[1]) {
                __threadfence();
                for (int f = tid; f < NF; f += K::NTHR) {
                    float4 v = partials[(size_t)slot0 * NF + f];
                    for (int j = 1; j < nch; ++j) {
                        float4 w = partials[(size_t)(slot0 + j) * NF + f];
                        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
                    }
                    int col = f / K::BT4, q = f - col * K::BT4;
                    store4(col, q, v);
                }
                if (tid == 0) arrive[ls] = 0u;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ dispatch ---
typedef void (*tile_fn)(const GridParams, const PointRec *, const uint32_t *, const int4 *, const uint64_t *, int *,
                        uint32_t *, float4 *, int, int, float, float *, int64_t, int64_t, int);

template <int BT, int CT, int KK>
static tile_fn get_fn() { return k_tile<BT, CT, KK>; }

// Supported (Bt, CT) thread tiles; CT = layers per thread.
#define STKDE_TILES(X) X(16, 4) X(16, 8) X(32, 8) X(32, 16) X(64, 16)

static tile_fn select(int BT, int CT, int KK) {
#define STKDE_SEL(bt, ct) \
    if (BT == bt && CT == ct) return KK ? get_fn<bt, ct, 1>() : get_fn<bt, ct, 0>();
    STKDE_TILES(STKDE_SEL)
#undef STKDE_SEL
    return nullptr;
}

size_t tile_smem_bytes(int BT, int CT) {
#define STKDE_SM(bt, ct) \
    if (BT == bt && CT == ct) return Cfg<bt, ct>::BYTES;
    STKDE_TILES(STKDE_SM)
#undef STKDE_SM
    return 0;
}

int tile_threads(int BT, int CT) { return 64 * (BT / CT); }

int tile_occupancy(int BT, int CT, int KK, int *ctas_per_sm) {
    tile_fn f = select(BT, CT, KK);
    if (!f) return STKDE_EINVAL;
    size_t smem = tile_smem_bytes(BT, CT);
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return STKDE_ECUDA;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, tile_threads(BT, CT), smem) != cudaSuccess)
        return STKDE_ECUDA;
    *ctas_per_sm = occ;
    return STKDE_OK;
}

int launch_tile(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cnorm, float *out,
                cudaStream_t st) {
    const GridParams &g = p->g;
    tile_fn f = select(g.BT, p->CT, p->kernel);
    if (!f) return STKDE_EINVAL;
    const int nsl = g.NTX * g.NTY * (c1 - c0);
    const int64_t Ts = t_end - t_begin;
    const int vec_ok = (Ts % 4 == 0) && (t_begin % 4 == 0) && ((uintptr_t)out % 16 == 0);
    unsigned grid = (unsigned)std::min<int64_t>((int64_t)p->num_sms * p->ctas_per_sm, p->max_items);
    if (!p->wc_zeroed) cudaMemsetAsync(p->counters, 0, sizeof(int), st);   // (else by k_worklist_small)
    p->wc_zeroed = 0;
    const bool timed = p->timing && p->tev_used < p->tev_cap;
    if (timed) cudaEventRecord(p->tev[2 * p->tev_used], st);
    f<<<grid, p->tile_threads, p->smem_bytes, st>>>(g, p->rec_sorted, p->bucket_begin, p->items, p->chunk_off + nsl,
                                                    p->counters, p->arrive, reinterpret_cast<float4 *>(p->partials),
                                                    p->chunk, c0, cnorm, out, t_begin, t_end, vec_ok);
    if (timed) {
        cudaEventRecord(p->tev[2 * p->tev_used + 1], st);
        p->tev_used += 1;
    }
    p->last_own_launches += 1;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

}  // namespace stkde
