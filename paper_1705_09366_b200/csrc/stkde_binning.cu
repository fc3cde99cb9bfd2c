// stkde_binning.cu -- point preparation, home-tile binning, the tile work list,
// the exact contribution counter and the slab-gather kernel.
//
// Binning.  Every point is keyed by its HOME tile (the
// Bx x By x Bt tile holding its voxel (X_i, Y_i, T_i), clamped into the grid)
// and the (key, point index) pairs are sorted with a stable LSD radix sort,
// so every bucket lists its points in ascending input order.  A tile's
// candidate points are the buckets within Ra = ceil(H_s/Bx) tiles in X/Y and
// Rt = ceil(H_t/Bt) tiles in T: exactly the points whose box
// X_i +- H_s, Y_i +- H_s, T_i +- H_t (Alg. 2/3 loop bounds)
// can reach it -- the GPU analogue of PB-SYM-DD's "copy a point into every
// subdomain its cylinder intersects" (Alg. 4), without
// materialising the copies.
#include <cub/cub.cuh>

#include "stkde_internal.cuh"

namespace stkde {

// floor((x - x0)/sres) and the in-voxel fraction, FP64.
__device__ __forceinline__ bool make_rec(const GridParams &g, float x, float y, float t, PointRec *r) {
    if (!isfinite(x) || !isfinite(y) || !isfinite(t)) return false;
    const double LIM = 1073741824.0;  // 2^30
    double px = ((double)x - g.x0) / g.sres;
    double py = ((double)y - g.y0) / g.sres;
    double pt = ((double)t - g.t0) / g.tres;
    px = fmin(fmax(px, -LIM), LIM);
    py = fmin(fmax(py, -LIM), LIM);
    pt = fmin(fmax(pt, -LIM), LIM);
    double fx = floor(px), fy = floor(py), ft = floor(pt);
    r->X = (int)fx;
    r->Y = (int)fy;
    r->T = (int)ft;
    r->fx = (float)(px - fx);
    r->fy = (float)(py - fy);
    r->ft = (float)(pt - ft);
    // (float)(p - floor p) may round up to 1.0f; keep the fraction in [0,1)
    if (r->fx >= 1.0f) r->fx = 0.99999994f;
    if (r->fy >= 1.0f) r->fy = 0.99999994f;
    if (r->ft >= 1.0f) r->ft = 0.99999994f;
    r->x = x;
    r->y = y;
    return true;
}

// Box of the point reaches the grid at all?
__device__ __forceinline__ bool reaches_grid(const GridParams &g, const PointRec &r) {
    return r.X + g.Hs >= 0 && r.X - g.Hs < g.Gx && r.Y + g.Hs >= 0 && r.Y - g.Hs < g.Gy &&
           r.T + g.Ht >= 0 && r.T - g.Ht < g.Gt;
}

// Adaptive call: the point's (hs_i, ht_i) must be finite with 0 < hs_i <= hs and
// 0 < ht_i <= ht (the plan's bandwidths size the binning reach).
__device__ __forceinline__ bool make_bw(const GridParams &g, const float *__restrict__ bw, int64_t i, PointBw *b) {
    const float hs = bw[2 * i], ht = bw[2 * i + 1];
    if (!(hs > 0.f) || !(ht > 0.f) || !((double)hs <= g.hs) || !((double)ht <= g.ht)) return false;
    b->hs = hs;
    b->ht = ht;
    b->inv_rs = (float)(g.sres / (double)hs);
    b->inv_rt = (float)(g.tres / (double)ht);
    return true;
}

// K1: records, home-tile keys, bucket histogram.  Adaptive calls (bw != NULL) also
// write the per-point bandwidths and the maximum normalisation weight
// W_i = (sres/hs_i)^2 (tres/ht_i) (as float bits; positive floats order as unsigned).
// one point: its record and home-bucket key (sentinel: not binned); writes bw_rec[i] and,
// for a binned point, rec[i]
__device__ __forceinline__ uint32_t prep_point(const float *__restrict__ pts, int64_t i, const GridParams &g,
                                               PointRec *__restrict__ rec, int *__restrict__ err, uint32_t sentinel,
                                               const float *__restrict__ bw, PointBw *__restrict__ bw_rec,
                                               unsigned *__restrict__ wmax, int t_begin, int t_end) {
    float x = pts[3 * i], y = pts[3 * i + 1], t = pts[3 * i + 2];
    PointRec r;
    uint32_t key = sentinel;
    bool bw_ok = true;
    PointBw b{0.f, 0.f, 0.f, 0.f};
    if (bw) {
        bw_ok = make_bw(g, bw, i, &b);
        if (!bw_ok) atomicOr(err, 4);
        if (bw_rec) bw_rec[i] = b;
    }
    const bool rec_ok = make_rec(g, x, y, t, &r);
    if (bw && bw_ok && rec_ok) {
        // The fixed-point full scale of an adaptive call: max_i W_i s_i, s_i >= the point's largest
        // spatial factor over ALL voxel columns -- reached at the column nearest to it in x and in y
        // (k_s decreases in |u| and |v| separately).  A point whose disc holds no
        // voxel centre near its peak (sub-voxel hs_i) then no longer inflates the scale (DESIGN.md
        // section 5, "small contributions").  eps covers the FP32 rounding of the generators'
        // tile-relative position (|b_x| < 256: half an ulp <= 2^-17) times sres/hs_i, the 1.0001
        // their FP32 products and this value's own rounding, so W_i/scale * a_x * a_y <= 1 holds
        // for every column in the tile kernel's arithmetic.  Depends on the points only: every
        // slab of a grid sees the same scale (slabs stay bitwise equal to the full grid).
        const double ws = g.sres / (double)b.hs, wt = g.tres / (double)b.ht;
        const double is = (double)b.inv_rs, eps = is * 1.52587890625e-05 + 1e-6;
        const double ux = fabs(0.5 - (double)r.fx) * is, uy = fabs(0.5 - (double)r.fy) * is;
        double sp;
        if (g.kernel == STKDE_KERNEL_PRINTED) {
            const double ax = fmin(fmax(1.0 - ux, 0.0) + eps, 1.0), ay = fmin(fmax(1.0 - uy, 0.0) + eps, 1.0);
            sp = ax * ax * ay * ay;
        } else {
            sp = fmin(fmax(1.0 - ux * ux - uy * uy, 0.0) + 4.0 * eps, 1.0);
        }
        atomicMax(wmax, __float_as_uint((float)(ws * ws * wt * sp * 1.0001)));
    }
    if (!rec_ok) {
        atomicOr(err, 1);
    } else if (bw_ok && reaches_grid(g, r) && r.T + g.Ht >= t_begin && r.T - g.Ht < t_end &&
               r.X + g.Hs >= g.XA0 * BX && r.X - g.Hs < (g.XA0 + g.NXA) * BX) {
        // (points whose window [T_i - H_t, T_i + H_t] misses the requested slab are not binned)
        int a = min(max(r.X, 0), g.Gx - 1) / BX;
        int b = min(max(r.Y, 0), g.Gy - 1) / g.BY;
        int c = min(max(r.T, 0), g.Gt - 1) / g.BTH;
        key = (uint32_t)((c * g.NTY + b) * g.NTX + a);
    }
    // only binned records are read back (slab calls skip most); the counting-sort path writes
    // none here: its scatter recomputes each record from the point (k_scatter)
    if (key != sentinel && rec) rec[i] = r;
    return key;
}

__global__ void k_prep(const float *__restrict__ pts, int64_t n, GridParams g, PointRec *__restrict__ rec,
                       uint32_t *__restrict__ keys, uint32_t *__restrict__ vals,
                       uint32_t *__restrict__ bucket_cnt, int *__restrict__ err, uint32_t sentinel,
                       const float *__restrict__ bw, PointBw *__restrict__ bw_rec, unsigned *__restrict__ wmax,
                       int t_begin, int t_end, int ranks) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = prep_point(pts, i, g, ranks ? nullptr : rec, err, sentinel, bw, ranks ? nullptr : bw_rec,
                                    wmax, t_begin, t_end);
    // (unbinned points keep the sentinel key and sort last; they are not counted: with slab
    // culling most points of a slab call are unbinned, and one shared counter serialised them)
    // rank = this point's slot in its bucket (counting-sort path of the tcgen05 engine)
    keys[i] = key;
    const uint32_t rank = key != sentinel ? atomicAdd(&bucket_cnt[key], 1u) : 0u;   // (every path's counts)
    if (!ranks) vals[i] = (uint32_t)i;
    else if (key != sentinel) vals[i] = rank;     // unbinned points' ranks are never read
}

// K1b: records (and adaptive bandwidths) in bucket order (coalesced candidate reads
// in the tile kernel).
__global__ void k_permute(const PointRec *__restrict__ rec, const uint32_t *__restrict__ vals,
                          PointRec *__restrict__ out, int64_t n, const PointBw *__restrict__ bw_rec,
                          PointBw *__restrict__ bw_out, const uint32_t *__restrict__ nbinned) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n && j < (int64_t)*nbinned) {      // the unbinned (sentinel-key) records sort last
        const uint32_t v = vals[j];
        out[j] = rec[v];
        if (bw_rec) bw_out[j] = bw_rec[v];
    }
}

// Exact disc chords of every (sorted) point, for the tcgen05 engine.  Point i
// owns R8 = chord_rows(Hs) entries for the absolute rows Y = Y0(i) + e,
// Y0(i) = floor8(Y_i - H_s), so that the 8 rows of any 16x8-column tile are
// one aligned 16-byte block.  Entry = int8 (lo, hi): columns [X_i + lo,
// X_i + hi] whose centres pass the spatial gate of Alg. 1,
// (1, 0) for an empty row; computed once per point instead of once per
// (point, tile) visit.  Requires H_s <= 120.  Adaptive calls (bw != NULL): the
// disc of point i has its own radius hs_i (the table layout keeps the plan's H_s).
// One thread per point: its 8-row blocks are 16-byte stores of one contiguous table row.
__device__ __forceinline__ uint32_t chord_pack(int dl, int dh) {
    return (uint32_t)((uint8_t)(int8_t)dl) | ((uint32_t)(uint8_t)(int8_t)dh << 8);
}
// FP32 fast path in voxel-local coordinates: column X_i + k is inside iff (k - pc)^2 + dy^2 < r^2
// with pc = fx - 0.5.  The chord ends come from an approximate sqrt (rsqrt) and are then
// verified: both ends inside and both outer neighbours outside, each decided outside the FP64
// band.  Returns false when a decision falls within the band (or the estimate was off by a
// column): the caller then takes chord_entry_exact.
__device__ __forceinline__ bool chord_entry_fast(const GridParams &g, const PointRec &r, int Y, uint32_t &e) {
    e = chord_pack(1, 0);                                   // empty row
    const int dyi = Y - r.Y;
    if (dyi < -g.Hs || dyi > g.Hs) return true;
    const float dyv = (float)dyi + 0.5f - r.fy;
    const float dy2 = __fmul_rn(dyv, dyv);
    const float lo_b = g.rs2 * (1.0f - GATE_BAND), hi_b = g.rs2 * (1.0f + GATE_BAND);
    if (dy2 > hi_b) return true;
    if (!(dy2 < lo_b)) return false;
    const float pc = r.fx - 0.5f;
    const float c2 = g.rs2 - dy2;
    const float c = c2 * rsqrtf(c2);
    const int a = __float2int_rd(pc - c) + 1, b = __float2int_ru(pc + c) - 1;
    auto d2 = [&](int k) { const float dx = (float)k - pc; return __fadd_rn(__fmul_rn(dx, dx), dy2); };
    if (a <= b && d2(a) < lo_b && d2(b) < lo_b && d2(a - 1) > hi_b && d2(b + 1) > hi_b) {
        e = chord_pack(a, b);
        return true;
    }
    return false;
}
// exact chord (row_chord: Alg. 1's FP64 gate near the edge)
__device__ __forceinline__ uint32_t chord_entry_exact(const GridParams &g, const PointRec &r, int Y) {
    int lo, hi;
    row_chord(g, r, Y, &lo, &hi);
    return lo <= hi ? chord_pack(lo - r.X, hi - r.X) : chord_pack(1, 0);
}
// one 8-row block of a point's chord table: block rows Y0 .. Y0 + 7 -> 4 words; the rare
// rows the fast path cannot decide take the exact path in one (not unrolled) loop
__device__ __forceinline__ uint4 chord_block(const GridParams &g, const PointRec &r, int Y0) {
    uint32_t w[4];
    unsigned need = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t e0, e1;
        if (!chord_entry_fast(g, r, Y0 + 2 * k, e0)) need |= 1u << (2 * k);
        if (!chord_entry_fast(g, r, Y0 + 2 * k + 1, e1)) need |= 2u << (2 * k);
        w[k] = e0 | (e1 << 16);
    }
#pragma unroll 1
    while (need) {
        const int k = __ffs(need) - 1;
        need &= need - 1u;
        const uint32_t v = chord_entry_exact(g, r, Y0 + k);
        const int sh = 16 * (k & 1), wi = k >> 1;
        const uint32_t m = ~(0xFFFFu << sh);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q == wi) w[q] = (w[q] & m) | (v << sh);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Dense over the binned (sorted) points, so a slab call's few binned points cost only
// themselves.  finalize: after its chords a record's x / y are rewritten for the loader (below);
// the sweep (xy != NULL) keeps the world coordinates in a side buffer and sets x the same way.
#ifndef STKDE_CHORD_ROWS
#define STKDE_CHORD_ROWS 1
#endif
constexpr uint32_t EMPTY_PAIR = 0x00010001u;      // two empty rows: int8 (lo, hi) = (1, 0) each
constexpr int CHORD_STAGE_MAX = 48;               // table rows staged per thread (H_s <= 20)
__global__ void k_chords(PointRec *__restrict__ rec, int64_t n, GridParams gp, uint16_t *__restrict__ chords,
                         const PointBw *__restrict__ bw, const uint32_t *__restrict__ nbinned,
                         const float2 *__restrict__ xy, int finalize) {
    // each thread's table rows staged in shared memory (chord_stage_bytes: blockDim x
    // chord_rows(H_s) x 2 B when chord_rows(H_s) <= CHORD_STAGE_MAX, else none)
    extern __shared__ __align__(16) uint16_t stage_buf[];
    uint16_t *stage = (STKDE_CHORD_ROWS && chord_rows(gp.Hs) <= CHORD_STAGE_MAX) ? stage_buf : nullptr;
    const int nb = chord_rows(gp.Hs) / 8;            // 8-row blocks per point
    const int64_t total = min(n, (int64_t)*nbinned);  // binned points only (they sort first): dense
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        PointRec r = rec[i];
        if (xy) {
            const float2 c = xy[i];
            r.x = c.x;
            r.y = c.y;
            rec[i].x = __int_as_float((int)i);
        }
        const GridParams g = bw ? with_point_bw(gp, bw[i]) : gp;
        const int Y0 = (r.Y - g.Hs) & ~7;
        uint4 *dst = reinterpret_cast<uint4 *>(chords) + i * nb;
#if STKDE_CHORD_ROWS
        if (stage) {
            // only the point's own 2 H_s + 1 rows (at table offset e0 = (Y_i - H_s) mod 8): every
            // lane of the warp runs the same row count instead of the union of the lanes' ranges
            // (small discs, where the union is up to 7 rows longer than 2 H_s + 1: ornith chords
            // 0.309 -> 0.273 ms, social 0.036 -> 0.029 ms; stress, with 65 of 80 rows in every
            // point's range, was 4 % slower staged and keeps the block loop)
            uint16_t *my = stage + threadIdx.x * (nb * 8);
            uint32_t *my32 = reinterpret_cast<uint32_t *>(my);
            for (int e = 0; e < nb * 4; ++e) my32[e] = EMPTY_PAIR;
            const int e0 = (r.Y - gp.Hs) - Y0;
            for (int k = 0; k <= 2 * gp.Hs; ++k) {
                const int Y = r.Y - gp.Hs + k;
                uint32_t v;
                if (!chord_entry_fast(g, r, Y, v)) v = chord_entry_exact(g, r, Y);
                my[e0 + k] = (uint16_t)v;
            }
            const uint4 *src = reinterpret_cast<const uint4 *>(my);
            for (int blk = 0; blk < nb; ++blk) dst[blk] = src[blk];
        } else
#endif
        for (int blk = 0; blk < nb; ++blk) dst[blk] = chord_block(g, r, Y0 + 8 * blk);
        if (finalize) {
            // once the chords exist the tile kernel needs neither world coordinate of the sorted
            // record (its FP64 gates are in the chords): x carries the record's own sorted index,
            // so the loader finds a candidate's chord row without a search; adaptive calls: y
            // carries the point's own reach for the loader's cull -- its disc radius
            // rs_i = hs_i / sres rounded UP to 10 mantissa bits (conservative) with its window
            // H_t(i) = floor(ht_i / tres) + 1 <= Ht in the 13 freed low bits
            float2 xyw = make_float2(__int_as_float((int)i), r.y);
            if (bw) {
                const PointBw b = bw[i];
                const int hti = min(gp.Ht, (int)(1.0f / b.inv_rt) + 1);
                const uint32_t rb = (__float_as_uint(1.0f / b.inv_rs) + 0x1FFFu) & ~0x1FFFu;
                xyw.y = __uint_as_float(rb | (uint32_t)hti);
            }
            reinterpret_cast<float2 *>(&rec[i].x)[0] = xyw;
        }
    }
}

static inline size_t chord_stage_bytes(int Hs, int threads) {
    return (STKDE_CHORD_ROWS && chord_rows(Hs) <= CHORD_STAGE_MAX) ? (size_t)threads * chord_rows(Hs) * 2 : 0;
}

// K1c (tcgen05 engine): counting-sort scatter.  Record i goes to bucket_begin[key] + rank,
// its slot from k_prep's atomic bucket count: buckets are contiguous runs as with the radix
// sort, but the order inside a bucket is the atomics' order.  The tcgen05 tile sums are exact
// integers, independent of the candidates' order and grouping, and every voxel is rounded
// once from its sum, so the grid is bitwise the same for any order.  The chord
// table follows in a dense pass over the sorted records (k_chords with finalize).
__global__ void k_scatter(const float *__restrict__ pts, GridParams g, const uint32_t *__restrict__ keys,
                          const uint32_t *__restrict__ ranks, const uint32_t *__restrict__ bucket_begin,
                          uint32_t sentinel, int64_t n, PointRec *__restrict__ out, const float *__restrict__ bw,
                          PointBw *__restrict__ bw_out) {
    // each binned record recomputed from its point (the same FP64 prep as k_prep: bitwise the
    // same record) and written once at its bucket slot -- k_prep stores only keys and ranks
    // four keys per thread and iteration (one 16-B load): slab calls skip most points, so the
    // key reads are the pass's main traffic
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i0 < n; i0 += stride) {
        uint32_t kk[4];
        if (i0 + 4 <= n) {
            const uint4 k4 = *reinterpret_cast<const uint4 *>(keys + i0);
            kk[0] = k4.x; kk[1] = k4.y; kk[2] = k4.z; kk[3] = k4.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) kk[q] = i0 + q < n ? keys[i0 + q] : sentinel;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (kk[q] == sentinel) continue;
            const int64_t i = i0 + q;
            const int64_t j = (int64_t)bucket_begin[kk[q]] + ranks[i];
            PointRec r;
            make_rec(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &r);
            out[j] = r;
            if (bw) {
                PointBw b;
                make_bw(g, bw, i, &b);
                bw_out[j] = b;
            }
        }
    }
}

// Candidate count of a tile: sum of its home-bucket segments.
__device__ __forceinline__ uint32_t tile_candidates(const GridParams &g, const uint32_t *__restrict__ bb,
                                                    int a, int b, int c) {
    int a0 = max(a - g.Ra, 0), a1 = min(a + g.Ra, g.NTX - 1);
    int b0 = max(b - g.Ray, 0), b1 = min(b + g.Ray, g.NTY - 1);
    int c0, c1;
    home_t_range(g, c, &c0, &c1);
    uint32_t s = 0;
    for (int cc = c0; cc <= c1; ++cc)
        for (int bb2 = b0; bb2 <= b1; ++bb2) {
            int k = (cc * g.NTY + bb2) * g.NTX;
            s += bb[k + a1 + 1] - bb[k + a0];
        }
    return s;
}

// 8-bit log-class work-list keys (one radix pass; 0: exact 16-bit counts, two passes)
#ifndef STKDE_WL_KEY8
#define STKDE_WL_KEY8 1
#endif
// K3a: per slab tile, candidate count and work-list sort key (stable radix sort, ascending).
//   order 0 (LPT, "most loaded subdomain first"): descending count;
//   order 1 (locality): tiles with >= `heavy` candidates first by descending count, then the
//     rest in slab-tile order (x fastest, then y, then the layer block), so the persistent
//     CTAs work on neighbouring tiles at the same time and their candidate records and
//     chords are shared in L2 instead of re-read from DRAM.
// Counts are clamped to 16 bits in the key (the order only needs to be approximate; the
// exact count is kept in tcnt for the chunking).
__global__ void k_tile_counts(GridParams g, const uint32_t *__restrict__ bucket_begin, int c0, int nsl,
                              uint32_t *__restrict__ lkey, uint32_t *__restrict__ lval, uint32_t *__restrict__ tcnt,
                              int order, uint32_t heavy) {
    int ls = blockIdx.x * blockDim.x + threadIdx.x;
    if (ls >= nsl) return;
    int a = ls % g.NXA + g.XA0, b = (ls / g.NXA) % g.NTY, c = ls / (g.NXA * g.NTY) + c0;
    uint32_t cnt = tile_candidates(g, bucket_begin, a, b, c);
#if STKDE_WL_KEY8
    // 8-bit keys (one radix pass): the count's log class 16 log2(cnt + 1) from its leading bit
    // and the next four (steps of <= 6.25 %, monotone; capped at 254), descending; locality
    // order: the non-heavy tiles share key 255 and keep their slab-tile order (stable sort)
    const uint32_t v = cnt + 1u;
    const int e = 31 - __clz(v);
    const uint32_t frac = (e >= 4 ? v >> (e - 4) : v << (4 - e)) & 15u;
    const uint32_t cls = min(16u * (uint32_t)e + frac, 254u);
    lkey[ls] = (order == 0 || cnt >= heavy) ? 254u - cls : 255u;
#else
    // locality order in 16-bit keys: the non-heavy tiles share the largest key, and the stable
    // sort keeps them in slab-tile order (two radix passes instead of three)
    lkey[ls] = order == 0 ? 0xFFFFu - min(cnt, 0xFFFFu) : (cnt >= heavy ? 0xFFFEu - min(cnt, 0xFFFEu) : 0xFFFFu);
#endif
    lval[ls] = (uint32_t)ls;
    tcnt[ls] = cnt;
}

// K3b: chunks per tile (in work-list order) packed with split-slot demand.
// The whole work list of a small slab (nsl <= WL_CAP tiles) in ONE CTA, one tile per thread:
// candidate counts, the keys' stable order (a bitonic sort of key << 10 | tile in shared
// memory: ties keep the tile order, as the general path's stable radix sort does), chunk
// packing, the offset scan and the items -- the six kernels of the general path
// (k_tile_counts, radix sort, k_chunk_pack, scan, k_items) and the item-counter memset as
// one launch, for the launch-bound small grids (same keys, same order, same items).
constexpr int WL_THR = 1024, WL_CAP = WL_THR;
__global__ void __launch_bounds__(WL_THR, 1)
k_worklist_small(GridParams g, const uint32_t *__restrict__ bucket_begin, int c0, int nsl, int order,
                 uint32_t heavy, int chunk, uint32_t *__restrict__ tcnt, uint32_t *__restrict__ lval,
                 uint64_t *__restrict__ off_out, int4 *__restrict__ items, int64_t max_items, int64_t max_slots,
                 int *__restrict__ err, int *__restrict__ work_counter) {
    using Scan = cub::BlockScan<unsigned long long, WL_THR>;
    __shared__ typename Scan::TempStorage ts;
    __shared__ uint32_t sk[WL_CAP], scnt[WL_CAP];
    const int ls = threadIdx.x;
    uint32_t cnt = 0, ck = 0xFFFFFFFFu;                        // padding sorts last
    if (ls < nsl) {
        const int a = ls % g.NXA + g.XA0, b = (ls / g.NXA) % g.NTY, c = ls / (g.NXA * g.NTY) + c0;
        cnt = tile_candidates(g, bucket_begin, a, b, c);
        const uint32_t lpt = 0xFFFFu - min(cnt, 0xFFFFu);
        const uint32_t key = (order == 0 || cnt >= heavy) ? lpt : 0x10000u + (uint32_t)ls;   // < 2^17
        ck = key << 10 | (uint32_t)ls;
        tcnt[ls] = cnt;
    }
    scnt[ls] = cnt;
    // ascending bitonic sort of the nsl keys padded to NP = 2^ceil(log2 nsl) (block-uniform):
    // strides < 32 by warp shuffles, the others through shared memory
    int NP = 32;
    while (NP < nsl) NP <<= 1;
    uint32_t v = ck;
    for (int kk = 2; kk <= NP; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            uint32_t o;
            if (jj >= 32) {
                __syncthreads();                               // previous readers of sk done
                sk[ls] = v;
                __syncthreads();
                o = sk[ls ^ jj];
            } else {
                o = __shfl_xor_sync(0xFFFFFFFFu, v, jj);
            }
            const bool up = (ls & kk) == 0, lower = (ls & jj) == 0;
            v = (up == lower) ? min(v, o) : max(v, o);
        }
    unsigned long long pk = 0;
    const int k = ls;
    int tile = 0;
    __syncthreads();                                           // scnt complete
    if (k < nsl) {
        tile = (int)(v & 1023u);
        const uint32_t cc = scnt[tile];
        const uint32_t nch = cc == 0 ? 1u : (cc + chunk - 1) / chunk;
        pk = (unsigned long long)nch | ((unsigned long long)(nch > 1 ? nch : 0) << 32);
        lval[k] = (uint32_t)tile;
    }
    unsigned long long o, total;
    Scan(ts).ExclusiveSum(pk, o, total);
    if (k < nsl) {
        off_out[k] = o;
        const uint32_t i0 = (uint32_t)o, nch = (uint32_t)pk, s0 = (uint32_t)(o >> 32);
        if ((int64_t)i0 + nch > max_items || (nch > 1 && (int64_t)s0 + nch > max_slots)) {
            atomicOr(err, 2);
        } else {
            for (uint32_t q = 0; q < nch; ++q)
                items[i0 + q] = make_int4(tile, (int)q, (int)nch, nch > 1 ? (int)s0 : -1);
        }
    }
    if (k == 0) {
        off_out[nsl] = total;
        *work_counter = 0;                // the tile kernel's item counter (no separate memset)
    }
}
__global__ void k_chunk_pack(const uint32_t *__restrict__ lval, const uint32_t *__restrict__ tcnt, int nsl, int chunk,
                             uint64_t *__restrict__ pack) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > nsl) return;
    if (k == nsl) { pack[k] = 0; return; }
    uint32_t cnt = tcnt[lval[k]];
    uint32_t nch = cnt == 0 ? 1u : (cnt + chunk - 1) / chunk;
    uint64_t slots = nch > 1 ? nch : 0;
    pack[k] = (uint64_t)nch | (slots << 32);
}

// K3c: expand to work items {slab tile, chunk j, nchunks, slot base}.
__global__ void k_items(const uint32_t *__restrict__ lval, const uint64_t *__restrict__ off, int nsl,
                        int4 *__restrict__ items, int64_t max_items, int64_t max_slots, int *__restrict__ err) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nsl) return;
    uint64_t o = off[k], o1 = off[k + 1];
    uint32_t i0 = (uint32_t)o, nch = (uint32_t)o1 - i0;
    uint32_t s0 = (uint32_t)(o >> 32);
    if ((int64_t)i0 + nch > max_items || (nch > 1 && (int64_t)s0 + nch > max_slots)) {
        atomicOr(err, 2);
        return;
    }
    for (uint32_t j = 0; j < nch; ++j)
        items[i0 + j] = make_int4((int)lval[k], (int)j, (int)nch, nch > 1 ? (int)s0 : -1);
}

// Exact contribution count: one warp per point (adaptive: the point's own bandwidths).
__global__ void k_count(const float *__restrict__ pts, int64_t n, GridParams gp, int64_t t_begin, int64_t t_end,
                        unsigned long long *__restrict__ out, const float *__restrict__ bwin, int x_begin, int x_end) {
    __shared__ unsigned long long part[32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned long long mine = 0;
    if (i < n) {
        PointRec r;
        PointBw b{0.f, 0.f, 0.f, 0.f};
        const bool bw_ok = !bwin || make_bw(gp, bwin, i, &b);
        const GridParams g = bwin ? with_point_bw(gp, b) : gp;
        if (bw_ok && make_rec(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &r) && reaches_grid(gp, r)) {
            int cols = 0, lay = 0;
            int y0 = max(r.Y - g.Hs, 0), y1 = min(r.Y + g.Hs, g.Gy - 1);
            for (int Y = y0 + lane; Y <= y1; Y += 32) {
                int lo, hi;
                row_chord(g, r, Y, &lo, &hi);
                lo = max(lo, x_begin);
                hi = min(hi, x_end - 1);
                cols += max(hi - lo + 1, 0);
            }
            int t0 = (int)max((int64_t)r.T - g.Ht, t_begin), t1 = (int)min((int64_t)r.T + g.Ht, t_end - 1);
            const float pt = pts[3 * i + 2];   // exact temporal gate needs the original t
            for (int T = t0 + lane; T <= t1; T += 32) lay += gate_t_fp64(g, T, pt) ? 1 : 0;
            for (int o = 16; o; o >>= 1) {
                cols += __shfl_xor_sync(0xffffffffu, cols, o);
                lay += __shfl_xor_sync(0xffffffffu, lay, o);
            }
            mine = (unsigned long long)cols * (unsigned long long)lay;
        }
    }
    if (lane == 0) part[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
        if (s) atomicAdd(out, s);
    }
}

// Histogram of T_i (clamped) for the slab partition.
__global__ void k_hist_t(const float *__restrict__ pts, int64_t n, GridParams g, int *__restrict__ hist) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    PointRec r;
    if (!make_rec(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &r) || !reaches_grid(g, r)) return;
    atomicAdd(&hist[min(max(r.T, 0), g.Gt - 1)], 1);
}

// Histogram of X_i (clamped) for the x-slab partition.
__global__ void k_hist_x(const float *__restrict__ pts, int64_t n, GridParams g, int *__restrict__ hist) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    PointRec r;
    if (!make_rec(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &r) || !reaches_grid(g, r)) return;
    atomicAdd(&hist[min(max(r.X, 0), g.Gx - 1)], 1);
}

// Slab [t0,t1) of layout [Gx][Gy][t1-t0] -> full grid [Gx][Gy][Gt].
// On the root of a multi-device run `slab` is a peer pointer (NVLink).
__global__ void k_gather(const float *__restrict__ slab, int64_t rows, int64_t Gt, int64_t t0, int64_t ts,
                         float *__restrict__ full) {
    int64_t total = rows * ts;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = e / ts, t = e - row * ts;
        full[row * Gt + t0 + t] = slab[e];
    }
}

// ----------------------------------------------------------- launchers ---
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

int launch_binning(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st, int64_t t_begin,
                   int64_t t_end, bool with_chords, bool stable) {
    const GridParams &g = p->g;
    phase_call_begin(p, st);
    const bool ad = p->d_bw != nullptr;
    // tcgen05 engine: counting-sort scatter by the atomic bucket ranks (order-free exact sums);
    // the FP32 engines keep the stable radix sort (their sums depend on the order)
    // (stable: the FP64-output path sums each voxel in bucket-then-input order)
    const bool counting = p->engine == STKDE_ENGINE_TC && !stable;
    {
        Phase ph(p, st, STKDE_PHASE_PREP);
        cudaMemsetAsync(p->bucket_cnt, 0, (p->nbuckets + 1) * sizeof(uint32_t), st);
        if (ad) cudaMemsetAsync(p->counters + 6, 0, sizeof(int), st);
        k_prep<<<nblk(n, 256), 256, 0, st>>>(d_points, n, g, p->rec, p->keys_in, p->vals_in, p->bucket_cnt,
                                              p->counters + 1, (uint32_t)p->nbuckets, p->d_bw,
                                              ad ? p->bw_rec : nullptr, reinterpret_cast<unsigned *>(p->counters + 6),
                                              (int)t_begin, (int)t_end, counting ? 1 : 0);
    }
    size_t bytes = p->cub_bytes;
    if (!counting) {
        Phase ph(p, st, STKDE_PHASE_SORT);
        if (cub::DeviceRadixSort::SortPairs(p->cub_tmp, bytes, p->keys_in, p->keys_out, p->vals_in, p->vals_out,
                                            (int)n, 0, p->key_bits, st) != cudaSuccess)
            return STKDE_ECUDA;
        bytes = p->cub_bytes;
    }
    {
        Phase ph(p, st, STKDE_PHASE_SCAN);
        if (cub::DeviceScan::ExclusiveSum(p->cub_tmp, bytes, p->bucket_cnt, p->bucket_begin, (int)(p->nbuckets + 1),
                                          st) != cudaSuccess)
            return STKDE_ECUDA;
    }
    if (counting) {
        // bucket_begin[nbuckets] = the number of binned points
        {
            Phase ph(p, st, STKDE_PHASE_SCATTER);
            k_scatter<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk((n + 3) / 4, 256), (int64_t)p->num_sms * 16)),
                        256, 0, st>>>(d_points, g, p->keys_in, p->vals_in, p->bucket_begin,
                                                     (uint32_t)p->nbuckets, n, p->rec_sorted, p->d_bw,
                                                     p->bw_sorted);
        }
        p->last_own_launches += 2;
        p->last_cub_calls += 1;
        p->ridx_in_rec = 0;
        // the chord table over the binned (sorted, dense) points only: a slab call's few binned
        // points are not spread over every warp of an all-points pass
        if (with_chords) {
            Phase ph(p, st, STKDE_PHASE_CHORDS);
            const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, (int64_t)p->num_sms * 64));
            k_chords<<<blocks, 128, chord_stage_bytes(g.Hs, 128), st>>>(p->rec_sorted, n, g, p->chords, ad ? p->bw_sorted : nullptr,
                                             p->bucket_begin + p->nbuckets, nullptr, 1);
            p->ridx_in_rec = 1;
            p->last_own_launches += 1;
        }
    } else {
        p->ridx_in_rec = 0;
        // bucket_begin[nbuckets] = the number of binned points (the sentinel bucket sorts last)
        Phase ph(p, st, STKDE_PHASE_SCATTER);
        k_permute<<<nblk(n, 256), 256, 0, st>>>(p->rec, p->vals_out, p->rec_sorted, n, ad ? p->bw_rec : nullptr,
                                                 p->bw_sorted, p->bucket_begin + p->nbuckets);
        p->last_own_launches += 2;
        p->last_cub_calls += 2;
    }
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

__global__ void k_save_xy(const PointRec *__restrict__ rec, int64_t n, const uint32_t *__restrict__ nbinned,
                          float2 *__restrict__ xy) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n && j < (int64_t)*nbinned) xy[j] = make_float2(rec[j].x, rec[j].y);
}

int launch_chords(stkde_plan_s *p, int64_t n, cudaStream_t st, const float2 *xy) {
    Phase ph(p, st, STKDE_PHASE_CHORDS);
    if (n > 0) {
        const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)p->num_sms * 32);
        k_chords<<<blocks, 256, chord_stage_bytes(p->g.Hs, 256), st>>>(p->rec_sorted, n, p->g, p->chords, p->d_bw ? p->bw_sorted : nullptr,
                                         p->bucket_begin + p->nbuckets, xy, 0);
        p->last_own_launches += 1;
    }
    p->ridx_in_rec = xy ? 1 : 0;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_save_xy(stkde_plan_s *p, int64_t n, float2 *xy, cudaStream_t st) {
    Phase ph(p, st, STKDE_PHASE_SCATTER);
    if (n > 0) {
        k_save_xy<<<nblk(n, 256), 256, 0, st>>>(p->rec_sorted, n, p->bucket_begin + p->nbuckets, xy);
        p->last_own_launches += 1;
    }
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_worklist(stkde_plan_s *p, int c0, int c1, cudaStream_t st) {
    const GridParams &g = p->g;
    Phase ph(p, st, STKDE_PHASE_WORKLIST);
    int nsl = g.NXA * g.NTY * (c1 - c0);
    // locality order only for grids with many tiles per SM (few tiles: LPT balances the SMs)
    const int order = p->order >= 0 ? p->order : (nsl >= 64 * p->num_sms ? 1 : 0);
    const int kbits = STKDE_WL_KEY8 ? 8 : 16;        // LPT and locality keys (k_tile_counts)
    if (nsl <= WL_CAP && p->wl_small) {              // small slab: the whole work list in one CTA
        k_worklist_small<<<1, WL_THR, 0, st>>>(g, p->bucket_begin, c0, nsl, order, (uint32_t)p->heavy, p->chunk,
                                               p->tile_cnt, p->lpt_val_out, p->chunk_off, p->items, p->max_items,
                                               p->max_slots, p->counters + 1, p->counters);
        p->wc_zeroed = 1;
        p->last_own_launches += 1;
        return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
    }
    p->wc_zeroed = 0;
    k_tile_counts<<<nblk(nsl, 256), 256, 0, st>>>(g, p->bucket_begin, c0, nsl, p->lpt_key_in, p->lpt_val_in,
                                                  p->tile_cnt, order, (uint32_t)p->heavy);
    size_t bytes = p->cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(p->cub_tmp, bytes, p->lpt_key_in, p->lpt_key_out, p->lpt_val_in,
                                        p->lpt_val_out, nsl, 0, kbits, st) != cudaSuccess)
        return STKDE_ECUDA;
    k_chunk_pack<<<nblk(nsl + 1, 256), 256, 0, st>>>(p->lpt_val_out, p->tile_cnt, nsl, p->chunk, p->chunk_pack);
    bytes = p->cub_bytes;
    if (cub::DeviceScan::ExclusiveSum(p->cub_tmp, bytes, p->chunk_pack, p->chunk_off, nsl + 1, st) != cudaSuccess)
        return STKDE_ECUDA;
    k_items<<<nblk(nsl, 256), 256, 0, st>>>(p->lpt_val_out, p->chunk_off, nsl, p->items, p->max_items,
                                            p->max_slots, p->counters + 1);
    p->last_own_launches += 3;
    p->last_cub_calls += 2;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

// candidate count of every slab tile into p->tile_cnt (the x-slab partition's cost model)
int launch_tile_cost(stkde_plan_s *p, int nsl, cudaStream_t st) {
    Phase ph(p, st, STKDE_PHASE_WORKLIST);
    k_tile_counts<<<nblk(nsl, 256), 256, 0, st>>>(p->g, p->bucket_begin, 0, nsl, p->lpt_key_in, p->lpt_val_in,
                                                  p->tile_cnt, 0, 0u);
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_count(stkde_plan_s *p, const float *d_points, int64_t n, int64_t t_begin, int64_t t_end,
                 int64_t *d_count, cudaStream_t st, const float *d_bw, int64_t x_begin, int64_t x_end) {
    cudaMemsetAsync(d_count, 0, sizeof(int64_t), st);
    if (n > 0)
        k_count<<<nblk(n * 32, 256), 256, 0, st>>>(d_points, n, p->g, t_begin, t_end,
                                                   reinterpret_cast<unsigned long long *>(d_count), d_bw,
                                                   (int)x_begin, (int)x_end);
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_hist_t(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st) {
    cudaMemsetAsync(p->hist_t, 0, (p->g.Gt + 1) * sizeof(int), st);
    if (n > 0) k_hist_t<<<nblk(n, 256), 256, 0, st>>>(d_points, n, p->g, p->hist_t);
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_hist_x(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st) {
    cudaMemsetAsync(p->hist_x, 0, (p->g.Gx + 1) * sizeof(int), st);
    if (n > 0) k_hist_x<<<nblk(n, 256), 256, 0, st>>>(d_points, n, p->g, p->hist_x);
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

int launch_gather(const float *slab, int64_t Gx, int64_t Gy, int64_t Gt, int64_t t0, int64_t t1, float *full,
                  cudaStream_t st) {
    int64_t rows = Gx * Gy, ts = t1 - t0;
    int64_t total = rows * ts;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (total > 0) k_gather<<<blocks, 256, 0, st>>>(slab, rows, Gt, t0, ts, full);
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

}  // namespace stkde
