// stkde_tile_mma.cu -- tensor-core variant of the PB-SYM tile kernel.
//
// Per tile the accumulation of Alg. 3,
//     out[(x,y)][t] += sum_p  S[(x,y)][p] * K_t[p][t],   S = K_s (masked a_x a_y),
// is a contraction over the points p: D(256 x Bt) += S(256 x P) . T(P x Bt).
// Each warp owns two tile rows (2 x 16 columns = two m16 tiles) and all Bt
// layers (Bt/8 n8 tiles) and issues mma.sync m16n8k16 (FP16 in, FP32 acc).
// FP32 accuracy is kept with the 3-term split  a*b ~ ah*bh + ah*bl + al*bh,
// ah = fp16(a), al = fp16(a - ah)  (relative error ~2^-22 per product; the
// dropped al*bl term is below FP32 rounding of the sum).  The S operand is
// generated in registers in the A-fragment layout (no shared-memory round
// trip); the K_t operand is split once per sub-batch into B-fragment order in
// shared memory.  Warps skip m-tiles whose row misses all 16 discs of a
// k-step and n-tiles outside the union of the 16 windows.  Candidate staging,
// two-level summation and the exactly-once store are those of stkde_tile.cu.
#include <cuda_fp16.h>

#include "stkde_internal.cuh"

namespace stkde {

template <int BT>
struct CfgM {
    static constexpr int NTHR = 256;             // 8 warps; warp w owns rows 2w, 2w+1
    static constexpr int NWARP = 8;
    static constexpr int P = 32;                 // points per sub-batch
    static constexpr int KS = P / 16;            // k-steps per sub-batch
    static constexpr int FLUSH_SB = 4;           // sub-batches per register -> shared flush (128 points)
    static constexpr int NT = BT / 8;            // n8 tiles
    static constexpr int CAP = P + NTHR;
    static constexpr int RS = BT + 8;            // outer row stride (floats): conflict-free float2 flush
    static constexpr int AXS = P + 8;            // a_x row stride (floats): conflict-free float2 loads
    static constexpr size_t OFF_OUTER = 0;
    static constexpr size_t SZ_OUTER = 256ull * RS * 4;
    static constexpr size_t OFF_KTF = OFF_OUTER + SZ_OUTER;
    static constexpr size_t SZ_KTF = (size_t)KS * NT * 32 * 16;
    static constexpr size_t OFF_AX = OFF_KTF + SZ_KTF;
    static constexpr size_t SZ_AX = (size_t)16 * AXS * 4;
    static constexpr size_t OFF_ROW = OFF_AX + SZ_AX;
    static constexpr size_t SZ_ROW = (size_t)16 * P * 8;
    static constexpr size_t OFF_RING = OFF_ROW + SZ_ROW;
    static constexpr size_t SZ_RING = (size_t)CAP * sizeof(PointRec);
    static constexpr size_t OFF_META = OFF_RING + SZ_RING;
    static constexpr size_t SZ_META = (size_t)P * 4;
    static constexpr size_t OFF_BREC = OFF_META + SZ_META;       // linearised sub-batch
    static constexpr size_t SZ_BREC = (size_t)P * sizeof(PointRec);
    static constexpr size_t OFF_BP = OFF_BREC + SZ_BREC;         // bpx, bpy, bpt [P] each
    static constexpr size_t SZ_BP = (size_t)3 * P * 4;
    static constexpr size_t OFF_SEG = OFF_BP + SZ_BP;
    static constexpr size_t SZ_SEG = (size_t)(2 * MAXSEG + 1) * 4;
    static constexpr size_t OFF_MISC = OFF_SEG + SZ_SEG;
    static constexpr size_t SZ_MISC = 64 * 4;
    static constexpr size_t BYTES = OFF_MISC + SZ_MISC;
};

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }

// Operands are scaled by 2^15 into the FP16 range (|s|, K_t <= 1 -> <= 32768)
// and positive values are clamped up to the smallest normal FP16 (2^-14), so a
// positive product can never flush to zero (the support of the density is
// preserved exactly) while the clamp moves a value by < 2^-29 in true units.
constexpr float MMA_SCALE = 32768.0f;
constexpr float MMA_UNSCALE2 = 1.0f / (32768.0f * 32768.0f);
__device__ __forceinline__ float fp16_range(float v) {
    return v > 0.f ? fmaxf(v * MMA_SCALE, 6.103515625e-05f) : v * MMA_SCALE;
}

// (v0, v1) -> fp16x2 hi and fp16x2 residual lo (inputs already in FP16 range)
__device__ __forceinline__ void split2(float v0, float v1, uint32_t &hi, uint32_t &lo) {
    __half2 h = __floats2half2_rn(v0, v1);
    float2 f = __half22float2(h);
    hi = h2u(h);
    lo = h2u(__floats2half2_rn(v0 - f.x, v1 - f.y));
}

template <int BT, int KK>
__global__ void __launch_bounds__(256, (BT <= 16 ? 3 : 2))
k_tile_mma(const GridParams g, const PointRec *__restrict__ recs, const uint32_t *__restrict__ bucket_begin,
           const int4 *__restrict__ items, const uint64_t *__restrict__ nitems_ptr, int *__restrict__ work_counter,
           uint32_t *__restrict__ arrive, float4 *__restrict__ partials, const int chunk, const int c0,
           const float cscale, float *__restrict__ out, const int64_t t_begin, const int64_t t_end,
           const int vec_ok) {
    using K = CfgM<BT>;
    extern __shared__ __align__(16) unsigned char smem[];
    float *outer = reinterpret_cast<float *>(smem + K::OFF_OUTER);
    uint4 *ktf = reinterpret_cast<uint4 *>(smem + K::OFF_KTF);
    float *axT = reinterpret_cast<float *>(smem + K::OFF_AX);
    float2 *rowT = reinterpret_cast<float2 *>(smem + K::OFF_ROW);
    PointRec *ring = reinterpret_cast<PointRec *>(smem + K::OFF_RING);
    int *meta = reinterpret_cast<int *>(smem + K::OFF_META);
    PointRec *brec = reinterpret_cast<PointRec *>(smem + K::OFF_BREC);
    float *bpx = reinterpret_cast<float *>(smem + K::OFF_BP);
    float *bpy = bpx + K::P;
    float *bpt = bpy + K::P;
    int *seg_start = reinterpret_cast<int *>(smem + K::OFF_SEG);
    int *seg_pref = seg_start + MAXSEG;
    int *misc = reinterpret_cast<int *>(smem + K::OFF_MISC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;         // mma fragment coordinates
    const uint32_t nitems = (uint32_t)(*nitems_ptr);
    const int Ts = (int)(t_end - t_begin);

    if (tid == 0) misc[0] = atomicAdd(work_counter, 1);
    for (;;) {
        __syncthreads();
        const uint32_t it = (uint32_t)misc[0];
        if (it >= nitems) break;
        const int4 item = items[it];
        const int ls = item.x, jchunk = item.y, nch = item.z;
        const int ta = ls % g.NTX, tb = (ls / g.NTX) % g.NTY, tc = ls / (g.NTX * g.NTY) + c0;
        const int tX0 = ta * BX, tY0 = tb * BYW, tT0 = tc * BT;
        const int lt0 = max(0, (int)(t_begin - tT0));
        const int lt1 = min(BT, (int)min((int64_t)g.Gt, t_end) - tT0);
        const int xn = min(BX, g.Gx - tX0), yn = min(BYW, g.Gy - tY0);
        const int gt1 = min(BT, g.Gt - tT0);

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
        bool touched = false;   // the shared accumulator holds data (no zero-fill pass)
        __syncthreads();
        if (tid == 0) {
            misc[0] = atomicAdd(work_counter, 1);   // next item, fetched while this one runs
            int acc = 0;
            seg_pref[0] = 0;
            for (int k = 0; k < nseg; ++k) { acc += seg_pref[k + 1]; seg_pref[k + 1] = acc; }
        }
        __syncthreads();
        const int total = seg_pref[nseg];
        const int cbeg = jchunk * chunk, cend = min(total, cbeg + chunk);
        const float xmax = (float)(xn - 1), ymax = (float)(yn - 1);
        const int Tlo = tT0, Thi = tT0 + gt1 - 1;

        // MMA accumulators live across FLUSH_SB sub-batches; then they are added
        // into the shared tile accumulator [y*16+x][t] (two-level summation).
        float cacc[2][K::NT][4];
        auto zero_acc = [&]() {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < K::NT; ++nt)
#pragma unroll
                    for (int j = 0; j < 4; ++j) cacc[mt][nt][j] = 0.f;
        };
        int pending = 0;
        auto flush = [&]() {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int y = 2 * warp + mt;
#pragma unroll
                for (int nt = 0; nt < K::NT; ++nt) {
                    float2 *o0 = reinterpret_cast<float2 *>(&outer[(y * 16 + gq) * K::RS + 8 * nt + 2 * tq]);
                    float2 *o1 = reinterpret_cast<float2 *>(&outer[(y * 16 + gq + 8) * K::RS + 8 * nt + 2 * tq]);
                    float2 v0 = make_float2(cacc[mt][nt][0], cacc[mt][nt][1]);
                    float2 v1 = make_float2(cacc[mt][nt][2], cacc[mt][nt][3]);
                    if (touched) {       // first flush writes, later ones add
                        const float2 u0 = *o0, u1 = *o1;
                        v0.x += u0.x; v0.y += u0.y;
                        v1.x += u1.x; v1.y += u1.y;
                    }
                    *o0 = v0;
                    *o1 = v1;
                }
            }
            touched = true;
            pending = 0;
            zero_acc();
        };
        zero_acc();
        int head = 0, tail = 0;
        for (int cb = cbeg; cb < cend; cb += K::NTHR) {
            const int i = cb + tid;
            bool acc = false;
            PointRec r;
            if (i < cend) {
                int lo = 0, hi = nseg - 1;
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
                // ---------------- per-point invariants, operand layouts ----------------
                // (1) linearise the sub-batch: tile-local continuous coordinates of
                //     each point (column x is at offset x - px) and its n-tile mask.
                for (int p = tid; p < K::P; p += K::NTHR) {
                    int m = 0;
                    float4 q = make_float4(1e30f, 1e30f, 1e30f, 0.f);      // padding: far away
                    if (p < np) {
                        const PointRec pr = ring[(head + p) % K::CAP];
                        brec[p] = pr;
                        q = make_float4((float)(pr.X - tX0) + pr.fx - 0.5f, (float)(pr.Y - tY0) + pr.fy - 0.5f,
                                        (float)(pr.T - tT0) + pr.ft - 0.5f, 0.f);
                        int lo = max((int)floorf(q.z - g.rt) - 1, lt0);
                        int hi = min((int)ceilf(q.z + g.rt) + 1, lt1 - 1);
                        if (lo <= hi) m = ((2 << (hi >> 3)) - 1) & ~((1 << (lo >> 3)) - 1);
                    }
                    bpx[p] = q.x;
                    bpy[p] = q.y;
                    bpt[p] = q.z;
                    meta[p] = m;
                }
                __syncthreads();
                // (2) K_t in B-fragment order: [k-step][n-tile][lane] = {hi(k0,k0+1), hi(k0+8,k0+9), lo.., lo..}
                for (int e = tid; e < K::KS * K::NT * 32; e += K::NTHR) {
                    const int l = e & 31, nt = (e >> 5) % K::NT, ks = (e >> 5) / K::NT;
                    const float layer = (float)(8 * nt + (l >> 2));
                    const int pb = 16 * ks + 2 * (l & 3);
                    const float2 t01 = *reinterpret_cast<const float2 *>(&bpt[pb]);
                    const float2 t89 = *reinterpret_cast<const float2 *>(&bpt[pb + 8]);
                    const float tp[4] = {t01.x, t01.y, t89.x, t89.y};
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float w = fabsf(layer - tp[j]) * g.inv_rt;
                        float kv;
                        if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - w; kv = 0.75f * (a * a); }
                        else kv = 0.75f * (1.0f - w * w);
                        v[j] = fp16_range((w <= 1.0f) ? kv : 0.0f);
                    }
                    uint4 f;
                    split2(v[0], v[1], f.x, f.z);
                    split2(v[2], v[3], f.y, f.w);
                    ktf[e] = f;
                }
                for (int e = tid; e < 16 * K::P; e += K::NTHR) {           // a_x, transposed [x][p]
                    const int p = e & (K::P - 1), xx = e / K::P;
                    float u = fabsf((float)xx - bpx[p]) * g.inv_rs;
                    float av;
                    if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - u; av = a * a; }
                    else av = MMA_SCALE * (1.0f - u * u);        // additive form: both terms scaled
                    axT[xx * K::AXS + p] = (p < np) ? av : 0.f;
                }
                for (int e = tid; e < 16 * K::P; e += K::NTHR) {           // a_y and the chord, [y][p]
                    const int p = e & (K::P - 1), yy = e / K::P;
                    float ay = 0.f;
                    uint32_t m = 0u;
                    if (p < np) {
                        float v = fabsf((float)yy - bpy[p]) * g.inv_rs;
                        // a_y carries the 2^15 FP16-range scale of the S operand
                        if (KK == STKDE_KERNEL_PRINTED) { float a = 1.0f - v; ay = MMA_SCALE * (a * a); }
                        else ay = -MMA_SCALE * (v * v);
                        if (yy < yn && v < 1.0f + CULL_BAND) m = row_mask16(g, brec[p], tX0, tY0 + yy);
                    }
                    rowT[e] = make_float2(ay, __uint_as_float(m));
                }
                __syncthreads();
                // ---------------- tensor-core accumulation ----------------
#pragma unroll
                for (int ks = 0; ks < K::KS; ++ks) {
                    const int ntm = __reduce_or_sync(0xffffffffu, lane < 16 ? meta[16 * ks + lane] : 0);
                    if (ntm == 0) continue;
                    uint32_t ahi[2][4] = {}, alo[2][4] = {};
                    bool act[2];
                    float4 r01v[2], r89v[2];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        const int y = 2 * warp + mt;
                        r01v[mt] = *reinterpret_cast<const float4 *>(&rowT[y * K::P + 16 * ks + 2 * tq]);
                        r89v[mt] = *reinterpret_cast<const float4 *>(&rowT[y * K::P + 16 * ks + 2 * tq + 8]);
                        act[mt] = __any_sync(0xffffffffu, (__float_as_uint(r01v[mt].y) | __float_as_uint(r01v[mt].w) |
                                                           __float_as_uint(r89v[mt].y) | __float_as_uint(r89v[mt].w)) != 0u);
                    }
                    if (!act[0] && !act[1]) continue;
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        if (!act[mt]) continue;            // row misses all 16 discs: no A fragment
                        const float4 r01 = r01v[mt], r89 = r89v[mt];
                        const uint32_t m0 = __float_as_uint(r01.y), m1 = __float_as_uint(r01.w);
                        const uint32_t m8 = __float_as_uint(r89.y), m9 = __float_as_uint(r89.w);
                        const float2 ag01 = *reinterpret_cast<const float2 *>(&axT[gq * K::AXS + 16 * ks + 2 * tq]);
                        const float2 ag89 = *reinterpret_cast<const float2 *>(&axT[gq * K::AXS + 16 * ks + 2 * tq + 8]);
                        const float2 aG01 = *reinterpret_cast<const float2 *>(&axT[(gq + 8) * K::AXS + 16 * ks + 2 * tq]);
                        const float2 aG89 = *reinterpret_cast<const float2 *>(&axT[(gq + 8) * K::AXS + 16 * ks + 2 * tq + 8]);
                        const uint32_t bg = 1u << gq, bG = 1u << (gq + 8);
                        // s = mask ? K_s (scaled, > 0 inside the disc, clamped to the
                        // smallest normal FP16) : 0
                        auto ks_ = [](float a, float b) {
                            return KK == STKDE_KERNEL_PRINTED ? a * b : a + b;
                        };
                        constexpr float TINY = 6.103515625e-05f;
                        float s[8];
                        s[0] = (m0 & bg) ? fmaxf(ks_(ag01.x, r01.x), TINY) : 0.f;   // row x=g,   k=2t
                        s[1] = (m1 & bg) ? fmaxf(ks_(ag01.y, r01.z), TINY) : 0.f;   // row x=g,   k=2t+1
                        s[2] = (m0 & bG) ? fmaxf(ks_(aG01.x, r01.x), TINY) : 0.f;   // row x=g+8, k=2t
                        s[3] = (m1 & bG) ? fmaxf(ks_(aG01.y, r01.z), TINY) : 0.f;
                        s[4] = (m8 & bg) ? fmaxf(ks_(ag89.x, r89.x), TINY) : 0.f;   // row x=g,   k=2t+8
                        s[5] = (m9 & bg) ? fmaxf(ks_(ag89.y, r89.z), TINY) : 0.f;
                        s[6] = (m8 & bG) ? fmaxf(ks_(aG89.x, r89.x), TINY) : 0.f;   // row x=g+8, k=2t+8
                        s[7] = (m9 & bG) ? fmaxf(ks_(aG89.y, r89.z), TINY) : 0.f;
                        split2(s[0], s[1], ahi[mt][0], alo[mt][0]);
                        split2(s[2], s[3], ahi[mt][1], alo[mt][1]);
                        split2(s[4], s[5], ahi[mt][2], alo[mt][2]);
                        split2(s[6], s[7], ahi[mt][3], alo[mt][3]);
                    }
#pragma unroll
                    for (int nt = 0; nt < K::NT; ++nt) {
                        if (!((ntm >> nt) & 1)) continue;
                        const uint4 b = ktf[(ks * K::NT + nt) * 32 + lane];
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) {
                            if (!act[mt]) continue;
                            mma16816(cacc[mt][nt], ahi[mt], b.x, b.y);
                            mma16816(cacc[mt][nt], ahi[mt], b.z, b.w);
                            mma16816(cacc[mt][nt], alo[mt], b.x, b.y);
                        }
                    }
                }
                if (++pending == K::FLUSH_SB) flush();
                head += np;
                __syncthreads();
            }
        }
        if (pending) {
            flush();
            __syncthreads();
        }

        // ---------------- store: every voxel exactly once ----------------
        // f enumerates the tile as [col'][t4] with col' = y*16 + x; values are
        // scaled by the kernel constant and 1/(n hs^2 ht) here.
        auto store4 = [&](int col, int q, float4 v) {
            const int x = col & 15, y = col >> 4;
            if (x >= xn || y >= yn) return;
            v.x *= cscale; v.y *= cscale; v.z *= cscale; v.w *= cscale;
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
        constexpr int BT4 = BT / 4;
        constexpr int NF = 256 * BT4;
        const float4 *outer4 = reinterpret_cast<const float4 *>(outer);
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (nch == 1) {
            for (int f = tid; f < NF; f += K::NTHR) {
                int col = f / BT4, q = f - col * BT4;
                store4(col, q, touched ? outer4[col * (K::RS / 4) + q] : zero4);
            }
        } else {
            const int slot0 = item.w;
            float4 *mine = partials + (size_t)(slot0 + jchunk) * NF;
            for (int f = tid; f < NF; f += K::NTHR) {
                int col = f / BT4, q = f - col * BT4;
                mine[f] = touched ? outer4[col * (K::RS / 4) + q] : zero4;
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
                    int col = f / BT4, q = f - col * BT4;
                    store4(col, q, v);
                }
                if (tid == 0) arrive[ls] = 0u;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ dispatch ---
typedef void (*tile_mma_fn)(const GridParams, const PointRec *, const uint32_t *, const int4 *, const uint64_t *,
                            int *, uint32_t *, float4 *, int, int, float, float *, int64_t, int64_t, int);

static tile_mma_fn select_mma(int BT, int KK) {
#define STKDE_SELM(bt) \
    if (BT == bt) return KK ? (tile_mma_fn)k_tile_mma<bt, 1> : (tile_mma_fn)k_tile_mma<bt, 0>;
    STKDE_SELM(16) STKDE_SELM(32) STKDE_SELM(64)
#undef STKDE_SELM
    return nullptr;
}

size_t tile_mma_smem_bytes(int BT) {
    switch (BT) {
        case 16: return CfgM<16>::BYTES;
        case 32: return CfgM<32>::BYTES;
        case 64: return CfgM<64>::BYTES;
    }
    return 0;
}

int tile_mma_occupancy(int BT, int KK, int *ctas_per_sm) {
    tile_mma_fn f = select_mma(BT, KK);
    if (!f) return STKDE_EINVAL;
    size_t smem = tile_mma_smem_bytes(BT);
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return STKDE_ECUDA;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 256, smem) != cudaSuccess) return STKDE_ECUDA;
    *ctas_per_sm = occ;
    return STKDE_OK;
}

int launch_tile_mma(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cscale, float *out,
                    cudaStream_t st) {
    const GridParams &g = p->g;
    tile_mma_fn f = select_mma(g.BT, p->kernel);
    if (!f) return STKDE_EINVAL;
    const int nsl = g.NTX * g.NTY * (c1 - c0);
    const int64_t Ts = t_end - t_begin;
    const int vec_ok = (Ts % 4 == 0) && (t_begin % 4 == 0) && ((uintptr_t)out % 16 == 0);
    unsigned grid = (unsigned)std::min<int64_t>((int64_t)p->num_sms * p->ctas_per_sm, p->max_items);
    if (!p->wc_zeroed) cudaMemsetAsync(p->counters, 0, sizeof(int), st);   // (else by k_worklist_small)
    p->wc_zeroed = 0;
    const bool timed = p->timing && p->tev_used < p->tev_cap;
    if (timed) cudaEventRecord(p->tev[2 * p->tev_used], st);
    f<<<grid, 256, p->smem_bytes, st>>>(g, p->rec_sorted, p->bucket_begin, p->items, p->chunk_off + nsl, p->counters,
                                        p->arrive, reinterpret_cast<float4 *>(p->partials), p->chunk, c0,
                                        cscale * MMA_UNSCALE2,
                                        out, t_begin, t_end, vec_ok);
    if (timed) {
        cudaEventRecord(p->tev[2 * p->tev_used + 1], st);
        p->tev_used += 1;
    }
    p->last_own_launches += 1;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

}  // namespace stkde
