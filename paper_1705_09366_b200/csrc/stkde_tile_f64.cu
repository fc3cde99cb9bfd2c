// stkde_tile_f64.cu -- the FP64-output option.
//
// A gather-form voxel-tile kernel that evaluates every (point, voxel) term in
// FP64 with the IEEE operation sequence of Alg. 1 and the
// printed / classical kernels, and writes an FP64 grid
// (SPEC.md:48-54 keeps its volume in FP64).  Per pair, with no contraction
// (__d*_rn intrinsics):
//
//   x = x0 + (X + 0.5) sres          (voxel centre, reading R5)
//   dx = x - x_i, dy = y - y_i, d = sqrt(dx*dx + dy*dy);   inside iff d < hs      (strict)
//   dt = |t - t_i|;                                      inside iff dt <= ht     (inclusive)
//   k_s(|dx|/hs, |dy|/hs) * k_t(dt/ht)
//
// so each gate decision and each factor k_s, k_t is the same double as in a plain
// FP64 evaluation of the definition.  The per-voxel sum is acc = fma(k_s, k_t, acc)
// (one rounding per term instead of the product's and the sum's) in a fixed order
// (home-bucket order, ascending point index inside a bucket), hence results agree
// with an FP64 reference to (2m - 1) 2^-53 f for m terms, and the support (f > 0)
// agrees exactly.  The sum is divided by n hs^2 ht at the end (adaptive: k_s is
// divided by hs_i^2 ht_i first, the sum by n; reading R15).
//
// Layout: one CTA per (16 x BY columns, TL layers) of the slab, TL = 32 when H_t >= 16
// else 16; one thread per column accumulating its TL layers in registers (the FP64 gate and k_s once per
// (point, column)).  Candidates are the plan's home buckets within reach (the
// binning of stkde_binning.cu), staged 64 at a time; those whose box
// X_i +- H_s, Y_i +- H_s, T_i +- H_t misses the CTA's block are dropped by an
// order-preserving (ballot) compaction, the rest get their temporal line K_t[32] in
// shared memory (the PB-SYM separation,
// Alg. 3: k_t formed once per (point, layer), reused by every
// column).  The loop is FP64-pipe bound.
#include "stkde_internal.cuh"

namespace stkde {

namespace {

constexpr int F64_CH = 64;       // candidates staged per round
constexpr double PI_D = 3.14159265358979323846;

struct F64Cand {
    double px, py, pt;       // the point's FP32 coordinates, widened exactly
    double hs, ht, dn;       // its bandwidths; dn = hs*hs*ht (adaptive)
    double hs2;              // hs*hs (gate pre-test)
    int X, Y;                // its voxel column
    int cmask;               // bit q: some K_t of layers [8q, 8q + 8) of the block is non-zero
    int pad;
};

__device__ __forceinline__ double kt_f64(int kernel, double w) {
    if (kernel == STKDE_KERNEL_CLASSICAL) return __dmul_rn(0.75, __dsub_rn(1.0, __dmul_rn(w, w)));
    const double a = __dsub_rn(1.0, w);
    return __dmul_rn(0.75, __dmul_rn(a, a));
}

__device__ __forceinline__ double ks_f64(int kernel, double u, double v) {
    if (kernel == STKDE_KERNEL_CLASSICAL)
        return __dmul_rn(2.0 / PI_D, __dsub_rn(__dsub_rn(1.0, __dmul_rn(u, u)), __dmul_rn(v, v)));
    const double a = __dsub_rn(1.0, u), b = __dsub_rn(1.0, v);
    return __dmul_rn(__dmul_rn(PI_D / 2.0, __dmul_rn(a, a)), __dmul_rn(b, b));
}

}  // namespace

template <bool AD, int TL>
__global__ void __launch_bounds__(256) k_tile_f64(GridParams g, const PointRec *__restrict__ rec,
                                                   const uint32_t *__restrict__ vals,
                                                   const uint32_t *__restrict__ bucket_begin,
                                                   const float *__restrict__ pts, const float *__restrict__ bw,
                                                   int t_begin, int t_end, double den, double *__restrict__ out) {
    __shared__ F64Cand cand[F64_CH];
    __shared__ double ktab[F64_CH][TL];
    __shared__ uint32_t keep_bal[F64_CH / 32];

    const int tid = threadIdx.x, nthr = blockDim.x;     // one thread per column (BX x BY)
    const int col = tid;
    const int lane = tid & 31;
    const int a = blockIdx.x, b = blockIdx.y;
    const int X = a * BX + col / g.BY, Y = b * g.BY + col % g.BY;
    const int T0 = t_begin + (int)blockIdx.z * TL;  // first layer of the CTA
    const int Ts = t_end - t_begin;
    // this column's voxel centre, as Alg. 1 forms it
    const double cxv = __dadd_rn(g.x0, __dmul_rn(__dadd_rn((double)X, 0.5), g.sres));
    const double cyv = __dadd_rn(g.y0, __dmul_rn(__dadd_rn((double)Y, 0.5), g.sres));

    double acc[TL];
#pragma unroll
    for (int k = 0; k < TL; ++k) acc[k] = 0.0;
    // the CTA's block: columns [xa, xb] x [ya, yb], layers [T0, tl]

    // candidate home buckets: x tiles a +- Ra, y tiles b +- Ray, T buckets whose points'
    // windows [T_i - H_t, T_i + H_t] can meet layers [T0, T0 + TL)
    const int a0 = max(a - g.Ra, 0), a1 = min(a + g.Ra, g.NTX - 1);
    const int b0 = max(b - g.Ray, 0), b1 = min(b + g.Ray, g.NTY - 1);
    const int tl = min(T0 + TL, t_end) - 1;
    const int xa = a * BX, xb = xa + BX - 1, ya = b * g.BY, yb = ya + g.BY - 1;
    const int c0 = max(floordiv(T0 - g.Ht, g.BTH), 0), c1 = min(floordiv(tl + g.Ht, g.BTH), g.NTTH - 1);

    for (int cc = c0; cc <= c1; ++cc)
        for (int bb = b0; bb <= b1; ++bb) {
            const int k0 = (cc * g.NTY + bb) * g.NTX;
            const uint32_t s0 = bucket_begin[k0 + a0], s1 = bucket_begin[k0 + a1 + 1];
            for (uint32_t s = s0; s < s1; s += F64_CH) {
                const int craw = (int)min((uint32_t)F64_CH, s1 - s);
                __syncthreads();   // previous round's readers are done
                // keep the candidates whose box reaches the block; compact them in input order
                bool keep = false;
                PointRec r;
                if (tid < craw) {
                    r = rec[s + tid];
                    keep = r.X + g.Hs >= xa && r.X - g.Hs <= xb && r.Y + g.Hs >= ya && r.Y - g.Hs <= yb &&
                           r.T + g.Ht >= T0 && r.T - g.Ht <= tl;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (tid < F64_CH && lane == 0) keep_bal[tid >> 5] = bal;
                __syncthreads();
                int cnt = 0, pos = 0;
#pragma unroll
                for (int w = 0; w < F64_CH / 32; ++w) {
                    if (w == (tid >> 5)) pos = cnt + __popc(bal & ((1u << lane) - 1u));
                    cnt += __popc(keep_bal[w]);
                }
                if (keep) {
                    const uint32_t idx = vals[s + tid];
                    F64Cand c;
                    c.px = (double)pts[3 * (size_t)idx];
                    c.py = (double)pts[3 * (size_t)idx + 1];
                    c.pt = (double)pts[3 * (size_t)idx + 2];
                    if (AD) {
                        c.hs = (double)bw[2 * (size_t)idx];
                        c.ht = (double)bw[2 * (size_t)idx + 1];
                    } else {
                        c.hs = g.hs;
                        c.ht = g.ht;
                    }
                    c.hs2 = __dmul_rn(c.hs, c.hs);
                    c.dn = __dmul_rn(c.hs2, c.ht);
                    c.X = r.X;
                    c.Y = r.Y;
                    c.cmask = 0;
                    c.pad = 0;
                    cand[pos] = c;
                }
                if (cnt == 0) continue;   // CTA-uniform
                __syncthreads();
                // temporal lines: K_t of (candidate j, layer T0 + l), 0 outside the gate or the slab
                for (int e = tid; e < cnt * TL; e += nthr) {
                    const int j = e / TL, l = e % TL;
                    const int T = T0 + l;
                    double kt = 0.0;
                    if (T < t_end) {
                        const double ct = __dadd_rn(g.t0, __dmul_rn(__dadd_rn((double)T, 0.5), g.tres));
                        const double dt = fabs(__dsub_rn(ct, cand[j].pt));
                        if (dt <= cand[j].ht) kt = kt_f64(g.kernel, __ddiv_rn(dt, cand[j].ht));
                    }
                    ktab[j][l] = kt;
                    if (kt != 0.0) atomicOr(&cand[j].cmask, 1 << (l >> 3));
                }
                __syncthreads();
                for (int j = 0; j < cnt; ++j) {
                    const int cm = cand[j].cmask;                   // CTA-uniform
                    if (cm == 0) continue;
                    if (abs(X - cand[j].X) > g.Hs || abs(Y - cand[j].Y) > g.Hs) continue;
                    const double hs = cand[j].hs;
                    const double dx = __dsub_rn(cxv, cand[j].px), dy = __dsub_rn(cyv, cand[j].py);
                    const double q = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                    // Alg. 1 spatial gate sqrt(q) < hs (strict): decided by q vs hs^2 outside a
                    // 1e-12 band (>> the 3 roundings of q, hs^2 and the band), else by the sqrt
                    const double hs2 = cand[j].hs2;
                    if (q > __dmul_rn(hs2, 1.0 + 1e-12)) continue;
                    if (!(q < __dmul_rn(hs2, 1.0 - 1e-12)) && !(__dsqrt_rn(q) < hs)) continue;
                    double ks = ks_f64(g.kernel, __ddiv_rn(fabs(dx), hs), __ddiv_rn(fabs(dy), hs));
                    if (AD) ks = __ddiv_rn(ks, cand[j].dn);        // the term's 1/(hs_i^2 ht_i)
                    const double2 *kt = reinterpret_cast<const double2 *>(ktab[j]);
                    // acc += k_s k_t with one rounding (zero terms outside the window leave acc unchanged)
#pragma unroll
                    for (int qq = 0; qq < TL / 8; ++qq)
                        if ((cm >> qq) & 1) {
#pragma unroll
                            for (int k = 4 * qq; k < 4 * qq + 4; ++k) {
                                const double2 v = kt[k];
                                acc[2 * k] = __fma_rn(ks, v.x, acc[2 * k]);
                                acc[2 * k + 1] = __fma_rn(ks, v.y, acc[2 * k + 1]);
                            }
                        }
                }
            }
        }

    if (X < g.Gx && Y < g.Gy) {
        double *o = out + ((int64_t)X * g.Gy + Y) * Ts + (T0 - t_begin);
        const int nv = min(TL, t_end - T0);
        if (nv == TL && ((uintptr_t)o & 15) == 0) {
#pragma unroll
            for (int k = 0; k < TL; k += 2)
                *reinterpret_cast<double2 *>(o + k) = make_double2(__ddiv_rn(acc[k], den), __ddiv_rn(acc[k + 1], den));
        } else {
#pragma unroll
            for (int k = 0; k < TL; ++k)
                if (k < nv) o[k] = __ddiv_rn(acc[k], den);
        }
    }
}

int launch_tile_f64(stkde_plan_s *p, const float *d_points, const float *d_bw, int64_t t_begin, int64_t t_end,
                    double den, double *out, cudaStream_t st) {
    const GridParams &g = p->g;
    const int ncol = BX * g.BY;   // threads per CTA: 128 (tcgen05 binning) or 256
    // layers per CTA: 32 for deep windows (the gate and k_s amortised over more layers),
    // 16 otherwise (half the accumulators: 80 instead of 122 registers, 1.5x the warps)
    const int TL = g.Ht >= 16 ? 32 : 16;
    const int64_t nz = (t_end - t_begin + TL - 1) / TL;
    if (nz > 65535) { set_error("FP64 slab too deep (%lld layers)", (long long)(t_end - t_begin)); return STKDE_EINVAL; }
    const dim3 grid((unsigned)g.NTX, (unsigned)g.NTY, (unsigned)nz);
    const bool timed = p->timing && p->tev_used < p->tev_cap;
    if (timed) cudaEventRecord(p->tev[2 * p->tev_used], st);
    auto f = d_bw ? (TL == 32 ? k_tile_f64<true, 32> : k_tile_f64<true, 16>)
                  : (TL == 32 ? k_tile_f64<false, 32> : k_tile_f64<false, 16>);
    f<<<grid, ncol, 0, st>>>(g, p->rec_sorted, p->vals_out, p->bucket_begin, d_points, d_bw, (int)t_begin,
                             (int)t_end, den, out);
    if (timed) {
        cudaEventRecord(p->tev[2 * p->tev_used + 1], st);
        p->tev_used += 1;
    }
    p->last_own_launches += 1;
    return cudaGetLastError() == cudaSuccess ? STKDE_OK : STKDE_ECUDA;
}

}  // namespace stkde
