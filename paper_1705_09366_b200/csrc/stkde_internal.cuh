// stkde_internal.cuh -- plan layout, kernel parameters and the device-side
// geometry helpers (voxel mapping, exact gates, per-row disc chords) of the
// B200 STKDE library.  Nothing here is shared with oracle/.
//
// Paper references (PAPER.md = /root/reference/PAPER.md):
//   density and kernels     PAPER.md:120-133 (§2.1)
//   gates                   Alg. 1, PAPER.md:208 (spatial strict, temporal inclusive)
//   grid / H
//   PB-SYM separability     Alg. 3; Fig. 3
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stkde.h"

namespace stkde {

constexpr int BX = 16;            // tile width in X (voxels), all engines
constexpr int BYW = 16;           // tile width in Y of the SIMT / mma.sync engines (g.BY = 8 for tcgen05)
constexpr int MAXSEG = 256;       // max home-bucket segments per tile
// Relative band around the disc edge inside which the FP32 gate defers to
// the exact FP64 expression (reading R13): |d^2 - r^2| <= BAND r^2.
// The FP32 voxel-local d^2 is within ~3e-7 (relative) of the FP64 value, so
// 4e-6 leaves a >10x margin while keeping FP64 evaluations rare.
constexpr float GATE_BAND = 4e-6f;
// Conservative margin of the tile acceptance test (culling only).
constexpr float CULL_BAND = 1e-4f;

// Per-point record written by the prep kernel (32 B, one per input point).
//   X, Y, T     voxel of the point: floor((x - x0)/sres) ...
//   fx, fy, ft  fractional position inside that voxel, in voxel units, [0,1)
//   x, y        the original FP32 world coordinates (for the FP64 gate)
struct __align__(16) PointRec {
    int X, Y, T;
    float fx, fy, ft;
    float x, y;
};

// Per-point bandwidths of the adaptive estimator (reading R15), one per
// record: hs_i, ht_i as given (world units, exact FP64 gates) and the voxel-unit
// reciprocals sres/hs_i, tres/ht_i of the FP32 tables.
struct __align__(16) PointBw {
    float hs, ht;
    float inv_rs, inv_rt;
};

// Kernel-side view of a plan (passed by value).
struct GridParams {
    double x0, y0, t0;      // origin (world)
    double sres, tres;      // voxel sizes (world)
    double hs, ht;          // bandwidths (world)
    float rs, rt;           // hs/sres, ht/tres (voxel units)
    float rs2;              // rs*rs
    float inv_rs, inv_rt;   // sres/hs, tres/ht
    int Gx, Gy, Gt;         // grid (voxels)
    int Hs, Ht;             // ceil(hs/sres), ceil(ht/tres)
    int NTX, NTY, NTT;      // tiles per axis
    int BY, BT;             // tile width in Y (columns), tile height (layers)
    int BTH, NTTH;          // home-bucket depth in T (layers; BT for the legacy engines) and count
    int Ra, Ray, Rt;        // home-bucket reach in tiles: ceil(Hs/BX), ceil(Hs/BY), ceil(Ht/BT)
    int XA0, NXA;           // x-tile window of the current launch: tiles [XA0, XA0 + NXA) (x-slabs;
                            // the whole grid otherwise)
    int kernel;             // STKDE_KERNEL_*
};

// rows of a point's chord table (tcgen05 engine): the 8-aligned row blocks that
// cover [Y_i - H_s, Y_i + H_s] for any Y_i
__host__ __device__ inline int chord_rows(int Hs) { return ((2 * Hs + 1 + 7) / 8 + 1) * 8; }

// The plan's GridParams with the spatial bandwidth of one point (adaptive chords,
// gates and counts): everything the exact gates read, nothing the binning reads.
__host__ __device__ inline GridParams with_point_bw(const GridParams &g, const PointBw &b) {
    GridParams gi = g;
    gi.hs = (double)b.hs;
    gi.ht = (double)b.ht;
    const double rs = (double)b.hs / g.sres;
    gi.rs = (float)rs;
    gi.rs2 = (float)(rs * rs);
    gi.rt = (float)((double)b.ht / g.tres);
    gi.inv_rs = b.inv_rs;
    gi.inv_rt = b.inv_rt;
    return gi;
}

__host__ __device__ inline int floordiv(int a, int b) {
    int q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// Home T-blocks whose points can reach work-tile layer block c: the windows
// [T_i - H_t, T_i + H_t] meet [c BT, c BT + BT - 1] iff T_i is in
// [c BT - H_t, c BT + BT - 1 + H_t] (Alg. 2/3 loop bounds).
__host__ __device__ inline void home_t_range(const GridParams &g, int c, int *cc0, int *cc1) {
    const int t0 = c * g.BT;
    *cc0 = max(floordiv(t0 - g.Ht, g.BTH), 0);
    *cc1 = min(floordiv(t0 + g.BT - 1 + g.Ht, g.BTH), g.NTTH - 1);
}

// ---- exact FP64 gates: the same IEEE expression sequence as Alg. 1 ----
// x = x0 + (X + 0.5) sres (voxel centre), dx = x - x_i,
// inside iff sqrt(dx*dx + dy*dy) < hs.  No contraction: __dmul_rn/__dadd_rn.
__device__ __forceinline__ bool gate_s_fp64(const GridParams &g, int X, int Y, float px, float py) {
    double cx = __dadd_rn(g.x0, __dmul_rn(__dadd_rn((double)X, 0.5), g.sres));
    double cy = __dadd_rn(g.y0, __dmul_rn(__dadd_rn((double)Y, 0.5), g.sres));
    double dx = __dsub_rn(cx, (double)px);
    double dy = __dsub_rn(cy, (double)py);
    double d = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    return d < g.hs;
}
// |t - t_i| <= ht with t = t0 + (T + 0.5) tres.
__device__ __forceinline__ bool gate_t_fp64(const GridParams &g, int T, float pt) {
    double ct = __dadd_rn(g.t0, __dmul_rn(__dadd_rn((double)T, 0.5), g.tres));
    return fabs(__dsub_rn(ct, (double)pt)) <= g.ht;
}

// Spatial gate of column X in a row whose FP32 offset^2 is dy2 (voxel units):
// FP32 unless |d^2 - r^2| is within the band, then the exact FP64 gate.
__device__ __forceinline__ bool gate_s(const GridParams &g, const PointRec &r, int X, int Y, float dy2) {
    float dxv = (float)(X - r.X) + 0.5f - r.fx;
    float d2 = __fadd_rn(__fmul_rn(dxv, dxv), dy2);
    float diff = d2 - g.rs2;
    if (fabsf(diff) > GATE_BAND * g.rs2) return diff < 0.0f;
    return gate_s_fp64(g, X, Y, r.x, r.y);
}

// Exact chord of the disc of point r on row Y: the global column interval
// [*lo, *hi] whose voxel centres pass the spatial gate (empty: *lo > *hi).
// The in-set of a row is an interval because the FP64 gate is monotone in
// |X + 0.5 - p|; the FP32 estimate is within one column of each end and is
// corrected with the exact gate.
__device__ __forceinline__ void row_chord(const GridParams &g, const PointRec &r, int Y, int *lo, int *hi) {
    float dyv = (float)(Y - r.Y) + 0.5f - r.fy;
    float dy2 = __fmul_rn(dyv, dyv);
    if (dy2 > g.rs2 * (1.0f + GATE_BAND) || !gate_s(g, r, r.X, Y, dy2)) {
        *lo = 1; *hi = 0;
        return;
    }
    float c = sqrtf(fmaxf(g.rs2 - dy2, 0.0f));
    float pc = (float)r.X + r.fx - 0.5f;            // column coordinate of the point
    int a = (int)floorf(pc - c) + 1, b = (int)ceilf(pc + c) - 1;
    a = min(a, r.X);
    b = max(b, r.X);
    while (a < r.X && !gate_s(g, r, a, Y, dy2)) ++a;
    while (gate_s(g, r, a - 1, Y, dy2)) --a;
    while (b > r.X && !gate_s(g, r, b, Y, dy2)) --b;
    while (gate_s(g, r, b + 1, Y, dy2)) ++b;
    *lo = a;
    *hi = b;
}

// Row mask of the 16 tile columns [tX0, tX0+16) inside the disc on row Y.
__device__ __forceinline__ uint32_t row_mask16(const GridParams &g, const PointRec &r, int tX0, int Y) {
    float dyv = (float)(Y - r.Y) + 0.5f - r.fy;
    float dy2 = __fmul_rn(dyv, dyv);
    // quick accept / reject from the two tile-edge columns and the nearest column
    float p = (float)(r.X - tX0) + r.fx - 0.5f;     // point in tile-local column coordinates
    float e0 = p, e1 = 15.0f - p;                     // distances to the edge columns
    float far = fmaxf(fabsf(e0), fabsf(e1));
    if (__fadd_rn(__fmul_rn(far, far), dy2) < g.rs2 * (1.0f - GATE_BAND)) return 0xFFFFu;
    float nearx = fminf(fmaxf(p, 0.0f), 15.0f) - p;
    if (__fadd_rn(__fmul_rn(nearx, nearx), dy2) > g.rs2 * (1.0f + GATE_BAND)) return 0u;
    int lo, hi;
    row_chord(g, r, Y, &lo, &hi);
    lo = max(lo - tX0, 0);
    hi = min(hi - tX0, 15);
    if (lo > hi) return 0u;
    return ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

}  // namespace stkde

// ------------------------------------------------------------------ plan ---
struct stkde_plan_s {
    int device;
    int num_sms;
    stkde::GridParams g;
    int kernel;
    int CT;                   // layers per thread of the tile kernel (4 columns x CT)
    int engine;               // STKDE_ENGINE_*: 0 = FP32 FFMA2 (SIMT), 1 = mma.sync 3xFP16, 2 = tcgen05 kind::i8,
                              // 3 = short-window FP32 (WS)
    int tile_threads;
    int ctas_per_sm;
    int64_t max_n;
    int64_t ntiles;           // NTX*NTY*NTT (global work tiles)
    int64_t nbuckets;         // NTX*NTY*NTTH (home buckets)
    int key_bits;             // radix bits of the home-bucket keys
    int chunk;                // candidates per work item
    int64_t max_items;
    int64_t max_slots;        // split-tile partial slots
    size_t smem_bytes;

    // workspace
    void *ws;
    size_t ws_bytes;
    stkde::PointRec *rec, *rec_sorted;
    uint16_t *chords;           // tcgen05 engine: [max_n][chord_rows(Hs)] exact disc chords (int8 lo, hi - X_i)
    int ridx_in_rec;            // rec_sorted[j].x holds j (the fused scatter + chord pass), else world x
    stkde::PointBw *bw_rec, *bw_sorted;   // tcgen05 engine: per-point bandwidths of an adaptive call
    const float *d_bw;          // the current call's per-point bandwidths [n][2] (NULL: fixed bandwidth)
    uint32_t *keys_in, *keys_out, *vals_in, *vals_out;
    uint32_t *bucket_cnt;       // [ntiles + 1]
    uint32_t *bucket_begin;     // [ntiles + 2]
    uint32_t *lpt_key_in, *lpt_key_out, *lpt_val_in, *lpt_val_out;   // [ntiles]
    uint32_t *tile_cnt;         // [ntiles] candidate count per slab tile
    int order;                  // work-list order: 0 = LPT, 1 = heavy tiles by LPT, then locality, -1 = by size
    int heavy;                  // candidates from which a tile counts as heavy (order 1)
    int wl_small;               // STKDE_WL_SMALL (default 1): one-CTA work list for small slabs
    int wc_zeroed;              // the next tile launch's item counter was zeroed by k_worklist_small
    uint64_t *chunk_pack, *chunk_off;   // [ntiles + 1]
    int4 *items;                // [max_items]
    uint32_t *arrive;           // [ntiles]
    float *partials;            // [max_slots][256*BT]
    int *counters;              // [0] work counter, [1] error flag, [2..3] u64 issued MMA columns,
                                // [4..5] u64 issued k-blocks (tcgen05 engine instrumentation),
                                // [6] adaptive call: max_i (sres/hs_i)^2 (tres/ht_i) as float bits,
                                // [32..95] u64 [32] tcgen05 phase profile (stkde_plan_tc_profile)
    int tc_profile;             // STKDE_TC_PROF: record the tcgen05 kernel's phase profile
    int tc_watchdog;            // STKDE_TC_WATCHDOG: bounded mbarrier waits, record in counters[96..97]
    int no_tma;                 // STKDE_NO_TMA: epilogue stores by per-column bulk copies instead of TMA
    int out_remote;             // the current call's output lives on another device (peer / IPC): plain stores
    int plain_stores;           // STKDE_PLAIN_STORES: x-slab outputs always take the peer-output store path (tests)
    void *debug_progress;       // stkde_plan_debug_progress: per-(CTA, warp) protocol state (host-mapped)
    int *hist_t;                // [Gt + 1] slab-partition histogram
    int *hist_x;                // [Gx + 1] x-slab-partition histogram
    void *cub_tmp;
    size_t cub_bytes;

    // instrumentation
    int timing;
    cudaEvent_t *tev;         // [2 * tev_cap] start/stop pairs around tile launches
    int tev_cap, tev_used;
    double kernel_ms;
    int64_t kernel_launches;
    int last_own_launches, last_cub_calls;
    // per-phase timing (stkde_plan_enable_phase_timing): events recorded at phase ends on the
    // caller's stream, ph_id[k] = phase that ends at ph_ev[k] (-1: start of a call)
    int ph_on;
    cudaEvent_t *ph_ev;
    int8_t *ph_id;
    int ph_cap, ph_used;
    double ph_ms[STKDE_NPHASES];
    int64_t ph_calls;

    // NCCL communicator of the per-rank gather (stkde_plan_comm_init; NULL until then)
    void *comm;
    int comm_rank, comm_nranks;
    float *gather_stage;        // root's staging of the time-slab gather (lazily allocated)
    size_t gather_stage_bytes;
};

namespace stkde {
// launchers (stkde_binning.cu / stkde_tile.cu)
// bins the points whose window reaches layers [t_begin, t_end) (the slab being computed)
// (tcgen05 engine: counting-sort scatter unless `stable` (radix sort: each bucket in input
// order); with_chords also writes the chord table in the same pass)
int launch_binning(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st, int64_t t_begin,
                   int64_t t_end, bool with_chords = false, bool stable = false);
// (xy != NULL: the sweep's saved world coordinates; the records' x then carries the sorted index)
int launch_chords(stkde_plan_s *p, int64_t n, cudaStream_t st, const float2 *xy = nullptr);
int launch_save_xy(stkde_plan_s *p, int64_t n, float2 *xy, cudaStream_t st);
int launch_worklist(stkde_plan_s *p, int c0, int c1, cudaStream_t st);
int launch_tile_cost(stkde_plan_s *p, int nsl, cudaStream_t st);
int launch_tile(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float norm,
                float *out, cudaStream_t st);
int launch_count(stkde_plan_s *p, const float *d_points, int64_t n, int64_t t_begin,
                 int64_t t_end, int64_t *d_count, cudaStream_t st, const float *d_bw, int64_t x_begin,
                 int64_t x_end);
int launch_hist_t(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st);
int launch_hist_x(stkde_plan_s *p, const float *d_points, int64_t n, cudaStream_t st);
int launch_gather(const float *slab, int64_t Gx, int64_t Gy, int64_t Gt, int64_t t0, int64_t t1,
                  float *full, cudaStream_t st);
size_t tile_smem_bytes(int BT, int CT);
int tile_occupancy(int BT, int CT, int kernel, int *ctas_per_sm);
int tile_threads(int BT, int CT);
size_t tile_mma_smem_bytes(int BT);
int tile_mma_occupancy(int BT, int kernel, int *ctas_per_sm);
int launch_tile_mma(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cscale, float *out,
                    cudaStream_t st);
size_t tile_tc_smem_bytes(int BT);
int tile_tc_occupancy(int BT, int kernel, int *ctas_per_sm);
int launch_tile_tc(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cscale, float *out,
                   cudaStream_t st);
size_t tile_ws_smem_bytes(int Ht);
int tile_ws_occupancy(int Ht, int KK, size_t smem, int *ctas_per_sm);
int launch_tile_ws(stkde_plan_s *p, int c0, int c1, int64_t t_begin, int64_t t_end, float cscale, float *out,
                   cudaStream_t st);
int launch_tile_f64(stkde_plan_s *p, const float *d_points, const float *d_bw, int64_t t_begin, int64_t t_end,
                    double den, double *out, cudaStream_t st);
void set_error(const char *fmt, ...);
// phase timing + NVTX ranges (stkde_trace_comm.cu): phase_call_begin marks the start of a
// call on `st`; phase_begin opens the NVTX range of phase `ph`, phase_end closes it and
// charges the interval since the previous mark on the plan to `ph`
void phase_call_begin(stkde_plan_s *p, cudaStream_t st);
void phase_begin(int ph);
void phase_end(stkde_plan_s *p, cudaStream_t st, int ph);
struct Phase {
    stkde_plan_s *p;
    cudaStream_t st;
    int ph;
    Phase(stkde_plan_s *p_, cudaStream_t st_, int ph_) : p(p_), st(st_), ph(ph_) { phase_begin(ph); }
    ~Phase() { phase_end(p, st, ph); }
};
// frees the communicator, gather staging and phase events (stkde_plan_destroy)
void trace_comm_release(stkde_plan_s *p);
}  // namespace stkde
