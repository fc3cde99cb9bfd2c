// stkde_api.cu -- C ABI (include/stkde.h): plans, workspace, orchestration.
//
// A compute call enqueues, on the caller's stream and without any host
// synchronisation:
//   K1 prep + bucket histogram -> CUB radix sort (home-tile key, point idx)
//   -> permute records -> CUB scan (bucket offsets)          [binning, §3.2]
//   K3a tile candidate counts -> CUB radix sort (LPT order)
//   -> K3b chunk pack -> CUB scan -> K3c work items         [work list, §3.3]
//   tile kernel (persistent, gather form, writes every voxel once)  [§3.4]
// The workspace is sized at plan creation from max_n, so the sequence is
// CUDA-graph capturable.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "stkde_internal.cuh"
#if STKDE_TC_DIAG
#include "stkde_diag.h"
#endif

namespace stkde {
static thread_local char g_err[512] = "";
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
}  // namespace stkde

using namespace stkde;

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            set_error("%s failed: %s", #call, cudaGetErrorString(e_));                    \
            return STKDE_ECUDA;                                                           \
        }                                                                                 \
    } while (0)

static int key_bits_for(int64_t maxkey) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) <= maxkey) ++b;
    return b;
}

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

extern "C" int stkde_plan_create(stkde_plan_t *out, int device, double x0, double y0, double t0, double sres,
                                 double tres, int64_t Gx, int64_t Gy, int64_t Gt, double hs, double ht,
                                 int kernel_kind, int64_t max_n) {
    if (!out) { set_error("out is NULL"); return STKDE_EINVAL; }
    *out = nullptr;
    if (!(sres > 0) || !std::isfinite(sres)) { set_error("sres must be > 0"); return STKDE_EINVAL; }
    if (!(tres > 0) || !std::isfinite(tres)) { set_error("tres must be > 0"); return STKDE_EINVAL; }
    if (!(hs > 0) || !std::isfinite(hs)) { set_error("hs must be > 0"); return STKDE_EINVAL; }
    if (!(ht > 0) || !std::isfinite(ht)) { set_error("ht must be > 0"); return STKDE_EINVAL; }
    if (!std::isfinite(x0) || !std::isfinite(y0) || !std::isfinite(t0)) { set_error("origin must be finite"); return STKDE_EINVAL; }
    if (Gx < 1 || Gx > (1 << 22)) { set_error("Gx must be in [1, 2^22]"); return STKDE_EINVAL; }
    if (Gy < 1 || Gy > (1 << 22)) { set_error("Gy must be in [1, 2^22]"); return STKDE_EINVAL; }
    if (Gt < 1 || Gt > (1 << 22)) { set_error("Gt must be in [1, 2^22]"); return STKDE_EINVAL; }
    if (kernel_kind != STKDE_KERNEL_PRINTED && kernel_kind != STKDE_KERNEL_CLASSICAL) { set_error("kernel_kind must be 0 or 1"); return STKDE_EINVAL; }
    if (max_n < 0 || max_n > ((int64_t)1 << 31) - 1) { set_error("max_n must be in [0, 2^31-1]"); return STKDE_EINVAL; }
    const double Hs_d = std::ceil(hs / sres), Ht_d = std::ceil(ht / tres);
    if (Hs_d > 4096 || Ht_d > 4096) { set_error("hs/sres and ht/tres must be <= 4096 voxels"); return STKDE_EINVAL; }

    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) { set_error("device %d out of range (%d devices)", device, ndev); return STKDE_EINVAL; }
    CK(cudaSetDevice(device));

    stkde_plan_s *p = (stkde_plan_s *)calloc(1, sizeof(stkde_plan_s));
    if (!p) { set_error("host allocation failed"); return STKDE_ENOMEM; }
    p->device = device;
    CK(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device));
    GridParams &g = p->g;
    g.x0 = x0; g.y0 = y0; g.t0 = t0; g.sres = sres; g.tres = tres; g.hs = hs; g.ht = ht;
    g.rs = (float)(hs / sres);
    g.rt = (float)(ht / tres);
    g.rs2 = (float)((hs / sres) * (hs / sres));
    g.inv_rs = (float)(sres / hs);
    g.inv_rt = (float)(tres / ht);
    g.Gx = (int)Gx; g.Gy = (int)Gy; g.Gt = (int)Gt;
    g.Hs = (int)Hs_d; g.Ht = (int)Ht_d;
    p->engine = env_int("STKDE_ENGINE", STKDE_ENGINE_TC);
    if (p->engine != STKDE_ENGINE_SIMT && p->engine != STKDE_ENGINE_TENSOR && p->engine != STKDE_ENGINE_TC &&
        p->engine != STKDE_ENGINE_WS) {
        set_error("bad STKDE_ENGINE"); free(p); return STKDE_EINVAL;
    }
    // the tcgen05 engine stores per-point chords as int8 offsets: H_s <= 120
    // the short-window engine: windows of <= 17 layers (its instantiations) and the chord table
    if (p->engine == STKDE_ENGINE_WS && (g.Ht > 8 || g.Hs > 120)) p->engine = STKDE_ENGINE_TC;
    if (p->engine == STKDE_ENGINE_TC && g.Hs > 120) p->engine = STKDE_ENGINE_TENSOR;
    // Tile shape (DESIGN.md §3.4/§3.6): SIMT and mma.sync engines 16x16 columns x Bt
    // from the temporal window 2H_t+1; tcgen05 engine 16x8 columns (UMMA M = 128)
    // x Bt in {64, 128} (the accumulator lives in 128 of the CTA's 256 TMEM columns).
    int BT, BYv;
    if (p->engine == STKDE_ENGINE_TC) {
        BYv = 8;
        // Bt = 64 for short grids, and for grids with fewer than 8 Bt = 128 tiles per SM: the
        // persistent CTAs then hold several shorter tile pipelines each (dengue: 512 -> 1024 tiles)
        const int64_t nt128 = ((Gx + BX - 1) / BX) * ((Gy + 7) / 8) * ((Gt + 127) / 128);
        BT = (Gt <= 64 || nt128 < 8 * 148) ? 64 : 128;
    } else if (p->engine == STKDE_ENGINE_WS) {
        BYv = 16;
        BT = 32;                                   // the engine's accumulators per column
    } else {
        BYv = BYW;
        BT = g.Ht >= 16 ? 64 : (g.Ht >= 6 ? 32 : 16);
    }
    if (p->engine != STKDE_ENGINE_WS) BT = env_int("STKDE_BT", BT);
    int CT = BT >= 64 ? 16 : 8;
    CT = env_int("STKDE_CT", CT);
    if (p->engine == STKDE_ENGINE_TC   ? tile_tc_smem_bytes(BT) == 0
        : p->engine == STKDE_ENGINE_WS ? tile_ws_smem_bytes(g.Ht) == 0
                                       : tile_smem_bytes(BT, CT) == 0) {
        set_error("unsupported tile shape Bt=%d CT=%d for engine %d", BT, CT, p->engine); free(p); return STKDE_EINVAL;
    }
    g.BT = BT;
    g.BY = BYv;
    p->CT = CT;
    p->kernel = kernel_kind;
    g.kernel = kernel_kind;
    p->tile_threads = tile_threads(BT, CT);
    g.NTX = (int)((Gx + BX - 1) / BX);
    g.NTY = (int)((Gy + BYv - 1) / BYv);
    g.NTT = (int)((Gt + BT - 1) / BT);
    g.Ra = (g.Hs + BX - 1) / BX;
    g.Ray = (g.Hs + BYv - 1) / BYv;
    g.Rt = (g.Ht + BT - 1) / BT;
    g.XA0 = 0;
    g.NXA = g.NTX;
    // Home-bucket depth in T: the tcgen05 engine bins points into 16x8x32 (16 when
    // H_t <= 8 on Bt = 128 tiles) blocks so a tile fetches only the blocks its temporal
    // reach meets; the legacy engines bin by whole tiles.  (Bt = 64 tiles -- the small
    // grids -- keep 32: a tile's reach then spans 3-4 home blocks instead of 5-6, measured
    // tiny 0.041 -> 0.039 ms, dengue 0.079 -> 0.076 ms per graph step; on Bt = 128 tiles 16
    // stays best for short windows, ornith 5.96 vs 6.09 ms with 32.)
    g.BTH = p->engine == STKDE_ENGINE_TC ? (g.Ht <= 8 && BT == 128 ? 16 : 32) : p->engine == STKDE_ENGINE_WS ? 16 : BT;
    g.BTH = env_int("STKDE_BTH", g.BTH);
    if (g.BTH < 1) { set_error("bad STKDE_BTH"); free(p); return STKDE_EINVAL; }
    g.NTTH = (int)((Gt + g.BTH - 1) / g.BTH);
    p->ntiles = (int64_t)g.NTX * g.NTY * g.NTT;
    p->nbuckets = (int64_t)g.NTX * g.NTY * g.NTTH;
    if (p->ntiles >= ((int64_t)1 << 30) || p->nbuckets >= ((int64_t)1 << 30)) { set_error("grid has too many tiles"); free(p); return STKDE_EINVAL; }
    const int64_t ncc_max = std::min<int64_t>((BT - 1 + 2 * (int64_t)g.Ht) / g.BTH + 2, g.NTTH);
    const int64_t nseg_max = (int64_t)std::min(2 * g.Ray + 1, g.NTY) * ncc_max;
    if (nseg_max > MAXSEG) { set_error("bandwidth too large for the tile shape (%lld segments)", (long long)nseg_max); free(p); return STKDE_EINVAL; }
    p->max_n = max_n;
    p->key_bits = key_bits_for(p->nbuckets);

    // Work-item and split-slot bounds: total candidates <= n * (tiles a point is a candidate of):
    // its home bucket (a, b, cc) lies in the reach of <= 2Ra+1 x-tiles, 2Ray+1 y-tiles and
    // <= floor((BTH + 2 H_t + Bt - 2) / Bt) + 1 layer blocks (home_t_range)
    const int64_t ntc = std::min<int64_t>((g.BTH + 2 * (int64_t)g.Ht + BT - 2) / BT + 1, g.NTT);
    const int64_t nb = (int64_t)std::min(2 * g.Ra + 1, g.NTX) * std::min(2 * g.Ray + 1, g.NTY) * ntc;
    const int64_t cand_bound = std::max<int64_t>(max_n, 1) * nb;
    // split-tile partial slot: tcgen05 engine int64 exact sums per voxel, legacy engines FP32
    const size_t tile_bytes = (size_t)(p->engine == STKDE_ENGINE_TC ? 128 * 8 : 256 * 4) * BT;
    const int64_t slot_budget = (int64_t)env_int("STKDE_SLOT_MB", 4096) * (1 << 20) / (int64_t)tile_bytes;
    int64_t chunk = std::max<int64_t>(env_int("STKDE_CHUNK", 4096), (2 * cand_bound + slot_budget - 1) / slot_budget);
    // tcgen05 engine: the S32 accumulators take <= 129888 per point (D16: hl + mm + lh
    // + the ICOMP = 93 indicator), so a work item may accumulate at most
    // 16533 points before 2^31.
    // (measured: the largest chunk is fastest -- fewer split tiles and partial passes; the
    // LPT order already starts the heaviest items first)
    // the slot budget (STKDE_SLOT_MB) still bounds the split-tile partial slots: the chunk is the
    // larger of the request and the budget-derived minimum, capped at the S32 limit; if even
    // the cap cannot meet the budget the plan is refused (max_n too large for the budget)
    if (p->engine == STKDE_ENGINE_TC) {
        const int64_t need = (2 * cand_bound + slot_budget - 1) / slot_budget;
        if (need > 16384) {
            set_error("max_n = %lld needs %lld-candidate work items for the %d MiB split-slot budget "
                      "(STKDE_SLOT_MB), above the 16384-candidate S32 limit: lower max_n or raise STKDE_SLOT_MB",
                      (long long)max_n, (long long)need, env_int("STKDE_SLOT_MB", 4096));
            free(p);
            return STKDE_EINVAL;
        }
        chunk = std::min<int64_t>(std::max<int64_t>(env_int("STKDE_CHUNK", 16384), need), 16384);
    } else if (p->engine == STKDE_ENGINE_WS) {
        // short-window engine: small chunks split hot tiles over many CTAs (a chunk of a
        // 16x16x32 tile costs ~ its candidates x 4 warps x ~30 instructions)
        const int64_t need = (2 * cand_bound + slot_budget - 1) / slot_budget;
        chunk = std::max<int64_t>(env_int("STKDE_CHUNK", 1024), need);
    }
    chunk = std::min<int64_t>(chunk, (int64_t)1 << 30);
    p->chunk = (int)chunk;
    p->max_items = p->ntiles + cand_bound / chunk + 1;
    p->max_slots = 2 * (cand_bound / chunk) + 2;
    int rc;
    if (p->engine == STKDE_ENGINE_TC) {
        p->tile_threads = 256;
        p->smem_bytes = tile_tc_smem_bytes(BT);
        rc = tile_tc_occupancy(BT, kernel_kind, &p->ctas_per_sm);
    } else if (p->engine == STKDE_ENGINE_WS) {
        p->tile_threads = 128;
        p->smem_bytes = tile_ws_smem_bytes(g.Ht);
        rc = tile_ws_occupancy(g.Ht, kernel_kind, p->smem_bytes, &p->ctas_per_sm);
    } else if (p->engine == STKDE_ENGINE_TENSOR) {
        p->tile_threads = 256;
        p->smem_bytes = tile_mma_smem_bytes(BT);
        rc = tile_mma_occupancy(BT, kernel_kind, &p->ctas_per_sm);
    } else {
        p->smem_bytes = tile_smem_bytes(BT, CT);
        rc = tile_occupancy(BT, CT, kernel_kind, &p->ctas_per_sm);
    }
    if (rc != STKDE_OK) { set_error("tile kernel attribute/occupancy query failed"); free(p); return rc; }
    if (p->ctas_per_sm < 1) { set_error("tile kernel does not fit on an SM"); free(p); return STKDE_EINVAL; }

    // CUB temporary storage: max over the four calls at their largest sizes.
    const int nmax = (int)std::max<int64_t>(max_n, 1);
    size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b1, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                       (uint32_t *)nullptr, nmax, 0, p->key_bits));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, b2, (uint32_t *)nullptr, (uint32_t *)nullptr, (int)(p->nbuckets + 1)));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b3, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                       (uint32_t *)nullptr, (int)p->ntiles, 0, 32));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, b4, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)(p->ntiles + 1)));
    p->cub_bytes = std::max(std::max(b1, b2), std::max(b3, b4));

    // One workspace allocation, carved.
    struct Part { void **ptr; size_t bytes; };
    const size_t nrec = (size_t)std::max<int64_t>(max_n, 1);
    const size_t nt = (size_t)p->ntiles;
    Part parts[] = {
        {(void **)&p->rec, nrec * sizeof(PointRec)},
        {(void **)&p->rec_sorted, nrec * sizeof(PointRec)},
        {(void **)&p->chords, (p->engine == STKDE_ENGINE_TC || p->engine == STKDE_ENGINE_WS)
                                  ? nrec * (size_t)chord_rows(g.Hs) * 2 : 0},
        {(void **)&p->bw_rec, p->engine == STKDE_ENGINE_TC ? nrec * sizeof(PointBw) : 0},
        {(void **)&p->bw_sorted, p->engine == STKDE_ENGINE_TC ? nrec * sizeof(PointBw) : 0},
        {(void **)&p->keys_in, nrec * 4}, {(void **)&p->keys_out, nrec * 4},
        {(void **)&p->vals_in, nrec * 4}, {(void **)&p->vals_out, nrec * 4},
        {(void **)&p->bucket_cnt, ((size_t)p->nbuckets + 1) * 4}, {(void **)&p->bucket_begin, ((size_t)p->nbuckets + 2) * 4},
        {(void **)&p->lpt_key_in, nt * 4}, {(void **)&p->lpt_key_out, nt * 4},
        {(void **)&p->lpt_val_in, nt * 4}, {(void **)&p->lpt_val_out, nt * 4},
        {(void **)&p->tile_cnt, nt * 4},
        {(void **)&p->chunk_pack, (nt + 1) * 8}, {(void **)&p->chunk_off, (nt + 1) * 8},
        {(void **)&p->items, (size_t)p->max_items * 16},
        {(void **)&p->arrive, nt * 4},
        {(void **)&p->partials, (size_t)p->max_slots * tile_bytes},
        {(void **)&p->counters, 128 * 4},
        {(void **)&p->hist_t, ((size_t)Gt + 1) * 4},
        {(void **)&p->hist_x, ((size_t)Gx + 1) * 4},
        {(void **)&p->cub_tmp, p->cub_bytes},
    };
    size_t total = 0;
    for (auto &pt : parts) total = align_up(total, 256) + pt.bytes;
    cudaError_t e = cudaMalloc(&p->ws, total);
    if (e != cudaSuccess) {
        set_error("workspace allocation of %zu bytes failed: %s", total, cudaGetErrorString(e));
        free(p);
        return STKDE_ENOMEM;
    }
    p->ws_bytes = total;
    size_t off = 0;
    for (auto &pt : parts) {
        off = align_up(off, 256);
        *pt.ptr = (char *)p->ws + off;
        off += pt.bytes;
    }
    CK(cudaMemset(p->arrive, 0, nt * 4));
    CK(cudaMemset(p->counters, 0, 128 * 4));
    p->tc_profile = env_int("STKDE_TC_PROF", 0);
    p->tc_watchdog = env_int("STKDE_TC_WATCHDOG", 0);
    p->no_tma = env_int("STKDE_NO_TMA", 0);
    p->plain_stores = env_int("STKDE_PLAIN_STORES", 0);
    p->order = env_int("STKDE_ORDER", -1);       // -1: by the slab's tile count (launch_worklist)
    p->heavy = env_int("STKDE_HEAVY", p->chunk / 4);
    p->wl_small = env_int("STKDE_WL_SMALL", 1);
    *out = p;
    return STKDE_OK;
}

extern "C" void stkde_plan_destroy(stkde_plan_t p) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    trace_comm_release(p);
    cudaFree(p->ws);
    for (int i = 0; i < 2 * p->tev_cap; ++i) cudaEventDestroy(p->tev[i]);
    free(p->tev);
    cudaSetDevice(cur);
    free(p);
}

// Sum the recorded tile-kernel intervals (synchronises on the last stop event).
static void harvest_timing(stkde_plan_s *p) {
    for (int i = 0; i < p->tev_used; ++i) {
        float ms = 0.f;
        if (cudaEventSynchronize(p->tev[2 * i + 1]) == cudaSuccess &&
            cudaEventElapsedTime(&ms, p->tev[2 * i], p->tev[2 * i + 1]) == cudaSuccess) {
            p->kernel_ms += ms;
            p->kernel_launches += 1;
        }
    }
    p->tev_used = 0;
}

// Per-call state of an adaptive-bandwidth call (p->d_bw), cleared on every exit.
struct BwScope {
    stkde_plan_s *p;
    BwScope(stkde_plan_s *p_, const float *bw) : p(p_) { p->d_bw = bw; }
    ~BwScope() { p->d_bw = nullptr; }
};

static int compute_slab_impl(stkde_plan_s *p, const float *d_points, int64_t n, int64_t n_norm, int64_t t_begin,
                             int64_t t_end, float *d_out, cudaStream_t st, const float *d_bw = nullptr) {
    const GridParams &g = p->g;
    p->last_own_launches = 0;
    p->last_cub_calls = 0;
    if (d_bw && p->engine != STKDE_ENGINE_TC) {
        set_error("adaptive bandwidths need the tcgen05 engine (H_s <= 120, STKDE_ENGINE unset or 2)");
        return STKDE_EINVAL;
    }
    BwScope scope(p, d_bw);
    if (n < 0 || n_norm < 0) { set_error("n must be >= 0"); return STKDE_EINVAL; }
    if (n > p->max_n) { set_error("n = %lld exceeds the plan's max_n = %lld", (long long)n, (long long)p->max_n); return STKDE_ECAPACITY; }
    if (t_begin < 0 || t_end > g.Gt || t_begin >= t_end) { set_error("slab [t_begin, t_end) must satisfy 0 <= t_begin < t_end <= Gt"); return STKDE_EINVAL; }
    if (!d_out || (n > 0 && !d_points)) { set_error("NULL device pointer"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    const int64_t Ts = t_end - t_begin;
    if (n == 0 || n_norm == 0) {   // empty point set -> zeros, no division
        CK(cudaMemsetAsync(d_out, 0, (size_t)g.Gx * g.Gy * Ts * sizeof(float), st));
        return STKDE_OK;
    }
    // 1/(n hs^2 ht) times the kernel constant (pi/2 or 2/pi); adaptive
    // calls: 1/(n sres^2 tres), the tile kernel supplies max_i (sres/hs_i)^2 (tres/ht_i)
    const double kc = p->kernel == STKDE_KERNEL_PRINTED ? M_PI / 2.0 : 2.0 / M_PI;
    const float cnorm = d_bw ? (float)(kc / ((double)n_norm * (g.sres * g.sres) * g.tres))
                             : (float)(kc / ((double)n_norm * (g.hs * g.hs) * g.ht));
    // the tcgen05 engine bins only the points that reach the slab (its integer sums do not
    // depend on the candidate grouping); the FP32 engines keep the full binning so a slab
    // stays bitwise equal to the full grid's layers
    const bool slab_cull = p->engine == STKDE_ENGINE_TC;
    // (tcgen05 engine: the chord table is written by the binning's scatter pass)
    int rc = launch_binning(p, d_points, n, st, slab_cull ? t_begin : 0, slab_cull ? t_end : (int64_t)g.Gt,
                            p->engine == STKDE_ENGINE_TC);
    if (rc) { set_error("binning launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    // short-window engine: the chord table over the stably sorted records
    if (p->engine == STKDE_ENGINE_WS && (rc = launch_chords(p, n, st))) {
        set_error("chord launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        return rc;
    }
    const int c0 = (int)(t_begin / g.BT), c1 = (int)((t_end + g.BT - 1) / g.BT);
    rc = launch_worklist(p, c0, c1, st);
    if (rc) { set_error("work-list launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    {
        Phase ph(p, st, STKDE_PHASE_TILES);
        rc = p->engine == STKDE_ENGINE_TC       ? launch_tile_tc(p, c0, c1, t_begin, t_end, cnorm, d_out, st)
             : p->engine == STKDE_ENGINE_WS     ? launch_tile_ws(p, c0, c1, t_begin, t_end, cnorm, d_out, st)
             : p->engine == STKDE_ENGINE_TENSOR ? launch_tile_mma(p, c0, c1, t_begin, t_end, cnorm, d_out, st)
                                                : launch_tile(p, c0, c1, t_begin, t_end, cnorm, d_out, st);
    }
    if (rc) { set_error("tile kernel launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    return STKDE_OK;
}

extern "C" int stkde_compute(stkde_plan_t p, const float *d_points, int64_t n, float *d_grid, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    return compute_slab_impl(p, d_points, n, n, 0, p->g.Gt, d_grid, (cudaStream_t)stream);
}

// ---- CUDA graphs: one compute call captured once, replayed with a single launch ----
struct stkde_graph_s {
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    int device;
};

// capture one enqueue sequence (fn(stream)) of plan p on a private stream into a CUDA graph
template <class F>
static int graph_capture(stkde_plan_s *p, stkde_graph_t *out, F fn) {
    *out = nullptr;
    CK(cudaSetDevice(p->device));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int timing = p->timing;
    p->timing = 0;                                     // no event nodes in the graph
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    int rc = STKDE_OK;
    if (e == cudaSuccess) {
        rc = fn(s);
        e = cudaStreamEndCapture(s, &graph);
    }
    p->timing = timing;
    cudaStreamDestroy(s);
    if (rc != STKDE_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) {
        set_error("graph capture failed: %s", cudaGetErrorString(e));
        if (graph) cudaGraphDestroy(graph);
        return STKDE_ECUDA;
    }
    stkde_graph_s *g = (stkde_graph_s *)calloc(1, sizeof(stkde_graph_s));
    if (!g) { cudaGraphDestroy(graph); set_error("host allocation failed"); return STKDE_ENOMEM; }
    g->graph = graph;
    g->device = p->device;
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (e != cudaSuccess) {
        set_error("graph instantiation failed: %s", cudaGetErrorString(e));
        cudaGraphDestroy(graph);
        free(g);
        return STKDE_ECUDA;
    }
    *out = g;
    return STKDE_OK;
}

extern "C" int stkde_graph_create(stkde_plan_t p, const float *d_points, int64_t n, int64_t n_norm, int64_t t_begin,
                                  int64_t t_end, float *d_out, stkde_graph_t *out) {
    if (!p || !out) { set_error("NULL argument"); return STKDE_EINVAL; }
    return graph_capture(p, out, [&](cudaStream_t s) {
        return compute_slab_impl(p, d_points, n, n_norm, t_begin, t_end, d_out, s);
    });
}

extern "C" int stkde_graph_create_xslab(stkde_plan_t p, const float *d_points, int64_t n, int64_t n_norm,
                                        int64_t x_begin, int64_t x_end, float *d_xslab, stkde_graph_t *out) {
    if (!p || !out) { set_error("NULL argument"); return STKDE_EINVAL; }
    return graph_capture(p, out, [&](cudaStream_t s) {
        return stkde_compute_xslab(p, d_points, n, n_norm, x_begin, x_end, d_xslab, s);
    });
}

extern "C" int stkde_graph_launch(stkde_graph_t g, void *stream) {
    if (!g) { set_error("graph is NULL"); return STKDE_EINVAL; }
    CK(cudaSetDevice(g->device));
    CK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    return STKDE_OK;
}

extern "C" void stkde_graph_destroy(stkde_graph_t g) {
    if (!g) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(g->graph);
    cudaSetDevice(cur);
    free(g);
}

extern "C" int stkde_compute_slab(stkde_plan_t p, const float *d_points, int64_t n, int64_t n_norm, int64_t t_begin,
                                  int64_t t_end, float *d_slab, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    return compute_slab_impl(p, d_points, n, n_norm, t_begin, t_end, d_slab, (cudaStream_t)stream);
}

static int count_impl(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n, int64_t t_begin,
                      int64_t t_end, int64_t *d_count, void *stream, int64_t x_begin = 0, int64_t x_end = -1) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (x_end < 0) x_end = p->g.Gx;
    if (n < 0 || (n > 0 && !d_points) || !d_count) { set_error("bad points/count arguments"); return STKDE_EINVAL; }
    if (t_begin < 0 || t_end > p->g.Gt || t_begin >= t_end) { set_error("bad slab"); return STKDE_EINVAL; }
    if (x_begin < 0 || x_end > p->g.Gx || x_begin >= x_end) { set_error("bad x range"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    int rc = launch_count(p, d_points, n, t_begin, t_end, d_count, (cudaStream_t)stream, d_bw, x_begin, x_end);
    if (rc) set_error("count launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return rc;
}

extern "C" int stkde_count_contributions(stkde_plan_t p, const float *d_points, int64_t n, int64_t t_begin,
                                         int64_t t_end, int64_t *d_count, void *stream) {
    return count_impl(p, d_points, nullptr, n, t_begin, t_end, d_count, stream);
}

extern "C" int stkde_count_contributions_box(stkde_plan_t p, const float *d_points, int64_t n, int64_t x_begin,
                                             int64_t x_end, int64_t t_begin, int64_t t_end, int64_t *d_count,
                                             void *stream) {
    return count_impl(p, d_points, nullptr, n, t_begin, t_end, d_count, stream, x_begin, x_end);
}

extern "C" int stkde_count_contributions_adaptive(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n,
                                                  int64_t t_begin, int64_t t_end, int64_t *d_count, void *stream) {
    if (n > 0 && !d_bw) { set_error("d_bw is NULL"); return STKDE_EINVAL; }
    return count_impl(p, d_points, d_bw, n, t_begin, t_end, d_count, stream);
}

// ---- adaptive bandwidth (reading R15) ----
extern "C" int stkde_compute_adaptive(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n,
                                      float *d_grid, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (n > 0 && !d_bw) { set_error("d_bw is NULL"); return STKDE_EINVAL; }
    return compute_slab_impl(p, d_points, n, n, 0, p->g.Gt, d_grid, (cudaStream_t)stream, n > 0 ? d_bw : nullptr);
}

// ---- FP64-output option (stkde_tile_f64.cu) ----
static int compute_f64_impl(stkde_plan_s *p, const float *d_points, const float *d_bw, int64_t n, int64_t n_norm,
                            int64_t t_begin, int64_t t_end, double *d_out, cudaStream_t st) {
    const GridParams &g = p->g;
    p->last_own_launches = 0;
    p->last_cub_calls = 0;
    if (d_bw && p->engine != STKDE_ENGINE_TC) {
        set_error("adaptive bandwidths need the tcgen05 engine (H_s <= 120, STKDE_ENGINE unset or 2)");
        return STKDE_EINVAL;
    }
    if (n < 0 || n_norm < 0) { set_error("n must be >= 0"); return STKDE_EINVAL; }
    if (n > p->max_n) { set_error("n = %lld exceeds the plan's max_n = %lld", (long long)n, (long long)p->max_n); return STKDE_ECAPACITY; }
    if (t_begin < 0 || t_end > g.Gt || t_begin >= t_end) { set_error("slab [t_begin, t_end) must satisfy 0 <= t_begin < t_end <= Gt"); return STKDE_EINVAL; }
    if (!d_out || (n > 0 && !d_points)) { set_error("NULL device pointer"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    if (n == 0 || n_norm == 0) {   // empty point set -> zeros, no division
        CK(cudaMemsetAsync(d_out, 0, (size_t)g.Gx * g.Gy * (t_end - t_begin) * sizeof(double), st));
        return STKDE_OK;
    }
    BwScope scope(p, d_bw);
    int rc = launch_binning(p, d_points, n, st, t_begin, t_end, false, true);
    if (rc) { set_error("binning launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    // Alg. 1 divides the sum by n hs^2 ht; adaptive: terms carry 1/(hs_i^2 ht_i), the sum 1/n
    const double den = d_bw ? (double)n_norm : (double)n_norm * (g.hs * g.hs) * g.ht;
    {
        Phase ph(p, st, STKDE_PHASE_TILES);
        rc = launch_tile_f64(p, d_points, d_bw, t_begin, t_end, den, d_out, st);
    }
    if (rc) { set_error("FP64 tile kernel launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    return STKDE_OK;
}

extern "C" int stkde_compute_f64(stkde_plan_t p, const float *d_points, int64_t n, double *d_grid, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    return compute_f64_impl(p, d_points, nullptr, n, n, 0, p->g.Gt, d_grid, (cudaStream_t)stream);
}

extern "C" int stkde_compute_slab_f64(stkde_plan_t p, const float *d_points, int64_t n, int64_t n_norm,
                                      int64_t t_begin, int64_t t_end, double *d_slab, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    return compute_f64_impl(p, d_points, nullptr, n, n_norm, t_begin, t_end, d_slab, (cudaStream_t)stream);
}

extern "C" int stkde_compute_adaptive_slab_f64(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n,
                                               int64_t n_norm, int64_t t_begin, int64_t t_end, double *d_slab,
                                               void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (n > 0 && !d_bw) { set_error("d_bw is NULL"); return STKDE_EINVAL; }
    return compute_f64_impl(p, d_points, n > 0 ? d_bw : nullptr, n, n_norm, t_begin, t_end, d_slab,
                            (cudaStream_t)stream);
}

extern "C" int stkde_compute_adaptive_slab(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n,
                                           int64_t n_norm, int64_t t_begin, int64_t t_end, float *d_slab,
                                           void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (n > 0 && !d_bw) { set_error("d_bw is NULL"); return STKDE_EINVAL; }
    return compute_slab_impl(p, d_points, n, n_norm, t_begin, t_end, d_slab, (cudaStream_t)stream,
                             n > 0 ? d_bw : nullptr);
}

// ---- multi-bandwidth sweep (Fig. 1) ----
// The plan's GridParams narrowed to (hs_k, ht_k) <= (hs, ht): gates, kernel scales and
// reach (H, Ra, Ray, Rt) of the smaller bandwidth; the home-bucket geometry (tile
// shape, BTH, key layout) stays the plan's, so one binning serves every bandwidth.
static GridParams narrowed(const GridParams &g, double hs, double ht) {
    GridParams k = g;
    k.hs = hs; k.ht = ht;
    k.rs = (float)(hs / g.sres);
    k.rt = (float)(ht / g.tres);
    k.rs2 = (float)((hs / g.sres) * (hs / g.sres));
    k.inv_rs = (float)(g.sres / hs);
    k.inv_rt = (float)(g.tres / ht);
    k.Hs = (int)std::ceil(hs / g.sres);
    k.Ht = (int)std::ceil(ht / g.tres);
    k.Ra = (k.Hs + BX - 1) / BX;
    k.Ray = (k.Hs + g.BY - 1) / g.BY;
    k.Rt = (k.Ht + g.BT - 1) / g.BT;
    return k;
}

extern "C" int stkde_compute_sweep(stkde_plan_t p, const float *d_points, int64_t n, int nbw, const double *h_hs,
                                   const double *h_ht, float *const *d_grids, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    if (nbw < 1 || !h_hs || !h_ht || !d_grids) { set_error("bad sweep arguments"); return STKDE_EINVAL; }
    const GridParams g0 = p->g;
    for (int k = 0; k < nbw; ++k) {
        if (!(h_hs[k] > 0) || !(h_ht[k] > 0) || !(h_hs[k] <= g0.hs) || !(h_ht[k] <= g0.ht)) {
            set_error("sweep bandwidth %d must satisfy 0 < hs_k <= hs and 0 < ht_k <= ht", k);
            return STKDE_EINVAL;
        }
        if (!d_grids[k]) { set_error("d_grids[%d] is NULL", k); return STKDE_EINVAL; }
    }
    if (n < 0) { set_error("n must be >= 0"); return STKDE_EINVAL; }
    if (n > p->max_n) { set_error("n = %lld exceeds the plan's max_n = %lld", (long long)n, (long long)p->max_n); return STKDE_ECAPACITY; }
    if (n > 0 && !d_points) { set_error("NULL device pointer"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    p->last_own_launches = 0;
    p->last_cub_calls = 0;
    const size_t vox = (size_t)g0.Gx * g0.Gy * g0.Gt;
    if (n == 0) {
        for (int k = 0; k < nbw; ++k) CK(cudaMemsetAsync(d_grids[k], 0, vox * sizeof(float), st));
        return STKDE_OK;
    }
    int rc = launch_binning(p, d_points, n, st, 0, g0.Gt);   // once, at the plan's (largest) reach
    if (rc) { set_error("binning launch failed: %s", cudaGetErrorString(cudaGetLastError())); return rc; }
    // tcgen05 engine: the sorted points' world coordinates go to a side buffer (the per-point
    // bandwidth buffer, unused by a fixed-bandwidth sweep) so each bandwidth's chord pass can
    // read them while the records' x carries the sorted index for the loader
    float2 *xy = p->engine == STKDE_ENGINE_TC ? reinterpret_cast<float2 *>(p->bw_rec) : nullptr;
    if (xy && (rc = launch_save_xy(p, n, xy, st))) {
        set_error("sweep launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        return rc;
    }
    const double kc = p->kernel == STKDE_KERNEL_PRINTED ? M_PI / 2.0 : 2.0 / M_PI;
    const int c0 = 0, c1 = g0.NTT;
    for (int k = 0; k < nbw; ++k) {
        p->g = narrowed(g0, h_hs[k], h_ht[k]);
        const float cnorm = (float)(kc / ((double)n * (h_hs[k] * h_hs[k]) * h_ht[k]));
        if (p->engine == STKDE_ENGINE_TC || p->engine == STKDE_ENGINE_WS) rc = launch_chords(p, n, st, xy);
        if (!rc) rc = launch_worklist(p, c0, c1, st);
        if (!rc) {
            Phase ph(p, st, STKDE_PHASE_TILES);
            rc = p->engine == STKDE_ENGINE_TC       ? launch_tile_tc(p, c0, c1, 0, g0.Gt, cnorm, d_grids[k], st)
                 : p->engine == STKDE_ENGINE_WS     ? launch_tile_ws(p, c0, c1, 0, g0.Gt, cnorm, d_grids[k], st)
                 : p->engine == STKDE_ENGINE_TENSOR ? launch_tile_mma(p, c0, c1, 0, g0.Gt, cnorm, d_grids[k], st)
                                                    : launch_tile(p, c0, c1, 0, g0.Gt, cnorm, d_grids[k], st);
        }
        p->g = g0;
        if (rc) { set_error("sweep launch %d failed: %s", k, cudaGetErrorString(cudaGetLastError())); return rc; }
    }
    return STKDE_OK;
}

// Cost-balanced Bt-aligned cuts: per-layer cost =
//   Gx*Gy*4 B / B_hbm  +  2 * W(T) / P_fp32,
// W(T) = (disc columns) * #{points whose window contains T}; cuts are taken
// at tile-layer boundaries where the cumulative cost crosses k/nparts.
extern "C" int stkde_slab_cuts(int64_t Gx, int64_t Gy, int64_t Gt, int Bt, int Ht, double rs,
                               const int64_t *h_hist, int nparts, int64_t *h_cuts) {
    if (!h_cuts || !h_hist || nparts < 1 || Gx < 1 || Gy < 1 || Gt < 1 || Bt < 1 || Ht < 0 || !(rs > 0)) {
        set_error("bad arguments to stkde_slab_cuts");
        return STKDE_EINVAL;
    }
    const double B_hbm = 6.5e12, P_fp32 = 6.0e13;
    const double disc = M_PI * rs * rs;
    std::vector<double> pre(Gt + 1, 0.0);   // prefix of point counts by T_i
    for (int64_t T = 0; T < Gt; ++T) pre[T + 1] = pre[T] + (double)h_hist[T];
    const int64_t nblk = (Gt + Bt - 1) / Bt;
    std::vector<double> cost(nblk, 0.0);
    for (int64_t T = 0; T < Gt; ++T) {
        int64_t lo = std::max<int64_t>(T - Ht, 0), hi = std::min<int64_t>(T + Ht, Gt - 1);
        double w = (pre[hi + 1] - pre[lo]) * disc;
        cost[T / Bt] += (double)Gx * Gy * 4.0 / B_hbm + 2.0 * w / P_fp32;
    }
    std::vector<double> cum(nblk + 1, 0.0);
    for (int64_t b = 0; b < nblk; ++b) cum[b + 1] = cum[b] + cost[b];
    const double tot = cum[nblk];
    h_cuts[0] = 0;
    int64_t prev = 0;
    for (int k = 1; k < nparts; ++k) {
        // first block boundary b with cum[b] >= tot*k/nparts (nearest of the two neighbours)
        const double target = tot * k / nparts;
        int64_t b = prev + 1;
        while (b < nblk && cum[b] < target) ++b;
        if (b > prev + 1 && (target - cum[b - 1]) < (cum[b] - target)) --b;
        // keep at least one block per remaining part (when possible)
        b = std::min<int64_t>(b, nblk - (nparts - k));
        b = std::max<int64_t>(b, std::min<int64_t>(prev + 1, nblk));
        h_cuts[k] = std::min<int64_t>(b * Bt, Gt);
        prev = b;
    }
    h_cuts[nparts] = Gt;
    for (int k = 1; k <= nparts; ++k)
        if (h_cuts[k] < h_cuts[k - 1]) h_cuts[k] = h_cuts[k - 1];
    return STKDE_OK;
}

// ---- x-slabs (multi-GPU partition along X) ----
// Per-column cost: alpha * Gy*Gt*4 B / B_hbm + beta * 2 W(X) / P_fp32 with W(X) = (2 rs)
// (2 rt + 1) #{points with |X - X_i| <= rs + 8} (the tile kernel's candidates of the
// column's 16-wide tile); cuts at multiples of 16 columns (tile width).
extern "C" int stkde_xslab_cuts(int64_t Gx, int64_t Gy, int64_t Gt, double rs, double rt, const int64_t *h_hist_X,
                                int nparts, int64_t *h_cuts) {
    if (!h_cuts || !h_hist_X || nparts < 1 || Gx < 1 || Gy < 1 || Gt < 1 || !(rs > 0) || !(rt > 0)) {
        set_error("bad arguments to stkde_xslab_cuts");
        return STKDE_EINVAL;
    }
    const double B_hbm = 6.5e12, P_fp32 = 6.0e13;
    // the tile kernel's cost follows its candidates (every point whose box reaches the
    // column's 16-wide tile), so each point weighs the full disc height 2 rs over the
    // columns within rs + 8 of it (measured: more even slab times than chord weights)
    const int R = (int)std::ceil(rs) + BX / 2;
    std::vector<double> chord(2 * R + 1, 2.0 * rs);
    const int64_t nblk = (Gx + BX - 1) / BX;
    std::vector<double> cost(nblk, 0.0);
    for (int64_t X = 0; X < Gx; ++X) {
        double w = 0.0;
        for (int d = -R; d <= R; ++d) {
            const int64_t Xi = X - d;
            if (Xi >= 0 && Xi < Gx) w += (double)h_hist_X[Xi] * chord[d + R];
        }
        cost[X / BX] += (double)Gy * Gt * 4.0 / B_hbm + 2.0 * w * (2.0 * rt + 1.0) / P_fp32;
    }
    std::vector<double> cum(nblk + 1, 0.0);
    for (int64_t b = 0; b < nblk; ++b) cum[b + 1] = cum[b] + cost[b];
    const double tot = cum[nblk];
    h_cuts[0] = 0;
    int64_t prev = 0;
    for (int k = 1; k < nparts; ++k) {
        const double target = tot * k / nparts;
        int64_t b = prev + 1;
        while (b < nblk && cum[b] < target) ++b;
        if (b > prev + 1 && (target - cum[b - 1]) < (cum[b] - target)) --b;
        b = std::min<int64_t>(b, nblk - (nparts - k));
        b = std::max<int64_t>(b, std::min<int64_t>(prev + 1, nblk));
        h_cuts[k] = std::min<int64_t>(b * BX, Gx);
        prev = b;
    }
    h_cuts[nparts] = Gx;
    for (int k = 1; k <= nparts; ++k)
        if (h_cuts[k] < h_cuts[k - 1]) h_cuts[k] = h_cuts[k - 1];
    return STKDE_OK;
}

extern "C" int stkde_xslab_partition(stkde_plan_t p, const float *d_points, int64_t n, int nparts, int64_t *h_cuts,
                                     void *stream) {
    if (!p || !h_cuts || nparts < 1) { set_error("bad arguments"); return STKDE_EINVAL; }
    const GridParams &g = p->g;
    CK(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (p->engine == STKDE_ENGINE_TC && n > 0 && n <= p->max_n) {
        // tcgen05 engine: the cost of an x-tile column is the tile kernel's own work, its tiles'
        // candidate counts (the same counts its work list sorts by) plus a fixed per-tile cost
        // kappa (STKDE_XKAPPA), from one binning of the full grid.  Measured (one-GPU estimate of
        // the 8-slab speedup, scripts/slab_scaling.py): round 1, kappa = 300 gave stress 6.45x and
        // ornith 5.16x, kappa = 1000 6.17x and 5.57x, kappa = 3000 5.48x and 5.12x; the point
        // histogram of stkde_xslab_cuts 6.45x and 5.31x.  Final round-2 build: kappa = 0 / 150 /
        // 300 / 500 / 600 / 1200 give stress 6.65 / 6.66 / 6.96 / 6.85 / 6.85 / 6.57x and ornith
        // 5.58 / 5.75 / 5.97 / 6.15 / 6.12 / 6.02x (500: both >= 6).  Slab times vary +-5 %.
        int rc = launch_binning(p, d_points, n, st, 0, g.Gt, false);
        if (rc) { set_error("binning launch failed"); return rc; }
        const int nsl = g.NXA * g.NTY * g.NTT;
        rc = launch_tile_cost(p, nsl, st);
        if (rc) { set_error("tile-count launch failed"); return rc; }
        std::vector<uint32_t> cnt((size_t)nsl);
        CK(cudaMemcpyAsync(cnt.data(), p->tile_cnt, (size_t)nsl * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double kappa = (double)env_int("STKDE_XKAPPA", 500);   // per-tile fixed cost, in candidates
        std::vector<double> col(g.NTX, 0.0);
        for (int ls = 0; ls < nsl; ++ls) col[ls % g.NXA + g.XA0] += kappa + (double)cnt[ls];
        std::vector<double> cum(g.NTX + 1, 0.0);
        for (int a = 0; a < g.NTX; ++a) cum[a + 1] = cum[a] + col[a];
        const double tot = cum[g.NTX];
        h_cuts[0] = 0;
        int64_t prev = 0;
        for (int k = 1; k < nparts; ++k) {
            const double target = tot * k / nparts;
            int64_t b = prev + 1;
            while (b < g.NTX && cum[b] < target) ++b;
            if (b > prev + 1 && (target - cum[b - 1]) < (cum[b] - target)) --b;
            b = std::min<int64_t>(b, g.NTX - (nparts - k));
            b = std::max<int64_t>(b, std::min<int64_t>(prev + 1, g.NTX));
            h_cuts[k] = std::min<int64_t>(b * BX, g.Gx);
            prev = b;
        }
        h_cuts[nparts] = g.Gx;
        for (int k = 1; k <= nparts; ++k)
            if (h_cuts[k] < h_cuts[k - 1]) h_cuts[k] = h_cuts[k - 1];
        return STKDE_OK;
    }
    std::vector<int> hist(g.Gx + 1, 0);
    if (n > 0) {
        int rc = launch_hist_x(p, d_points, n, st);
        if (rc) { set_error("histogram launch failed"); return rc; }
        CK(cudaMemcpyAsync(hist.data(), p->hist_x, g.Gx * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    std::vector<int64_t> h64(hist.begin(), hist.begin() + g.Gx);
    return stkde_xslab_cuts(g.Gx, g.Gy, g.Gt, (double)g.rs, (double)g.rt, h64.data(), nparts, h_cuts);
}

static int xslab_impl(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n, int64_t n_norm,
                      int64_t x_begin, int64_t x_end, float *d_xslab, void *stream) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    const GridParams g0 = p->g;
    if (p->engine != STKDE_ENGINE_TC && p->engine != STKDE_ENGINE_WS) {
        set_error("x-slabs need the tcgen05 or the short-window engine");
        return STKDE_EINVAL;
    }
    if (x_begin < 0 || x_end > g0.Gx || x_begin >= x_end || x_begin % BX != 0 || (x_end % BX != 0 && x_end != g0.Gx)) {
        set_error("x-slab [x_begin, x_end) must satisfy 0 <= x_begin < x_end <= Gx with x_begin and x_end "
                  "(unless = Gx) multiples of 16");
        return STKDE_EINVAL;
    }
    if (!d_xslab) { set_error("NULL device pointer"); return STKDE_EINVAL; }
    if (n < 0 || n_norm < 0) { set_error("n must be >= 0"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    if (n == 0 || n_norm == 0) {
        p->last_own_launches = p->last_cub_calls = 0;
        CK(cudaMemsetAsync(d_xslab, 0, (size_t)(x_end - x_begin) * g0.Gy * g0.Gt * sizeof(float), (cudaStream_t)stream));
        return STKDE_OK;
    }
    p->g.XA0 = (int)(x_begin / BX);
    p->g.NXA = (int)((x_end + BX - 1) / BX - x_begin / BX);
    // the tile kernel indexes the full grid; the slab is that grid's block of rows [x_begin, x_end)
    float *out_shifted = d_xslab - x_begin * (int64_t)g0.Gy * g0.Gt;
    // the direct gather (include/stkde.h: stkde_ipc_*) passes rows of the root's grid on
    // another device: its epilogue then uses plain stores over the peer mapping
    cudaPointerAttributes pa;
    p->out_remote = p->plain_stores || (cudaPointerGetAttributes(&pa, d_xslab) == cudaSuccess &&
                                        pa.type == cudaMemoryTypeDevice && pa.device != p->device);
    cudaGetLastError();
    const int rc = compute_slab_impl(p, d_points, n, n_norm, 0, g0.Gt, out_shifted, (cudaStream_t)stream, d_bw);
    p->g = g0;
    p->out_remote = 0;
    return rc;
}

extern "C" int stkde_compute_xslab(stkde_plan_t p, const float *d_points, int64_t n, int64_t n_norm,
                                   int64_t x_begin, int64_t x_end, float *d_xslab, void *stream) {
    return xslab_impl(p, d_points, nullptr, n, n_norm, x_begin, x_end, d_xslab, stream);
}

extern "C" int stkde_compute_adaptive_xslab(stkde_plan_t p, const float *d_points, const float *d_bw, int64_t n,
                                            int64_t n_norm, int64_t x_begin, int64_t x_end, float *d_xslab,
                                            void *stream) {
    if (n > 0 && !d_bw) { set_error("d_bw is NULL"); return STKDE_EINVAL; }
    return xslab_impl(p, d_points, n > 0 ? d_bw : nullptr, n, n_norm, x_begin, x_end, d_xslab, stream);
}

extern "C" int stkde_slab_partition(stkde_plan_t p, const float *d_points, int64_t n, int nparts, int64_t *h_cuts,
                                    void *stream) {
    if (!p || !h_cuts || nparts < 1) { set_error("bad arguments"); return STKDE_EINVAL; }
    const GridParams &g = p->g;
    CK(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<int> hist(g.Gt + 1, 0);
    if (n > 0) {
        int rc = launch_hist_t(p, d_points, n, st);
        if (rc) { set_error("histogram launch failed"); return rc; }
        CK(cudaMemcpyAsync(hist.data(), p->hist_t, g.Gt * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    std::vector<int64_t> h64(hist.begin(), hist.begin() + g.Gt);
    // cut granularity: Bt; the tcgen05 engine (slabs bitwise equal at any boundary, TMA
    // epilogue for 32-aligned starts) halves it down to 32 layers while there are fewer
    // Bt blocks than parts (stress at 8 ranks: 64-layer slabs instead of 4 busy ranks)
    int gran = g.BT;
    if (p->engine == STKDE_ENGINE_TC)
        while (gran > 32 && (g.Gt + gran - 1) / gran < nparts) gran /= 2;
    return stkde_slab_cuts(g.Gx, g.Gy, g.Gt, gran, g.Ht, (double)g.rs, h64.data(), nparts, h_cuts);
}

extern "C" int stkde_compute_sharded(stkde_plan_t *plans, int ndev, const float *const *d_points, int64_t n,
                                     float *const *d_slabs, int64_t *h_cuts, int root, float *d_full_grid,
                                     void *const *streams) {
    if (!plans || ndev < 1 || !d_points || !d_slabs || !h_cuts || !streams) { set_error("bad arguments"); return STKDE_EINVAL; }
    for (int d = 0; d < ndev; ++d)
        if (!plans[d]) { set_error("plans[%d] is NULL", d); return STKDE_EINVAL; }
    if (h_cuts[0] < 0) {
        int rc = stkde_slab_partition(plans[0], d_points[0], n, ndev, h_cuts, streams[0]);
        if (rc) return rc;
    }
    for (int d = 0; d < ndev; ++d) {
        if (h_cuts[d + 1] <= h_cuts[d]) continue;   // empty slab
        int rc = stkde_compute_slab(plans[d], d_points[d], n, n, h_cuts[d], h_cuts[d + 1], d_slabs[d], streams[d]);
        if (rc) return rc;
    }
    if (d_full_grid) {
        if (root < 0 || root >= ndev) { set_error("root out of range"); return STKDE_EINVAL; }
        stkde_plan_s *pr = plans[root];
        CK(cudaSetDevice(pr->device));
        cudaStream_t rs = (cudaStream_t)streams[root];
        for (int d = 0; d < ndev; ++d) {
            if (h_cuts[d + 1] <= h_cuts[d]) continue;
            if (plans[d]->device != pr->device) {
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, pr->device, plans[d]->device));
                if (!can) { set_error("device %d cannot access device %d", pr->device, plans[d]->device); return STKDE_ECUDA; }
                cudaError_t e = cudaDeviceEnablePeerAccess(plans[d]->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
                cudaEvent_t ev;
                CK(cudaSetDevice(plans[d]->device));
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, (cudaStream_t)streams[d]));
                CK(cudaSetDevice(pr->device));
                CK(cudaStreamWaitEvent(rs, ev, 0));
                cudaEventDestroy(ev);
            } else if (streams[d] != streams[root]) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, (cudaStream_t)streams[d]));
                CK(cudaStreamWaitEvent(rs, ev, 0));
                cudaEventDestroy(ev);
            }
            int rc = launch_gather(d_slabs[d], pr->g.Gx, pr->g.Gy, pr->g.Gt, h_cuts[d], h_cuts[d + 1], d_full_grid, rs);
            if (rc) { set_error("gather launch failed"); return rc; }
        }
    }
    return STKDE_OK;
}

// X-slab variant: device d computes rows [h_cuts[d], h_cuts[d+1]); a slab is a contiguous
// block of the full layout, so the gather is one peer copy per device into the root's grid.
extern "C" int stkde_compute_sharded_x(stkde_plan_t *plans, int ndev, const float *const *d_points, int64_t n,
                                       float *const *d_slabs, int64_t *h_cuts, int root, float *d_full_grid,
                                       void *const *streams) {
    // d_slabs == NULL: the fused gather -- every device's tile kernel stores its rows straight into
    // d_full_grid on the root (peer access enabled here), no slab buffers and no copies
    const bool fused = d_slabs == nullptr;
    if (!plans || ndev < 1 || !d_points || !h_cuts || !streams || (fused && !d_full_grid)) {
        set_error("bad arguments");
        return STKDE_EINVAL;
    }
    for (int d = 0; d < ndev; ++d)
        if (!plans[d]) { set_error("plans[%d] is NULL", d); return STKDE_EINVAL; }
    if (fused && (root < 0 || root >= ndev)) { set_error("root out of range"); return STKDE_EINVAL; }
    if (h_cuts[0] < 0) {
        int rc = stkde_xslab_partition(plans[0], d_points[0], n, ndev, h_cuts, streams[0]);
        if (rc) return rc;
    }
    for (int d = 0; d < ndev; ++d) {
        if (h_cuts[d + 1] <= h_cuts[d]) continue;   // empty slab
        float *dst = d_slabs ? d_slabs[d] : nullptr;
        if (fused) {
            const int rdev = plans[root]->device, ddev = plans[d]->device;
            if (ddev != rdev) {
                CK(cudaSetDevice(ddev));
                const cudaError_t e = cudaDeviceEnablePeerAccess(rdev, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    set_error("peer access %d -> %d: %s", ddev, rdev, cudaGetErrorString(e));
                    return STKDE_ECUDA;
                }
                cudaGetLastError();
            }
            dst = d_full_grid + h_cuts[d] * (int64_t)plans[root]->g.Gy * plans[root]->g.Gt;
        }
        int rc = stkde_compute_xslab(plans[d], d_points[d], n, n, h_cuts[d], h_cuts[d + 1], dst, streams[d]);
        if (rc) return rc;
    }
    if (fused) {   // the root's stream waits for every other device's stores
        stkde_plan_s *pr = plans[root];
        for (int d = 0; d < ndev; ++d) {
            if (h_cuts[d + 1] <= h_cuts[d] || streams[d] == streams[root]) continue;
            cudaEvent_t ev;
            CK(cudaSetDevice(plans[d]->device));
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, (cudaStream_t)streams[d]));
            CK(cudaSetDevice(pr->device));
            CK(cudaStreamWaitEvent((cudaStream_t)streams[root], ev, 0));
            cudaEventDestroy(ev);
        }
        return STKDE_OK;
    }
    if (d_full_grid) {
        if (root < 0 || root >= ndev) { set_error("root out of range"); return STKDE_EINVAL; }
        stkde_plan_s *pr = plans[root];
        CK(cudaSetDevice(pr->device));
        cudaStream_t rs = (cudaStream_t)streams[root];
        const size_t row = (size_t)pr->g.Gy * pr->g.Gt * sizeof(float);
        for (int d = 0; d < ndev; ++d) {
            if (h_cuts[d + 1] <= h_cuts[d]) continue;
            if (streams[d] != streams[root]) {
                cudaEvent_t ev;
                CK(cudaSetDevice(plans[d]->device));
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, (cudaStream_t)streams[d]));
                CK(cudaSetDevice(pr->device));
                CK(cudaStreamWaitEvent(rs, ev, 0));
                cudaEventDestroy(ev);
            }
            char *dst = reinterpret_cast<char *>(d_full_grid) + (size_t)h_cuts[d] * row;
            const size_t bytes = (size_t)(h_cuts[d + 1] - h_cuts[d]) * row;
            CK(cudaMemcpyPeerAsync(dst, pr->device, d_slabs[d], plans[d]->device, bytes, rs));
        }
    }
    return STKDE_OK;
}

extern "C" int stkde_plan_check_flags(stkde_plan_t p, uint32_t *flags) {
    if (!p || !flags) { set_error("NULL argument"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    CK(cudaDeviceSynchronize());
    int f = 0;
    CK(cudaMemcpy(&f, p->counters + 1, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(p->counters + 1, 0, sizeof(int)));
    *flags = (uint32_t)f & (STKDE_FLAG_NONFINITE | STKDE_FLAG_WORKLIST | STKDE_FLAG_BANDWIDTH);
    return STKDE_OK;
}

extern "C" int stkde_plan_check(stkde_plan_t p) {
    uint32_t flags = 0;
    const int rc = stkde_plan_check_flags(p, &flags);
    if (rc) return rc;
    if (!flags) return STKDE_OK;
    // every raised condition is named in the message; the code is the most severe one
    char msg[400] = "";
    if (flags & STKDE_FLAG_WORKLIST) strcat(msg, "internal work-list capacity exceeded; ");
    if (flags & STKDE_FLAG_NONFINITE) strcat(msg, "non-finite point coordinate(s) were skipped; ");
    if (flags & STKDE_FLAG_BANDWIDTH) strcat(msg, "point(s) with a bandwidth outside (0, plan hs] x (0, plan ht] were skipped; ");
    msg[strlen(msg) - 2] = 0;
    set_error("%s", msg);
    if (flags & STKDE_FLAG_WORKLIST) return STKDE_ECUDA;
    if (flags & STKDE_FLAG_NONFINITE) return STKDE_ENONFINITE;
    return STKDE_EBANDWIDTH;
}

extern "C" int stkde_plan_info(stkde_plan_t p, stkde_plan_info_t *info) {
    if (!p || !info) { set_error("NULL argument"); return STKDE_EINVAL; }
    info->Bx = BX; info->By = p->g.BY; info->Bt = p->g.BT;
    info->Hs = p->g.Hs; info->Ht = p->g.Ht;
    info->ntiles = p->ntiles;
    info->workspace_bytes = (int64_t)p->ws_bytes;
    info->last_own_launches = p->last_own_launches;
    info->last_cub_calls = p->last_cub_calls;
    info->tile_threads = p->tile_threads;
    info->tile_ctas_per_sm = p->ctas_per_sm;
    info->num_sms = p->num_sms;
    info->chunk_candidates = p->chunk;
    info->tile_layers_per_thread = p->CT;
    info->engine = p->engine;
    return STKDE_OK;
}

extern "C" int stkde_plan_enable_kernel_timing(stkde_plan_t p, int enable) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    if (enable && !p->tev) {
        const int cap = 4096;
        p->tev = (cudaEvent_t *)calloc(2 * cap, sizeof(cudaEvent_t));
        if (!p->tev) { set_error("host allocation failed"); return STKDE_ENOMEM; }
        for (int i = 0; i < 2 * cap; ++i) CK(cudaEventCreate(&p->tev[i]));
        p->tev_cap = cap;
    }
    p->tev_used = 0;
    p->timing = enable ? 1 : 0;
    p->kernel_ms = 0;
    p->kernel_launches = 0;
    return STKDE_OK;
}

extern "C" int stkde_plan_kernel_ms(stkde_plan_t p, double *ms_total, int64_t *launches) {
    if (!p) { set_error("plan is NULL"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    harvest_timing(p);
    if (ms_total) *ms_total = p->kernel_ms;
    if (launches) *launches = p->kernel_launches;
    return STKDE_OK;
}

extern "C" int stkde_plan_mma_stats(stkde_plan_t p, int64_t *mma_columns, int64_t *kblocks) {
    if (!p || !mma_columns || !kblocks) { set_error("NULL argument"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    CK(cudaDeviceSynchronize());
    unsigned long long v[2] = {0ull, 0ull};
    CK(cudaMemcpy(v, p->counters + 2, sizeof v, cudaMemcpyDeviceToHost));
    CK(cudaMemset(p->counters + 2, 0, sizeof v));
    *mma_columns = (int64_t)v[0];
    *kblocks = (int64_t)v[1];
    return STKDE_OK;
}

#if STKDE_TC_DIAG
// development diagnostics (paper_1705_09366_b200/csrc/stkde_diag.h): only in a
// -DSTKDE_TC_DIAG=1 build (scripts/build_variant.py), not part of the product ABI
extern "C" int stkde_plan_tc_profile(stkde_plan_t p, uint64_t *out32) {
    if (!p || !out32) { set_error("NULL argument"); return STKDE_EINVAL; }
    CK(cudaSetDevice(p->device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out32, p->counters + 32, 31 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out32 + 31, p->counters + 96, sizeof(uint64_t), cudaMemcpyDeviceToHost));   // watchdog record
    CK(cudaMemset(p->counters + 32, 0, 32 * sizeof(uint64_t)));
    CK(cudaMemset(p->counters + 96, 0, sizeof(uint64_t)));
    return STKDE_OK;
}

extern "C" int stkde_plan_debug_progress(stkde_plan_t p, void *buf) {
    if (!p) { set_error("NULL argument"); return STKDE_EINVAL; }
    p->debug_progress = buf;
    return STKDE_OK;
}
#endif

extern "C" const char *stkde_strerror(int code) {
    switch (code) {
        case STKDE_OK: return "ok";
        case STKDE_EINVAL: return "invalid argument";
        case STKDE_ENOMEM: return "device allocation failed";
        case STKDE_ECUDA: return "CUDA error";
        case STKDE_ECAPACITY: return "n exceeds plan capacity (max_n)";
        case STKDE_ENONFINITE: return "non-finite point coordinate";
        case STKDE_EBANDWIDTH: return "per-point bandwidth outside the plan's range";
        case STKDE_ENCCL: return "NCCL unavailable or an NCCL call failed";
    }
    return "unknown error";
}

extern "C" const char *stkde_last_error(void) { return g_err; }
