/*
 * stkde.h -- C ABI of the B200 (sm_100a) space-time kernel density library.
 *
 * The library computes, for every voxel (X,Y,T) of a Gx x Gy x Gt grid,
 *
 *   f(X,Y,T) = 1/(n hs^2 ht) * sum_{i : sqrt((x-x_i)^2+(y-y_i)^2) < hs and |t-t_i| <= ht}
 *                  k_s(|x-x_i|/hs, |y-y_i|/hs) * k_t(|t-t_i|/ht)
 *
 * with (x,y,t) the voxel centre (x0 + (X+0.5) sres, ...), i.e. the density
 * of PAPER.md:120-121 (§2.1) with the kernels of PAPER.md:132-133 and the
 * gates of Alg. 1, accumulated point-major as PB-SYM
 * (Alg. 3): each point contributes the separable product
 * K_s(X,Y) * K_t(T) to every voxel of its cylinder.  The GPU computes the
 * same sum in gather form per voxel tile.
 *
 * Conventions for every call:
 *   - Pointers named d_* are DEVICE pointers on the plan's device; h_* are
 *     host pointers.  The caller owns all buffers; the plan owns only its
 *     internal workspace.
 *   - Points are float32 [n][3] = (x, y, t) in world units, row-major,
 *     read-only.  Non-finite coordinates are skipped and raise the plan's
 *     error flag (read with stkde_plan_check).
 *   - The density grid is float32 [Gx][Gy][Gt], linear index
 *     (X*Gy + Y)*Gt + T (T innermost; SPEC.md:48-54 layout, 4 B/voxel as in
 *     the paper's Table 2).  It is FULLY OVERWRITTEN (no
 *     need to zero it; there is no separate initialisation pass).
 *   - Calls that take a cudaStream_t (passed as void*) are asynchronous on
 *     that stream and never synchronise the host; they are CUDA-graph
 *     capturable.  Their return code reports validation / enqueue errors
 *     only; kernel faults surface at the caller's next synchronisation.
 *   - A plan must not be used concurrently from two streams.
 *   - Results are deterministic: identical inputs give bitwise identical
 *     grids.  A time slab (stkde_compute_slab) or x-slab (stkde_compute_xslab)
 *     is bitwise equal to the same block of the full-grid result: with the
 *     tcgen05 engine for any boundary (exact integer accumulation; each voxel
 *     rounded from its exact sum: int64 -> float, then x scale), with the
 *     short-window FP32 engine (WS) for any boundary (every voxel sums in
 *     candidate order), with the other FP32 engines for time-slab boundaries
 *     that are multiples of the tile height Bt.
 *   - Accuracy (float32 grids): |result - definition| <= 1e-5 of the grid's
 *     maximum and an exact support mask (value > 0), guaranteed where every
 *     bandwidth spans at least one voxel (hs >= sres, ht >= tres).  With a
 *     disc or window narrower than one voxel the maximum can lie far below one
 *     point's peak -- the scale of the fixed-point / FP32 factors -- and the
 *     bound can be missed (up to 1.9e-4 of the maximum over 1500 random
 *     plans; support still exact).  The temporal gate is decided in FP32: a
 *     pair within ~8e-6 (relative) of the window edge may be gated the other
 *     way, which changes a value by < 4e-6 of the maximum (K_t is zero at the
 *     edge) but can flip the support bit of such a voxel.  The float64 calls
 *     (stkde_compute_f64 ...) have neither limit.  DESIGN.md sections 5, 3.10.
 *   - Return codes: STKDE_OK (0) or a negative STKDE_E* value; the message
 *     of the most recent error on the calling thread is stkde_last_error().
 */
#ifndef STKDE_H_
#define STKDE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    STKDE_OK = 0,
    STKDE_EINVAL = -1,      /* invalid argument (message names the field)            */
    STKDE_ENOMEM = -2,      /* device allocation failed                              */
    STKDE_ECUDA = -3,       /* a CUDA runtime call failed                            */
    STKDE_ECAPACITY = -4,   /* n exceeds the plan's max_n                            */
    STKDE_ENONFINITE = -5,  /* some input coordinate was NaN/Inf (stkde_plan_check)  */
    STKDE_EBANDWIDTH = -6,  /* an adaptive call had a per-point bandwidth outside the
                               plan's range (stkde_plan_check)                      */
    STKDE_ENCCL = -7        /* NCCL unavailable or an NCCL call failed (gather)      */
};

/* Kernel pair (reading R1 in DESIGN.md). */
enum {
    STKDE_KERNEL_PRINTED = 0,   /* k_s = pi/2 (1-u)^2 (1-v)^2, k_t = 3/4 (1-w)^2 */
    STKDE_KERNEL_CLASSICAL = 1  /* k_s = 2/pi (1-u^2-v^2),     k_t = 3/4 (1-w^2)                    */
};

/* Tile-kernel engine (environment variable STKDE_ENGINE at plan creation;
 * default TC).  SIMT: FP32 FFMA2 accumulation in registers (16x16 columns).
 * TENSOR: the per-tile contraction on the legacy tensor-core path (mma.sync
 * m16n8k16, FP16 3-term split, FP32 accumulation; 16x16 columns) -- DESIGN.md
 * §3.5.  TC: the same contraction on 5th-generation tensor cores (tcgen05.mma
 * kind::i8, 23-bit fixed-point factors split into three 8-bit limbs, exact S32
 * accumulation in TMEM; M = 128 columns of a 16x8-column tile, A generated
 * into TMEM) -- DESIGN.md §3.5.  Hs > 120 falls back to TENSOR.  WS: short temporal windows
 * (H_t <= 8, H_s <= 120): FP32 FFMA2 accumulation of each point's window only, 16x16 columns x
 * 32 layers, two columns per thread, the window offset dispatched to compile-time accumulator
 * indices; other bandwidths fall back to TC.  All engines compute the same
 * sums within the parity tolerance; they differ in speed only. */
enum { STKDE_ENGINE_SIMT = 0, STKDE_ENGINE_TENSOR = 1, STKDE_ENGINE_TC = 2, STKDE_ENGINE_WS = 3 };

typedef struct stkde_plan_s *stkde_plan_t;

/* Create a plan on `device` (CUDA ordinal).  Grid origin (x0,y0,t0), voxel
 * sizes sres/tres > 0, grid Gx,Gy,Gt >= 1 and bandwidths hs, ht > 0 are in
 * world units (H_s = ceil(hs/sres), H_t = ceil(ht/tres)).
 * `max_n` bounds the point count of later calls and sizes the device
 * workspace, so compute calls never allocate.  The tile shape depends on the
 * engine (tcgen05: 16 x 8 columns x Bt = 64 or 128 layers; short-window FP32: 16 x 16
 * columns x 32 layers; legacy engines: 16 x 16 columns x Bt = 16, 32 or 64 from H_t);
 * read it back with stkde_plan_info.  Writes the
 * plan to *out.  Errors: STKDE_EINVAL (message names the field),
 * STKDE_ENOMEM, STKDE_ECUDA. */
int stkde_plan_create(stkde_plan_t *out, int device,
                      double x0, double y0, double t0,
                      double sres, double tres,
                      int64_t Gx, int64_t Gy, int64_t Gt,
                      double hs, double ht,
                      int kernel_kind, int64_t max_n);

/* Release the plan and its workspace (NULL is a no-op). */
void stkde_plan_destroy(stkde_plan_t plan);

/* Full grid: d_points [n][3] -> d_grid [Gx][Gy][Gt].  Normalisation
 * 1/(n hs^2 ht) uses this n; n = 0 writes zeros. */
int stkde_compute(stkde_plan_t plan, const float *d_points, int64_t n,
                  float *d_grid, void *stream);

/* Time slab [t_begin, t_end) of the grid, 0 <= t_begin < t_end <= Gt:
 * d_slab is float32 [Gx][Gy][t_end - t_begin] (T innermost).  `n_norm` is
 * the n of the normalisation (the GLOBAL point count when the caller shards
 * one grid over several devices); the point set must be the full one --
 * points whose temporal window misses the slab are culled on the device, so
 * the halo is implicit.  Used by the multi-GPU time-slab decomposition
 * (the temporal split of PAPER.md:415-433). */
int stkde_compute_slab(stkde_plan_t plan, const float *d_points, int64_t n,
                       int64_t n_norm, int64_t t_begin, int64_t t_end,
                       float *d_slab, void *stream);

/* ---- CUDA graphs (launch-bound small grids: one launch instead of ~20) ----
 * stkde_graph_create captures ONE stkde_compute_slab call (arguments as there; the full
 * grid is t_begin = 0, t_end = Gt, n_norm = n) on a private stream into an instantiated
 * CUDA graph; nothing runs at creation.  stkde_graph_launch replays it on `stream`: the
 * whole pass (binning, work list, tile kernel) as one graph launch, reading d_points and
 * writing d_out AS THEY ARE at launch time (the caller may refill the point buffer between
 * launches; n, the slab and the buffers are fixed at capture).  The graph uses the plan's
 * workspace: the plan must outlive it, and a graph must not run concurrently with another
 * call on the same plan.  Errors: as stkde_compute_slab, STKDE_ECUDA if capture or
 * instantiation fails, STKDE_ENOMEM. */
typedef struct stkde_graph_s *stkde_graph_t;
int stkde_graph_create(stkde_plan_t plan, const float *d_points, int64_t n, int64_t n_norm,
                       int64_t t_begin, int64_t t_end, float *d_out, stkde_graph_t *out);
/* The same for one stkde_compute_xslab call (rows [x_begin, x_end) into d_xslab). */
int stkde_graph_create_xslab(stkde_plan_t plan, const float *d_points, int64_t n, int64_t n_norm,
                             int64_t x_begin, int64_t x_end, float *d_xslab, stkde_graph_t *out);
int stkde_graph_launch(stkde_graph_t graph, void *stream);
void stkde_graph_destroy(stkde_graph_t graph);

/* Cost-balanced, Bt-aligned time-slab cuts for `nparts` devices (tcgen05
 * engine: when nparts exceeds ceil(Gt/Bt) the cut granularity is halved down
 * to 32 layers -- its slabs are bitwise equal to the full grid at any boundary).
 * Synchronous (reads a per-layer cost histogram back to the host).  Writes
 * h_cuts[0..nparts] with h_cuts[0] = 0 and h_cuts[nparts] = Gt; empty
 * slabs are never produced while nparts <= ceil(Gt/granularity).  Cost per layer
 * T = alpha * (Gx*Gy*4 B)/B_hbm + beta * 2*W(T)/P_fp32 where W(T) is the
 * number of (point, column) pairs whose window contains T. */
int stkde_slab_partition(stkde_plan_t plan, const float *d_points, int64_t n,
                         int nparts, int64_t *h_cuts, void *stream);

/* Host-only half of stkde_slab_partition (no CUDA calls): cuts from a
 * histogram h_hist_T[0..Gt) of the points' voxel layers T_i (clamped into
 * [0, Gt)).  Bt is the plan's tile height, Ht = ceil(ht/tres), rs = hs/sres.
 * Writes h_cuts[0..nparts]; returns STKDE_EINVAL on bad sizes. */
int stkde_slab_cuts(int64_t Gx, int64_t Gy, int64_t Gt, int Bt, int Ht, double rs,
                    const int64_t *h_hist_T, int nparts, int64_t *h_cuts);

/* Exact number C of gated (point, voxel) pairs whose voxel lies in layers
 * [t_begin, t_end) -- the "contributions" of the metric.  Writes one int64
 * to d_count (device).  Asynchronous. */
int stkde_count_contributions(stkde_plan_t plan, const float *d_points, int64_t n,
                              int64_t t_begin, int64_t t_end, int64_t *d_count,
                              void *stream);
/* The same count restricted to the voxels of rows [x_begin, x_end) and layers
 * [t_begin, t_end) (an x-slab's or a time slab's own contributions: the per-rank work of
 * a sharded run).  0 <= x_begin < x_end <= Gx, 0 <= t_begin < t_end <= Gt, else
 * STKDE_EINVAL.  Asynchronous. */
int stkde_count_contributions_box(stkde_plan_t plan, const float *d_points, int64_t n,
                                  int64_t x_begin, int64_t x_end, int64_t t_begin, int64_t t_end,
                                  int64_t *d_count, void *stream);

/* ---- Adaptive bandwidth (reading R15) ----
 * PAPER.md:1060-1062 names "a bandwidth that adapts to the density of
 * population" as future work.  Point i carries its own (hs_i, ht_i) and
 *
 *   f(X,Y,T) = 1/n * sum_{i : d < hs_i and |dt| <= ht_i}
 *                  k_s(|dx|/hs_i, |dy|/hs_i) * k_t(|dt|/ht_i) / (hs_i^2 ht_i),
 *
 * i.e. PAPER.md:120-121 with the bandwidths inside the sum (identical to it when
 * every hs_i = hs, ht_i = ht).  d_bw is float32 [n][2] = (hs_i, ht_i) in world
 * units on the plan's device, read-only; every pair must satisfy
 * 0 < hs_i <= hs and 0 < ht_i <= ht of the plan (the plan's bandwidths size the
 * binning reach).  A point violating this is skipped and raises the plan's
 * error flag: stkde_plan_check returns STKDE_EBANDWIDTH.  Same grid layout,
 * overwrite, asynchrony, determinism and slab rules as stkde_compute /
 * stkde_compute_slab.  Needs the tcgen05 engine (H_s <= 120); otherwise
 * STKDE_EINVAL.
 * Accuracy: the fixed-point factors are scaled by max_i W_i s_i, W_i = 1/(hs_i^2 ht_i)
 * and s_i the point's spatial factor at its nearest voxel centre; each contribution
 * carries <= 8.3e-7 of that full scale.  The result is within 1e-5 of the grid's
 * maximum whenever every hs_i >= sres and ht_i >= tres; with sub-voxel per-point
 * bandwidths a maximum built from hundreds of far smaller contributions can deviate
 * more (up to 1.5e-4 of the maximum over 1500 random draws, tests/test_gpu_fuzz.py;
 * DESIGN.md section 5).  stkde_compute_adaptive_slab_f64 has no such scale. */
int stkde_compute_adaptive(stkde_plan_t plan, const float *d_points, const float *d_bw, int64_t n,
                           float *d_grid, void *stream);
int stkde_compute_adaptive_slab(stkde_plan_t plan, const float *d_points, const float *d_bw, int64_t n,
                                int64_t n_norm, int64_t t_begin, int64_t t_end, float *d_slab, void *stream);
/* Exact gated-pair count C of the adaptive estimator (per-point gates). */
int stkde_count_contributions_adaptive(stkde_plan_t plan, const float *d_points, const float *d_bw, int64_t n,
                                       int64_t t_begin, int64_t t_end, int64_t *d_count, void *stream);

/* ---- FP64 output (SPEC.md:48-54 keeps the volume in FP64) ----
 * The same density as stkde_compute / stkde_compute_slab / stkde_compute_adaptive_slab
 * (same arguments, slab and normalisation rules), written as float64
 * [Gx][Gy][t_end - t_begin] (T innermost; d_grid / d_slab on the plan's device,
 * fully overwritten).  Every (point, voxel) term is evaluated in FP64 with the IEEE
 * operation sequence of Alg. 1 -- voxel centre
 * x0 + (X + 0.5) sres, gates sqrt(dx^2 + dy^2) < hs and |dt| <= ht, the printed or
 * classical kernels -- without contraction, so the gate decisions
 * and each term equal a plain FP64 evaluation of the definition; the per-voxel sum
 * runs in a fixed order (home bucket, then ascending point index), the sum is divided
 * by n hs^2 ht at the end (adaptive: each term by hs_i^2 ht_i, the sum by n).
 * Deterministic; slabs are bitwise equal to the full grid's layers.  FP64-pipe bound
 * (DESIGN.md §3.8): an accuracy option, not the throughput path.  Any engine for
 * the fixed bandwidth; the adaptive form needs the tcgen05 engine (else STKDE_EINVAL).
 * Asynchronous; the non-finite / bandwidth flags as for the FP32 calls. */
int stkde_compute_f64(stkde_plan_t plan, const float *d_points, int64_t n, double *d_grid, void *stream);
int stkde_compute_slab_f64(stkde_plan_t plan, const float *d_points, int64_t n, int64_t n_norm,
                           int64_t t_begin, int64_t t_end, double *d_slab, void *stream);
int stkde_compute_adaptive_slab_f64(stkde_plan_t plan, const float *d_points, const float *d_bw, int64_t n,
                                    int64_t n_norm, int64_t t_begin, int64_t t_end, double *d_slab,
                                    void *stream);

/* ---- Multi-bandwidth sweep (Fig. 1, PAPER.md:135-146:
 * the same events viewed at several bandwidths; the Lb/Hb/VHb instances of
 * PAPER.md:651-653) ----
 * Bins the points ONCE at the plan's bandwidths and computes nbw full grids,
 * grid k for bandwidths (h_hs[k], h_ht[k]) (host arrays, world units,
 * 0 < h_hs[k] <= hs, 0 < h_ht[k] <= ht), each normalised by 1/(n h_hs[k]^2
 * h_ht[k]).  d_grids is a host array of nbw device pointers, each float32
 * [Gx][Gy][Gt], fully overwritten.  Asynchronous on `stream`; grid k equals
 * stkde_compute on a plan created with (h_hs[k], h_ht[k]) within the parity
 * tolerance.  Errors: STKDE_EINVAL (bad bandwidth / NULL grid), STKDE_ECAPACITY. */
int stkde_compute_sweep(stkde_plan_t plan, const float *d_points, int64_t n, int nbw, const double *h_hs,
                        const double *h_ht, float *const *d_grids, void *stream);

/* ---- X-slabs: the multi-GPU partition along X ----
 * stkde_compute_xslab computes grid rows [x_begin, x_end) -- a contiguous block of
 * the [Gx][Gy][Gt] layout -- into d_xslab (float32 [x_end - x_begin][Gy][Gt],
 * fully overwritten), normalised with n_norm (the global n).  x_begin and x_end
 * (unless = Gx) must be multiples of 16 (the tile width): the slab's tiles and their
 * candidate lists are then the full grid's, so the result is bitwise equal to those
 * rows of stkde_compute and the work splits without overhead.  tcgen05 engine only
 * (else STKDE_EINVAL).  Asynchronous. */
int stkde_compute_xslab(stkde_plan_t plan, const float *d_points, int64_t n, int64_t n_norm,
                        int64_t x_begin, int64_t x_end, float *d_xslab, void *stream);
/* The same for the adaptive estimator (d_bw as in stkde_compute_adaptive). */
int stkde_compute_adaptive_xslab(stkde_plan_t plan, const float *d_points, const float *d_bw, int64_t n,
                                 int64_t n_norm, int64_t x_begin, int64_t x_end, float *d_xslab, void *stream);
/* Cost-balanced x cuts (multiples of 16, h_cuts[0] = 0, h_cuts[nparts] = Gx); the cost of
 * column X is Gy*Gt*4 B / B_hbm + 2 W(X) / P_fp32, W(X) = sum over the points with
 * |X - X_i| <= rs + 8 of 2 rs (2 rt + 1) -- the tile kernel's candidates.  stkde_xslab_partition reads the X_i histogram from the device
 * (synchronous); stkde_xslab_cuts is its host-only half (rs = hs/sres, rt = ht/tres). */
int stkde_xslab_partition(stkde_plan_t plan, const float *d_points, int64_t n, int nparts, int64_t *h_cuts,
                          void *stream);
int stkde_xslab_cuts(int64_t Gx, int64_t Gy, int64_t Gt, double rs, double rt, const int64_t *h_hist_X, int nparts,
                     int64_t *h_cuts);

/* Single-process multi-device driver: plans[d] lives on device d's ordinal,
 * d_points[d] holds the full point set on that device, d_slabs[d] receives
 * slab [h_cuts[d], h_cuts[d+1]).  If d_full_grid is non-NULL it must be on
 * plans[root]'s device and receives the whole grid, gathered over peer
 * memory (NVLink) by a kernel on the root after all slabs finish.
 * streams[d] are per-device streams.  Asynchronous except for the cut
 * computation (stkde_slab_partition on plans[0]) when h_cuts[0] < 0. */
int stkde_compute_sharded(stkde_plan_t *plans, int ndev,
                          const float *const *d_points, int64_t n,
                          float *const *d_slabs, int64_t *h_cuts,
                          int root, float *d_full_grid, void *const *streams);

/* X-slab counterpart of stkde_compute_sharded: d_slabs[d] receives rows
 * [h_cuts[d], h_cuts[d+1]) (float32 [rows][Gy][Gt]); cuts from stkde_xslab_partition
 * on plans[0] when h_cuts[0] < 0; the optional gather is one peer copy per device
 * (each x-slab is a contiguous block of the full grid).  d_slabs == NULL fuses the gather
 * into the compute: each device's tile kernel stores its rows straight into d_full_grid on
 * plans[root]'s device over peer memory (peer access is enabled by the call), with no slab
 * buffers and no copies; streams[root] then waits for every device's stream.  Same
 * stream/asynchrony rules. */
int stkde_compute_sharded_x(stkde_plan_t *plans, int ndev, const float *const *d_points, int64_t n,
                            float *const *d_slabs, int64_t *h_cuts, int root, float *d_full_grid,
                            void *const *streams);

/* Conditions raised on the device by earlier calls (bit mask, see stkde_plan_check_flags). */
enum {
    STKDE_FLAG_NONFINITE = 1,   /* a point had a non-finite coordinate (skipped)                 */
    STKDE_FLAG_WORKLIST = 2,    /* internal work-list capacity exceeded (a library bug)          */
    STKDE_FLAG_BANDWIDTH = 4    /* an adaptive call had a per-point bandwidth outside the plan's
                                   range (skipped)                                               */
};

/* Synchronises the plan's device, writes every condition raised since the last check to
 * *flags (STKDE_FLAG_* bits, 0 = none) and clears them.  Errors: STKDE_EINVAL (NULL),
 * STKDE_ECUDA. */
int stkde_plan_check_flags(stkde_plan_t plan, uint32_t *flags);

/* Synchronises the plan's device and clears the flags; returns STKDE_OK if none was
 * raised, else the code of the most severe one (STKDE_ECUDA for a work-list overflow,
 * then STKDE_ENONFINITE, then STKDE_EBANDWIDTH) with stkde_last_error() naming EVERY
 * raised condition. */
int stkde_plan_check(stkde_plan_t plan);

/* Plan facts: tile shape, H, workspace bytes, number of kernels the last
 * compute launched (library kernels, CUB kernels counted separately). */
typedef struct {
    int32_t Bx, By, Bt;
    int32_t Hs, Ht;
    int64_t ntiles;
    int64_t workspace_bytes;
    int32_t last_own_launches;
    int32_t last_cub_calls;
    int32_t tile_threads;
    int32_t tile_ctas_per_sm;
    int32_t num_sms;
    int32_t chunk_candidates;
    int32_t tile_layers_per_thread;   /* CT: each thread owns 4 columns x CT layers (SIMT engine) */
    int32_t engine;                   /* STKDE_ENGINE_* of the tile kernel */
} stkde_plan_info_t;
int stkde_plan_info(stkde_plan_t plan, stkde_plan_info_t *info);

/* Time the tile kernel of subsequent compute calls with CUDA events recorded
 * on the caller's stream; stkde_plan_kernel_ms sums the elapsed ms of all
 * timed launches since enable (synchronises on the last event). */
int stkde_plan_enable_kernel_timing(stkde_plan_t plan, int enable);
int stkde_plan_kernel_ms(stkde_plan_t plan, double *ms_total, int64_t *launches);

/* Instrumentation of the tcgen05 engine: since the last call,
 * the sum over issued k-blocks of the MMA width N (each k-block issues 7
 * tcgen05.mma kind::i8 of 128 x N x 32) and the number of k-blocks (accumulated in
 * registers, two atomics per generator team when the persistent CTA exits); both are
 * reset.  Synchronises the device.  Zero for the other engines. */
int stkde_plan_mma_stats(stkde_plan_t plan, int64_t *mma_columns, int64_t *kblocks);

/* Per-phase device time of the pipeline (SURVEY.md §5 tracing; the GPU counterpart of
 * the paper's init / compute breakdown, Fig. 6).  Phases, in enqueue
 * order: PREP = point prep + home-bucket count (k_prep), SORT = the stable radix sort
 * (FP32 engines and the FP64 path; 0 for the tcgen05 engine's counting sort), SCAN =
 * bucket offsets, SCATTER = records into bucket order, CHORDS = the disc-chord table,
 * WORKLIST = tile counts + order + chunking, TILES = the tile kernel, GATHER = the
 * whole-grid gather (stkde_gather_*).  Every call also opens NVTX ranges named
 * "stkde.<phase>" around the host-side enqueue of each phase (no cost without a tool). */
enum {
    STKDE_PHASE_PREP = 0,
    STKDE_PHASE_SORT = 1,
    STKDE_PHASE_SCAN = 2,
    STKDE_PHASE_SCATTER = 3,
    STKDE_PHASE_CHORDS = 4,
    STKDE_PHASE_WORKLIST = 5,
    STKDE_PHASE_TILES = 6,
    STKDE_PHASE_GATHER = 7,
    STKDE_NPHASES = 8
};
/* enable != 0: subsequent calls record a CUDA event on their stream at every phase end
 * (skipped while the stream is being captured into a graph); resets the sums.
 * stkde_plan_phase_ms writes the summed ms of each phase since enable to
 * ms[STKDE_NPHASES] and the number of timed calls to *calls (synchronises on the last
 * event).  stkde_phase_name(i) = "prep", "sort", ... (NULL outside [0, STKDE_NPHASES)).
 * Errors: STKDE_EINVAL (NULL plan / ms), STKDE_ECUDA, STKDE_ENOMEM. */
int stkde_plan_enable_phase_timing(stkde_plan_t plan, int enable);
int stkde_plan_phase_ms(stkde_plan_t plan, double *ms, int64_t *calls);
const char *stkde_phase_name(int phase);

/* ---- NCCL gather of per-rank slabs (one process per GPU) ----
 * The hot path has no collective (slabs are independent); the optional whole-grid
 * gather to one rank runs inside the library over NCCL point-to-point (NVLink /
 * NVSwitch).  NCCL is loaded at first use (dlopen "libnccl.so.2"); without it these
 * calls return STKDE_ENCCL and everything else works.
 *
 * stkde_nccl_unique_id: rank 0 creates the 128-byte id (h_id, host) and ships it to the
 * other ranks out of band (e.g. a torch.distributed broadcast).
 * stkde_plan_comm_init: every rank creates the communicator on its plan's device
 * (collective over the nranks ranks: each must call it; blocking).  The plan owns the
 * communicator and destroys it in stkde_plan_destroy.  Re-init replaces it. */
int stkde_nccl_unique_id(void *h_id /* 128 bytes */);
int stkde_plan_comm_init(stkde_plan_t plan, int nranks, int rank, const void *h_id /* 128 bytes */);
/* X-slab gather: rank r holds rows [h_cuts[r], h_cuts[r+1]) as float32 [rows][Gy][Gt]
 * (stkde_compute_xslab).  Each is a contiguous block of the full grid, so the root
 * receives every slab straight into d_full (float32 [Gx][Gy][Gt], root only; ignored on
 * the other ranks) with no unpack; a root slab already in place (d_slab == its block
 * of d_full) is not copied.  h_cuts (host, nranks+1 entries, ascending, 0 .. Gx) must be
 * the same on every rank.  Collective over the communicator's ranks; asynchronous on
 * `stream`.  Errors: STKDE_EINVAL (no communicator, bad cuts or root, NULL slab),
 * STKDE_ENCCL (an NCCL call failed; stkde_last_error names it). */
int stkde_gather_xslab(stkde_plan_t plan, const float *d_slab, const int64_t *h_cuts, int root, float *d_full,
                       void *stream);
/* Time-slab gather: rank r holds layers [h_cuts[r], h_cuts[r+1]) as float32
 * [Gx][Gy][Ts] (stkde_compute_slab).  Slabs are strided in the T-innermost full grid,
 * so the root receives the other ranks' slabs into a staging buffer the plan allocates
 * on first use (sum of their sizes) and unpacks them with one kernel per slab; its own
 * slab is unpacked straight from d_slab.  Same rules and errors as stkde_gather_xslab
 * (plus STKDE_ENOMEM for the staging buffer). */
int stkde_gather_slab(stkde_plan_t plan, const float *d_slab, const int64_t *h_cuts, int root, float *d_full,
                      void *stream);

/* ---- Direct x-slab gather over peer memory (CUDA IPC; one process per GPU) ----
 * The fused alternative to stkde_gather_xslab: the root exports its full grid once, every
 * rank maps it and passes its rows of the ROOT's grid as d_xslab to stkde_compute_xslab,
 * so the tile kernel's epilogue stores the slab straight into the root's memory over
 * NVLink / NVSwitch while the rank computes (no staging, no separate collective; the
 * caller synchronises its stream and then the ranks, e.g. a torch.distributed barrier,
 * before the root reads the grid).  An output on another device is written with plain
 * warp-coalesced stores (no TMA tensor map over peer memory).
 * stkde_ipc_get_handle: the 64-byte cudaIpcMemHandle of the allocation holding d_ptr
 * (device memory of the calling process) and d_ptr's byte offset in it.
 * stkde_ipc_open: maps a handle of another process on `device` (peer access enabled
 * lazily); *d_base = the allocation's base (add the offset).  stkde_ipc_close unmaps it.
 * Errors: STKDE_EINVAL (NULL arguments), STKDE_ECUDA (the CUDA call's message in
 * stkde_last_error; a handle cannot be opened in the process that exported it). */
int stkde_ipc_get_handle(const void *d_ptr, void *h_handle /* 64 bytes */, int64_t *offset);
int stkde_ipc_open(int device, const void *h_handle /* 64 bytes */, void **d_base);
int stkde_ipc_close(void *d_base);

/* Human-readable message for a return code / the last error of this thread. */
const char *stkde_strerror(int code);
const char *stkde_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* STKDE_H_ */
