/*
 * stkde_oracle.c -- FP64 CPU oracle for space-time kernel density estimation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_1705_09366_b200/ and never calls it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, §2.1-§3.2):
 *
 *   f(X,Y,T) = 1/(n hs^2 ht) * sum_{i : sqrt((x-x_i)^2+(y-y_i)^2) < hs  and  |t-t_i| <= ht}
 *                  k_s(|x-x_i|/hs, |y-y_i|/hs) * k_t(|t-t_i|/ht)
 *
 *   - density formula: PAPER.md:120-121 (§2.1);
 *   - kernels as printed: k_s(u,v) = pi/2 (1-u)^2 (1-v)^2, k_t(w) = 3/4 (1-w)^2
 *     (PAPER.md:132-133); the classical Epanechnikov pair (2/pi)(1-u^2-v^2),
 *     3/4 (1-w^2) behind kernel = 1 (reading R1);
 *   - gates exactly as Alg. 1 prints them: spatial strict sqrt(...) < hs,
 *     temporal inclusive |t_i - t| <= ht (reading R3);
 *   - (x,y,t) of voxel (X,Y,T) is the voxel centre, x = x0 + (X+0.5) sres
 *     (reading R5);
 *   - sum of k_s k_t per voxel, divided by n hs^2 ht at the end (Alg. 1,
 *     PAPER.md:202-216); n = 0 gives zeros without dividing;
 *   - G and H from PAPER.md:158-166: H_s = ceil(hs/sres), H_t = ceil(ht/tres).
 *
 * oracle_vb   : Alg. 1 (VB) written out -- every voxel, every point.
 * oracle_pb   : the same sum organised point-major as Alg. 3 (PB-SYM,
 *               PAPER.md:302-335): per point the temporal line K_t[T] is formed
 *               once, then every (X,Y) of the box X_i +- H_s, Y_i +- H_s
 *               (Alg. 2/3 loop bounds, with T_i +- H_t for the printed
 *               "T_i - T_s .. T_i + H_s" typo, reading R4) is gated and
 *               accumulated.  Parallelism is PB-SYM-DD with an A x 1 x 1 split
 *               (PAPER.md:387-413): thread chunks own disjoint X ranges and
 *               visit their candidate points in input order, so every voxel
 *               sums in input order and the result is bitwise identical to
 *               oracle_vb and independent of the thread count.
 * oracle_vb_voxels : Alg. 1 at a caller-chosen list of voxels (full-size sampling).
 *
 * Adaptive bandwidth (PAPER.md:1060-1062 names "a bandwidth
 * that adapts to the density of population" as future work; reading R15 in
 * DESIGN.md): point i carries its own (hs_i, ht_i) and the density is the
 * sample-point estimator
 *
 *   f(X,Y,T) = 1/n * sum_{i : d < hs_i and |dt| <= ht_i}
 *                  k_s(|dx|/hs_i, |dy|/hs_i) k_t(|dt|/ht_i) / (hs_i^2 ht_i),
 *
 * which is PAPER.md:120-121 with h_s, h_t moved inside the sum (equal to it
 * when every hs_i = hs, ht_i = ht).  oracle_*_adaptive take bw = float[n][2]
 * (hs_i, ht_i), widened exactly to FP64; the grid's hs/ht only bound the loops
 * (every hs_i <= hs, ht_i <= ht; violations return -3).  Each term is
 * (k_s k_t) / (hs_i*hs_i*ht_i), summed in input order, then divided by n.
 *
 * Optional outputs: per-voxel ambiguity flag and slack (reading R10/R11):
 * a (point, voxel) pair is ambiguous when |sqrt(d^2)/hs - 1| <= 1e-6 or
 * ||dt|/ht - 1| <= 1e-6 while the other coordinate is inside (or itself
 * ambiguous); slack is the sum of such pairs' |k_s k_t|/(n hs^2 ht).
 * `contributions` counts the gated (point, voxel) pairs (the metric's C).
 *
 * Compiled with -O2 -ffp-contract=off so every gate expression is the plain
 * IEEE sequence written here.  Parity unpinned: none -- see tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double x0, y0, t0;      /* grid origin (world units)                 */
    double sres, tres;      /* voxel size in space / time                */
    double hs, ht;          /* bandwidths (world units)                  */
    int64_t Gx, Gy, Gt;     /* grid size in voxels                       */
    int32_t kernel;         /* 0 = printed, 1 = classical */
    int32_t pad_;
} oracle_grid_t;

#define ORACLE_AMB_REL 1e-6
static const double PI = 3.14159265358979323846;

/* ---- kernels ---- */
static double k_s(const oracle_grid_t *g, double u, double v) {
    if (g->kernel == 1) return (2.0 / PI) * (1.0 - u * u - v * v);
    double a = 1.0 - u, b = 1.0 - v;
    return (PI / 2.0) * (a * a) * (b * b);
}
static double k_t(const oracle_grid_t *g, double w) {
    if (g->kernel == 1) return 0.75 * (1.0 - w * w);
    double a = 1.0 - w;
    return 0.75 * (a * a);
}

/* voxel centre (reading R5) */
static double cx(const oracle_grid_t *g, int64_t X) { return g->x0 + ((double)X + 0.5) * g->sres; }
static double cy(const oracle_grid_t *g, int64_t Y) { return g->y0 + ((double)Y + 0.5) * g->sres; }
static double ct(const oracle_grid_t *g, int64_t T) { return g->t0 + ((double)T + 0.5) * g->tres; }

/* PAPER.md:164-166 */
int64_t oracle_H(double h, double res) { return (int64_t)ceil(h / res); }

int oracle_check_grid(const oracle_grid_t *g) {
    if (!(g->sres > 0) || !(g->tres > 0) || !(g->hs > 0) || !(g->ht > 0)) return -1;
    if (g->Gx < 1 || g->Gy < 1 || g->Gt < 1) return -1;
    return 0;
}

/* Per-pair evaluation shared by VB and PB (same expressions, same order).
 * Spatial half of a (point, voxel) pair: gate, ambiguity, and k_s. */
static int eval_pair(const oracle_grid_t *g, double hs, double px, double py, int64_t X, int64_t Y,
                     double *ksv, int *s_amb_out, int *s_in_out) {
    double dx = cx(g, X) - px;
    double dy = cy(g, Y) - py;
    double d = sqrt(dx * dx + dy * dy);       /* Alg. 1 gate */
    int s_in = d < hs;
    int s_amb = fabs(d / hs - 1.0) <= ORACLE_AMB_REL;
    *s_in_out = s_in;
    *s_amb_out = s_amb;
    if (s_in || s_amb) *ksv = k_s(g, fabs(dx) / hs, fabs(dy) / hs);
    else *ksv = 0.0;
    return s_in;
}

/* Per-point bandwidths of the adaptive estimator (NULL bw: the grid's). */
static void point_bw(const oracle_grid_t *g, const float *bw, int64_t i, double *hs, double *ht) {
    if (bw) { *hs = (double)bw[2 * i]; *ht = (double)bw[2 * i + 1]; }
    else { *hs = g->hs; *ht = g->ht; }
}
static int check_bw(const oracle_grid_t *g, const float *bw, int64_t n) {
    if (!bw) return 0;
    for (int64_t i = 0; i < n; ++i) {
        double hs = bw[2 * i], ht = bw[2 * i + 1];
        if (!(hs > 0) || !(ht > 0) || hs > g->hs || ht > g->ht) return -3;
    }
    return 0;
}

/* ------------------------------------------------------------------ VB --- */
static int vb_impl(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                   double *vol, double *slack, uint8_t *amb, int64_t *contributions) {
    if (oracle_check_grid(g)) return -1;
    if (check_bw(g, bw, n)) return -3;
    const int64_t Gx = g->Gx, Gy = g->Gy, Gt = g->Gt;
    const double den = (double)n * (g->hs * g->hs) * g->ht;
    int64_t C = 0;
    for (int64_t X = 0; X < Gx; ++X)
        for (int64_t Y = 0; Y < Gy; ++Y)
            for (int64_t T = 0; T < Gt; ++T) {
                double sum = 0.0, sl = 0.0;
                int a = 0;
                for (int64_t i = 0; i < n; ++i) {
                    double px = pts[3 * i], py = pts[3 * i + 1], pt = pts[3 * i + 2];
                    double hs, ht;
                    point_bw(g, bw, i, &hs, &ht);
                    double dt = fabs(ct(g, T) - pt);
                    int t_in = dt <= ht;
                    int t_amb = fabs(dt / ht - 1.0) <= ORACLE_AMB_REL;
                    if (!t_in && !t_amb) continue;
                    double ksv; int s_amb, s_in;
                    eval_pair(g, hs, px, py, X, Y, &ksv, &s_amb, &s_in);
                    /* fixed bandwidth: sum k_s k_t, divide by n hs^2 ht at the end;
                       adaptive: each term divided by its own hs_i^2 ht_i, then by n */
                    const double dn = bw ? hs * hs * ht : 1.0;
                    if (s_in && t_in) {
                        sum += bw ? ksv * k_t(g, dt / ht) / dn : ksv * k_t(g, dt / ht);
                        ++C;
                    }
                    if ((s_amb && (t_in || t_amb)) || (t_amb && (s_in || s_amb))) {
                        a = 1;
                        sl += bw ? fabs(ksv * k_t(g, dt / ht)) / dn : fabs(ksv * k_t(g, dt / ht));
                    }
                }
                int64_t v = (X * Gy + Y) * Gt + T;
                const double dd = bw ? (double)n : den;
                vol[v] = n > 0 ? sum / dd : 0.0;
                if (slack) slack[v] = n > 0 ? sl / dd : 0.0;
                if (amb) amb[v] = (uint8_t)a;
            }
    if (contributions) *contributions = C;
    return 0;
}

int oracle_vb(const float *pts, int64_t n, const oracle_grid_t *g,
              double *vol, double *slack, uint8_t *amb, int64_t *contributions) {
    return vb_impl(pts, NULL, n, g, vol, slack, amb, contributions);
}
int oracle_vb_adaptive(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                       double *vol, double *slack, uint8_t *amb, int64_t *contributions) {
    if (!bw) return -1;
    return vb_impl(pts, bw, n, g, vol, slack, amb, contributions);
}

/* ------------------------------------------------------------------ PB --- */
typedef struct { int64_t key; int64_t idx; } kv_t;
static int cmp_kv(const void *a, const void *b) {
    const kv_t *p = (const kv_t *)a, *q = (const kv_t *)b;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    return p->idx < q->idx ? -1 : (p->idx > q->idx);
}
static int cmp_i64(const void *a, const void *b) {
    int64_t p = *(const int64_t *)a, q = *(const int64_t *)b;
    return p < q ? -1 : (p > q);
}
static int64_t clamp64(double v, int64_t lo, int64_t hi) {
    if (!(v >= (double)lo)) return lo;   /* also catches NaN */
    if (v > (double)hi) return hi;
    return (int64_t)v;
}

static int pb_impl(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                   double *vol, double *slack, uint8_t *amb, int64_t *contributions,
                   int nthreads) {
    if (oracle_check_grid(g)) return -1;
    if (check_bw(g, bw, n)) return -3;
    const int64_t Gx = g->Gx, Gy = g->Gy, Gt = g->Gt;
    const int64_t Hs = oracle_H(g->hs, g->sres), Ht = oracle_H(g->ht, g->tres);
    const int64_t nvox = Gx * Gy * Gt;
    memset(vol, 0, (size_t)nvox * sizeof(double));
    if (slack) memset(slack, 0, (size_t)nvox * sizeof(double));
    if (amb) memset(amb, 0, (size_t)nvox);
    if (contributions) *contributions = 0;
    if (n == 0) return 0;
    const double den = (double)n * (g->hs * g->hs) * g->ht;
    const int64_t BIG = Gx + Hs + 2;

    /* X_i = floor((x_i - x0)/sres), used only for loop bounds. */
    kv_t *order = (kv_t *)malloc((size_t)n * sizeof(kv_t));
    if (!order) return -2;
    for (int64_t i = 0; i < n; ++i) {
        double p = floor(((double)pts[3 * i] - g->x0) / g->sres);
        order[i].key = clamp64(p, -BIG, BIG);
        order[i].idx = i;
    }
    qsort(order, (size_t)n, sizeof(kv_t), cmp_kv);

    const int64_t CH = 4;                       /* X rows per work chunk */
    const int64_t nch = (Gx + CH - 1) / CH;
    int64_t Ctot = 0;
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : Ctot)
    {
        int64_t *cand = (int64_t *)malloc((size_t)n * sizeof(int64_t));
        double *kt = (double *)malloc((size_t)(2 * Ht + 1) * sizeof(double));
        int *tin = (int *)malloc((size_t)(2 * Ht + 1) * sizeof(int));
        int *tam = (int *)malloc((size_t)(2 * Ht + 1) * sizeof(int));
        if (!cand || !kt || !tin || !tam) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t c = 0; c < nch; ++c) {
            if (!cand || !kt || !tin || !tam) continue;
            const int64_t xa = c * CH, xb = (xa + CH < Gx) ? xa + CH : Gx;
            /* candidates: X_i in [xa - Hs, xb - 1 + Hs], then restore input order */
            int64_t lo = 0, hi = n;
            while (lo < hi) { int64_t m = (lo + hi) / 2; if (order[m].key < xa - Hs) lo = m + 1; else hi = m; }
            int64_t m0 = lo; hi = n;
            while (lo < hi) { int64_t m = (lo + hi) / 2; if (order[m].key <= xb - 1 + Hs) lo = m + 1; else hi = m; }
            int64_t nc = lo - m0;
            for (int64_t k = 0; k < nc; ++k) cand[k] = order[m0 + k].idx;
            qsort(cand, (size_t)nc, sizeof(int64_t), cmp_i64);

            for (int64_t k = 0; k < nc; ++k) {
                const int64_t i = cand[k];
                const double px = pts[3 * i], py = pts[3 * i + 1], pt = pts[3 * i + 2];
                double hs, ht;
                point_bw(g, bw, i, &hs, &ht);
                /* the point's own box (adaptive: H_s(i) = ceil(hs_i/sres) <= H_s) */
                const int64_t Hsi = bw ? oracle_H(hs, g->sres) : Hs, Hti = bw ? oracle_H(ht, g->tres) : Ht;
                const double dn = bw ? hs * hs * ht : 1.0;
                const int64_t Xi = clamp64(floor((px - g->x0) / g->sres), -BIG, BIG);
                const int64_t Yi = clamp64(floor((py - g->y0) / g->sres), -(Gy + Hs + 2), Gy + Hs + 2);
                const int64_t Ti = clamp64(floor((pt - g->t0) / g->tres), -(Gt + Ht + 2), Gt + Ht + 2);
                const int64_t X0 = Xi - Hsi > xa ? Xi - Hsi : xa, X1 = Xi + Hsi < xb - 1 ? Xi + Hsi : xb - 1;
                const int64_t Y0 = Yi - Hsi > 0 ? Yi - Hsi : 0, Y1 = Yi + Hsi < Gy - 1 ? Yi + Hsi : Gy - 1;
                const int64_t T0 = Ti - Hti > 0 ? Ti - Hti : 0, T1 = Ti + Hti < Gt - 1 ? Ti + Hti : Gt - 1;
                if (X0 > X1 || Y0 > Y1 || T0 > T1) continue;
                /* K_t[T] once per point (Alg. 3) */
                int any_t = 0;
                for (int64_t T = T0; T <= T1; ++T) {
                    double dt = fabs(ct(g, T) - pt);
                    tin[T - T0] = dt <= ht;
                    tam[T - T0] = fabs(dt / ht - 1.0) <= ORACLE_AMB_REL;
                    kt[T - T0] = k_t(g, dt / ht);
                    any_t |= tin[T - T0] | tam[T - T0];
                }
                if (!any_t) continue;
                for (int64_t X = X0; X <= X1; ++X)
                    for (int64_t Y = Y0; Y <= Y1; ++Y) {
                        double ksv; int s_amb, s_in;
                        eval_pair(g, hs, px, py, X, Y, &ksv, &s_amb, &s_in);
                        if (!s_in && !s_amb) continue;
                        double *col = vol + (X * Gy + Y) * Gt;
                        if (s_in)
                            for (int64_t T = T0; T <= T1; ++T)
                                if (tin[T - T0]) {
                                    col[T] += bw ? ksv * kt[T - T0] / dn : ksv * kt[T - T0];
                                    ++Ctot;
                                }
                        if (slack || amb)
                            for (int64_t T = T0; T <= T1; ++T) {
                                int ti = tin[T - T0], ta = tam[T - T0];
                                if ((s_amb && (ti || ta)) || (ta && (s_in || s_amb))) {
                                    int64_t v = (X * Gy + Y) * Gt + T;
                                    if (slack) slack[v] += bw ? fabs(ksv * kt[T - T0]) / dn : fabs(ksv * kt[T - T0]);
                                    if (amb) amb[v] = 1;
                                }
                            }
                    }
            }
        }
        free(cand); free(kt); free(tin); free(tam);
    }
    free(order);
    if (err) return -2;
    const double dd = bw ? (double)n : den;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvox; ++v) {
        vol[v] = vol[v] / dd;
        if (slack) slack[v] = slack[v] / dd;
    }
    if (contributions) *contributions = Ctot;
    return 0;
}

int oracle_pb(const float *pts, int64_t n, const oracle_grid_t *g,
              double *vol, double *slack, uint8_t *amb, int64_t *contributions,
              int nthreads) {
    return pb_impl(pts, NULL, n, g, vol, slack, amb, contributions, nthreads);
}
int oracle_pb_adaptive(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                       double *vol, double *slack, uint8_t *amb, int64_t *contributions,
                       int nthreads) {
    if (!bw) return -1;
    return pb_impl(pts, bw, n, g, vol, slack, amb, contributions, nthreads);
}

/* ---------------------------------------------------- VB at sampled voxels --- */
static int vb_voxels_impl(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                          const int64_t *vox, int64_t m, double *val, double *slack,
                          uint8_t *amb, int nthreads) {
    if (oracle_check_grid(g)) return -1;
    if (check_bw(g, bw, n)) return -3;
    const int64_t Gy = g->Gy, Gt = g->Gt;
    const double den = (double)n * (g->hs * g->hs) * g->ht;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = 0; k < m; ++k) {
        const int64_t v = vox[k];
        const int64_t X = v / (Gy * Gt), Y = (v / Gt) % Gy, T = v % Gt;
        double sum = 0.0, sl = 0.0;
        int a = 0;
        for (int64_t i = 0; i < n; ++i) {
            double px = pts[3 * i], py = pts[3 * i + 1], pt = pts[3 * i + 2];
            double hs, ht;
            point_bw(g, bw, i, &hs, &ht);
            double dt = fabs(ct(g, T) - pt);
            int t_in = dt <= ht;
            int t_amb = fabs(dt / ht - 1.0) <= ORACLE_AMB_REL;
            if (!t_in && !t_amb) continue;
            double ksv; int s_amb, s_in;
            eval_pair(g, hs, px, py, X, Y, &ksv, &s_amb, &s_in);
            const double dn = bw ? hs * hs * ht : 1.0;
            if (s_in && t_in) sum += bw ? ksv * k_t(g, dt / ht) / dn : ksv * k_t(g, dt / ht);
            if ((s_amb && (t_in || t_amb)) || (t_amb && (s_in || s_amb))) {
                a = 1;
                sl += bw ? fabs(ksv * k_t(g, dt / ht)) / dn : fabs(ksv * k_t(g, dt / ht));
            }
        }
        const double dd = bw ? (double)n : den;
        val[k] = n > 0 ? sum / dd : 0.0;
        if (slack) slack[k] = n > 0 ? sl / dd : 0.0;
        if (amb) amb[k] = (uint8_t)a;
    }
    return 0;
}
int oracle_vb_voxels(const float *pts, int64_t n, const oracle_grid_t *g,
                     const int64_t *vox, int64_t m, double *val, double *slack,
                     uint8_t *amb, int nthreads) {
    return vb_voxels_impl(pts, NULL, n, g, vox, m, val, slack, amb, nthreads);
}
int oracle_vb_voxels_adaptive(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                              const int64_t *vox, int64_t m, double *val, double *slack,
                              uint8_t *amb, int nthreads) {
    if (!bw) return -1;
    return vb_voxels_impl(pts, bw, n, g, vox, m, val, slack, amb, nthreads);
}

/* Exact gated-pair count C = sum_i (#disc columns in grid) * (#window layers in grid). */
static int contributions_impl(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                              int64_t *out, int nthreads) {
    if (oracle_check_grid(g)) return -1;
    if (check_bw(g, bw, n)) return -3;
    const int64_t Hs = oracle_H(g->hs, g->sres), Ht = oracle_H(g->ht, g->tres);
    int64_t C = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : C)
    for (int64_t i = 0; i < n; ++i) {
        const double px = pts[3 * i], py = pts[3 * i + 1], pt = pts[3 * i + 2];
        double hs, ht;
        point_bw(g, bw, i, &hs, &ht);
        const int64_t Xi = clamp64(floor((px - g->x0) / g->sres), -(g->Gx + Hs + 2), g->Gx + Hs + 2);
        const int64_t Yi = clamp64(floor((py - g->y0) / g->sres), -(g->Gy + Hs + 2), g->Gy + Hs + 2);
        const int64_t Ti = clamp64(floor((pt - g->t0) / g->tres), -(g->Gt + Ht + 2), g->Gt + Ht + 2);
        int64_t cols = 0, lay = 0;
        for (int64_t X = Xi - Hs; X <= Xi + Hs; ++X) {
            if (X < 0 || X >= g->Gx) continue;
            for (int64_t Y = Yi - Hs; Y <= Yi + Hs; ++Y) {
                if (Y < 0 || Y >= g->Gy) continue;
                double dx = cx(g, X) - px, dy = cy(g, Y) - py;
                if (sqrt(dx * dx + dy * dy) < hs) ++cols;
            }
        }
        for (int64_t T = Ti - Ht; T <= Ti + Ht; ++T) {
            if (T < 0 || T >= g->Gt) continue;
            if (fabs(ct(g, T) - pt) <= ht) ++lay;
        }
        C += cols * lay;
    }
    *out = C;
    return 0;
}
int oracle_contributions(const float *pts, int64_t n, const oracle_grid_t *g,
                         int64_t *out, int nthreads) {
    return contributions_impl(pts, NULL, n, g, out, nthreads);
}
int oracle_contributions_adaptive(const float *pts, const float *bw, int64_t n, const oracle_grid_t *g,
                                  int64_t *out, int nthreads) {
    if (!bw) return -1;
    return contributions_impl(pts, bw, n, g, out, nthreads);
}

/* Single kernel evaluations, exported for the closed-form pins. */
double oracle_k_s(int32_t kernel, double u, double v) {
    oracle_grid_t g; memset(&g, 0, sizeof g); g.kernel = kernel; return k_s(&g, u, v);
}
double oracle_k_t(int32_t kernel, double w) {
    oracle_grid_t g; memset(&g, 0, sizeof g); g.kernel = kernel; return k_t(&g, w);
}
