/*
 * o3g_oracle.c — CPU ORACLE for the point-to-plane ICP iteration.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing on the product path may link, load or
 * call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it. It shares no code, header,
 * constant or helper with the CUDA library (paper_1801_09847_b200/csrc).
 *
 * Plain, slow, obviously-correct C99, compiled with
 *   -O2 -ffp-contract=off -fno-fast-math   (SSE2 fp64, no FMA contraction)
 * so every floating-point operation below is one IEEE-754 binary64
 * operation in the order written.
 *
 * What it computes (citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
 * R#n = reading n of DESIGN.md §3 "Readings of the paper"):
 *   - registration_icp(..., TransformationEstimationPointToPlane())
 *     P:203-212 (§3.3), loop semantics S:282-290, refs [2],[4] P:267,P:269.
 *   - Gauss-Newton step x <- x - (J^T J)^{-1} J^T r, Eq. 2, with
 *     J^T J and J^T r summed over the data records.
 *   - nearest neighbour within max_correspondence_distance,
 *     inclusive d <= dmax, ties -> lower target index (R#1-R#3).
 *   - fitness = inliers/|source|, inlier_rmse over the
 *     correspondences (R#7).
 *   - LDLT without pivoting + singularity guard (R#6).
 *   - SE(3) exponential, twist (omega, v) rotation first, series for
 *     |omega| < 1e-6 (R#5).
 *   - convergence |dfit| < relative_fitness and |drmse| < relative_rmse
 *     between consecutive passes (R#8: parity unpinned by paper).
 *
 * Correspondence search has two forms:
 *   - brute force over every target point: the DEFINITION;
 *   - a grid accelerator (cells of size dmax*(1+2^-24), 27-cell scan) that
 *     tests/test_oracle.py checks equal to brute force.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FP_FAST_FMA) && !defined(O3G_ORACLE_ALLOW_FMA)
/* -ffp-contract=off is what matters; __FP_FAST_FMA only says FMA exists. */
#endif

/* ------------------------------------------------------------------ A3 */
/* s' = T s with the fixed order ((T00 sx + T01 sy) + T02 sz) + T03
 * (R#2), sx = (double) of the fp32 input. T is row-major 4x4.           */
void orc_transform_point(const double T[16], const float p[3], double out[3])
{
    const double x = (double)p[0], y = (double)p[1], z = (double)p[2];
    for (int r = 0; r < 3; ++r) {
        double a = T[4 * r + 0] * x;
        double b = T[4 * r + 1] * y;
        double c = T[4 * r + 2] * z;
        out[r] = ((a + b) + c) + T[4 * r + 3];
    }
}

void orc_transform(const double T[16], const float *p, int64_t n, double *out)
{
    for (int64_t i = 0; i < n; ++i) orc_transform_point(T, p + 3 * i, out + 3 * i);
}

/* ------------------------------------------------------------------ A4 */
/* d^2 = ((dx*dx + dy*dy) + dz*dz), dx = s'x - (double)qx (R#2).          */
static double dist2(const double s[3], const float *q)
{
    double dx = s[0] - (double)q[0];
    double dy = s[1] - (double)q[1];
    double dz = s[2] - (double)q[2];
    double xx = dx * dx, yy = dy * dy, zz = dz * dz;
    return (xx + yy) + zz;
}

/* Keep j if d2 <= r2 (inclusive, R#1); the winner is the minimum d2 and,
 * among equal d2, the lowest target index (R#3).                        */
static int better(double d2, int64_t j, double best_d2, int64_t best_j)
{
    if (best_j < 0) return 1;
    if (d2 < best_d2) return 1;
    if (d2 == best_d2 && j < best_j) return 1;
    return 0;
}

/* Brute force: the definition. Returns the index or -1.                 */
int64_t orc_nn_brute(const double s[3], const float *tgt, int64_t m, double r2, double *d2_out)
{
    int64_t best = -1;
    double bd = 0.0;
    for (int64_t j = 0; j < m; ++j) {
        double d2 = dist2(s, tgt + 3 * j);
        if (d2 <= r2 && better(d2, j, bd, best)) { best = j; bd = d2; }
    }
    if (d2_out) *d2_out = bd;
    return best;
}

/* ---------------------------------------------------------- grid (accel) */
typedef struct { int64_t cz, cy, cx; int64_t idx; } orc_cellpt;

typedef struct {
    const float *tgt;
    int64_t m;
    double o[3];     /* componentwise min of the target */
    double h;        /* cell size dmax*(1+2^-24) */
    orc_cellpt *pts; /* sorted by (cz, cy, cx, idx) */
} orc_grid;

static int cmp_cellpt(const void *a_, const void *b_)
{
    const orc_cellpt *a = (const orc_cellpt *)a_, *b = (const orc_cellpt *)b_;
    if (a->cz != b->cz) return a->cz < b->cz ? -1 : 1;
    if (a->cy != b->cy) return a->cy < b->cy ? -1 : 1;
    if (a->cx != b->cx) return a->cx < b->cx ? -1 : 1;
    if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
    return 0;
}

static int64_t cell_coord(double x, double o, double h)
{
    double c = floor((x - o) / h);
    if (c < -1099511627776.0) c = -1099511627776.0; /* clamp far queries: 2^40 */
    if (c > 1099511627776.0) c = 1099511627776.0;
    return (int64_t)c;
}

orc_grid *orc_grid_build(const float *tgt, int64_t m, double dmax)
{
    orc_grid *g = (orc_grid *)calloc(1, sizeof(orc_grid));
    if (!g) return NULL;
    g->tgt = tgt;
    g->m = m;
    g->h = dmax * (1.0 + 5.9604644775390625e-08); /* 2^-24 margin */
    for (int a = 0; a < 3; ++a) g->o[a] = INFINITY;
    for (int64_t j = 0; j < m; ++j)
        for (int a = 0; a < 3; ++a)
            if ((double)tgt[3 * j + a] < g->o[a]) g->o[a] = (double)tgt[3 * j + a];
    g->pts = (orc_cellpt *)malloc(sizeof(orc_cellpt) * (size_t)(m > 0 ? m : 1));
    if (!g->pts) { free(g); return NULL; }
    for (int64_t j = 0; j < m; ++j) {
        g->pts[j].cx = cell_coord((double)tgt[3 * j + 0], g->o[0], g->h);
        g->pts[j].cy = cell_coord((double)tgt[3 * j + 1], g->o[1], g->h);
        g->pts[j].cz = cell_coord((double)tgt[3 * j + 2], g->o[2], g->h);
        g->pts[j].idx = j;
    }
    qsort(g->pts, (size_t)m, sizeof(orc_cellpt), cmp_cellpt);
    return g;
}

void orc_grid_free(orc_grid *g)
{
    if (g) { free(g->pts); free(g); }
}

/* first position whose (cz,cy,cx) >= key (idx ignored) */
static int64_t lower(const orc_grid *g, int64_t cz, int64_t cy, int64_t cx)
{
    int64_t lo = 0, hi = g->m;
    orc_cellpt key = {cz, cy, cx, -1};
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (cmp_cellpt(&g->pts[mid], &key) < 0) lo = mid + 1; else hi = mid;
    }
    return lo;
}

int64_t orc_nn_grid(const orc_grid *g, const double s[3], double r2, double *d2_out)
{
    int64_t cx = cell_coord(s[0], g->o[0], g->h);
    int64_t cy = cell_coord(s[1], g->o[1], g->h);
    int64_t cz = cell_coord(s[2], g->o[2], g->h);
    int64_t best = -1;
    double bd = 0.0;
    for (int64_t dz = -1; dz <= 1; ++dz)
        for (int64_t dy = -1; dy <= 1; ++dy)
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t k = lower(g, cz + dz, cy + dy, cx + dx);
                for (; k < g->m; ++k) {
                    const orc_cellpt *c = &g->pts[k];
                    if (c->cz != cz + dz || c->cy != cy + dy || c->cx != cx + dx) break;
                    double d2 = dist2(s, g->tgt + 3 * c->idx);
                    if (d2 <= r2 && better(d2, c->idx, bd, best)) { best = c->idx; bd = d2; }
                }
            }
    if (d2_out) *d2_out = bd;
    return best;
}

/* ------------------------------------------------------------ A5 / A6 */
/* Neumaier-compensated accumulator, plus the sum of |terms| used by the
 * reduction tolerance (R#14).                                           */
typedef struct { double s, c, a; } acc_t;

static void acc_add(acc_t *x, double v)
{
    double t = x->s + v;
    if (fabs(x->s) >= fabs(v)) x->c += (x->s - t) + v;
    else x->c += (v - t) + x->s;
    x->s = t;
    x->a += fabs(v);
}

/* 29 terms: JTJ upper triangle row-major (i<=j, 21), JTr (6), count, sum d^2 */
enum { ORC_NTERMS = 29 };

/* One correspondence record: r = (s'-q).n, J = [s' x n ; n] (R#4).       */
static void record(const double s[3], const float *qf, const float *nf, double d2, acc_t acc[ORC_NTERMS])
{
    double q[3] = {(double)qf[0], (double)qf[1], (double)qf[2]};
    double n[3] = {(double)nf[0], (double)nf[1], (double)nf[2]};
    double r = ((s[0] - q[0]) * n[0] + (s[1] - q[1]) * n[1]) + (s[2] - q[2]) * n[2];
    double J[6];
    J[0] = s[1] * n[2] - s[2] * n[1];
    J[1] = s[2] * n[0] - s[0] * n[2];
    J[2] = s[0] * n[1] - s[1] * n[0];
    J[3] = n[0];
    J[4] = n[1];
    J[5] = n[2];
    int k = 0;
    for (int i = 0; i < 6; ++i)
        for (int j = i; j < 6; ++j) acc_add(&acc[k++], J[i] * J[j]);
    for (int i = 0; i < 6; ++i) acc_add(&acc[21 + i], J[i] * r);
    acc_add(&acc[27], 1.0);
    acc_add(&acc[28], d2);
}

/* One pass at fixed T over source indices idx[0..k) (idx NULL -> 0..n).
 * corr[t] gets the target index of idx[t] (or -1); d2out likewise.
 * sums/abssums: the 29 terms and their sums of |term|.                  */
void orc_pass_subset(const double T[16], const float *src, int64_t n, const int64_t *idx, int64_t k,
                     const float *tgt, const float *nrm, int64_t m, const orc_grid *g, double dmax,
                     int32_t *corr, double *d2out, double *sums, double *abssums)
{
    acc_t acc[ORC_NTERMS];
    memset(acc, 0, sizeof(acc));
    const double r2 = dmax * dmax;
    int64_t cnt = idx ? k : n;
    for (int64_t t = 0; t < cnt; ++t) {
        int64_t i = idx ? idx[t] : t;
        double s[3], d2 = 0.0;
        orc_transform_point(T, src + 3 * i, s);
        int64_t j = g ? orc_nn_grid(g, s, r2, &d2) : orc_nn_brute(s, tgt, m, r2, &d2);
        if (corr) corr[t] = (int32_t)j;
        if (d2out) d2out[t] = j >= 0 ? d2 : -1.0;
        if (j >= 0) record(s, tgt + 3 * j, nrm + 3 * j, d2, acc);
    }
    for (int t = 0; t < ORC_NTERMS; ++t) {
        if (sums) sums[t] = acc[t].s + acc[t].c;
        if (abssums) abssums[t] = acc[t].a;
    }
}

void orc_pass(const double T[16], const float *src, int64_t n, const float *tgt, const float *nrm,
              int64_t m, const orc_grid *g, double dmax, int32_t *corr, double *sums, double *abssums)
{
    orc_pass_subset(T, src, n, NULL, 0, tgt, nrm, m, g, dmax, corr, NULL, sums, abssums);
}

/* Deterministic OpenMP mode (SURVEY §8(c) "a fixed chunk partition, with
 * partials summed in chunk order"; the paper's own parallelisation of the
 * J^T J / J^T r evaluation, "OpenMP reduction ... for each data record",
 * P:238-248, Eq. 2). The records are split into fixed chunks of
 * ORC_CHUNK queries in source order, independent of the thread count; each
 * chunk is accumulated exactly like orc_pass_subset (Neumaier), and the
 * chunk partials (their compensated values s + c) are then summed in chunk
 * order by the same accumulator. The result is therefore bitwise the same
 * for any nthreads (0/1 = run the chunks on the calling thread). The
 * correspondences are per-query, hence identical to orc_pass_subset's.   */
#define ORC_CHUNK 4096
int orc_pass_chunked(const double T[16], const float *src, int64_t n, const int64_t *idx, int64_t k,
                     const float *tgt, const float *nrm, int64_t m, const orc_grid *g, double dmax,
                     int32_t *corr, double *d2out, double *sums, double *abssums, int32_t nthreads)
{
    const int64_t cnt = idx ? k : n;
    const int64_t nch = (cnt + ORC_CHUNK - 1) / ORC_CHUNK;
    acc_t *part = (acc_t *)calloc((size_t)(nch > 0 ? nch : 1) * ORC_NTERMS, sizeof(acc_t));
    if (!part) return 1;
    const double r2 = dmax * dmax;
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < nch; ++c) {
        acc_t *acc = part + c * ORC_NTERMS;
        const int64_t t1 = (c + 1) * ORC_CHUNK < cnt ? (c + 1) * ORC_CHUNK : cnt;
        for (int64_t t = c * ORC_CHUNK; t < t1; ++t) {
            int64_t i = idx ? idx[t] : t;
            double s[3], d2 = 0.0;
            orc_transform_point(T, src + 3 * i, s);
            int64_t j = g ? orc_nn_grid(g, s, r2, &d2) : orc_nn_brute(s, tgt, m, r2, &d2);
            if (corr) corr[t] = (int32_t)j;
            if (d2out) d2out[t] = j >= 0 ? d2 : -1.0;
            if (j >= 0) record(s, tgt + 3 * j, nrm + 3 * j, d2, acc);
        }
    }
    acc_t tot[ORC_NTERMS];
    memset(tot, 0, sizeof(tot));
    for (int64_t c = 0; c < nch; ++c)
        for (int t = 0; t < ORC_NTERMS; ++t) {
            const acc_t *a = &part[c * ORC_NTERMS + t];
            double a_abs = tot[t].a + a->a;
            acc_add(&tot[t], a->s + a->c);
            tot[t].a = a_abs;   /* sum of |records|, not of |chunk sums| */
        }
    for (int t = 0; t < ORC_NTERMS; ++t) {
        if (sums) sums[t] = tot[t].s + tot[t].c;
        if (abssums) abssums[t] = tot[t].a;
    }
    free(part);
    return 0;
}

/* ------------------------------------------------------------------ A8 */
/* Full symmetric 6x6 from the 21 upper-triangle terms.                  */
void orc_expand_jtj(const double *terms, double A[36])
{
    int k = 0;
    for (int i = 0; i < 6; ++i)
        for (int j = i; j < 6; ++j) { A[6 * i + j] = terms[k]; A[6 * j + i] = terms[k]; ++k; }
}

/* LDL^T without pivoting (R#6). Returns 0 on success, 1 if singular:
 * some D_k <= 1e-12 * max_i A_ii (or max_i A_ii <= 0).                  */
int orc_ldlt_solve(const double A[36], const double b[6], double x[6])
{
    double L[36] = {0}, D[6], y[6];
    double dmax = 0.0;
    for (int i = 0; i < 6; ++i) if (A[7 * i] > dmax) dmax = A[7 * i];
    if (!(dmax > 0.0)) return 1;
    for (int j = 0; j < 6; ++j) {
        double d = A[6 * j + j];
        for (int k = 0; k < j; ++k) d -= L[6 * j + k] * L[6 * j + k] * D[k];
        if (!(d > 1e-12 * dmax)) return 1;
        D[j] = d;
        L[6 * j + j] = 1.0;
        for (int i = j + 1; i < 6; ++i) {
            double v = A[6 * i + j];
            for (int k = 0; k < j; ++k) v -= L[6 * i + k] * L[6 * j + k] * D[k];
            L[6 * i + j] = v / d;
        }
    }
    for (int i = 0; i < 6; ++i) {            /* L y = b */
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= L[6 * i + k] * y[k];
        y[i] = v;
    }
    for (int i = 0; i < 6; ++i) y[i] /= D[i]; /* D z = y */
    for (int i = 5; i >= 0; --i) {           /* L^T x = z */
        double v = y[i];
        for (int k = i + 1; k < 6; ++k) v -= L[6 * k + i] * x[k];
        x[i] = v;
    }
    return 0;
}

/* SE(3) exponential of xi = (omega, v) (R#5):
 *   R = I + A W + B W^2,  V = I + B W + C W^2,  t = V v,
 *   A = sin(th)/th, B = (1-cos th)/th^2, C = (th - sin th)/th^3,
 *   series 1 - th^2/6, 1/2 - th^2/24, 1/6 - th^2/120 for th < 1e-6.      */
void orc_exp_se3(const double xi[6], double T[16])
{
    const double w[3] = {xi[0], xi[1], xi[2]}, v[3] = {xi[3], xi[4], xi[5]};
    double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double th = sqrt(th2), A, B, C;
    if (th < 1e-6) {
        A = 1.0 - th2 / 6.0;
        B = 0.5 - th2 / 24.0;
        C = 1.0 / 6.0 - th2 / 120.0;
    } else {
        A = sin(th) / th;
        B = (1.0 - cos(th)) / th2;
        C = (th - sin(th)) / (th2 * th);
    }
    double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    double W2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += W[3 * i + k] * W[3 * k + j];
            W2[3 * i + j] = s;
        }
    double R[9], V[9];
    for (int i = 0; i < 9; ++i) {
        double I = (i % 4 == 0) ? 1.0 : 0.0;
        R[i] = I + A * W[i] + B * W2[i];
        V[i] = I + B * W[i] + C * W2[i];
    }
    memset(T, 0, 16 * sizeof(double));
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) T[4 * i + j] = R[3 * i + j];
        T[4 * i + 3] = V[3 * i + 0] * v[0] + V[3 * i + 1] * v[1] + V[3 * i + 2] * v[2];
    }
    T[15] = 1.0;
}

/* C = A B for 4x4 row-major rigid transforms; bottom row set exactly.   */
void orc_compose(const double A[16], const double B[16], double C[16])
{
    double out[16];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += A[4 * i + k] * B[4 * k + j];
            out[4 * i + j] = s;
        }
    out[12] = 0.0; out[13] = 0.0; out[14] = 0.0; out[15] = 1.0;
    memcpy(C, out, sizeof(out));
}

/* ------------------------------------------------------------ the loop */
enum { ORC_FLAG_NO_CORR = 1, ORC_FLAG_DEGENERATE = 2 };

/* registration_icp, point-to-plane.
 * max_iterations counts updates; passes = updates + 1. Returns fitness and
 * rmse of the last pass, i.e. at the returned T. hist_* (nullable) get one
 * entry per pass (max_iterations + 1 capacity).                         */
int orc_icp(const float *src, int64_t n, const float *tgt, const float *nrm, int64_t m,
            const double T0[16], double dmax, int32_t max_iterations, double relative_fitness,
            double relative_rmse, int32_t use_grid, double T_out[16], double *fitness,
            double *inlier_rmse, int32_t *iterations, int32_t *flags, int32_t *converged,
            double *hist_fit, double *hist_rmse, int32_t nthreads)
{
    orc_grid *g = use_grid ? orc_grid_build(tgt, m, dmax) : NULL;
    if (use_grid && !g) return -1;
    double T[16], sums[ORC_NTERMS];
    memcpy(T, T0, sizeof(T));
    int32_t it = 0, fl = 0, conv = 0, passes = 0;

    /* nthreads > 0: the deterministic chunked (OpenMP) pass */
#define ORC_PASS()                                                                          \
    (nthreads > 0 ? (void)orc_pass_chunked(T, src, n, NULL, 0, tgt, nrm, m, g, dmax, NULL, NULL, \
                                           sums, NULL, nthreads)                            \
                  : orc_pass(T, src, n, tgt, nrm, m, g, dmax, NULL, sums, NULL))
    ORC_PASS();
    double cnt = sums[27];
    double fit = cnt / (double)n, rmse = cnt > 0 ? sqrt(sums[28] / cnt) : 0.0;
    if (hist_fit) hist_fit[passes] = fit;
    if (hist_rmse) hist_rmse[passes] = rmse;
    ++passes;
    double fp = fit, rp = rmse;
    while (it < max_iterations) {
        if (cnt == 0.0) { fl |= ORC_FLAG_NO_CORR; break; }
        double A[36], b[6], xi[6], dT[16];
        orc_expand_jtj(sums, A);
        for (int i = 0; i < 6; ++i) b[i] = -sums[21 + i];
        if (cnt < 6.0 || orc_ldlt_solve(A, b, xi)) { fl |= ORC_FLAG_DEGENERATE; break; }
        orc_exp_se3(xi, dT);
        orc_compose(dT, T, T);
        ++it;
        ORC_PASS();
        cnt = sums[27];
        fit = cnt / (double)n;
        rmse = cnt > 0 ? sqrt(sums[28] / cnt) : 0.0;
        if (hist_fit) hist_fit[passes] = fit;
        if (hist_rmse) hist_rmse[passes] = rmse;
        ++passes;
        if (fabs(fit - fp) < relative_fitness && fabs(rmse - rp) < relative_rmse) { conv = 1; break; }
        fp = fit;
        rp = rmse;
    }
    if (cnt == 0.0) fl |= ORC_FLAG_NO_CORR;
    memcpy(T_out, T, sizeof(T));
    *fitness = fit;
    *inlier_rmse = rmse;
    *iterations = it;
    *flags = fl;
    *converged = conv;
    orc_grid_free(g);
#undef ORC_PASS
    return passes;
}

/* ------------------------------------------------- voxel_down_sample (NEXT 1) */
/* SPEC S:58-61 (Fig. 1 "voxel_size = 0.05"): each output point is the
 * arithmetic mean of the input points in one occupied voxel of the grid
 * anchored at the cloud's minimum bound, voxel index floor((p - min)/voxel)
 * (floor semantics); normals averaged the same way then renormalised;
 * output in ascending lexicographic (ix, iy, iz) order. Sums are fp64 in
 * original index order; mean = sum / count rounded once to fp32; normal =
 * s / sqrt((sx*sx + sy*sy) + sz*sz) (zero if the sum is zero). Returns the
 * number of output points.                                               */
typedef struct { int64_t ix, iy, iz, idx; } orc_vox;

static int cmp_vox(const void *a_, const void *b_)
{
    const orc_vox *a = (const orc_vox *)a_, *b = (const orc_vox *)b_;
    if (a->ix != b->ix) return a->ix < b->ix ? -1 : 1;
    if (a->iy != b->iy) return a->iy < b->iy ? -1 : 1;
    if (a->iz != b->iz) return a->iz < b->iz ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

int64_t orc_voxel_down_sample(const float *p, const float *nrm, int64_t n, double voxel,
                              float *out_p, float *out_n)
{
    if (n <= 0 || !(voxel > 0.0)) return -1;
    double mn[3] = {INFINITY, INFINITY, INFINITY};
    for (int64_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a)
            if ((double)p[3 * i + a] < mn[a]) mn[a] = (double)p[3 * i + a];
    orc_vox *v = (orc_vox *)malloc(sizeof(orc_vox) * (size_t)n);
    if (!v) return -2;
    for (int64_t i = 0; i < n; ++i) {
        v[i].ix = (int64_t)floor(((double)p[3 * i + 0] - mn[0]) / voxel);
        v[i].iy = (int64_t)floor(((double)p[3 * i + 1] - mn[1]) / voxel);
        v[i].iz = (int64_t)floor(((double)p[3 * i + 2] - mn[2]) / voxel);
        v[i].idx = i;
    }
    qsort(v, (size_t)n, sizeof(orc_vox), cmp_vox);
    int64_t out = 0;
    for (int64_t s = 0; s < n;) {
        int64_t e = s;
        double sp[3] = {0, 0, 0}, sn[3] = {0, 0, 0};
        while (e < n && v[e].ix == v[s].ix && v[e].iy == v[s].iy && v[e].iz == v[s].iz) {
            for (int a = 0; a < 3; ++a) {
                sp[a] += (double)p[3 * v[e].idx + a];
                if (nrm) sn[a] += (double)nrm[3 * v[e].idx + a];
            }
            ++e;
        }
        const double cnt = (double)(e - s);
        for (int a = 0; a < 3; ++a) out_p[3 * out + a] = (float)(sp[a] / cnt);
        if (nrm && out_n) {
            double nn = sqrt((sn[0] * sn[0] + sn[1] * sn[1]) + sn[2] * sn[2]);
            for (int a = 0; a < 3; ++a) out_n[3 * out + a] = nn > 0.0 ? (float)(sn[a] / nn) : 0.0f;
        }
        ++out;
        s = e;
    }
    free(v);
    return out;
}

/* Multi-scale registration (NEXT 1; SURVEY §8(c) reading R13): for each
 * scale s, downsample source and target at voxel[s] (target normals
 * averaged), run orc_icp with dmax[s] and iters[s] from the current T, and
 * carry T to the next scale. fit/rmse/iterations of each scale are written
 * to the per-scale arrays (nullable).                                      */
int orc_icp_multiscale(const float *src, int64_t n, const float *tgt, const float *nrm, int64_t m,
                       const double T0[16], int32_t nscales, const double *voxel, const double *dmax,
                       const int32_t *iters, double relative_fitness, double relative_rmse,
                       double T_out[16], double *fit_s, double *rmse_s, int32_t *iters_s,
                       int64_t *nsrc_s, int32_t nthreads)
{
    double T[16];
    memcpy(T, T0, sizeof(T));
    float *sp = (float *)malloc(sizeof(float) * 3 * (size_t)n);
    float *tp = (float *)malloc(sizeof(float) * 3 * (size_t)m);
    float *tn = (float *)malloc(sizeof(float) * 3 * (size_t)m);
    if (!sp || !tp || !tn) { free(sp); free(tp); free(tn); return -1; }
    for (int32_t s = 0; s < nscales; ++s) {
        int64_t ns = orc_voxel_down_sample(src, NULL, n, voxel[s], sp, NULL);
        int64_t ms = orc_voxel_down_sample(tgt, nrm, m, voxel[s], tp, tn);
        double fit, rmse, Tn[16];
        int32_t it, fl, cv;
        if (ns <= 0 || ms <= 0) { free(sp); free(tp); free(tn); return -1; }
        orc_icp(sp, ns, tp, tn, ms, T, dmax[s], iters[s], relative_fitness, relative_rmse, 1, Tn,
                &fit, &rmse, &it, &fl, &cv, NULL, NULL, nthreads);
        memcpy(T, Tn, sizeof(T));
        if (fit_s) fit_s[s] = fit;
        if (rmse_s) rmse_s[s] = rmse;
        if (iters_s) iters_s[s] = it;
        if (nsrc_s) nsrc_s[s] = ns;
    }
    memcpy(T_out, T, sizeof(T));
    free(sp); free(tp); free(tn);
    return 0;
}

/* ------------------------------------------ point-to-point ICP (NEXT 2) */
/* TransformationEstimationPointToPoint(False) ("Other ICP variants
 * are implemented as well" P:212): closed-form rigid fit
 * minimising sum |R s'_i + t - q_i|^2 over the correspondences, no scale,
 * reflection corrected so det R = +1 (Kabsch/SVD). The 29 terms of a pass:
 * [0..8] sum s'_a q_b (row-major a,b), [9..11] sum s', [12..14] sum q,
 * [27] count, [28] sum d^2; the correspondence rule is the same as above. */
static void record_p2p(const double s[3], const float *qf, double d2, acc_t acc[ORC_NTERMS])
{
    double q[3] = {(double)qf[0], (double)qf[1], (double)qf[2]};
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) acc_add(&acc[3 * a + b], s[a] * q[b]);
    for (int a = 0; a < 3; ++a) acc_add(&acc[9 + a], s[a]);
    for (int a = 0; a < 3; ++a) acc_add(&acc[12 + a], q[a]);
    acc_add(&acc[27], 1.0);
    acc_add(&acc[28], d2);
}

void orc_pass_p2p(const double T[16], const float *src, int64_t n, const float *tgt, int64_t m,
                  const orc_grid *g, double dmax, int32_t *corr, double *sums)
{
    acc_t acc[ORC_NTERMS];
    memset(acc, 0, sizeof(acc));
    const double r2 = dmax * dmax;
    for (int64_t i = 0; i < n; ++i) {
        double s[3], d2 = 0.0;
        orc_transform_point(T, src + 3 * i, s);
        int64_t j = g ? orc_nn_grid(g, s, r2, &d2) : orc_nn_brute(s, tgt, m, r2, &d2);
        if (corr) corr[i] = (int32_t)j;
        if (j >= 0) record_p2p(s, tgt + 3 * j, d2, acc);
    }
    for (int t = 0; t < ORC_NTERMS; ++t) sums[t] = acc[t].s + acc[t].c;
}

/* Jacobi eigen-decomposition of a symmetric 3x3 A (destroyed): eigenvalues
 * in w, eigenvectors in the columns of V (row-major).                     */
static void jacobi3(double A[9], double w[3], double V[9])
{
    for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = fabs(A[1]) + fabs(A[2]) + fabs(A[5]);
        double dia = fabs(A[0]) + fabs(A[4]) + fabs(A[8]);
        if (off <= 1e-300 || off <= 1e-18 * dia) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = A[3 * p + q];
                if (apq == 0.0) continue;
                double theta = (A[3 * q + q] - A[3 * p + p]) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {   /* A <- J^T A J */
                    double akp = A[3 * k + p], akq = A[3 * k + q];
                    A[3 * k + p] = c * akp - s * akq;
                    A[3 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    double apk = A[3 * p + k], aqk = A[3 * q + k];
                    A[3 * p + k] = c * apk - s * aqk;
                    A[3 * q + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    double vkp = V[3 * k + p], vkq = V[3 * k + q];
                    V[3 * k + p] = c * vkp - s * vkq;
                    V[3 * k + q] = s * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < 3; ++i) w[i] = A[4 * i];
}

/* Kabsch: R, t minimising sum |R s + t - q|^2 from the p2p terms. Returns 0,
 * or 1 if degenerate (count < 3 or rank(H) < 2: sigma_2 <= 1e-6 sigma_1, R15).
 * H = sum s q^T - n mu_s mu_q^T = U S V^T  ->  R = V diag(1,1,d) U^T,
 * d = sign det(V U^T); t = mu_q - R mu_s.                                  */
int orc_kabsch(const double *terms, double Tout[16])
{
    const double cnt = terms[27];
    if (!(cnt >= 3.0)) return 1;
    double ms[3], mq[3], H[9];
    for (int a = 0; a < 3; ++a) { ms[a] = terms[9 + a] / cnt; mq[a] = terms[12 + a] / cnt; }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) H[3 * a + b] = terms[3 * a + b] - cnt * ms[a] * mq[b];
    double HtH[9], w[3], V[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += H[3 * k + i] * H[3 * k + j];
            HtH[3 * i + j] = s;
        }
    jacobi3(HtH, w, V);
    int order[3] = {0, 1, 2};   /* sort eigenpairs descending */
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (w[order[j]] > w[order[i]]) { int tmp = order[i]; order[i] = order[j]; order[j] = tmp; }
    double sig[3], Vs[9], U[9];
    for (int c = 0; c < 3; ++c) {
        sig[c] = sqrt(w[order[c]] > 0.0 ? w[order[c]] : 0.0);
        for (int r = 0; r < 3; ++r) Vs[3 * r + c] = V[3 * r + order[c]];
    }
    if (!(sig[0] > 0.0) || !(sig[1] > 1e-6 * sig[0])) return 1;   /* R15: sigma via H^T H */
    for (int c = 0; c < 2; ++c)          /* U_c = H V_c / sigma_c */
        for (int r = 0; r < 3; ++r) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += H[3 * r + k] * Vs[3 * k + c];
            U[3 * r + c] = s / sig[c];
        }
    U[2] = U[3] * U[7] - U[6] * U[4];    /* U_2 = U_0 x U_1 */
    U[5] = U[6] * U[1] - U[0] * U[7];
    U[8] = U[0] * U[4] - U[3] * U[1];
    double R[9];                         /* R = V diag(1,1,d) U^T, det(R) = +1 */
    for (int pass = 0; pass < 2; ++pass) {
        double d = pass == 0 ? 1.0 : -1.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                R[3 * i + j] = Vs[3 * i + 0] * U[3 * j + 0] + Vs[3 * i + 1] * U[3 * j + 1] +
                               d * Vs[3 * i + 2] * U[3 * j + 2];
        double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                     R[2] * (R[3] * R[7] - R[4] * R[6]);
        if (det > 0.0) break;
    }
    memset(Tout, 0, 16 * sizeof(double));
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) Tout[4 * i + j] = R[3 * i + j];
        Tout[4 * i + 3] = mq[i] - (R[3 * i] * ms[0] + R[3 * i + 1] * ms[1] + R[3 * i + 2] * ms[2]);
    }
    Tout[15] = 1.0;
    return 0;
}

/* registration_icp with TransformationEstimationPointToPoint(False): the
 * same loop, criteria and flags as orc_icp, with the Kabsch
 * update T <- T_est T.                                                    */
int orc_icp_p2p(const float *src, int64_t n, const float *tgt, int64_t m, const double T0[16],
                double dmax, int32_t max_iterations, double relative_fitness, double relative_rmse,
                double T_out[16], double *fitness, double *inlier_rmse, int32_t *iterations,
                int32_t *flags, int32_t *converged)
{
    orc_grid *g = orc_grid_build(tgt, m, dmax);
    if (!g) return -1;
    double T[16], sums[ORC_NTERMS];
    memcpy(T, T0, sizeof(T));
    int32_t it = 0, fl = 0, conv = 0, passes = 0;
    orc_pass_p2p(T, src, n, tgt, m, g, dmax, NULL, sums);
    double cnt = sums[27];
    double fit = cnt / (double)n, rmse = cnt > 0 ? sqrt(sums[28] / cnt) : 0.0;
    ++passes;
    double fp = fit, rp = rmse;
    while (it < max_iterations) {
        if (cnt == 0.0) { fl |= ORC_FLAG_NO_CORR; break; }
        double dT[16];
        if (orc_kabsch(sums, dT)) { fl |= ORC_FLAG_DEGENERATE; break; }
        orc_compose(dT, T, T);
        ++it;
        orc_pass_p2p(T, src, n, tgt, m, g, dmax, NULL, sums);
        cnt = sums[27];
        fit = cnt / (double)n;
        rmse = cnt > 0 ? sqrt(sums[28] / cnt) : 0.0;
        ++passes;
        if (fabs(fit - fp) < relative_fitness && fabs(rmse - rp) < relative_rmse) { conv = 1; break; }
        fp = fit;
        rp = rmse;
    }
    if (cnt == 0.0) fl |= ORC_FLAG_NO_CORR;
    memcpy(T_out, T, sizeof(T));
    *fitness = fit;
    *inlier_rmse = rmse;
    *iterations = it;
    *flags = fl;
    *converged = conv;
    orc_grid_free(g);
    return passes;
}

/* ---------------------------------------------- estimate_normals (NEXT 4) */
/* SPEC S:67-75 (Fig. 1b "KDTreeSearchParamHybrid(radius = 0.1, max_nn =
 * 30)", "normal estimation ... #pragma omp for"): for each point the
 * hybrid neighbourhood = the min(max_nn, count) nearest points within the
 * radius (the point itself included; d^2 in fp64 as in A4, inclusive, ties
 * -> lower index), ordered by (d^2, index); mean and covariance in
 * fp64 summed in that order (cov divides by k); normal = unit eigenvector of
 * the smallest eigenvalue (Jacobi); sign: the component of largest absolute
 * value made positive (first such component on exact ties). Fewer than 3
 * neighbours -> (0,0,1), counted. Returns that count (or -1 on error).      */
typedef struct { double d2; int64_t idx; } orc_nb;

static int cmp_nb(const void *a_, const void *b_)
{
    const orc_nb *a = (const orc_nb *)a_, *b = (const orc_nb *)b_;
    if (a->d2 != b->d2) return a->d2 < b->d2 ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

int64_t orc_estimate_normals(const float *p, int64_t n, double radius, int32_t max_nn, float *out_n,
                             int32_t *nbr_count)
{
    if (n < 3 || !(radius > 0.0) || max_nn < 1) return -1;
    orc_grid *g = orc_grid_build(p, n, radius);
    orc_nb *buf = (orc_nb *)malloc(sizeof(orc_nb) * (size_t)n);
    if (!g || !buf) { orc_grid_free(g); free(buf); return -1; }
    const double r2 = radius * radius;
    int64_t fallback = 0;
    for (int64_t i = 0; i < n; ++i) {
        double s[3] = {(double)p[3 * i], (double)p[3 * i + 1], (double)p[3 * i + 2]};
        int64_t cx = cell_coord(s[0], g->o[0], g->h), cy = cell_coord(s[1], g->o[1], g->h),
                cz = cell_coord(s[2], g->o[2], g->h);
        int64_t cnt = 0;
        for (int64_t dz = -1; dz <= 1; ++dz)
            for (int64_t dy = -1; dy <= 1; ++dy)
                for (int64_t dx = -1; dx <= 1; ++dx)
                    for (int64_t k = lower(g, cz + dz, cy + dy, cx + dx); k < g->m; ++k) {
                        const orc_cellpt *c = &g->pts[k];
                        if (c->cz != cz + dz || c->cy != cy + dy || c->cx != cx + dx) break;
                        double d2 = dist2(s, p + 3 * c->idx);
                        if (d2 <= r2) { buf[cnt].d2 = d2; buf[cnt].idx = c->idx; ++cnt; }
                    }
        qsort(buf, (size_t)cnt, sizeof(orc_nb), cmp_nb);
        int64_t k = cnt < max_nn ? cnt : max_nn;
        if (nbr_count) nbr_count[i] = (int32_t)k;
        if (k < 3) {
            out_n[3 * i] = 0.0f, out_n[3 * i + 1] = 0.0f, out_n[3 * i + 2] = 1.0f;
            ++fallback;
            continue;
        }
        double mu[3] = {0, 0, 0};
        for (int64_t t = 0; t < k; ++t)
            for (int a = 0; a < 3; ++a) mu[a] += (double)p[3 * buf[t].idx + a];
        for (int a = 0; a < 3; ++a) mu[a] /= (double)k;
        double C[9] = {0};
        for (int64_t t = 0; t < k; ++t) {
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = (double)p[3 * buf[t].idx + a] - mu[a];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) C[3 * a + b] += d[a] * d[b];
        }
        for (int a = 0; a < 9; ++a) C[a] /= (double)k;
        double w[3], V[9];
        jacobi3(C, w, V);
        int sm = 0;
        for (int a = 1; a < 3; ++a) if (w[a] < w[sm]) sm = a;
        double v[3] = {V[sm], V[3 + sm], V[6 + sm]};
        double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        int big = 0;
        for (int a = 1; a < 3; ++a) if (fabs(v[a]) > fabs(v[big])) big = a;
        double sg = v[big] < 0.0 ? -1.0 : 1.0;
        for (int a = 0; a < 3; ++a) out_n[3 * i + a] = (float)(sg * v[a] / nv);
    }
    free(buf);
    orc_grid_free(g);
    return fallback;
}
