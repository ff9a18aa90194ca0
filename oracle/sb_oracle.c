/*
 * sb_oracle.c -- CPU restatement of the reference `streambench` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: it may be
 * linked/called only by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg.  The product (libsb200.so and the
 * paper_2009_10917_b200 package) never calls it.
 *
 * Parity pinned: every function below is checked against golden vectors
 * produced by the unmodified reference (tests/golden/make_golden.py imports
 * /root/reference/pkg/src/streambench) in tests/test_oracle_golden.py.
 *
 * Citations are relative to the reference tree (pkg/src/streambench/...).
 * Compile with -ffp-contract=off: every multiply and add must round
 * separately, exactly like numpy's materialised temporaries.
 *
 * Threading mirrors parallel.py:43-69 (contiguous spans, worker-count
 * invariant results); the thread count only changes speed.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOMEM 2

static int g_threads = 1;

/* parallel.py:17-25 set_num_workers */
void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int or_get_threads(void) { return g_threads; }
int or_max_threads(void) { return omp_get_num_procs(); }

/* ---------------------------------------------------------------- BS1/BS2 */

/* kernels.py:90-93 bs1_copy: y = x */
void or_bs1_copy(const double *x, double *y, int64_t n) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) y[i] = x[i];
}

/* kernels.py:96-103 bs2_axpy: y = (alpha*x) + (beta*y), each op rounded */
void or_bs2_axpy(double alpha, const double *x, double beta, double *y, int64_t n) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double a = alpha * x[i];
        double b = beta * y[i];
        y[i] = a + b;
    }
}

/* ---------------------------------------------------- lattice reduction */

/* kernels.py:63-69 _tree_fold on one row of length bs (power of two >= 2) */
static double tree_fold(double *row, int64_t bs) {
    for (int64_t k = bs / 2; k > 1; k >>= 1)
        for (int64_t s = 0; s < k; s++) row[s] = row[s] + row[s + k];
    return row[0] + row[1];
}

/* kernels.py:38-60 _accumulate_lattice.  Slot s accumulates
 * u[s + c*S]*v[s + c*S] for c = 0,1,... in order, from +0.0. */
static void accumulate_lattice(const double *u, const double *v, int64_t n,
                               int64_t bs, int64_t nb, double *lat) {
    const int64_t S = bs * nb;
    /* spans of whole blocks, as parallel.run_spans(..., nb) does */
#pragma omp parallel num_threads(g_threads)
    {
        int nt = omp_get_num_threads(), t = omp_get_thread_num();
        int64_t parts = nt < nb ? nt : nb;
        if (t < parts) {
            int64_t step = nb / parts, extra = nb % parts;
            int64_t blo = t * step + (t < extra ? t : extra);
            int64_t bhi = blo + step + (t < extra ? 1 : 0);
            int64_t lo = blo * bs, hi = bhi * bs;
            for (int64_t s = lo; s < hi; s++) lat[s] = 0.0;
            for (int64_t base = 0; base + lo < n; base += S) {
                int64_t a = base + lo;
                int64_t b = base + hi < n ? base + hi : n;
                double *seg = lat + lo;
                for (int64_t i = 0; i < b - a; i++) {
                    double pr = u[a + i] * v[a + i];
                    seg[i] = seg[i] + pr;
                }
            }
        }
    }
}

/* kernels.py:72-87 _final_reduce / _reduce_product */
int or_reduce_product(const double *u, const double *v, int64_t n, int64_t bs,
                      int64_t nb, double *result) {
    if (bs < 2 || (bs & (bs - 1)) || nb < 1) return OR_EINVAL;
    const int64_t S = bs * nb;
    double *lat = (double *)malloc(sizeof(double) * (size_t)S);
    double *partials = (double *)malloc(sizeof(double) * (size_t)nb);
    double *s = (double *)malloc(sizeof(double) * (size_t)bs);
    if (!lat || !partials || !s) { free(lat); free(partials); free(s); return OR_ENOMEM; }
    accumulate_lattice(u, v, n, bs, nb, lat);
    for (int64_t b = 0; b < nb; b++) partials[b] = tree_fold(lat + b * bs, bs);
    for (int64_t t = 0; t < bs; t++) s[t] = 0.0;
    for (int64_t base = 0; base < nb; base += bs) {
        int64_t m = nb - base < bs ? nb - base : bs;
        for (int64_t t = 0; t < m; t++) s[t] = s[t] + partials[base + t];
    }
    *result = tree_fold(s, bs);
    free(lat); free(partials); free(s);
    return OR_OK;
}

/* kernels.py:106-114 */
int or_bs3_norm2(const double *x, int64_t n, int64_t bs, int64_t nb, double *out) {
    return or_reduce_product(x, x, n, bs, nb, out);
}
int or_bs4_dot(const double *x, const double *y, int64_t n, int64_t bs, int64_t nb, double *out) {
    return or_reduce_product(x, y, n, bs, nb, out);
}

/* kernels.py:117-132 bs5_fused_cg_update: x += alpha*p; r -= alpha*ap;
 * returns _reduce_product(r, r). */
int or_bs5_fused_cg_update(double alpha, const double *p, const double *ap,
                           double *x, double *r, int64_t n, int64_t bs,
                           int64_t nb, double *out) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double a = alpha * p[i];
        x[i] = x[i] + a;
        double b = alpha * ap[i];
        r[i] = r[i] - b;
    }
    return or_reduce_product(r, r, n, bs, nb, out);
}

/* ------------------------------------------------------------ BS6 / BS7 */

/* gs.py:10-39 bs6_gather (== reference.py:46-55 gather_rowwise):
 * out[r] = +0.0 + sum of q[col_ids[c]] for c ascending in row r.
 * `carry` (may be NULL) seeds rows [0, n_carry) instead of +0.0: this is the
 * multi-rank carry-halo composition. */
void or_bs6_gather(const int32_t *row_starts, const int32_t *col_ids, int64_t ng,
                   const double *q, double *out, const double *carry, int64_t n_carry) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t r = 0; r < ng; r++) {
        double acc = (carry && r < n_carry) ? carry[r] : 0.0;
        for (int64_t c = row_starts[r]; c < row_starts[r + 1]; c++) acc = acc + q[col_ids[c]];
        out[r] = acc;
    }
}

/* gs.py:42-61 bs7_scatter: q_local[n] = q_global[ids[n]] where ids[n] >= 0 */
void or_bs7_scatter(const int32_t *ids, int64_t nl, const double *qg, double *ql) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < nl; i++) {
        int32_t id = ids[i];
        if (id >= 0) ql[i] = qg[id];
    }
}

/* ------------------------------------------------------------- builders */

/* mesh.py:73-97 build_mesh.  Returns OR_EINVAL for K<1, p<1 or g^3 > INT32_MAX
 * (the reference's own checks, mesh.py:80-84). */
int or_build_mesh(int64_t K, int64_t p, int32_t *l2g) {
    if (K < 1 || p < 1) return OR_EINVAL;
    const int64_t g = K * p + 1;
    if (g * g * g > INT32_MAX) return OR_EINVAL;
    const int64_t npe = p + 1, npe3 = npe * npe * npe, ne = K * K * K;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        int64_t ex = e % K, ey = (e / K) % K, ez = e / (K * K);
        for (int64_t nd = 0; nd < npe3; nd++) {
            int64_t i = nd % npe, j = (nd / npe) % npe, k = nd / (npe * npe);
            int64_t ax = ex * p + i, ay = ey * p + j, az = ez * p + k;
            l2g[e * npe3 + nd] = (int32_t)((az * g + ay) * g + ax);
        }
    }
    return OR_OK;
}

/* mesh.py:113-147 build_gather.
 *  counts = bincount(l2g); reject counts.min() < 1 (ret 3) and
 *  counts.max() > nodes_per_block (ret 4);
 *  col_ids = stable argsort(l2g)  (a stable counting sort is identical);
 *  row_starts = [0, cumsum(counts)];
 *  block_starts = greedy: next = searchsorted(row_starts, rs[row]+npb, 'right')-1,
 *                 clamped to [row+1, ng].
 * block_starts must have room for ng+1 entries; *n_blocks gets the count-1. */
int or_build_gather(const int32_t *l2g, int64_t nl, int64_t ng, int64_t npb,
                    int32_t *row_starts, int32_t *col_ids, int32_t *block_starts,
                    int64_t *n_blocks) {
    int64_t *cnt = (int64_t *)calloc((size_t)ng + 1, sizeof(int64_t));
    if (!cnt) return OR_ENOMEM;
    for (int64_t i = 0; i < nl; i++) {
        int32_t id = l2g[i];
        if (id < 0 || id >= ng) { free(cnt); return OR_EINVAL; }
        cnt[id]++;
    }
    int64_t cmin = INT64_MAX, cmax = 0;
    for (int64_t r = 0; r < ng; r++) {
        if (cnt[r] < cmin) cmin = cnt[r];
        if (cnt[r] > cmax) cmax = cnt[r];
    }
    if (ng > 0 && cmin < 1) { free(cnt); return 3; }
    if (cmax > npb) { free(cnt); return 4; }
    row_starts[0] = 0;
    for (int64_t r = 0; r < ng; r++) row_starts[r + 1] = (int32_t)(row_starts[r] + cnt[r]);
    /* stable counting sort == np.argsort(kind="stable") */
    for (int64_t r = 0; r < ng; r++) cnt[r] = row_starts[r];
    for (int64_t i = 0; i < nl; i++) col_ids[cnt[l2g[i]]++] = (int32_t)i;
    free(cnt);
    int64_t nb = 0, row = 0;
    block_starts[0] = 0;
    while (row < ng) {
        int64_t limit = (int64_t)row_starts[row] + npb;
        /* searchsorted(side="right") - 1: last j with row_starts[j] <= limit */
        int64_t lo = 0, hi = ng + 1; /* first index with rs > limit in [lo, hi) */
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if ((int64_t)row_starts[mid] <= limit) lo = mid + 1; else hi = mid;
        }
        int64_t nxt = lo - 1;
        if (nxt < row + 1) nxt = row + 1;
        if (nxt > ng) nxt = ng;
        block_starts[++nb] = (int32_t)nxt;
        row = nxt;
    }
    *n_blocks = nb;
    return OR_OK;
}

/* mesh.py:100-110 build_scatter_ids: ids = l2g with masked gids -> -1.
 * `masked` is a dense 0/1 byte array of length ng. */
void or_build_scatter_ids(const int32_t *l2g, int64_t nl, const uint8_t *masked, int32_t *ids) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < nl; i++) ids[i] = (masked && masked[l2g[i]]) ? -1 : l2g[i];
}
