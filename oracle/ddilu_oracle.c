/*
 * ddilu_oracle.c -- TEST INFRASTRUCTURE ONLY (CPU oracle, plain C, serial).
 *
 * A restatement of the reference package's numba kernels (ddilu 0.1.0,
 * the .py files under /root/reference/pkg/src/ddilu) for the DD-ILU + FGMRES hot path.  It is
 * the checker for the CUDA product in paper_2303_08881_b200/ and the
 * "cpu_baseline" leg of bench.py.  Nothing under paper_2303_08881_b200/ may
 * link, import or call this file.
 *
 * Parity is PINNED: tests/test_oracle_golden.py compares every function here
 * against fixtures produced by the unmodified reference (tests/golden/,
 * generator: tests/golden/make_golden.py).
 *
 * Arithmetic notes: the reference accumulates strictly left to right and numba
 * does not contract a*b+c into an FMA; build with -ffp-contract=off (see
 * oracle/Makefile) so every product is rounded before it is added.
 * Index type is int64 like the reference (sparse.py:95-96).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* Optional host threading for the TIMED reference arm of bench.py only (`bench.py --impl reference`): the
 * reference is strictly serial and g_threads = 1 (the default) IS the pinned oracle.  With more threads SpMV
 * rows and axpy entries are split (same bits) and the dot product is summed in g_threads chunks. */
#define ORC_MAX_THREADS 256
static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : (n > ORC_MAX_THREADS ? ORC_MAX_THREADS : n); }

/* fork-join over contiguous index ranges (pthreads: the image has no libgomp); a call costs ~20 us per thread,
 * it is used on vectors of >= 65536 entries only */
typedef struct {
    void (*fn)(i64 lo, i64 hi, int t, void *ctx);
    void *ctx;
    i64 lo, hi;
    int t;
} orc_task;
static void *orc_task_run(void *p)
{
    orc_task *k = (orc_task *)p;
    k->fn(k->lo, k->hi, k->t, k->ctx);
    return NULL;
}
static void orc_parallel(i64 n, int nt, void (*fn)(i64, i64, int, void *), void *ctx)
{
    pthread_t th[ORC_MAX_THREADS];
    orc_task task[ORC_MAX_THREADS];
    int started[ORC_MAX_THREADS];
    if (nt < 1)
        nt = 1;
    if (nt > ORC_MAX_THREADS)
        nt = ORC_MAX_THREADS;
    memset(task, 0, sizeof(orc_task));
    for (int t = 0; t < nt; ++t) {
        task[t].fn = fn;
        task[t].ctx = ctx;
        task[t].lo = n * t / nt;
        task[t].hi = n * (t + 1) / nt;
        task[t].t = t;
        started[t] = t > 0 && pthread_create(&th[t], NULL, orc_task_run, &task[t]) == 0;
    }
    orc_task_run(&task[0]);
    for (int t = 1; t < nt; ++t) {
        if (started[t])
            pthread_join(th[t], NULL);
        else
            orc_task_run(&task[t]);
    }
}

/* ------------------------------------------------------------------ */
/* sparse core                                                          */

/* sparse.py:219-225 (_spmv): row-serial, left-to-right sum. */
typedef struct { const i64 *rp, *ci; const double *v, *x; double *out; } spmv_ctx;
static void spmv_rows(i64 lo, i64 hi, int t, void *p)
{
    const spmv_ctx *c = (const spmv_ctx *)p;
    (void)t;
    for (i64 i = lo; i < hi; ++i) {
        double s = 0.0;
        for (i64 k = c->rp[i]; k < c->rp[i + 1]; ++k)
            s += c->v[k] * c->x[c->ci[k]];
        c->out[i] = s;
    }
}
void orc_spmv(i64 n_rows, const i64 *rp, const i64 *ci, const double *v,
              const double *x, double *out)
{
    spmv_ctx c = {rp, ci, v, x, out};
    /* rows are independent: splitting them over threads keeps every bit */
    if (g_threads > 1 && n_rows > 65536)
        orc_parallel(n_rows, g_threads, spmv_rows, &c);
    else
        spmv_rows(0, n_rows, 0, &c);
}

/* sparse.py:228-249 (_lower_solve): returns -1 or the failing row. */
i64 orc_lower_solve(i64 n, const i64 *rp, const i64 *ci, const double *v,
                    const double *b, double *x, int unit_diag)
{
    for (i64 i = 0; i < n; ++i) {
        double s = b[i], diag = 1.0;
        int seen = 0;
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            i64 j = ci[k];
            if (j < i)
                s -= v[k] * x[j];
            else if (j == i) {
                diag = v[k];
                seen = 1;
            }
        }
        if (unit_diag)
            x[i] = s;
        else {
            if (!seen || fabs(diag) < 1e-300)
                return i;
            x[i] = s / diag;
        }
    }
    return -1;
}

/* sparse.py:252-272 (_upper_solve). */
i64 orc_upper_solve(i64 n, const i64 *rp, const i64 *ci, const double *v,
                    const double *b, double *x, int unit_diag)
{
    for (i64 i = n - 1; i >= 0; --i) {
        double s = b[i], diag = 1.0;
        int seen = 0;
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            i64 j = ci[k];
            if (j > i)
                s -= v[k] * x[j];
            else if (j == i) {
                diag = v[k];
                seen = 1;
            }
        }
        if (unit_diag)
            x[i] = s;
        else {
            if (!seen || fabs(diag) < 1e-300)
                return i;
            x[i] = s / diag;
        }
    }
    return -1;
}

/* sparse.py:275-280 (_vdot). */
typedef struct { const double *a, *b; double *part; } dot_ctx;
static void dot_chunk(i64 lo, i64 hi, int t, void *p)
{
    const dot_ctx *c = (const dot_ctx *)p;
    double s = 0.0;
    for (i64 i = lo; i < hi; ++i)
        s += c->a[i] * c->b[i];
    c->part[t] = s;
}
double orc_vdot(i64 n, const double *a, const double *b)
{
    if (g_threads > 1 && n > 65536) {
        /* timed reference arm only: g_threads contiguous chunks, partial sums added in chunk order (NOT the
         * reference's single left-to-right sum; agrees to rounding) */
        double part[ORC_MAX_THREADS];
        const int nt = g_threads;
        dot_ctx c = {a, b, part};
        orc_parallel(n, nt, dot_chunk, &c);
        double s = 0.0;
        for (int t = 0; t < nt; ++t)
            s += part[t];
        return s;
    }
    double s = 0.0;
    for (i64 i = 0; i < n; ++i)
        s += a[i] * b[i];
    return s;
}

/* krylov.py:74-77 (_axpy): w += alpha * v. */
typedef struct { double alpha; const double *v; double *w; } axpy_ctx;
static void axpy_range(i64 lo, i64 hi, int t, void *p)
{
    const axpy_ctx *c = (const axpy_ctx *)p;
    (void)t;
    for (i64 i = lo; i < hi; ++i)
        c->w[i] += c->alpha * c->v[i];
}
void orc_axpy(i64 n, double alpha, const double *v, double *w)
{
    axpy_ctx c = {alpha, v, w};
    if (g_threads > 1 && n > 65536)
        orc_parallel(n, g_threads, axpy_range, &c);
    else
        axpy_range(0, n, 0, &c);
}

/* sort one CSR row segment by column (columns are unique, so any sort gives
 * the argsort result of sparse.py:298-300 / :328-330). */
static void sort_row(i64 *c, double *v, i64 len)
{
    for (i64 a = 1; a < len; ++a) {
        i64 cc = c[a];
        double vv = v[a];
        i64 b = a - 1;
        while (b >= 0 && c[b] > cc) {
            c[b + 1] = c[b];
            v[b + 1] = v[b];
            --b;
        }
        c[b + 1] = cc;
        v[b + 1] = vv;
    }
}

/* sparse.py:283-300 (_permute): B[fwd[i], fwd[j]] = A[i, j]; new_rp is given. */
void orc_permute(i64 n, const i64 *rp, const i64 *ci, const double *v,
                 const i64 *fwd, const i64 *new_rp, i64 *new_ci, double *new_v)
{
    for (i64 i = 0; i < n; ++i) {
        i64 p = new_rp[fwd[i]];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k, ++p) {
            new_ci[p] = fwd[ci[k]];
            new_v[p] = v[k];
        }
    }
    for (i64 i = 0; i < n; ++i)
        sort_row(new_ci + new_rp[i], new_v + new_rp[i], new_rp[i + 1] - new_rp[i]);
}

/* sparse.py:303-311 (_gather_rows_count). */
void orc_gather_rows_count(const i64 *rp, const i64 *ci, i64 n_sel,
                           const i64 *rows, const i64 *colmap, i64 *counts)
{
    for (i64 r = 0; r < n_sel; ++r) {
        i64 i = rows[r], c = 0;
        for (i64 k = rp[i]; k < rp[i + 1]; ++k)
            if (colmap[ci[k]] >= 0)
                ++c;
        counts[r] = c;
    }
}

/* sparse.py:314-330 (_gather_rows_fill). */
void orc_gather_rows_fill(const i64 *rp, const i64 *ci, const double *v,
                          i64 n_sel, const i64 *rows, const i64 *colmap,
                          const i64 *out_rp, i64 *out_ci, double *out_v,
                          int resort)
{
    for (i64 r = 0; r < n_sel; ++r) {
        i64 i = rows[r], p = out_rp[r];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            i64 m = colmap[ci[k]];
            if (m >= 0) {
                out_ci[p] = m;
                out_v[p] = v[k];
                ++p;
            }
        }
        if (resort)
            sort_row(out_ci + out_rp[r], out_v + out_rp[r], out_rp[r + 1] - out_rp[r]);
    }
}

/* sparse.py:373-382 (_transpose); out_rp prepared by the caller (sparse.py:508-512). */
void orc_transpose(i64 n_rows, i64 n_cols, const i64 *rp, const i64 *ci,
                   const double *v, const i64 *out_rp, i64 *out_ci, double *out_v)
{
    i64 *fill = (i64 *)malloc(sizeof(i64) * (size_t)(n_cols > 0 ? n_cols : 1));
    memcpy(fill, out_rp, sizeof(i64) * (size_t)n_cols);
    for (i64 i = 0; i < n_rows; ++i)
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            i64 p = fill[ci[k]]++;
            out_ci[p] = i;
            out_v[p] = v[k];
        }
    free(fill);
}

/* ------------------------------------------------------------------ */
/* orderings                                                            */

/* ordering.py:32-70 (_sym_merge_count / _sym_merge_fill): pattern(A) U
 * pattern(A^T) minus the diagonal.  With out_ci == NULL only counts. */
void orc_sym_merge(i64 n, const i64 *rp, const i64 *ci, const i64 *trp,
                   const i64 *tci, i64 *counts, const i64 *out_rp, i64 *out_ci)
{
    for (i64 i = 0; i < n; ++i) {
        i64 a = rp[i], ae = rp[i + 1], b = trp[i], be = trp[i + 1];
        i64 c = 0, p = out_ci ? out_rp[i] : 0;
        while (a < ae || b < be) {
            i64 j;
            if (a < ae && (b >= be || ci[a] <= tci[b])) {
                j = ci[a];
                if (b < be && tci[b] == j)
                    ++b;
                ++a;
            } else {
                j = tci[b];
                ++b;
            }
            if (j != i) {
                if (out_ci)
                    out_ci[p++] = j;
                ++c;
            }
        }
        if (counts)
            counts[i] = c;
    }
}

/* ordering.py:88-94 (_mark_exterior). */
void orc_mark_exterior(i64 n, const i64 *rp, const i64 *ci, const i64 *owner,
                       uint8_t *exterior)
{
    for (i64 i = 0; i < n; ++i)
        for (i64 k = rp[i]; k < rp[i + 1]; ++k)
            if (owner[ci[k]] != owner[i]) {
                exterior[i] = 1;
                break;
            }
}

/* ordering.py:97-127 (_grow_regions): greedy BFS partition fallback. */
void orc_grow_regions(i64 n, const i64 *rp, const i64 *ci, i64 n_dom,
                      const i64 *sizes, i64 *owner)
{
    i64 *queue = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 *queued = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    for (i64 i = 0; i < n; ++i)
        queued[i] = -1;
    i64 scan = 0;
    for (i64 d = 0; d < n_dom; ++d) {
        i64 need = sizes[d], count = 0, head = 0, tail = 0;
        while (count < need) {
            if (head == tail) {
                while (owner[scan] >= 0)
                    ++scan;
                queue[tail++] = scan;
                queued[scan] = d;
            }
            i64 u = queue[head++];
            if (owner[u] >= 0)
                continue;
            owner[u] = d;
            if (++count == need)
                break;
            for (i64 k = rp[u]; k < rp[u + 1]; ++k) {
                i64 w = ci[k];
                if (owner[w] < 0 && queued[w] != d) {
                    queued[w] = d;
                    queue[tail++] = w;
                }
            }
        }
    }
    free(queue);
    free(queued);
}

/* ordering.py:304-337 (_bfs_ecc): level BFS from root; returns the
 * eccentricity and (through *last) the min-degree / min-index node of the
 * last level. */
static i64 bfs_ecc(const i64 *rp, const i64 *ci, i64 root, i64 *dist, i64 stamp,
                   i64 *mark, i64 *q, i64 *last)
{
    i64 head = 0, tail = 0, ecc = 0;
    q[tail++] = root;
    mark[root] = stamp;
    dist[root] = 0;
    while (head < tail) {
        i64 u = q[head++], du = dist[u];
        if (du > ecc)
            ecc = du;
        for (i64 k = rp[u]; k < rp[u + 1]; ++k) {
            i64 w = ci[k];
            if (mark[w] != stamp) {
                mark[w] = stamp;
                dist[w] = du + 1;
                q[tail++] = w;
            }
        }
    }
    i64 best = -1, best_deg = 0;
    for (i64 t = 0; t < tail; ++t) {
        i64 u = q[t];
        if (dist[u] == ecc) {
            i64 deg = rp[u + 1] - rp[u];
            if (best == -1 || deg < best_deg || (deg == best_deg && u < best)) {
                best = u;
                best_deg = deg;
            }
        }
    }
    *last = best;
    return ecc;
}

/* ordering.py:340-397 (_rcm_order): Cuthill-McKee order (not yet reversed) of
 * the symmetrised adjacency (rp, ci), components by smallest index, George-Liu
 * pseudo-peripheral roots, neighbours by (degree, index). */
void orc_cm_order(i64 n, const i64 *rp, const i64 *ci, i64 *order)
{
    uint8_t *visited = (uint8_t *)calloc((size_t)(n + 1), 1);
    i64 *dist = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 *mark = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 *q = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 *nbrs = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    for (i64 i = 0; i < n; ++i)
        mark[i] = -1;
    i64 pos = 0, scan = 0, stamp = 0;
    while (pos < n) {
        while (visited[scan])
            ++scan;
        i64 root = scan, cand, nxt;
        i64 ecc_root = bfs_ecc(rp, ci, root, dist, stamp++, mark, q, &cand);
        for (;;) {
            i64 ecc_cand = bfs_ecc(rp, ci, cand, dist, stamp++, mark, q, &nxt);
            if (ecc_cand > ecc_root) {
                root = cand;
                ecc_root = ecc_cand;
                cand = nxt;
            } else
                break;
        }
        i64 head = pos;
        visited[root] = 1;
        order[pos++] = root;
        while (head < pos) {
            i64 u = order[head++], cnt = 0;
            for (i64 k = rp[u]; k < rp[u + 1]; ++k) {
                i64 w = ci[k];
                if (!visited[w]) {
                    visited[w] = 1;
                    nbrs[cnt++] = w;
                }
            }
            for (i64 a = 1; a < cnt; ++a) {
                i64 w = nbrs[a], dw = rp[w + 1] - rp[w], b = a - 1;
                while (b >= 0) {
                    i64 y = nbrs[b], dy = rp[y + 1] - rp[y];
                    if (dy > dw || (dy == dw && y > w)) {
                        nbrs[b + 1] = y;
                        --b;
                    } else
                        break;
                }
                nbrs[b + 1] = w;
            }
            for (i64 a = 0; a < cnt; ++a)
                order[pos++] = nbrs[a];
        }
    }
    free(visited);
    free(dist);
    free(mark);
    free(q);
    free(nbrs);
}

/* Level schedule (absent from the reference; defined in
 * SURVEY.md 8c): lev[i] = 1 + max lev[j] over stored j < i (lower) or j > i
 * (upper), 0 for rows with no such entry.  Returns the number of levels. */
i64 orc_levels(i64 n, const i64 *rp, const i64 *ci, int upper, i64 *lev)
{
    i64 depth = 0;
    if (!upper) {
        for (i64 i = 0; i < n; ++i) {
            i64 l = 0;
            for (i64 k = rp[i]; k < rp[i + 1]; ++k)
                if (ci[k] < i && lev[ci[k]] + 1 > l)
                    l = lev[ci[k]] + 1;
            lev[i] = l;
            if (l + 1 > depth)
                depth = l + 1;
        }
    } else {
        for (i64 i = n - 1; i >= 0; --i) {
            i64 l = 0;
            for (i64 k = rp[i]; k < rp[i + 1]; ++k)
                if (ci[k] > i && lev[ci[k]] + 1 > l)
                    l = lev[ci[k]] + 1;
            lev[i] = l;
            if (l + 1 > depth)
                depth = l + 1;
        }
    }
    return n ? depth : 0;
}

/* ------------------------------------------------------------------ */
/* factorisations                                                       */

/* factor.py:198-216 (_split_counts). */
void orc_split_counts(i64 n, const i64 *a_rp, const i64 *a_ci, i64 n_elim,
                      i64 *pc, i64 *kc)
{
    for (i64 i = 0; i < n; ++i) {
        i64 lim = i < n_elim ? i : n_elim, npv = 0, nk = 0;
        int has_diag = 0;
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            i64 j = a_ci[s];
            if (j < lim)
                ++npv;
            else {
                ++nk;
                if (j == i)
                    has_diag = 1;
            }
        }
        if (!has_diag)
            ++nk;
        pc[i] = npv;
        kc[i] = nk;
    }
}

/* factor.py:219-246 (_split_fill). */
void orc_split_fill(i64 n, const i64 *a_rp, const i64 *a_ci, const double *a_v,
                    i64 n_elim, const i64 *p_rp, i64 *p_ci, double *p_v,
                    const i64 *k_rp, i64 *k_ci, double *k_v)
{
    for (i64 i = 0; i < n; ++i) {
        i64 lim = i < n_elim ? i : n_elim, pp = p_rp[i], kp = k_rp[i];
        int placed = 0;
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            i64 j = a_ci[s];
            if (j < lim) {
                p_ci[pp] = j;
                p_v[pp++] = a_v[s];
            } else {
                if (!placed && j > i) {
                    k_ci[kp] = i;
                    k_v[kp++] = 0.0;
                    placed = 1;
                }
                if (j == i)
                    placed = 1;
                k_ci[kp] = j;
                k_v[kp++] = a_v[s];
            }
        }
        if (!placed) {
            k_ci[kp] = i;
            k_v[kp++] = 0.0;
        }
    }
}

/* factor.py:435-443 (_row_inf_norms). */
void orc_row_inf_norms(i64 n, const i64 *a_rp, const double *a_v, double *out)
{
    for (i64 i = 0; i < n; ++i) {
        double m = 0.0;
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            double t = fabs(a_v[s]);
            if (t > m)
                m = t;
        }
        out[i] = m > 0.0 ? m : 1.0;
    }
}

/* factor.py:397-432 (_factor_split): IKJ elimination on the fixed split
 * pattern; MILU compensation and the pivot safeguard for rows < n_elim. */
void orc_factor_split(i64 n, const i64 *p_rp, const i64 *p_ci, double *p_v,
                      const i64 *k_rp, const i64 *k_ci, double *k_v, i64 n_elim,
                      int milu, const double *target, const double *wvec,
                      double delta, const double *rownorm)
{
    i64 *where = (i64 *)calloc((size_t)(n + 1), sizeof(i64));
    for (i64 i = 0; i < n; ++i) {
        for (i64 s = p_rp[i]; s < p_rp[i + 1]; ++s)
            where[p_ci[s]] = -(s + 1);
        for (i64 s = k_rp[i]; s < k_rp[i + 1]; ++s)
            where[k_ci[s]] = s + 1;
        double hy = 0.0;
        for (i64 s = p_rp[i]; s < p_rp[i + 1]; ++s) {
            i64 k = p_ci[s];
            double lik = p_v[s] / k_v[k_rp[k]];
            p_v[s] = lik;
            for (i64 t = k_rp[k] + 1; t < k_rp[k + 1]; ++t) {
                i64 j = k_ci[t];
                double upd = lik * k_v[t];
                i64 w = where[j];
                if (w > 0)
                    k_v[w - 1] -= upd;
                else if (w < 0)
                    p_v[-w - 1] -= upd;
                else if (milu)
                    hy -= upd * target[j];
            }
        }
        if (i < n_elim) {
            i64 sd = k_rp[i];
            if (milu)
                k_v[sd] += (hy - wvec[i]) / target[i];
            double rn = rownorm[i], d = k_v[sd];
            if (fabs(d) < delta * rn)
                k_v[sd] = d >= 0.0 ? delta * rn : -delta * rn;
        }
        for (i64 s = p_rp[i]; s < p_rp[i + 1]; ++s)
            where[p_ci[s]] = 0;
        for (i64 s = k_rp[i]; s < k_rp[i + 1]; ++s)
            where[k_ci[s]] = 0;
    }
    free(where);
}

/* factor.py:465-479 (_select_largest): ties toward the smaller column. */
static void select_largest(const double *vals, i64 count, i64 keep, uint8_t *sel)
{
    for (i64 s = 0; s < count; ++s)
        sel[s] = 0;
    i64 m = keep < count ? keep : count;
    for (i64 r = 0; r < m; ++r) {
        i64 best = -1;
        double bestv = -1.0;
        for (i64 s = 0; s < count; ++s)
            if (!sel[s] && fabs(vals[s]) > bestv) {
                best = s;
                bestv = fabs(vals[s]);
            }
        sel[best] = 1;
    }
}

typedef struct {
    i64 *ci;
    double *v;
    i64 cap;
} grow_t;

static void grow_reserve(grow_t *g, i64 need)
{
    if (need <= g->cap)
        return;
    i64 cap = g->cap * 2 > need ? g->cap * 2 : need;
    g->ci = (i64 *)realloc(g->ci, sizeof(i64) * (size_t)cap);
    g->v = (double *)realloc(g->v, sizeof(double) * (size_t)cap);
    g->cap = cap;
}

/* factor.py:482-656 (_ilut_factor): dual-threshold ILUT, rows >= n_elim are
 * Schur rows (own tolerance tau_s, no cap, no safeguard).  l_rp / u_rp have
 * n+1 entries; the entry arrays are malloc'ed here and handed back through
 * the out pointers (free with orc_free). */
void orc_ilut_factor(i64 n, const i64 *a_rp, const i64 *a_ci, const double *a_v,
                     i64 n_elim, double tau, i64 maxfill, double tau_s,
                     double delta, i64 *l_rp, i64 **l_ci_out, double **l_v_out,
                     i64 *u_rp, i64 **u_ci_out, double **u_v_out)
{
    grow_t L = {0, 0, 0}, U = {0, 0, 0};
    grow_reserve(&L, a_rp[n] + 16);
    grow_reserve(&U, a_rp[n] + n + 16);
    double *udiag = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    i64 *nxt = (i64 *)malloc(sizeof(i64) * (size_t)(n + 2));
    double *w = (double *)calloc((size_t)(n + 1), sizeof(double));
    i64 *cand_c = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    double *cand_v = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    uint8_t *sel = (uint8_t *)malloc((size_t)(n + 1));
    l_rp[0] = 0;
    u_rp[0] = 0;
    for (i64 i = 0; i < n; ++i) {
        i64 lim = i < n_elim ? i : n_elim;
        double nrm = 0.0, mx = 0.0;
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            double t = a_v[s];
            nrm += t * t;
            if (fabs(t) > mx)
                mx = fabs(t);
        }
        nrm = sqrt(nrm);
        double thresh = nrm > 0.0 ? tau * nrm : 0.0;
        if (mx == 0.0)
            mx = 1.0;
        /* sorted linked list of the row, diagonal inserted (value 0) if absent */
        i64 head = n, last = -1;
        int placed = 0;
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            i64 j = a_ci[s];
            if (!placed && j >= i) {
                if (j > i) {
                    if (last < 0)
                        head = i;
                    else
                        nxt[last] = i;
                    nxt[i] = n;
                    w[i] = 0.0;
                    last = i;
                }
                placed = 1;
            }
            if (last < 0)
                head = j;
            else
                nxt[last] = j;
            nxt[j] = n;
            w[j] = a_v[s];
            last = j;
        }
        if (!placed) {
            if (last < 0)
                head = i;
            else
                nxt[last] = i;
            nxt[i] = n;
            w[i] = 0.0;
        }
        /* eliminate pivots in increasing column order */
        for (i64 k = head; k < lim; k = nxt[k]) {
            double lik = w[k] / udiag[k];
            if (fabs(lik) < thresh) {
                w[k] = 0.0;
                continue;
            }
            w[k] = lik;
            i64 cursor = k;
            for (i64 t = u_rp[k]; t < u_rp[k + 1]; ++t) {
                i64 j = U.ci[t];
                if (j == k)
                    continue;
                double upd = lik * U.v[t];
                while (nxt[cursor] <= j)
                    cursor = nxt[cursor];
                if (cursor == j)
                    w[j] -= upd;
                else {
                    nxt[j] = nxt[cursor];
                    nxt[cursor] = j;
                    w[j] = -upd;
                }
            }
        }
        /* L part */
        i64 nl = 0;
        for (i64 j = head; j < lim; j = nxt[j])
            if (fabs(w[j]) >= thresh && w[j] != 0.0) {
                cand_c[nl] = j;
                cand_v[nl++] = w[j];
            }
        select_largest(cand_v, nl, maxfill, sel);
        i64 pp = l_rp[i];
        grow_reserve(&L, pp + nl);
        for (i64 s = 0; s < nl; ++s)
            if (sel[s]) {
                L.ci[pp] = cand_c[s];
                L.v[pp++] = cand_v[s];
            }
        l_rp[i + 1] = pp;
        /* U / kept part */
        i64 nu = 0, nc = 0;
        for (i64 j = head; j < n; j = nxt[j])
            if (j >= lim) {
                cand_c[nu] = j;
                cand_v[nu++] = w[j];
            }
        if (i < n_elim) {
            for (i64 s = 0; s < nu; ++s)
                if (cand_c[s] == i || fabs(cand_v[s]) >= thresh) {
                    cand_c[nc] = cand_c[s];
                    cand_v[nc++] = cand_v[s];
                }
            select_largest(cand_v, nc, maxfill, sel);
            for (i64 s = 0; s < nc; ++s)
                if (cand_c[s] == i)
                    sel[s] = 1;
        } else {
            double snrm = 0.0;
            for (i64 s = 0; s < nu; ++s)
                snrm += cand_v[s] * cand_v[s];
            snrm = sqrt(snrm);
            double sth = tau_s * snrm;
            for (i64 s = 0; s < nu; ++s)
                if (cand_c[s] == i || fabs(cand_v[s]) >= sth) {
                    cand_c[nc] = cand_c[s];
                    cand_v[nc++] = cand_v[s];
                }
            for (i64 s = 0; s < nc; ++s)
                sel[s] = 1;
        }
        i64 kp = u_rp[i];
        grow_reserve(&U, kp + nc);
        for (i64 s = 0; s < nc; ++s)
            if (sel[s]) {
                if (cand_c[s] == i && i < n_elim) {
                    double d = cand_v[s];
                    if (fabs(d) < delta * mx)
                        d = d >= 0.0 ? delta * mx : -delta * mx;
                    cand_v[s] = d;
                    udiag[i] = d;
                }
                U.ci[kp] = cand_c[s];
                U.v[kp++] = cand_v[s];
            }
        u_rp[i + 1] = kp;
    }
    free(udiag);
    free(nxt);
    free(w);
    free(cand_c);
    free(cand_v);
    free(sel);
    *l_ci_out = L.ci;
    *l_v_out = L.v;
    *u_ci_out = U.ci;
    *u_v_out = U.v;
}

/* factor.py:270-369 (_iluk_symbolic): level-of-fill pattern.  Row i starts as
 * pattern(A_i) plus the diagonal, all at level 0; every pivot k < lim of the
 * working row (in increasing column order, fill included) merges the kept
 * part of row k beyond its diagonal with level lev(i,k) + lev(k,j) + 1, kept
 * if <= klevel, the smaller level winning on a position already present.
 * The working row is a sorted array here (the reference threads a linked
 * list through an n-vector; the visiting order and the results are the same).
 * p_rp / k_rp have n+1 entries, column arrays are malloc'ed (orc_free). */
void orc_iluk_symbolic(i64 n, const i64 *a_rp, const i64 *a_ci, i64 n_elim,
                       i64 klevel, i64 *p_rp, i64 **p_ci_out, i64 *k_rp,
                       i64 **k_ci_out)
{
    i64 pcap = a_rp[n] + 16, kcap = a_rp[n] + n + 16;
    i64 *p_ci = (i64 *)malloc(sizeof(i64) * (size_t)pcap);
    i64 *k_ci = (i64 *)malloc(sizeof(i64) * (size_t)kcap);
    i64 *k_lv = (i64 *)malloc(sizeof(i64) * (size_t)kcap);
    i64 wcap = 64;
    i64 *wc = (i64 *)malloc(sizeof(i64) * (size_t)wcap);   /* working row: columns  */
    i64 *wl = (i64 *)malloc(sizeof(i64) * (size_t)wcap);   /* ... and their levels  */
    p_rp[0] = 0;
    k_rp[0] = 0;
    for (i64 i = 0; i < n; ++i) {
        const i64 lim = i < n_elim ? i : n_elim;
        i64 len = 0;
        int have_diag = 0;
        if (a_rp[i + 1] - a_rp[i] + 1 > wcap) {
            wcap = 2 * (a_rp[i + 1] - a_rp[i] + 1);
            wc = (i64 *)realloc(wc, sizeof(i64) * (size_t)wcap);
            wl = (i64 *)realloc(wl, sizeof(i64) * (size_t)wcap);
        }
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            const i64 j = a_ci[s];
            if (!have_diag && j >= i) {
                if (j > i) {
                    wc[len] = i;
                    wl[len++] = 0;
                }
                have_diag = 1;
            }
            wc[len] = j;
            wl[len++] = 0;
        }
        if (!have_diag) {
            wc[len] = i;
            wl[len++] = 0;
        }
        for (i64 pos = 0; pos < len && wc[pos] < lim; ++pos) {
            const i64 k = wc[pos], lk = wl[pos];
            i64 at = pos;                      /* merge cursor: columns only grow */
            for (i64 t = k_rp[k] + 1; t < k_rp[k + 1]; ++t) {
                const i64 j = k_ci[t], nl = lk + k_lv[t] + 1;
                if (nl > klevel)
                    continue;
                while (at + 1 < len && wc[at + 1] <= j)
                    ++at;
                if (wc[at] == j) {
                    if (nl < wl[at])
                        wl[at] = nl;
                } else {                       /* insert after `at` */
                    if (len + 1 > wcap) {
                        wcap *= 2;
                        wc = (i64 *)realloc(wc, sizeof(i64) * (size_t)wcap);
                        wl = (i64 *)realloc(wl, sizeof(i64) * (size_t)wcap);
                    }
                    memmove(wc + at + 2, wc + at + 1, sizeof(i64) * (size_t)(len - at - 1));
                    memmove(wl + at + 2, wl + at + 1, sizeof(i64) * (size_t)(len - at - 1));
                    wc[at + 1] = j;
                    wl[at + 1] = nl;
                    ++len;
                    ++at;
                }
            }
        }
        i64 np = 0;
        while (np < len && wc[np] < lim)
            ++np;
        if (p_rp[i] + np > pcap) {
            pcap = 2 * pcap > p_rp[i] + np ? 2 * pcap : p_rp[i] + np;
            p_ci = (i64 *)realloc(p_ci, sizeof(i64) * (size_t)pcap);
        }
        if (k_rp[i] + len - np > kcap) {
            kcap = 2 * kcap > k_rp[i] + len - np ? 2 * kcap : k_rp[i] + len - np;
            k_ci = (i64 *)realloc(k_ci, sizeof(i64) * (size_t)kcap);
            k_lv = (i64 *)realloc(k_lv, sizeof(i64) * (size_t)kcap);
        }
        memcpy(p_ci + p_rp[i], wc, sizeof(i64) * (size_t)np);
        memcpy(k_ci + k_rp[i], wc + np, sizeof(i64) * (size_t)(len - np));
        memcpy(k_lv + k_rp[i], wl + np, sizeof(i64) * (size_t)(len - np));
        p_rp[i + 1] = p_rp[i] + np;
        k_rp[i + 1] = k_rp[i] + len - np;
    }
    free(k_lv);
    free(wc);
    free(wl);
    *p_ci_out = p_ci;
    *k_ci_out = k_ci;
}

/* factor.py:372-390 (_prefill): values of A into the matching slots of a
 * superset pattern; fill positions keep 0.  upper_part 0: columns < lim of
 * every row, 1: columns >= lim (lim = min(i, n_elim)). */
void orc_prefill(i64 n, const i64 *a_rp, const i64 *a_ci, const double *a_v,
                 const i64 *rp, const i64 *ci, double *v, i64 n_elim, int upper_part)
{
    for (i64 i = 0; i < n; ++i) {
        const i64 lim = i < n_elim ? i : n_elim;
        i64 t = rp[i];
        for (i64 s = a_rp[i]; s < a_rp[i + 1]; ++s) {
            const i64 j = a_ci[s];
            if ((upper_part == 0) != (j < lim))
                continue;
            while (t < rp[i + 1] && ci[t] < j)
                ++t;
            if (t < rp[i + 1] && ci[t] == j)
                v[t++] = a_v[s];
        }
    }
}

void orc_free(void *p) { free(p); }

/* factor.py:756-781 (_col_split_counts / _col_split_fill): rows [r0, r1) cut
 * at column csplit; the high part is shifted to start at column 0.  With
 * lo_ci == NULL only the low counts are produced. */
void orc_col_split(const i64 *rp, const i64 *ci, const double *v, i64 r0, i64 r1,
                   i64 csplit, i64 *lo_counts, const i64 *lo_rp, i64 *lo_ci,
                   double *lo_v, const i64 *hi_rp, i64 *hi_ci, double *hi_v)
{
    for (i64 r = r0; r < r1; ++r) {
        if (!lo_ci) {
            i64 lo = 0;
            for (i64 s = rp[r]; s < rp[r + 1]; ++s)
                if (ci[s] < csplit)
                    ++lo;
            lo_counts[r - r0] = lo;
            continue;
        }
        i64 lp = lo_rp[r - r0], hp = hi_rp[r - r0];
        for (i64 s = rp[r]; s < rp[r + 1]; ++s) {
            i64 j = ci[s];
            if (j < csplit) {
                lo_ci[lp] = j;
                lo_v[lp++] = v[s];
            } else {
                hi_ci[hp] = j - csplit;
                hi_v[hp++] = v[s];
            }
        }
    }
}

/* precond.py:154-159 (_keep_cross_block). */
void orc_keep_cross_block(i64 n_rows, const i64 *rp, const i64 *ci,
                          const i64 *block_of, uint8_t *keep)
{
    for (i64 i = 0; i < n_rows; ++i)
        for (i64 t = rp[i]; t < rp[i + 1]; ++t)
            keep[t] = block_of[ci[t]] != block_of[i];
}

/* precond.py:84-92 (_l1_row_shifts). */
void orc_l1_row_shifts(const i64 *rp, const i64 *ci, const double *v,
                       const i64 *owner, i64 n_sel, const i64 *rows, i64 dom,
                       double *out)
{
    for (i64 k = 0; k < n_sel; ++k) {
        i64 r = rows[k];
        double s = 0.0;
        for (i64 t = rp[r]; t < rp[r + 1]; ++t)
            if (owner[ci[t]] != dom)
                s += fabs(v[t]);
        out[k] = s;
    }
}
