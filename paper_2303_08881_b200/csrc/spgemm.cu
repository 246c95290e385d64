// Sparse product C = A B with the exact structural pattern (replaces sparse.py:333-370 `_spgemm_count`,
// `_spgemm_fill` behind `sparse_matmul`, sparse.py:487-505; used for explicit Schur-complement assembly options).
//
// The reference walks row i of A, and for every entry (i, k) the row k of B, accumulating acc[j] with a marker
// array: the FIRST product that reaches column j is assigned, later ones are added in traversal order, and the
// row is emitted in ascending column order with cancelled entries kept.  Here: (1) an upper bound of the row's
// products = sum of the B row lengths (count kernel, scanned by the caller); (2) one thread per row expands its
// products in the same traversal order into scratch and insertion-sorts them stably by column, so equal
// columns stay in traversal order, and counts the distinct columns; (3) after the scan of those counts the
// runs of equal columns are summed left to right -- the reference's additions, in the reference's order, every
// product rounded before it is added (-fmad=false): bit-exact values and pattern.
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

__global__ void spgemm_bound_kernel(int n_rows, const int *__restrict__ a_rp, const int *__restrict__ a_ci,
                                    const int *__restrict__ b_rp, int *__restrict__ bound) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    int c = 0;
    for (int ka = a_rp[i], ke = a_rp[i + 1]; ka < ke; ++ka) {
        const int k = a_ci[ka];
        c += b_rp[k + 1] - b_rp[k];
    }
    bound[i] = c;
}

__global__ void spgemm_expand_kernel(int n_rows, const int *__restrict__ a_rp, const int *__restrict__ a_ci,
                                     const double *__restrict__ a_v, const int *__restrict__ b_rp,
                                     const int *__restrict__ b_ci, const double *__restrict__ b_v,
                                     const int *__restrict__ off, int *__restrict__ s_col, double *__restrict__ s_val,
                                     int *__restrict__ counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const int base = off[i];
    int m = 0;
    for (int ka = a_rp[i], ke = a_rp[i + 1]; ka < ke; ++ka) {
        const int k = a_ci[ka];
        const double av = a_v[ka];
        for (int kb = b_rp[k], kbe = b_rp[k + 1]; kb < kbe; ++kb) {
            // stable insertion by column: an equal column stays BEHIND the earlier products of that column
            const int j = b_ci[kb];
            const double pv = av * b_v[kb];
            int q = base + m;
            while (q > base && s_col[q - 1] > j) {
                s_col[q] = s_col[q - 1];
                s_val[q] = s_val[q - 1];
                --q;
            }
            s_col[q] = j;
            s_val[q] = pv;
            ++m;
        }
    }
    int distinct = 0;
    for (int q = base; q < base + m; ++q)
        if (q == base || s_col[q] != s_col[q - 1]) ++distinct;
    counts[i] = distinct;
}

__global__ void spgemm_compact_kernel(int n_rows, const int *__restrict__ off, const int *__restrict__ s_col,
                                      const double *__restrict__ s_val, const int *__restrict__ out_rp,
                                      int *__restrict__ out_ci, double *__restrict__ out_v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const int b = off[i], e = off[i + 1];
    int p = out_rp[i] - 1;
    double acc = 0.0;
    for (int q = b; q < e; ++q) {
        if (q == b || s_col[q] != s_col[q - 1]) {
            if (p >= out_rp[i]) out_v[p] = acc;
            ++p;
            out_ci[p] = s_col[q];
            acc = s_val[q];                 // first product of the column is assigned ...
        } else {
            acc += s_val[q];                // ... the others are added in traversal order
        }
    }
    if (p >= out_rp[i]) out_v[p] = acc;
}

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

extern "C" int ddilu_spgemm_bound(int n_rows, const int *a_rp, const int *a_ci, const int *b_rp, int *bound,
                                  void *stream) {
    if (n_rows <= 0) return DDILU_OK;
    spgemm_bound_kernel<<<div_up(n_rows, 256), 256, 0, ST(stream)>>>(n_rows, a_rp, a_ci, b_rp, bound);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_spgemm_expand(int n_rows, const int *a_rp, const int *a_ci, const double *a_v, const int *b_rp,
                                   const int *b_ci, const double *b_v, const int *off, int *s_col, double *s_val,
                                   int *counts, void *stream) {
    if (n_rows <= 0) return DDILU_OK;
    spgemm_expand_kernel<<<div_up(n_rows, 128), 128, 0, ST(stream)>>>(n_rows, a_rp, a_ci, a_v, b_rp, b_ci, b_v, off,
                                                                     s_col, s_val, counts);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_spgemm_compact(int n_rows, const int *off, const int *s_col, const double *s_val,
                                    const int *out_rp, int *out_ci, double *out_v, void *stream) {
    if (n_rows <= 0) return DDILU_OK;
    spgemm_compact_kernel<<<div_up(n_rows, 128), 128, 0, ST(stream)>>>(n_rows, off, s_col, s_val, out_rp, out_ci,
                                                                      out_v);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
