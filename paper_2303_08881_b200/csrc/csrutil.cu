// CSR plumbing for the setup phase: classification of interface (exterior)
// nodes, local-block extraction with column remapping, symmetrised adjacency.
// Replaces ordering.py:88-94 (`_mark_exterior`), sparse.py:303-330
// (`_gather_rows_*`), ordering.py:32-81 (`_sym_*`), precond.py:154-170.
// Streaming count -> scan -> fill passes, one thread per row (rows are short).
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

#define GRID_STRIDE(i, n) \
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

// A node is exterior when the symmetrised pattern couples it to another owner:
// an entry (i, j) with owner[i] != owner[j] marks both ends.
__global__ void mark_exterior(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                              const int *__restrict__ owner, int *exterior) {
    GRID_STRIDE(i, n) {
        const int oi = owner[i];
        bool mine = false;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (owner[j] != oi) {
                mine = true;
                exterior[j] = 1;
            }
        }
        if (mine) exterior[i] = 1;
    }
}

// key[i] = exterior[i] * p + owner[i]; val[i] = i  (sorted by key = layout order)
__global__ void layout_keys(int n, const int *__restrict__ owner, const int *__restrict__ exterior, int p,
                            int *__restrict__ keys, int *__restrict__ vals) {
    GRID_STRIDE(i, n) {
        keys[i] = (exterior[i] ? p : 0) + owner[i];
        vals[i] = (int)i;
    }
}

// out[k] = first position q with sorted[q] >= k, for k = 0..nkeys
__global__ void lower_bounds(const int *__restrict__ sorted, int n, int nkeys, int *__restrict__ out) {
    GRID_STRIDE(k, nkeys + 1) {
        int lo = 0, hi = n;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (sorted[mid] < (int)k) lo = mid + 1; else hi = mid;
        }
        out[k] = lo;
    }
}

// map[nodes[k]] = offset + k
__global__ void build_map(int n_nodes, const int *__restrict__ nodes, int offset, int *__restrict__ map) {
    GRID_STRIDE(k, n_nodes) map[nodes[k]] = offset + (int)k;
}

// filter: 0 keep all mapped columns, 1 only same-domain, 2 only different-domain, +4 drop the diagonal
__device__ __forceinline__ bool keep_entry(int i, int j, const int *colmap, const int *dom, int filter) {
    if (colmap[j] < 0) return false;
    if ((filter & 4) && i == j) return false;
    const int f = filter & 3;
    if (f == 0) return true;
    const bool same = dom[i] == dom[j];
    return f == 1 ? same : !same;
}

__global__ void gather_count(int n_sel, const int *__restrict__ rows, const int *__restrict__ rp,
                             const int *__restrict__ ci, const int *__restrict__ colmap, const int *__restrict__ dom,
                             int filter, int *__restrict__ counts) {
    GRID_STRIDE(r, n_sel) {
        const int i = rows ? rows[r] : (int)r;
        int c = 0;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) c += keep_entry(i, ci[k], colmap, dom, filter);
        counts[r] = c;
    }
}

__global__ void gather_fill(int n_sel, const int *__restrict__ rows, const int *__restrict__ rp,
                            const int *__restrict__ ci, const double *__restrict__ v, const int *__restrict__ colmap,
                            const int *__restrict__ dom, int filter, const int *__restrict__ out_rp,
                            int *__restrict__ out_ci, double *__restrict__ out_v, int resort) {
    GRID_STRIDE(r, n_sel) {
        const int i = rows ? rows[r] : (int)r;
        const int p0 = out_rp[r];
        int p = p0;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (keep_entry(i, j, colmap, dom, filter)) {
                out_ci[p] = colmap[j];
                if (out_v) out_v[p] = v[k];
                ++p;
            }
        }
        if (resort) {  // columns are unique: any sort equals the reference's argsort
            const int len = p - p0;
            for (int gap = len >> 1; gap > 0; gap >>= 1)
                for (int a = gap; a < len; ++a) {
                    const int cc = out_ci[p0 + a];
                    const double vv = out_v ? out_v[p0 + a] : 0.0;
                    int b = a - gap;
                    while (b >= 0 && out_ci[p0 + b] > cc) {
                        out_ci[p0 + b + gap] = out_ci[p0 + b];
                        if (out_v) out_v[p0 + b + gap] = out_v[p0 + b];
                        b -= gap;
                    }
                    out_ci[p0 + b + gap] = cc;
                    if (out_v) out_v[p0 + b + gap] = vv;
                }
        }
    }
}

// symmetrisation: for every off-diagonal (i, j) whose mirror (j, i) is not
// stored, count one extra neighbour for row j (rows are column-sorted)
__device__ __forceinline__ bool has_entry(const int *rp, const int *ci, int row, int col) {
    int lo = rp[row], hi = rp[row + 1];
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        int c = ci[mid];
        if (c == col) return true;
        if (c < col) lo = mid + 1; else hi = mid;
    }
    return false;
}

__global__ void sym_count(int n, const int *__restrict__ rp, const int *__restrict__ ci, int *counts) {
    GRID_STRIDE(i, n) {
        int own = 0;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (j == i) continue;
            ++own;
            if (!has_entry(rp, ci, j, (int)i)) atomicAdd(counts + j, 1);
        }
        atomicAdd(counts + i, own);
    }
}

__global__ void sym_fill(int n, const int *__restrict__ rp, const int *__restrict__ ci, const int *__restrict__ out_rp,
                         int *cursor, int *out_ci) {
    GRID_STRIDE(i, n) {
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (j == i) continue;
            out_ci[out_rp[i] + atomicAdd(cursor + i, 1)] = j;
            if (!has_entry(rp, ci, j, (int)i)) out_ci[out_rp[j] + atomicAdd(cursor + j, 1)] = (int)i;
        }
    }
}

// halo planning: flag every column of the selected rows that is not mapped locally
__global__ void mark_foreign_cols(int n_sel, const int *__restrict__ rows, const int *__restrict__ rp,
                                  const int *__restrict__ ci, const int *__restrict__ colmap, int *flags) {
    GRID_STRIDE(r, n_sel) {
        const int i = rows[r];
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k)
            if (colmap[ci[k]] < 0) flags[ci[k]] = 1;
    }
}

// send planning: rows owned by another rank that touch one of my exterior
// columns (extmap[j] >= 0) flag it for that rank: flags[rank * n_ext + extmap[j]] = 1
__global__ void mark_sends(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                           const int *__restrict__ owner, int doms_per_rank, int my_rank,
                           const int *__restrict__ extmap, int n_ext, int *flags) {
    GRID_STRIDE(i, n) {
        const int r = owner[i] / doms_per_rank;
        if (r == my_rank) continue;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k) {
            const int m = extmap[ci[k]];
            if (m >= 0) flags[(long long)r * n_ext + m] = 1;
        }
    }
}

// sort the column indices of every row (used after the symmetrisation appended mirrored entries)
__global__ void sort_rows(int n, const int *__restrict__ rp, int *ci) {
    GRID_STRIDE(i, n) {
        const int p0 = rp[i], len = rp[i + 1] - p0;
        for (int gap = len >> 1; gap > 0; gap >>= 1)
            for (int a = gap; a < len; ++a) {
                const int cc = ci[p0 + a];
                int b = a - gap;
                while (b >= 0 && ci[p0 + b] > cc) {
                    ci[p0 + b + gap] = ci[p0 + b];
                    b -= gap;
                }
                ci[p0 + b + gap] = cc;
            }
    }
}

// ordering.py:97-127 `_grow_regions`: greedy breadth-first growth of the domains, one after the
// other, seeded at the lowest unassigned index.  The sweep is inherently serial (every step depends
// on the queue state left by the previous one), so it runs as ONE thread; it is the rarely used
// fallback of `partition` for unstructured matrices.  owner / queued preset to -1.
__global__ void grow_regions(int n, const int *__restrict__ rp, const int *__restrict__ ci, int n_dom,
                             const int *__restrict__ sizes, int *owner, int *queue, int *queued) {
    if (blockIdx.x || threadIdx.x) return;
    int scan = 0;
    for (int d = 0; d < n_dom; ++d) {
        const int need = sizes[d];
        int count = 0, head = 0, tail = 0;
        while (count < need) {
            if (head == tail) {
                while (owner[scan] >= 0) ++scan;
                queue[tail++] = scan;
                queued[scan] = d;
            }
            const int u = queue[head++];
            if (owner[u] >= 0) continue;
            owner[u] = d;
            if (++count == need) break;
            for (int k = rp[u], ke = rp[u + 1]; k < ke; ++k) {
                const int w = ci[k];
                if (owner[w] < 0 && queued[w] != d) {
                    queued[w] = d;
                    queue[tail++] = w;
                }
            }
        }
    }
}

// precond.py:84-92 `_l1_row_shifts`: off-domain absolute row sums of the selected rows
__global__ void l1_shifts(int n_sel, const int *__restrict__ rows, const int *__restrict__ rp,
                          const int *__restrict__ ci, const double *__restrict__ v, const int *__restrict__ owner,
                          double *__restrict__ out) {
    GRID_STRIDE(r, n_sel) {
        const int i = rows[r], d = owner[i];
        double s = 0.0;
        for (int k = rp[i], ke = rp[i + 1]; k < ke; ++k)
            if (owner[ci[k]] != d) s += fabs(v[k]);
        out[r] = s;
    }
}

// precond.py:105-115 `_add_to_diagonal` (diagonal present); *missing counts rows that would need an insertion
__global__ void add_to_diag(int n, const int *__restrict__ rp, const int *__restrict__ ci, double *v,
                            const double *__restrict__ shifts, int *missing) {
    GRID_STRIDE(i, n) {
        int lo = rp[i], hi = rp[i + 1];
        bool found = false;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ci[mid] == (int)i) {
                v[mid] += shifts[i];
                found = true;
                break;
            }
            if (ci[mid] < (int)i) lo = mid + 1; else hi = mid;
        }
        if (!found && shifts[i] != 0.0) atomicAdd(missing, 1);
    }
}

// factor.py:806-822 `_drop_small_rows`: keep the diagonal and entries with |v| >= tol * ||row||_2
__device__ __forceinline__ double row_norm2(const double *v, int k0, int k1) {
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s += v[k] * v[k];
    return sqrt(s);
}

__global__ void drop_small_count(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                 const double *__restrict__ v, double tol, int *__restrict__ counts) {
    GRID_STRIDE(i, n) {
        const int k0 = rp[i], k1 = rp[i + 1];
        const double thr = tol * row_norm2(v, k0, k1);
        int c = 0;
        for (int k = k0; k < k1; ++k) c += !(fabs(v[k]) < thr && ci[k] != (int)i);
        counts[i] = c;
    }
}

__global__ void drop_small_fill(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                const double *__restrict__ v, double tol, const int *__restrict__ out_rp,
                                int *__restrict__ out_ci, double *__restrict__ out_v) {
    GRID_STRIDE(i, n) {
        const int k0 = rp[i], k1 = rp[i + 1];
        const double thr = tol * row_norm2(v, k0, k1);
        int p = out_rp[i];
        for (int k = k0; k < k1; ++k)
            if (!(fabs(v[k]) < thr && ci[k] != (int)i)) {
                out_ci[p] = ci[k];
                out_v[p++] = v[k];
            }
    }
}

__global__ void diff_kernel(int n, const int *__restrict__ rp, int *__restrict__ out) {
    GRID_STRIDE(i, n) out[i] = rp[i + 1] - rp[i];
}

__global__ void narrow_i64(long long n, const long long *__restrict__ in, int *__restrict__ out) {
    GRID_STRIDE(i, n) out[i] = (int)in[i];
}

__global__ void widen_i32(long long n, const int *__restrict__ in, long long *__restrict__ out) {
    GRID_STRIDE(i, n) out[i] = in[i];
}

// structured box partition (ordering.py:171-187): owner = sum_ax chunk_ax * dstride_ax,
// chunk by np.array_split bounds: the first (d % f) chunks have d/f + 1 cells
__global__ void box_owner(int n, int nd, int d0, int d1, int d2, int f0, int f1, int f2, int *__restrict__ owner) {
    GRID_STRIDE(i, n) {
        const int dims[3] = {d0, d1, d2}, fac[3] = {f0, f1, f2};
        long long rem = i;
        int own = 0, dstride = 1;
        for (int a = 0; a < nd; ++a) {
            const int c = (int)(rem % dims[a]);
            rem /= dims[a];
            const int base = dims[a] / fac[a], extra = dims[a] % fac[a];
            const int cut = extra * (base + 1);
            const int chunk = c < cut ? c / (base + 1) : extra + (base ? (c - cut) / base : 0);
            own += chunk * dstride;
            dstride *= fac[a];
        }
        owner[i] = own;
    }
}

}  // namespace ddilu

using namespace ddilu;
#define ST(s) ((cudaStream_t)(s))
#define G1(n) stream_grid((n), 256), 256, 0

extern "C" int ddilu_mark_exterior(int n, const int *rp, const int *ci, const int *owner, int *exterior, void *stream) {
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(exterior, 0, sizeof(int) * (size_t)n, ST(stream)));
    mark_exterior<<<G1(n), ST(stream)>>>(n, rp, ci, owner, exterior);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_layout_keys(int n, const int *owner, const int *exterior, int p, int *keys, int *vals,
                                 void *stream) {
    if (n <= 0) return DDILU_OK;
    layout_keys<<<G1(n), ST(stream)>>>(n, owner, exterior, p, keys, vals);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_lower_bounds(const int *sorted, int n, int nkeys, int *out, void *stream) {
    lower_bounds<<<G1(nkeys + 1), ST(stream)>>>(sorted, n, nkeys, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_build_map(int n_nodes, const int *nodes, int offset, int *map, void *stream) {
    if (n_nodes <= 0) return DDILU_OK;
    build_map<<<G1(n_nodes), ST(stream)>>>(n_nodes, nodes, offset, map);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_gather_rows_count(int n_sel, const int *rows, const int *rp, const int *ci, const int *colmap,
                                       const int *dom, int filter, int *counts, void *stream) {
    if (n_sel <= 0) return DDILU_OK;
    if ((filter & 3) && !dom) return DDILU_ERR_ARG;
    gather_count<<<G1(n_sel), ST(stream)>>>(n_sel, rows, rp, ci, colmap, dom, filter, counts);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_gather_rows_fill(int n_sel, const int *rows, const int *rp, const int *ci, const double *v,
                                      const int *colmap, const int *dom, int filter, const int *out_rp, int *out_ci,
                                      double *out_v, int resort, void *stream) {
    if (n_sel <= 0) return DDILU_OK;
    if ((filter & 3) && !dom) return DDILU_ERR_ARG;
    gather_fill<<<G1(n_sel), ST(stream)>>>(n_sel, rows, rp, ci, v, colmap, dom, filter, out_rp, out_ci, out_v, resort);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sym_adj_count(int n, const int *rp, const int *ci, int *counts, void *stream) {
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)n, ST(stream)));
    sym_count<<<G1(n), ST(stream)>>>(n, rp, ci, counts);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sym_adj_fill(int n, const int *rp, const int *ci, const int *out_rp, int *cursor, int *out_ci,
                                  void *stream) {
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(cursor, 0, sizeof(int) * (size_t)n, ST(stream)));
    sym_fill<<<G1(n), ST(stream)>>>(n, rp, ci, out_rp, cursor, out_ci);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_mark_foreign_cols(int n_sel, const int *rows, const int *rp, const int *ci, const int *colmap,
                                       int *flags, void *stream) {
    if (n_sel <= 0) return DDILU_OK;
    mark_foreign_cols<<<G1(n_sel), ST(stream)>>>(n_sel, rows, rp, ci, colmap, flags);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_mark_sends(int n, const int *rp, const int *ci, const int *owner, int doms_per_rank, int my_rank,
                                const int *extmap, int n_ext, int *flags, void *stream) {
    if (n <= 0 || n_ext <= 0) return DDILU_OK;
    mark_sends<<<G1(n), ST(stream)>>>(n, rp, ci, owner, doms_per_rank, my_rank, extmap, n_ext, flags);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sort_rows_i32(int n, const int *rp, int *ci, void *stream) {
    if (n <= 0) return DDILU_OK;
    sort_rows<<<G1(n), ST(stream)>>>(n, rp, ci);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_grow_regions(int n, const int *adj_rp, const int *adj_ci, int n_dom, const int *sizes,
                                  int *owner, int *work, void *stream) {
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(owner, 0xFF, sizeof(int) * (size_t)n, ST(stream)));
    DDILU_CHECK(cudaMemsetAsync(work + n, 0xFF, sizeof(int) * (size_t)n, ST(stream)));
    grow_regions<<<1, 1, 0, ST(stream)>>>(n, adj_rp, adj_ci, n_dom, sizes, owner, work, work + n);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_l1_row_shifts(int n_sel, const int *rows, const int *rp, const int *ci, const double *v,
                                   const int *owner, double *out, void *stream) {
    if (n_sel <= 0) return DDILU_OK;
    l1_shifts<<<G1(n_sel), ST(stream)>>>(n_sel, rows, rp, ci, v, owner, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_add_to_diagonal(int n, const int *rp, const int *ci, double *v, const double *shifts,
                                     int *missing, void *stream) {
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(missing, 0, sizeof(int), ST(stream)));
    add_to_diag<<<G1(n), ST(stream)>>>(n, rp, ci, v, shifts, missing);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_drop_small_count(int n, const int *rp, const int *ci, const double *v, double tol, int *counts,
                                      void *stream) {
    if (n <= 0) return DDILU_OK;
    drop_small_count<<<G1(n), ST(stream)>>>(n, rp, ci, v, tol, counts);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_drop_small_fill(int n, const int *rp, const int *ci, const double *v, double tol,
                                     const int *out_rp, int *out_ci, double *out_v, void *stream) {
    if (n <= 0) return DDILU_OK;
    drop_small_fill<<<G1(n), ST(stream)>>>(n, rp, ci, v, tol, out_rp, out_ci, out_v);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_row_lengths(int n, const int *rp, int *out, void *stream) {
    if (n <= 0) return DDILU_OK;
    diff_kernel<<<G1(n), ST(stream)>>>(n, rp, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_narrow_i64(long long n, const long long *in, int *out, void *stream) {
    if (n <= 0) return DDILU_OK;
    narrow_i64<<<G1(n), ST(stream)>>>(n, in, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_widen_i32(long long n, const int *in, long long *out, void *stream) {
    if (n <= 0) return DDILU_OK;
    widen_i32<<<G1(n), ST(stream)>>>(n, in, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_box_owner(int n, int nd, const int *dims, const int *factors, int *owner, void *stream) {
    if (n <= 0) return DDILU_OK;
    if (nd < 1 || nd > 3) return DDILU_ERR_ARG;
    int d[3] = {1, 1, 1}, f[3] = {1, 1, 1};
    for (int a = 0; a < nd; ++a) {
        d[a] = dims[a];
        f[a] = factors[a];
    }
    box_owner<<<G1(n), ST(stream)>>>(n, nd, d[0], d[1], d[2], f[0], f[1], f[2], owner);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
