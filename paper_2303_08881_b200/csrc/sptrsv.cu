// Sparse triangular solves and their level schedules.
//
// Replaces sparse.py:228-272 (`_lower_solve`, `_upper_solve`).  The reference
// sweeps rows serially; here ONE persistent launch runs the whole solve:
//
//   * rows are visited in level order (schedule built once per factor; every
//     level is padded to a multiple of 32 slots so a warp never holds two rows
//     that depend on each other),
//   * one thread owns one row and accumulates its entries strictly left to
//     right (bit-identical to the reference; -fmad=false),
//   * there is no barrier between levels: the solution vector itself is the
//     ready flag.  x is preset to an all-ones NaN pattern; a consumer polls
//     x[j] in L2 until the pattern is gone (8-byte stores are single-copy
//     atomic), so a dependency hop costs one L2 store + one L2 load instead of
//     a grid-wide barrier or a kernel launch per level,
//   * CTAs take chunks of the schedule round-robin; the launch is cooperative
//     so all CTAs are co-resident and every dependency (always in an earlier
//     chunk) is owned by a running CTA: no deadlock.
//
// Algorithmic bytes: 12*nnz + 4*(n+1) + 8n (b) + 8n (x).
// Critical path: n_levels dependent L2 hops; both bounds are reported by bench.py.
#include <string.h>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int TRSV_THREADS = 256;
constexpr int TRSV_UNROLL = 4;

struct TrsvTuning {
    int blocks_per_sm = 4;
    unsigned sleep_ns = 0;
};
static TrsvTuning g_trsv;

template <bool UPPER>
__global__ void __launch_bounds__(TRSV_THREADS) sptrsv_syncfree(int n_slots, const int *__restrict__ order,
                                                                const int *__restrict__ rp, const int *__restrict__ ci,
                                                                const double *__restrict__ val,
                                                                const double *__restrict__ b, double *x, int unit_diag,
                                                                int *err, unsigned sleep_ns) {
    for (long long base = (long long)blockIdx.x * TRSV_THREADS; base < n_slots;
         base += (long long)gridDim.x * TRSV_THREADS) {
        const long long slot = base + threadIdx.x;
        if (slot >= n_slots) continue;
        const int row = order[slot];
        if (row < 0) continue;
        int k = rp[row];
        const int ke = rp[row + 1];
        double s = b[row], diag = 1.0;
        bool seen = false;
        while (k < ke) {
            int j[TRSV_UNROLL];
            double a[TRSV_UNROLL], xv[TRSV_UNROLL];
            bool dep[TRSV_UNROLL];
#pragma unroll
            for (int u = 0; u < TRSV_UNROLL; ++u) {
                const bool in = k + u < ke;
                j[u] = in ? ci[k + u] : row;
                a[u] = in ? val[k + u] : 0.0;
                dep[u] = in && (UPPER ? j[u] > row : j[u] < row);
                if (in && j[u] == row) {
                    diag = a[u];
                    seen = true;
                }
            }
            // all polls of this group are in flight together
#pragma unroll
            for (int u = 0; u < TRSV_UNROLL; ++u) xv[u] = dep[u] ? ld_l2(x + j[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < TRSV_UNROLL; ++u) {
                if (dep[u]) {
                    while (is_sentinel(xv[u])) {
                        if (sleep_ns) __nanosleep(sleep_ns);
                        xv[u] = ld_l2(x + j[u]);
                    }
                    s -= a[u] * xv[u];
                }
            }
            k += TRSV_UNROLL;
        }
        double res = s;
        if (!unit_diag) {
            if (!seen || fabs(diag) < 1e-300) {
                atomicMin(err, row);
                res = __longlong_as_double(0x7FF8000000000000LL);
            } else {
                res = s / diag;
            }
        }
        st_l2(x + row, scrub_sentinel(res));
    }
}

// Topological level of every row (lev[i] = 1 + max lev[j] over dependencies),
// rows visited in index order (reverse for U).  lev is preset to -1 and is its
// own ready flag.  Dependencies may sit in the same warp here, so the loop
// never blocks: a lane that cannot advance simply retries on the next trip.
template <bool UPPER>
__global__ void __launch_bounds__(TRSV_THREADS) levels_syncfree(int n, const int *__restrict__ rp,
                                                                const int *__restrict__ ci, int *lev, int *max_lev) {
    for (long long base = (long long)blockIdx.x * TRSV_THREADS; base < n; base += (long long)gridDim.x * TRSV_THREADS) {
        const long long idx = base + threadIdx.x;
        const bool active = idx < n;
        const int row = active ? (UPPER ? n - 1 - (int)idx : (int)idx) : 0;
        int k = active ? rp[row] : 0;
        const int ke = active ? rp[row + 1] : 0;
        int l = 0;
        bool done = !active;
        while (!done) {
            while (k < ke) {
                const int j = ci[k];
                if (UPPER ? j > row : j < row) {
                    const int lj = ld_l2(lev + j);
                    if (lj < 0) break;
                    l = max(l, lj + 1);
                }
                ++k;
            }
            if (k == ke) {
                st_l2(lev + row, l);
                done = true;
            }
        }
        const int m = __reduce_max_sync(0xffffffffu, active ? l : 0);
        if ((threadIdx.x & 31) == 0) atomicMax(max_lev, m);
    }
}

__global__ void sched_init(int n, const int *__restrict__ lev, int upper, int *__restrict__ keys,
                           int *__restrict__ vals) {
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        int row = upper ? n - 1 - (int)q : (int)q;
        keys[q] = lev[row];
        vals[q] = row;
    }
}

__global__ void sched_bounds(int n, const int *__restrict__ keys, int n_levels, int *__restrict__ level_ptr) {
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        if (q == 0 || keys[q] != keys[q - 1]) level_ptr[keys[q]] = (int)q;
        if (q == n - 1) level_ptr[n_levels] = n;
    }
}

// single CTA: padded slot offsets slot_ptr[l] = sum_{l'<l} roundup32(count[l'])
__global__ void sched_slots(int n_levels, const int *__restrict__ level_ptr, int *__restrict__ slot_ptr) {
    __shared__ int carry_s;
    __shared__ int wtot[32];
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < n_levels; base += blockDim.x) {
        int l = base + threadIdx.x;
        int v = l < n_levels ? ((level_ptr[l + 1] - level_ptr[l] + 31) & ~31) : 0;
        int inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        int wbase = 0, all = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) wbase += wtot[w];
            all += wtot[w];
        }
        int carry = carry_s;
        if (l < n_levels) slot_ptr[l] = carry + wbase + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + all;
        __syncthreads();
    }
    if (threadIdx.x == 0) slot_ptr[n_levels] = carry_s;
}

__global__ void sched_place(int n, const int *__restrict__ keys, const int *__restrict__ rows,
                            const int *__restrict__ level_ptr, const int *__restrict__ slot_ptr,
                            int *__restrict__ order) {
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        int l = keys[q];
        order[slot_ptr[l] + ((int)q - level_ptr[l])] = rows[q];
    }
}

template <typename K>
static int coop_grid(K kernel, int threads, int blocks_per_sm_cap, long long work_items) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0);
    if (occ < 1) occ = 1;
    if (blocks_per_sm_cap > 0 && occ > blocks_per_sm_cap) occ = blocks_per_sm_cap;
    long long grid = (long long)occ * device_info().sm_count;
    long long need = (work_items + threads - 1) / threads;
    if (need < 1) need = 1;
    return (int)(grid < need ? grid : need);
}

}  // namespace ddilu

using namespace ddilu;

extern "C" int ddilu_set_tuning(const char *key, int value) {
    if (!key) return DDILU_ERR_ARG;
    if (!strcmp(key, "trsv_blocks_per_sm")) g_trsv.blocks_per_sm = value;
    else if (!strcmp(key, "trsv_sleep_ns")) g_trsv.sleep_ns = (unsigned)value;
    else return DDILU_ERR_ARG;
    return DDILU_OK;
}

extern "C" int ddilu_levels(int n, const int *row_ptr, const int *col_idx, int upper, int *lev, int *max_lev,
                            void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    DDILU_CHECK(cudaMemsetAsync(max_lev, 0, sizeof(int), st));
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(lev, 0xFF, sizeof(int) * (size_t)n, st));
    void *args[] = {&n, &row_ptr, &col_idx, &lev, &max_lev};
    if (upper) {
        int grid = coop_grid(levels_syncfree<true>, TRSV_THREADS, 0, n);
        DDILU_CHECK(cudaLaunchCooperativeKernel((void *)levels_syncfree<true>, grid, TRSV_THREADS, args, 0, st));
    } else {
        int grid = coop_grid(levels_syncfree<false>, TRSV_THREADS, 0, n);
        DDILU_CHECK(cudaLaunchCooperativeKernel((void *)levels_syncfree<false>, grid, TRSV_THREADS, args, 0, st));
    }
    return DDILU_OK;
}

extern "C" int ddilu_schedule_build(int n, const int *lev, int n_levels, int upper, int *keys, int *rows,
                                    int *keys_alt, int *rows_alt, int *sort_tmp, int *level_ptr, int *slot_ptr,
                                    int *order, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0 || n_levels <= 0) return DDILU_OK;
    int bits = 1;
    while ((1LL << bits) < n_levels) ++bits;
    int grid = stream_grid(n, 256);
    sched_init<<<grid, 256, 0, st>>>(n, lev, upper, keys, rows);
    int rc = ddilu_sort_pairs_i32(keys, rows, keys_alt, rows_alt, n, bits, sort_tmp, stream);
    if (rc) return rc;
    sched_bounds<<<grid, 256, 0, st>>>(n, keys, n_levels, level_ptr);
    sched_slots<<<1, 1024, 0, st>>>(n_levels, level_ptr, slot_ptr);
    DDILU_CHECK(cudaMemsetAsync(order, 0xFF, sizeof(int) * ((size_t)n + 32 * (size_t)n_levels), st));
    sched_place<<<grid, 256, 0, st>>>(n, keys, rows, level_ptr, slot_ptr, order);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sptrsv(int n, int n_slots, const int *order, const int *row_ptr, const int *col_idx,
                            const double *values, const double *b, double *x, int upper, int unit_diag, int *err,
                            void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (x == b) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    unsigned sleep_ns = g_trsv.sleep_ns;
    void *args[] = {&n_slots, &order, &row_ptr, &col_idx, &values, &b, &x, &unit_diag, &err, &sleep_ns};
    if (upper) {
        int grid = coop_grid(sptrsv_syncfree<true>, TRSV_THREADS, g_trsv.blocks_per_sm, n_slots);
        DDILU_CHECK(cudaLaunchCooperativeKernel((void *)sptrsv_syncfree<true>, grid, TRSV_THREADS, args, 0, st));
    } else {
        int grid = coop_grid(sptrsv_syncfree<false>, TRSV_THREADS, g_trsv.blocks_per_sm, n_slots);
        DDILU_CHECK(cudaLaunchCooperativeKernel((void *)sptrsv_syncfree<false>, grid, TRSV_THREADS, args, 0, st));
    }
    return DDILU_OK;
}
