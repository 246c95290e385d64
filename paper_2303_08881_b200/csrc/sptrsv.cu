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
    int blocks_per_sm = 3;
    int wr_blocks_per_sm = 0;  // warp-per-row kernel: CTAs per SM (0: as many as fit; measured best, scripts/probe_warprow.py)
    unsigned sleep_ns = 0;
    int pipe = 0;            // 1: software-pipelined SELL kernel, 0: plain SELL kernel
    int pipe_warps_per_sm = 8;
    int win_threads = 0;   // CTA size of the window sweep (0: BL_THREADS)
    int stage_mask = -1;     // -1: by level width (measured: narrow levels -> 3, wide levels -> 4)
                             // bit0: far stage (sleep-poll 3 levels back), bit1: mid stage (spin 2 levels
                             // back), bit2: near stage (spin on the group's own latest dependency)
    int far_sleep_ns = 400;
    int chunk = 0;           // dependencies polled per round by the SELL kernel; 0: by average row width
    int depth = 24;          // resident warps ~ depth x (groups per level): enough lookahead to hide the
                             // startup loads of a group, few enough pollers not to slow the producers
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

// Warp-per-row variant for LONG rows (ILUT / ILU(k) / 27-point factors: 10-20 dependencies per row, factors that
// neither tile nor fit a block sweep).  The thread-per-row kernels above poll a row's dependencies in rounds of
// 4-16 and add the products one after the other in ONE thread: 3.5 us per level on the 27-point interior factors
// (3 % of the HBM roofline).  Here a warp owns a row: the lanes fetch the row's entries with one coalesced load,
// poll all dependencies at once (x is its own ready flag, as above), round their products, and lane 0 adds them
// in storage order (sparse.py:228-272: same operations, same order -> same bits).  Warps take the schedule slots
// round-robin; the launch is cooperative, so the earliest unfinished row always belongs to a resident warp.
constexpr int WR_WARPS = 8;
template <bool UPPER>
__global__ void __launch_bounds__(32 * WR_WARPS) sptrsv_warprow(int n_slots, const int *__restrict__ order,
                                                                const int *__restrict__ rp, const int *__restrict__ ci,
                                                                const double *__restrict__ val,
                                                                const double *__restrict__ b, double *x, int unit_diag,
                                                                int *err, unsigned sleep_ns) {
    __shared__ double prod[WR_WARPS][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long n_warps = (long long)gridDim.x * WR_WARPS;
    long long slot = (long long)blockIdx.x * WR_WARPS + wib;
    // software pipeline: row id, row bounds and right-hand side of the NEXT slot are fetched while this one waits
    int row = slot < n_slots ? order[slot] : -1;
    int k0 = 0, k1 = 0;
    double rhs = 0.0;
    if (row >= 0) {
        k0 = rp[row];
        k1 = rp[row + 1];
        rhs = b[row];
    }
    for (; slot < n_slots; slot += n_warps) {
        const long long nslot = slot + n_warps;
        const int nrow = nslot < n_slots ? order[nslot] : -1;
        int nk0 = 0, nk1 = 0;
        double nrhs = 0.0;
        if (nrow >= 0) {
            nk0 = rp[nrow];
            nk1 = rp[nrow + 1];
            nrhs = b[nrow];
        }
        if (row >= 0) {
            double s = rhs, diag = 1.0;
            bool seen = false;
            for (int base = k0; base < k1; base += 32) {
                const int k = base + lane;
                const bool in = k < k1;
                const int col = in ? ci[k] : row;
                const double a = in ? val[k] : 0.0;
                const bool dep = in && (UPPER ? col > row : col < row);
                const unsigned dmask = __ballot_sync(0xffffffffu, in && col == row);
                if (dmask) {
                    diag = __shfl_sync(0xffffffffu, a, __ffs(dmask) - 1);
                    seen = true;
                }
                double v = 0.0;
                if (dep) {
                    v = ld_l2(x + col);
                    while (is_sentinel(v)) {
                        if (sleep_ns) __nanosleep(sleep_ns);
                        v = ld_l2(x + col);
                    }
                }
                prod[wib][lane] = dep ? a * v : 0.0;          // every product rounded (-fmad=false)
                __syncwarp();
                if (lane == 0) {
                    const int cnt = min(32, k1 - base);
                    for (int q = 0; q < cnt; ++q) s -= prod[wib][q];   // storage order; non-dependencies subtract 0.0
                }
                __syncwarp();
            }
            if (lane == 0) {
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
        row = nrow;
        k0 = nk0;
        k1 = nk1;
        rhs = nrhs;
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


// ---------------------------------------------------------------------------
// Schedule-ordered sliced-ELL (SELL-32) form of a triangular factor.
//
// A group = 32 consecutive schedule slots (= one warp, all in one level).  The
// dependencies of its rows are stored column-major inside the group
// (entry k of lane l at goff[g] + 32*k + l), padded with col = -1 to the
// longest row of the group; the diagonal (U, or a non-unit L) is kept per slot.
// Every load of the solve is then a coalesced 128/256-byte access and the chain
// of dependent loads is descriptor -> (cols, vals, row id) -> x.
__global__ void sched_positions(int n_slots, const int *__restrict__ order, int *__restrict__ pos) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += (long long)gridDim.x * blockDim.x)
        if (order[s] >= 0) pos[order[s]] = (int)s;
}

// out[g] = gwait of the group that produces gwait[g]: an indicator one level further back
__global__ void compose_wait(int n_groups, const int *__restrict__ gwait, const int *__restrict__ pos,
                             const int *__restrict__ prev, int *__restrict__ out) {
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n_groups; g += (long long)gridDim.x * blockDim.x) {
        const int c = prev[g];
        out[g] = c >= 0 ? gwait[pos[c] >> 5] : -1;
    }
}

// gwait[g] = the dependency of group g that sits LATEST in the schedule (-1 if the
// group has none): the warp spins on that single address before it checks the rest,
// so a waiting warp costs one 32-byte L2 sector per poll instead of ~30.
__global__ void sell_width(int n_groups, const int *__restrict__ order, const int *__restrict__ rp,
                           const int *__restrict__ ci, const double *__restrict__ val, int upper, int unit_diag,
                           int *__restrict__ gw32, double *__restrict__ sdiag, int *bad_row,
                           const int *__restrict__ pos, int *__restrict__ gwait) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long g = warp; g < n_groups; g += nw) {
        const int row = order[g * 32 + lane];
        int deps = 0;
        double d = 1.0;
        bool seen = false;
        long long last = -1;  // (schedule position << 32) | column of the latest dependency
        if (row >= 0) {
            for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
                const int j = ci[k];
                if (upper ? j > row : j < row) {
                    ++deps;
                    if (pos) {
                        const long long key = ((long long)pos[j] << 32) | (unsigned)j;
                        last = key > last ? key : last;
                    }
                } else if (j == row) {
                    d = val[k];
                    seen = true;
                }
            }
            if (!unit_diag && (!seen || fabs(d) < 1e-300)) atomicMin(bad_row, row);
        }
        if (sdiag) sdiag[g * 32 + lane] = unit_diag ? 1.0 : d;
        const int w = __reduce_max_sync(0xffffffffu, deps);
        if (lane == 0) gw32[g] = w * 32;
        if (gwait) {
            for (int o = 16; o > 0; o >>= 1) {
                const long long other = __shfl_xor_sync(0xffffffffu, last, o);
                last = other > last ? other : last;
            }
            if (lane == 0) gwait[g] = last < 0 ? -1 : (int)(last & 0xffffffffLL);
        }
    }
}

__global__ void sell_fill(int n_groups, const int *__restrict__ order, const int *__restrict__ rp,
                          const int *__restrict__ ci, const double *__restrict__ val, int upper,
                          const int *__restrict__ goff, int uw, int *__restrict__ scol, double *__restrict__ sval) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long g = warp; g < n_groups; g += nw) {
        const int row = order[g * 32 + lane];
        const long long off = goff ? goff[g] : g * 32LL * uw;
        const int w = goff ? (goff[g + 1] - (int)off) >> 5 : uw;
        int k2 = 0;
        if (row >= 0) {
            for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
                const int j = ci[k];
                if (upper ? j > row : j < row) {
                    scol[off + 32 * k2 + lane] = j;
                    sval[off + 32 * k2 + lane] = val[k];
                    ++k2;
                }
            }
        }
        for (; k2 < w; ++k2) {
            scol[off + 32 * k2 + lane] = -1;
            sval[off + 32 * k2 + lane] = 0.0;
        }
    }
}

constexpr int SELL_THREADS = 256;
constexpr int SELL_CHUNK = 4;

// Wait until every dependency of the chunk is available.  The first round has
// all polls in flight together; a dependency that is still missing is then
// re-polled on its own.  (Measured on B200: re-issuing ALL pending polls every
// round is slower -- more simultaneous polls of the line the producer is about
// to store to: 0.81 vs 0.48 us per level on a one-warp-per-level chain.)
template <int C>
__device__ __forceinline__ void poll_chunk(const double *x, const int (&c)[C], double (&xv)[C]) {
#pragma unroll
    for (int u = 0; u < C; ++u) xv[u] = c[u] >= 0 ? ld_l2(x + c[u]) : 0.0;
    bool pending;
    do {
        pending = false;
#pragma unroll
        for (int u = 0; u < C; ++u)
            if (is_sentinel(xv[u])) {
                xv[u] = ld_l2(x + c[u]);
                pending |= is_sentinel(xv[u]);
            }
    } while (pending);
}

// CHUNK = dependencies of a row polled together: 4 for stencil-length rows, 12 for long rows (27-point /
// ILUT / ILU(k) factors: a 19-entry row is 2 poll rounds instead of 5)
template <bool HAS_DIAG, int CHUNK>
__global__ void __launch_bounds__(SELL_THREADS) sptrsv_sell(int n_groups, const int *__restrict__ order,
                                                            const int *__restrict__ goff, int uw,
                                                            const int *__restrict__ scol,
                                                            const double *__restrict__ sval,
                                                            const double *__restrict__ sdiag,
                                                            const int *__restrict__ gwait,
                                                            const int *__restrict__ gfar1,
                                                            const int *__restrict__ gfar2, unsigned far_sleep_ns,
                                                            const double *__restrict__ b, double *x) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long g = warp; g < n_groups; g += nw) {
        // uniform-width layout (goff == nullptr): no descriptor load on the dependency chain
        const long long off = goff ? goff[g] : g * 32LL * uw;
        const int w = goff ? (goff[g + 1] - (int)off) >> 5 : uw;
        const int row = order[g * 32 + lane];
        const int wait_col = gwait ? gwait[g] : -1;
        const int far1 = gfar1 ? gfar1[g] : -1, far2 = gfar2 ? gfar2[g] : -1;
        double s = row >= 0 ? b[row] : 0.0;
        const double d = HAS_DIAG ? sdiag[g * 32 + lane] : 1.0;
        // staged waiting: every stage polls ONE address (one 32-byte sector for the whole warp)
        //   far  (an indicator 3 levels back not yet written): sleep between polls, latency is irrelevant here
        //   mid  (2 levels back): tight single-sector spin
        //   near (optional, the group's own latest dependency): tight single-sector spin
        // afterwards the real dependencies are polled directly.
        if (far2 >= 0)
            while (is_sentinel(ld_l2(x + far2))) __nanosleep(far_sleep_ns);
        if (far1 >= 0)
            while (is_sentinel(ld_l2(x + far1))) {
            }
        if (wait_col >= 0)
            while (is_sentinel(ld_l2(x + wait_col))) {
            }
        for (int k0 = 0; k0 < w; k0 += CHUNK) {
            int c[CHUNK];
            double a[CHUNK], xv[CHUNK];
#pragma unroll
            for (int u = 0; u < CHUNK; ++u) {
                const bool in = k0 + u < w;
                c[u] = in ? scol[off + 32 * (k0 + u) + lane] : -1;
                a[u] = in ? sval[off + 32 * (k0 + u) + lane] : 0.0;
            }
            poll_chunk(x, c, xv);
#pragma unroll
            for (int u = 0; u < CHUNK; ++u)
                if (c[u] >= 0) s -= a[u] * xv[u];
        }
        if (row >= 0) st_l2(x + row, scrub_sentinel(HAS_DIAG ? s / d : s));
    }
}

// Software-pipelined variant: while a warp polls the dependencies of its
// current group it already holds the next group's row ids, first SELL_CHUNK
// entries, right-hand sides and pivots in registers and the descriptor of the
// group after that.  The startup chain (descriptor -> entries -> x) is thus off
// the critical path and a SMALL number of resident warps is enough, which keeps
// the L2 polling traffic (the thing that inflates every dependency hop) low.
#ifdef DDILU_EXPERIMENTS   // measured-slower alternatives: pipelined SELL solve, CTA-per-block sweeps
struct SellRow {
    int row, w;
    long long off;
    int c[SELL_CHUNK];
    double a[SELL_CHUNK];
    double rhs, piv;
};

template <bool HAS_DIAG>
__device__ __forceinline__ void sell_load(SellRow &r, long long g, int lane, const int *__restrict__ order,
                                          const int *__restrict__ scol, const double *__restrict__ sval,
                                          const double *__restrict__ sdiag, const double *__restrict__ b) {
    r.row = order[g * 32 + lane];
    r.rhs = r.row >= 0 ? b[r.row] : 0.0;
    r.piv = HAS_DIAG ? sdiag[g * 32 + lane] : 1.0;
#pragma unroll
    for (int u = 0; u < SELL_CHUNK; ++u) {
        const bool in = u < r.w;
        r.c[u] = in ? scol[r.off + 32 * u + lane] : -1;
        r.a[u] = in ? sval[r.off + 32 * u + lane] : 0.0;
    }
}

template <bool HAS_DIAG>
__global__ void __launch_bounds__(128) sptrsv_sell_pipe(int n_groups, const int *__restrict__ order,
                                                        const int *__restrict__ goff, int uw,
                                                        const int *__restrict__ scol,
                                                        const double *__restrict__ sval,
                                                        const double *__restrict__ sdiag,
                                                        const double *__restrict__ b, double *x) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    long long g = warp;
    if (g >= n_groups) return;
    SellRow cur, nxt;
    cur.off = goff ? goff[g] : g * 32LL * uw;
    cur.w = goff ? (goff[g + 1] - (int)cur.off) >> 5 : uw;
    sell_load<HAS_DIAG>(cur, g, lane, order, scol, sval, sdiag, b);
    long long gn = g + nw;
    bool have_n = gn < n_groups;
    nxt.off = have_n ? (goff ? goff[gn] : gn * 32LL * uw) : 0;
    nxt.w = have_n ? (goff ? (goff[gn + 1] - (int)nxt.off) >> 5 : uw) : 0;
    for (;;) {
        // prefetch: next group's rows, descriptor of the one after
        long long gnn = gn + nw;
        const bool have_nn = have_n && gnn < n_groups;
        long long off_nn = 0;
        int w_nn = 0;
        if (have_n) sell_load<HAS_DIAG>(nxt, gn, lane, order, scol, sval, sdiag, b);
        if (have_nn) {
            off_nn = goff ? goff[gnn] : gnn * 32LL * uw;
            w_nn = goff ? (goff[gnn + 1] - (int)off_nn) >> 5 : uw;
        }
        // ---- current group: poll all pending dependencies of a chunk together
        double s = cur.rhs;
        {
            double xv[SELL_CHUNK];
            poll_chunk(x, cur.c, xv);
#pragma unroll
            for (int u = 0; u < SELL_CHUNK; ++u)
                if (cur.c[u] >= 0) s -= cur.a[u] * xv[u];
        }
        for (int k0 = SELL_CHUNK; k0 < cur.w; k0 += SELL_CHUNK) {  // long rows: remaining chunks on the fly
            int c[SELL_CHUNK];
            double a[SELL_CHUNK], xv[SELL_CHUNK];
#pragma unroll
            for (int u = 0; u < SELL_CHUNK; ++u) {
                const bool in = k0 + u < cur.w;
                c[u] = in ? scol[cur.off + 32 * (k0 + u) + lane] : -1;
                a[u] = in ? sval[cur.off + 32 * (k0 + u) + lane] : 0.0;
            }
            poll_chunk(x, c, xv);
#pragma unroll
            for (int u = 0; u < SELL_CHUNK; ++u)
                if (c[u] >= 0) s -= a[u] * xv[u];
        }
        if (cur.row >= 0) st_l2(x + cur.row, scrub_sentinel(HAS_DIAG ? s / cur.piv : s));
        if (!have_n) break;
        cur = nxt;
        gn = gnn;
        have_n = have_nn;
        nxt.off = off_nn;
        nxt.w = w_nn;
    }
}


// ---------------------------------------------------------------------------
// Block-local solve for SMALL, DEEP factors that are block diagonal (the
// interface factors L_S / U_S of the two-level preconditioners: one independent
// block per subdomain, ~100-400 rows per level).  One CTA owns one block and
// walks its levels with __syncthreads() in between: a level costs one L2 load of
// the dependencies + a CTA barrier (deterministic, no polling, no cooperative
// launch); the row data of the next level is prefetched into registers before
// the current level is finished.  Row sums in storage order: bit-identical.
constexpr int BL_THREADS = 1024;
constexpr int BL_PRE = 6;  // entries of a row kept in registers

__global__ void blocklocal_table(int n, int n_blocks, const int *__restrict__ seg_ptr, int n_levels,
                                 const int *__restrict__ lev, const int *__restrict__ level_rows,
                                 int *start, int *cnt) {
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int row = level_rows[q];
        int lo = 0, hi = n_blocks;  // largest d with seg_ptr[d] <= row
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (seg_ptr[mid] <= row) lo = mid; else hi = mid;
        }
        const long long slot = (long long)lo * n_levels + lev[row];
        atomicMin(start + slot, (int)q);
        atomicAdd(cnt + slot, 1);
    }
}

struct BlRow {
    int row, k, ke;
    int c[BL_PRE];
    double a[BL_PRE];
    double rhs;
};

__device__ __forceinline__ void bl_load(BlRow &r, bool active, int q, const int *__restrict__ level_rows,
                                        const int *__restrict__ rp, const int *__restrict__ ci,
                                        const double *__restrict__ val, const double *__restrict__ b) {
    r.row = -1;
    r.k = r.ke = 0;
    r.rhs = 0.0;
    if (active) {
        r.row = level_rows[q];
        r.k = rp[r.row];
        r.ke = rp[r.row + 1];
        r.rhs = b[r.row];
    }
#pragma unroll
    for (int u = 0; u < BL_PRE; ++u) {
        const bool in = r.k + u < r.ke;
        r.c[u] = in ? ci[r.k + u] : -1;
        r.a[u] = in ? val[r.k + u] : 0.0;
    }
}

template <bool UPPER>
__device__ __forceinline__ void bl_finish(const BlRow &r, const int *__restrict__ ci, const double *__restrict__ val,
                                          double *x, int unit_diag, int *err) {
    if (r.row < 0) return;
    double s = r.rhs, diag = 1.0;
    bool seen = false;
#pragma unroll
    for (int u = 0; u < BL_PRE; ++u) {
        const int j = r.c[u];
        if (j < 0) continue;
        if (UPPER ? j > r.row : j < r.row) s -= r.a[u] * x[j];
        else if (j == r.row) {
            diag = r.a[u];
            seen = true;
        }
    }
    for (int k = r.k + BL_PRE; k < r.ke; ++k) {  // long rows
        const int j = ci[k];
        if (UPPER ? j > r.row : j < r.row) s -= val[k] * x[j];
        else if (j == r.row) {
            diag = val[k];
            seen = true;
        }
    }
    if (!unit_diag) {
        if (!seen || fabs(diag) < 1e-300) {
            atomicMin(err, r.row);
            s = __longlong_as_double(0x7FF8000000000000LL);
        } else {
            s = s / diag;
        }
    }
    x[r.row] = s;
}

template <bool UPPER>
__global__ void __launch_bounds__(BL_THREADS) sptrsv_blocklocal(int n_levels, const int *__restrict__ start,
                                                                const int *__restrict__ cnt,
                                                                const int *__restrict__ level_rows,
                                                                const int *__restrict__ rp, const int *__restrict__ ci,
                                                                const double *__restrict__ val,
                                                                const double *__restrict__ b, double *x, int unit_diag,
                                                                int *err) {
    const int *st = start + (long long)blockIdx.x * n_levels;
    const int *ct = cnt + (long long)blockIdx.x * n_levels;
    BlRow cur, nxt;
    int c0 = n_levels > 0 ? ct[0] : 0;
    bl_load(nxt, (int)threadIdx.x < c0, n_levels > 0 ? st[0] + (int)threadIdx.x : 0, level_rows, rp, ci, val, b);
    for (int l = 0; l < n_levels; ++l) {
        cur = nxt;
        const int c = c0, s0 = st[l];
        if (l + 1 < n_levels) {
            c0 = ct[l + 1];
            bl_load(nxt, (int)threadIdx.x < c0, st[l + 1] + (int)threadIdx.x, level_rows, rp, ci, val, b);
        }
        bl_finish<UPPER>(cur, ci, val, x, unit_diag, err);
        for (int t = threadIdx.x + BL_THREADS; t < c; t += BL_THREADS) {  // levels wider than the CTA
            BlRow extra;
            bl_load(extra, true, s0 + t, level_rows, rp, ci, val, b);
            bl_finish<UPPER>(extra, ci, val, x, unit_diag, err);
        }
        __syncthreads();
    }
}


// Block-local sweep on the schedule-ordered SELL arrays: the address of every
// operand of slot s is computable from s, so the register prefetch is one load
// deep (row id two levels ahead; entries, pivot and right-hand side one level ahead).
struct BsRow {
    int row;
    int c[SELL_CHUNK];
    double a[SELL_CHUNK];
    double rhs, piv;
    long long off;
    int w, lane;
};

template <bool HAS_DIAG>
__device__ __forceinline__ void bs_load(BsRow &r, int row, bool active, int slot, const int *__restrict__ goff, int uw,
                                        const int *__restrict__ scol, const double *__restrict__ sval,
                                        const double *__restrict__ sdiag, const double *__restrict__ b) {
    r.row = active ? row : -1;
    r.w = 0;
    r.off = 0;
    r.lane = slot & 31;
    r.rhs = 0.0;
    r.piv = 1.0;
    if (active) {
        const long long g = slot >> 5;
        r.off = goff ? goff[g] : g * 32LL * uw;
        r.w = goff ? (goff[g + 1] - (int)r.off) >> 5 : uw;
        if (r.row >= 0) r.rhs = b[r.row];
        if (HAS_DIAG) r.piv = sdiag[slot];
    }
#pragma unroll
    for (int u = 0; u < SELL_CHUNK; ++u) {
        const bool in = u < r.w;
        r.c[u] = in ? scol[r.off + 32 * u + r.lane] : -1;
        r.a[u] = in ? sval[r.off + 32 * u + r.lane] : 0.0;
    }
}

template <bool HAS_DIAG>
__device__ __forceinline__ void bs_finish(const BsRow &r, const int *__restrict__ scol, const double *__restrict__ sval,
                                          double *x) {
    if (r.row < 0) return;
    double s = r.rhs;
#pragma unroll
    for (int u = 0; u < SELL_CHUNK; ++u)
        if (r.c[u] >= 0) s -= r.a[u] * x[r.c[u]];
    for (int k = SELL_CHUNK; k < r.w; ++k) {
        const int j = scol[r.off + 32 * k + r.lane];
        if (j >= 0) s -= sval[r.off + 32 * k + r.lane] * x[j];
    }
    x[r.row] = HAS_DIAG ? s / r.piv : s;
}

template <bool HAS_DIAG>
__global__ void __launch_bounds__(BL_THREADS) sptrsv_blocklocal_sell(int n_levels, const int *__restrict__ sstart,
                                                                     const int *__restrict__ cnt,
                                                                     const int *__restrict__ order,
                                                                     const int *__restrict__ goff, int uw,
                                                                     const int *__restrict__ scol,
                                                                     const double *__restrict__ sval,
                                                                     const double *__restrict__ sdiag,
                                                                     const double *__restrict__ b, double *x) {
    const int *st = sstart + (long long)blockIdx.x * n_levels;
    const int *ct = cnt + (long long)blockIdx.x * n_levels;
    const int tid = threadIdx.x;
    // prologue: row ids of levels 0 and 1, operands of level 0
    int c_cur = n_levels > 0 ? ct[0] : 0, c_n = n_levels > 1 ? ct[1] : 0;
    int s_cur = n_levels > 0 ? st[0] : 0, s_n = n_levels > 1 ? st[1] : 0;
    int row0 = tid < c_cur ? order[s_cur + tid] : -1;
    int row_n = tid < c_n ? order[s_n + tid] : -1;
    BsRow cur, nxt;
    bs_load<HAS_DIAG>(nxt, row0, tid < c_cur, s_cur + tid, goff, uw, scol, sval, sdiag, b);
    for (int l = 0; l < n_levels; ++l) {
        cur = nxt;
        const int c = c_cur, s0 = s_cur;
        // stage A: row ids of level l+2;  stage B: operands of level l+1
        int c_nn = 0, s_nn = 0, row_nn = -1;
        if (l + 2 < n_levels) {
            c_nn = ct[l + 2];
            s_nn = st[l + 2];
            if (tid < c_nn) row_nn = order[s_nn + tid];
        }
        if (l + 1 < n_levels) bs_load<HAS_DIAG>(nxt, row_n, tid < c_n, s_n + tid, goff, uw, scol, sval, sdiag, b);
        bs_finish<HAS_DIAG>(cur, scol, sval, x);
        for (int t = tid + BL_THREADS; t < c; t += BL_THREADS) {  // levels wider than the CTA
            BsRow extra;
            bs_load<HAS_DIAG>(extra, order[s0 + t], true, s0 + t, goff, uw, scol, sval, sdiag, b);
            bs_finish<HAS_DIAG>(extra, scol, sval, x);
        }
        __syncthreads();
        c_cur = c_n; s_cur = s_n;
        c_n = c_nn; s_n = s_nn; row_n = row_nn;
    }
}

// Block-local sweep with the block's part of x in a SHARED-MEMORY window.  The rows of a block in schedule
// order (level by level) get block-local positions 0, 1, 2, ...; `scol_loc` holds the position of every
// dependency, and result p lives in xs[p & wmask] until position p + W is written.  Setup checks that no row
// reads further back than the window (device.enable_block_window), so a level costs a shared-memory round
// trip + one CTA barrier instead of the L2 round trip of the variant above (0.77 us per level).  The pivot
// division uses the reciprocal prepared at setup (exact_div: bits of the IEEE quotient).
struct BwRow {
    int row;
    int c[SELL_CHUNK];
    double a[SELL_CHUNK];
    double rhs, piv, rinv;
    long long off;
    int w, lane;
};

template <bool HAS_DIAG>
__device__ __forceinline__ void bw_load(BwRow &r, int row, bool active, int slot,
                                        const int *__restrict__ goff, int uw,
                                        const int *__restrict__ scol, const double *__restrict__ sval,
                                        const double *__restrict__ sdiag, const double *__restrict__ sdinv,
                                        const double *__restrict__ b) {
    r.row = active ? row : -1;
    r.lane = slot & 31;
    r.off = 0;
    r.w = 0;
    if (active) {
        const long long g = slot >> 5;
        r.off = goff ? goff[g] : g * 32LL * uw;
        r.w = goff ? (goff[g + 1] - (int)r.off) >> 5 : uw;
    }
    r.rhs = 0.0;
    r.piv = 1.0;
    r.rinv = 1.0;
    if (active && r.row >= 0) {
        r.rhs = b[r.row];
        if (HAS_DIAG) {
            r.piv = sdiag[slot];
            r.rinv = sdinv[slot];
        }
    }
#pragma unroll
    for (int u = 0; u < SELL_CHUNK; ++u) {
        const bool in = u < r.w;
        r.c[u] = in ? scol[r.off + 32 * u + r.lane] : -1;
        r.a[u] = in ? sval[r.off + 32 * u + r.lane] : 0.0;
    }
}

template <bool HAS_DIAG>
__device__ __forceinline__ void bw_finish(const BwRow &r, const int *__restrict__ scol,
                                          const double *__restrict__ sval, double *xs, int wmask, int pos, double *x) {
    if (r.row < 0) return;
    double s = r.rhs;
#pragma unroll
    for (int u = 0; u < SELL_CHUNK; ++u)
        if (r.c[u] >= 0) s -= r.a[u] * xs[r.c[u] & wmask];
    for (int k = SELL_CHUNK; k < r.w; ++k) {
        const int j = scol[r.off + 32 * k + r.lane];
        if (j >= 0) s -= sval[r.off + 32 * k + r.lane] * xs[j & wmask];
    }
    if (HAS_DIAG) s = exact_div(s, r.piv, r.rinv);
    xs[pos & wmask] = s;
    x[r.row] = s;
}

template <bool HAS_DIAG>
__global__ void __launch_bounds__(BL_THREADS) sptrsv_blockwin_sell(int n_levels, const int *__restrict__ sstart,
                                                                   const int *__restrict__ cnt,
                                                                   const int *__restrict__ lbase,
                                                                   const int *__restrict__ order,
                                                                   const int *__restrict__ goff, int uw,
                                                                   const int *__restrict__ scol,
                                                                   const double *__restrict__ sval,
                                                                   const double *__restrict__ sdiag,
                                                                   const double *__restrict__ sdinv, int wmask,
                                                                   const double *__restrict__ b, double *x) {
    extern __shared__ double xs_win[];
    const int *st = sstart + (long long)blockIdx.x * n_levels;
    const int *ct = cnt + (long long)blockIdx.x * n_levels;
    const int *lb = lbase + (long long)blockIdx.x * n_levels;
    const int tid = threadIdx.x;
    int c_cur = n_levels > 0 ? ct[0] : 0, c_n = n_levels > 1 ? ct[1] : 0;
    int s_cur = n_levels > 0 ? st[0] : 0, s_n = n_levels > 1 ? st[1] : 0;
    int p_cur = n_levels > 0 ? lb[0] : 0, p_n = n_levels > 1 ? lb[1] : 0;
    int row0 = tid < c_cur ? order[s_cur + tid] : -1;
    int row_n = tid < c_n ? order[s_n + tid] : -1;
    BwRow cur, nxt;
    bw_load<HAS_DIAG>(nxt, row0, tid < c_cur, s_cur + tid, goff, uw, scol, sval, sdiag, sdinv, b);
    for (int l = 0; l < n_levels; ++l) {
        cur = nxt;
        const int c = c_cur, s0 = s_cur, p0 = p_cur;
        int c_nn = 0, s_nn = 0, p_nn = 0, row_nn = -1;
        if (l + 2 < n_levels) {
            c_nn = ct[l + 2];
            s_nn = st[l + 2];
            p_nn = lb[l + 2];
            if (tid < c_nn) row_nn = order[s_nn + tid];
        }
        if (l + 1 < n_levels) bw_load<HAS_DIAG>(nxt, row_n, tid < c_n, s_n + tid, goff, uw, scol, sval, sdiag, sdinv, b);
        bw_finish<HAS_DIAG>(cur, scol, sval, xs_win, wmask, p0 + tid, x);
        for (int t = tid + (int)blockDim.x; t < c; t += (int)blockDim.x) {  // levels wider than the CTA
            BwRow extra;
            bw_load<HAS_DIAG>(extra, order[s0 + t], true, s0 + t, goff, uw, scol, sval, sdiag, sdinv, b);
            bw_finish<HAS_DIAG>(extra, scol, sval, xs_win, wmask, p0 + t, x);
        }
        __syncthreads();
        c_cur = c_n; s_cur = s_n; p_cur = p_n;
        c_n = c_nn; s_n = s_nn; p_n = p_nn; row_n = row_nn;
    }
}

#endif  // DDILU_EXPERIMENTS
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

#ifdef DDILU_EXPERIMENTS   // tuning knobs of the probes
extern "C" int ddilu_set_tuning(const char *key, int value) {
    if (!key) return DDILU_ERR_ARG;
    if (!strcmp(key, "trsv_blocks_per_sm")) g_trsv.blocks_per_sm = value;
    else if (!strcmp(key, "trsv_sleep_ns")) g_trsv.sleep_ns = (unsigned)value;
    else if (!strcmp(key, "wr_blocks_per_sm")) g_trsv.wr_blocks_per_sm = value;
    else if (!strcmp(key, "trsv_pipe")) g_trsv.pipe = value;
    else if (!strcmp(key, "trsv_depth")) g_trsv.depth = value;
    else if (!strcmp(key, "trsv_chunk")) g_trsv.chunk = value;
    else if (!strcmp(key, "trsv_stage_mask")) g_trsv.stage_mask = value;
    else if (!strcmp(key, "trsv_far_sleep_ns")) g_trsv.far_sleep_ns = value;
    else if (!strcmp(key, "trsv_pipe_warps_per_sm")) g_trsv.pipe_warps_per_sm = value;
    else if (!strcmp(key, "win_threads")) g_trsv.win_threads = value;
    else return DDILU_ERR_ARG;
    return DDILU_OK;
}

#endif  // DDILU_EXPERIMENTS
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

/* the same solve with a warp per row (long rows: ILUT / ILU(k) / 27-point factors) */
extern "C" int ddilu_sptrsv_warprow(int n, int n_slots, const int *order, const int *row_ptr, const int *col_idx,
                                    const double *values, const double *b, double *x, int upper, int unit_diag,
                                    int *err, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (x == b) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    unsigned sleep_ns = g_trsv.sleep_ns;
    void *args[] = {&n_slots, &order, &row_ptr, &col_idx, &values, &b, &x, &unit_diag, &err, &sleep_ns};
    void *fn = upper ? (void *)sptrsv_warprow<true> : (void *)sptrsv_warprow<false>;
    int occ = 0;
    DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * WR_WARPS, 0));
    if (occ < 1) occ = 1;
    if (g_trsv.wr_blocks_per_sm > 0 && occ > g_trsv.wr_blocks_per_sm) occ = g_trsv.wr_blocks_per_sm;
    long long grid = (long long)occ * device_info().sm_count;
    const long long need = ((long long)n_slots + WR_WARPS - 1) / WR_WARPS;
    if (grid > need) grid = need < 1 ? 1 : need;
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, 32 * WR_WARPS, args, 0, st));
    return DDILU_OK;
}

extern "C" int ddilu_sell_width(int n_slots, const int *order, const int *row_ptr, const int *col_idx,
                                const double *values, int upper, int unit_diag, int *gw32, double *sdiag,
                                int *bad_row, int *pos_work, int *gwait, void *stream) {
    if (n_slots <= 0) return DDILU_OK;
    if (n_slots & 31) return DDILU_ERR_ARG;
    if (gwait && !pos_work) return DDILU_ERR_ARG;
    const int n_groups = n_slots >> 5;
    if (gwait)
        sched_positions<<<stream_grid(n_slots, 256), 256, 0, (cudaStream_t)stream>>>(n_slots, order, pos_work);
    sell_width<<<stream_grid((long long)n_groups * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        n_groups, order, row_ptr, col_idx, values, upper, unit_diag, gw32, sdiag, bad_row, gwait ? pos_work : nullptr,
        gwait);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sell_fill(int n_slots, const int *order, const int *row_ptr, const int *col_idx,
                               const double *values, int upper, const int *goff, int uniform_width, int *scol,
                               double *sval, void *stream) {
    if (n_slots <= 0) return DDILU_OK;
    const int n_groups = n_slots >> 5;
    sell_fill<<<stream_grid((long long)n_groups * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        n_groups, order, row_ptr, col_idx, values, upper, goff, uniform_width, scol, sval);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_compose_wait(int n_groups, const int *gwait, const int *pos, const int *prev, int *out,
                                  void *stream) {
    if (n_groups <= 0) return DDILU_OK;
    compose_wait<<<stream_grid(n_groups, 256), 256, 0, (cudaStream_t)stream>>>(n_groups, gwait, pos, prev, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sptrsv_sell(int n, int n_slots, int n_levels, const int *order, const int *goff,
                                 int uniform_width, const int *scol, const double *sval, const double *sdiag,
                                 const int *gwait, const int *gfar1, const int *gfar2, double avg_width,
                                 const double *b, double *x, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (x == b || (n_slots & 31)) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    int n_groups = n_slots >> 5;
    int mask = g_trsv.stage_mask;
    if (mask < 0) mask = (n_levels > 0 && n_groups / n_levels >= 256) ? 4 : 3;
    const int *w0 = (mask & 4) ? gwait : nullptr;
    const int *w1 = (mask & 2) ? gfar1 : nullptr;
    const int *w2 = (mask & 1) ? gfar2 : nullptr;
    unsigned far_sleep = (unsigned)g_trsv.far_sleep_ns;
    void *args[] = {&n_groups, &order, &goff, &uniform_width, &scol, &sval, &sdiag, &w0, &w1, &w2, &far_sleep, &b, &x};
#ifdef DDILU_EXPERIMENTS
    if (g_trsv.pipe) {
        void *pargs[] = {&n_groups, &order, &goff, &uniform_width, &scol, &sval, &sdiag, &b, &x};
        // few resident warps: pipe_warps_per_sm warps on every SM, 4 warps per CTA
        int ctas_per_sm = (g_trsv.pipe_warps_per_sm + 3) / 4;
        if (ctas_per_sm < 1) ctas_per_sm = 1;
        void *fn = sdiag ? (void *)sptrsv_sell_pipe<true> : (void *)sptrsv_sell_pipe<false>;
        int occ = 0;
        if (sdiag) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sptrsv_sell_pipe<true>, 128, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sptrsv_sell_pipe<false>, 128, 0);
        if (occ < 1) occ = 1;
        if (ctas_per_sm > occ) ctas_per_sm = occ;
        long long grid = (long long)ctas_per_sm * device_info().sm_count;
        long long need = ((long long)n_groups + 3) / 4;
        if (grid > need) grid = need;
        DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, 128, pargs, 0, st));
        return DDILU_OK;
    }
#endif  // DDILU_EXPERIMENTS
    // dependencies polled per round: 4 for stencil-length rows, 8 / 16 for long rows (ILUT / ILU(k) /
    // 27-point factors); avg_width = average padded entries per lane of the layout
    if (avg_width <= 0.0) avg_width = uniform_width;
    int chunk = g_trsv.chunk;
    if (chunk <= 0) chunk = avg_width > 14.0 ? 16 : (avg_width > 6.0 ? 8 : 4);
    void *fn;
    if (chunk >= 16) fn = sdiag ? (void *)sptrsv_sell<true, 16> : (void *)sptrsv_sell<false, 16>;
    else if (chunk >= 8) fn = sdiag ? (void *)sptrsv_sell<true, 8> : (void *)sptrsv_sell<false, 8>;
    else fn = sdiag ? (void *)sptrsv_sell<true, 4> : (void *)sptrsv_sell<false, 4>;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, SELL_THREADS, 0);
    if (occ < 1) occ = 1;
    if (g_trsv.blocks_per_sm > 0 && occ > g_trsv.blocks_per_sm) occ = g_trsv.blocks_per_sm;
    long long cap = (long long)occ * device_info().sm_count;
    long long need_blocks = ((long long)n_slots + SELL_THREADS - 1) / SELL_THREADS;
    int grid = (int)(cap < need_blocks ? cap : (need_blocks < 1 ? 1 : need_blocks));
    if (g_trsv.depth > 0 && n_levels > 0) {
        // narrow levels: cap the resident warps at depth x (groups per level)
        long long want_warps = (long long)g_trsv.depth * ((n_groups + n_levels - 1) / n_levels);
        long long want = (want_warps + SELL_THREADS / 32 - 1) / (SELL_THREADS / 32);
        if (want < 16) want = 16;
        if (want < grid) grid = (int)want;
    }
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, grid, SELL_THREADS, args, 0, st));
    return DDILU_OK;
}

#ifdef DDILU_EXPERIMENTS
extern "C" int ddilu_blocklocal_table(int n, int n_blocks, const int *seg_ptr, int n_levels, const int *lev,
                                      const int *level_rows, int *start, int *cnt, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0 || n_blocks <= 0 || n_levels <= 0) return DDILU_OK;
    size_t slots = (size_t)n_blocks * n_levels;
    DDILU_CHECK(cudaMemsetAsync(start, 0x7F, sizeof(int) * slots, st));
    DDILU_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * slots, st));
    blocklocal_table<<<stream_grid(n, 256), 256, 0, st>>>(n, n_blocks, seg_ptr, n_levels, lev, level_rows, start, cnt);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sptrsv_blocklocal(int n_blocks, int n_levels, const int *start, const int *cnt,
                                       const int *level_rows, const int *row_ptr, const int *col_idx,
                                       const double *values, const double *b, double *x, int upper, int unit_diag,
                                       int *err, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_blocks <= 0 || n_levels <= 0) return DDILU_OK;
    if (x == b) return DDILU_ERR_ARG;
    if (upper)
        sptrsv_blocklocal<true><<<n_blocks, BL_THREADS, 0, st>>>(n_levels, start, cnt, level_rows, row_ptr, col_idx,
                                                                values, b, x, unit_diag, err);
    else
        sptrsv_blocklocal<false><<<n_blocks, BL_THREADS, 0, st>>>(n_levels, start, cnt, level_rows, row_ptr, col_idx,
                                                                 values, b, x, unit_diag, err);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* block-local sweep with x in a shared-memory window of wmask + 1 doubles */
extern "C" int ddilu_sptrsv_blockwin_sell(int n_blocks, int n_levels, const int *sstart, const int *cnt,
                                          const int *lbase, const int *order, const int *goff, int uniform_width,
                                          const int *scol_loc,
                                          const double *sval, const double *sdiag, const double *sdinv, int wmask,
                                          const double *b, double *x, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_blocks <= 0 || n_levels <= 0) return DDILU_OK;
    if (x == b || wmask < 0 || ((wmask + 1) & wmask) || (sdiag && !sdinv)) return DDILU_ERR_ARG;
    const size_t smem = sizeof(double) * (size_t)(wmask + 1);
    if (smem > 200 * 1024) return DDILU_ERR_ARG;
    void *fn = sdiag ? (void *)sptrsv_blockwin_sell<true> : (void *)sptrsv_blockwin_sell<false>;
    static size_t attr[2] = {0, 0};
    if (attr[sdiag ? 1 : 0] < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[sdiag ? 1 : 0] = smem;
    }
    const int threads = g_trsv.win_threads > 0 ? g_trsv.win_threads : BL_THREADS;
    if (sdiag)
        sptrsv_blockwin_sell<true><<<n_blocks, threads, smem, st>>>(n_levels, sstart, cnt, lbase, order, goff,
                                                                      uniform_width, scol_loc, sval, sdiag, sdinv, wmask,
                                                                      b, x);
    else
        sptrsv_blockwin_sell<false><<<n_blocks, threads, smem, st>>>(n_levels, sstart, cnt, lbase, order, goff,
                                                                       uniform_width, scol_loc, sval, sdiag, sdinv,
                                                                       wmask, b, x);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sptrsv_blocklocal_sell(int n_blocks, int n_levels, const int *sstart, const int *cnt,
                                            const int *order, const int *goff, int uniform_width, const int *scol,
                                            const double *sval, const double *sdiag, const double *b, double *x,
                                            void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_blocks <= 0 || n_levels <= 0) return DDILU_OK;
    if (x == b) return DDILU_ERR_ARG;
    if (sdiag)
        sptrsv_blocklocal_sell<true><<<n_blocks, BL_THREADS, 0, st>>>(n_levels, sstart, cnt, order, goff, uniform_width,
                                                                     scol, sval, sdiag, b, x);
    else
        sptrsv_blocklocal_sell<false><<<n_blocks, BL_THREADS, 0, st>>>(n_levels, sstart, cnt, order, goff,
                                                                      uniform_width, scol, sval, sdiag, b, x);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
#endif  // DDILU_EXPERIMENTS
