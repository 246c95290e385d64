// Lattice sparse triangular solve: the fast path of sptrsv for factors of
// 7-point-type stencils (<= 3 dependencies per row) on a structured grid.
//
// Replaces sparse.py:228-272 (`_lower_solve`, `_upper_solve`) like tiled.cu; same
// arithmetic, same storage-order row sums: bit-exact.
//
// Why another kernel.  The rotating-warp kernel (tiled.cu) walks a box tile level
// by level with a named barrier per level: ~450 cycles per level for ~23 rows, 4
// such chains per SM -> 35 % of the HBM roofline.  Here ONE WARP owns a tile and
// nothing but the warp's own shared-memory line buffer sits between two levels:
//
//   * a box tile (t0 x t1 x t2 grid nodes, t1*t2 <= 64) is read as t1*t2 LINES
//     along grid axis 0; lane (line & 31), register slot (line >> 5) owns a line;
//   * after the build kernel has oriented every axis of the tile so that all
//     in-tile dependencies point to the directed coordinate minus one, row
//     (a, b, c) is solved at STEP a + b + c: its in-tile dependencies (a-1, b, c),
//     (a, b-1, c), (a, b, c-1) were solved exactly one step earlier, each by a
//     known line.  A step is: read <= 3 values from the warp's line buffer (the
//     previous step's results) or from the tile's boundary values, 3 multiplies,
//     3 subtractions in storage order (+ the exact reciprocal division for U),
//     store into the other half of the line buffer, __syncwarp.  No named
//     barrier, no other warp, ~100 cycles per step;
//   * the rows' static records (coefficients, operand codes, row id [, pivot])
//     are stored in (step, slot, lane) order, compacted over the active lanes,
//     and stream through a per-warp cp.async ring D steps ahead; the right-hand
//     side b[row] follows D/2 steps ahead (cp.async 8 B gather, the row id comes
//     out of the record that has already landed);
//   * boundary dependencies (values of rows in other tiles) are gathered once per
//     tile after the producer tiles have raised their per-tile flags
//     (release/acquire, <= 11 producers per tile; 3 on a 7-point grid).  No
//     sentinel preset of x, no polling per value.
//
// Nothing about the ORDERING is assumed: the build kernel checks per tile that
// every in-tile dependency is a lattice neighbour, that the orientation of each
// axis is consistent and that rows have <= 3 dependencies; any failure makes the
// caller fall back to the general tiled / sync-free kernels.  Tiles are taken in
// a topological order of the tile graph (the same ddilu_tile_* machinery), warp w
// takes tiles w, w + W, ... and the launch is cooperative, so the lowest
// unfinished tile is always some warp's current tile: deadlock-free.
//
// Bytes moved per row: 32 (L) / 48 (U) record + 8 b + 8 x (+ 12 per boundary
// value) against the algorithmic 12 nnz + 4 + 16 = 56 (L) / 68 (U) of a 7-point
// ILU(0) factor row.
#include <stdint.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int LAT_MAX_ROWS = 1024;
constexpr int LAT_MAX_STEPS = 32;     // one table entry per lane
constexpr int LAT_MAX_DEPS = 11;      // producer tiles listed in the table (lanes 5..15)
constexpr int LAT_XE = 448;           // boundary values per tile held in shared memory
constexpr int LAT_ZERO_CODE = 1023;   // operand code of a padded entry
constexpr int LAT_WPB = 1;            // warps per CTA (independent of each other; 1 = finest shared-memory packing)

// table entry of lane i of a tile (int4): x = active lanes of slot 0 at step i, y = of slot 1, z = record
// offset of step i, w = header word i:
enum { LW_NSTEPS = 0, LW_NEXT, LW_BLK16, LW_REC16, LW_NDEPS, LW_DEP0, LW_T = 16, LW_BYTES16 = 17 };

__device__ __forceinline__ int lat_pad16(int bytes) { return (bytes + 15) & ~15; }

__device__ __forceinline__ int lat_block_scan(int v, int *total, int *wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = wsum[lane], winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, winc, o);
            if (lane >= o) winc += t;
        }
        wsum[lane] = winc - w;
        if (lane == 31) wsum[32] = winc;
    }
    __syncthreads();
    *total = wsum[32];
    return wsum[warp] + inc - v;
}

// One CTA (1024 threads, one per row) per tile, tiles in schedule order.
//   FILL = false: checks the lattice property, sizes the tile's block -> blk16[q], maxima -> stats
//   FILL = true : writes the table entry tab[32 q ..] and the block (boundary columns, records)
// stats: [0] failure flag, [1] max boundary values, [2] max steps, [3] first bad pivot row, [4] max producers,
//        [5] max block bytes, [6] max rows
template <bool FILL>
__global__ void __launch_bounds__(LAT_MAX_ROWS)
lattice_build(int n_tiles, const int *__restrict__ tsched, const int *__restrict__ tile_pos,
              const int *__restrict__ tile_ptr, const int *__restrict__ trows, const int *__restrict__ tile_of,
              const int *__restrict__ rp, const int *__restrict__ ci, const double *__restrict__ val,
              const int *__restrict__ nodes, int d0, int d1, int t0, int t1, int t2, int upper, int has_diag,
              int4 *__restrict__ tab, int *blk16, int *stats, unsigned char *blob) {
    __shared__ int s_sign[3];
    __shared__ int s_dep[LAT_MAX_DEPS];
    __shared__ int s_minmax[2];
    __shared__ unsigned s_mask[LAT_MAX_STEPS][2];
    __shared__ int s_off[LAT_MAX_STEPS + 1];
    __shared__ int s_ne[LAT_MAX_ROWS];
    __shared__ int s_wsum[33];
    __shared__ int s_fail;
    const int q = blockIdx.x;
    const int t = tsched[q];
    const int base = tile_ptr[t], T = tile_ptr[t + 1] - base;
    const int i = threadIdx.x;
    const bool active = i < T;
    if (i < 3) s_sign[i] = 0;
    if (i < LAT_MAX_DEPS) s_dep[i] = -1;
    if (i == 0) {
        s_minmax[0] = 0x7FFFFFFF;
        s_minmax[1] = -1;
        s_fail = 0;
    }
    if (i < LAT_MAX_STEPS) s_mask[i][0] = s_mask[i][1] = 0u;
    s_ne[i] = 0;
    __syncthreads();
    const int row = active ? trows[base + i] : -1;
    int l[3] = {0, 0, 0}, c[3] = {0, 0, 0};
    auto coords = [&](int r, int *cc) {
        const int g = nodes[r];
        cc[0] = g % d0;
        cc[1] = (g / d0) % d1;
        cc[2] = g / (d0 * d1);
    };
    int nd = 0, ne = 0;
    if (active) {
        coords(row, c);
        l[0] = c[0] % t0;
        l[1] = c[1] % t1;
        l[2] = c[2] % t2;
        for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (!(upper ? j > row : j < row)) continue;
            ++nd;
            const int tj = tile_of[j];
            if (tj == t) {
                int cj[3];
                coords(j, cj);
                int ax = -1, nz = 0, dl = 0;
                for (int a = 0; a < 3; ++a)
                    if (cj[a] != c[a]) {
                        ++nz;
                        ax = a;
                        dl = cj[a] - c[a];
                    }
                if (nz != 1 || (dl != 1 && dl != -1))
                    s_fail = 1;   // not a lattice neighbour
                else
                    atomicOr(&s_sign[ax], dl > 0 ? 1 : 2);
            } else {
                ++ne;
                bool placed = false;
                for (int s = 0; s < LAT_MAX_DEPS && !placed; ++s) {
                    const int old = atomicCAS(&s_dep[s], -1, tj);
                    placed = old == -1 || old == tj;
                }
                if (!placed) s_fail = 1;   // more producer tiles than the table holds
            }
        }
        if (nd > 3) s_fail = 1;
    }
    __syncthreads();
    if (s_sign[0] == 3 || s_sign[1] == 3 || s_sign[2] == 3) s_fail = 1;   // both orientations along one axis
    __syncthreads();
    if (s_fail) {
        if (i == 0) atomicOr(stats + 0, 1);
        if (!FILL && i == 0) blk16[q] = 0;
        return;
    }
    // directed coordinates: dependencies sit at the coordinate minus one
    const bool rev0 = s_sign[0] & 1, rev1 = s_sign[1] & 1, rev2 = s_sign[2] & 1;
    const int a_ = rev0 ? t0 - 1 - l[0] : l[0], b_ = rev1 ? t1 - 1 - l[1] : l[1], c_ = rev2 ? t2 - 1 - l[2] : l[2];
    const int step_raw = a_ + b_ + c_;
    const int line = b_ + t1 * c_;
    const int lane = line & 31, slot = line >> 5;
    if (active) {
        atomicMin(&s_minmax[0], step_raw);
        atomicMax(&s_minmax[1], step_raw);
    }
    __syncthreads();
    const int smin = s_minmax[0], n_steps = s_minmax[1] - smin + 1;
    const int st = step_raw - smin;
    if (n_steps > LAT_MAX_STEPS) {
        if (i == 0) atomicOr(stats + 0, 1);
        if (!FILL && i == 0) blk16[q] = 0;
        return;
    }
    if (active) atomicOr(&s_mask[st][slot], 1u << lane);
    __syncthreads();
    if (i == 0) {
        int run = 0;
        for (int s = 0; s < n_steps; ++s) {
            s_off[s] = run;
            run += __popc(s_mask[s][0]) + __popc(s_mask[s][1]);
        }
        s_off[n_steps] = run;
    }
    __syncthreads();
    int p = 0;
    if (active) {
        const unsigned lt = (1u << lane) - 1u;
        p = s_off[st] + (slot ? __popc(s_mask[st][0]) : 0) + __popc(s_mask[st][slot] & lt);
        s_ne[p] = ne;
    }
    __syncthreads();
    int n_ext;
    const int eoff_i = lat_block_scan(s_ne[i], &n_ext, s_wsum);   // boundary values numbered in record order
    __syncthreads();
    s_ne[i] = eoff_i;
    __syncthreads();
    int n_deps = 0;
    for (int s = 0; s < LAT_MAX_DEPS; ++s) n_deps += s_dep[s] >= 0 ? 1 : 0;
    const int recb = has_diag ? 48 : 32;
    const int off_rec = lat_pad16(4 * n_ext);
    const int bytes = off_rec + recb * T;
    if (!FILL) {
        if (i == 0) {
            blk16[q] = bytes >> 4;
            atomicMax(stats + 1, n_ext);
            atomicMax(stats + 2, n_steps);
            atomicMax(stats + 4, n_deps);
            atomicMax(stats + 5, bytes);
            atomicMax(stats + 6, T);
        }
        return;
    }
    unsigned char *blk = blob + 16LL * blk16[q];
    if (i < 32) {
        int w = 0;
        switch (i) {
            case LW_NSTEPS: w = n_steps; break;
            case LW_NEXT: w = n_ext; break;
            case LW_BLK16: w = blk16[q]; break;
            case LW_REC16: w = off_rec >> 4; break;
            case LW_NDEPS: w = n_deps; break;
            case LW_T: w = T; break;
            case LW_BYTES16: w = bytes >> 4; break;
            default: break;
        }
        if (i >= LW_DEP0 && i < LW_DEP0 + LAT_MAX_DEPS) {
            // compact the producer list (slots fill from the front: CAS on the first free one)
            const int d = s_dep[i - LW_DEP0];
            w = d >= 0 ? tile_pos[d] : -1;
        }
        tab[32LL * q + i] = make_int4(i < n_steps ? (int)s_mask[i][0] : 0, i < n_steps ? (int)s_mask[i][1] : 0,
                                      i < n_steps ? s_off[i] : 0, w);
    }
    // alignment tail of the boundary-column list
    for (int pz = 4 * n_ext + i; pz < off_rec; pz += LAT_MAX_ROWS) blk[pz] = 0;
    if (!active) return;
    int *ext_out = (int *)blk;
    unsigned char *rec = blk + off_rec + (size_t)recb * p;
    double av[3] = {0.0, 0.0, 0.0};
    unsigned code[3] = {LAT_ZERO_CODE, LAT_ZERO_CODE, LAT_ZERO_CODE};
    int kk = 0, e = s_ne[p];
    double diag = 1.0;
    bool seen = false, bad = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (upper ? j > row : j < row) {
            unsigned cd;
            if (tile_of[j] == t) {
                int cj[3];
                coords(j, cj);
                const int lj0 = cj[0] % t0, lj1 = cj[1] % t1, lj2 = cj[2] % t2;
                const int aj = rev0 ? t0 - 1 - lj0 : lj0, bj = rev1 ? t1 - 1 - lj1 : lj1,
                          cjj = rev2 ? t2 - 1 - lj2 : lj2;
                if (aj + bj + cjj - smin != st - 1) bad = true;   // must have been solved one step earlier
                cd = (unsigned)(bj + t1 * cjj);
            } else {
                cd = 64u + (unsigned)e;
                ext_out[e] = j;
                ++e;
            }
            if (kk < 3) {
                av[kk] = val[k];
                code[kk] = cd;
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    if (bad) atomicOr(stats + 0, 1);
    double *rd = (double *)rec;
    rd[0] = av[0];
    rd[1] = av[1];
    rd[2] = av[2];
    ((unsigned *)rec)[6] = code[0] | (code[1] << 10) | (code[2] << 20);
    ((int *)rec)[7] = row;
    if (has_diag) {
        rd[4] = diag;
        rd[5] = safe_reciprocal(diag);
        if (!seen || fabs(diag) < 1e-300) atomicMin(stats + 3, row);
    }
}

// ---------------------------------------------------------------------------
// solve

__device__ __forceinline__ uint32_t lat_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double ld_cg(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void lat_mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lat_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void lat_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lat_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void lat_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     lat_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(lat_smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool lat_mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(lat_smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

// shared memory of one warp (bytes): 2 mbarriers | 2 tile blocks | 2 right-hand-side buffers | line buffers,
// boundary values and the zero slot
__host__ __device__ inline size_t lat_warp_bytes(int blkmax, int tmax, int xemax) {
    return 16 + 2 * (size_t)blkmax + 2 * 8 * (size_t)((tmax + 1) & ~1) + 8 * (size_t)(128 + xemax + 2);
}

// One warp per CTA; warp w of W takes the tiles w, w + W, ... of the schedule.  The WHOLE static block of a
// tile (boundary columns + row records, contiguous) arrives by one TMA bulk copy into one of two buffers
// while the previous tile is being solved; its right-hand side is gathered (cp.async, 8 B per row) as soon as
// the block has landed.  When the producers' flags are up, nothing but shared memory sits on the tile's
// critical path: boundary gather -> n_steps x (3 loads, 3 multiply/subtract, store, __syncwarp) -> flag.
template <bool HAS_DIAG, int NS>
__global__ void __launch_bounds__(32)
sptrsv_lattice(int n_tiles, const int4 *__restrict__ tab, const unsigned char *__restrict__ blob, int *flags,
               int blkmax, int tmax, int xemax, long long *dbg, const double *__restrict__ b, double *x) {
    constexpr int RECB = HAS_DIAG ? 48 : 32;
    extern __shared__ __align__(128) unsigned char lat_smem[];
    const int lane = threadIdx.x;
    uint64_t *mbar = (uint64_t *)lat_smem;
    unsigned char *blk0 = lat_smem + 16;
    const int tpad = (tmax + 1) & ~1;
    double *rhs0 = (double *)(blk0 + 2 * (size_t)blkmax);
    double *xs = rhs0 + 2 * (size_t)tpad;        // [2][64] lines | [xemax] boundary | zero
    const int ZIDX = 128 + xemax;
    const int W = gridDim.x;
    const int gw = blockIdx.x;
    const int nk = gw < n_tiles ? (n_tiles - gw + W - 1) / W : 0;
    if (nk == 0) return;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    if (lane == 0) {
        lat_mbar_init(&mbar[0], 1);
        lat_mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        xs[ZIDX] = 0.0;
    }
    __syncwarp();
    auto load_tab = [&](int k) -> int4 {
        return k < nk ? __ldg(tab + 32LL * (gw + (long long)k * W) + lane) : make_int4(0, 0, 0, 0);
    };
    auto issue_block = [&](const int4 &tb, int k) {   // TMA of tile k's block into buffer k & 1
        if (k >= nk) return;
        const int blk16 = __shfl_sync(full, tb.w, LW_BLK16), bytes16 = __shfl_sync(full, tb.w, LW_BYTES16);
        if (lane == 0) {
            lat_mbar_expect_tx(&mbar[k & 1], (uint32_t)bytes16 << 4);
            lat_bulk_g2s(blk0 + (size_t)(k & 1) * blkmax, blob + 16LL * blk16, (uint32_t)bytes16 << 4, &mbar[k & 1]);
        }
    };
    auto block_landed = [&](int k) -> bool {
        int ok = 0;
        if (lane == 0) ok = lat_mbar_test(&mbar[k & 1], (uint32_t)((k >> 1) & 1)) ? 1 : 0;
        return __shfl_sync(full, ok, 0) != 0;
    };
    auto issue_rhs = [&](const int4 &tb, int k) {     // right-hand side of tile k: b[row] -> rhs[k & 1][p]
        const int T = __shfl_sync(full, tb.w, LW_T), rec16 = __shfl_sync(full, tb.w, LW_REC16);
        const unsigned char *recs = blk0 + (size_t)(k & 1) * blkmax + 16 * rec16;
        double *rh = rhs0 + (size_t)(k & 1) * tpad;
        for (int p = lane; p < T; p += 32) {
            const int rowid = *(const int *)(recs + (size_t)RECB * p + 28);
            cp_async8(lat_smem_u32(rh + p), b + rowid);
        }
        cp_async_commit();
    };
    long long t_all = 0, t_dep = 0, t_gather = 0, t_steps = 0, t_rhs = 0, t_blk = 0, t_fence = 0;
    if (dbg) t_all = clock64();
    int4 tb0 = load_tab(0), tb1 = load_tab(1), tb2 = load_tab(2);
    issue_block(tb0, 0);
    issue_block(tb1, 1);
    while (!block_landed(0)) {}
    issue_rhs(tb0, 0);
    for (int k = 0; k < nk; ++k) {
        const int cur = k & 1;
        const unsigned char *blk = blk0 + (size_t)cur * blkmax;
        double *rh = rhs0 + (size_t)cur * tpad;     // b[row] of record p, replaced by x[row] as the rows are solved
        long long c0 = 0;
        if (dbg) c0 = clock64();
        cp_async_wait<0>();     // rhs of tile k (the block itself was awaited before the rhs was issued)
        __syncwarp();
        if (dbg) t_rhs += clock64() - c0, c0 = clock64();
        // ---- producers finished?
        const int n_deps = __shfl_sync(full, tb0.w, LW_NDEPS);
        const int depq = __shfl_sync(full, tb0.w, (LW_DEP0 + lane) & 31);
        if (lane < n_deps)
            while (ld_acquire(flags + depq) == 0) __nanosleep(32);
        __syncwarp();
        if (dbg) t_dep += clock64() - c0, c0 = clock64();
        // ---- boundary values
        const int n_ext = __shfl_sync(full, tb0.w, LW_NEXT);
        const int *ext = (const int *)blk;
        for (int e0 = 0; e0 < n_ext; e0 += 128) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                v[u] = e < n_ext ? ld_cg(x + ext[e]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < n_ext) xs[128 + e] = v[u];
            }
        }
        __syncwarp();
        if (dbg) t_gather += clock64() - c0, c0 = clock64();
        // ---- the steps
        const int ns = __shfl_sync(full, tb0.w, LW_NSTEPS);
        const unsigned char *recs = blk + 16 * __shfl_sync(full, tb0.w, LW_REC16);
        bool next_rhs = k + 1 >= nk;
        auto row_step = [&](int p, int rdbase, int wrslot) {
            const unsigned char *rec = recs + (size_t)RECB * p;
            const double2 c01 = *(const double2 *)rec;
            const double c2 = *(const double *)(rec + 16);
            const uint2 meta = *(const uint2 *)(rec + 24);
            const double rhs = rh[p];
            const int k0 = (int)(meta.x & 1023u), k1 = (int)((meta.x >> 10) & 1023u), k2 = (int)((meta.x >> 20) & 1023u);
            const int i0 = k0 < 64 ? rdbase + k0 : min(k0 + 64, ZIDX);
            const int i1 = k1 < 64 ? rdbase + k1 : min(k1 + 64, ZIDX);
            const int i2 = k2 < 64 ? rdbase + k2 : min(k2 + 64, ZIDX);
            const double v0 = xs[i0], v1 = xs[i1], v2 = xs[i2];
            double sum = rhs;
            sum -= c01.x * v0;
            sum -= c01.y * v1;
            sum -= c2 * v2;
            if (HAS_DIAG) {
                const double2 pr = *(const double2 *)(rec + 32);
                sum = exact_div(sum, pr.x, pr.y);
            }
            xs[wrslot] = sum;
            rh[p] = sum;      // NOT to global memory here: __syncwarp behind a global store waits for the store's
                              // round trip to L2 (measured: ~2000 cycles per step); the tile's results leave at its end
        };
        for (int t = 0; t < ns; ++t) {
            const unsigned m0 = (unsigned)__shfl_sync(full, tb0.x, t);
            const unsigned m1 = NS > 1 ? (unsigned)__shfl_sync(full, tb0.y, t) : 0u;
            const int off = __shfl_sync(full, tb0.z, t);
            const int rd = ((t + 1) & 1) * 64, wr = (t & 1) * 64;
            if ((m0 >> lane) & 1u) row_step(off + __popc(m0 & lt), rd, wr + lane);
            if (NS > 1 && ((m1 >> lane) & 1u)) row_step(off + __popc(m0) + __popc(m1 & lt), rd, wr + 32 + lane);
            __syncwarp();
            if (!next_rhs && (t & 3) == 3 && block_landed(k + 1)) {   // next tile's block is here: start its gather
                issue_rhs(tb1, k + 1);
                next_rhs = true;
            }
        }
        if (dbg) t_steps += clock64() - c0, c0 = clock64();
        // ---- tile finished: results to global memory, visible, then the flag
        {
            const int T = __shfl_sync(full, tb0.w, LW_T);
            for (int p = lane; p < T; p += 32) x[*(const int *)(recs + (size_t)RECB * p + 28)] = rh[p];
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(flags + gw + (long long)k * W, 1);
        if (dbg) t_fence += clock64() - c0, c0 = clock64();
        if (!next_rhs) {
            while (!block_landed(k + 1)) {}
            issue_rhs(tb1, k + 1);
        }
        if (dbg) t_blk += clock64() - c0;
        // this buffer is free again: tile k + 2
        issue_block(tb2, k + 2);
        tb0 = tb1;
        tb1 = tb2;
        tb2 = load_tab(k + 3);
    }
    if (dbg && lane == 0) {
        long long *o = dbg + 8LL * gw;
        o[0] = clock64() - t_all;
        o[1] = t_rhs;
        o[2] = t_dep;
        o[3] = t_gather;
        o[4] = t_steps;
        o[5] = t_fence;
        o[6] = t_blk;
        o[7] = nk;
    }
}

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

extern "C" int ddilu_lattice_build(int fill, int n_tiles, const int *tsched, const int *tile_pos, const int *tile_ptr,
                                   const int *trows, const int *tile_of, const int *row_ptr, const int *col_idx,
                                   const double *values, const int *nodes, const int *dims3, const int *tdims3,
                                   int upper, int has_diag, void *tab, int *blk16, int *stats, unsigned char *blob,
                                   void *stream) {
    if (n_tiles <= 0) return DDILU_OK;
    const int d0 = dims3[0], d1 = dims3[1], t0 = tdims3[0], t1 = tdims3[1], t2 = tdims3[2];
    if (t0 < 1 || t1 < 1 || t2 < 1 || t1 * t2 > 64 || t0 + t1 + t2 - 2 > LAT_MAX_STEPS ||
        (long long)t0 * t1 * t2 > LAT_MAX_ROWS)
        return DDILU_ERR_ARG;
    if (fill)
        lattice_build<true><<<n_tiles, LAT_MAX_ROWS, 0, ST(stream)>>>(n_tiles, tsched, tile_pos, tile_ptr, trows,
                                                                      tile_of, row_ptr, col_idx, values, nodes, d0, d1,
                                                                      t0, t1, t2, upper, has_diag, (int4 *)tab, blk16,
                                                                      stats, blob);
    else
        lattice_build<false><<<n_tiles, LAT_MAX_ROWS, 0, ST(stream)>>>(n_tiles, tsched, tile_pos, tile_ptr, trows,
                                                                       tile_of, row_ptr, col_idx, values, nodes, d0,
                                                                       d1, t0, t1, t2, upper, has_diag, (int4 *)tab,
                                                                       blk16, stats, blob);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_lattice_max_ext(void) { return LAT_XE; }

namespace {
struct LatTuning {
    int ctas_per_sm = 0;            // 0: as many as fit (one warp per CTA)
    long long *debug = nullptr;     // optional device buffer: 8 int64 cycle counters per warp
};
LatTuning g_lat;

template <bool HAS_DIAG, int NS>
int launch_lattice(int n_tiles, const void *tab, const unsigned char *blob, int *flags, int blkmax, int tmax,
                   int xemax, const double *b, double *x, cudaStream_t st) {
    const size_t smem = lat_warp_bytes(blkmax, tmax, xemax);
    void *fn = (void *)sptrsv_lattice<HAS_DIAG, NS>;
    struct Cfg { size_t smem; int occ; };
    static std::mutex mu;
    static size_t attr = 0;
    static Cfg cache[8];
    static int n_cache = 0;
    int occ = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        int hit = -1;
        for (int i = 0; i < n_cache; ++i)
            if (cache[i].smem == smem) hit = i;
        if (hit < 0) {
            if (attr < smem) {
                DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                attr = smem;
            }
            int o = 0;
            DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32, smem));
            hit = n_cache < 8 ? n_cache++ : 7;
            cache[hit] = {smem, o};
        }
        occ = cache[hit].occ;
    }
    if (occ < 1) return DDILU_ERR_ARG;
    if (g_lat.ctas_per_sm > 0 && occ > g_lat.ctas_per_sm) occ = g_lat.ctas_per_sm;
    long long grid = (long long)occ * device_info().sm_count;
    if (grid > n_tiles) grid = n_tiles;
    DDILU_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)n_tiles, st));
    const int4 *tabp = (const int4 *)tab;
    long long *dbg = g_lat.debug;
    void *args[] = {&n_tiles, &tabp, &blob, &flags, &blkmax, &tmax, &xemax, &dbg, &b, &x};
    // cooperative: a warp waits on tiles of other warps, all CTAs must be resident
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, 32, args, smem, st));
    return DDILU_OK;
}
}  // namespace

extern "C" long long ddilu_lattice_smem_bytes(int blkmax, int tmax, int xemax) {
    return (long long)lat_warp_bytes(blkmax, tmax, xemax);
}

extern "C" int ddilu_lattice_set_debug(long long *buf) {
    g_lat.debug = buf;
    return DDILU_OK;
}

extern "C" int ddilu_lattice_set_tuning(const char *key, int value) {
    const std::string k(key ? key : "");
    if (k == "ctas_per_sm") g_lat.ctas_per_sm = value;
    else return DDILU_ERR_ARG;
    return DDILU_OK;
}

/* x = T^-1 b on the lattice layout; n_slots = 1 (<= 32 lines per tile) or 2; blkmax / tmax / xemax = the
 * largest block (bytes), row count and boundary-value count of a tile (stats of ddilu_lattice_build) */
extern "C" int ddilu_sptrsv_lattice(int n_tiles, const void *tab, const unsigned char *blob, int *flags, int n_slots,
                                    int has_diag, int blkmax, int tmax, int xemax, const double *b, double *x,
                                    void *stream) {
    cudaStream_t st = ST(stream);
    if (n_tiles <= 0) return DDILU_OK;
    if (x == b || (n_slots != 1 && n_slots != 2) || (blkmax & 15) || xemax > LAT_XE) return DDILU_ERR_ARG;
    if (has_diag)
        return n_slots == 1 ? launch_lattice<true, 1>(n_tiles, tab, blob, flags, blkmax, tmax, xemax, b, x, st)
                            : launch_lattice<true, 2>(n_tiles, tab, blob, flags, blkmax, tmax, xemax, b, x, st);
    return n_slots == 1 ? launch_lattice<false, 1>(n_tiles, tab, blob, flags, blkmax, tmax, xemax, b, x, st)
                        : launch_lattice<false, 2>(n_tiles, tab, blob, flags, blkmax, tmax, xemax, b, x, st);
}
