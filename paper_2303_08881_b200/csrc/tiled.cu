// Tiled sparse triangular solve: the production path for factors whose rows can
// be clustered into tiles with a one-way (acyclic) tile dependency graph
// (structured problems: box tiles of the grid; checked, not assumed).
//
// Replaces sparse.py:228-272 (`_lower_solve`, `_upper_solve`) like sptrsv.cu.
// Why a second kernel: the sync-free solve pays one L2 round trip (0.4-1.9 us)
// per LEVEL because consecutive levels live in different warps / SMs.  Here a
// CTA owns a tile of <= 1024 rows and walks the tile's levels with the tile's
// part of x in SHARED memory; only the dependencies that cross a tile boundary
// travel through L2.  Roles inside a CTA (sptrsv_tiled):
//   warp 0  feeder   one cp.async.bulk (TMA) per tile of the tile's contiguous
//                    "static block" (level starts, per-warp work items, row ids,
//                    external columns, pivot pairs, values, 16-bit local column
//                    codes) into a 2-deep shared-memory ring (mbarrier), then the
//                    gather of the tile's right-hand side INTO its x slots
//   warp 1  poller   polls the tile's boundary dependencies in L2 (x is preset to
//                    an all-ones NaN: the value is its own flag), in the order
//                    the levels need them
//   warps 2-5 compute: level l is cut into chunks of 32 rows, chunk c belongs to
//                    warp (l + c) mod 4; a warp holds its NEXT chunk's operands
//                    in registers, syncs on the named barrier of the level
//                    before, runs  x loads -> multiply/subtract chain -> store,
//                    ARRIVES at this level's barrier (and at those of the levels
//                    it skips) and only then sends the results to L2
// Row sums keep the storage order of the reference: bit-exact.
//
// Deadlock freedom: tiles are listed in a topological order of the tile graph,
// CTA c takes tiles c, c+G, c+2G, ... in that order and the launch is
// cooperative (all CTAs co-resident); the lowest unfinished tile of the list is
// always the current tile of its CTA and all its producers are finished.
//
// Algorithmic bytes: 12*nnz + 4*(n+1) + 16n; this layout moves
// 10*nnz + 4n (row ids) + 16n (+ 4 per boundary dependency).
#include <stdint.h>

#include "common.cuh"
#include <mutex>
#include "ddilu_b200.h"

namespace ddilu {

constexpr int TILE_MAX_ROWS = 1024;
constexpr int TILE_HDR_BYTES = 96;
constexpr int TILE_NW = 4;          // compute warps of the solve kernel (the item lists are cut for them)
constexpr int ITEM_SYNC = 1 << 8;   // first chunk of this warp in a level >= 1: wait for the previous level
constexpr int TILE_NBUF = 2;
constexpr int TILE_HELPERS = 64;   // warp 0: TMA + right-hand side, warp 1: external dependencies

// header ints of a static block
enum { H_T = 0, H_NLEV, H_NEXT, H_NENT, H_OFF_ROWS, H_OFF_EXT, H_OFF_PIV, H_OFF_VAL, H_OFF_CODE, H_BYTES, H_OFF_ITEMS,
       H_NITEMS = 12, H_FIRST = 16 };   // H_NITEMS..+3: items per compute warp, H_FIRST..+3: its first level

struct TiledTuning {
    int ctas_per_sm = 0;  // 0: as many as fit
    int grid_cap = 0;     // diagnostics: at most this many CTAs
    long long *debug = nullptr;  // optional device buffer: 8 int64 per CTA of cycle counters (scripts/probe_tiled.py)
};
static TiledTuning g_tiled;
// timing probes of the rotating kernel (scripts/probe_tiled.py --probe): 1 = right-hand side read from CONTIGUOUS
// (wrong) addresses, 2 = every result stored to L2 twice, 4 = right-hand side gathered twice.  Flags 2 and 4 keep the
// results intact; flag 1 does not (timing only).  They measure how much the scattered 8-byte accesses cost.
__device__ int d_tile_probe = 0;


#define GRID_STRIDE_Q(i, n) \
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

__global__ void tile_box_keys(int n, const int *__restrict__ nodes, int d0, int d1, int t0, int t1, int t2, int nb0,
                              int nb1, int nboxes, const int *__restrict__ owner, int *__restrict__ keys) {
    GRID_STRIDE_Q(i, n) {
        const int g = nodes ? nodes[i] : (int)i;
        const int c0 = g % d0, c1 = (g / d0) % d1, c2 = g / (d0 * d1);
        int key = ((c2 / t2) * nb1 + (c1 / t1)) * nb0 + (c0 / t0);
        if (owner) key += owner[g] * nboxes;
        keys[i] = key;
    }
}

// "Wavefront slab" tiles: footprint box in the first two grid coordinates x a range of `delta` consecutive
// LEVELS of the factor.  On a wavefront-ordered stencil factor every level of such a tile holds the whole
// footprint (t0*t1 rows), so a tile of t0*t1*delta rows has only delta levels (a t^3 box has 3t-2).
#ifdef DDILU_EXPERIMENTS   // wavefront-slab tiles
__global__ void tile_slab_keys(int n, const int *__restrict__ nodes, int d0, int d1, int t0, int t1, int nb0, int nb1,
                               const int *__restrict__ lev, int delta, int n_slabs, const int *__restrict__ owner,
                               int *__restrict__ keys) {
    GRID_STRIDE_Q(i, n) {
        const int g = nodes ? nodes[i] : (int)i;
        const int c0 = g % d0, c1 = (g / d0) % d1;
        int key = (c1 / t1) * nb0 + (c0 / t0);
        if (owner) key += owner[g] * (nb0 * nb1);
        keys[i] = key * n_slabs + lev[i] / delta;
    }
}

#endif  // DDILU_EXPERIMENTS
__global__ void tile_heads(int n, const int *__restrict__ skeys, int *__restrict__ flags) {
    GRID_STRIDE_Q(q, n) flags[q] = (q == 0 || skeys[q] != skeys[q - 1]) ? 1 : 0;
}

__global__ void tile_assign(int n, const int *__restrict__ skeys, const int *__restrict__ scan,
                            const int *__restrict__ srows, int *__restrict__ tile_of, int *__restrict__ tpos,
                            int *__restrict__ tile_ptr) {
    GRID_STRIDE_Q(q, n) {
        const bool head = q == 0 || skeys[q] != skeys[q - 1];
        const int tid = scan[q] + (head ? 0 : -1);
        const int row = srows[q];
        tile_of[row] = tid;
        tpos[row] = (int)q;
        if (head) tile_ptr[tid] = (int)q;
        if (q == n - 1) tile_ptr[tid + 1] = n;
    }
}

// cross-tile dependencies as (producer tile, consumer tile) pairs
template <bool FILL>
__global__ void tile_edges(int n, const int *__restrict__ rp, const int *__restrict__ ci, int upper,
                           const int *__restrict__ tile_of, int *__restrict__ cnt, const int *__restrict__ off,
                           int2 *__restrict__ edges) {
    GRID_STRIDE_Q(i, n) {
        const int row = (int)i, t = tile_of[row];
        int c = 0, last = -1;
        long long o = FILL ? off[row] : 0;
        for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (upper ? j > row : j < row) {
                const int tj = tile_of[j];
                if (tj != t && tj != last) {   // runs of the same producer tile collapse
                    if (FILL) edges[o + c] = make_int2(tj, t);
                    ++c;
                    last = tj;
                }
            }
        }
        if (!FILL) cnt[row] = c;
    }
}

// one relaxation sweep of tlev[consumer] = max(tlev[consumer], tlev[producer] + 1)
__global__ void tile_relax(long long n_edges, const int2 *__restrict__ edges, int n_tiles, int *tlev, int *flags) {
    GRID_STRIDE_Q(e, n_edges) {
        const int2 ed = edges[e];
        const int s = tlev[ed.x] + 1;
        if (s > tlev[ed.y]) {
            if (s >= n_tiles) {
                flags[1] = 1;   // a path longer than the number of tiles: the tile graph has a cycle
            } else {
                atomicMax(tlev + ed.y, s);
                flags[0] = 1;
            }
        }
    }
}

__device__ __forceinline__ int block_excl_scan(int v, int *total, int *wsum) {
    // 1024 threads; wsum: 33 ints of shared memory
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();   // wsum may still be read from a previous call
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

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ int pad16(int bytes) { return (bytes + 15) & ~15; }

// One CTA (1024 threads, one per row) per tile, tiles in schedule order.
//   COUNT (FILL = false): size of the tile's static block -> blk16[q] (16-byte units), maxima -> stats
//   FILL: writes the static block at blob + 16 * blk16[q]
// The rows of a tile are sorted by (global level of the factor, local index): rows of
// one level never depend on each other, so the distinct levels met in a tile are its
// local levels.
template <bool FILL>
__global__ void __launch_bounds__(TILE_MAX_ROWS)
tile_build(int n_tiles, const int *__restrict__ tsched, const int *__restrict__ tile_ptr,
           const int *__restrict__ trows, const int *__restrict__ tile_of, const int *__restrict__ tpos,
           const int *__restrict__ rp, const int *__restrict__ ci, const double *__restrict__ val,
           const int *__restrict__ glev, int upper, int has_diag, int nw, int *blk16, int *stats,
           unsigned char *blob) {
    __shared__ int s_key[TILE_MAX_ROWS];     // level of local row i, later level index of slot s
    __shared__ int s_slot[TILE_MAX_ROWS];    // slot of local row i
    __shared__ int s_skey[TILE_MAX_ROWS];    // level key of slot s
    __shared__ int s_lstart[TILE_MAX_ROWS + 1];
    __shared__ int s_lk[TILE_MAX_ROWS];      // widest row of level l
    __shared__ int s_lent[TILE_MAX_ROWS + 1];
    __shared__ int s_eoff[TILE_MAX_ROWS + 1];
    __shared__ int s_wsum[33];
    const int q = blockIdx.x;
    const int t = tsched[q];
    const int base = tile_ptr[t], T = tile_ptr[t + 1] - base;
    const int i = threadIdx.x;
    const bool active = i < T;
    const int row = active ? trows[base + i] : -1;
    const int key = active ? glev[row] : 0x7FFFFFFF;
    s_key[i] = key;
    s_lk[i] = 0;
    __syncthreads();
    // rank = slot
    int slot = 0;
    if (active) {
        for (int j = 0; j < T; ++j) {
            const int kj = s_key[j];
            slot += (kj < key || (kj == key && j < i)) ? 1 : 0;
        }
        s_slot[i] = slot;
        s_skey[slot] = key;
    }
    __syncthreads();
    // level index of every slot
    int total;
    const int head = (i < T && (i == 0 || s_skey[i] != s_skey[i - 1])) ? 1 : 0;
    const int lidx_of_slot_i = block_excl_scan(head, &total, s_wsum) + head - 1;
    const int n_lev = total;
    if (i < T) {
        if (head) s_lstart[lidx_of_slot_i] = i;
        s_key[i] = lidx_of_slot_i;   // s_key now: level index by SLOT
    }
    if (i == 0) s_lstart[n_lev] = T;
    __syncthreads();
    // dependencies of my row
    int nd = 0, ne = 0;
    const int my_l = active ? s_key[slot] : 0;
    if (active) {
        for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (upper ? j > row : j < row) {
                ++nd;
                if (tile_of[j] != t) ++ne;
            }
        }
        atomicMax(&s_lk[my_l], nd);
        s_eoff[slot] = ne;
    }
    __syncthreads();
    // external offsets by slot
    const int ne_slot = i < T ? s_eoff[i] : 0;
    int n_ext;
    const int eoff_i = block_excl_scan(ne_slot, &n_ext, s_wsum);
    __syncthreads();
    if (i < T) s_eoff[i] = eoff_i;
    if (i == 0) s_eoff[T] = n_ext;
    // entry offsets by level
    const int lw = i < n_lev ? s_lk[i] * (s_lstart[i + 1] - s_lstart[i]) : 0;
    int n_ent;
    const int lent_i = block_excl_scan(lw, &n_ent, s_wsum);
    if (i < n_lev) s_lent[i] = lent_i;
    if (i == 0) s_lent[n_lev] = n_ent;
    __syncthreads();
    // work items: level l is cut into chunks of 32 rows, chunk c belongs to compute warp (l + c) mod 4;
    // every warp gets the ordered list of its chunks, so the solve kernel never scans level tables
    // (nw = 4: the rotating-warp kernel; nw = 1: the warp-per-tile kernel, one list in (level, chunk) order)
    int cntw[TILE_NW], basew[TILE_NW], totw[TILE_NW];
#pragma unroll
    for (int cwp = 0; cwp < TILE_NW; ++cwp) {
        cntw[cwp] = 0;
        if (i < n_lev && cwp < nw) {
            const int nch = (s_lstart[i + 1] - s_lstart[i] + 31) >> 5;
            const int c0 = (cwp - i) & (nw - 1);
            cntw[cwp] = c0 < nch ? (nch - c0 + nw - 1) / nw : 0;
        }
    }
#pragma unroll
    for (int cwp = 0; cwp < TILE_NW; ++cwp) basew[cwp] = block_excl_scan(cntw[cwp], &totw[cwp], s_wsum);
    const int n_items = totw[0] + totw[1] + totw[2] + totw[3];
    // layout.  nw == 0 ("lean", rows with <= 3 dependencies only): no work items; per level {slot start,
    // externals needed}, per slot two 16-byte records {a0, a1} and {a2, x-slot indices 0..2} (padding:
    // coefficient 0, the tile's zero slot), 32 spare records so that idle lanes may read past a level.
    const bool lean = nw == 0;
    const int off_lst = TILE_HDR_BYTES;
    const int off_items = off_lst + pad16((lean ? 8 : 4) * (n_lev + 1));
    const int off_rows = off_items + (lean ? 0 : 32 * n_items);
    const int off_ext = off_rows + pad16(4 * T);
    const int off_piv = off_ext + pad16(4 * n_ext);
    const int off_val = off_piv + (has_diag ? 16 * T : 0);   // (pivot, reciprocal) pairs
    const int off_code = off_val + (lean ? 16 * (T + 32) : pad16(8 * n_ent));
    const int bytes = off_code + (lean ? 16 * (T + 32) : pad16(2 * n_ent));
    if (!FILL) {
        if (i == 0) {
            blk16[q] = bytes >> 4;
            atomicMax(stats + 0, T);
            atomicMax(stats + 1, n_ext);
            atomicMax(stats + 2, bytes);
        }
        if (i < n_lev) atomicMax(stats + 4, s_lk[i]);
        return;
    }
    unsigned char *blk = blob + 16LL * blk16[q];
    int *hdr = (int *)blk;
    // first level with a chunk of warp cwp after level `from` (n_lev + 1 if none)
    auto next_level_of = [&](int cwp, int from) {
        for (int l = from; l < n_lev; ++l) {
            const int nch = (s_lstart[l + 1] - s_lstart[l] + 31) >> 5;
            if (((cwp - l) & (nw - 1)) < nch) return l;
        }
        return n_lev + 1;
    };
    if (i < TILE_HDR_BYTES / 4) {
        int v = 0;
        switch (i) {
            case H_T: v = T; break;
            case H_NLEV: v = n_lev; break;
            case H_NEXT: v = n_ext; break;
            case H_NENT: v = n_ent; break;
            case H_OFF_ROWS: v = off_rows; break;
            case H_OFF_EXT: v = off_ext; break;
            case H_OFF_PIV: v = has_diag ? off_piv : 0; break;
            case H_OFF_VAL: v = off_val; break;
            case H_OFF_CODE: v = off_code; break;
            case H_BYTES: v = bytes; break;
            case H_OFF_ITEMS: v = off_items; break;
            default: break;
        }
        if (i >= H_NITEMS && i < H_NITEMS + TILE_NW) v = totw[i - H_NITEMS];
        if (i >= H_FIRST && i < H_FIRST + nw) v = next_level_of(i - H_FIRST, 0);
        hdr[i] = v;
    }
    if (lean) {
        int2 *lvl2 = (int2 *)(blk + off_lst);
        if (i <= n_lev) lvl2[i] = make_int2(s_lstart[i], i < n_lev ? s_eoff[s_lstart[i + 1]] : n_ext);
        double2 *recA = (double2 *)(blk + off_val);
        uint4 *recB = (uint4 *)(blk + off_code);
        if (i < 32) {   // spare records
            recA[T + i] = make_double2(0.0, 0.0);
            recB[T + i] = make_uint4(0u, 0u, 0u, 0u);
        }
        {
            const int tails[3][2] = {{off_lst + 8 * (n_lev + 1), off_rows}, {off_rows + 4 * T, off_ext},
                                     {off_ext + 4 * n_ext, off_piv}};
            if (i < 3)
                for (int p = tails[i][0]; p < tails[i][1]; ++p) blk[p] = 0;
        }
        if (!active) return;
        ((int *)(blk + off_rows))[slot] = row;
        int *ext_out = (int *)(blk + off_ext);
        const unsigned zs = (unsigned)(T + n_ext);
        double av[3] = {0.0, 0.0, 0.0};
        unsigned ix[3] = {zs, zs, zs};
        int kk = 0, e = s_eoff[slot];
        double diag = 1.0;
        bool seen = false;
        for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
            const int j = ci[k];
            if (upper ? j > row : j < row) {
                unsigned code;
                if (tile_of[j] == t) {
                    code = (unsigned)s_slot[tpos[j] - base];
                } else {
                    code = (unsigned)(T + e);
                    ext_out[e] = j;
                    ++e;
                }
                if (kk < 3) {
                    av[kk] = val[k];
                    ix[kk] = code;
                }
                ++kk;
            } else if (j == row) {
                diag = val[k];
                seen = true;
            }
        }
        recA[slot] = make_double2(av[0], av[1]);
        recB[slot] = make_uint4((unsigned)__double2loint(av[2]), (unsigned)__double2hiint(av[2]), ix[0] | (ix[1] << 16),
                                ix[2]);
        if (has_diag) {
            ((double2 *)(blk + off_piv))[slot] = make_double2(diag, safe_reciprocal(diag));
            if (!seen || fabs(diag) < 1e-300) atomicMin(stats + 3, row);
        }
        return;
    }
    int *lst = (int *)(blk + off_lst);
    if (i <= n_lev) lst[i] = s_lstart[i];
    if (i < n_lev) {
        const int l0 = s_lstart[i], wl = s_lstart[i + 1] - l0, nch = (wl + 31) >> 5;
        const int need = s_eoff[s_lstart[i + 1]];   // externals needed by the levels up to and including this one
        int wbase = 0;
#pragma unroll
        for (int cwp = 0; cwp < TILE_NW; ++cwp) {
            if (cwp >= nw) break;
            int4 *it = (int4 *)(blk + off_items) + 2 * (wbase + basew[cwp]);
            const int c0 = (cwp - i) & (nw - 1);
            int nth = 0;
            for (int c = c0; c < nch; c += nw, ++nth) {
                const bool first = c == c0, last = c + nw >= nch;
                int n_arr = 0;
                if (last) {
                    const int nxt = next_level_of(cwp, i + 1);
                    n_arr = nxt > n_lev ? n_lev - i : nxt - 1 - i;
                }
                const int cnt = wl - c * 32 < 32 ? wl - c * 32 : 32;
                const int flags = cnt | ((first && i >= 1) ? ITEM_SYNC : 0);
                it[2 * nth] = make_int4(l0 + c * 32, s_lent[i] + c * 32, wl, s_lk[i]);
                it[2 * nth + 1] = make_int4(i, need, flags, n_arr);
            }
            wbase += totw[cwp];
        }
    }
    // zero the alignment tails so the blob is fully defined
    {
        const int tails[6][2] = {{off_lst + 4 * (n_lev + 1), off_items}, {off_rows + 4 * T, off_ext},
                                 {off_ext + 4 * n_ext, off_piv}, {off_val, off_val},
                                 {off_val + 8 * n_ent, off_code}, {off_code + 2 * n_ent, bytes}};
        if (i < 6)
            for (int p = tails[i][0]; p < tails[i][1]; ++p) blk[p] = 0;
    }
    if (!active) return;
    int *rows_out = (int *)(blk + off_rows);
    int *ext_out = (int *)(blk + off_ext);
    double *piv_out = (double *)(blk + off_piv);
    double *val_out = (double *)(blk + off_val);
    unsigned short *code_out = (unsigned short *)(blk + off_code);
    rows_out[slot] = row;
    const int l0 = s_lstart[my_l], w = s_lstart[my_l + 1] - l0, K = s_lk[my_l];
    const long long e0 = (long long)s_lent[my_l] + (slot - l0);
    int kk = 0, e = s_eoff[slot];
    double diag = 1.0;
    bool seen = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (upper ? j > row : j < row) {
            int code;
            if (tile_of[j] == t) {
                code = s_slot[tpos[j] - base];
            } else {
                code = T + e;
                ext_out[e] = j;
                ++e;
            }
            code_out[e0 + (long long)kk * w] = (unsigned short)code;
            val_out[e0 + (long long)kk * w] = val[k];
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {   // padding: coefficient 0 times the tile's zero slot (x[T + n_ext] = 0)
        code_out[e0 + (long long)kk * w] = (unsigned short)(T + n_ext);
        val_out[e0 + (long long)kk * w] = 0.0;
    }
    if (has_diag) {
        ((double2 *)piv_out)[slot] = make_double2(diag, safe_reciprocal(diag));
        if (!seen || fabs(diag) < 1e-300) atomicMin(stats + 3, row);
    }
}

// ---------------------------------------------------------------------------
// solve

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void level_arrive(int l, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(1 + (l & (TILE_NW - 1))), "r"(threads) : "memory");
}
__device__ __forceinline__ void level_sync(int l, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (l & (TILE_NW - 1))), "r"(threads) : "memory");
}

struct TileCtl {
    uint64_t mbar[TILE_NBUF];
    unsigned long long ext_prog[2];   // (tile ordinal << 32) | externals delivered
    int b_ready[2];                   // tile ordinal + 1 whose right-hand side sits in bs[buf]
    int comp_done;                    // tiles finished by the compute warps
    int poll_done;                    // tiles whose boundary dependencies the poller has delivered
    int pad[3];
};

__global__ void fastdiv_selftest(long long n, unsigned long long seed, unsigned long long *mismatch) {
    unsigned long long bad = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        // splitmix64 stream per sample
        unsigned long long z = seed + 0x9E3779B97F4A7C15ULL * (unsigned long long)(i + 1);
        auto next = [&]() {
            z += 0x9E3779B97F4A7C15ULL;
            unsigned long long x = z;
            x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
            x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
            return x ^ (x >> 31);
        };
        unsigned long long ms = next(), md = next(), m = next();
        // exponents: mostly near 1, sometimes anywhere (incl. subnormal / inf / nan), sometimes at the window edges
        auto expo = [&](unsigned long long r) -> unsigned long long {
            const unsigned sel = (unsigned)(r & 7);
            const unsigned v = (unsigned)(r >> 8);
            if (sel < 4) return 1023 - 40 + v % 81;
            if (sel < 6) return v % 2048;
            return (v & 1) ? 623 - 3 + (v >> 1) % 7 : 1423 - 3 + (v >> 1) % 7;
        };
        unsigned long long fs = ms & 0xFFFFFFFFFFFFFULL, fd = md & 0xFFFFFFFFFFFFFULL;
        // adversarial mantissas: all ones, all zeros, few bits, near-all-ones
        switch ((m >> 20) & 15) {
            case 0: fd = 0xFFFFFFFFFFFFFULL; break;
            case 1: fd = 0; break;
            case 2: fd = 0xFFFFFFFFFFFFFULL ^ (1ULL << (m % 52)); break;
            case 3: fd = 1ULL << (m % 52); break;
            case 4: fs = 0xFFFFFFFFFFFFFULL; break;
            case 5: fs = 0; break;
            case 6: fs = fd; break;
            case 7: fs = 0xFFFFFFFFFFFFFULL ^ (1ULL << (m % 52)); break;
            default: break;
        }
        const unsigned long long bs = ((m >> 62) & 1) << 63 | expo(m >> 24) << 52 | fs;
        const unsigned long long bd = ((m >> 63) & 1) << 63 | expo(m >> 40) << 52 | fd;
        const double sv = __longlong_as_double((long long)bs), dv = __longlong_as_double((long long)bd);
        const double ref = sv / dv;
        const double got = exact_div(sv, dv, safe_reciprocal(dv));
        const long long br = __double_as_longlong(ref), bg = __double_as_longlong(got);
        if (br != bg && !(ref != ref && got != got)) ++bad;   // NaN payloads may differ, values may not
    }
    if (bad) atomicAdd(mismatch, bad);
}

// One work item (a chunk of <= 32 rows of one level) as a compute warp holds it one item ahead:
// everything that does not depend on x is in registers before the level's barrier opens.
template <int KP>
struct TileItem {
    int level, need, flags, n_arr;   // flags: rows in the chunk | ITEM_SYNC
    int ent0, w, K;                  // entry k of lane i: ent0 + k*w + i (long rows, k >= KP)
    uint32_t xaddr[KP];              // shared-memory byte address of the x operand of entry k
    uint32_t saddr;                  // where this lane's result goes
    int bar;                         // hardware barrier id of this item's level
    int row;                         // global row of this lane's result (-1: idle lane)
    double a[KP];
    double rhs, piv, rinv;
};

template <bool HAS_DIAG, int KP>
__device__ __forceinline__ void tile_item_load(TileItem<KP> &r, const int4 *it, int lane,
                                               const double *xsk, int zslot, const double *piv, const int *rows,
                                               const unsigned short *codes, const double *vals) {
    const int4 A = it[0], B = it[1];   // A = {slot0, ent0, w, K}, B = {level, need, flags, n_arr}
    r.level = B.x;
    r.need = B.y;
    r.flags = B.z;
    r.n_arr = B.w;
    r.ent0 = A.y;
    r.w = A.z;
    r.K = A.w;
    const bool act = lane < (B.z & 0xff);
    const int s = A.x + lane;
    r.saddr = smem_u32(xsk + (act ? s : zslot + 1));   // idle lanes store into a scratch slot: no predicate on the chain
    r.row = act ? rows[s] : -1;
    r.rhs = act ? xsk[s] : 1.0;   // the feeder parked b[row] in the row's own x slot (idle lanes: keep the
                                  // division on its fast path)
    const double2 pr = (HAS_DIAG && act) ? ((const double2 *)piv)[s] : make_double2(1.0, 1.0);
    r.piv = pr.x;
    r.rinv = pr.y;
    r.bar = 1 + (B.x & (TILE_NW - 1));
#pragma unroll
    for (int u = 0; u < KP; ++u) {
        const bool in = act && u < A.w;
        const int c = in ? (int)codes[A.y + u * A.z + lane] : zslot;
        r.a[u] = in ? vals[A.y + u * A.z + lane] : 0.0;
        r.xaddr[u] = smem_u32(xsk + c);
    }
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// LONG: some row of the factor has more than KP dependencies (compiled out for 7-point ILU(0) factors)
template <bool HAS_DIAG, int KP, bool LONG>
__global__ void __launch_bounds__(TILE_HELPERS + TILE_NW * 32)
sptrsv_tiled(int n_tiles, const int *__restrict__ blk_off16, const unsigned char *__restrict__ blob, int stat_max,
             int tmax, int emax, long long *dbg, const double *__restrict__ b, double *x) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *stat = smem;
    double *xs = (double *)(smem + (size_t)TILE_NBUF * stat_max);
    const int xstride = tmax + emax + 2;   // + the zero slot that padded entries point to
    TileCtl *ctl = (TileCtl *)(xs + 2 * (size_t)xstride);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int nk = (n_tiles - (int)blockIdx.x + G - 1) / G;   // my tiles: blockIdx.x + k*G
    if (tid == 0) {
        for (int s = 0; s < TILE_NBUF; ++s) mbar_init(&ctl->mbar[s], 1);
        ctl->ext_prog[0] = ctl->ext_prog[1] = 0ULL;
        ctl->b_ready[0] = ctl->b_ready[1] = 0;
        ctl->comp_done = 0;
        ctl->poll_done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    volatile int *comp_done = &ctl->comp_done;
    volatile int *poll_done = &ctl->poll_done;

    if (warp == 0) {
        // ---------------- feeder: TMA of the static blocks + right-hand side gather
        auto issue = [&](int k) {
            const long long qq = (long long)blockIdx.x + (long long)k * G;
            const int o0 = blk_off16[qq], o1 = blk_off16[qq + 1];
            const uint32_t bytes = (uint32_t)(o1 - o0) << 4;
            uint64_t *bar = &ctl->mbar[k % TILE_NBUF];
            mbar_expect_tx(bar, bytes);
            bulk_g2s(stat + (size_t)(k % TILE_NBUF) * stat_max, blob + 16LL * o0, bytes, bar);
        };
        // Tile j needs: its ring slot and x buffer free (tile j-2 computed and its boundary values
        // delivered), then the TMA of its static block, then the right-hand side gathered INTO its x slots.
        // All of that happens while tile j-1 is being computed.  The waits sleep (the ncu profile of the
        // first version showed 40 % of all issued instructions in helper-warp spin loops, and the kernel is
        // issue-bound).
        for (int j = 0; j < nk; ++j) {
            if (j >= 2)
                while (*comp_done < j - 1 || *poll_done < j - 1) __nanosleep(600);
            if (lane == 0) issue(j);
            mbar_wait(&ctl->mbar[j % TILE_NBUF], (uint32_t)((j / TILE_NBUF) & 1));
            const unsigned char *blk = stat + (size_t)(j % TILE_NBUF) * stat_max;
            const int *hdr = (const int *)blk;
            const int T = hdr[H_T];
            const int *rows = (const int *)(blk + hdr[H_OFF_ROWS]);
            double *xsk = xs + (size_t)(j & 1) * xstride;   // slot s holds b[row] until the row is solved
            const int probe = d_tile_probe;
            const long long fake0 = ((long long)blockIdx.x + (long long)j * G) * 448;
            for (int s0 = 0; s0 < T; s0 += 256) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int s = s0 + u * 32 + lane;
                    v[u] = s < T ? __ldg(b + ((probe & 1) ? fake0 + s : (long long)rows[s])) : 0.0;
                }
                if (probe & 4) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int s = s0 + u * 32 + lane;
                        if (s < T) v[u] += 0.0 * ld_l2(b + rows[s]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int s = s0 + u * 32 + lane;
                    if (s < T) xsk[s] = v[u];
                }
            }
            __syncwarp();
            __threadfence_block();
            if (lane == 0) *(volatile int *)&ctl->b_ready[j & 1] = j + 1;
        }
    } else if (warp == 1) {
        // ---------------- poller: boundary dependencies, in the order the levels need them
        for (int k = 0; k < nk; ++k) {
            if (k >= 2)
                while (*comp_done < k - 1) __nanosleep(600);   // x buffer of tile k-2 still in use
            mbar_wait(&ctl->mbar[k % TILE_NBUF], (uint32_t)((k / TILE_NBUF) & 1));
            const unsigned char *blk = stat + (size_t)(k % TILE_NBUF) * stat_max;
            const int *hdr = (const int *)blk;
            const int T = hdr[H_T], n_ext = hdr[H_NEXT];
            const int *ext = (const int *)(blk + hdr[H_OFF_EXT]);
            double *xe = xs + (size_t)(k & 1) * xstride + T;
            volatile unsigned long long *prog = &ctl->ext_prog[k & 1];
            for (int base = 0; base < n_ext; base += 128) {
                int c[4];
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = base + u * 32 + lane;
                    c[u] = e < n_ext ? ext[e] : -1;
                }
                // all polls of the chunk in flight together; delivered and published 32 at a time, in order
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = c[u] >= 0 ? ld_l2(x + c[u]) : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (base + u * 32 < n_ext) {
                        if (c[u] >= 0) {
                            while (is_sentinel(v[u])) v[u] = ld_l2(x + c[u]);
                            xe[base + u * 32 + lane] = v[u];
                        }
                        __syncwarp();
                        __threadfence_block();
                        const int upto = base + (u + 1) * 32 < n_ext ? base + (u + 1) * 32 : n_ext;
                        if (lane == 0) *prog = ((unsigned long long)(unsigned)k << 32) | (unsigned)upto;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) *poll_done = k + 1;
        }
    } else {
        // ---------------- compute warps
        // Level l of a tile is cut into chunks of 32 rows; chunk c goes to compute warp (l + c) mod 4.
        // Every level has a chunk 0, so a warp works at least every 4th level and is otherwise free
        // to prefetch its next chunk (TilePre) while the other warps compute.  Barrier B_l (hardware
        // id 1 + l mod 4) completes when every warp has passed level l: a warp ARRIVES (non-blocking)
        // at the levels it skips and SYNCS only on the level right before its next chunk, so the
        // per-level critical path is  wake-up -> x loads -> multiply/subtract chain -> store -> arrive.
        const int cw = warp - TILE_HELPERS / 32;
        constexpr int NC = TILE_NW * 32;
        const bool probe2 = (d_tile_probe & 2) != 0;
        long long t_start = 0, t_wait_tile = 0, t_wait_ext = 0, t_levels = 0, n_lv = 0;
        if (dbg) t_start = clock64();
        for (int k = 0; k < nk; ++k) {
            long long t0 = 0;
            if (dbg) t0 = clock64();
            mbar_wait(&ctl->mbar[k % TILE_NBUF], (uint32_t)((k / TILE_NBUF) & 1));
            while (*(volatile int *)&ctl->b_ready[k & 1] != k + 1) __nanosleep(200);
            asm volatile("" ::: "memory");
            if (dbg) t_wait_tile += clock64() - t0;
            const unsigned char *blk = stat + (size_t)(k % TILE_NBUF) * stat_max;
            const int *hdr = (const int *)blk;
            const int n_lev = hdr[H_NLEV];
            const int *rows = (const int *)(blk + hdr[H_OFF_ROWS]);
            const double *piv = (const double *)(blk + hdr[H_OFF_PIV]);
            const double *vals = (const double *)(blk + hdr[H_OFF_VAL]);
            const unsigned short *codes = (const unsigned short *)(blk + hdr[H_OFF_CODE]);
            double *xsk = xs + (size_t)(k & 1) * xstride;
            const int zslot = hdr[H_T] + hdr[H_NEXT];
            volatile unsigned long long *prog = &ctl->ext_prog[k & 1];
            int n_it = 0, it_base = 0;
#pragma unroll
            for (int q = 0; q < TILE_NW; ++q) {
                const int nq = hdr[H_NITEMS + q];
                if (q < cw) it_base += nq;
                if (q == cw) n_it = nq;
            }
            const int4 *items = (const int4 *)(blk + hdr[H_OFF_ITEMS]) + 2 * it_base;
            const int first = hdr[H_FIRST + cw];
            if (lane == 0) xsk[zslot] = 0.0;   // every warp writes the same value; its own reads follow in order
            __syncwarp();
            // levels before my first chunk (all levels if I have none): arrive at once
            for (int l = 0; l <= (n_it ? first - 2 : n_lev - 1); ++l) level_arrive(l, NC);
            TileItem<KP> itm;
            if (n_it) tile_item_load<HAS_DIAG, KP>(itm, items, lane, xsk, zslot, piv, rows, codes, vals);
            int have = 0;
            for (int q = 0; q < n_it; ++q) {
                if (itm.flags & ITEM_SYNC) level_sync(itm.level - 1, NC);
                if (itm.need > have) {
                    long long t1 = 0;
                    if (dbg) t1 = clock64();
                    const unsigned long long want = ((unsigned long long)(unsigned)k << 32) | (unsigned)itm.need;
                    unsigned long long got = *prog;
                    while (got < want) got = *prog;
                    have = (int)(got & 0xffffffffULL);
                    if (dbg) t_wait_ext += clock64() - t1;
                }
                // ---- the level's critical path: x loads -> multiply/subtract chain -> store -> arrive
                double xv[KP];
#pragma unroll
                for (int u = 0; u < KP; ++u) xv[u] = lds_f64(itm.xaddr[u]);
                double sum = itm.rhs;
#pragma unroll
                for (int u = 0; u < KP; ++u) sum -= itm.a[u] * xv[u];
                if (LONG && itm.K > KP) {   // long rows: the remaining entries straight from the static block
                    const unsigned short *cp = codes + itm.ent0 + lane;
                    const double *vp = vals + itm.ent0 + lane;
                    if (lane < (itm.flags & 0xff))
                        for (int kk = KP; kk < itm.K; ++kk) sum -= vp[kk * itm.w] * xsk[cp[kk * itm.w]];
                }
                if (HAS_DIAG) sum = exact_div(sum, itm.piv, itm.rinv);
                sts_f64(itm.saddr, sum);
                // release this level and every level I skip right away; then the next item's prefetch,
                // off everybody's critical path
                asm volatile(
                    "{\n .reg .pred p;\n setp.gt.s32 p, %2, 0;\n @p bar.arrive %0, %1;\n}" ::"r"(itm.bar), "r"(NC),
                    "r"(itm.n_arr)
                    : "memory");   // predicated: no branch between the store and the arrive
                for (int j = 1; j < itm.n_arr; ++j) level_arrive(itm.level + j, NC);
                // publish to L2 AFTER the arrives: a barrier operation issued behind a global store waits for
                // the store (an L2 round trip); this warp's next barrier operation is >= 1 level away
                if (itm.row >= 0) st_l2(x + itm.row, scrub_sentinel(sum));
                if (probe2 && itm.row >= 0) st_l2(x + itm.row, scrub_sentinel(sum));
                if (q + 1 < n_it)
                    tile_item_load<HAS_DIAG, KP>(itm, items + 2 * (q + 1), lane, xsk, zslot, piv, rows, codes, vals);
            }
            asm volatile("bar.sync 5, %0;" ::"r"(NC) : "memory");   // tile finished by every compute warp
            if (dbg) {
                t_levels += clock64() - t0;
                n_lv += n_lev;
            }
            if (cw == 0 && lane == 0) {
                __threadfence_block();
                *comp_done = k + 1;
            }
        }
        if (dbg && lane == 0)   // boundary waits of ALL compute warps (each level's wait is seen by its owner only)
            atomicAdd((unsigned long long *)(dbg + 8LL * blockIdx.x + 6), (unsigned long long)t_wait_ext);
        if (dbg && cw == 0 && lane == 0) {
            long long *o = dbg + 8LL * blockIdx.x;
            o[0] = clock64() - t_start;   // whole CTA life
            o[1] = t_wait_tile;           // waiting for the static block / right-hand side
            o[2] = t_wait_ext;            // waiting for boundary dependencies (at this warp's levels)
            o[3] = t_levels;              // tile time including both waits
            o[4] = n_lv;
            o[5] = nk;
        }
    }
}

#ifdef DDILU_EXPERIMENTS   // warp-per-tile and lean kernels: measured slower
// ---------------------------------------------------------------------------
// Warp-per-tile variant (tiles whose levels are mostly <= 32 rows wide: 8x8x4 interior boxes, 16x16
// interface patches).  Every WARP owns a stream of tiles and is completely independent of the other
// warps of its CTA: its own 2-deep TMA ring, its own x slots, no named barrier, no helper warps.  A level
// is one `__syncwarp()` away from the next, the operands of the next chunk are loaded (shared memory ->
// registers) before the current chain starts, finished rows go straight to L2 (no barrier follows a
// global store here), boundary dependencies are polled 32 at a time with the next batch already in
// flight.  Latencies that a warp cannot hide itself (right-hand-side gather, TMA, polls) are hidden by
// the other 6-9 resident warps of the SM, which is what the rotating-warp kernel could not do: it keeps
// at most 4 level chains per SM in flight, this one 7-9.
// Execution barrier of a warp WITHOUT the memory-fence semantics of __syncwarp(): a shuffle makes the
// lanes converge, and shared-memory accesses of one warp are performed in issue order, so the level's
// STS are visible to the next level's LDS.  (__syncwarp / bar.warp.sync additionally waits until the
// lanes' outstanding GLOBAL stores are performed -- an L2 round trip per level, measured.)
__device__ __forceinline__ void warp_converge() {
    int t = 0;
    asm volatile("shfl.sync.idx.b32 %0, %0, 0, 0x1f, 0xffffffff;" : "+r"(t)::"memory");
}

// Boundary dependencies of a warp's tile.  At tile start every dependency is polled ONCE, 8 per lane in
// flight (the producers are usually long finished): the value -- or the not-ready pattern -- goes to the
// tile's x slots.  A level that needs dependency e < need re-polls only what is still missing.
__device__ __forceinline__ void ext_prefetch(const double *x, const int *ext, int n_ext, double *xe, int lane) {
    for (int e0 = 0; e0 < n_ext; e0 += 256) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 32 + lane;
            v[u] = e < n_ext ? ld_l2(x + ext[e]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 32 + lane;
            if (e < n_ext) xe[e] = v[u];
        }
    }
}
__device__ __forceinline__ int ext_deliver(const double *x, const int *ext, int n_ext, double *xe, int lane, int have,
                                           int need) {
    while (need > have) {
        const int e = have + lane;
        if (e < n_ext) {
            double v = xe[e];
            if (is_sentinel(v)) {
                do v = ld_l2(x + ext[e]); while (is_sentinel(v));
                xe[e] = v;
            }
        }
        have += 32;
    }
    warp_converge();
    return have;
}

template <int KP>
struct WarpItem {
    int need, cnt, ent0, w, K, row;
    uint32_t xaddr[KP], saddr;
    double a[KP];
    double rhs, piv, rinv;
};

template <bool HAS_DIAG, int KP>
__device__ __forceinline__ void warp_item_load(WarpItem<KP> &r, const int4 *it, int lane, const double *xsk, int zslot,
                                               const double *piv, const int *rows, const unsigned short *codes,
                                               const double *vals) {
    const int4 A = it[0], B = it[1];   // A = {slot0, ent0, w, K}, B = {level, need, flags, n_arr}
    r.need = B.y;
    r.cnt = B.z & 0xff;
    r.ent0 = A.y;
    r.w = A.z;
    r.K = A.w;
    const bool act = lane < r.cnt;
    const int s = A.x + lane;
    r.saddr = smem_u32(xsk + s);
    r.row = act ? rows[s] : 0;
    r.rhs = act ? xsk[s] : 1.0;
    const double2 pr = (HAS_DIAG && act) ? ((const double2 *)piv)[s] : make_double2(1.0, 1.0);
    r.piv = pr.x;
    r.rinv = pr.y;
#pragma unroll
    for (int u = 0; u < KP; ++u) {
        const bool in = act && u < A.w;
        const int c = in ? (int)codes[A.y + u * A.z + lane] : zslot;
        r.a[u] = in ? vals[A.y + u * A.z + lane] : 0.0;
        r.xaddr[u] = smem_u32(xsk + c);
    }
}

template <bool HAS_DIAG, int KP>
__global__ void __launch_bounds__(512)
sptrsv_warptile(int n_tiles, const int *__restrict__ blk_off16, const unsigned char *__restrict__ blob, int stat_max,
                int xcap, int per_warp, const double *__restrict__ b, double *x) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    unsigned char *base = smem + (size_t)warp * per_warp;
    unsigned char *stat = base;
    double *xs = (double *)(base + 2 * (size_t)stat_max);
    uint64_t *mbar = (uint64_t *)(xs + xcap);
    const long long gw = (long long)blockIdx.x * wpb + warp, nwt = (long long)gridDim.x * wpb;
    const int nk = gw < n_tiles ? (int)((n_tiles - gw + nwt - 1) / nwt) : 0;   // my tiles: gw + k * nwt
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int k) {
        const long long qq = gw + (long long)k * nwt;
        const int o0 = blk_off16[qq], o1 = blk_off16[qq + 1];
        const uint32_t bytes = (uint32_t)(o1 - o0) << 4;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the slot was read by this warp before
        mbar_expect_tx(&mbar[k & 1], bytes);
        bulk_g2s(stat + (size_t)(k & 1) * stat_max, blob + 16LL * o0, bytes, &mbar[k & 1]);
    };
    if (lane == 0 && nk > 0) issue(0);
    for (int k = 0; k < nk; ++k) {
        if (lane == 0 && k + 1 < nk) issue(k + 1);   // its slot held tile k-1, which this warp has finished
        mbar_wait(&mbar[k & 1], (uint32_t)((k >> 1) & 1));
        const unsigned char *blk = stat + (size_t)(k & 1) * stat_max;
        const int *hdr = (const int *)blk;
        const int T = hdr[H_T], n_ext = hdr[H_NEXT], n_it = hdr[H_NITEMS];
        const int *rows = (const int *)(blk + hdr[H_OFF_ROWS]);
        const int *ext = (const int *)(blk + hdr[H_OFF_EXT]);
        const double *piv = (const double *)(blk + hdr[H_OFF_PIV]);
        const double *vals = (const double *)(blk + hdr[H_OFF_VAL]);
        const unsigned short *codes = (const unsigned short *)(blk + hdr[H_OFF_CODE]);
        const int4 *items = (const int4 *)(blk + hdr[H_OFF_ITEMS]);
        const int zslot = T + n_ext;
        double *xe = xs + T;
        int have = 0;
        ext_prefetch(x, ext, n_ext, xe, lane);
        for (int s0 = 0; s0 < T; s0 += 256) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u * 32 + lane;
                v[u] = s < T ? __ldg(b + rows[s]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u * 32 + lane;
                if (s < T) xs[s] = v[u];
            }
        }
        if (lane == 0) xs[zslot] = 0.0;
        __syncwarp();
        WarpItem<KP> cur, nxt;
        if (n_it) warp_item_load<HAS_DIAG, KP>(cur, items, lane, xs, zslot, piv, rows, codes, vals);
        for (int q = 0; q < n_it; ++q) {
            // the next chunk never belongs to this level's consumers' producers: its right-hand side and
            // coefficients can be read now (its x operands are only ADDRESSES here)
            if (q + 1 < n_it)
                warp_item_load<HAS_DIAG, KP>(nxt, items + 2 * (q + 1), lane, xs, zslot, piv, rows, codes, vals);
            if (cur.need > have) have = ext_deliver(x, ext, n_ext, xe, lane, have, cur.need);
            double xv[KP];
#pragma unroll
            for (int u = 0; u < KP; ++u) xv[u] = lds_f64(cur.xaddr[u]);
            double sum = cur.rhs;
#pragma unroll
            for (int u = 0; u < KP; ++u) sum -= cur.a[u] * xv[u];
            if (cur.K > KP) {   // long rows: the remaining entries straight from the static block
                const unsigned short *cp = codes + cur.ent0 + lane;
                const double *vp = vals + cur.ent0 + lane;
                if (lane < cur.cnt)
                    for (int kk = KP; kk < cur.K; ++kk) sum -= vp[kk * cur.w] * xs[cp[kk * cur.w]];
            }
            if (HAS_DIAG) sum = exact_div(sum, cur.piv, cur.rinv);
            if (lane < cur.cnt) {
                sts_f64(cur.saddr, sum);
                st_l2(x + cur.row, scrub_sentinel(sum));
            }
            warp_converge();
            cur = nxt;
        }
    }
}

// ---------------------------------------------------------------------------
// Lean warp-per-tile kernel for factors whose rows have at most 3 dependencies (ILU(0) of 7-point
// problems: the headline workload).  Same execution model as sptrsv_warptile (independent warps, own TMA
// ring, own x slots, no barriers), but the static block holds PRE-DIGESTED 16-byte records per row
// ({a0, a1}, {a2, three 16-bit x-slot indices}) so that a level costs ~40 instructions: a lone warp issues
// dependent instructions at ~6-8 cycles each, so the instruction count IS the per-level latency.
template <bool HAS_DIAG>
__global__ void __launch_bounds__(512)
sptrsv_lean(int n_tiles, const int *__restrict__ blk_off16, const unsigned char *__restrict__ blob, int stat_max,
            int xcap, int per_warp, const double *__restrict__ b, double *x) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    unsigned char *base = smem + (size_t)warp * per_warp;
    unsigned char *stat = base;
    double *xs = (double *)(base + 2 * (size_t)stat_max);
    uint64_t *mbar = (uint64_t *)(xs + xcap);
    const uint32_t xs_a = smem_u32(xs);
    const long long gw = (long long)blockIdx.x * wpb + warp, nwt = (long long)gridDim.x * wpb;
    const int nk = gw < n_tiles ? (int)((n_tiles - gw + nwt - 1) / nwt) : 0;   // my tiles: gw + k * nwt
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int k) {
        const long long qq = gw + (long long)k * nwt;
        const int o0 = blk_off16[qq], o1 = blk_off16[qq + 1];
        const uint32_t bytes = (uint32_t)(o1 - o0) << 4;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the slot was read by this warp before
        mbar_expect_tx(&mbar[k & 1], bytes);
        bulk_g2s(stat + (size_t)(k & 1) * stat_max, blob + 16LL * o0, bytes, &mbar[k & 1]);
    };
    if (lane == 0 && nk > 0) issue(0);
    for (int k = 0; k < nk; ++k) {
        if (lane == 0 && k + 1 < nk) issue(k + 1);   // its slot held tile k-1, which this warp has finished
        mbar_wait(&mbar[k & 1], (uint32_t)((k >> 1) & 1));
        const unsigned char *blk = stat + (size_t)(k & 1) * stat_max;
        const int *hdr = (const int *)blk;
        const int T = hdr[H_T], n_ext = hdr[H_NEXT], n_lev = hdr[H_NLEV];
        const int2 *lvl2 = (const int2 *)(blk + TILE_HDR_BYTES);
        const int *rows = (const int *)(blk + hdr[H_OFF_ROWS]);
        const int *ext = (const int *)(blk + hdr[H_OFF_EXT]);
        const double2 *piv = (const double2 *)(blk + hdr[H_OFF_PIV]);
        const double2 *recA = (const double2 *)(blk + hdr[H_OFF_VAL]);
        const uint4 *recB = (const uint4 *)(blk + hdr[H_OFF_CODE]);
        double *xe = xs + T;
        int have = 0;
        ext_prefetch(x, ext, n_ext, xe, lane);
        for (int s0 = 0; s0 < T; s0 += 256) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u * 32 + lane;
                v[u] = s < T ? __ldg(b + rows[s]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u * 32 + lane;
                if (s < T) xs[s] = v[u];
            }
        }
        if (lane == 0) xs[T + n_ext] = 0.0;
        __syncwarp();
        int2 lv = lvl2[0];
        for (int l = 0; l < n_lev; ++l) {
            const int2 ln = lvl2[l + 1];
            if (lv.y > have) have = ext_deliver(x, ext, n_ext, xe, lane, have, lv.y);
            for (int c = lv.x; c < ln.x; c += 32) {
                const int slot = c + lane;   // idle lanes read a neighbour's (or a spare) record and store nothing
                const double2 A = recA[slot];
                const uint4 B = recB[slot];
                const double rhs = xs[slot];
                const int row = rows[slot < T ? slot : 0];
                const double x0 = lds_f64(xs_a + ((B.z & 0xffffu) << 3));
                const double x1 = lds_f64(xs_a + ((B.z >> 16) << 3));
                const double x2 = lds_f64(xs_a + ((B.w & 0xffffu) << 3));
                double sum = rhs - A.x * x0;
                sum -= A.y * x1;
                sum -= __hiloint2double((int)B.y, (int)B.x) * x2;
                if (HAS_DIAG) {
                    const double2 pr = piv[slot < T ? slot : 0];
                    if (slot >= ln.x) sum = 1.0;   // idle lanes: stay on the fast path of the division
                    sum = exact_div(sum, pr.x, pr.y);
                }
                if (slot < ln.x) {
                    xs[slot] = sum;
                    st_l2(x + row, scrub_sentinel(sum));
                }
            }
            warp_converge();
            lv = ln;
        }
    }
}

#endif  // DDILU_EXPERIMENTS
}  // namespace ddilu

using namespace ddilu;
#define ST(s) ((cudaStream_t)(s))

#ifdef DDILU_EXPERIMENTS
extern "C" int ddilu_tiled_set_tuning(const char *key, int value) {
    if (!key) return DDILU_ERR_ARG;
    const char *k = key;
    auto eq = [&](const char *s) {
        int i = 0;
        while (s[i] && k[i] == s[i]) ++i;
        return s[i] == 0 && k[i] == 0;
    };
    if (eq("ctas_per_sm")) {
        g_tiled.ctas_per_sm = value;
    } else if (eq("grid_cap")) {
        g_tiled.grid_cap = value;
    } else if (eq("probe")) {
        DDILU_CHECK(cudaMemcpyToSymbol(d_tile_probe, &value, sizeof(int)));

    } else {
        return DDILU_ERR_ARG;
    }
    return DDILU_OK;
}

#endif  // DDILU_EXPERIMENTS
extern "C" int ddilu_fastdiv_selftest(long long n_samples, unsigned long long seed, unsigned long long *mismatch,
                                      void *stream) {
    DDILU_CHECK(cudaMemsetAsync(mismatch, 0, sizeof(unsigned long long), ST(stream)));
    if (n_samples <= 0) return DDILU_OK;
    fastdiv_selftest<<<stream_grid(n_samples, 256, 64), 256, 0, ST(stream)>>>(n_samples, seed, mismatch);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

#ifdef DDILU_EXPERIMENTS
extern "C" int ddilu_tiled_set_debug(long long *device_buf) {
    g_tiled.debug = device_buf;
    return DDILU_OK;
}

#endif  // DDILU_EXPERIMENTS
extern "C" int ddilu_tile_box_keys(int n, const int *nodes, int nd, const int *dims_h, const int *tdims_h,
                                   const int *owner, int *keys, long long *n_keys_h, void *stream) {
    if (nd < 1 || nd > 3) return DDILU_ERR_ARG;
    int d[3] = {1, 1, 1}, t[3] = {1, 1, 1}, nb[3];
    for (int a = 0; a < nd; ++a) {
        d[a] = dims_h[a];
        t[a] = tdims_h[a] < 1 ? 1 : tdims_h[a];
    }
    long long nboxes = 1;
    for (int a = 0; a < 3; ++a) {
        nb[a] = (d[a] + t[a] - 1) / t[a];
        nboxes *= nb[a];
    }
    if (n_keys_h) *n_keys_h = nboxes;
    if (nboxes > 0x7FFFFFFF) return DDILU_ERR_ARG;
    if (n <= 0) return DDILU_OK;
    tile_box_keys<<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, nodes, d[0], d[1], t[0], t[1], t[2], nb[0], nb[1],
                                                              (int)nboxes, owner, keys);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

#ifdef DDILU_EXPERIMENTS
extern "C" int ddilu_tile_slab_keys(int n, const int *nodes, int nd, const int *dims_h, const int *tdims_h,
                                    const int *lev, int n_levels, int delta, const int *owner, int n_owners, int *keys,
                                    long long *n_keys_h, void *stream) {
    if (nd < 2 || nd > 3 || delta < 1 || n_levels < 1 || n_owners < 1) return DDILU_ERR_ARG;
    const int d0 = dims_h[0], d1 = dims_h[1];
    const int t0 = tdims_h[0] < 1 ? 1 : tdims_h[0], t1 = tdims_h[1] < 1 ? 1 : tdims_h[1];
    const int nb0 = (d0 + t0 - 1) / t0, nb1 = (d1 + t1 - 1) / t1, n_slabs = (n_levels + delta - 1) / delta;
    const long long range = (long long)nb0 * nb1 * n_slabs * n_owners;
    if (n_keys_h) *n_keys_h = range;
    if (range > 0x7FFFFFFF) return DDILU_ERR_ARG;
    if (n <= 0) return DDILU_OK;
    tile_slab_keys<<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, nodes, d0, d1, t0, t1, nb0, nb1, lev, delta, n_slabs,
                                                               owner, keys);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

#endif  // DDILU_EXPERIMENTS
extern "C" int ddilu_tile_heads(int n, const int *sorted_keys, int *flags, void *stream) {
    if (n <= 0) return DDILU_OK;
    tile_heads<<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, sorted_keys, flags);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_tile_assign(int n, const int *sorted_keys, const int *head_scan, const int *sorted_rows,
                                 int *tile_of, int *tpos, int *tile_ptr, void *stream) {
    if (n <= 0) return DDILU_OK;
    tile_assign<<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, sorted_keys, head_scan, sorted_rows, tile_of, tpos,
                                                            tile_ptr);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_tile_edges_count(int n, const int *row_ptr, const int *col_idx, int upper, const int *tile_of,
                                      int *cnt, void *stream) {
    if (n <= 0) return DDILU_OK;
    tile_edges<false><<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, row_ptr, col_idx, upper, tile_of, cnt, nullptr,
                                                                  nullptr);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_tile_edges_fill(int n, const int *row_ptr, const int *col_idx, int upper, const int *tile_of,
                                     const int *off, int *edges, void *stream) {
    if (n <= 0) return DDILU_OK;
    tile_edges<true><<<stream_grid(n, 256), 256, 0, ST(stream)>>>(n, row_ptr, col_idx, upper, tile_of, nullptr, off,
                                                                 (int2 *)edges);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* flags[0] = did the LAST of the `passes` sweeps change a level, flags[1] = cycle detected */
extern "C" int ddilu_tile_relax(long long n_edges, const int *edges, int n_tiles, int *tlev, int *flags, int passes,
                                void *stream) {
    if (n_edges <= 0 || passes <= 0) {
        DDILU_CHECK(cudaMemsetAsync(flags, 0, sizeof(int), ST(stream)));
        return DDILU_OK;
    }
    for (int p = 0; p < passes; ++p) {
        if (p == passes - 1) DDILU_CHECK(cudaMemsetAsync(flags, 0, sizeof(int), ST(stream)));
        tile_relax<<<stream_grid(n_edges, 256), 256, 0, ST(stream)>>>(n_edges, (const int2 *)edges, n_tiles, tlev,
                                                                     flags);
    }
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_tile_build(int fill, int n_tiles, const int *tsched, const int *tile_ptr, const int *trows,
                                const int *tile_of, const int *tpos, const int *row_ptr, const int *col_idx,
                                const double *values, const int *glev, int upper, int has_diag, int item_warps,
                                int *blk16, int *stats, unsigned char *blob, void *stream) {
    if (n_tiles <= 0) return DDILU_OK;
    if (item_warps != 0 && item_warps != 1 && item_warps != TILE_NW) return DDILU_ERR_ARG;
    const int nw = item_warps;
    if (fill)
        tile_build<true><<<n_tiles, TILE_MAX_ROWS, 0, ST(stream)>>>(n_tiles, tsched, tile_ptr, trows, tile_of, tpos,
                                                                   row_ptr, col_idx, values, glev, upper, has_diag,
                                                                   nw, blk16, stats, blob);
    else
        tile_build<false><<<n_tiles, TILE_MAX_ROWS, 0, ST(stream)>>>(n_tiles, tsched, tile_ptr, trows, tile_of, tpos,
                                                                    row_ptr, col_idx, values, glev, upper, has_diag,
                                                                    nw, blk16, stats, blob);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" long long ddilu_tiled_smem_bytes(int stat_max, int tmax, int emax) {
    return (long long)TILE_NBUF * stat_max + 16LL * (tmax + emax + 2) + (long long)sizeof(TileCtl) + 128;
}

extern "C" int ddilu_sptrsv_tiled(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max,
                                  int tmax, int emax, int kmax, int has_diag, const double *b, double *x,
                                  void *stream) {
    cudaStream_t st = ST(stream);
    if (n <= 0 || n_tiles <= 0) return DDILU_OK;
    if (x == b || (stat_max & 15)) return DDILU_ERR_ARG;
    const size_t smem = (size_t)ddilu_tiled_smem_bytes(stat_max, tmax, emax);
    const int threads = TILE_HELPERS + TILE_NW * 32;
    // entries of a row held in registers: 3 covers 7-point factors, 6 everything else (+ a loop for the rest)
    const int sel = kmax <= 3 ? 0 : (kmax <= 6 ? 1 : 2);   // 0: KP 3, 1: KP 6, 2: KP 6 + loop over the rest
    void *fns[2][3] = {
        {(void *)sptrsv_tiled<false, 3, false>, (void *)sptrsv_tiled<false, 6, false>, (void *)sptrsv_tiled<false, 6, true>},
        {(void *)sptrsv_tiled<true, 3, false>, (void *)sptrsv_tiled<true, 6, false>, (void *)sptrsv_tiled<true, 6, true>}};
    void *fn = fns[has_diag ? 1 : 0][sel];
    // occupancy is looked up once per (kernel, shared-memory size): a solve alternates between factors of
    // different tile sizes (L_B / L_S share an instance), so the cache holds a few sizes per instance and the
    // opt-in shared-memory attribute only ever grows.  Guarded: the Python host may call from several threads.
    struct Cfg { size_t smem; int occ; };
    struct Inst { size_t attr; int n; Cfg c[8]; };
    static Inst cache[2][3];
    static std::mutex cache_mu;
    int occ = 0;
    {
        std::lock_guard<std::mutex> lock(cache_mu);
        Inst &in = cache[has_diag ? 1 : 0][sel];
        int hit = -1;
        for (int i = 0; i < in.n; ++i)
            if (in.c[i].smem == smem) hit = i;
        if (hit < 0) {
            if (in.attr < smem) {
                DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                in.attr = smem;
            }
            int o = 0;
            DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem));
            hit = in.n < 8 ? in.n++ : 7;
            in.c[hit] = {smem, o};
        }
        occ = in.c[hit].occ;
    }
    if (occ < 1) return DDILU_ERR_ARG;
    if (g_tiled.ctas_per_sm > 0 && occ > g_tiled.ctas_per_sm) occ = g_tiled.ctas_per_sm;
    long long grid = (long long)occ * device_info().sm_count;
    if (grid > n_tiles) grid = n_tiles;
    if (g_tiled.grid_cap > 0 && grid > g_tiled.grid_cap) grid = g_tiled.grid_cap;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    long long *dbg = g_tiled.debug;
    void *args[] = {&n_tiles, &blk_off16, &blob, &stat_max, &tmax, &emax, &dbg, &b, &x};
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, threads, args, smem, st));
    return DDILU_OK;
}

#ifdef DDILU_EXPERIMENTS
extern "C" long long ddilu_warptile_smem_per_warp(int stat_max, int tmax, int emax) {
    long long b = 2LL * stat_max + 8LL * (tmax + emax + 2) + 16;
    return (b + 127) & ~127LL;
}

/* warp-per-tile solve: static blocks must have been built with item_warps = 1 */
extern "C" int ddilu_sptrsv_warptile(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max,
                                     int tmax, int emax, int kmax, int has_diag, const double *b, double *x,
                                     void *stream) {
    cudaStream_t st = ST(stream);
    if (n <= 0 || n_tiles <= 0) return DDILU_OK;
    if (x == b || (stat_max & 15)) return DDILU_ERR_ARG;
    int per_warp = (int)ddilu_warptile_smem_per_warp(stat_max, tmax, emax);
    int xcap = tmax + emax + 2;
    int wpb = (226 * 1024) / per_warp;     // one CTA per SM holding as many independent warps as fit
    if (wpb > 16) wpb = 16;
    if (g_tiled.ctas_per_sm > 0 && wpb > g_tiled.ctas_per_sm) wpb = g_tiled.ctas_per_sm;   // diagnostics: warps per SM
    if (wpb < 1) return DDILU_ERR_ARG;
    const size_t smem = (size_t)wpb * per_warp;
    const int wide = kmax > 3 ? 1 : 0;
    void *fns[2][2] = {{(void *)sptrsv_warptile<false, 3>, (void *)sptrsv_warptile<false, 6>},
                       {(void *)sptrsv_warptile<true, 3>, (void *)sptrsv_warptile<true, 6>}};
    void *fn = fns[has_diag ? 1 : 0][wide];
    static size_t attr[2][2] = {{0, 0}, {0, 0}};
    if (attr[has_diag ? 1 : 0][wide] < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[has_diag ? 1 : 0][wide] = smem;
    }
    long long grid = device_info().sm_count;
    const long long need = ((long long)n_tiles + wpb - 1) / wpb;
    if (grid > need) grid = need;
    if (g_tiled.grid_cap > 0 && grid > g_tiled.grid_cap) grid = g_tiled.grid_cap;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    void *args[] = {&n_tiles, &blk_off16, &blob, &stat_max, &xcap, &per_warp, &b, &x};
    // cooperative: every warp waits on tiles of other warps, all CTAs must be resident
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, wpb * 32, args, smem, st));
    return DDILU_OK;
}

/* lean warp-per-tile solve (rows with <= 3 dependencies): static blocks built with item_warps = 0 */
extern "C" int ddilu_sptrsv_lean(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max,
                                 int tmax, int emax, int kmax, int has_diag, const double *b, double *x, void *stream) {
    cudaStream_t st = ST(stream);
    if (n <= 0 || n_tiles <= 0) return DDILU_OK;
    if (x == b || (stat_max & 15) || kmax > 3) return DDILU_ERR_ARG;
    int per_warp = (int)ddilu_warptile_smem_per_warp(stat_max, tmax + 32, emax);
    int xcap = tmax + 32 + emax + 2;
    int wpb = (226 * 1024) / per_warp;
    if (wpb > 16) wpb = 16;
    if (g_tiled.ctas_per_sm > 0 && wpb > g_tiled.ctas_per_sm) wpb = g_tiled.ctas_per_sm;   // diagnostics: warps per SM
    if (wpb < 1) return DDILU_ERR_ARG;
    const size_t smem = (size_t)wpb * per_warp;
    void *fn = has_diag ? (void *)sptrsv_lean<true> : (void *)sptrsv_lean<false>;
    static size_t attr[2] = {0, 0};
    if (attr[has_diag ? 1 : 0] < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[has_diag ? 1 : 0] = smem;
    }
    long long grid = device_info().sm_count;
    const long long need = ((long long)n_tiles + wpb - 1) / wpb;
    if (grid > need) grid = need;
    if (g_tiled.grid_cap > 0 && grid > g_tiled.grid_cap) grid = g_tiled.grid_cap;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    void *args[] = {&n_tiles, &blk_off16, &blob, &stat_max, &xcap, &per_warp, &b, &x};
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, wpb * 32, args, smem, st));
    return DDILU_OK;
}
#endif  // DDILU_EXPERIMENTS
