// Tile sweep: L^-1 b or U^-1 b for the INTERIOR factors of a structured problem (sparse.py:228-272 `_lower_solve`,
// `_upper_solve`; bit-exact: row sums left to right in storage order, every product rounded, IEEE division), with
// the level loop of the block sweep (csrc/sweep.cu) applied to large box tiles (16 x 16 x 16 grid nodes, 4096
// rows, 46 wavefront levels of ~90 rows).
//
// What is different from the rotating-warp tile kernel (csrc/tiled.cu, 8 x 8 x 8 tiles, 23 rows per level, 9.5
// warp instructions per row, 35 % of the HBM roofline):
//   * VECTORS ARE IN TILE ORDER.  The caller keeps right-hand side and solution in the order the sweep walks
//     them: tiles one after the other (each padded to whole 256-row pages, pads hold 0), rows of a tile in
//     level-major order of the L factor.  The U factor of a structurally symmetric stencil walks exactly the
//     reverse order (checked at setup), so ONE ordering serves both solves: a page of the right-hand side is a
//     contiguous 2 KB slice that arrives by TMA next to the page of operands, and the results leave by ONE bulk
//     store per page.  No row ids, no gathers, no scattered stores: 30 (L) / 46 (U) bytes of operands + 16 bytes
//     of vectors per row against the algorithmic 56 / 68.
//   * levels of ~90 rows keep whole warps busy: ~3.5 warp instructions per row.
//   * a tile's boundary dependencies (values of rows in <= 3 neighbour tiles) are gathered once, by a helper
//     warp, one tile AHEAD of the compute warps (double-buffered level table / window / boundary values), after
//     the producer tiles have raised their flags (release / acquire at gpu scope); tiles are taken in a
//     topological order of the tile graph by persistent CTAs of a cooperative launch (deadlock-free: the lowest
//     unfinished tile is always some CTA's current tile).
//
// Roles in a CTA: NS sets of nct compute threads taking the levels in turn (see sweep.cu), an issuer thread (TMA
// of operand pages + right-hand-side slices into an S-deep ring, running ahead across tile boundaries), a gate
// thread (pages landed so far), a gather warp (next tile's level table and boundary values), a writer thread
// (bulk store of finished pages, tile flag).
#include <stdint.h>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int TS_PAGE = 256;
constexpr int TS_HELPERS = 128;          // warp 0: issuer, warp 1: gate, warp 2: gather, warp 3: writer
constexpr int TS_MAX_STAGES = 16;
constexpr int TS_HDR = 16;               // ints per tile header
enum { TH_ROWS = 0, TH_PAGE0, TH_NLEV, TH_LEVOFF, TH_NEXT, TH_EXTOFF, TH_NPROD, TH_PRODOFF, TH_FRONT };

__host__ __device__ constexpr int ts_page_bytes(int K, bool upper) { return TS_PAGE * (upper ? 10 * K + 16 : 10 * K); }
__host__ __device__ constexpr int ts_stage_bytes(int K, bool upper) { return ts_page_bytes(K, upper) + TS_PAGE * 8; }

__device__ __forceinline__ uint32_t ts_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ts_mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ts_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ts_mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ts_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ts_mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ts_u32(bar)) : "memory");
}
__device__ __forceinline__ void ts_mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(ts_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void ts_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ts_u32(dst)),
                 "l"(src), "r"(bytes), "r"(ts_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void ts_bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(ts_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ts_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ int ts_ld_vol(const int *p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(ts_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void ts_st_vol(int *p, int v) {
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(ts_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ts_ld_acq(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(ts_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void ts_st_rel(int *p, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(ts_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ double ts_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ double ts_lds_at(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ uint32_t ts_lds_u16_at(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
__device__ __forceinline__ int2 ts_lds_v2(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void ts_sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ int ts_gt(int a, int b) {
    int v;
    asm volatile("{\n .reg .pred q;\n setp.gt.s32 q, %1, %2;\n selp.s32 %0, 1, 0, q;\n}" : "=r"(v) : "r"(a), "r"(b));
    return v;
}
template <int ID>
__device__ __forceinline__ void ts_bar_sync(int threads) {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(threads) : "memory");
}
template <int ID>
__device__ __forceinline__ void ts_bar_arrive(int threads) {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(threads) : "memory");
}
__device__ __forceinline__ double ts_ld_cg(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

struct TsArgs {
    const int *tiles;               // TS_HDR ints per tile, tiles in schedule (topological) order
    const int *levtab;              // level END positions (tile-local, in the factor's own position space)
    const int *extpos;              // vector positions of the boundary dependencies
    const int *prods;               // schedule ordinals of the producer tiles
    const unsigned char *pages;     // page q of the factor's page space at q * ts_page_bytes(K, UPPER)
    int *flags;                     // per tile (schedule ordinal): 1 when its results are in x (zeroed by the caller)
    const double *b;                // right-hand side, tile order
    double *x;                      // solution, tile order
    int n_tiles;
    int wmask;                      // window - 1
    int xe_cap;                     // boundary values per tile buffer
    int max_lev;                    // levels per tile buffer
    int stages, sets, nct;
};

__host__ __device__ inline size_t ts_ctl_bytes() { return (2 * TS_MAX_STAGES + 4) * 8 + 16; }
__host__ __device__ inline size_t ts_xs_bytes(int window, int xe_cap) {
    return (((size_t)(window + 1 + xe_cap) * 8) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t ts_smem_bytes(int K, bool upper, int stages, int window, int xe_cap, int max_lev) {
    size_t b = ts_ctl_bytes();
    b += 2 * ((((size_t)max_lev * 8) + 15) & ~(size_t)15);
    b += 2 * ts_xs_bytes(window, xe_cap);
    b = (b + 127) & ~(size_t)127;
    return b + (size_t)stages * ts_stage_bytes(K, upper);
}

// the level loop of one tile (see sweep.cu `sweep_levels`: operands in registers before the named barrier of the
// previous level opens; everything the chain does not need is decided before the barrier)
template <int K, bool UPPER, int BAR_IN, int BAR_OUT>
__device__ __forceinline__ void ts_levels(int set, int NS, int t, int nct, uint32_t lev_u32, int nlev, int gq0,
                                          int smask, const int *landed, int &have, uint32_t stage0_u32,
                                          uint32_t xs_u32, int wmask, int *progress, int done_base) {
    constexpr int P = TS_PAGE;
    constexpr int OFF_PIV = 8 * K * P;                       // U: d[P], r[P]
    constexpr int OFF_CODE = UPPER ? 8 * K * P + 16 * P : 8 * K * P;
    constexpr int OFF_RHS = ts_page_bytes(K, UPPER);
    constexpr int STAGE = ts_stage_bytes(K, UPPER);
    const int pair = 2 * nct;
    double c[K], rhs = 0.0, d = 1.0, r = 1.0;
    uint32_t sa[K], wa = 0, slot = 0;
#define TS_OPERANDS(p)                                                                                  \
    do {                                                                                                \
        const int g_ = gq0 + ((p) >> 8);                                                                \
        if (g_ >= have) {                                                                               \
            while ((have = ts_ld_acq(landed)) <= g_) {}                                                 \
        }                                                                                               \
        const uint32_t off_ = (uint32_t)((p) & (P - 1));                                                \
        const uint32_t a8_ = stage0_u32 + (uint32_t)(g_ & smask) * STAGE + off_ * 8u;                   \
        const uint32_t a2_ = a8_ - off_ * 6u + OFF_CODE;                                                \
        uint32_t code_[K];                                                                              \
        if (K >= 1) { c[0] = ts_lds_at<0>(a8_); code_[0] = ts_lds_u16_at<0>(a2_); }                     \
        if (K >= 2) { c[1 % K] = ts_lds_at<8 * P>(a8_); code_[1 % K] = ts_lds_u16_at<2 * P>(a2_); }     \
        if (K >= 3) { c[2 % K] = ts_lds_at<16 * P>(a8_); code_[2 % K] = ts_lds_u16_at<4 * P>(a2_); }    \
        if (K >= 4) { c[3 % K] = ts_lds_at<24 * P>(a8_); code_[3 % K] = ts_lds_u16_at<6 * P>(a2_); }    \
        if (K >= 8) {                                                                                   \
            c[4 % K] = ts_lds_at<32 * P>(a8_); code_[4 % K] = ts_lds_u16_at<8 * P>(a2_);                \
            c[5 % K] = ts_lds_at<40 * P>(a8_); code_[5 % K] = ts_lds_u16_at<10 * P>(a2_);               \
            c[6 % K] = ts_lds_at<48 * P>(a8_); code_[6 % K] = ts_lds_u16_at<12 * P>(a2_);               \
            c[7 % K] = ts_lds_at<56 * P>(a8_); code_[7 % K] = ts_lds_u16_at<14 * P>(a2_);               \
        }                                                                                               \
        if (UPPER) {                                                                                    \
            d = ts_lds_at<OFF_PIV>(a8_);                                                                \
            r = ts_lds_at<OFF_PIV + 8 * P>(a8_);                                                        \
            /* the vector slice of a U page is in memory (= L) order: mirrored inside the page */      \
            slot = a8_ - off_ * 16u + (OFF_RHS + 8 * (P - 1));                                          \
        } else {                                                                                        \
            slot = a8_ + OFF_RHS;                                                                       \
        }                                                                                               \
        rhs = ts_lds(slot);                                                                             \
        wa = xs_u32 + 8u * (uint32_t)((p) & wmask);                                                     \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) sa[k_] = xs_u32 + 8u * code_[k_];              \
    } while (0)
#define TS_FINISH()                                                                                     \
    do {                                                                                                \
        double v_[K];                                                                                   \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) v_[k_] = ts_lds(sa[k_]);                       \
        double sum_ = rhs;                                                                              \
        /* -fmad=false: every product is rounded before it is subtracted */                            \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) sum_ -= c[k_] * v_[k_];                        \
        if (UPPER) sum_ = exact_div(sum_, d, r);                                                        \
        ts_sts(wa, sum_);                                                                               \
        ts_sts(slot, sum_);      /* the page's vector slice now holds the result: it leaves by bulk store */ \
    } while (0)
    uint32_t lp = lev_u32 + 8u * (uint32_t)set;
    for (int l = set; l < nlev; l += NS, lp += 8u * (uint32_t)NS) {
        const int2 se = ts_lds_v2(lp);
        const int p0 = se.x + t, e = se.y;
        const int wide = ts_gt(e - se.x, nct), more = ts_gt(nlev, l + 1);
        const bool first = l == 0;
        const bool act = p0 < e;
        if (act) TS_OPERANDS(p0);
        if (!first) ts_bar_sync<BAR_IN>(pair);
        if (act) TS_FINISH();
        if (wide) {
            for (int p = p0 + nct; p < e; p += nct) {
                TS_OPERANDS(p);
                TS_FINISH();
            }
        }
        if (more) ts_bar_arrive<BAR_OUT>(pair);
        if (t == 0) ts_st_vol(progress, done_base + se.x);
    }
#undef TS_OPERANDS
#undef TS_FINISH
}

template <int K, bool UPPER>
__global__ void __launch_bounds__(768, 1) tsweep_kernel(const TsArgs a) {
    constexpr int P = TS_PAGE;
    constexpr int STAGE = ts_stage_bytes(K, UPPER);
    constexpr int OFF_RHS = ts_page_bytes(K, UPPER);
    constexpr uint32_t PB = ts_page_bytes(K, UPPER);
    extern __shared__ __align__(128) unsigned char ts_smem[];
    const int S = a.stages, smask = S - 1, nct = a.nct, NS = a.sets;
    uint64_t *full = (uint64_t *)ts_smem;
    uint64_t *empty = full + TS_MAX_STAGES;
    uint64_t *tile_ready = empty + TS_MAX_STAGES;   // [2]
    uint64_t *tile_free = tile_ready + 2;           // [2]
    int *progress = (int *)(tile_free + 2);
    int *landed = progress + 1;
    unsigned char *lev0 = ts_smem + ts_ctl_bytes();
    const size_t lev_bytes = (((size_t)a.max_lev * 8) + 15) & ~(size_t)15;
    unsigned char *xs0 = lev0 + 2 * lev_bytes;
    const size_t xs_bytes = ts_xs_bytes(a.wmask + 1, a.xe_cap);
    size_t off = (size_t)(xs0 - ts_smem) + 2 * xs_bytes;
    off = (off + 127) & ~(size_t)127;
    unsigned char *stage0 = ts_smem + off;
    const int tid = threadIdx.x;
    const int G = gridDim.x, c0 = blockIdx.x;
    const int my_tiles = c0 < a.n_tiles ? (a.n_tiles - c0 + G - 1) / G : 0;
    if (my_tiles == 0) return;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            ts_mbar_init(&full[s], 1);
            ts_mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ts_mbar_init(&tile_ready[i], 1);
            ts_mbar_init(&tile_free[i], 1);
        }
        *progress = 0;
        *landed = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ncomp = NS * nct;
    if (tid < ncomp) {
        // ------------------------------------------------------------ compute sets
        const int set = tid / nct, t = tid - set * nct;
        const uint32_t stage0_u32 = ts_u32(stage0);
        int have = 0, gq0 = 0, done_base = 0;
        for (int k = 0; k < my_tiles; ++k) {
            const int par = k & 1;
            const int *hdr = a.tiles + (size_t)TS_HDR * (c0 + (size_t)k * G);
            const int n_rows = __ldg(hdr + TH_ROWS), nlev = __ldg(hdr + TH_NLEV);
            const int n_pages = (n_rows + (UPPER ? __ldg(hdr + TH_FRONT) : 0) + P - 1) / P;
            ts_mbar_wait(&tile_ready[par], (uint32_t)((k >> 1) & 1));
            const uint32_t lev_u32 = ts_u32(lev0 + par * lev_bytes), xs_u32 = ts_u32(xs0 + par * xs_bytes);
#define TS_CALL(IN, OUT)                                                                                      \
    ts_levels<K, UPPER, IN, OUT>(set, NS, t, nct, lev_u32, nlev, gq0, smask, landed, have, stage0_u32, xs_u32, \
                                 a.wmask, progress, done_base)
            if (set == 0) {
                if (NS == 2) TS_CALL(2, 1);
                else TS_CALL(3, 1);
            } else if (set == 1) {
                TS_CALL(1, 2);
            } else {
                TS_CALL(2, 3);
            }
#undef TS_CALL
            ts_bar_sync<4>(ncomp);                    // every row of the tile is stored
            gq0 += n_pages;
            done_base += n_pages * P;
            if (tid == 0) {
                ts_st_vol(progress, done_base);
                ts_mbar_arrive(&tile_free[par]);      // level table / window / boundary buffer of this parity are free
            }
        }
    } else if (tid == ncomp) {
        // ------------------------------------------------------------ issuer
        int i = 0;
        for (int k = 0; k < my_tiles; ++k) {
            const int *hdr = a.tiles + (size_t)TS_HDR * (c0 + (size_t)k * G);
            const int n_rows = __ldg(hdr + TH_ROWS), page0 = __ldg(hdr + TH_PAGE0);
            const int n_pages = (n_rows + (UPPER ? __ldg(hdr + TH_FRONT) : 0) + P - 1) / P;
            for (int q = 0; q < n_pages; ++q, ++i) {
                const int s = i & smask;
                if (i >= S) ts_mbar_wait(&empty[s], (uint32_t)(((i / S) - 1) & 1));
                unsigned char *st = stage0 + (size_t)s * STAGE;
                // U page q (U position space) holds the vector positions of L page n_pages - 1 - q
                const int vq = UPPER ? n_pages - 1 - q : q;
                ts_mbar_arrive_tx(&full[s], PB + P * 8);
                ts_bulk_g2s(st, a.pages + (size_t)(page0 + q) * PB, PB, &full[s]);
                ts_bulk_g2s(st + OFF_RHS, a.b + (size_t)(page0 + vq) * P, P * 8, &full[s]);
            }
            if (k + 1 < my_tiles) {     // operands of the next tile towards L2 while this one is worked on
                const int *h2 = a.tiles + (size_t)TS_HDR * (c0 + (size_t)(k + 1) * G);
                const int r2 = __ldg(h2 + TH_ROWS), p2 = __ldg(h2 + TH_PAGE0);
                const int np2 = (r2 + (UPPER ? __ldg(h2 + TH_FRONT) : 0) + P - 1) / P;
                for (int q = 0; q < np2; ++q) ts_prefetch_l2(a.pages + (size_t)(p2 + q) * PB, PB);
            }
        }
    } else if (tid == ncomp + 32) {
        // ------------------------------------------------------------ gate: pages landed so far
        int total = 0;
        for (int k = 0; k < my_tiles; ++k) {
            const int *hdr = a.tiles + (size_t)TS_HDR * (c0 + (size_t)k * G);
            total += (__ldg(hdr + TH_ROWS) + (UPPER ? __ldg(hdr + TH_FRONT) : 0) + P - 1) / P;
        }
        for (int i = 0; i < total; ++i) {
            ts_mbar_wait(&full[i & smask], (uint32_t)((i / S) & 1));
            ts_st_rel(landed, i + 1);
        }
    } else if (tid >= ncomp + 64 && tid < ncomp + 96) {
        // ------------------------------------------------------------ gather warp: level table + boundary values,
        // one tile ahead of the compute sets
        const int lane = tid - ncomp - 64;
        for (int k = 0; k < my_tiles; ++k) {
            const int par = k & 1;
            const int q_tile = c0 + k * G;
            const int *hdr = a.tiles + (size_t)TS_HDR * q_tile;
            const int nlev = __ldg(hdr + TH_NLEV), lev_off = __ldg(hdr + TH_LEVOFF), n_ext = __ldg(hdr + TH_NEXT),
                      ext_off = __ldg(hdr + TH_EXTOFF), n_prod = __ldg(hdr + TH_NPROD), prod_off = __ldg(hdr + TH_PRODOFF),
                      front = UPPER ? __ldg(hdr + TH_FRONT) : 0;
            if (k >= 2) ts_mbar_wait(&tile_free[par], (uint32_t)(((k >> 1) - 1) & 1));
            int *levs = (int *)(lev0 + par * lev_bytes);
            double *xs = (double *)(xs0 + par * xs_bytes);
            for (int i = lane; i < nlev; i += 32) {
                levs[2 * i] = i ? __ldg(a.levtab + lev_off + i - 1) : front;
                levs[2 * i + 1] = __ldg(a.levtab + lev_off + i);
            }
            if (lane == 0) xs[a.wmask + 1] = 0.0;
            // producers finished?
            for (int i = lane; i < n_prod; i += 32) {
                const int *f = a.flags + __ldg(a.prods + prod_off + i);
                while (ld_acquire(f) == 0) __nanosleep(64);
            }
            __syncwarp();
            for (int e0 = 0; e0 < n_ext; e0 += 128) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * 32 + lane;
                    v[u] = e < n_ext ? ts_ld_cg(a.x + __ldg(a.extpos + ext_off + e)) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * 32 + lane;
                    if (e < n_ext) xs[a.wmask + 2 + e] = v[u];
                }
            }
            __syncwarp();
            if (lane == 0) ts_mbar_arrive(&tile_ready[par]);
        }
    } else if (tid == ncomp + 96) {
        // ------------------------------------------------------------ writer: finished pages leave by bulk store
        int i = 0, done_base = 0;
        for (int k = 0; k < my_tiles; ++k) {
            const int q_tile = c0 + k * G;
            const int *hdr = a.tiles + (size_t)TS_HDR * q_tile;
            const int n_rows = __ldg(hdr + TH_ROWS), page0 = __ldg(hdr + TH_PAGE0);
            const int front = UPPER ? __ldg(hdr + TH_FRONT) : 0;
            const int n_pages = (n_rows + front + P - 1) / P;
            for (int q = 0; q < n_pages; ++q, ++i) {
                const int s = i & smask;
                // rows of the page are complete when the progress counter has passed its last REAL position
                const int last = UPPER ? (q + 1) * P : min((q + 1) * P, n_rows);
                while (ts_ld_vol(progress) < done_base + last) __nanosleep(40);
                ts_mbar_wait(&full[s], (uint32_t)((i / S) & 1));
                asm volatile("fence.acq_rel.cta;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic stores -> bulk (async proxy) read
                const int vq = UPPER ? n_pages - 1 - q : q;
                ts_bulk_s2g(a.x + (size_t)(page0 + vq) * P, stage0 + (size_t)s * STAGE + OFF_RHS, P * 8);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the stage may be refilled
                ts_mbar_arrive(&empty[s]);
            }
            done_base += n_pages * P;
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");            // the tile's results are written
            __threadfence();
            st_release(a.flags + q_tile, 1);
        }
    }
}

// operands of a factor into its pages (tile order); ecode[k] = boundary slot of entry k (window + 1 + e) or -1
template <bool UPPER>
__global__ void tsweep_fill_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                   const double *__restrict__ val, int K, const int *__restrict__ gpos,
                                   const int *__restrict__ lpos, const int *__restrict__ ecode, int wmask,
                                   unsigned char *pages, int *bad_row) {
    constexpr int P = TS_PAGE;
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const int g = gpos[row], q = g >> 8, off = g & (P - 1);
    const size_t pb = (size_t)P * (UPPER ? 10 * K + 16 : 10 * K);
    unsigned char *pg = pages + (size_t)q * pb;
    double *cf = (double *)pg;
    unsigned short *cd = (unsigned short *)(pg + (UPPER ? 8 * K * P + 16 * P : 8 * K * P));
    int kk = 0;
    double diag = 1.0;
    bool seen = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (UPPER ? j > row : j < row) {
            if (kk < K) {
                cf[kk * P + off] = val[k];
                const int ec = ecode[k];
                cd[kk * P + off] = (unsigned short)(ec >= 0 ? ec : (lpos[j] & wmask));
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {
        cf[kk * P + off] = 0.0;
        cd[kk * P + off] = (unsigned short)(wmask + 1);
    }
    if (UPPER) {
        double *pv = (double *)(pg + 8 * K * P);
        pv[off] = diag;
        pv[P + off] = safe_reciprocal(diag);
        if (!seen || fabs(diag) < 1e-300) atomicMin(bad_row, row);
    }
}

// vector between the row order and the tile order: out[pos[i]] = in[i] (to_tile) or out[i] = in[pos[i]]
__global__ void tsweep_permute_kernel(int n, const int *__restrict__ pos, const double *__restrict__ in,
                                      double *__restrict__ out, int to_tile) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (to_tile) out[pos[i]] = in[i];
    else out[i] = in[pos[i]];
}

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

extern "C" long long ddilu_tsweep_page_bytes(int k, int upper) { return ts_page_bytes(k, upper != 0); }

extern "C" long long ddilu_tsweep_smem_bytes(int k, int upper, int stages, int window, int xe_cap, int max_lev) {
    return (long long)ts_smem_bytes(k, upper != 0, stages, window, xe_cap, max_lev);
}

extern "C" int ddilu_tsweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                                 const int *gpos, const int *lpos, const int *ecode, int window, unsigned char *pages,
                                 int *bad_row, void *stream) {
    if (n <= 0) return DDILU_OK;
    if (k < 1 || k > 8 || window < 32 || (window & (window - 1)) || window > 16384) return DDILU_ERR_ARG;
    const int threads = 256, grid = div_up(n, threads);
    if (upper)
        tsweep_fill_kernel<true><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, lpos, ecode,
                                                                   window - 1, pages, bad_row);
    else
        tsweep_fill_kernel<false><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, lpos, ecode,
                                                                    window - 1, pages, bad_row);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_tsweep_permute(int n, const int *pos, const double *in, double *out, int to_tile, void *stream) {
    if (n <= 0) return DDILU_OK;
    tsweep_permute_kernel<<<div_up(n, 256), 256, 0, ST(stream)>>>(n, pos, in, out, to_tile);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

namespace {
template <int K, bool UPPER>
int launch_tsweep(const TsArgs &a, size_t smem, int *flags, cudaStream_t st) {
    static size_t attr = 0;
    static int occ_smem = -1, occ_threads = -1, occ = 0;
    void *fn = (void *)tsweep_kernel<K, UPPER>;
    const int threads = a.sets * a.nct + TS_HELPERS;
    if (attr < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    if (occ_smem != (int)smem || occ_threads != threads) {
        DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
        occ_smem = (int)smem;
        occ_threads = threads;
    }
    if (occ < 1) return DDILU_ERR_ARG;
    long long grid = (long long)occ * device_info().sm_count;
    if (grid > a.n_tiles) grid = a.n_tiles;
    DDILU_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)a.n_tiles, st));
    TsArgs args = a;
    void *kargs[] = {&args};
    // cooperative: a CTA waits on tiles of other CTAs, all of them must be resident
    DDILU_CHECK(cudaLaunchCooperativeKernel(fn, (int)grid, threads, kargs, smem, st));
    return DDILU_OK;
}
}  // namespace

/* x = T^-1 b with b and x in TILE ORDER (see the header of this file); tiles = 16 ints per tile in schedule order
 * {rows, first page, levels, offset into levtab, boundary values, offset into extpos, producer tiles, offset into
 * prods, pad rows in front (U), 0...} */
extern "C" int ddilu_tsweep_solve(int n_tiles, const int *tiles, const int *levtab, const int *extpos, const int *prods,
                                  const unsigned char *pages, int *flags, int k, int upper, int window, int xe_cap,
                                  int max_lev, int stages, int sets, int nct, const double *b, double *x, void *stream) {
    if (n_tiles <= 0) return DDILU_OK;
    if (x == b || stages < 2 || stages > TS_MAX_STAGES || (stages & (stages - 1)) || sets < 2 || sets > 3 || nct < 32 ||
        (nct & 31) || sets * nct + TS_HELPERS > 768 || window < 32 || (window & (window - 1)) ||
        window + 2 + xe_cap > 65535)
        return DDILU_ERR_ARG;
    TsArgs a{tiles, levtab, extpos, prods, pages, flags, b, x, n_tiles, window - 1, xe_cap, max_lev, stages, sets, nct};
    const size_t smem = ts_smem_bytes(k, upper != 0, stages, window, xe_cap, max_lev);
    if (smem > 227 * 1024) return DDILU_ERR_ARG;
    cudaStream_t st = ST(stream);
#define TS_DISPATCH(KK)                                                          \
    case KK:                                                                     \
        return upper ? launch_tsweep<KK, true>(a, smem, flags, st) : launch_tsweep<KK, false>(a, smem, flags, st)
    switch (k) {
        TS_DISPATCH(2);
        TS_DISPATCH(3);
        TS_DISPATCH(4);
        TS_DISPATCH(8);
        default: return DDILU_ERR_ARG;
    }
#undef TS_DISPATCH
}
