// Block sweep: L^-1 / U^-1 / U^-1 L^-1 on a block-diagonal factor pair with narrow levels -- the interface
// (Schur) factors L_S, U_S of the two-level preconditioners, one independent diagonal block per subdomain
// (precond.py:239-249 `_schur_solve` inside `reduced_matvec`, precond.py:361-366 `_coarse_precond`; the
// arithmetic is sparse.py:228-272 `_lower_solve` / `_upper_solve`: row sums left to right in storage order,
// every product rounded, IEEE division -> bit-exact).
//
// Why its own kernel.  These factors are tiny (390 k rows, 20 MB at 256^3) and deep (382 levels of ~190 rows
// per subdomain): any kernel that pays an L2 round trip or a tile hand-over per level is latency-bound (the
// tiled kernel: 83 / 120 us per solve, 3 % of the HBM roofline, as much time per outer iteration as the
// interior solves that move 100x the bytes).  Here ONE CTA owns a diagonal block and walks its levels with
// nothing but shared memory on the dependency chain:
//
//   * rows of a block are numbered in schedule order (level-major); result p lives in xs[p & (W - 1)], a
//     shared-memory window (setup checks that no row reads further back than W positions behind the END of
//     its own level);
//   * the rows' operands -- K coefficients, K 16-bit window slots, the row id, (pivot, reciprocal) for U --
//     are stored as PAGES of 256 rows in schedule order, structure-of-arrays, and stream through an S-deep
//     shared-memory ring by TMA (cp.async.bulk + mbarrier complete_tx), together with the 2 KB slice of the
//     right-hand side, which the caller provides IN SCHEDULE ORDER (ddilu_sweep_rhs: a gather, or the fused
//     product base -/+ A y with the coupling block E_off or W, precond.py:247, 242-243);
//   * compute thread t owns row s + t of the level [s, e): its operands are in registers BEFORE the level's
//     named barrier opens; behind the barrier only K shared-memory loads, the multiply/subtract chain (+ the
//     exact reciprocal division for U), two shared-memory stores (window, page) remain;
//   * three writer warps follow the compute warps (progress counter in shared memory), each taking every third
//     page, and scatter the results to global memory -- L results go to the U phase's right-hand-side buffer
//     in U schedule order, U results to out[row] (+ the added vector, staged in U schedule order with the
//     page: the `y + S^-1 E y` of precond.py:249) -- then free the page;
//   * L and U run back to back in ONE launch: after the last L page has been flushed (fence.proxy.async +
//     mbarrier) the issuer streams the U pages with the right-hand side the L phase wrote.
//
// Algorithmic bytes per row: 12 nnz + 4 + 16; moved here: 10 K + 8 (L) / 10 K + 20 (U) of
// operands + 8 right-hand side + 8 result.
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int SW_PAGE = 256;            // rows per page (short rows); long rows (K > 8) use 64-row pages
constexpr int SW_WRITER_WARPS = 3;      // each takes every 3rd page: the flush latencies of consecutive pages overlap
constexpr int SW_WRITERS = 32 * SW_WRITER_WARPS;
constexpr int SW_HELPERS = 64 + SW_WRITERS;   // warp 0: TMA issuer (one lane), warp 1: gate (one lane), then the writer warps
constexpr int SW_MAX_STAGES = 24;
constexpr int SW_BLOCK_INTS = 8;        // per block: n_rows, page0, nlev_l, nlev_u, lev_off, 0, 0, 0

__host__ __device__ constexpr int sw_page_bytes(int K, bool upper, int P = SW_PAGE) {
    return P * (upper ? 10 * K + 20 : 10 * K + 8);
}
// stage = operands page | right-hand side slice | slice of the vector added to the result (U phase)
__host__ __device__ constexpr int sw_stage_bytes(int K, int P = SW_PAGE) { return sw_page_bytes(K, true, P) + P * 16; }
__host__ __device__ constexpr int sw_shift(int P) { return P == 256 ? 8 : (P == 128 ? 7 : (P == 64 ? 6 : 5)); }

__device__ __forceinline__ uint32_t sw_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sw_mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sw_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void sw_mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sw_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void sw_mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sw_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sw_mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(sw_smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void sw_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sw_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(sw_smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void sw_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sw_bar_sync(int threads) {
    asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
}
__device__ __forceinline__ int sw_ld_progress(const int *p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(sw_smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void sw_st_progress(int *p, int v) {
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sw_smem_u32(p)), "r"(v) : "memory");
}
// pages-landed counter: release / acquire, so that ptxas cannot move a thread's operand loads in front of the
// load that tells it the page is there (it did, with plain volatile accesses)
__device__ __forceinline__ int sw_ld_landed(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(sw_smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void sw_st_landed(int *p, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(sw_smem_u32(p)), "r"(v) : "memory");
}

struct SweepArgs {
    const int *blocks;              // SW_BLOCK_INTS per block
    const int *levtab;              // per block: end positions (block-local) of its L levels, then of its U levels
    const unsigned char *pages_l;   // page q of the global page space at q * sw_page_bytes(K, false)
    const unsigned char *pages_u;
    const double *rhs;              // right-hand side in schedule order of the FIRST phase that runs
    double *tmp;                    // U-phase right-hand side written by the L phase (phases = 3)
    double *out;                    // results by row id
    const double *add;              // optional, in U schedule order (ddilu_sweep_rhs): out[row] = add[U position] + x
    int phases;                     // 1: L, 2: U, 3: L then U
    int wmask;                      // window size - 1 (power of two); slot W holds 0.0 for padded operands
    int stages;                     // ring depth, a power of two
    int sets;                       // compute sets (2 or 3)
    int nct;                        // compute threads per set (multiple of 32); two sets take the levels alternately
    int max_lev;                    // largest nlev_l + nlev_u of a block (shared-memory table size)
    int wsleep;                     // writers' poll back-off (ns)
    int flags;                      // diagnostics: 1 = writers skip the global stores, 2 = no L2 prefetch
    long long *dbg;                 // optional: 64 cycle counters per block (16 per compute set, thread 0 of the set): L phase, U phase, waiting for pages, then operands / barrier / chain of L and of U
};

// shared memory: [full[S] | empty[S] | lflush | progress] [levels] [window] [stages]
__host__ __device__ inline size_t sw_ctl_bytes() { return (2 * SW_MAX_STAGES + 2) * 8; }   // + progress, landed (2 ints)
__host__ __device__ inline size_t sw_smem_bytes(int K, int stages, int window, int max_lev, int P = SW_PAGE) {
    size_t b = sw_ctl_bytes();
    b += ((size_t)max_lev * 8 + 15) & ~(size_t)15;      // (start, end) pair per level
    b += ((size_t)(window + 1) * 8 + 15) & ~(size_t)15;
    b = (b + 127) & ~(size_t)127;
    return b + (size_t)stages * sw_stage_bytes(K, P);
}

__device__ __forceinline__ double sw_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ double sw_lds_at(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ uint32_t sw_lds_u16_at(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
__device__ __forceinline__ int sw_lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t sw_lds_u16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sw_sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sw_bar_sync_id(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void sw_bar_arrive_id(int id, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void sw_mbar_wait_u32(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ int sw_gt(int a, int b) {     // a > b, evaluated where it is written
    int v;
    asm volatile("{\n .reg .pred q;\n setp.gt.s32 q, %1, %2;\n selp.s32 %0, 1, 0, q;\n}" : "=r"(v) : "r"(a), "r"(b));
    return v;
}
template <int ID>
__device__ __forceinline__ void sw_bar_sync_c(int threads) {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(threads) : "memory");
}
template <int ID>
__device__ __forceinline__ void sw_bar_arrive_c(int threads) {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(threads) : "memory");
}
__device__ __forceinline__ int2 sw_lds_v2(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}

// The compute threads form NS (2 or 3) sets that take the levels in turn: while one set runs the chain of level
// l (K window loads, multiply/subtract chain [, division], two stores per row), the next set has the operands
// of level l + 1 in registers already and waits on the named barrier the first set arrives at -- operand fetch
// and address arithmetic are off the dependency chain.  A thread owns R rows of its level (row s + t + j nct).
// Barrier 1 + (l % NS) = 1 + set: arrived at by the set of level l, synced on by the set of level l + 1.
// The kernel is bound by instruction issue (ncu: 1.8 warp instructions per cycle and SM, ~500 per level before
// this loop was trimmed): every instruction a warp executes per level counts, also in warps that own no row of
// the level, so the loop carries nothing but the (start, end) pair of the level, the barrier pair and, for the
// rows that exist, operand fetch and chain.  DBG (experiments build) adds cycle counters and the strip flags
// of scripts/probe_sweep.py.
template <int K, int R, bool UPPER, bool DBG, int BAR_IN, int BAR_OUT, int P>
__device__ __forceinline__ void sweep_levels(int set, int NS, int t, int nct, uint32_t lev_u32, int nlev, int gq0,
                                              int smask, const int *landed, uint32_t stage0_u32, uint32_t xs_u32,
                                              int wmask, int *progress, int done_base, long long *dbg, int xflags) {
    constexpr int PSH = sw_shift(P);
    // long-row instances (64-row pages): non-blocking operand prefetch, see SW_OPERANDS; the short-row instances
    // keep the blocking prefetch (their plans satisfy the stricter residency rule of device.build_sweep) and
    // with it a chain without the pending-row checks
    constexpr bool NB = P < SW_PAGE;
    constexpr int OFF_PIV = 8 * K * P;                                   // U: d[P], r[P]
    constexpr int OFF_CODE = UPPER ? 8 * K * P + 20 * P : 8 * K * P + 8 * P;
    constexpr int OFF_RHS = sw_page_bytes(K, true, P);
    constexpr int STAGE = sw_stage_bytes(K, P);
    const int pair = 2 * nct;                 // threads of a producer set + a consumer set
    int have = 0;                             // ring ordinals below `have` are known to have landed
    long long wait_cycles = 0, t_begin = 0, t_ops = 0, t_fin = 0;
    if (DBG && dbg) t_begin = clock64();
    double c[R][K], rhs[R], d[R], r[R];
    uint32_t sa[R][K], wa[R], slot[R];
    /* BLOCK = false: prefetch before the level barrier -- if the row's page has not landed yet the row is marked   \
     * pending and fetched behind the barrier (BLOCK = true).  A prefetch that waited for its page could wait for   \
     * ever: the page may need a ring stage that is freed only when the progress counter moves, and the progress   \
     * counter is moved by this very set behind its barrier. */                                                  \
#define SW_OPERANDS(j, p, BLOCK)                                                                       \
    do {                                                                                               \
        if (DBG && (xflags & 128)) break;                                                              \
        const int g_ = gq0 + ((p) >> PSH);                                                             \
        if (g_ >= have) {                                                                              \
            have = sw_ld_landed(landed);                                                               \
            if (have <= g_) {                                                                          \
                if (NB && !(BLOCK)) {                                                                  \
                    pend |= 1 << (j);                                                                  \
                    break;                                                                             \
                }                                                                                      \
                long long w0_ = 0;                                                                     \
                if (DBG && dbg) w0_ = clock64();                                                       \
                while ((have = sw_ld_landed(landed)) <= g_) {}                                         \
                if (DBG && dbg) wait_cycles += clock64() - w0_;                                        \
            }                                                                                          \
        }                                                                                              \
        if (DBG && (xflags & 64)) break;                                                               \
        const uint32_t off_ = (uint32_t)((p) & (P - 1));                                               \
        const uint32_t a8_ = stage0_u32 + (uint32_t)(g_ & smask) * STAGE + off_ * 8u;                  \
        const uint32_t a2_ = a8_ - off_ * 6u + OFF_CODE;                                               \
        uint32_t code_[K];                                                                             \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) {      /* offsets fold into immediates after unrolling */ \
            c[j][k_] = sw_lds(a8_ + (uint32_t)(k_ * 8 * P));                                           \
            code_[k_] = sw_lds_u16(a2_ + (uint32_t)(k_ * 2 * P));                                      \
        }                                                                                              \
        rhs[j] = sw_lds_at<OFF_RHS>(a8_);                                                              \
        if (UPPER) {                                                                                   \
            d[j] = sw_lds_at<OFF_PIV>(a8_);                                                            \
            r[j] = sw_lds_at<OFF_PIV + 8 * P>(a8_);                                                    \
        }                                                                                              \
        slot[j] = a8_ + OFF_RHS;                                                                       \
        wa[j] = xs_u32 + 8u * (uint32_t)((p) & wmask);                                                 \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) sa[j][k_] = xs_u32 + 8u * code_[k_];          \
    } while (0)
#define SW_FINISH(j)                                                                                   \
    do {                                                                                               \
        double v_[K];                                                                                  \
        _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_)                                               \
            v_[k_] = (DBG && (xflags & 4)) ? 1.0 : sw_lds(sa[j][k_]);                                  \
        double sum_ = rhs[j];                                                                          \
        if (!(DBG && (xflags & 8))) {                                                                  \
            /* -fmad=false: every product is rounded before it is subtracted */                       \
            _Pragma("unroll") for (int k_ = 0; k_ < K; ++k_) sum_ -= c[j][k_] * v_[k_];                \
            if (UPPER) sum_ = exact_div(sum_, d[j], r[j]);                                             \
        }                                                                                              \
        if (!(DBG && (xflags & 32))) sw_sts(wa[j], sum_);                                              \
        /* the writer warps take the result from the page (the window slot is reused W rows later) */  \
        if (!(DBG && (xflags & 16))) sw_sts(slot[j], sum_);                                            \
    } while (0)
    uint32_t lp = lev_u32 + 8u * (uint32_t)set;
    const int cover = R * nct;                      // rows of a level the prefetched slots cover
    for (int l = set; l < nlev; l += NS, lp += 8u * (uint32_t)NS) {
        const int2 se = sw_lds_v2(lp);              // positions [start, end) of the level
        const int p0 = se.x + t, e = se.y;
        // everything the chain does not need is decided BEFORE the barrier: what sits between the barrier and the
        // arrive is the dependency chain of the whole solve
        // (inline asm keeps the compiler from sinking the comparisons behind the chain)
        const int wide = sw_gt(e - se.x, cover), more = sw_gt(nlev, l + 1);
        const bool first = l == 0;
        long long c0 = 0, c1 = 0;
        if (DBG && dbg) c0 = clock64();
        int pend = 0;                               // rows whose page had not landed at prefetch time
#pragma unroll
        for (int j = 0; j < R; ++j)
            if (p0 + j * nct < e) SW_OPERANDS(j, p0 + j * nct, false);
        if (DBG && dbg) c1 = clock64();
        if (!first) sw_bar_sync_c<BAR_IN>(pair);    // results of the previous level are in the window
        // rows below the level's start are complete: the writers may flush their pages, the ring moves on (with the
        // non-blocking prefetch this must come before any wait for a page of this level)
        if (NB && t == 0) sw_st_progress(progress, done_base + se.x);
#pragma unroll
        for (int j = 0; j < R; ++j)
            if (p0 + j * nct < e) {
                if (NB && (pend & (1 << j))) SW_OPERANDS(j, p0 + j * nct, true);
                SW_FINISH(j);
            }
        if (wide) {                                 // levels wider than R rows per thread (rare)
            for (int p = p0 + cover; p < e; p += nct) {
                SW_OPERANDS(0, p, true);
                SW_FINISH(0);
            }
        }
        if (more) sw_bar_arrive_c<BAR_OUT>(pair);
        if (!NB && t == 0) sw_st_progress(progress, done_base + se.x);   // rows below the level's start are complete
        if (DBG && dbg) {
            t_ops += c1 - c0;
            t_fin += clock64() - c1;
        }
    }
#undef SW_OPERANDS
#undef SW_FINISH
    if (DBG && dbg && t == 0) {
        long long *o = dbg + 16 * set;
        o[UPPER ? 1 : 0] = clock64() - t_begin;
        o[2] += wait_cycles;
        o[UPPER ? 6 : 3] = t_ops;
        o[UPPER ? 8 : 5] = t_fin;
    }
}

// barrier ids as immediates (a register id makes the compiler pack id and count around every barrier instruction)
template <int K, int R, bool UPPER, bool DBG, int P>
__device__ __forceinline__ void sweep_compute(int set, int NS, int t, int nct, uint32_t lev_u32, int nlev, int gq0,
                                              int smask, const int *landed, uint32_t stage0_u32, uint32_t xs_u32,
                                              int wmask, int *progress, int done_base, long long *dbg, int xflags) {
#define SW_CALL(IN, OUT)                                                                                        \
    sweep_levels<K, R, UPPER, DBG, IN, OUT, P>(set, NS, t, nct, lev_u32, nlev, gq0, smask, landed, stage0_u32, xs_u32, \
                                            wmask, progress, done_base, dbg, xflags)
    if (set == 0) {
        if (NS == 2) SW_CALL(2, 1);
        else SW_CALL(3, 1);
    } else if (set == 1) {
        SW_CALL(1, 2);
    } else {
        SW_CALL(2, 3);
    }
#undef SW_CALL
    // end of the phase: every row is stored.  ONE barrier instruction for all sets (the level loops above are
    // separate instances per set; a barrier inside them would be reached at different program counters)
    sw_bar_sync_id(4, NS * nct);
    if (set == 0 && t == 0) {
        const int last = nlev ? sw_lds_v2(lev_u32 + 8u * (uint32_t)(nlev - 1)).y : 0;
        sw_st_progress(progress, done_base + last);
    }
}

template <int K, int R, int MAXT, bool DBG, int P>
__global__ void __launch_bounds__(MAXT, 1) sweep_kernel(const SweepArgs a) {
    constexpr int STAGE = sw_stage_bytes(K, P);
    constexpr int OFF_RHS = sw_page_bytes(K, true, P);
    extern __shared__ __align__(128) unsigned char sw_smem[];
    const int *blk = a.blocks + SW_BLOCK_INTS * blockIdx.x;
    const int n_rows = blk[0], page0 = blk[1], nlev_l = blk[2], nlev_u = blk[3], lev_off = blk[4];
    if (n_rows <= 0) return;
    const int S = a.stages, smask = S - 1, nct = a.nct, NS = a.sets;
    uint64_t *full = (uint64_t *)sw_smem;
    uint64_t *empty = full + SW_MAX_STAGES;
    uint64_t *lflush = empty + SW_MAX_STAGES;
    int *progress = (int *)(lflush + 1);
    int *landed = progress + 1;
    int *levs = (int *)(sw_smem + sw_ctl_bytes());
    double *xs = (double *)((unsigned char *)levs + (((size_t)a.max_lev * 8 + 15) & ~(size_t)15));
    size_t off = (size_t)((unsigned char *)xs - sw_smem) + ((((size_t)a.wmask + 2) * 8 + 15) & ~(size_t)15);
    off = (off + 127) & ~(size_t)127;
    unsigned char *stage0 = sw_smem + off;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            sw_mbar_init(&full[s], 1);
            sw_mbar_init(&empty[s], 1);
        }
        sw_mbar_init(lflush, SW_WRITERS);
        *progress = 0;
        *landed = 0;
        xs[a.wmask + 1] = 0.0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // level table as (start, end) position pairs: one shared-memory load per level in the compute loop
    for (int i = tid; i < nlev_l + nlev_u; i += blockDim.x) {
        const int e = a.levtab[lev_off + i];
        const int st = (i == 0 || i == nlev_l) ? 0 : a.levtab[lev_off + i - 1];
        levs[2 * i] = st;
        levs[2 * i + 1] = e;
    }
    __syncthreads();
    const int n_pages = (n_rows + P - 1) / P;
    const bool do_l = a.phases & 1, do_u = a.phases & 2;
    const int gq_u = do_l ? n_pages : 0;             // first ring ordinal of the U pages
    const int done_u = do_l ? n_rows : 0;
    const int total = n_pages * ((do_l ? 1 : 0) + (do_u ? 1 : 0));
    const int ncomp = NS * nct;
    if (tid < ncomp) {
        // ------------------------------------------------------------ compute warps (NS sets)
        const int set = tid / nct, t = tid - set * nct;
        long long *dbg = (DBG && a.dbg) ? a.dbg + 64 * blockIdx.x : nullptr;
        if (DBG && dbg && t == 0) dbg[16 * set + 2] = 0;
        const uint32_t stage0_u32 = sw_smem_u32(stage0), xs_u32 = sw_smem_u32(xs), lev_u32 = sw_smem_u32(levs);
        if (do_l)
            sweep_compute<K, R, false, DBG, P>(set, NS, t, nct, lev_u32, nlev_l, 0, smask, landed, stage0_u32, xs_u32,
                                            a.wmask, progress, 0, dbg, a.flags);
        if (do_u)
            sweep_compute<K, R, true, DBG, P>(set, NS, t, nct, lev_u32 + 8u * (uint32_t)nlev_l, nlev_u, gq_u, smask,
                                           landed, stage0_u32, xs_u32, a.wmask, progress, done_u, dbg, a.flags);
    } else if (DBG && (a.flags & 256)) {
        // diagnostics: no helper warps at all (with flags 252: the bare level hand-over of the compute sets)
    } else if (tid == ncomp) {
        // ------------------------------------------------------------ issuer: one TMA group per page
        for (int i = 0; i < total; ++i) {
            const bool upper = !(do_l && i < n_pages);
            const int q = upper ? i - gq_u : i;
            const int s = i & smask;
            if (i >= S) sw_mbar_wait(&empty[s], (uint32_t)(((i / S) - 1) & 1));
            if (upper && do_l && q == 0) sw_mbar_wait(lflush, 0);   // the U right-hand side is complete and visible
            const uint32_t pb = upper ? sw_page_bytes(K, true, P) : sw_page_bytes(K, false, P);
            const unsigned char *src = (upper ? a.pages_u : a.pages_l) + (size_t)(page0 + q) * pb;
            const double *rsrc = ((upper && do_l) ? a.tmp : a.rhs) + (size_t)(page0 + q) * P;
            unsigned char *st = stage0 + (size_t)s * STAGE;
            const bool with_add = upper && a.add;
            sw_mbar_arrive_tx(&full[s], pb + P * (with_add ? 16 : 8));
            sw_bulk_g2s(st, src, pb, &full[s]);
            sw_bulk_g2s(st + OFF_RHS, rsrc, P * 8, &full[s]);
            if (with_add) sw_bulk_g2s(st + OFF_RHS + P * 8, a.add + (size_t)(page0 + q) * P, P * 8, &full[s]);
            // pull the operands of a page further ahead than the ring into L2 (HBM latency > ring depth)
            const int j = i + 2 * S;
            if (j < total && !(DBG && (a.flags & 2))) {
                const bool up2 = !(do_l && j < n_pages);
                const int q2 = up2 ? j - gq_u : j;
                const uint32_t pb2 = up2 ? sw_page_bytes(K, true, P) : sw_page_bytes(K, false, P);
                sw_prefetch_l2((up2 ? a.pages_u : a.pages_l) + (size_t)(page0 + q2) * pb2, pb2);
            }
        }
    } else if (tid == ncomp + 32) {
        // ------------------------------------------------------------ gate: pages landed so far, one counter the
        // compute threads read with a plain load (a try_wait per thread and page cost ~400 cycles per level)
        for (int i = 0; i < total; ++i) {
            sw_mbar_wait(&full[i & smask], (uint32_t)((i / S) & 1));
            sw_st_landed(landed, i + 1);
        }
    } else if (tid >= ncomp + 64) {
        // ------------------------------------------------------------ writers: warp w takes pages w, w + 3, ...
        const int wt = tid - ncomp - 64, lane = wt & 31, ww = wt >> 5;
        for (int ph = 0; ph < 2; ++ph) {
            const bool upper = ph == 1;
            if (upper ? !do_u : !do_l) continue;
            const int gq0 = upper ? gq_u : 0, done_base = upper ? done_u : 0;
            const bool to_tmp = !upper && do_u;
            const bool with_add = upper && a.add;
            for (int q = ww; q < n_pages; q += SW_WRITER_WARPS) {
                const int gq = gq0 + q, s = gq & smask;
                const int rows = min(P, n_rows - q * P);
                while (sw_ld_progress(progress) < done_base + q * P + rows) __nanosleep(a.wsleep);
                sw_mbar_wait(&full[s], (uint32_t)((gq / S) & 1));    // (complete long ago) async-proxy visibility
                asm volatile("fence.acq_rel.cta;" ::: "memory");
                const unsigned char *st = stage0 + (size_t)s * STAGE;
                const double *xv = (const double *)(st + OFF_RHS);
                const int *ids = (const int *)(st + 8 * K * P + (upper ? 16 * P : 0)) + (to_tmp ? P : 0);
                double x[P / 32];
                int id[P / 32];
#pragma unroll
                for (int u = 0; u < P / 32; ++u) {
                    const int o = u * 32 + lane;
                    x[u] = xv[o];
                    if (with_add) x[u] = xv[P + o] + x[u];
                    id[u] = ids[o];
                }
                double *dst = to_tmp ? a.tmp : a.out;     // tmp: U schedule position of the row; out: the row
#pragma unroll
                for (int u = 0; u < P / 32; ++u)
                    if (u * 32 + lane < rows && !(DBG && (a.flags & 1))) dst[id[u]] = x[u];
                __syncwarp();
                if (lane == 0) sw_mbar_arrive(&empty[s]);
            }
            if (to_tmp) {
                // generic-proxy stores -> the issuer's bulk (async-proxy) loads
                __threadfence();
                asm volatile("fence.proxy.async;" ::: "memory");
                sw_mbar_arrive(lflush);
            }
        }
    }
}

// right-hand side in schedule order: out[i] = base[row] -/+ (A y)[row] for row = rowof[i] (0 for padding)
//   rp == nullptr: out[i] = base[row]        mode 0: (A y)[row]   mode 1: base - A y   mode 2: base + A y
// and, for the fused `add + x`, add_out[i] = add[rowof_u[i]] (the added vector in U schedule order)
__global__ void sweep_rhs_kernel(int npad, const int *__restrict__ rowof, const int *__restrict__ rp,
                                 const int *__restrict__ ci, const double *__restrict__ val,
                                 const double *__restrict__ y, const double *__restrict__ base, int mode,
                                 double *__restrict__ out, const int *__restrict__ rowof_u,
                                 const double *__restrict__ add, double *__restrict__ add_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npad) return;
    if (add_out) {
        const int ru = rowof_u[i];
        add_out[i] = ru >= 0 ? add[ru] : 0.0;
    }
    const int row = rowof[i];
    double res = 0.0;
    if (row >= 0) {
        if (rp) {
            double s = 0.0;
            for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) s += val[k] * y[ci[k]];
            res = mode == 0 ? s : (mode == 1 ? base[row] - s : base[row] + s);
        } else {
            res = base[row];
        }
    }
    out[i] = res;
}

// one thread per row: operands of the row into its page slot
template <bool UPPER>
__global__ void sweep_fill_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                  const double *__restrict__ val, int K, const int *__restrict__ gpos,
                                  const int *__restrict__ lpos, const int *__restrict__ gpos_u, int wmask,
                                  int P, unsigned char *pages, int *bad_row) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const int g = gpos[row], q = g / P, off = g & (P - 1);
    const size_t pb = (size_t)P * (UPPER ? 10 * K + 20 : 10 * K + 8);
    unsigned char *pg = pages + (size_t)q * pb;
    double *cf = (double *)pg;
    unsigned short *cd = (unsigned short *)(pg + (UPPER ? 8 * K * P + 20 * P : 8 * K * P + 8 * P));
    int kk = 0;
    double diag = 1.0;
    bool seen = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (UPPER ? j > row : j < row) {
            if (kk < K) {
                cf[kk * P + off] = val[k];
                cd[kk * P + off] = (unsigned short)(lpos[j] & wmask);
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {       // padding: coefficient 0 times the window's zero slot
        cf[kk * P + off] = 0.0;
        cd[kk * P + off] = (unsigned short)(wmask + 1);
    }
    if (UPPER) {
        double *pv = (double *)(pg + 8 * K * P);
        pv[off] = diag;
        pv[P + off] = safe_reciprocal(diag);
        ((int *)(pg + 8 * K * P + 16 * P))[off] = row;
        if (!seen || fabs(diag) < 1e-300) atomicMin(bad_row, row);
    } else {
        int *ids = (int *)(pg + 8 * K * P);
        ids[off] = row;
        ids[P + off] = gpos_u[row];
    }
}

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

/* rows per operand page for k operand slots per row: 256, or 64 for long rows (k > 8: the pages of the levels the
 * compute sets work on at once must fit the ring) */
extern "C" int ddilu_sweep_page_rows(int k) { return k > 8 ? 64 : SW_PAGE; }

extern "C" int ddilu_sweep_helper_threads(void) { return SW_HELPERS; }

extern "C" long long ddilu_sweep_page_bytes(int k, int upper) {
    return sw_page_bytes(k, upper != 0, ddilu_sweep_page_rows(k));
}

extern "C" long long ddilu_sweep_smem_bytes(int k, int stages, int window, int max_lev) {
    return (long long)sw_smem_bytes(k, stages, window, max_lev, ddilu_sweep_page_rows(k));
}

extern "C" int ddilu_sweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                                const int *gpos, const int *lpos, const int *gpos_u, int window,
                                unsigned char *pages, int *bad_row, void *stream) {
    if (n <= 0) return DDILU_OK;
    if (k < 1 || k > 24 || window < 32 || (window & (window - 1)) || window > 32768) return DDILU_ERR_ARG;
    const int threads = 256, grid = div_up(n, threads), page_rows = ddilu_sweep_page_rows(k);
    if (upper)
        sweep_fill_kernel<true><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, lpos, gpos_u,
                                                                  window - 1, page_rows, pages, bad_row);
    else
        sweep_fill_kernel<false><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, lpos, gpos_u,
                                                                   window - 1, page_rows, pages, bad_row);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_sweep_rhs(int npad, const int *rowof, const int *row_ptr, const int *col_idx,
                               const double *values, const double *y, const double *base, int mode, double *out,
                               const int *rowof_u, const double *add, double *add_out, void *stream) {
    if (npad <= 0) return DDILU_OK;
    if (mode < 0 || mode > 2 || (!row_ptr && !base) || (row_ptr && mode != 0 && !base) || (add_out && (!add || !rowof_u)))
        return DDILU_ERR_ARG;
    sweep_rhs_kernel<<<div_up(npad, 256), 256, 0, ST(stream)>>>(npad, rowof, row_ptr, col_idx, values, y, base, mode,
                                                               out, rowof_u, add, add_out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

namespace {
long long *g_sweep_dbg = nullptr;
int g_sweep_wsleep = 100, g_sweep_flags = 0;
template <int K, int R, int MAXT, bool DBG, int P>
int launch_sweep_one(int n_blocks, const SweepArgs &a, size_t smem, cudaStream_t st) {
    static size_t attr = 0;     // monotone: the largest dynamic shared-memory size requested so far
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (attr < smem) {
            DDILU_CHECK(cudaFuncSetAttribute(sweep_kernel<K, R, MAXT, DBG, P>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = smem;
        }
    }
    sweep_kernel<K, R, MAXT, DBG, P><<<n_blocks, a.sets * a.nct + SW_HELPERS, smem, st>>>(a);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
template <int K, int R>
int launch_sweep_kr(int n_blocks, const SweepArgs &a, size_t smem, cudaStream_t st) {
    const int threads = a.sets * a.nct + SW_HELPERS;      // register budget follows the CTA size
#ifdef DDILU_EXPERIMENTS
    if (a.dbg || a.flags) return launch_sweep_one<K, R, 1024, true, SW_PAGE>(n_blocks, a, smem, st);
#endif
    if (threads <= 768) return launch_sweep_one<K, R, 768, false, SW_PAGE>(n_blocks, a, smem, st);
    return launch_sweep_one<K, R, 1024, false, SW_PAGE>(n_blocks, a, smem, st);
}
template <int K>
int launch_sweep(int rows_per_thread, int n_blocks, const SweepArgs &a, size_t smem, cudaStream_t st) {
    switch (rows_per_thread) {
        case 1: return launch_sweep_kr<K, 1>(n_blocks, a, smem, st);
        case 2: return launch_sweep_kr<K, 2>(n_blocks, a, smem, st);
        default: return DDILU_ERR_ARG;
    }
}
// long rows (ILUT / ILU(k) / 27-point interface factors, up to 24 dependencies): the K coefficients and K window
// addresses of a row take ~100 registers, so the CTA is capped at 512 threads (one row per thread), and the pages
// hold 64 rows so that the levels in flight fit the ring
template <int K>
int launch_sweep_long(int rows_per_thread, int n_blocks, const SweepArgs &a, size_t smem, cudaStream_t st) {
    if (rows_per_thread != 1 || a.sets * a.nct + SW_HELPERS > 512) return DDILU_ERR_ARG;
    return launch_sweep_one<K, 1, 512, false, 64>(n_blocks, a, smem, st);
}
}  // namespace

#ifdef DDILU_EXPERIMENTS   // diagnostics of scripts/probe_sweep.py
/* diagnostics: 64 int64 cycle counters per block */
extern "C" int ddilu_sweep_set_debug(long long *buf) {
    g_sweep_dbg = buf;
    return DDILU_OK;
}

extern "C" int ddilu_sweep_set_tuning(int writer_sleep_ns, int flags) {
    g_sweep_wsleep = writer_sleep_ns;
    g_sweep_flags = flags;
    return DDILU_OK;
}

#endif  // DDILU_EXPERIMENTS
/* phases: 1 = x = L^-1 rhs, 2 = x = U^-1 rhs, 3 = x = U^-1 L^-1 rhs; rhs in the schedule order of the first
 * phase (ddilu_sweep_rhs), results by row: out[row] = x (+ add[U position of the row], phases 2 and 3) */
extern "C" int ddilu_sweep_solve(int n_blocks, const int *blocks, const int *levtab, const unsigned char *pages_l,
                                 const unsigned char *pages_u, int k, int window, int stages, int sets, int nct,
                                 int rows_per_thread, int max_lev, int phases, const double *rhs, double *tmp,
                                 double *out, const double *add, void *stream) {
    if (n_blocks <= 0) return DDILU_OK;
    if (phases < 1 || phases > 3 || stages < 4 || stages > SW_MAX_STAGES || (stages & (stages - 1)) || sets < 2 ||
        sets > 3 || nct < 32 || (nct & 31) || sets * nct + SW_HELPERS > 1024 || window < 32 || (window & (window - 1)) || window > 32768 || (phases == 3 && !tmp) ||
        (add && !(phases & 2)))
        return DDILU_ERR_ARG;
    SweepArgs a{blocks, levtab, pages_l, pages_u, rhs, tmp, out, add, phases, window - 1, stages, sets, nct, max_lev,
                g_sweep_wsleep, g_sweep_flags, g_sweep_dbg};
    const size_t smem = sw_smem_bytes(k, stages, window, max_lev, ddilu_sweep_page_rows(k));
    if (smem > 227 * 1024) return DDILU_ERR_ARG;
    switch (k) {
        case 2: return launch_sweep<2>(rows_per_thread, n_blocks, a, smem, ST(stream));
        case 3: return launch_sweep<3>(rows_per_thread, n_blocks, a, smem, ST(stream));
        case 4: return launch_sweep<4>(rows_per_thread, n_blocks, a, smem, ST(stream));
        case 8: return launch_sweep<8>(rows_per_thread, n_blocks, a, smem, ST(stream));
        case 16: return launch_sweep_long<16>(rows_per_thread, n_blocks, a, smem, ST(stream));
        case 24: return launch_sweep_long<24>(rows_per_thread, n_blocks, a, smem, ST(stream));
        default: return DDILU_ERR_ARG;
    }
}
