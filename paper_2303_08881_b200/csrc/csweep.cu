// Cluster sweep: L^-1 / U^-1 on a block-diagonal factor whose blocks are LARGE and deep -- the interior factors
// L_B / U_B of the two-level preconditioners, one independent diagonal block per subdomain (precond.py:236-238,
// 244-246 `_interior_solve`; arithmetic of sparse.py:228-272 `_lower_solve` / `_upper_solve`: row sums left to
// right in storage order, every product rounded, IEEE division -> bit-exact).
//
// Why its own kernel.  At 256^3 / p = 8 an interior factor has 16.4 M rows in 379 levels of ~5 k rows per
// subdomain.  The tiled kernel (csrc/tiled.cu) pays 22 in-tile levels per 512 rows plus the wavefront of 46 tile
// levels and sits at 0.35 of the HBM roofline; a CTA per block (csrc/sweep.cu) has one SM's bandwidth.  Here a
// THREAD-BLOCK CLUSTER of up to 16 CTAs owns a block and walks its levels together:
//
//   * every level of the block is cut into contiguous chunks, chunk r belongs to CTA r of the cluster;
//   * a CTA keeps every value IT needs in a window of W doubles (4 095; 8 191 for long rows) of its OWN shared memory:
//     its own results and the results of other CTAs that its rows depend on (halo values), numbered level by level
//     (own rows of the level, then the level's halo values), value p in xs[p mod W]; setup checks that no row reads
//     further back than W positions behind the end of its own level.  A dependency is a 16-bit window slot, read
//     with a plain shared-memory load; slot W holds 0.0 for padded operands;
//   * a producer PUSHES a result to the (<= 3; long rows: 4) other CTAs that need it: st.async through distributed
//     shared memory into the consumer's window slot, completing bytes on the consumer's mbarrier -- data and signal
//     travel together, no fence, no cluster-scope release (barrier.cluster.arrive.release costs a MEMBAR.ALL.GPU per
//     level, ~700 cycles: measured);
//   * ONE mbarrier wait per level: the phase of level l completes when all warps of the own CTA have stored their
//     level-l rows, all halo bytes of level l have landed (expect_tx) and every warp of every CTA this one exchanges
//     values with has finished level l (a token arrive -- the flow control that makes the window slots safe to
//     overwrite; CTAs that exchange nothing are not coupled);
//   * a STEP is (a part of) a CTA's chunk of a level, at most one row per compute thread; chunks wider than the CTA
//     are cut into several steps at setup.  Operands are structure-of-arrays in the CTA's schedule order (K
//     coefficients, K slots + push targets packed in 32-bit words, (pivot, reciprocal) pairs for U, the row id
//     only when a chunk is not a range of consecutive rows); ONE lane of a 25th warp streams them into a ring of
//     shared-memory stages with bulk copies (cp.async.bulk + complete_tx on full[stage]), the compute threads take
//     them with plain loads and free the stage through empty[stage]; the results leave by row after the arrive.
//     (Operands prefetched into registers stalled every consumer on the youngest load in flight -- six scoreboards
//     per warp --, per-thread cp.async cost ~200 warp instructions per step: DESIGN.md 5.8.)
//
// Bytes moved per row (three dependencies): 24 + 12 (+ 16 pivot pair) operands + 8 right-hand side + 8 result = 52 (L)
// / 68 (U), against the algorithmic 12 nnz + 4 + 16 = 56 / 68.
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int CS_STEP_INTS = 8;       // per CTA and step: first / end operand position, window slot of the first row,
                                      // first row (-1: row ids), halo bytes of the level, flags, 0, 0
constexpr int CS_CTA_INTS = 4;        // per CTA: first position in the operand arrays, signal mask | arrivals << 16, first step, number of steps
constexpr unsigned CS_NO_PUSH = 0xffffu;
constexpr int CS_WAIT = 1, CS_ARRIVE = 2;   // step flags: first / last step of its level
constexpr int CS_MAX_DEPTH = 4;

// Two shapes of the kernel, chosen by the operand slots per row K:
//   short rows (K <= 4: 5- / 7-point ILU(0) factors): wide levels -- 768 compute threads, a window of 4 095 doubles,
//     three push targets per row as slot << 4 | rank (clusters up to 16), the step table in shared memory;
//   long rows (K = 20: 27-point / ILUT factors): narrow deep levels that reach further back -- 256 compute threads, a
//     window of 8 191 doubles, four push targets as slot << 3 | rank (clusters up to 8), the step table (thousands
//     of levels) read from global memory one step ahead.
template <int K>
struct CsCfg {
    static constexpr bool LONG = K > 4;
    static constexpr int NT = LONG ? 256 : 768;           // compute threads = rows of a step at most; one more warp feeds the ring
    static constexpr int WIN = LONG ? 8191 : 4095;        // doubles per CTA; slot WIN holds 0.0
    static constexpr int RB = LONG ? 3 : 4;               // rank bits of a push target
    static constexpr int NP = LONG ? 4 : 3;               // push targets per row
    static constexpr int NW = (K + NP + 1) / 2;           // 32-bit words holding a row's K slots and NP push targets
    static constexpr bool TABLE_IN_SMEM = !LONG;
};
__host__ __device__ constexpr bool cs_long(int K) { return K > 4; }
__host__ __device__ constexpr int cs_nt(int K) { return cs_long(K) ? 256 : 768; }
__host__ __device__ constexpr int cs_win(int K) { return cs_long(K) ? 8191 : 4095; }
__host__ __device__ constexpr int cs_rb(int K) { return cs_long(K) ? 3 : 4; }
__host__ __device__ constexpr int cs_np(int K) { return cs_long(K) ? 4 : 3; }
__host__ __device__ constexpr int cs_words(int K) { return (K + cs_np(K) + 1) / 2; }

struct CSweepArgs {
    const int *ctas;                  // CS_CTA_INTS per CTA (block-major, rank-minor)
    const int *steps;                 // CS_STEP_INTS per CTA and step
    const double *coef;               // [K][np]
    const unsigned *code;             // [cs_words(K)][np]: 16-bit halves = K window slots of the dependencies, then the
                                      // push targets slot << rank bits | rank (0xffff = none)
    const int *rowid;                 // [np]
    const double *piv;                // [np][2]: pivot, reciprocal (upper)
    const unsigned char *blob;        // long rows instead of the four arrays: the operands STEP BY STEP, one contiguous block
                                      // per step (r4 = rows rounded up to 4): coef[K][r4] | piv[2][r4] (upper) |
                                      // words[NW][r4] | row ids[r4] -- one bulk copy per step
    const double *b;                  // right-hand side by row
    double *out;                      // results by row
    long long np;
    int max_steps;
    int depth;                        // stages of the operand ring
    long long *dbg;                   // experiments build: 16 cycle counters per CTA and probe thread (first, last)
};

// a stage of the operand ring (structure of arrays, slot = row of the step):
// coef[K][NT] | pivot pairs[2][NT] (upper) | rhs[NT + 2] | words[NW][NT] | row ids[NT]
__host__ __device__ constexpr int cs_stage_bytes(int K, bool upper) {
    return cs_nt(K) * (8 * K + (upper ? 16 : 0) + 4 * cs_words(K) + 4) + 8 * (cs_nt(K) + 2);
}
__host__ __device__ inline size_t cs_ctl_bytes() { return (2 + 2 * CS_MAX_DEPTH) * 8; }   // level pair, full[], empty[]
__host__ __device__ inline size_t cs_table_bytes(int K, int max_steps) {
    return cs_long(K) ? 0 : (size_t)max_steps * CS_STEP_INTS * 4;
}
__host__ __device__ inline size_t cs_smem_bytes(int K, bool upper, int depth, int max_steps) {
    size_t b = cs_ctl_bytes() + cs_table_bytes(K, max_steps) + ((size_t)cs_win(K) + 1) * 8;
    b = (b + 127) & ~(size_t)127;
    return b + (size_t)depth * cs_stage_bytes(K, upper);
}

__device__ __forceinline__ uint32_t cs_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cs_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cs_mapa(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ double cs_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ double cs_lds_at(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
template <int OFF>
__device__ __forceinline__ uint32_t cs_lds_u32_at(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
__device__ __forceinline__ double2 cs_lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void cs_sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ int4 cs_lds_v4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
// a result into another CTA's window, completing 8 bytes on that CTA's mbarrier
__device__ __forceinline__ void cs_push(uint32_t remote_slot, double v, uint32_t remote_bar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_slot),
                 "l"(__double_as_longlong(v)), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void cs_mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void cs_mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cs_mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cs_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive on the own mbarrier: release.cta orders the warp's window stores (made visible to the arriving lane by
// __syncwarp) before the arrive for the readers of the own CTA
__device__ __forceinline__ void cs_mbar_arrive_release(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// token arrive on the mbarrier of another CTA of the cluster: it carries no data (that CTA gets its data through
// cs_push), it only says that this warp's reads of the level are done
__device__ __forceinline__ void cs_mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cs_mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(1000000u)      /* suspend-time hint (ns): sleep until the phase completes */
            : "memory");
    } while (!done);
}
// global -> shared memory, bytes a multiple of 16, both addresses 16-byte aligned; completes bytes on the mbarrier
__device__ __forceinline__ void cs_bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cs_cp_async8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ int cs_ldg_s32(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t cs_half(const uint32_t *w, int i) {     // 16-bit half i of the packed words
    return (i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xffffu);
}

// One CTA of the cluster that owns block blockIdx.x / cluster size.  A CTA walks its STEPS: a step is (a part of)
// the CTA's chunk of a level, at most one row per compute thread -- levels wider than the CTA are cut into several
// steps at setup; only the first step of a level waits, only the last one signals.  Compute thread t owns row t of
// every step; every warp instruction of its loop counts (24 warps share four schedulers), so the operands do NOT
// come by per-thread loads: lane 0 of the feeder warp streams every operand array of a step into a stage of a
// shared-memory ring with one bulk copy each (steps start at multiples of 4 positions, so every run is 16-byte
// aligned), `depth` steps ahead, and a compute thread takes its operands with plain shared-memory loads.
// per step      feeder: wait until the stage is free, bulk copies with complete_tx on full[stage]
//               compute: wait full[stage]; operands -> registers; arrive empty[stage];
//                        (first step of a level) wait for the mbarrier phase of the previous level: own rows
//                        stored, halo landed, every warp of the cluster past it;
//                        K window loads, multiply / subtract chain [, division], window store, pushes;
//                        (last step of a level) arrive at every CTA's mbarrier of the level; result to global memory
template <int K, bool UPPER>
__global__ void __launch_bounds__(CsCfg<K>::NT + 32, 1) csweep_kernel(const CSweepArgs a) {
    using Cfg = CsCfg<K>;
    constexpr int NT = Cfg::NT, NW = Cfg::NW, CS_WINDOW = Cfg::WIN, CS_NP = Cfg::NP, RB = Cfg::RB;
    constexpr int CS_THREADS = NT + 32;
    constexpr uint32_t RMASK = (1u << RB) - 1u;
    constexpr int STAGE = cs_stage_bytes(K, UPPER);
    // short rows: coef[K][NT] | piv[NT][2] (upper) | rhs[NT + 2] | words[NW][NT] | row ids[NT]
    // long rows:  rhs[NT + 2] (unused: b[row id] is loaded directly) | the step's operand block as it lies in the blob
    constexpr int OFF_PIV = 8 * K * NT, OFF_RHS = Cfg::LONG ? 0 : OFF_PIV + (UPPER ? 16 * NT : 0),
                  OFF_W = OFF_PIV + (UPPER ? 16 * NT : 0) + 8 * (NT + 2), OFF_ID = OFF_W + 4 * NW * NT;
    constexpr int OFF_BLK = 8 * (NT + 2);                                  // long rows
    constexpr int REC = 8 * K + (UPPER ? 16 : 0) + 4 * NW + 4;            // operand bytes of a row
    extern __shared__ __align__(128) unsigned char cs_smem[];
    const int *cta = a.ctas + CS_CTA_INTS * blockIdx.x;
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctaid.x;" : "=r"(csize));
    const long long base = cta[0];
    const int step_off = cta[2], nsteps = cta[3];
    // the CTAs this one signals at the end of a level (itself and the CTAs it exchanges values with, a symmetric
    // relation: a producer must know that its consumer is done reading before it overwrites the consumer's window
    // slots, and a coupled pair stays within one level of each other), and how many CTAs signal this one
    const uint32_t sigmask = (uint32_t)cta[1] & 0xffffu;
    const int signallers = cta[1] >> 16;
    const int tid = threadIdx.x, lane = tid & 31;
    const int D = a.depth;
    uint64_t *bars = (uint64_t *)cs_smem;                     // [2]: levels of even / odd index, then full[], empty[]
    int4 *steps = (int4 *)(cs_smem + cs_ctl_bytes());
    double *xs = (double *)((unsigned char *)steps + cs_table_bytes(K, a.max_steps));
    size_t ring_off = cs_ctl_bytes() + cs_table_bytes(K, a.max_steps) + ((size_t)CS_WINDOW + 1) * 8;
    ring_off = (ring_off + 127) & ~(size_t)127;
    const int4 *gsteps = (const int4 *)a.steps + 2 * (size_t)step_off;      // this CTA's step table
    if (Cfg::TABLE_IN_SMEM)
        for (int i = tid; i < 2 * nsteps; i += CS_THREADS) steps[i] = gsteps[i];
    const uint32_t bar_u32 = cs_smem_u32(bars), full_u32 = bar_u32 + 16, empty_u32 = full_u32 + 8 * CS_MAX_DEPTH;
    if (tid == 0) {
        xs[CS_WINDOW] = 0.0;                  // padded operands: coefficient 0 times this slot
        cs_mbar_init(bar_u32, (NT / 32) * signallers);
        cs_mbar_init(bar_u32 + 8, (NT / 32) * signallers);
        for (int s = 0; s < D; ++s) {
            // the feeder's arrive.expect_tx and its asynchronous cp.async arrive
            cs_mbar_init(full_u32 + 8 * s, 2);
            cs_mbar_init(empty_u32 + 8 * s, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cs_cluster_sync();                        // every CTA of the cluster is running, its mbarriers are initialised
    const uint32_t st_u32 = cs_smem_u32(steps), xs_u32 = cs_smem_u32(xs), ring_u32 = cs_smem_u32(cs_smem + ring_off);
    const long long np = a.np;
    // half h (0: positions, slot, first row; 1: halo bytes, flags) of the table entry of step i
    auto entry = [&](int i, int h) -> int4 {
        return Cfg::TABLE_IN_SMEM ? cs_lds_v4(st_u32 + 32u * (uint32_t)i + 16u * (uint32_t)h) : __ldg(gsteps + 2 * i + h);
    };

    if (tid >= NT) {
        // ------------------------------------------------------------ feeder (one lane)
        if (lane == 0) {
            const double *cf = a.coef + base;
            const unsigned *cd = a.code + base;
            const int *ids = a.rowid + base;
            const double *pv = a.piv + 2 * base;
            const int4 none = make_int4(0, 0, 0, 0);
            int4 sv = nsteps > 0 ? entry(0, 0) : none;      // (long rows: the table is in global memory, an entry ahead)
            int4 tfc = (Cfg::LONG && nsteps > 0) ? entry(0, 1) : none;
            int s = 0;
            uint32_t round = 0;               // how often the ring has wrapped
            for (int i = 0; i < nsteps; ++i) {
                const int4 sv1 = i + 1 < nsteps ? entry(i + 1, 0) : none;
                const int4 tf1 = (Cfg::LONG && i + 1 < nsteps) ? entry(i + 1, 1) : none;
                const int rows = sv.y - sv.x;
                const uint32_t st = ring_u32 + (uint32_t)(s * STAGE), full = full_u32 + 8u * (uint32_t)s;
                if (round) cs_mbar_wait(empty_u32 + 8u * (uint32_t)s, (round - 1) & 1u);
                if (rows > 0 && Cfg::LONG) {
                    // long rows: the whole operand block of the step with one bulk copy (35 copies of ~1 KB each, one
                    // per array, made the feeder the bottleneck of the deep narrow levels); b[row id] is loaded by
                    // the compute threads (chunks of 27-point blocks are not row ranges)
                    const uint32_t r4 = (uint32_t)(rows + 3) & ~3u;
                    const uint32_t bytes = r4 * (uint32_t)REC;
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
                    cs_mbar_arrive_tx(full, bytes);
                    cs_bulk_g2s(st + OFF_BLK, a.blob + 16ull * (unsigned long long)(unsigned)tfc.z, bytes, full);
                } else if (rows > 0) {
                    const uint32_t r4 = (uint32_t)(rows + 3) & ~3u;                 // whole 16-byte pieces of every array
                    uint32_t tx = r4 * (uint32_t)(8 * K + 4 * NW + (UPPER ? 16 : 0));
                    uint32_t nb_bulk = 0;
                    const double *bsrc = nullptr;
                    uint32_t bdst = 0;
                    if (sv.w >= 0) {
                        // right-hand side b[row0 .. row0 + rows): element j of the step lands at rhs[j + head] with
                        // head = row0 & 1 -- the 16-byte aligned run by one bulk copy, an odd head / tail element by
                        // an 8-byte cp.async of this thread (signalled through the asynchronous arrive below)
                        const int head = sv.w & 1;
                        const int body = (rows - head) & ~1;
                        bsrc = a.b + sv.w + head;
                        bdst = st + OFF_RHS + 8u * (uint32_t)(2 * head);
                        nb_bulk = 8u * (uint32_t)body;
                        tx += nb_bulk;
                        if (head) cs_cp_async8(st + OFF_RHS + 8u, a.b + sv.w);
                        if (head + body < rows) cs_cp_async8(st + OFF_RHS + 8u * (uint32_t)(head + rows - 1), a.b + sv.w + rows - 1);
                    } else {
                        tx += r4 * 4u;
                    }
                    // second arrival of the phase: when this thread's cp.async copies (if any) have landed
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
                    cs_mbar_arrive_tx(full, tx);
#pragma unroll
                    for (int k = 0; k < K; ++k) cs_bulk_g2s(st + (uint32_t)(8 * k * NT), cf + (long long)k * np + sv.x, 8u * r4, full);
#pragma unroll
                    for (int k = 0; k < NW; ++k) cs_bulk_g2s(st + OFF_W + (uint32_t)(4 * k * NT), cd + (long long)k * np + sv.x, 4u * r4, full);
                    if (UPPER) cs_bulk_g2s(st + OFF_PIV, pv + 2 * (long long)sv.x, 16u * r4, full);      // (pivot, reciprocal) pairs
                    if (sv.w >= 0) {
                        if (nb_bulk) cs_bulk_g2s(bdst, bsrc, nb_bulk, full);
                    } else {
                        cs_bulk_g2s(st + OFF_ID, ids + sv.x, 4u * r4, full);
                    }
                } else {
                    cs_mbar_arrive(full);
                    cs_mbar_arrive(full);
                }
                sv = sv1;
                tfc = tf1;
                if (++s == D) {
                    s = 0;
                    ++round;
                }
            }
        }
    } else {
        // ------------------------------------------------------------ compute threads
        // lane r signals CTA r when the mask says so: the address of that CTA's mbarrier pair (the own CTA's through
        // its shared::cta address)
        uint32_t my_rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(my_rank));
        const bool self = (uint32_t)lane == my_rank;
        const bool signals = (uint32_t)lane < csize && ((sigmask >> lane) & 1u) && !self;
        const uint32_t peer_bar = cs_mapa(bar_u32, signals ? (uint32_t)lane : 0u);
        const uint32_t my8 = ring_u32 + 8u * (uint32_t)tid, my4 = ring_u32 + 4u * (uint32_t)tid;
#ifdef DDILU_EXPERIMENTS
        unsigned tq[6] = {0, 0, 0, 0, 0, 0}, t0 = 0, t1 = 0;
        const bool probe = a.dbg && (tid == 0 || tid == NT - 1);
#define CS_TICK(i)                  \
    if (probe) {                    \
        t1 = (unsigned)clock();     \
        tq[i] += t1 - t0;           \
        t0 = t1;                    \
    }
        if (probe) t0 = (unsigned)clock();
#else
#define CS_TICK(i)
#endif
        int lev = 0;                          // level of the current step
        int s = 0;
        uint32_t round = 0;
        // the table entry of a step is loaded one step ahead (its two shared-memory loads head the step's chain)
        int4 sv_n = make_int4(0, 0, 0, 0), tf_n = sv_n;
        if (nsteps) {
            sv_n = entry(0, 0);
            tf_n = entry(0, 1);
        }
        for (int i = 0; i < nsteps; ++i) {
            const int4 sv = sv_n;
            const int4 tf = tf_n;                                            // halo bytes of the level, flags
            if (i + 1 < nsteps) {
                sv_n = entry(i + 1, 0);
                tf_n = entry(i + 1, 1);
            }
            const uint32_t mybar = bar_u32 + 8u * (uint32_t)(lev & 1);       // phase of this level: own and (offset) peers'
            // the halo bytes of the level (before this warp's arrive: the phase cannot complete without them)
            if (tid == 0 && tf.x) cs_mbar_expect_tx(mybar, (uint32_t)tf.x);
            const uint32_t so = (uint32_t)(s * STAGE);
            const bool have = tid < sv.y - sv.x;
            CS_TICK(0)
            cs_mbar_wait(full_u32 + 8u * (uint32_t)s, round & 1u);
            CS_TICK(1)
            double c[K], rhs = 0.0, d = 1.0, r = 0.0;
            uint32_t w[NW], ad[K];
            int id = 0;
            if (have && Cfg::LONG) {
                const uint32_t r4 = (uint32_t)(sv.y - sv.x + 3) & ~3u;       // the block's arrays have r4 entries each
                const uint32_t blk = ring_u32 + so + OFF_BLK;
                uint32_t p8 = blk + 8u * (uint32_t)tid;
#pragma unroll
                for (int k = 0; k < K; ++k, p8 += 8u * r4) c[k] = cs_lds(p8);
                if (UPPER) {
                    d = cs_lds(p8);
                    r = cs_lds(p8 + 8u * r4);
                }
                uint32_t p4 = blk + (uint32_t)(8 * K + (UPPER ? 16 : 0)) * r4 + 4u * (uint32_t)tid;
#pragma unroll
                for (int k = 0; k < NW; ++k, p4 += 4u * r4) w[k] = cs_lds_u32_at<0>(p4);
                id = (int)cs_lds_u32_at<0>(p4);
                rhs = __ldg(a.b + id);
#pragma unroll
                for (int k = 0; k < K; ++k) ad[k] = xs_u32 + 8u * cs_half(w, k);
            } else if (have) {
#pragma unroll
                for (int k = 0; k < K; ++k) c[k] = cs_lds(my8 + so + (uint32_t)(8 * k * NT));
#pragma unroll
                for (int k = 0; k < NW; ++k) w[k] = cs_lds_u32_at<OFF_W>(my4 + so + (uint32_t)(4 * k * NT));
                if (UPPER) {
                    const double2 dr = cs_lds_f64x2(ring_u32 + so + OFF_PIV + 16u * (uint32_t)tid);
                    d = dr.x;
                    r = dr.y;
                }
                if (sv.w >= 0) {
                    id = sv.w + tid;
                    rhs = cs_lds_at<OFF_RHS>(my8 + so + 8u * (uint32_t)(sv.w & 1));
                } else {                                // rows by id (27-point blocks under RCM): a dependent load on the
                    id = (int)cs_lds_u32_at<OFF_ID>(my4 + so);      // spot -- a gather by the feeder warp measured slower
                    rhs = __ldg(a.b + id);
                }
#pragma unroll
                for (int k = 0; k < K; ++k) ad[k] = xs_u32 + 8u * cs_half(w, k);
            }
            // the stage may be refilled (the loads above have returned: their values were used)
            __syncwarp();
            if (lane == 0) cs_mbar_arrive(empty_u32 + 8u * (uint32_t)s);
            if (++s == D) {
                s = 0;
                ++round;
            }
            CS_TICK(2)
            // previous level: own rows stored, halo landed, every warp of the cluster past it
            if ((tf.y & CS_WAIT) && lev) cs_mbar_wait(bar_u32 + 8u * (uint32_t)((lev - 1) & 1), (uint32_t)(((lev - 1) >> 1) & 1));
            CS_TICK(3)
            double res = 0.0;
            if (have) {
                double v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) v[k] = cs_lds(ad[k]);
                double sum = rhs;
                // -fmad=false: every product is rounded before it is subtracted
#pragma unroll
                for (int k = 0; k < K; ++k) sum -= c[k] * v[k];
                if (UPPER) sum = exact_div(sum, d, r);
                int sl = sv.z + tid;
                sl -= sl >= CS_WINDOW ? CS_WINDOW : 0;
                cs_sts(xs_u32 + 8u * (uint32_t)sl, sum);
                // to the other CTAs that need the value (rows on the border of a chunk; the targets of a row are
                // stored front to back, so one test tells the common case "none")
                if (cs_half(w, K) != CS_NO_PUSH) {
#pragma unroll
                    for (int k = 0; k < CS_NP; ++k) {
                        const uint32_t pp = cs_half(w, K + k);
                        if (pp != CS_NO_PUSH) cs_push(cs_mapa(xs_u32 + 8u * (pp >> RB), pp & RMASK), sum, cs_mapa(mybar, pp & RMASK));
                    }
                }
                res = sum;
            }
            CS_TICK(4)
            if (tf.y & CS_ARRIVE) {
                // this warp is through the level: one arrive per CTA of the cluster (lane r -> CTA r)
                __syncwarp();
                if (self) cs_mbar_arrive_release(mybar);
                if (signals) cs_mbar_arrive_cluster(peer_bar + 8u * (uint32_t)(lev & 1));
                ++lev;
            }
            // behind the arrive: the hand-over must not wait for the store
            if (have) a.out[id] = res;
            CS_TICK(5)
        }
        // the last phase: nobody pushes into this CTA's window or signals its mbarriers any more
        if (lev) cs_mbar_wait(bar_u32 + 8u * (uint32_t)((lev - 1) & 1), (uint32_t)(((lev - 1) >> 1) & 1));
#ifdef DDILU_EXPERIMENTS
        if (probe) {
            long long *o = a.dbg + 16 * (2 * blockIdx.x + (tid ? 1 : 0));
            for (int q = 0; q < 6; ++q) o[q] = tq[q];
        }
#endif
#undef CS_TICK
    }
    cs_cluster_sync();
}

// one thread per row: operands of the row into its position of the CTA-local schedule order
template <bool UPPER>
__global__ void csweep_fill_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                   const double *__restrict__ val, int K, const int *__restrict__ gpos,
                                   const int *__restrict__ dep_slot, int window, long long np, double *coef,
                                   unsigned short *code, int *rowid, double *piv, int *bad_row) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const long long g = gpos[row];
    int kk = 0;
    double diag = 1.0;
    bool seen = false;
    // half kk of the row's packed words: word kk / 2 of the [words][np] array, 16-bit half kk % 2
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (UPPER ? j > row : j < row) {
            if (kk < K) {
                coef[(long long)kk * np + g] = val[k];
                code[2 * ((long long)(kk >> 1) * np + g) + (kk & 1)] = (unsigned short)dep_slot[k];
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {       // padding: coefficient 0 times the zero slot
        coef[(long long)kk * np + g] = 0.0;
        code[2 * ((long long)(kk >> 1) * np + g) + (kk & 1)] = (unsigned short)window;
    }
    rowid[g] = row;
    if (UPPER) {
        piv[2 * g] = diag;
        piv[2 * g + 1] = safe_reciprocal(diag);
        if (!seen || fabs(diag) < 1e-300) atomicMin(bad_row, row);
    }
}

// long rows: the record of a row inside the operand block of its step (block at byte blk_base[row], arrays of r4[row]
// entries, the row at entry off[row])
template <bool UPPER>
__global__ void csweep_fill_long_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                        const double *__restrict__ val, int K, int NW, int NP,
                                        const long long *__restrict__ blk_base, const int *__restrict__ r4s,
                                        const int *__restrict__ offs, const int *__restrict__ dep_slot, int window,
                                        unsigned char *blob, int *bad_row) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const long long r4 = r4s[row], off = offs[row];
    unsigned char *blk = blob + blk_base[row];
    double *cf = (double *)blk;
    double *pv = cf + (long long)K * r4;
    unsigned short *hv = (unsigned short *)(blk + (8LL * K + (UPPER ? 16 : 0)) * r4);
    int *ids = (int *)(blk + (8LL * K + (UPPER ? 16 : 0) + 4LL * NW) * r4);
    int kk = 0;
    double diag = 1.0;
    bool seen = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (UPPER ? j > row : j < row) {
            if (kk < K) {
                cf[kk * r4 + off] = val[k];
                hv[2 * ((kk >> 1) * r4 + off) + (kk & 1)] = (unsigned short)dep_slot[k];
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {       // padding: coefficient 0 times the zero slot
        cf[kk * r4 + off] = 0.0;
        hv[2 * ((kk >> 1) * r4 + off) + (kk & 1)] = (unsigned short)window;
    }
    for (int q = K; q < K + NP; ++q) hv[2 * ((q >> 1) * r4 + off) + (q & 1)] = (unsigned short)0xffff;    // no push target (yet)
    ids[off] = row;
    if (UPPER) {
        pv[off] = diag;
        pv[r4 + off] = safe_reciprocal(diag);
        if (!seen || fabs(diag) < 1e-300) atomicMin(bad_row, row);
    }
}

namespace {
long long *g_csweep_dbg = nullptr;
template <int K, bool UPPER>
int cs_prepare(size_t smem) {
    if (smem > 227 * 1024) return DDILU_ERR_ARG;
    static size_t attr = 0;
    static bool nonportable = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!nonportable) {
        DDILU_CHECK(cudaFuncSetAttribute(csweep_kernel<K, UPPER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        nonportable = true;
    }
    if (attr < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(csweep_kernel<K, UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    return DDILU_OK;
}

inline void cs_config(cudaLaunchConfig_t &cfg, cudaLaunchAttribute *at, int n_clusters, int csize, int threads,
                      size_t smem, cudaStream_t st) {
    cfg = cudaLaunchConfig_t{};
    cfg.gridDim = dim3((unsigned)(n_clusters * csize));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
}

template <int K, bool UPPER>
int cs_launch(int n_blocks, int csize, const CSweepArgs &a, cudaStream_t st) {
    const size_t smem = cs_smem_bytes(K, UPPER, a.depth, a.max_steps);
    const int rc = cs_prepare<K, UPPER>(smem);
    if (rc) return rc;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cs_config(cfg, at, n_blocks, csize, cs_nt(K) + 32, smem, st);
    DDILU_CHECK(cudaLaunchKernelEx(&cfg, csweep_kernel<K, UPPER>, a));
    return DDILU_OK;
}

template <int K, bool UPPER>
int cs_active(int csize, size_t smem, int *out) {
    const int rc = cs_prepare<K, UPPER>(smem);
    if (rc) return rc;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cs_config(cfg, at, 64, csize, cs_nt(K) + 32, smem, nullptr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, csweep_kernel<K, UPPER>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *out = n;
    return DDILU_OK;
}
}  // namespace

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

#ifdef DDILU_EXPERIMENTS   // diagnostics of scripts/probe_csweep.py: 16 int64 cycle counters per CTA and probe thread
extern "C" int ddilu_csweep_set_debug(long long *buf) {
    g_csweep_dbg = buf;
    return DDILU_OK;
}
#endif

/* k = operand slots per row (3, 4: short rows; 20: long rows) selects the shape of the kernel */
/* compute threads of a CTA of the cluster sweep = rows of a step at most */
extern "C" int ddilu_csweep_threads(int k) { return cs_nt(k); }

/* doubles of a CTA's window (own and halo values): no row may read further back (device.build_csweep checks) */
extern "C" int ddilu_csweep_window(int k) { return cs_win(k); }

/* CTAs other than its own that may need a row's result */
extern "C" int ddilu_csweep_max_push(int k) { return cs_np(k); }

/* a push target is slot << rank_bits | rank: clusters of at most 1 << rank_bits CTAs */
extern "C" int ddilu_csweep_rank_bits(int k) { return cs_rb(k); }

/* 32-bit words per row holding its k dependency slots and its push targets */
extern "C" int ddilu_csweep_code_words(int k) { return cs_words(k); }

extern "C" long long ddilu_csweep_smem_bytes(int k, int upper, int depth, int max_steps) {
    return (long long)cs_smem_bytes(k, upper != 0, depth, max_steps);
}

/* clusters of `cluster_size` CTAs of the sweep kernel that can be resident at once (0: the size cannot be launched) */
extern "C" int ddilu_csweep_active_clusters(int cluster_size, int k, int depth, int max_steps) {
    if (cluster_size < 1 || cluster_size > 16 || depth < 2 || depth > CS_MAX_DEPTH) return 0;
    int n = 0, rc = DDILU_ERR_ARG;
    if (k == 3) rc = cs_active<3, true>(cluster_size, cs_smem_bytes(3, true, depth, max_steps), &n);
    if (k == 4) rc = cs_active<4, true>(cluster_size, cs_smem_bytes(4, true, depth, max_steps), &n);
    if (k == 20) rc = cs_active<20, true>(cluster_size, cs_smem_bytes(20, true, depth, max_steps), &n);
    return rc == DDILU_OK ? n : 0;
}

extern "C" int ddilu_csweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                                 const int *gpos, const int *dep_slot, long long np, double *coef, unsigned *code,
                                 int *rowid, double *piv, int *bad_row, void *stream) {
    if (n <= 0) return DDILU_OK;
    if (k != 3 && k != 4 && k != 20) return DDILU_ERR_ARG;
    const int threads = 256, grid = div_up(n, threads);
    if (upper)
        csweep_fill_kernel<true><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, dep_slot,
                                                                   cs_win(k), np, coef, (unsigned short *)code, rowid,
                                                                   piv, bad_row);
    else
        csweep_fill_kernel<false><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, dep_slot,
                                                                    cs_win(k), np, coef, (unsigned short *)code, rowid,
                                                                    piv, bad_row);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* long rows (k = 20): a row's operands inside the block of its step */
extern "C" int ddilu_csweep_fill_long(int n, const int *row_ptr, const int *col_idx, const double *values, int upper,
                                      int k, const long long *blk_base, const int *r4, const int *off,
                                      const int *dep_slot, unsigned char *blob, int *bad_row, void *stream) {
    if (n <= 0) return DDILU_OK;
    if (!cs_long(k) || k != 20) return DDILU_ERR_ARG;
    const int threads = 256, grid = div_up(n, threads);
    if (upper)
        csweep_fill_long_kernel<true><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, cs_words(k), cs_np(k),
                                                                        blk_base, r4, off, dep_slot, cs_win(k), blob, bad_row);
    else
        csweep_fill_long_kernel<false><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, cs_words(k), cs_np(k),
                                                                         blk_base, r4, off, dep_slot, cs_win(k), blob, bad_row);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* bytes of a row's operands in a long-row block */
extern "C" int ddilu_csweep_long_record_bytes(int k, int upper) { return 8 * k + (upper ? 16 : 0) + 4 * cs_words(k) + 4; }

/* out[row] = (L^-1 b)[row] (upper 0, unit diagonal) or (U^-1 b)[row] (upper 1) for a block-diagonal factor laid out
 * by ddilu_csweep_fill: n_blocks clusters of cluster_size CTAs */
extern "C" int ddilu_csweep_solve(int n_blocks, int cluster_size, const int *ctas, const int *steps, const double *coef,
                                  const unsigned *code, const int *rowid, const double *piv,
                                  const unsigned char *blob, long long np, int k, int upper, int max_steps, int depth,
                                  const double *b, double *out, void *stream) {
    if (n_blocks <= 0) return DDILU_OK;
    if (cluster_size < 1 || cluster_size > 16 || depth < 2 || depth > CS_MAX_DEPTH) return DDILU_ERR_ARG;
    if (cs_long(k) ? !blob : (!coef || !code || !rowid || (upper && !piv))) return DDILU_ERR_ARG;
    CSweepArgs a{ctas, steps, coef, code, rowid, piv, blob, b, out, np, max_steps, depth, g_csweep_dbg};
    if (k == 3) return upper ? cs_launch<3, true>(n_blocks, cluster_size, a, ST(stream)) : cs_launch<3, false>(n_blocks, cluster_size, a, ST(stream));
    if (k == 4) return upper ? cs_launch<4, true>(n_blocks, cluster_size, a, ST(stream)) : cs_launch<4, false>(n_blocks, cluster_size, a, ST(stream));
    if (k == 20) {
        if (cluster_size > (1 << cs_rb(20))) return DDILU_ERR_ARG;
        return upper ? cs_launch<20, true>(n_blocks, cluster_size, a, ST(stream)) : cs_launch<20, false>(n_blocks, cluster_size, a, ST(stream));
    }
    return DDILU_ERR_ARG;
}
