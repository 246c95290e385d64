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
//   * a CTA keeps every value IT needs in a window of W = 4095 doubles of its OWN shared memory: its own results
//     and the results of other CTAs that its rows depend on (halo values), numbered level by level (own rows of
//     the level, then the level's halo values), value p in xs[p mod W]; setup checks that no row reads further
//     back than W positions behind the end of its own level.  A dependency is a 16-bit window slot, read with a
//     plain shared-memory load; slot W holds 0.0 for padded operands;
//   * a producer PUSHES a result to the (<= 3) other CTAs that need it: st.async through distributed shared memory
//     into the consumer's window slot, completing bytes on the consumer's mbarrier -- data and signal travel
//     together, no fence, no cluster-scope release (barrier.cluster.arrive.release costs a MEMBAR.ALL.GPU per
//     level, ~700 cycles: measured);
//   * ONE mbarrier wait per level: the phase of level l completes when all warps of the own CTA have stored their
//     level-l rows, all halo bytes of level l have landed (expect_tx) and every warp of every other CTA has
//     finished level l (a token arrive -- the flow control that makes the window slots safe to overwrite);
//   * operands are one 48-byte record per row (4 coefficients, 8 halves: K slots and <= 3 push targets; + the pivot
//     pair for U; the row id only when a level chunk is not a contiguous row range) in the CTA's schedule order and
//     travel to thread-private shared-memory slots by cp.async, D - 1 steps ahead (coalesced); a step is at
//     most one row per thread, chunks wider than the CTA are cut into several steps at setup; the results leave
//     by row after the arrive.  Every thread computes: there are no helper warps and no flags.
//
// Bytes moved per row: 48 (+ 16 pivot pair) (+ 4 row id) operands + 8 right-hand side + 8 result = 64 (L) / 80 (U),
// against the algorithmic 12 nnz + 4 + 16 = 56 / 68 for three dependencies.
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int CS_WINDOW = 4095;       // doubles per CTA; slot CS_WINDOW holds 0.0
constexpr int CS_STEP_INTS = 8;       // per CTA and step: first / end operand position, window slot of the first row,
                                      // first row (-1: row ids), halo bytes of the level, flags, 0, 0
constexpr int CS_CTA_INTS = 4;        // per CTA: first position in the operand arrays, rows, offset into steps, number of steps
constexpr int CS_NP = 3;              // push targets per row
constexpr unsigned CS_NO_PUSH = 0xffffu;
constexpr int CS_WAIT = 1, CS_ARRIVE = 2;   // step flags: first / last step of its level
constexpr int CS_REC = 48;            // bytes of a row's record without the pivot pair

struct CSweepArgs {
    const int *ctas;                  // CS_CTA_INTS per CTA (block-major, rank-minor)
    const int *steps;                 // CS_STEP_INTS per CTA and step
    const unsigned char *recs;        // [np] records of 48 (lower) / 64 (upper) bytes: c[4] | 8 halves: K window slots of the
                                      // dependencies, then CS_NP push targets slot << 4 | rank (0xffff = none) | upper: d, 1/d
    const int *rowid;                 // [np]
    const double *b;                  // right-hand side by row
    double *out;                      // results by row
    long long np;
    int max_steps;
    long long *dbg;                   // experiments build: 16 cycle counters per CTA and probe thread (first, last)
};

__host__ __device__ constexpr int cs_threads(bool upper, int depth) {
    return (upper && depth > 3) ? 640 : 768;
}
// a stage of the operand ring: per thread the row's record, right-hand side, pivot pair (upper)
__host__ __device__ constexpr int cs_stage_bytes(bool upper, int threads) {
    return threads * (CS_REC + 8 + (upper ? 16 : 0));
}
__host__ __device__ inline size_t cs_smem_bytes(bool upper, int depth, int max_steps) {
    return 16 + (size_t)max_steps * CS_STEP_INTS * 4 + ((size_t)CS_WINDOW + 1) * 8 +
           (size_t)depth * cs_stage_bytes(upper, cs_threads(upper, depth));
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
__device__ __forceinline__ void cs_sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ int4 cs_lds_v4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ int2 cs_lds_v2(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
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
// arrive on the mbarrier of a CTA of the cluster (own included); release.cta orders the warp's window stores before
// the arrive for the readers of the own CTA -- other CTAs get their data through cs_push
__device__ __forceinline__ void cs_mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cs_mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
// operand loads: read once, keep them out of L1
__device__ __forceinline__ double cs_ldg_f64(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t cs_ldg_u32(const unsigned *p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int cs_ldg_s32(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t cs_lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
// global -> shared memory without a register (and without a scoreboard): completion by cp.async.wait_group
__device__ __forceinline__ void cs_cp_async8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cs_cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ double2 cs_lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 cs_lds_u32x4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t cs_half(const uint32_t *w, int i) {     // 16-bit half i of the packed words
    return (i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xffffu);
}

// the registers of one step of one thread
template <int K>
struct CsRow {
    double c[K], rhs, d, r;
    uint32_t ad[K];           // shared-memory addresses of the dependencies
    uint32_t push[2];         // halves K .. K + 2 of the record's tail: push targets (K = 3: halves 3, 4, 5; K = 4: 4, 5, 6)
    int id, slot;             // row (CS_NO_ROW: the thread has no row in the step), window slot (before wrap-around)
};
constexpr int CS_NO_ROW = (int)0x80000000;

// One CTA of the cluster that owns block blockIdx.x / cluster size.  A CTA walks its STEPS: a step is (a part of)
// the CTA's chunk of a level, at most one row per thread -- levels wider than the CTA are cut into several steps at
// setup; only the first step of a level waits, only the last one signals.  Thread t owns row t of every step.
// Operands travel global -> shared memory by cp.async (16-byte pieces of the row's record into thread-private
// slots of a D-deep stage ring, D - 1 steps ahead; completion by cp.async.wait_group, i.e. NOT through the six
// register scoreboards of a warp: operands prefetched into registers made every consumer wait for the youngest
// load in flight), and shared memory -> registers one step ahead:
// iteration i   B: operands of step i + 1 from the ring into registers, slots -> shared-memory addresses
//               A: operands of step i + D requested
//               C: (first step of a level) mbarrier phase of the previous level: own rows stored, halo landed,
//                  every warp of the cluster past it
//               D: the row: K window loads, multiply / subtract chain [, division], window store, pushes
//               E: (last step of a level) arrive at every CTA's mbarrier of the level; result to global memory
template <int K, bool UPPER, int D>
__global__ void __launch_bounds__(cs_threads(UPPER, D), 1) csweep_kernel(const CSweepArgs a) {
    constexpr int NT = cs_threads(UPPER, D);
    constexpr int STAGE = cs_stage_bytes(UPPER, NT);
    // stage layout (slot = thread): records[NT][48] | rhs[NT][8] | pivot pairs[NT][16] (upper)
    constexpr int OFF_RHS = CS_REC * NT, OFF_PIV = OFF_RHS + 8 * NT;
    extern __shared__ __align__(16) unsigned char cs_smem[];
    const int *cta = a.ctas + CS_CTA_INTS * blockIdx.x;
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctaid.x;" : "=r"(csize));
    const long long base = cta[0];
    const int step_off = cta[2], nsteps = cta[3];
    const int tid = threadIdx.x, lane = tid & 31;
    uint64_t *bars = (uint64_t *)cs_smem;                     // [2]: levels of even / odd index
    int4 *steps = (int4 *)(cs_smem + 16);
    double *xs = (double *)(cs_smem + 16 + (size_t)a.max_steps * CS_STEP_INTS * 4);
    unsigned char *ring = (unsigned char *)(xs + CS_WINDOW + 1);
    {
        const int4 *src = (const int4 *)a.steps + 2 * (size_t)step_off;
        for (int i = tid; i < 2 * nsteps; i += NT) steps[i] = src[i];
    }
    const uint32_t bar_u32 = cs_smem_u32(bars);
    if (tid == 0) {
        xs[CS_WINDOW] = 0.0;                  // padded operands: coefficient 0 times this slot
        cs_mbar_init(bar_u32, (NT / 32) * (int)csize);
        cs_mbar_init(bar_u32 + 8, (NT / 32) * (int)csize);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cs_cluster_sync();                        // every CTA of the cluster is running, its mbarriers are initialised
    const uint32_t st_u32 = cs_smem_u32(steps), xs_u32 = cs_smem_u32(xs);
    const uint32_t rec_u32 = cs_smem_u32(ring) + (uint32_t)(CS_REC * tid);     // this thread's slots of stage 0
    const uint32_t rhs_u32 = cs_smem_u32(ring) + OFF_RHS + 8u * (uint32_t)tid;
    const uint32_t piv_u32 = cs_smem_u32(ring) + OFF_PIV + 16u * (uint32_t)tid;
    const unsigned char *recs = a.recs + (size_t)base * (UPPER ? CS_REC + 16 : CS_REC);
    const int *ids = a.rowid + base;
    // lane r < cluster size signals CTA r: the address of that CTA's mbarrier pair
    const uint32_t peer_bar = cs_mapa(bar_u32, (uint32_t)lane < csize ? (uint32_t)lane : 0u);
    const bool signals = (uint32_t)lane < csize;

    // A: request the operands of step i into a stage (an empty group when the warp has no row there).  The records
    // of a warp's 32 rows are one contiguous run in global memory AND in the stage: lane j copies the 16-byte
    // pieces j, j + 32, ... of the run (fully coalesced) -- a thread's record is assembled by its whole warp, so
    // fetch() synchronises the warp behind its wait
    constexpr int PIECES = UPPER ? 4 : 3;     // 16-byte pieces of a record in global memory (the 4th: pivot pair)
    const uint32_t wrec_u32 = cs_smem_u32(ring) + (uint32_t)(CS_REC * (tid - lane));      // stage 0 slots of the warp's lane 0
    const uint32_t wpiv_u32 = cs_smem_u32(ring) + OFF_PIV + 16u * (uint32_t)(tid - lane);
    auto issue = [&](int i, uint32_t stage_off) {
        if (i < nsteps) {
            const int4 sv = cs_lds_v4(st_u32 + 32u * (uint32_t)i);
            const int p0 = sv.x + tid - lane;                 // position of the warp's first row
            const int rows = min(32, sv.y - p0);              // rows of the warp in this step
            if (rows > 0) {
                const unsigned char *g = recs + (size_t)p0 * (16 * PIECES);
#pragma unroll
                for (int q = 0; q < PIECES; ++q) {
                    const int m = lane + 32 * q;              // piece of the run
                    if (m < rows * PIECES) {
                        const int t = UPPER ? m >> 2 : m / 3, o = UPPER ? m & 3 : m - 3 * t;      // row of the warp, piece of its record
                        const uint32_t dst = (UPPER && o == 3) ? wpiv_u32 + 16u * (uint32_t)t : wrec_u32 + (uint32_t)(CS_REC * t + 16 * o);
                        cs_cp_async16(dst + stage_off, g + 16 * m);
                    }
                }
                if (lane < rows && sv.w >= 0) cs_cp_async8(rhs_u32 + stage_off, a.b + sv.w + tid);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // B: the operands of step i (requested D - 1 iterations ago) from their stage into registers
    auto fetch = [&](int i, uint32_t stage_off, CsRow<K> &x) {
        x.id = CS_NO_ROW;
        if (i >= nsteps) return;
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
        __syncwarp();                         // the record was copied by the other lanes of the warp
        const int4 sv = cs_lds_v4(st_u32 + 32u * (uint32_t)i);
        const int p = sv.x + tid;
        if (p < sv.y) {
            x.slot = sv.z + tid;
            const double2 c01 = cs_lds_f64x2(rec_u32 + stage_off), c23 = cs_lds_f64x2(rec_u32 + stage_off + 16u);
            const uint4 h = cs_lds_u32x4(rec_u32 + stage_off + 32u);
            x.c[0] = c01.x, x.c[1] = c01.y, x.c[2] = c23.x;
            if (K > 3) x.c[3] = c23.y;
            if (UPPER) {
                const double2 dr = cs_lds_f64x2(piv_u32 + stage_off);
                x.d = dr.x, x.r = dr.y;
            }
            if (sv.w >= 0) {
                x.id = sv.w + tid;
                x.rhs = cs_lds(rhs_u32 + stage_off);
            } else {                                    // rows by id: two dependent loads on the spot (rare layouts)
                x.id = cs_ldg_s32(ids + p);
                x.rhs = __ldg(a.b + x.id);
            }
            // halves: K slots, then the push targets
            const uint32_t w[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
            for (int k = 0; k < K; ++k) x.ad[k] = xs_u32 + 8u * cs_half(w, k);
            if (K == 3) x.push[0] = (h.y >> 16) | (h.z << 16), x.push[1] = h.z >> 16;      // halves 3, 4 | 5
            else x.push[0] = h.z, x.push[1] = h.w & 0xffffu;                                // halves 4, 5 | 6
        }
    };

#ifdef DDILU_EXPERIMENTS
    unsigned tq[6] = {0, 0, 0, 0, 0, 0}, t0 = 0, t1 = 0;
    const bool probe = a.dbg && (tid == 0 || tid == NT - 1);
#define CS_TICK(i)                  \
    if (probe) {                    \
        t1 = (unsigned)clock();     \
        tq[i] += t1 - t0;           \
        t0 = t1;                    \
    }
#else
#define CS_TICK(i)
#endif
    int lev = 0;                              // level of the current step
    uint32_t stage_off = 0;                   // stage of the current step
    // one step: `cur` holds its operands, `nxt` receives those of the next step
    auto step = [&](int i, const CsRow<K> &cur, CsRow<K> &nxt) {
        const uint32_t cur_stage = stage_off;
        stage_off = stage_off + STAGE == (uint32_t)(D * STAGE) ? 0u : stage_off + STAGE;
        const int2 tf = cs_lds_v2(st_u32 + 32u * (uint32_t)i + 16u);         // halo bytes of the level, flags
        const uint32_t mybar = bar_u32 + 8u * (uint32_t)(lev & 1);           // phase of this level: own and (offset) peers'
        // the halo bytes of the level (before this warp's arrive: the phase cannot complete without them)
        if (tid == 0 && tf.x) cs_mbar_expect_tx(mybar, (uint32_t)tf.x);
        CS_TICK(0)
        fetch(i + 1, stage_off, nxt);
        CS_TICK(1)
        issue(i + D, cur_stage);              // the stage of step i is free: its operands are in registers
        CS_TICK(2)
        // previous level: own rows stored, halo landed, every warp of the cluster past it
        if ((tf.y & CS_WAIT) && lev) cs_mbar_wait(bar_u32 + 8u * (uint32_t)((lev - 1) & 1), (uint32_t)(((lev - 1) >> 1) & 1));
        CS_TICK(3)
        double res = 0.0;
        const bool have = cur.id != CS_NO_ROW;
        if (have) {
            double v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = cs_lds(cur.ad[k]);
            double sum = cur.rhs;
            // -fmad=false: every product is rounded before it is subtracted
#pragma unroll
            for (int k = 0; k < K; ++k) sum -= cur.c[k] * v[k];
            if (UPPER) sum = exact_div(sum, cur.d, cur.r);
            int sl = cur.slot;
            sl -= sl >= CS_WINDOW ? CS_WINDOW : 0;
            cs_sts(xs_u32 + 8u * (uint32_t)sl, sum);
            // to the other CTAs that need the value (rare: rows on the border of a chunk)
            if ((cur.push[0] & cur.push[1]) != 0xffffffffu || false) {
#pragma unroll
                for (int k = 0; k < CS_NP; ++k) {
                    const uint32_t pp = k == 0 ? (cur.push[0] & 0xffffu) : (k == 1 ? cur.push[0] >> 16 : (cur.push[1] & 0xffffu));
                    if (pp != CS_NO_PUSH) cs_push(cs_mapa(xs_u32 + 8u * (pp >> 4), pp & 15u), sum, cs_mapa(mybar, pp & 15u));
                }
            }
            res = sum;
        }
        CS_TICK(4)
        if (tf.y & CS_ARRIVE) {
            // this warp is through the level: one arrive per CTA of the cluster (lane r -> CTA r)
            __syncwarp();
            if (signals) cs_mbar_arrive_cluster(peer_bar + 8u * (uint32_t)(lev & 1));
            ++lev;
        }
        // behind the arrive: the hand-over must not wait for the store
        if (have) a.out[cur.id] = res;
        CS_TICK(5)
    };

    // prologue: D groups in flight, step 0 in registers
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s, (uint32_t)(s * STAGE));
    CsRow<K> r0, r1;
    fetch(0, 0, r0);
#ifdef DDILU_EXPERIMENTS
    if (probe) t0 = (unsigned)clock();
#endif
    for (int i = 0; i < nsteps; i += 2) {     // two register sets take the steps in turn
        step(i, r0, r1);
        if (i + 1 < nsteps) step(i + 1, r1, r0);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    // the last phase: nobody pushes into this CTA's window or signals its mbarriers any more
    if (lev) cs_mbar_wait(bar_u32 + 8u * (uint32_t)((lev - 1) & 1), (uint32_t)(((lev - 1) >> 1) & 1));
    cs_cluster_sync();
#ifdef DDILU_EXPERIMENTS
    if (probe) {
        long long *o = a.dbg + 16 * (2 * blockIdx.x + (tid ? 1 : 0));
        for (int q = 0; q < 6; ++q) o[q] = tq[q];
    }
#endif
#undef CS_TICK
}

// one thread per row: the record of the row at its position of the CTA-local schedule order
// record: c[4] (32 bytes) | 8 halves: K dependency slots, then CS_NP push targets (written by the caller) | upper: d, 1/d
template <bool UPPER>
__global__ void csweep_fill_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                   const double *__restrict__ val, int K, const int *__restrict__ gpos,
                                   const int *__restrict__ dep_slot, unsigned char *recs, int *rowid, int *bad_row) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const long long g = gpos[row];
    unsigned char *rec = recs + (size_t)g * (UPPER ? CS_REC + 16 : CS_REC);
    double *cf = (double *)rec;
    unsigned short *hv = (unsigned short *)(rec + 32);
    int kk = 0;
    double diag = 1.0;
    bool seen = false;
    for (int k = rp[row], ke = rp[row + 1]; k < ke; ++k) {
        const int j = ci[k];
        if (UPPER ? j > row : j < row) {
            if (kk < K) {
                cf[kk] = val[k];
                hv[kk] = (unsigned short)dep_slot[k];
            }
            ++kk;
        } else if (j == row) {
            diag = val[k];
            seen = true;
        }
    }
    for (; kk < K; ++kk) {       // padding: coefficient 0 times the zero slot
        cf[kk] = 0.0;
        hv[kk] = (unsigned short)CS_WINDOW;
    }
    rowid[g] = row;
    if (UPPER) {
        double *pv = (double *)(rec + CS_REC);
        pv[0] = diag;
        pv[1] = safe_reciprocal(diag);
        if (!seen || fabs(diag) < 1e-300) atomicMin(bad_row, row);
    }
}

namespace {
long long *g_csweep_dbg = nullptr;
template <int K, bool UPPER, int NSET>
int cs_prepare(size_t smem) {
    if (smem > 227 * 1024) return DDILU_ERR_ARG;
    static size_t attr = 0;
    static bool nonportable = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!nonportable) {
        DDILU_CHECK(cudaFuncSetAttribute(csweep_kernel<K, UPPER, NSET>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        nonportable = true;
    }
    if (attr < smem) {
        DDILU_CHECK(cudaFuncSetAttribute(csweep_kernel<K, UPPER, NSET>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
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

template <int K, bool UPPER, int NSET>
int cs_launch(int n_blocks, int csize, const CSweepArgs &a, size_t smem, cudaStream_t st) {
    const int rc = cs_prepare<K, UPPER, NSET>(smem);
    if (rc) return rc;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cs_config(cfg, at, n_blocks, csize, cs_threads(UPPER, NSET), smem, st);
    DDILU_CHECK(cudaLaunchKernelEx(&cfg, csweep_kernel<K, UPPER, NSET>, a));
    return DDILU_OK;
}

template <int K, bool UPPER, int NSET>
int cs_active(int csize, size_t smem, int *out) {
    const int rc = cs_prepare<K, UPPER, NSET>(smem);
    if (rc) return rc;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cs_config(cfg, at, 64, csize, cs_threads(UPPER, NSET), smem, nullptr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, csweep_kernel<K, UPPER, NSET>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *out = n;
    return DDILU_OK;
}

template <int K>
int cs_dispatch(int upper, int depth, int n_blocks, int csize, const CSweepArgs &a, cudaStream_t st) {
    const size_t smem = cs_smem_bytes(upper != 0, depth, a.max_steps);
    if (depth == 2) return upper ? cs_launch<K, true, 2>(n_blocks, csize, a, smem, st) : cs_launch<K, false, 2>(n_blocks, csize, a, smem, st);
    if (depth == 3) return upper ? cs_launch<K, true, 3>(n_blocks, csize, a, smem, st) : cs_launch<K, false, 3>(n_blocks, csize, a, smem, st);
    if (depth == 4) return upper ? cs_launch<K, true, 4>(n_blocks, csize, a, smem, st) : cs_launch<K, false, 4>(n_blocks, csize, a, smem, st);
    return DDILU_ERR_ARG;
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

/* threads of a CTA of the cluster sweep (= rows of a step) for a kernel shape (depth = stages of the operand ring) */
extern "C" int ddilu_csweep_threads(int upper, int depth) { return cs_threads(upper != 0, depth); }

/* doubles of a CTA's window (own and halo values): no row may read further back (device.build_csweep checks) */
extern "C" int ddilu_csweep_window(void) { return CS_WINDOW; }

/* CTAs other than its own that may need a row's result */
extern "C" int ddilu_csweep_max_push(void) { return CS_NP; }

/* bytes of a row's record in the operand array */
extern "C" int ddilu_csweep_record_bytes(int upper) { return upper ? CS_REC + 16 : CS_REC; }

extern "C" long long ddilu_csweep_smem_bytes(int upper, int depth, int max_steps) {
    return (long long)cs_smem_bytes(upper != 0, depth, max_steps);
}

/* clusters of `cluster_size` CTAs of the sweep kernel that can be resident at once (0: the size cannot be launched) */
extern "C" int ddilu_csweep_active_clusters(int cluster_size, int depth, int max_steps) {
    if (cluster_size < 1 || cluster_size > 16) return 0;
    int n = 0, rc = DDILU_ERR_ARG;
    if (depth == 2) rc = cs_active<3, true, 2>(cluster_size, cs_smem_bytes(true, 2, max_steps), &n);
    if (depth == 3) rc = cs_active<3, true, 3>(cluster_size, cs_smem_bytes(true, 3, max_steps), &n);
    if (depth == 4) rc = cs_active<3, true, 4>(cluster_size, cs_smem_bytes(true, 4, max_steps), &n);
    return rc == DDILU_OK ? n : 0;
}

extern "C" int ddilu_csweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                                 const int *gpos, const int *dep_slot, unsigned char *recs, int *rowid, int *bad_row,
                                 void *stream) {
    if (n <= 0) return DDILU_OK;
    if (k != 3 && k != 4) return DDILU_ERR_ARG;
    const int threads = 256, grid = div_up(n, threads);
    if (upper)
        csweep_fill_kernel<true><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, dep_slot, recs,
                                                                   rowid, bad_row);
    else
        csweep_fill_kernel<false><<<grid, threads, 0, ST(stream)>>>(n, row_ptr, col_idx, values, k, gpos, dep_slot, recs,
                                                                    rowid, bad_row);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* out[row] = (L^-1 b)[row] (upper 0, unit diagonal) or (U^-1 b)[row] (upper 1) for a block-diagonal factor laid out
 * by ddilu_csweep_fill: n_blocks clusters of cluster_size CTAs */
extern "C" int ddilu_csweep_solve(int n_blocks, int cluster_size, const int *ctas, const int *steps,
                                  const unsigned char *recs, const int *rowid, long long np, int k, int upper,
                                  int max_steps, int depth, const double *b, double *out, void *stream) {
    if (n_blocks <= 0) return DDILU_OK;
    if (cluster_size < 1 || cluster_size > 16) return DDILU_ERR_ARG;
    CSweepArgs a{ctas, steps, recs, rowid, b, out, np, max_steps, g_csweep_dbg};
    switch (k) {
        case 3: return cs_dispatch<3>(upper, depth, n_blocks, cluster_size, a, ST(stream));
        case 4: return cs_dispatch<4>(upper, depth, n_blocks, cluster_size, a, ST(stream));
        default: return DDILU_ERR_ARG;
    }
}
