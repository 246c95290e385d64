// Cuthill-McKee ordering on the device, bit-identical to the serial reference
// (ordering.py:304-397 `_bfs_ecc`, `_rcm_order`).
//
// One persistent cooperative launch orders the whole graph.  The serial queue
// discipline is reproduced level by level:
//   * a node is claimed by the earliest-positioned frontier node adjacent to it
//     (atomicMin over the parent position = "first to dequeue wins"),
//   * every parent emits its own children sorted by (degree, index); the
//     children of parent q start at the prefix sum of the child counts of the
//     parents before q (grid-wide scan), which is exactly the order in which the
//     serial loop appends them,
//   * components are taken up by smallest index; each one starts from the
//     George-Liu pseudo-peripheral node found by repeated level BFS with the
//     reference's tie rule (last level, min degree, then min index).
// The graph is the symmetrised adjacency without the diagonal; only neighbour
// SETS and degrees matter to the result, so neighbour lists need not be sorted.
#include <cooperative_groups.h>

#include <climits>

#include "common.cuh"
#include "ddilu_b200.h"

namespace cg = cooperative_groups;

namespace ddilu {

constexpr int RCM_THREADS = 512;
constexpr int RCM_MAX_LOCAL = 32;

struct RcmState {
    int found;
    int fcnt[3];
    unsigned long long best;
    int total;
    unsigned barrier;   // monotone arrival counter of the CTA group that owns this state
    int pad;
};

// A group of consecutive CTAs that orders one independent segment of the graph (one subdomain's
// interior block).  sync() is a barrier over the group's CTAs only (monotone counter in L2): the
// segments advance concurrently instead of paying every grid barrier once per segment.
struct CtaGroup {
    unsigned *bar;
    int nblk, blk;      // CTAs in the group, my index inside it
    unsigned phase;
    __device__ __forceinline__ void sync() {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(bar, 1u);
            const unsigned target = (phase + 1u) * (unsigned)nblk;
            while ((int)(ld_acquire((const int *)bar) - (int)target) < 0) {
            }
            __threadfence();
        }
        ++phase;
        __syncthreads();
    }
};

__device__ __forceinline__ int block_excl_scan_512(int v, int *total, int *wtot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    int base = 0, all = 0;
#pragma unroll
    for (int w = 0; w < RCM_THREADS / 32; ++w) {
        int t = wtot[w];
        if (w < warp) base += t;
        all += t;
    }
    __syncthreads();
    *total = all;
    return base + inc - v;
}

__device__ __forceinline__ unsigned long long node_key(const int *rp, int v) {
    return ((unsigned long long)(unsigned)(rp[v + 1] - rp[v]) << 32) | (unsigned)v;
}

// level BFS from `root`; returns eccentricity, *last = min (degree, index) node of the last level
__device__ int bfs_ecc(CtaGroup &grid, int n, const int *__restrict__ rp, const int *__restrict__ ci, int root,
                       int stamp, int *mark, int *fa, int *fb, RcmState *st, int *last) {
    const long long gtid = (long long)grid.blk * blockDim.x + threadIdx.x, gsize = (long long)grid.nblk * blockDim.x;
    if (gtid == 0) {
        fa[0] = root;
        mark[root] = stamp;
        st->fcnt[1] = 0;
        st->best = ~0ULL;
    }
    int *cur = fa, *nxt = fb;
    int cur_cnt = 1, level = 0;
    for (;;) {
        grid.sync();
        if (gtid == 0) st->fcnt[(level + 2) % 3] = 0;
        int *next_cnt = &st->fcnt[(level + 1) % 3];
        for (long long q = gtid; q < cur_cnt; q += gsize) {
            const int u = ld_l2(cur + q);
            for (int k = rp[u], ke = rp[u + 1]; k < ke; ++k) {
                const int w = ci[k];
                if (ld_l2(mark + w) != stamp && atomicExch(mark + w, stamp) != stamp) nxt[atomicAdd(next_cnt, 1)] = w;
            }
        }
        grid.sync();
        const int c = ld_l2(next_cnt);
        if (c == 0) break;
        int *t = cur; cur = nxt; nxt = t;
        cur_cnt = c;
        ++level;
    }
    for (long long q = gtid; q < cur_cnt; q += gsize) atomicMin(&st->best, node_key(rp, ld_l2(cur + q)));
    grid.sync();
    *last = (int)(unsigned)(*(volatile unsigned long long *)&st->best & 0xffffffffULL);
    grid.sync();  // everyone has read best before the next sweep resets it
    return level;
}

// n_seg segments [seg_ptr[s], seg_ptr[s+1]) with no edges between them (n_seg = 1, seg_ptr = NULL: the
// whole graph); the CTAs are dealt to the segments in equal groups.  Scratch arrays are indexed by node or
// by position, both of which stay inside the segment, so the groups never touch each other's data.
__global__ void __launch_bounds__(RCM_THREADS) cm_order_kernel(int n_all, const int *__restrict__ rp,
                                                               const int *__restrict__ ci, int n_seg,
                                                               const int *__restrict__ seg_ptr, int *order,
                                                               int *visited, int *mark, int *ppos, int *fa, int *fb,
                                                               int *cnt, int *tile_tot_all, RcmState *st_all) {
    __shared__ int wtot[RCM_THREADS / 32];
    __shared__ int sh_base, sh_total;
    const int per_seg = (int)gridDim.x / n_seg;           // CTAs per segment (the remainder idles)
    const int seg = (int)blockIdx.x / per_seg;
    if (seg >= n_seg) return;
    RcmState *st = st_all + seg;
    CtaGroup grid{&st->barrier, per_seg, (int)blockIdx.x - seg * per_seg, 0u};
    int *tile_tot = tile_tot_all + seg * per_seg;
    const int node0 = seg_ptr ? seg_ptr[seg] : 0;
    const int n = seg_ptr ? seg_ptr[seg + 1] : n_all;      // nodes of this segment: [node0, n)
    // frontier / count scratch of this segment starts at its first node
    fa += node0;
    fb += node0;
    cnt += node0;
    const long long gtid = (long long)grid.blk * blockDim.x + threadIdx.x, gsize = (long long)grid.nblk * blockDim.x;
    const int G = grid.nblk;
    int pos = node0, scan = node0, stamp = 0;
    while (pos < n) {
        // ---- smallest unvisited index >= scan
        int root;
        for (;;) {
            if (gtid == 0) st->found = INT_MAX;
            grid.sync();
            const long long idx = scan + gtid;
            if (idx < n && ld_l2(visited + idx) == 0) atomicMin(&st->found, (int)idx);
            grid.sync();
            root = ld_l2(&st->found);
            grid.sync();
            if (root != INT_MAX) break;
            scan += (int)min((long long)n - scan, gsize);
        }
        scan = root;
        // ---- George-Liu pseudo-peripheral node (ordering.py:354-365)
        int cand, nxt;
        int ecc_root = bfs_ecc(grid, n, rp, ci, root, stamp++, mark, fa, fb, st, &cand);
        for (;;) {
            int ecc_cand = bfs_ecc(grid, n, rp, ci, cand, stamp++, mark, fa, fb, st, &nxt);
            if (ecc_cand > ecc_root) {
                root = cand;
                ecc_root = ecc_cand;
                cand = nxt;
            } else {
                break;
            }
        }
        // ---- Cuthill-McKee sweep (ordering.py:366-397)
        if (gtid == 0) {
            order[pos] = root;
            visited[root] = 1;
        }
        int lo = pos, hi = pos + 1;
        for (;;) {
            grid.sync();
            // claim: first parent (smallest position) wins
            for (long long q = lo + gtid; q < hi; q += gsize) {
                const int u = ld_l2(order + q);
                for (int k = rp[u], ke = rp[u + 1]; k < ke; ++k) {
                    const int w = ci[k];
                    if (ld_l2(visited + w) == 0) atomicMin(ppos + w, (int)q);
                }
            }
            grid.sync();
            // count children per parent; scan inside this CTA's contiguous tile
            const int F = hi - lo;
            const int per = (F + G - 1) / G;
            const int bx = grid.blk;
            const int t0 = lo + (int)min((long long)F, (long long)bx * per);
            const int t1 = lo + (int)min((long long)F, (long long)(bx + 1) * per);
            int running = 0;
            for (int base = t0; base < t1; base += RCM_THREADS) {
                const int q = base + threadIdx.x;
                int c = 0;
                if (q < t1) {
                    const int u = ld_l2(order + q);
                    for (int k = rp[u], ke = rp[u + 1]; k < ke; ++k) c += (ld_l2(ppos + ci[k]) == q);
                }
                int tot;
                const int ex = block_excl_scan_512(c, &tot, wtot);
                if (q < t1) cnt[q - lo] = running + ex;
                running += tot;
            }
            if (threadIdx.x == 0) tile_tot[grid.blk] = running;
            grid.sync();
            // CTA base = totals of the CTAs before this one
            {
                int mine = 0, all = 0;
                for (int c = threadIdx.x; c < G; c += RCM_THREADS) {
                    const int t = ld_l2(tile_tot + c);
                    all += t;
                    if (c < grid.blk) mine += t;
                }
                int tb, ta;
                block_excl_scan_512(mine, &tb, wtot);
                block_excl_scan_512(all, &ta, wtot);
                if (threadIdx.x == 0) {
                    sh_base = tb;
                    sh_total = ta;
                }
                __syncthreads();
            }
            const int cta_base = sh_base, total = sh_total;
            // emit children of each parent sorted by (degree, index)
            for (int q = t0 + threadIdx.x; q < t1; q += RCM_THREADS) {
                const int u = ld_l2(order + q);
                const int ks = rp[u], ke = rp[u + 1];
                int out = hi + cta_base + ld_l2(cnt + (q - lo));
                unsigned long long keys[RCM_MAX_LOCAL];
                int c = 0;
                bool overflow = false;
                for (int k = ks; k < ke; ++k) {
                    const int w = ci[k];
                    if (ld_l2(ppos + w) == q) {
                        if (c == RCM_MAX_LOCAL) {
                            overflow = true;
                            break;
                        }
                        const unsigned long long key = node_key(rp, w);
                        int b = c - 1;
                        while (b >= 0 && keys[b] > key) {
                            keys[b + 1] = keys[b];
                            --b;
                        }
                        keys[b + 1] = key;
                        ++c;
                    }
                }
                if (!overflow) {
                    for (int b = 0; b < c; ++b) {
                        const int w = (int)(unsigned)(keys[b] & 0xffffffffULL);
                        order[out + b] = w;
                        visited[w] = 1;
                    }
                } else {  // many children: repeated selection of the next-larger key
                    unsigned long long prev = 0;
                    bool first = true;
                    for (;;) {
                        unsigned long long best = ~0ULL;
                        for (int k = ks; k < ke; ++k) {
                            const int w = ci[k];
                            if (ld_l2(ppos + w) == q) {
                                const unsigned long long key = node_key(rp, w);
                                if ((first || key > prev) && key < best) best = key;
                            }
                        }
                        if (best == ~0ULL) break;
                        const int w = (int)(unsigned)(best & 0xffffffffULL);
                        order[out++] = w;
                        visited[w] = 1;
                        prev = best;
                        first = false;
                    }
                }
            }
            if (total == 0) break;
            lo = hi;
            hi += total;
        }
        pos = hi;
    }
}

// reverse the CM order inside every segment (one segment per domain block):
// out[seg_ptr[s] + k] = cm[seg_ptr[s+1] - 1 - k]
__global__ void reverse_segments(int n, const int *__restrict__ cm, int n_seg, const int *__restrict__ seg_ptr,
                                 int *__restrict__ out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = n_seg;  // largest s with seg_ptr[s] <= i
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (seg_ptr[mid] <= i) lo = mid; else hi = mid;
        }
        out[i] = cm[seg_ptr[lo] + (seg_ptr[lo + 1] - 1 - (int)i)];
    }
}

}  // namespace ddilu

using namespace ddilu;

extern "C" long long ddilu_cm_work_elems(int n) {
    // visited, mark, ppos, fa, fb, cnt: n each; tile totals + one state per segment group
    return 6LL * (n > 0 ? n : 1) + 4096 + 16 * 256;
}

static int cm_order_launch(int n, const int *adj_rp, const int *adj_ci, int n_seg, const int *seg_ptr, int *order,
                           int *work, cudaStream_t st) {
    if (n <= 0) return DDILU_OK;
    const long long nn = n;
    int *visited = work, *mark = work + nn, *ppos = work + 2 * nn, *fa = work + 3 * nn, *fb = work + 4 * nn,
        *cnt = work + 5 * nn, *tile_tot = work + 6 * nn;
    RcmState *state = (RcmState *)(work + 6 * nn + 4096);
    int grid = device_info().sm_count;  // one CTA per SM keeps the barriers cheap
    if (grid > 4096) grid = 4096;
    if (n_seg < 1 || !seg_ptr) {
        n_seg = 1;
        seg_ptr = nullptr;
    }
    if (n_seg > grid || n_seg > 256) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaMemsetAsync(visited, 0, sizeof(int) * nn, st));
    DDILU_CHECK(cudaMemsetAsync(mark, 0xFF, sizeof(int) * nn, st));
    DDILU_CHECK(cudaMemsetAsync(ppos, 0x7F, sizeof(int) * nn, st));  // 0x7F7F7F7F > any position
    DDILU_CHECK(cudaMemsetAsync(state, 0, sizeof(RcmState) * n_seg, st));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cm_order_kernel, RCM_THREADS, 0);
    if (occ < 1) return DDILU_ERR_ARG;
    void *args[] = {&n, &adj_rp, &adj_ci, &n_seg, &seg_ptr, &order, &visited, &mark, &ppos, &fa, &fb, &cnt, &tile_tot,
                    &state};
    // cooperative launch: the group barriers need every CTA resident
    DDILU_CHECK(cudaLaunchCooperativeKernel((void *)cm_order_kernel, grid, RCM_THREADS, args, 0, st));
    return DDILU_OK;
}

extern "C" int ddilu_cm_order(int n, const int *adj_rp, const int *adj_ci, int *order, int *work, void *stream) {
    return cm_order_launch(n, adj_rp, adj_ci, 1, nullptr, order, work, (cudaStream_t)stream);
}

/* the same for a graph whose node ranges [seg_ptr[s], seg_ptr[s+1]) are not connected to each other
 * (one range per subdomain): the ranges are ordered concurrently by disjoint CTA groups */
extern "C" int ddilu_cm_order_segments(int n, const int *adj_rp, const int *adj_ci, int n_seg, const int *seg_ptr,
                                       int *order, int *work, void *stream) {
    return cm_order_launch(n, adj_rp, adj_ci, n_seg, seg_ptr, order, work, (cudaStream_t)stream);
}

extern "C" int ddilu_reverse_segments(int n, const int *cm, int n_seg, const int *seg_ptr, int *out, void *stream) {
    if (n <= 0) return DDILU_OK;
    reverse_segments<<<stream_grid(n, 256), 256, 0, (cudaStream_t)stream>>>(n, cm, n_seg, seg_ptr, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
