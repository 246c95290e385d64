// Symbolic phase of the level-of-fill factorisation ILU(k) (replaces
// factor.py:270-369 `_iluk_symbolic`) and the value prefill of the resulting
// pattern (factor.py:372-390 `_prefill`).  The numeric phase is the fixed-pattern
// kernel of factor.cu (the reference calls the same `_factor_split`).
//
// The pattern of a row depends on the kept rows (and their fill LEVELS) of all
// its pivots, fill included, so - like ILUT - there is no schedule to
// precompute: one persistent cooperative launch, warps take rows round-robin in
// index order, the working row is a sorted (column, level) array in shared
// memory, pivots are visited in increasing column order; for pivot k the warp
// waits on done[k] (release/acquire), reads the kept row of k from L2 (lanes =
// entries beyond its diagonal) and merges it with level lev(i,k)+lev(k,j)+1 <=
// klevel: the minimum wins on a present position, new positions are inserted
// with a warp-parallel two-buffer merge.  Integer work only: bit-exact.
//
// Output: fixed-capacity row slabs (cap entries per row for the pivot part and
// for the kept part), compacted to CSR by ddilu_compact_cols.  status != 0: a
// row outgrew cap, the host retries with a larger one.
#include <climits>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int ILUK_WARPS = 4;

__global__ void __launch_bounds__(ILUK_WARPS * 32)
iluk_symbolic_kernel(int n, const int *__restrict__ a_rp, const int *__restrict__ a_ci, int n_elim, int klevel, int cap,
                     int *p_cnt, int *p_ci, int *k_cnt, int *k_ci, int *k_lv, int *done, int *status,
                     const int *__restrict__ order) {
    extern __shared__ int iluk_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int *ca = iluk_smem + (size_t)wib * (4 * cap + 32), *cb = ca + cap, *la = cb + cap, *lb = la + cap;
    int *insj = lb + cap;
    const long long W = (long long)gridDim.x * ILUK_WARPS;
    // rows in PROCESSING order (order[slot], any order in which a row follows its pivot rows: the caller interleaves
    // the independent diagonal blocks so that all of them advance at once), else index order
    for (long long slot = (long long)blockIdx.x * ILUK_WARPS + wib; slot < n; slot += W) {
        const int i = order ? order[slot] : (int)slot;
        const int lim = i < n_elim ? i : n_elim;
        const int a0 = a_rp[i], len0 = a_rp[i + 1] - a0;
        bool overflow = false;
        // ---- pattern of A's row plus the diagonal, level 0 (factor.py:285-317)
        int nless = 0, hasd = 0;
        for (int s = lane; s < len0; s += 32) {
            const int c = a_ci[a0 + s];
            nless += c < i;
            hasd |= c == i;
        }
        for (int o = 16; o > 0; o >>= 1) {
            nless += __shfl_xor_sync(0xffffffffu, nless, o);
            hasd |= __shfl_xor_sync(0xffffffffu, hasd, o);
        }
        int len = len0 + (hasd ? 0 : 1);
        if (len > cap) {
            overflow = true;
            len = 0;
        } else {
            for (int s = lane; s < len0; s += 32) {
                const int c = a_ci[a0 + s];
                const int dst = s + ((!hasd && c > i) ? 1 : 0);
                ca[dst] = c;
                la[dst] = 0;
            }
            if (!hasd && lane == 0) {
                ca[nless] = i;
                la[nless] = 0;
            }
        }
        __syncwarp();
        // ---- merge the kept rows of all pivots below the boundary (factor.py:318-337)
        int pos = 0;
        while (!overflow && pos < len) {
            const int k = ca[pos];
            if (k >= lim) break;
            const int lk = la[pos];
            if (lane == 0)
                while (ld_acquire(done + k) == 0) {
                }
            __syncwarp();
            const long long kb = (long long)k * cap;
            const int kcount = ld_l2(k_cnt + k);
            for (int t0 = 1; t0 < kcount && !overflow; t0 += 32) {
                const int t = t0 + lane;
                int j = INT_MAX, nl = INT_MAX;
                if (t < kcount) {
                    j = ld_l2(k_ci + kb + t);
                    nl = lk + ld_l2(k_lv + kb + t) + 1;
                }
                const bool valid = t < kcount && nl <= klevel;
                int lo = pos + 1, hi = len;   // first index in (pos, len) with column >= j
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (ca[mid] < j) lo = mid + 1; else hi = mid;
                }
                const bool found = valid && lo < len && ca[lo] == j;
                if (found && nl < la[lo]) la[lo] = nl;
                const bool ins = valid && !found;
                const unsigned m = __ballot_sync(0xffffffffu, ins);
                const int nins = __popc(m), irank = __popc(m & ((1u << lane) - 1u));
                if (nins) {
                    if (len + nins > cap) {
                        overflow = true;
                    } else {
                        __syncwarp();
                        if (ins) insj[irank] = j;
                        __syncwarp();
                        for (int e = lane; e < len; e += 32) {   // entries move up by the inserts below them
                            const int c = ca[e];
                            int sh = 0;
                            if (e > pos)
                                for (int q = 0; q < nins; ++q) sh += insj[q] < c;
                            cb[e + sh] = c;
                            lb[e + sh] = la[e];
                        }
                        if (ins) {
                            cb[lo + irank] = j;
                            lb[lo + irank] = nl;
                        }
                        __syncwarp();
                        int *tc = ca; ca = cb; cb = tc;
                        int *tl = la; la = lb; lb = tl;
                        len += nins;
                    }
                }
                __syncwarp();
            }
            ++pos;
        }
        // ---- emit: [0, pos) pivot part, [pos, len) kept part with levels (factor.py:338-368)
        if (!overflow) {
            const long long ob = (long long)i * cap;
            for (int e = lane; e < pos; e += 32) p_ci[ob + e] = ca[e];
            for (int e = pos + lane; e < len; e += 32) {
                k_ci[ob + e - pos] = ca[e];
                k_lv[ob + e - pos] = la[e];
            }
        }
        if (lane == 0) {
            p_cnt[i] = overflow ? 0 : pos;
            k_cnt[i] = overflow ? 1 : len - pos;   // later rows then see "diagonal only"
            if (overflow) {
                k_ci[(long long)i * cap] = i;
                k_lv[(long long)i * cap] = 0;
                atomicExch(status, 1);
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(done + i, 1);
    }
}

// slab -> CSR columns
__global__ void compact_cols(int n, int cap, const int *__restrict__ cnt, const int *__restrict__ ci,
                             const int *__restrict__ out_rp, int *__restrict__ out_ci) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < n; i += nw) {
        const int c = cnt[i], dst = out_rp[i];
        for (int e = lane; e < c; e += 32) out_ci[dst + e] = ci[i * cap + e];
    }
}

// factor.py:372-390: copy A's values into the matching slots of the superset pattern
// (fill keeps 0); part 0: columns < lim of every row, part 1: columns >= lim
__global__ void prefill(int n, const int *__restrict__ a_rp, const int *__restrict__ a_ci,
                        const double *__restrict__ a_v, const int *__restrict__ rp, const int *__restrict__ ci,
                        double *__restrict__ v, int n_elim, int upper_part) {
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)q;
        const int lim = i < n_elim ? i : n_elim;
        int t = rp[i];
        const int te = rp[i + 1];
        for (int u = t; u < te; ++u) v[u] = 0.0;
        for (int s = a_rp[i], se = a_rp[i + 1]; s < se; ++s) {
            const int j = a_ci[s];
            if ((upper_part == 0) != (j < lim)) continue;
            while (t < te && ci[t] < j) ++t;
            if (t < te && ci[t] == j) v[t++] = a_v[s];
        }
    }
}

}  // namespace ddilu

using namespace ddilu;

extern "C" long long ddilu_iluk_smem_bytes(int row_cap) {
    return (long long)ILUK_WARPS * (4LL * row_cap + 32) * (long long)sizeof(int);
}

extern "C" int ddilu_iluk_symbolic(int n, const int *a_rp, const int *a_ci, int n_elim, int klevel, int row_cap,
                                   int *p_cnt, int *p_ci, int *k_cnt, int *k_ci, int *k_lv, int *done, int *status,
                                   const int *order, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (row_cap < 2 || klevel < 0) return DDILU_ERR_ARG;
    const size_t smem = (size_t)ddilu_iluk_smem_bytes(row_cap);
    if (smem > 200 * 1024) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaFuncSetAttribute(iluk_symbolic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DDILU_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * (size_t)n, st));
    DDILU_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
    int occ = 0;
    DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, iluk_symbolic_kernel, ILUK_WARPS * 32, smem));
    if (occ < 1) return DDILU_ERR_ARG;
    long long grid = (long long)occ * device_info().sm_count;
    const long long need = div_up(n, ILUK_WARPS);
    if (grid > need) grid = need;
    int g = (int)grid;
    void *args[] = {&n, &a_rp, &a_ci, &n_elim, &klevel, &row_cap, &p_cnt, &p_ci, &k_cnt, &k_ci, &k_lv, &done, &status,
                    &order};
    DDILU_CHECK(cudaLaunchCooperativeKernel((void *)iluk_symbolic_kernel, g, ILUK_WARPS * 32, args, smem, st));
    return DDILU_OK;
}

extern "C" int ddilu_compact_cols(int n, int cap, const int *cnt, const int *ci, const int *out_rp, int *out_ci,
                                  void *stream) {
    if (n <= 0) return DDILU_OK;
    compact_cols<<<stream_grid(n, 256, 1, 16), 256, 0, (cudaStream_t)stream>>>(n, cap, cnt, ci, out_rp, out_ci);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_prefill(int n, const int *a_rp, const int *a_ci, const double *a_v, const int *rp, const int *ci,
                             double *v, int n_elim, int upper_part, void *stream) {
    if (n <= 0) return DDILU_OK;
    prefill<<<stream_grid(n, 256), 256, 0, (cudaStream_t)stream>>>(n, a_rp, a_ci, a_v, rp, ci, v, n_elim, upper_part);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
