// Dual-threshold ILUT with a dynamic pattern (replaces factor.py:482-656
// `_ilut_factor` and :465-479 `_select_largest`).
//
// The pattern of a row is only known once its pivot rows are final, so there is
// no level schedule to precompute.  One persistent cooperative launch: warps
// take rows round-robin in index order; a warp keeps its working row as a
// sorted (column, value) array in shared memory, walks the pivots in increasing
// column order and, for each pivot k, waits on done[k] (release/acquire), reads
// U-row k from L2 and merges it (lanes = U entries; fill is inserted with a
// warp-parallel two-buffer merge).  Every arithmetic step that decides a drop
// follows the reference's order: row norms are accumulated serially in storage
// order, updates are applied pivot by pivot, and the largest-magnitude
// selection ranks by (|v| descending, column ascending) which is exactly the
// reference's first-largest scan.  Patterns and values are bit-identical.
//
// Output goes to fixed-capacity row slabs (compacted to CSR by
// ddilu_compact_rows): L rows hold <= lcap entries; U rows of eliminated rows
// hold <= ucap entries and start with the diagonal; Schur rows (>= n_elim) are
// uncapped in the reference and get `row_cap` entries here.  status != 0 means
// a working row or a Schur row outgrew row_cap: the host retries with a larger cap.
#include <climits>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int ILUT_WARPS = 4;  // warps per CTA

struct IlutSlabs {
    int n_elim, lcap, ucap, scap;
    __host__ __device__ long long loff(int i) const { return (long long)i * lcap; }
    __host__ __device__ long long uoff(int i) const {
        return i < n_elim ? (long long)i * ucap : (long long)n_elim * ucap + (long long)(i - n_elim) * scap;
    }
};

// warp-wide exclusive position of this lane among the lanes with flag set; *total = number set
__device__ __forceinline__ int warp_compact_pos(bool flag, int *total) {
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    *total = __popc(m);
    return __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
}

// keep the `keep` largest |v| of cand[0..cnt) (ties: smaller index = smaller column);
// sel[c] = 1 if kept.  force_col >= 0 is always kept (the diagonal).
__device__ void warp_select(const int *cc, const double *cv, int cnt, int keep, int force_col, unsigned char *sel) {
    const int lane = threadIdx.x & 31;
    for (int c = lane; c < cnt; c += 32) {
        int rank = 0;
        if (cnt > keep) {
            const double mine = fabs(cv[c]);
            for (int o = 0; o < cnt; ++o) {
                const double other = fabs(cv[o]);
                rank += (other > mine) || (other == mine && o < c);
            }
        }
        sel[c] = (rank < keep) || (cc[c] == force_col);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(ILUT_WARPS * 32) ilut_kernel(int n, const int *__restrict__ a_rp,
                                                               const int *__restrict__ a_ci,
                                                               const double *__restrict__ a_v, double tau, int maxfill,
                                                               double tau_s, double delta, int cap, IlutSlabs sl,
                                                               int *l_cnt, int *l_ci, double *l_v, int *u_cnt,
                                                               int *u_ci, double *u_v, int *done, int *status,
                                                               const int *__restrict__ order) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // per-warp carve: valsA, valsB (double[cap]), colsA, colsB (int[cap]), insj (int[32]), sel (uchar[cap])
    const size_t per_warp = (size_t)cap * (2 * sizeof(double) + 2 * sizeof(int)) + 32 * sizeof(int) + ((cap + 7) & ~7);
    unsigned char *base = smem_raw + per_warp * wib;
    double *va = (double *)base, *vb = va + cap;
    int *ca = (int *)(vb + cap), *cb = ca + cap;
    int *insj = cb + cap;
    unsigned char *sel = (unsigned char *)(insj + 32);
    const int n_elim = sl.n_elim;
    const long long W = (long long)gridDim.x * ILUT_WARPS;

    // rows are taken in PROCESSING order: order[slot] (any order in which a row comes after its pivot rows; the
    // caller interleaves the independent diagonal blocks so that all of them advance at once), else index order
    for (long long slot = (long long)blockIdx.x * ILUT_WARPS + wib; slot < n; slot += W) {
        const int i = order ? order[slot] : (int)slot;
        const int lim = i < n_elim ? i : n_elim;
        const int a0 = a_rp[i], len0 = a_rp[i + 1] - a0;
        bool overflow = false;
        // ---- norms in storage order (factor.py:500-511)
        double nrm = 0.0, mx = 0.0;
        if (lane == 0) {
            for (int s = 0; s < len0; ++s) {
                const double t = a_v[a0 + s];
                nrm += t * t;
                mx = fmax(mx, fabs(t));
            }
            nrm = sqrt(nrm);
        }
        nrm = __shfl_sync(0xffffffffu, nrm, 0);
        mx = __shfl_sync(0xffffffffu, mx, 0);
        const double thresh = nrm > 0.0 ? tau * nrm : 0.0;
        if (mx == 0.0) mx = 1.0;
        // ---- load the row, diagonal inserted with value 0 if absent (factor.py:512-541)
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
                va[dst] = a_v[a0 + s];
            }
            if (!hasd && lane == 0) {
                ca[nless] = i;
                va[nless] = 0.0;
            }
        }
        __syncwarp();
        // ---- eliminate pivots in increasing column order (factor.py:542-564)
        int pos = 0;
        while (!overflow && pos < len) {
            const int k = ca[pos];
            if (k >= lim) break;
            if (lane == 0)
                while (ld_acquire(done + k) == 0) {
                }
            __syncwarp();
            const long long ub = sl.uoff(k);
            const int ucount = ld_l2(u_cnt + k);
            const double lik = va[pos] / ld_l2(u_v + ub);
            __syncwarp();
            if (fabs(lik) < thresh) {
                if (lane == 0) va[pos] = 0.0;
                __syncwarp();
                ++pos;
                continue;
            }
            if (lane == 0) va[pos] = lik;
            __syncwarp();
            for (int t0 = 1; t0 < ucount && !overflow; t0 += 32) {
                const int t = t0 + lane;
                const bool valid = t < ucount;
                const int j = valid ? ld_l2(u_ci + ub + t) : INT_MAX;
                const double upd = valid ? lik * ld_l2(u_v + ub + t) : 0.0;
                // first index in (pos, len) with column >= j
                int lo = pos + 1, hi = len;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (ca[mid] < j) lo = mid + 1; else hi = mid;
                }
                const bool found = valid && lo < len && ca[lo] == j;
                if (found) va[lo] -= upd;
                const bool ins = valid && !found;
                int nins;
                const int irank = warp_compact_pos(ins, &nins);
                if (nins) {
                    if (len + nins > cap) {
                        overflow = true;
                    } else {
                        __syncwarp();
                        if (ins) insj[irank] = j;
                        __syncwarp();
                        // existing entries move up by the number of inserted columns below them
                        for (int e = lane; e < len; e += 32) {
                            const int c = ca[e];
                            int sh = 0;
                            if (e > pos)
                                for (int q = 0; q < nins; ++q) sh += insj[q] < c;
                            cb[e + sh] = c;
                            vb[e + sh] = va[e];
                        }
                        if (ins) {
                            cb[lo + irank] = j;
                            vb[lo + irank] = -upd;
                        }
                        __syncwarp();
                        int *tc = ca; ca = cb; cb = tc;
                        double *tv = va; va = vb; vb = tv;
                        len += nins;
                    }
                }
                __syncwarp();
            }
            ++pos;
        }
        // pos = number of entries below lim (the L part); [pos, len) is the U / Schur part
        // ---- L part (factor.py:565-593): |w| >= thresh and w != 0, keep the maxfill largest
        int nl = 0;
        for (int b0 = 0; b0 < pos; b0 += 32) {
            const int e = b0 + lane;
            const bool c = e < pos && fabs(va[e]) >= thresh && va[e] != 0.0;
            int tot;
            const int r = warp_compact_pos(c, &tot);
            if (c) {
                cb[nl + r] = ca[e];
                vb[nl + r] = va[e];
            }
            nl += tot;
        }
        __syncwarp();
        warp_select(cb, vb, nl, maxfill, -1, sel);
        int lout = 0;
        const long long lb = sl.loff(i);
        for (int b0 = 0; b0 < nl; b0 += 32) {
            const int e = b0 + lane;
            const bool c = e < nl && sel[e];
            int tot;
            const int r = warp_compact_pos(c, &tot);
            if (c && lout + r < sl.lcap) {
                l_ci[lb + lout + r] = cb[e];
                l_v[lb + lout + r] = vb[e];
            }
            lout += tot;
        }
        if (lout > sl.lcap) {
            overflow = true;
            lout = sl.lcap;
        }
        __syncwarp();
        // ---- U part (factor.py:594-655)
        int nu = 0;
        const bool schur_row = i >= n_elim;
        if (!schur_row) {
            for (int b0 = pos; b0 < len; b0 += 32) {
                const int e = b0 + lane;
                const bool c = e < len && (ca[e] == i || fabs(va[e]) >= thresh);
                int tot;
                const int r = warp_compact_pos(c, &tot);
                if (c) {
                    cb[nu + r] = ca[e];
                    vb[nu + r] = va[e];
                }
                nu += tot;
            }
            __syncwarp();
            warp_select(cb, vb, nu, maxfill, i, sel);
        } else {
            // Schur row: own tolerance relative to the 2-norm of the kept part, no cap
            double snrm = 0.0;
            if (lane == 0) {
                for (int e = pos; e < len; ++e) snrm += va[e] * va[e];
                snrm = sqrt(snrm);
            }
            snrm = __shfl_sync(0xffffffffu, snrm, 0);
            const double sth = tau_s * snrm;
            for (int b0 = pos; b0 < len; b0 += 32) {
                const int e = b0 + lane;
                const bool c = e < len && (ca[e] == i || fabs(va[e]) >= sth);
                int tot;
                const int r = warp_compact_pos(c, &tot);
                if (c) {
                    cb[nu + r] = ca[e];
                    vb[nu + r] = va[e];
                }
                nu += tot;
            }
            __syncwarp();
            for (int e = lane; e < nu; e += 32) sel[e] = 1;
            __syncwarp();
        }
        const int ucap_row = schur_row ? sl.scap : sl.ucap;
        int uout = 0;
        const long long ubo = sl.uoff(i);
        for (int b0 = 0; b0 < nu; b0 += 32) {
            const int e = b0 + lane;
            const bool c = e < nu && sel[e];
            int tot;
            const int r = warp_compact_pos(c, &tot);
            if (c && uout + r < ucap_row) {
                double d = vb[e];
                if (cb[e] == i && !schur_row) {  // pivot safeguard (factor.py:646-651)
                    if (fabs(d) < delta * mx) d = d >= 0.0 ? delta * mx : -(delta * mx);
                }
                u_ci[ubo + uout + r] = cb[e];
                u_v[ubo + uout + r] = d;
            }
            uout += tot;
        }
        if (uout > ucap_row) {
            overflow = true;
            uout = ucap_row;
        }
        if (overflow && !schur_row && lane == 0) {  // keep later rows from dividing by garbage
            u_ci[ubo] = i;
            u_v[ubo] = 1.0;
            if (uout < 1) uout = 1;
        }
        if (lane == 0) {
            l_cnt[i] = lout;
            u_cnt[i] = uout;
            if (overflow) atomicExch(status, 1);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(done + i, 1);
    }
}

// slab -> CSR; offsets as in IlutSlabs (cap_a for rows < n_split, cap_b after)
__global__ void compact_rows(int n, int n_split, int cap_a, int cap_b, const int *__restrict__ cnt,
                             const int *__restrict__ ci, const double *__restrict__ v,
                             const int *__restrict__ out_rp, int *__restrict__ out_ci, double *__restrict__ out_v) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < n; i += nw) {
        const long long src = i < n_split ? i * cap_a : (long long)n_split * cap_a + (i - n_split) * cap_b;
        const int c = cnt[i], dst = out_rp[i];
        for (int e = lane; e < c; e += 32) {
            out_ci[dst + e] = ci[src + e];
            out_v[dst + e] = v[src + e];
        }
    }
}

static size_t ilut_smem(int cap) {
    size_t per_warp = (size_t)cap * (2 * sizeof(double) + 2 * sizeof(int)) + 32 * sizeof(int) + ((cap + 7) & ~7);
    return per_warp * ILUT_WARPS;
}

}  // namespace ddilu

using namespace ddilu;

extern "C" long long ddilu_ilut_smem_bytes(int row_cap) { return (long long)ilut_smem(row_cap); }

// slab sizes for the host: {lcap, ucap, scap}
extern "C" int ddilu_ilut_caps(int maxfill, int row_cap, int *caps_h) {
    caps_h[0] = maxfill < row_cap ? maxfill : row_cap;
    caps_h[1] = maxfill + 1 < row_cap ? maxfill + 1 : row_cap;
    caps_h[2] = row_cap;
    return DDILU_OK;
}

extern "C" int ddilu_ilut_factor(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim, double tau,
                                 int maxfill, double tau_s, double delta, int row_cap, int *l_cnt, int *l_ci,
                                 double *l_v, int *u_cnt, int *u_ci, double *u_v, int *done, int *status,
                                 const int *order, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (row_cap < 2) return DDILU_ERR_ARG;
    IlutSlabs sl;
    sl.n_elim = n_elim;
    sl.lcap = maxfill < row_cap ? maxfill : row_cap;
    sl.ucap = maxfill + 1 < row_cap ? maxfill + 1 : row_cap;
    sl.scap = row_cap;
    const size_t smem = ilut_smem(row_cap);
    if (smem > 200 * 1024) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaFuncSetAttribute(ilut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DDILU_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * (size_t)n, st));
    DDILU_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
    int occ = 0;
    DDILU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ilut_kernel, ILUT_WARPS * 32, smem));
    if (occ < 1) return DDILU_ERR_ARG;
    long long grid = (long long)occ * device_info().sm_count;
    const long long need = div_up(n, ILUT_WARPS);
    if (grid > need) grid = need;
    int g = (int)grid;
    void *args[] = {&n, &a_rp, &a_ci, &a_v, &tau, &maxfill, &tau_s, &delta, &row_cap, &sl,
                    &l_cnt, &l_ci, &l_v, &u_cnt, &u_ci, &u_v, &done, &status, &order};
    DDILU_CHECK(cudaLaunchCooperativeKernel((void *)ilut_kernel, g, ILUT_WARPS * 32, args, smem, st));
    return DDILU_OK;
}

extern "C" int ddilu_compact_rows(int n, int n_split, int cap_a, int cap_b, const int *cnt, const int *ci,
                                  const double *v, const int *out_rp, int *out_ci, double *out_v, void *stream) {
    if (n <= 0) return DDILU_OK;
    compact_rows<<<stream_grid(n, 256, 1, 16), 256, 0, (cudaStream_t)stream>>>(n, n_split, cap_a, cap_b, cnt, ci, v,
                                                                              out_rp, out_ci, out_v);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
