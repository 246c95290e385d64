// Level-0 split and numeric ILU(0) / MILU(0) / partial ILU(0).
//
// Replaces factor.py:198-246 (`_split_counts`, `_split_fill`), :435-443
// (`_row_inf_norms`) and :397-432 (`_factor_split`).
//
// The numeric kernel is the same sync-free design as the triangular solve:
// rows are visited in the level order of the L pattern by one persistent
// cooperative launch, one thread per row; a row waits on a per-row `done`
// flag (release/acquire at gpu scope) of each pivot row, reads that row's U
// values from L2, and applies the updates in exactly the reference order
// (pivots ascending, U entries ascending, product rounded then subtracted),
// so L/U values are bit-identical to the serial reference.
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

// pass 1: per-row sizes of the pivot (L) and kept (U, diagonal inserted) parts,
// and the row inf-norm of A used by the pivot safeguard.
__global__ void split_count(int n, const int *__restrict__ a_rp, const int *__restrict__ a_ci,
                            const double *__restrict__ a_v, int n_elim, int *__restrict__ pc, int *__restrict__ kc,
                            double *__restrict__ rownorm) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int lim = i < n_elim ? (int)i : n_elim;
        int npv = 0, nk = 0;
        bool has_diag = false;
        double m = 0.0;
        for (int s = a_rp[i], se = a_rp[i + 1]; s < se; ++s) {
            const int j = a_ci[s];
            if (j < lim) ++npv;
            else {
                ++nk;
                has_diag |= (j == i);
            }
            m = fmax(m, fabs(a_v[s]));
        }
        pc[i] = npv;
        kc[i] = nk + (has_diag ? 0 : 1);
        if (rownorm) rownorm[i] = m > 0.0 ? m : 1.0;
    }
}

__global__ void split_fill(int n, const int *__restrict__ a_rp, const int *__restrict__ a_ci,
                           const double *__restrict__ a_v, int n_elim, const int *__restrict__ p_rp,
                           int *__restrict__ p_ci, double *__restrict__ p_v, const int *__restrict__ k_rp,
                           int *__restrict__ k_ci, double *__restrict__ k_v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int lim = i < n_elim ? (int)i : n_elim;
        int pp = p_rp[i], kp = k_rp[i];
        bool placed = false;
        for (int s = a_rp[i], se = a_rp[i + 1]; s < se; ++s) {
            const int j = a_ci[s];
            if (j < lim) {
                p_ci[pp] = j;
                p_v[pp++] = a_v[s];
            } else {
                if (!placed && j > i) {
                    k_ci[kp] = (int)i;
                    k_v[kp++] = 0.0;
                    placed = true;
                }
                if (j == i) placed = true;
                k_ci[kp] = j;
                k_v[kp++] = a_v[s];
            }
        }
        if (!placed) {
            k_ci[kp] = (int)i;
            k_v[kp] = 0.0;
        }
    }
}

constexpr int ILU_THREADS = 128;

__global__ void __launch_bounds__(ILU_THREADS) ilu0_numeric(int n_slots, const int *__restrict__ order,
                                                            const int *__restrict__ p_rp, const int *__restrict__ p_ci,
                                                            double *p_v, const int *__restrict__ k_rp,
                                                            const int *__restrict__ k_ci, double *k_v, int n_elim,
                                                            int milu, const double *__restrict__ target,
                                                            const double *__restrict__ wvec, double delta,
                                                            const double *__restrict__ rownorm, int *done) {
    for (long long base = (long long)blockIdx.x * ILU_THREADS; base < n_slots;
         base += (long long)gridDim.x * ILU_THREADS) {
        const long long slot = base + threadIdx.x;
        if (slot >= n_slots) continue;
        const int i = order[slot];
        if (i < 0) continue;
        const int lim = i < n_elim ? i : n_elim;
        const int ps = p_rp[i], pe = p_rp[i + 1];
        const int ks = k_rp[i], ke = k_rp[i + 1];
        double hy = 0.0;
        for (int s = ps; s < pe; ++s) {
            const int k = p_ci[s];
            while (ld_acquire(done + k) == 0) {
            }
            const int ts = k_rp[k], te = k_rp[k + 1];
            const double lik = p_v[s] / ld_l2(k_v + ts);
            p_v[s] = lik;
            int pp = s + 1, kp = ks;  // both target lists are sorted: merge walk
            for (int t = ts + 1; t < te; ++t) {
                const int j = k_ci[t];
                const double upd = lik * ld_l2(k_v + t);
                if (j < lim) {
                    while (pp < pe && p_ci[pp] < j) ++pp;
                    if (pp < pe && p_ci[pp] == j) p_v[pp] -= upd;
                    else if (milu) hy -= upd * target[j];
                } else {
                    while (kp < ke && k_ci[kp] < j) ++kp;
                    if (kp < ke && k_ci[kp] == j) k_v[kp] -= upd;
                    else if (milu) hy -= upd * target[j];
                }
            }
        }
        if (i < n_elim) {
            if (milu) k_v[ks] += (hy - wvec[i]) / target[i];
            const double rn = rownorm[i], d = k_v[ks];
            if (fabs(d) < delta * rn) k_v[ks] = d >= 0.0 ? delta * rn : -(delta * rn);
        }
        __threadfence();
        st_release(done + i, 1);
    }
}

// rows [r0, r1) x columns [c0, c1) of a row-sorted CSR matrix, columns shifted by -c0
__global__ void block_count(const int *__restrict__ rp, const int *__restrict__ ci, int r0, int r1, int c0, int c1,
                            int *__restrict__ counts) {
    for (long long r = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
         r += (long long)gridDim.x * blockDim.x) {
        int c = 0;
        for (int s = rp[r], se = rp[r + 1]; s < se; ++s) c += (ci[s] >= c0 && ci[s] < c1);
        counts[r - r0] = c;
    }
}

__global__ void block_fill(const int *__restrict__ rp, const int *__restrict__ ci, const double *__restrict__ v, int r0,
                           int r1, int c0, int c1, const int *__restrict__ out_rp, int *__restrict__ out_ci,
                           double *__restrict__ out_v) {
    for (long long r = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
         r += (long long)gridDim.x * blockDim.x) {
        int p = out_rp[r - r0];
        for (int s = rp[r], se = rp[r + 1]; s < se; ++s) {
            const int j = ci[s];
            if (j >= c0 && j < c1) {
                out_ci[p] = j - c0;
                out_v[p++] = v[s];
            }
        }
    }
}

}  // namespace ddilu

using namespace ddilu;

extern "C" int ddilu_split_count(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim, int *pc,
                                 int *kc, double *rownorm, void *stream) {
    if (n <= 0) return DDILU_OK;
    split_count<<<stream_grid(n, 256), 256, 0, (cudaStream_t)stream>>>(n, a_rp, a_ci, a_v, n_elim, pc, kc, rownorm);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_split_fill(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim,
                                const int *p_rp, int *p_ci, double *p_v, const int *k_rp, int *k_ci, double *k_v,
                                void *stream) {
    if (n <= 0) return DDILU_OK;
    split_fill<<<stream_grid(n, 256), 256, 0, (cudaStream_t)stream>>>(n, a_rp, a_ci, a_v, n_elim, p_rp, p_ci, p_v,
                                                                      k_rp, k_ci, k_v);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_ilu0_numeric(int n, int n_slots, const int *order, const int *p_rp, const int *p_ci, double *p_v,
                                  const int *k_rp, const int *k_ci, double *k_v, int n_elim, int milu,
                                  const double *target, const double *wvec, double delta, const double *rownorm,
                                  int *done, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    if (milu && (!target || !wvec)) return DDILU_ERR_ARG;
    DDILU_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * (size_t)n, st));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ilu0_numeric, ILU_THREADS, 0);
    if (occ < 1) occ = 1;
    long long grid = (long long)occ * device_info().sm_count;
    long long need = div_up(n_slots, ILU_THREADS);
    if (grid > need) grid = need;
    int g = (int)grid;
    void *args[] = {&n_slots, &order, &p_rp, &p_ci, &p_v, &k_rp, &k_ci, &k_v, &n_elim,
                    &milu, &target, &wvec, &delta, &rownorm, &done};
    DDILU_CHECK(cudaLaunchCooperativeKernel((void *)ilu0_numeric, g, ILU_THREADS, args, 0, st));
    return DDILU_OK;
}

extern "C" int ddilu_csr_block_count(const int *rp, const int *ci, int r0, int r1, int c0, int c1, int *counts,
                                     void *stream) {
    if (r1 <= r0) return DDILU_OK;
    block_count<<<stream_grid(r1 - r0, 256), 256, 0, (cudaStream_t)stream>>>(rp, ci, r0, r1, c0, c1, counts);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_csr_block_fill(const int *rp, const int *ci, const double *v, int r0, int r1, int c0, int c1,
                                    const int *out_rp, int *out_ci, double *out_v, void *stream) {
    if (r1 <= r0) return DDILU_OK;
    block_fill<<<stream_grid(r1 - r0, 256), 256, 0, (cudaStream_t)stream>>>(rp, ci, v, r0, r1, c0, c1, out_rp, out_ci,
                                                                             out_v);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
