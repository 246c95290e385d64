// Instrumented twin of sptrsv_sell (diagnostics only; scripts/trace_trsv.py):
// records per group the global timer at (0) group start, (1) single-address spin
// satisfied, (2) all dependencies loaded, (3) result stored, plus the SM id.
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

__device__ __forceinline__ long long gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int smid() {
    int s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

constexpr int TR_CHUNK = 4;

__global__ void __launch_bounds__(256) sptrsv_sell_trace(int n_groups, const int *__restrict__ order,
                                                         const int *__restrict__ goff, int uw,
                                                         const int *__restrict__ scol, const double *__restrict__ sval,
                                                         const double *__restrict__ sdiag,
                                                         const int *__restrict__ gwait, const double *__restrict__ b,
                                                         double *x, long long *stamps) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long g = warp; g < n_groups; g += nw) {
        const long long off = goff ? goff[g] : g * 32LL * uw;
        const int w = goff ? (goff[g + 1] - (int)off) >> 5 : uw;
        const int row = order[g * 32 + lane];
        const int wait_col = gwait ? gwait[g] : -1;
        double s = row >= 0 ? b[row] : 0.0;
        const double d = sdiag ? sdiag[g * 32 + lane] : 1.0;
        int c[TR_CHUNK];
        double a[TR_CHUNK];
#pragma unroll
        for (int u = 0; u < TR_CHUNK; ++u) {
            const bool in = u < w;
            c[u] = in ? scol[off + 32 * u + lane] : -1;
            a[u] = in ? sval[off + 32 * u + lane] : 0.0;
        }
        // make sure the operands have arrived before the first stamp
        long long dep = (long long)row + c[0] + c[1] + c[2] + c[3] + (long long)(a[0] + a[1] + a[2] + a[3] + s + d);
        const long long t0 = gtime() + (dep == 0x7fffffffffffffffLL);
        long long spins = 0;
        if (wait_col >= 0)
            while (is_sentinel(ld_l2(x + wait_col))) ++spins;
        const long long t1 = gtime();
        double xv[TR_CHUNK];
#pragma unroll
        for (int u = 0; u < TR_CHUNK; ++u) xv[u] = c[u] >= 0 ? ld_l2(x + c[u]) : 0.0;
        bool pending;
        long long rounds = 0;
        do {
            pending = false;
#pragma unroll
            for (int u = 0; u < TR_CHUNK; ++u)
                if (is_sentinel(xv[u])) {
                    xv[u] = ld_l2(x + c[u]);
                    pending |= is_sentinel(xv[u]);
                }
            rounds += __any_sync(0xffffffffu, pending) ? 1 : 0;
        } while (__any_sync(0xffffffffu, pending));
        const long long t2 = gtime();
#pragma unroll
        for (int u = 0; u < TR_CHUNK; ++u)
            if (c[u] >= 0) s -= a[u] * xv[u];
        for (int k = TR_CHUNK; k < w; ++k) {  // long rows (not traced separately)
            const int j = scol[off + 32 * k + lane];
            if (j >= 0) {
                double v = ld_l2(x + j);
                while (is_sentinel(v)) v = ld_l2(x + j);
                s -= sval[off + 32 * k + lane] * v;
            }
        }
        if (row >= 0) st_l2(x + row, scrub_sentinel(sdiag ? s / d : s));
        const long long t3 = gtime();
        if (lane == 0) {
            long long *o = stamps + g * 8;
            o[0] = t0; o[1] = t1; o[2] = t2; o[3] = t3; o[4] = smid(); o[5] = spins; o[6] = rounds; o[7] = warp;
        }
    }
}

}  // namespace ddilu

using namespace ddilu;

extern "C" int ddilu_sptrsv_sell_trace(int n, int n_slots, int blocks_per_sm, const int *order, const int *goff,
                                       int uniform_width, const int *scol, const double *sval, const double *sdiag,
                                       const int *gwait, const double *b, double *x, long long *stamps, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return DDILU_OK;
    DDILU_CHECK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n, st));
    int n_groups = n_slots >> 5;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sptrsv_sell_trace, 256, 0);
    if (occ < 1) occ = 1;
    if (blocks_per_sm > 0 && occ > blocks_per_sm) occ = blocks_per_sm;
    long long grid = (long long)occ * device_info().sm_count;
    long long need = ((long long)n_slots + 255) / 256;
    if (grid > need) grid = need;
    int g = (int)grid;
    void *args[] = {&n_groups, &order, &goff, &uniform_width, &scol, &sval, &sdiag, &gwait, &b, &x, &stamps};
    DDILU_CHECK(cudaLaunchCooperativeKernel((void *)sptrsv_sell_trace, g, 256, args, 0, st));
    return DDILU_OK;
}
