// CSR SpMV, fp64 values / int32 indices (replaces sparse.py:219-225 `_spmv`).
//
// "CSR-stream": a CTA owns ROWS consecutive rows; their entries are one
// contiguous slice of (col_idx, values), read with fully coalesced loads, the
// products val*x[col] are staged in shared memory, then one thread per row adds
// its products strictly left to right.  Each product is rounded before it is
// added (-fmad=false), so the result is bit-identical to the serial reference.
// x may carry a halo tail (columns >= n_local hold interface values received
// from other ranks); interior rows never touch it, so the caller launches the
// interior row range while the halo is still in flight.
//
// Algorithmic bytes: 12*nnz + 4*(rows+1) + 8*cols_touched + 8*rows (+8*rows for b).
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int SPMV_UNROLL = 8;       // entries per thread and round

// mode 0: y = A x      mode 1: y = b - A x      mode 2: y = b + A x
// ROWS rows (= threads) per CTA, STAGE products staged per CTA: chosen by the launcher from the average
// row length so that a CTA's entries fit the stage and as many CTAs as possible are resident
template <int MODE, int ROWS, int STAGE>
__global__ void __launch_bounds__(ROWS) spmv_stream(int r0, int r1, const int *__restrict__ rp,
                                                    const int *__restrict__ ci, const double *__restrict__ val,
                                                    const double *__restrict__ x, const double *__restrict__ b,
                                                    double *__restrict__ y) {
    __shared__ double prod[STAGE];
    __shared__ int srp[ROWS + 1];
    const int row0 = r0 + blockIdx.x * ROWS;
    const int nrows = min(ROWS, r1 - row0);
    if (threadIdx.x < nrows) srp[threadIdx.x] = rp[row0 + threadIdx.x];
    if (threadIdx.x == 0) srp[nrows] = rp[row0 + nrows];
    __syncthreads();
    const int e0 = srp[0], e1 = srp[nrows];
    const int row = row0 + threadIdx.x;
    if (e1 - e0 <= STAGE) {
        // all (column, value) loads of a round in flight together, then all the x gathers: eight
        // independent 2-deep load chains per thread instead of one (HBM latency x bandwidth needs ~44 KB
        // in flight per SM)
        for (int base = e0 + threadIdx.x; base < e1; base += SPMV_UNROLL * ROWS) {
            int c[SPMV_UNROLL];
            double v[SPMV_UNROLL], xv[SPMV_UNROLL];
#pragma unroll
            for (int u = 0; u < SPMV_UNROLL; ++u) {
                const int e = base + u * ROWS;
                const bool in = e < e1;
                c[u] = in ? ci[e] : -1;
                v[u] = in ? val[e] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SPMV_UNROLL; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : 0.0;
#pragma unroll
            for (int u = 0; u < SPMV_UNROLL; ++u)
                if (c[u] >= 0) prod[base + u * ROWS - e0] = v[u] * xv[u];
        }
        __syncthreads();
        if (threadIdx.x < nrows) {
            double s = 0.0;
            for (int k = srp[threadIdx.x] - e0, ke = srp[threadIdx.x + 1] - e0; k < ke; ++k) s += prod[k];
            if (MODE == 1) s = b[row] - s;
            if (MODE == 2) s = b[row] + s;
            y[row] = s;
        }
    } else if (threadIdx.x < nrows) {  // long rows: plain row loop, same summation order
        double s = 0.0;
        for (int k = srp[threadIdx.x], ke = srp[threadIdx.x + 1]; k < ke; ++k) s += val[k] * x[ci[k]];
        if (MODE == 1) s = b[row] - s;
        if (MODE == 2) s = b[row] + s;
        y[row] = s;
    }
}

template <int ROWS, int STAGE>
static int spmv_launch(int row_begin, int row_end, const int *rp, const int *ci, const double *val, const double *x,
                       const double *b, double *y, int mode, cudaStream_t st) {
    const int grid = div_up(row_end - row_begin, ROWS);
    if (mode == 0) spmv_stream<0, ROWS, STAGE><<<grid, ROWS, 0, st>>>(row_begin, row_end, rp, ci, val, x, b, y);
    else if (mode == 1) spmv_stream<1, ROWS, STAGE><<<grid, ROWS, 0, st>>>(row_begin, row_end, rp, ci, val, x, b, y);
    else spmv_stream<2, ROWS, STAGE><<<grid, ROWS, 0, st>>>(row_begin, row_end, rp, ci, val, x, b, y);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

}  // namespace ddilu

using namespace ddilu;

/* avg_row_len: entries per row of the range (0 = unknown) -- picks rows per CTA and stage size */
extern "C" int ddilu_spmv_csr_f64_tuned(int row_begin, int row_end, const int *row_ptr, const int *col_idx,
                                        const double *values, const double *x, const double *b, double *y, int mode,
                                        double avg_row_len, void *stream) {
    if (row_end <= row_begin) return DDILU_OK;
    if ((mode != 0 && !b) || mode < 0 || mode > 2) return DDILU_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (avg_row_len > 0.0 && avg_row_len <= 7.5)
        return spmv_launch<256, 2048>(row_begin, row_end, row_ptr, col_idx, values, x, b, y, mode, st);
    if (avg_row_len <= 0.0 || avg_row_len <= 15.0)
        return spmv_launch<256, 4096>(row_begin, row_end, row_ptr, col_idx, values, x, b, y, mode, st);
    if (avg_row_len <= 30.0)
        return spmv_launch<128, 4096>(row_begin, row_end, row_ptr, col_idx, values, x, b, y, mode, st);
    return spmv_launch<64, 4096>(row_begin, row_end, row_ptr, col_idx, values, x, b, y, mode, st);
}

extern "C" int ddilu_spmv_csr_f64(int row_begin, int row_end, const int *row_ptr, const int *col_idx,
                                  const double *values, const double *x, const double *b, double *y, int mode,
                                  void *stream) {
    return ddilu_spmv_csr_f64_tuned(row_begin, row_end, row_ptr, col_idx, values, x, b, y, mode, 0.0, stream);
}
