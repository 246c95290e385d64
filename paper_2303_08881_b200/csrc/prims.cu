// Scan and stable radix-sort primitives used by the setup kernels
// (count -> scan -> fill pipelines; level-schedule bucketing; layout ordering).
// HBM-bound integer work: coalesced tiles, shared-memory staging.
#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int block_exclusive_scan(int v, int *total) {
    // 256 threads: warp shuffles + one shared exchange
    __shared__ int warp_tot[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    int base = 0, all = 0;
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
        int t = warp_tot[w];
        if (w < warp) base += t;
        all += t;
    }
    __syncthreads();
    *total = all;
    return base + inc - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_sums(const int *__restrict__ in, long long n,
                                                               int *__restrict__ sums) {
    const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
        if (base + k < n) s += in[base + k];
    int total;
    block_exclusive_scan(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// single CTA: exclusive scan of the tile sums in place; sums[nb] = grand total
__global__ void __launch_bounds__(SCAN_THREADS) scan_sums(int *sums, int nb) {
    __shared__ int carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += SCAN_THREADS) {
        int i = base + threadIdx.x;
        int v = i < nb ? sums[i] : 0;
        int total;
        int ex = block_exclusive_scan(v, &total);
        int carry = carry_s;
        if (i < nb) sums[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nb] = carry_s;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_apply(const int *in, long long n, const int *__restrict__ sums,
                                                           int nb, int *out) {
    const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    int total;
    int run = block_exclusive_scan(s, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (blockIdx.x == nb - 1 && threadIdx.x == 0) out[n] = sums[nb];
}

__global__ void scan_empty(int *out) { out[0] = 0; }

// ---------------------------------------------------------------- radix sort
constexpr int RS_WARPS = 8, RS_ROUNDS = 8, RS_TILE = RS_WARPS * RS_ROUNDS * 32;

__device__ __forceinline__ void radix_count(const int *__restrict__ keys, long long n, int shift, int *digit,
                                            int (*wh)[256]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b = threadIdx.x; b < RS_WARPS * 256; b += blockDim.x) (&wh[0][0])[b] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * RS_TILE + (long long)warp * RS_ROUNDS * 32 + lane;
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        long long i = base + r * 32;
        int d = i < n ? ((keys[i] >> shift) & 255) : 256;
        digit[r] = d;
        unsigned m = __match_any_sync(0xffffffffu, d);
        if (d < 256 && lane == __ffs(m) - 1) wh[warp][d] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(RS_WARPS * 32) radix_hist(const int *__restrict__ keys, long long n, int shift,
                                                            int *__restrict__ hist, int nb) {
    __shared__ int wh[RS_WARPS][256];
    int digit[RS_ROUNDS];
    radix_count(keys, n, shift, digit, wh);
    int bin = threadIdx.x, t = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) t += wh[w][bin];
    hist[(long long)bin * nb + blockIdx.x] = t;
}

__global__ void __launch_bounds__(RS_WARPS * 32) radix_scatter(const int *__restrict__ keys, const int *__restrict__ vals,
                                                               int *__restrict__ keys_out, int *__restrict__ vals_out,
                                                               long long n, int shift, const int *__restrict__ offs,
                                                               int nb) {
    __shared__ int wh[RS_WARPS][256];
    int digit[RS_ROUNDS];
    radix_count(keys, n, shift, digit, wh);
    {
        int bin = threadIdx.x;
        int run = offs[(long long)bin * nb + blockIdx.x];
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            int c = wh[w][bin];
            wh[w][bin] = run;
            run += c;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long base = (long long)blockIdx.x * RS_TILE + (long long)warp * RS_ROUNDS * 32 + lane;
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        long long i = base + r * 32;
        int d = digit[r];
        unsigned m = __match_any_sync(0xffffffffu, d);
        int pos = 0;
        if (d < 256) pos = wh[warp][d] + __popc(m & ((1u << lane) - 1u));
        __syncwarp();
        if (d < 256 && lane == __ffs(m) - 1) wh[warp][d] += __popc(m);
        __syncwarp();
        if (d < 256) {
            keys_out[pos] = keys[i];
            if (vals) vals_out[pos] = vals[i];
        }
    }
}

}  // namespace ddilu

using namespace ddilu;

extern "C" long long ddilu_scan_tmp_elems(long long n) { return div_up(n, SCAN_TILE) + 2; }

extern "C" int ddilu_exclusive_scan_i32(const int *in, int *out, long long n, int *tmp, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0) return DDILU_ERR_ARG;
    if (n == 0) {
        scan_empty<<<1, 1, 0, st>>>(out);
        DDILU_LAUNCH_CHECK();
        return DDILU_OK;
    }
    int nb = div_up(n, SCAN_TILE);
    scan_tile_sums<<<nb, SCAN_THREADS, 0, st>>>(in, n, tmp);
    scan_sums<<<1, SCAN_THREADS, 0, st>>>(tmp, nb);
    scan_apply<<<nb, SCAN_THREADS, 0, st>>>(in, n, tmp, nb, out);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" long long ddilu_sort_tmp_elems(long long n) {
    long long nb = div_up(n > 0 ? n : 1, RS_TILE);
    long long h = 256 * nb;
    return h + 1 + ddilu_scan_tmp_elems(h);
}

// Stable LSD radix sort of (key, value) int32 pairs on the low `bits` key bits.
// The sorted pairs end in (keys, vals); (keys_alt, vals_alt) is scratch.
extern "C" int ddilu_sort_pairs_i32(int *keys, int *vals, int *keys_alt, int *vals_alt, long long n, int bits,
                                    int *tmp, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 1) return DDILU_OK;
    int nb = div_up(n, RS_TILE);
    long long h = 256LL * nb;
    int *hist = tmp, *scan_tmp = tmp + h + 1;
    int passes = (bits + 7) / 8;
    if (passes < 1) passes = 1;
    int *ka = keys, *va = vals, *kb = keys_alt, *vb = vals_alt;
    for (int p = 0; p < passes; ++p) {
        radix_hist<<<nb, RS_WARPS * 32, 0, st>>>(ka, n, 8 * p, hist, nb);
        int rc = ddilu_exclusive_scan_i32(hist, hist, h, scan_tmp, stream);
        if (rc) return rc;
        radix_scatter<<<nb, RS_WARPS * 32, 0, st>>>(ka, va, kb, vb, n, 8 * p, hist, nb);
        DDILU_LAUNCH_CHECK();
        int *t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    if (ka != keys) {
        DDILU_CHECK(cudaMemcpyAsync(keys, ka, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
        if (vals) DDILU_CHECK(cudaMemcpyAsync(vals, va, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    }
    return DDILU_OK;
}
