// Krylov vector kernels (replace sparse.py:275-280 `_vdot`, krylov.py:74-77
// `_axpy` and the numpy vector expressions inside krylov.py `_restarted` /
// `fixed_gmres`).  All HBM-bound streaming passes: 16-byte vector loads, a
// whole number of waves, deterministic two-stage reductions (per-CTA partials,
// the last CTA to finish adds them in CTA order), scalars kept on the device so
// an Arnoldi step is a chain of launches with no host round trip.
//
// Algorithmic bytes: dot 16n; axpy 24n; fused axpy+dot 32n (the reference's
// separate dot and axpy move 40n per MGS step).
#include <string.h>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

constexpr int VEC_THREADS = 256;
constexpr int RED_MAX_BLOCKS = 1024;  // partial buffer: RED_MAX_BLOCKS doubles + ticket

struct RedWs {
    double partial[RED_MAX_BLOCKS];
    unsigned int ticket;
};

__device__ __forceinline__ bool aligned16(const void *a, const void *b) {
    return (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[VEC_THREADS / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < VEC_THREADS / 32 ? ws[threadIdx.x] : 0.0;
        t = warp_sum(t);
    }
    return t;  // valid in warp 0
}

// publish this CTA's partial; the last CTA adds all partials in index order
__device__ __forceinline__ void finish_reduction(double part, RedWs *ws, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        ws->partial[blockIdx.x] = part;
        __threadfence();
        unsigned t = atomicAdd(&ws->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
        __threadfence();
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) s += ld_l2(&ws->partial[b]);
        s = warp_sum(s);
        if (threadIdx.x == 0) {
            *out = s;
            ws->ticket = 0;
        }
    }
}

// out = sum x[i]*y[i]
__global__ void __launch_bounds__(VEC_THREADS) dot_kernel(long long n, const double *__restrict__ x,
                                                          const double *__restrict__ y, RedWs *ws, double *out,
                                                          int reverse) {
    double acc = 0.0;
    const long long n2 = aligned16(x, y) ? n >> 1 : 0;  // 16-byte path only when both operands allow it
    const double2 *x2 = reinterpret_cast<const double2 *>(x), *y2 = reinterpret_cast<const double2 *>(y);
    for (long long q = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; q < n2; q += (long long)gridDim.x * VEC_THREADS) {
        const long long i = reverse ? n2 - 1 - q : q;
        double2 a = x2[i], b = y2[i];
        acc += a.x * b.x;
        acc += a.y * b.y;
    }
    for (long long i = 2 * n2 + (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS)
        acc += x[i] * y[i];
    double part = block_sum(acc);
    finish_reduction(part, ws, out);
}

// w += (sign * *alpha_dev or alpha_host) * v ; optionally out = dot(u, w_new)
// (u == w gives the squared norm).  One pass: 32n bytes with the dot, 24n without.
template <bool DOT>
// reverse: walk the vectors from the end.  Consecutive MGS steps alternate the direction, so a step starts
// with the ~L2-sized tail of w and of the basis vector that the previous step touched last.
__global__ void __launch_bounds__(VEC_THREADS) axpy_dot_kernel(long long n, const double *alpha_dev, double alpha_host,
                                                               const double *__restrict__ v, double *w, const double *u,
                                                               RedWs *ws, double *out, int reverse) {
    const double alpha = alpha_dev ? alpha_host * (*alpha_dev) : alpha_host;
    double acc = 0.0;
    const long long n2 = (aligned16(v, w) && aligned16(u ? u : w, w)) ? n >> 1 : 0;
    const double2 *v2 = reinterpret_cast<const double2 *>(v);
    double2 *w2 = reinterpret_cast<double2 *>(w);
    const double2 *u2 = reinterpret_cast<const double2 *>(u);
    const bool self = (u == w);
    for (long long q = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; q < n2; q += (long long)gridDim.x * VEC_THREADS) {
        const long long i = reverse ? n2 - 1 - q : q;
        double2 a = v2[i], b = w2[i];
        b.x += alpha * a.x;
        b.y += alpha * a.y;
        w2[i] = b;
        if (DOT) {
            double2 c = self ? b : u2[i];
            acc += c.x * b.x;
            acc += c.y * b.y;
        }
    }
    for (long long i = 2 * n2 + (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS) {
        double b = w[i] + alpha * v[i];
        w[i] = b;
        if (DOT) acc += (self ? b : u[i]) * b;
    }
    if (DOT) {
        double part = block_sum(acc);
        finish_reduction(part, ws, out);
    }
}

// ---- blocked modified Gram-Schmidt (krylov.py:131-136 restated for blocks of up to MGS_K basis vectors) ----------
// MGS orthogonalises w against v_0..v_j one vector at a time: h_i = <v_i, w_i>, w_{i+1} = w_i - h_i v_i; every
// step is a pass over w.  Inside a block of k vectors the same coefficients follow from ONE pass:
//   d_i = <v_i, w_0>,  G_il = <v_i, v_l> (l < i)   =>   h_i = d_i - sum_{l<i} h_l G_il   ( = <v_i, w_i> ),
// so a pass (a) subtracts the previous block, w -= sum h_l v_l in the MGS order, and (b) accumulates d and G of
// the next block against the updated w.  Traffic per MGS step: (16/k + 16) n bytes instead of 32 n.
// The raw sums [d_0..d_{k-1}, G_10, G_20, G_21, G_30, ...] go through the same deterministic two-stage
// reduction as the dots (and through ONE allreduce with several ranks); the k x k recurrence is redone by every
// thread of the consuming pass, whose first thread also stores the coefficients into the Hessenberg column.
constexpr int MGS_K = 8;
constexpr int MGS_NRED = MGS_K + MGS_K * (MGS_K - 1) / 2;

struct MgsWs {
    double partial[MGS_NRED][RED_MAX_BLOCKS];
    unsigned int ticket;
    unsigned int bar[3];  // grid barriers of mgs_small_step_kernel (two counters + the exit ticket that clears them)
};

template <int NA>
__device__ __forceinline__ void finish_reduction_multi(const double (&acc)[NA], MgsWs *ws, double *out) {
    __shared__ double sm[NA][VEC_THREADS / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        double v = warp_sum(acc[a]);
        if (lane == 0) sm[a][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < VEC_THREADS / 32; ++q) t += sm[threadIdx.x][q];
        ws->partial[threadIdx.x][blockIdx.x] = t;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = atomicAdd(&ws->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        for (int a = warp; a < NA; a += VEC_THREADS / 32) {
            double s = 0.0;
            for (unsigned b = lane; b < gridDim.x; b += 32) s += ld_l2(&ws->partial[a][b]);
            s = warp_sum(s);
            if (lane == 0) out[a] = s;
        }
        if (threadIdx.x == 0) ws->ticket = 0;
    }
}

// one pass: w -= sum_{l<KP} h_l vprev_l (h from raw_prev, stored to hout), then raw sums of vnext_0..KN-1 against
// the updated w into out[0 .. KN + KN(KN-1)/2); KN == 0: out[0] = <w, w>.
template <int KP, int KN>
__global__ void __launch_bounds__(VEC_THREADS) mgs_block_kernel(long long n, long long ld,
                                                                const double *__restrict__ vprev,
                                                                const double *__restrict__ raw_prev, double *hout,
                                                                double *w, const double *__restrict__ vnext, MgsWs *ws,
                                                                double *out, int reverse) {
    constexpr int KPA = KP > 0 ? KP : 1;
    constexpr int NA = KN > 0 ? KN + KN * (KN - 1) / 2 : 1;
    double nh[KPA];
    if (KP > 0) {
        double h[KPA];
        int g = KP;
#pragma unroll
        for (int i = 0; i < KP; ++i) {
            double s = raw_prev[i];
#pragma unroll
            for (int l = 0; l < i; ++l) s -= h[l] * raw_prev[g++];
            h[i] = s;
            nh[i] = -s;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < KP; ++i) hout[i] = h[i];
        }
    }
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    const bool al = ((((uintptr_t)w | (uintptr_t)(KP > 0 ? vprev : w) | (uintptr_t)(KN > 0 ? vnext : w)) & 15) == 0) &&
                    ((ld & 1) == 0);
    const long long n2 = al ? n >> 1 : 0, ld2 = ld >> 1;
    double2 *w2 = reinterpret_cast<double2 *>(w);
    const double2 *p2 = reinterpret_cast<const double2 *>(vprev), *q2 = reinterpret_cast<const double2 *>(vnext);
    for (long long q = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; q < n2; q += (long long)gridDim.x * VEC_THREADS) {
        const long long i = reverse ? n2 - 1 - q : q;
        double2 b = w2[i];
        if (KP > 0) {
            double2 a[KPA];
#pragma unroll
            for (int l = 0; l < KP; ++l) a[l] = p2[l * ld2 + i];
#pragma unroll
            for (int l = 0; l < KP; ++l) {
                b.x += nh[l] * a[l].x;
                b.y += nh[l] * a[l].y;
            }
            w2[i] = b;
        }
        if (KN > 0) {
            double2 c[KN > 0 ? KN : 1];
#pragma unroll
            for (int j = 0; j < KN; ++j) c[j] = q2[j * ld2 + i];
            int g = KN;
#pragma unroll
            for (int j = 0; j < KN; ++j) {
                acc[j] += c[j].x * b.x;
                acc[j] += c[j].y * b.y;
#pragma unroll
                for (int l = 0; l < j; ++l) {
                    acc[g] += c[j].x * c[l].x;
                    acc[g] += c[j].y * c[l].y;
                    ++g;
                }
            }
        } else {
            acc[0] += b.x * b.x;
            acc[0] += b.y * b.y;
        }
    }
    for (long long i = 2 * n2 + (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS) {
        double b = w[i];
        if (KP > 0) {
#pragma unroll
            for (int l = 0; l < KP; ++l) b += nh[l] * vprev[l * ld + i];
            w[i] = b;
        }
        if (KN > 0) {
            double c[KN > 0 ? KN : 1];
#pragma unroll
            for (int j = 0; j < KN; ++j) c[j] = vnext[j * ld + i];
            int g = KN;
#pragma unroll
            for (int j = 0; j < KN; ++j) {
                acc[j] += c[j] * b;
#pragma unroll
                for (int l = 0; l < j; ++l) acc[g++] += c[j] * c[l];
            }
        } else {
            acc[0] += b * b;
        }
    }
    finish_reduction_multi<NA>(acc, ws, out);
}

template <int KP>
static void mgs_launch_kn(int kn, int grid, cudaStream_t st, long long n, long long ld, const double *vprev,
                          const double *raw_prev, double *hout, double *w, const double *vnext, MgsWs *ws, double *out,
                          int reverse) {
#define DDILU_MGS_CASE(KN)                                                                                           \
    case KN:                                                                                                         \
        mgs_block_kernel<KP, KN><<<grid, VEC_THREADS, 0, st>>>(n, ld, vprev, raw_prev, hout, w, vnext, ws, out, reverse); \
        break;
    switch (kn) {
        DDILU_MGS_CASE(0)
        DDILU_MGS_CASE(1)
        DDILU_MGS_CASE(2)
        DDILU_MGS_CASE(3)
        DDILU_MGS_CASE(4)
        DDILU_MGS_CASE(5)
        DDILU_MGS_CASE(6)
        DDILU_MGS_CASE(7)
        DDILU_MGS_CASE(8)
    }
#undef DDILU_MGS_CASE
}

// ---- one Arnoldi step on a SHORT vector in one launch (the inner GMRES of the two-level preconditioners works on
// the interface unknowns: a few hundred thousand doubles, every kernel there is launch-bound).  Phases = the three
// launches it replaces, with the same grid, the same per-thread loops and the same reduction order, so the bits
// are the same: (1) mgs_block_kernel<0, K>: raw sums of v_0..v_{K-1} against w, (2) mgs_block_kernel<K, 0>:
// w -= sum h_l v_l, <w, w>, (3) scale_kernel: vout = w / sqrt(<w, w>).  Between the phases a grid barrier (the grid
// is launched cooperatively: all CTAs resident) after which EVERY CTA adds the partials in the order the last CTA
// of the separate kernels would.  hout[0..K) = h, hout[K] = <w, w>.
__device__ __forceinline__ void grid_barrier(unsigned int *counter) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        while (ld_l2(reinterpret_cast<const int *>(counter)) < (int)gridDim.x) __nanosleep(20);
        __threadfence();
    }
    __syncthreads();
}

template <int K>
__global__ void __launch_bounds__(VEC_THREADS, 4) mgs_small_step_kernel(long long n, long long ld,
                                                                        const double *__restrict__ v, double *w,
                                                                        double *hout, double *vout, MgsWs *ws,
                                                                        int reverse_dots, int reverse_update) {
    constexpr int NA = K + K * (K - 1) / 2;
    constexpr int ROW2 = MGS_NRED - 1;   // partial row of the phase-2 sum: phase-1 rows may still be read by slower CTAs
    __shared__ double sm[NA][VEC_THREADS / 32];
    __shared__ double tot[NA + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool al = ((((uintptr_t)w | (uintptr_t)v) & 15) == 0) && ((ld & 1) == 0);
    const long long n2 = al ? n >> 1 : 0, ld2 = ld >> 1;
    double2 *w2 = reinterpret_cast<double2 *>(w);
    const double2 *p2 = reinterpret_cast<const double2 *>(v);
    const long long q0 = (long long)blockIdx.x * VEC_THREADS + threadIdx.x, qs = (long long)gridDim.x * VEC_THREADS;

    // phase 1: raw sums (mgs_block_kernel<0, K>)
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    for (long long q = q0; q < n2; q += qs) {
        const long long i = reverse_dots ? n2 - 1 - q : q;
        const double2 b = w2[i];
        double2 c[K];
#pragma unroll
        for (int j = 0; j < K; ++j) c[j] = p2[j * ld2 + i];
        int g = K;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            acc[j] += c[j].x * b.x;
            acc[j] += c[j].y * b.y;
#pragma unroll
            for (int l = 0; l < j; ++l) {
                acc[g] += c[j].x * c[l].x;
                acc[g] += c[j].y * c[l].y;
                ++g;
            }
        }
    }
    for (long long i = 2 * n2 + q0; i < n; i += qs) {
        const double b = w[i];
        double c[K];
#pragma unroll
        for (int j = 0; j < K; ++j) c[j] = v[j * ld + i];
        int g = K;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            acc[j] += c[j] * b;
#pragma unroll
            for (int l = 0; l < j; ++l) acc[g++] += c[j] * c[l];
        }
    }
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        const double t = warp_sum(acc[a]);
        if (lane == 0) sm[a][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < VEC_THREADS / 32; ++q) t += sm[threadIdx.x][q];
        st_l2(&ws->partial[threadIdx.x][blockIdx.x], t);
        __threadfence();
    }
    grid_barrier(&ws->bar[0]);
    for (int a = warp; a < NA; a += VEC_THREADS / 32) {
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += ld_l2(&ws->partial[a][b]);
        s = warp_sum(s);
        if (lane == 0) tot[a] = s;
    }
    __syncthreads();

    // phase 2: coefficients of the block recurrence, update, <w, w> (mgs_block_kernel<K, 0>)
    double h[K], nh[K];
    {
        int g = K;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            double s = tot[i];
#pragma unroll
            for (int l = 0; l < i; ++l) s -= h[l] * tot[g++];
            h[i] = s;
            nh[i] = -s;
        }
    }
    double ww = 0.0;
    for (long long q = q0; q < n2; q += qs) {
        const long long i = reverse_update ? n2 - 1 - q : q;
        double2 b = w2[i];
        double2 a[K];
#pragma unroll
        for (int l = 0; l < K; ++l) a[l] = p2[l * ld2 + i];
#pragma unroll
        for (int l = 0; l < K; ++l) {
            b.x += nh[l] * a[l].x;
            b.y += nh[l] * a[l].y;
        }
        w2[i] = b;
        ww += b.x * b.x;
        ww += b.y * b.y;
    }
    for (long long i = 2 * n2 + q0; i < n; i += qs) {
        double b = w[i];
#pragma unroll
        for (int l = 0; l < K; ++l) b += nh[l] * v[l * ld + i];
        w[i] = b;
        ww += b * b;
    }
    __syncthreads();   // sm[0] is reused
    {
        const double t = warp_sum(ww);
        if (lane == 0) sm[0][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < VEC_THREADS / 32; ++q) t += sm[0][q];
        st_l2(&ws->partial[ROW2][blockIdx.x], t);
        __threadfence();
    }
    grid_barrier(&ws->bar[1]);
    if (warp == 0) {
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += ld_l2(&ws->partial[ROW2][b]);
        s = warp_sum(s);
        if (lane == 0) tot[NA] = s;
    }
    __syncthreads();
    const double w_sq = tot[NA];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) hout[i] = h[i];
        hout[K] = w_sq;
        ws->bar[0] = 0;   // every CTA is past the first barrier
    }

    // phase 3: vout = w / sqrt(<w, w>) (scale_kernel); a thread reads back what it stored itself
    const double sc = sqrt(w_sq);
    const bool alo = al && (((uintptr_t)vout & 15) == 0);
    double2 *o2 = reinterpret_cast<double2 *>(vout);
    for (long long q = q0; q < n2; q += qs) {
        const long long i = reverse_update ? n2 - 1 - q : q;
        const double2 b = w2[i];
        if (alo) {
            o2[i] = make_double2(b.x / sc, b.y / sc);
        } else {
            vout[2 * i] = b.x / sc;
            vout[2 * i + 1] = b.y / sc;
        }
    }
    for (long long i = 2 * n2 + q0; i < n; i += qs) vout[i] = w[i] / sc;

    // the last CTA to get here clears the second barrier and the exit ticket for the next launch
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(&ws->bar[2], 1u);
        if (t == gridDim.x - 1) {
            ws->bar[1] = 0;
            ws->bar[2] = 0;
        }
    }
}

// y = x / sqrt(<x, x>), *out = <x, x> in one cooperative launch: dot_kernel (its loop, block_sum and the order in
// which the last CTA adds the partials) + scale_kernel(take_sqrt) with one grid barrier in between -- the first two
// launches of an inner GMRES solve (krylov.py:226-232: beta = ||b||, v_0 = b / beta).  Same bits as the two launches.
__global__ void __launch_bounds__(VEC_THREADS, 4) norm_scale_small_kernel(long long n, const double *__restrict__ x,
                                                                          double *out, double *y, MgsWs *ws) {
    constexpr int ROW2 = MGS_NRED - 1;
    __shared__ double tot;
    double acc = 0.0;
    const bool al = aligned16(x, x);
    const long long n2 = al ? n >> 1 : 0;
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
    const long long q0 = (long long)blockIdx.x * VEC_THREADS + threadIdx.x, qs = (long long)gridDim.x * VEC_THREADS;
    for (long long q = q0; q < n2; q += qs) {
        const double2 a = x2[q];
        acc += a.x * a.x;
        acc += a.y * a.y;
    }
    for (long long i = 2 * n2 + q0; i < n; i += qs) acc += x[i] * x[i];
    const double part = block_sum(acc);
    if (threadIdx.x == 0) {
        st_l2(&ws->partial[ROW2][blockIdx.x], part);
        __threadfence();
    }
    grid_barrier(&ws->bar[1]);
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) s += ld_l2(&ws->partial[ROW2][b]);
        s = warp_sum(s);
        if (threadIdx.x == 0) tot = s;
    }
    __syncthreads();
    const double xx = tot;
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = xx;
    const double sc = sqrt(xx);
    for (long long i = q0; i < n; i += qs) y[i] = x[i] / sc;
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(&ws->bar[2], 1u);
        if (t == gridDim.x - 1) {
            ws->bar[1] = 0;
            ws->bar[2] = 0;
        }
    }
}

// all CTAs of `grid` resident at once?  (cooperative launches fail otherwise; asked once per instance)
template <int K>
static bool small_step_fits(int grid) {
    static int resident = -1;
    if (resident < 0) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgs_small_step_kernel<K>, VEC_THREADS, 0) != cudaSuccess)
            per_sm = 0;
        resident = per_sm * device_info().sm_count;
    }
    return grid <= resident;
}

template <int K>
static cudaError_t small_step_launch(int grid, cudaStream_t st, long long n, long long ld, const double *v, double *w,
                                     double *hout, double *vout, MgsWs *ws, int r1, int r2) {
    void *args[] = {&n, &ld, &v, &w, &hout, &vout, &ws, &r1, &r2};
    return cudaLaunchCooperativeKernel((const void *)mgs_small_step_kernel<K>, dim3(grid), dim3(VEC_THREADS), args, 0, st);
}

// y = x / s, y = x * s or y = copy, with s = *alpha_dev (optionally sqrt'ed) or alpha_host
// mode: 0 divide, 1 multiply
__global__ void __launch_bounds__(VEC_THREADS) scale_kernel(long long n, const double *__restrict__ x,
                                                            const double *alpha_dev, double alpha_host, int take_sqrt,
                                                            int mode, double *__restrict__ y) {
    double s = alpha_dev ? *alpha_dev : alpha_host;
    if (take_sqrt) s = sqrt(s);
    for (long long i = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS)
        y[i] = mode == 0 ? x[i] / s : x[i] * s;
}

// x += sum_i coef[i] * basis[i*ld + :], added in increasing i (same order as the
// reference's sequence of axpys: krylov.py:160-162, 264-267)
__global__ void __launch_bounds__(VEC_THREADS) multi_axpy_kernel(long long n, int k, const double *__restrict__ basis,
                                                                 long long ld, const double *__restrict__ coef,
                                                                 double *x, int overwrite) {
    extern __shared__ double c[];
    for (int i = threadIdx.x; i < k; i += VEC_THREADS) c[i] = coef[i];
    __syncthreads();
    for (long long e = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; e < n; e += (long long)gridDim.x * VEC_THREADS) {
        double s = overwrite ? 0.0 : x[e];
        for (int i = 0; i < k; ++i) s += c[i] * basis[i * ld + e];
        x[e] = s;
    }
}

// z = a op b elementwise: op 0: a + b, 1: a - b, 2: -a
__global__ void __launch_bounds__(VEC_THREADS) ewise_kernel(long long n, const double *a, const double *b, int op,
                                                            double *z) {
    for (long long i = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS)
        z[i] = op == 0 ? a[i] + b[i] : (op == 1 ? a[i] - b[i] : -a[i]);
}

__global__ void __launch_bounds__(VEC_THREADS) gather_kernel(long long n, const int *__restrict__ idx,
                                                             const double *__restrict__ src, double *__restrict__ dst) {
    for (long long i = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS)
        dst[i] = src[idx[i]];
}

__global__ void __launch_bounds__(VEC_THREADS) scatter_kernel(long long n, const int *__restrict__ idx,
                                                              const double *__restrict__ src, double *__restrict__ dst) {
    for (long long i = (long long)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_THREADS)
        dst[idx[i]] = src[i];
}

// The host arithmetic of `fixed_gmres` (krylov.py:233-268) for the few-step inner solve, on the device so that a
// preconditioner application needs no host read: Givens rotations on the Hessenberg columns, back substitution,
// coefficients of the basis combination.  H row j = [h_0j .. h_jj, |w_j|^2] (stride ldh), *bbp = <b, b>.
// Same operations in the same order as the host code (products rounded: -fmad=false; IEEE sqrt and division;
// hypot may differ from CPython's by an ulp).  Any early exit of the reference (zero right-hand side, happy
// breakdown before the last step) and any non-finite number raises *flag: the caller redoes the application step
// by step on the host path.
constexpr int SMALL_GMRES_MAX = 8;
__global__ void gmres_small_solve_kernel(int m, const double *__restrict__ H, int ldh, const double *__restrict__ bbp,
                                         double happy_tol, double *__restrict__ coef, int *flag) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double h[SMALL_GMRES_MAX + 1][SMALL_GMRES_MAX], cs[SMALL_GMRES_MAX], sn[SMALL_GMRES_MAX], g[SMALL_GMRES_MAX + 1],
        y[SMALL_GMRES_MAX];
    for (int i = 0; i <= m; ++i) {
        g[i] = 0.0;
        for (int j = 0; j < m; ++j) h[i][j] = 0.0;
    }
    for (int j = 0; j < m; ++j) coef[j] = 0.0;
    const double bb = *bbp;
    const double beta = sqrt(bb);
    bool bad = !(beta > 0.0) || !isfinite(beta);
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m && !bad; ++j) {
        const double *col = H + (long long)j * ldh;
        for (int i = 0; i <= j; ++i) h[i][j] = col[i];
        const double w2 = col[j + 1];
        const double hnext = w2 > 0.0 ? sqrt(w2) : 0.0;
        h[j + 1][j] = hnext;
        for (int i = 0; i < j; ++i) {                       // krylov.py:137-140
            const double t = cs[i] * h[i][j] + sn[i] * h[i + 1][j];
            h[i + 1][j] = -sn[i] * h[i][j] + cs[i] * h[i + 1][j];
            h[i][j] = t;
        }
        const double denom = hypot(h[j][j], hnext);         // krylov.py:141
        if (denom == 0.0) {
            cs[j] = 1.0;
            sn[j] = 0.0;
        } else {
            cs[j] = h[j][j] / denom;
            sn[j] = hnext / denom;
        }
        h[j][j] = cs[j] * h[j][j] + sn[j] * hnext;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        k = j + 1;
        if (!isfinite(w2) || !isfinite(h[j][j])) bad = true;
        if (hnext < happy_tol) {
            if (j + 1 < m) bad = true;                      // the queued steps behind a breakdown divided by ~0
            break;
        }
    }
    if (bad) {
        atomicExch(flag, 1);
        return;
    }
    for (int i = k - 1; i >= 0; --i) {                      // krylov.py:86-93
        double s = g[i];
        for (int j = i + 1; j < k; ++j) s -= h[i][j] * y[j];
        y[i] = h[i][i] != 0.0 ? s / h[i][i] : 0.0;
    }
    for (int i = 0; i < k; ++i) coef[i] = y[i];
}

static int red_grid(long long n) {
    int g = stream_grid(n, VEC_THREADS, 4, 4);
    return g > RED_MAX_BLOCKS ? RED_MAX_BLOCKS : g;
}

}  // namespace ddilu

using namespace ddilu;

extern "C" long long ddilu_reduce_ws_bytes(void) { return (long long)sizeof(RedWs); }

extern "C" int ddilu_dot(long long n, const double *x, const double *y, double *out, void *ws, void *stream) {
    dot_kernel<<<red_grid(n), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, x, y, (RedWs *)ws, out, 0);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* the same walking the vectors from the end when reverse != 0 (see ddilu_axpy_dot_dir) */
extern "C" int ddilu_dot_dir(long long n, const double *x, const double *y, double *out, void *ws, int reverse,
                             void *stream) {
    dot_kernel<<<red_grid(n), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, x, y, (RedWs *)ws, out, reverse);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

static int axpy_dot_launch(long long n, const double *alpha_dev, double alpha_host, const double *v, double *w,
                           const double *u, double *out, void *ws, int reverse, cudaStream_t st) {
    if (u) {
        if (!out || !ws) return DDILU_ERR_ARG;
        axpy_dot_kernel<true><<<red_grid(n), VEC_THREADS, 0, st>>>(n, alpha_dev, alpha_host, v, w, u, (RedWs *)ws, out,
                                                                  reverse);
    } else {
        if (n <= 0) return DDILU_OK;
        axpy_dot_kernel<false><<<stream_grid(n, VEC_THREADS, 4), VEC_THREADS, 0, st>>>(n, alpha_dev, alpha_host, v, w,
                                                                                       nullptr, nullptr, nullptr,
                                                                                       reverse);
    }
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_axpy_dot(long long n, const double *alpha_dev, double alpha_host, const double *v, double *w,
                              const double *u, double *out, void *ws, void *stream) {
    return axpy_dot_launch(n, alpha_dev, alpha_host, v, w, u, out, ws, 0, (cudaStream_t)stream);
}

/* the same, walking the vectors from the end when reverse != 0 (consecutive MGS steps alternate: the step
 * starts with what the previous one left in L2) */
extern "C" int ddilu_axpy_dot_dir(long long n, const double *alpha_dev, double alpha_host, const double *v, double *w,
                                  const double *u, double *out, void *ws, int reverse, void *stream) {
    return axpy_dot_launch(n, alpha_dev, alpha_host, v, w, u, out, ws, reverse, (cudaStream_t)stream);
}

extern "C" long long ddilu_mgs_ws_bytes(void) { return (long long)sizeof(MgsWs); }
extern "C" int ddilu_mgs_max_block(void) { return MGS_K; }

/* one pass of the blocked modified Gram-Schmidt (see mgs_block_kernel) */
extern "C" int ddilu_mgs_block(long long n, long long ld, int kp, const double *vprev, const double *raw_prev,
                               double *hout, double *w, int kn, const double *vnext, double *out, void *ws,
                               int reverse, void *stream) {
    if (kp < 0 || kp > MGS_K || kn < 0 || kn > MGS_K || !w || !out || !ws) return DDILU_ERR_ARG;
    if (kp > 0 && (!vprev || !raw_prev || !hout)) return DDILU_ERR_ARG;
    if (kn > 0 && !vnext) return DDILU_ERR_ARG;
    const int grid = red_grid(n);
    cudaStream_t st = (cudaStream_t)stream;
    MgsWs *m = (MgsWs *)ws;
    switch (kp) {
        case 0: mgs_launch_kn<0>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 1: mgs_launch_kn<1>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 2: mgs_launch_kn<2>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 3: mgs_launch_kn<3>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 4: mgs_launch_kn<4>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 5: mgs_launch_kn<5>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 6: mgs_launch_kn<6>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 7: mgs_launch_kn<7>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
        case 8: mgs_launch_kn<8>(kn, grid, st, n, ld, vprev, raw_prev, hout, w, vnext, m, out, reverse); break;
    }
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* One Arnoldi step of the inner GMRES (krylov.py:236-256) on a short vector in ONE cooperative launch: the k <=
 * ddilu_mgs_small_max() basis vectors v[0..k) (leading dimension ld), w orthogonalised in place,
 * hout[0..k) = the MGS coefficients, hout[k] = <w, w>, vout = w / sqrt(<w, w>).  Same bits as
 * ddilu_mgs_block(0, k) + ddilu_mgs_block(k, 0) + ddilu_scale (which it falls back to when the grid of the
 * reductions cannot be resident at once); raw = scratch of k + k(k-1)/2 doubles for that fallback. */
extern "C" int ddilu_scale(long long n, const double *x, const double *alpha_dev, double alpha_host, int take_sqrt,
                           int mode, double *y, void *stream);
extern "C" int ddilu_mgs_small_max(void) { return 4; }
extern "C" int ddilu_mgs_small_step(long long n, long long ld, int k, const double *v, double *w, double *hout,
                                    double *vout, double *raw, void *ws, int reverse_dots, int reverse_update,
                                    void *stream) {
    if (k < 1 || k > 4 || n <= 0 || !v || !w || !hout || !vout || !raw || !ws) return DDILU_ERR_ARG;
    const int grid = red_grid(n);
    cudaStream_t st = (cudaStream_t)stream;
    MgsWs *m = (MgsWs *)ws;
    bool fits = false;
    switch (k) {
        case 1: fits = small_step_fits<1>(grid); break;
        case 2: fits = small_step_fits<2>(grid); break;
        case 3: fits = small_step_fits<3>(grid); break;
        case 4: fits = small_step_fits<4>(grid); break;
    }
    if (!fits) {
        int rc = ddilu_mgs_block(n, ld, 0, nullptr, nullptr, nullptr, w, k, v, raw, ws, reverse_dots, stream);
        if (rc != DDILU_OK) return rc;
        rc = ddilu_mgs_block(n, ld, k, v, raw, hout, w, 0, nullptr, hout + k, ws, reverse_update, stream);
        if (rc != DDILU_OK) return rc;
        return ddilu_scale(n, w, hout + k, 0.0, 1, 0, vout, stream);
    }
    cudaError_t e = cudaSuccess;
    switch (k) {
        case 1: e = small_step_launch<1>(grid, st, n, ld, v, w, hout, vout, m, reverse_dots, reverse_update); break;
        case 2: e = small_step_launch<2>(grid, st, n, ld, v, w, hout, vout, m, reverse_dots, reverse_update); break;
        case 3: e = small_step_launch<3>(grid, st, n, ld, v, w, hout, vout, m, reverse_dots, reverse_update); break;
        case 4: e = small_step_launch<4>(grid, st, n, ld, v, w, hout, vout, m, reverse_dots, reverse_update); break;
    }
    DDILU_CHECK(e);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* krylov.py:226-232, the start of `fixed_gmres` on one rank: *out = <x, x>, y = x / sqrt(<x, x>) in ONE cooperative
 * launch (ddilu_dot + ddilu_scale(take_sqrt) with a grid barrier in between; same bits, falls back to the two
 * launches when the grid cannot be resident at once).  ws: the ddilu_mgs_block workspace, red_ws: ddilu_dot's. */
extern "C" int ddilu_norm_scale_small(long long n, const double *x, double *out, double *y, void *ws, void *red_ws,
                                      void *stream) {
    if (n <= 0 || !x || !out || !y || !ws || !red_ws) return DDILU_ERR_ARG;
    const int grid = red_grid(n);
    static int resident = -1;
    if (resident < 0) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, norm_scale_small_kernel, VEC_THREADS, 0) != cudaSuccess)
            per_sm = 0;
        resident = per_sm * device_info().sm_count;
    }
    if (grid > resident) {
        int rc = ddilu_dot(n, x, x, out, red_ws, stream);
        if (rc != DDILU_OK) return rc;
        return ddilu_scale(n, x, out, 0.0, 1, 0, y, stream);
    }
    MgsWs *m = (MgsWs *)ws;
    void *args[] = {&n, &x, &out, &y, &m};
    DDILU_CHECK(cudaLaunchCooperativeKernel((const void *)norm_scale_small_kernel, dim3(grid), dim3(VEC_THREADS), args, 0,
                                            (cudaStream_t)stream));
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_scale(long long n, const double *x, const double *alpha_dev, double alpha_host, int take_sqrt,
                           int mode, double *y, void *stream) {
    if (n <= 0) return DDILU_OK;
    scale_kernel<<<stream_grid(n, VEC_THREADS, 2), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, x, alpha_dev, alpha_host,
                                                                                          take_sqrt, mode, y);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_multi_axpy(long long n, int k, const double *basis, long long ld, const double *coef, double *x,
                                int overwrite, void *stream) {
    if (n <= 0 || k < 0) return DDILU_OK;
    multi_axpy_kernel<<<stream_grid(n, VEC_THREADS, 2), VEC_THREADS, sizeof(double) * (k > 0 ? k : 1),
                        (cudaStream_t)stream>>>(n, k, basis, ld, coef, x, overwrite);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_gmres_small_max(void) { return SMALL_GMRES_MAX; }

extern "C" int ddilu_gmres_small_solve(int m, const double *H, int ldh, const double *bb, double happy_tol,
                                       double *coef, int *flag, void *stream) {
    if (m < 1 || m > SMALL_GMRES_MAX || ldh < m + 2) return DDILU_ERR_ARG;
    gmres_small_solve_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m, H, ldh, bb, happy_tol, coef, flag);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_ewise(long long n, const double *a, const double *b, int op, double *z, void *stream) {
    if (n <= 0) return DDILU_OK;
    ewise_kernel<<<stream_grid(n, VEC_THREADS, 2), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, a, b, op, z);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_gather(long long n, const int *idx, const double *src, double *dst, void *stream) {
    if (n <= 0) return DDILU_OK;
    gather_kernel<<<stream_grid(n, VEC_THREADS, 2), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_scatter(long long n, const int *idx, const double *src, double *dst, void *stream) {
    if (n <= 0) return DDILU_OK;
    scatter_kernel<<<stream_grid(n, VEC_THREADS, 2), VEC_THREADS, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

/* L2 residency hint for the Arnoldi work vector w (no reference equivalent): every MGS step reads and writes
 * w while the basis vectors stream through once; with w pinned in the persisting part of L2 a step moves
 * 16n + (1 - hit) 16n bytes from HBM instead of 32n.  bytes = 0 clears the window and the persisting lines. */
extern "C" int ddilu_l2_persist_window(const void *ptr, long long bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, max_persist = 0, max_window = 0;
    DDILU_CHECK(cudaGetDevice(&dev));
    DDILU_CHECK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    DDILU_CHECK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    cudaStreamAttrValue attr;
    memset(&attr, 0, sizeof(attr));
    if (bytes <= 0 || !ptr || max_persist <= 0) {
        attr.accessPolicyWindow.num_bytes = 0;
        DDILU_CHECK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
        DDILU_CHECK(cudaCtxResetPersistingL2Cache());
        return DDILU_OK;
    }
    // leave a quarter of the allowed set-aside to everything else that wants L2
    const long long set_aside = (long long)max_persist * 3 / 4;
    DDILU_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)set_aside));
    const long long win = bytes < max_window ? bytes : max_window;
    double ratio = (double)set_aside / (double)win;
    if (ratio > 1.0) ratio = 1.0;
    attr.accessPolicyWindow.base_ptr = const_cast<void *>(ptr);
    attr.accessPolicyWindow.num_bytes = (size_t)win;
    attr.accessPolicyWindow.hitRatio = (float)ratio;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    DDILU_CHECK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
    return DDILU_OK;
}
