// Shared device/host helpers for libddilu_b200 (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DDILU_OK 0
#define DDILU_ERR_ARG (-1000)

// Every C-ABI entry returns 0 or -(cudaError_t); launch errors are picked up
// right after the launch (no device synchronisation inside the library).
#define DDILU_CHECK(expr)                                   \
    do {                                                    \
        cudaError_t e__ = (expr);                           \
        if (e__ != cudaSuccess) return -(int)e__;           \
    } while (0)
#define DDILU_LAUNCH_CHECK() DDILU_CHECK(cudaGetLastError())

namespace ddilu {

constexpr int kWarp = 32;

struct DeviceInfo {
    int sm_count;
    int max_threads_per_sm;
};

// one query per process; B200 = 148 SMs, 2048 threads/SM
inline const DeviceInfo &device_info() {
    static DeviceInfo info = [] {
        DeviceInfo d{148, 2048};
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) {
            cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&d.max_threads_per_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
        }
        return d;
    }();
    return info;
}

inline int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

// grid for a grid-stride streaming kernel: a whole number of waves
inline int stream_grid(long long n, int threads, int per_thread = 1, int waves = 8) {
    long long want = (n + (long long)threads * per_thread - 1) / ((long long)threads * per_thread);
    long long cap = (long long)device_info().sm_count * waves;
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

// ---- "value is the flag" sentinel used by the sync-free triangular solves:
// the all-ones bit pattern (a NaN no arithmetic produces; cudaMemset 0xFF).
__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == -1LL; }
__device__ __forceinline__ double scrub_sentinel(double v) {
    return is_sentinel(v) ? __longlong_as_double(0x7FF8000000000000LL) : v;
}

// L2-coherent accesses (bypass the non-coherent L1)
__device__ __forceinline__ double ld_l2(const double *p) {
    double v;
    asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_l2(double *p, double v) {
    asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// gpu-scope relaxed (coherent at L2, no system-scope semantics)
__device__ __forceinline__ double ld_gpu(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_gpu(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ int ld_l2(const int *p) {
    int v;
    asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_l2(int *p, int v) {
    asm volatile("st.volatile.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// s / d with the pivot's reciprocal r = RN(1/d) precomputed at setup: one multiply and two
// remainder/correction FMA pairs instead of the ~30-instruction division routine on every level's
// critical path.  q1 = RN(s r) is within 2 ulp of s/d, q2 is faithful, and by Markstein's theorem
// (r correctly rounded, the remainder s - d q2 exact) the last correction rounds exactly like the
// IEEE division, so the result has the bits of the reference's `s / d` (sparse.py:271).  Operands
// outside a safe exponent window (zero, subnormal, huge, inf/nan: the remainder would not be exact)
// and pivots flagged r = 0 at setup take the real division.  Verified bit-for-bit on random and
// adversarial operands by ddilu_fastdiv_selftest (tests/test_gpu_tiled.py).
// the rare real division, kept out of line: inlined, the compiler starts its reciprocal iteration (six dependent
// FMAs) speculatively on every call, in front of the corrections below
static __device__ __noinline__ double exact_div_slow(double s, double d) { return s / d; }

__device__ __forceinline__ double exact_div(double s, double d, double r) {
    // the corrections start at once; the operand check runs beside them and only a failing check branches
    // (the check-then-branch form put ~25 cycles in front of the five dependent operations on every level)
    const double q1 = s * r;
    const double e1 = __fma_rn(-d, q1, s);
    const double q2 = __fma_rn(e1, r, q1);
    const double e2 = __fma_rn(-d, q2, s);
    double q = __fma_rn(e2, r, q2);
    const unsigned es = ((unsigned)__double2hiint(s) >> 20) & 0x7ffu;
    const unsigned rh = (unsigned)__double2hiint(r) & 0x7fffffffu;   // r == +-0.0 <=> no exponent / mantissa bits
    const bool ok = ((rh | (unsigned)__double2loint(r)) != 0u) && (es - 623u <= 800u);
    if (!ok) q = exact_div_slow(s, d);
    return q;
}
// reciprocal to store for a pivot, 0 = "always divide" (pivot outside the safe exponent window)
__device__ __forceinline__ double safe_reciprocal(double d) {
    const unsigned ed = ((unsigned)__double2hiint(d) >> 20) & 0x7ffu;
    return (ed - 623u <= 800u) ? 1.0 / d : 0.0;
}

}  // namespace ddilu
