// Measures the store->poll latency through L2 between SMs: a chain of CTAs,
// each waits for its predecessor's value and publishes its own.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double ld_l2(const double *p) { double v; asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_l2(double *p, double v) { asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }
__global__ void chain(double *x, int links, int stride) {
    // CTA c handles links c, c+G, ...; link i waits on x[(i-1)*stride]
    for (int i = blockIdx.x; i < links; i += gridDim.x) {
        if (threadIdx.x == 0) {
            double v = 1.0;
            if (i > 0) { do { v = ld_l2(x + (size_t)(i - 1) * stride); } while (__double_as_longlong(v) == -1LL); }
            st_l2(x + (size_t)i * stride, v + 1.0);
        }
    }
}
int main() {
    int links = 20000;
    for (int stride : {1, 16, 1024}) {
        double *x; cudaMalloc(&x, sizeof(double) * (size_t)links * stride);
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(x, 0xFF, sizeof(double) * (size_t)links * stride);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            void *args[] = {&x, &links, &stride};
            cudaLaunchCooperativeKernel((void *)chain, 148, 32, args, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("stride %d: %d links in %.3f ms -> %.1f ns per hop (%s)\n", stride, links, ms, ms * 1e6 / links, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(x);
    }
    return 0;
}
