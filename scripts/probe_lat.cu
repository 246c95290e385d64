// Latency probes for the per-level critical path of the tiled SpTRSV (one CTA, B200):
// dependent fp64 mul/sub chain, fp64 division, shared-memory load chain, named barrier,
// warp-to-warp handoff through bar.arrive / bar.sync, volatile global store issue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o probe_lat probe_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double *out, long long *cyc, double seed, double *g) {
    __shared__ double sm[1024];
    __shared__ int chase[1024];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) {
        sm[i] = seed + i;
        chase[i] = (i * 37 + 11) & 1023;
    }
    __syncthreads();
    const int N = 256;
    long long t0, t1;
    double s = seed, a = 1.0000001;
    // (0) dependent DMUL + DADD pairs
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) s -= a * s;
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / N;
    // (1) dependent DADD
    double s1 = s;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) s1 = s1 - a;
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[1] = (t1 - t0) / N;
    // (2) dependent division
    double s2 = s1 + 3.0;
    t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N; ++i) s2 = (s2 + 1.5) / a;
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[2] = (t1 - t0) / N;
    // (3) shared-memory pointer chase
    int p = lane;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) p = chase[p];
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[3] = (t1 - t0) / N;
    // (4) named barrier, all warps
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[4] = (t1 - t0) / N;
    // (5) ring handoff: warp w waits for warp w-1 (bar ids 1..4), does one sts, passes on
    __syncthreads();
    const int nw = blockDim.x >> 5;
    t0 = clock64();
    for (int i = 0; i < N && nw > 1; ++i) {
        // level l = i*nw + warp is "owned" by this warp
        const int l = i * nw + warp;
        if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((l - 1) % nw)), "r"(64) : "memory");
        sm[lane] = s2 + l;
        asm volatile("bar.arrive %0, %1;" ::"r"(8 + (l % nw)), "r"(64) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[5] = (t1 - t0) / (N * nw);   // per handoff
    if (nw > 1 && warp == 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((N * nw - 1) % nw)), "r"(64) : "memory");
    __syncthreads();
    // (6) volatile global store + barrier per iteration
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(g + tid), "d"(s2) : "memory");
        asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[6] = (t1 - t0) / N;
    // (7) sts -> bar -> dependent lds of another thread's value -> dmul/dadd x3 -> sts  (one "level")
    double v = s2;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        sm[tid] = v;
        asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
        const double x0 = sm[(tid + 1) & 127], x1 = sm[(tid + 5) & 127], x2 = sm[(tid + 9) & 127];
        v = v - a * x0;
        v = v - a * x1;
        v = v - a * x2;
        asm volatile("bar.sync 2, %0;" ::"r"((int)blockDim.x) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[7] = (t1 - t0) / N;
    // (8) like (6) but every store goes to a fresh line
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(g + tid + 128 * i), "d"(s2) : "memory");
        asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[8] = (t1 - t0) / N;
    // (9) ring handoff with a level's work: sync, 3 lds, 3 mul/sub, sts, volatile global store (fresh line), arrive
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N && nw > 1; ++i) {
        const int l = i * nw + warp;
        if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((l - 1) % nw)), "r"(64) : "memory");
        const double x0 = sm[(lane + 1) & 31], x1 = sm[(lane + 5) & 31], x2 = sm[(lane + 9) & 31];
        v = v - a * x0;
        v = v - a * x1;
        v = v - a * x2;
        sm[lane] = v;
        asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(g + lane + 32 * (l & 1023)), "d"(v) : "memory");
        asm volatile("bar.arrive %0, %1;" ::"r"(8 + (l % nw)), "r"(64) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[9] = (t1 - t0) / (N * nw);
    // (10) the same with a plain (weak) global store
    if (nw > 1 && warp == 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((N * nw - 1) % nw)), "r"(64) : "memory");
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N && nw > 1; ++i) {
        const int l = i * nw + warp;
        if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((l - 1) % nw)), "r"(64) : "memory");
        const double x0 = sm[(lane + 1) & 31], x1 = sm[(lane + 5) & 31], x2 = sm[(lane + 9) & 31];
        v = v - a * x0;
        v = v - a * x1;
        v = v - a * x2;
        sm[lane] = v;
        g[lane + 32 * (l & 1023)] = v;
        asm volatile("bar.arrive %0, %1;" ::"r"(8 + (l % nw)), "r"(64) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[10] = (t1 - t0) / (N * nw);
    // (11) without any global store
    if (nw > 1 && warp == 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((N * nw - 1) % nw)), "r"(64) : "memory");
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N && nw > 1; ++i) {
        const int l = i * nw + warp;
        if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((l - 1) % nw)), "r"(64) : "memory");
        const double x0 = sm[(lane + 1) & 31], x1 = sm[(lane + 5) & 31], x2 = sm[(lane + 9) & 31];
        v = v - a * x0;
        v = v - a * x1;
        v = v - a * x2;
        sm[lane] = v;
        asm volatile("bar.arrive %0, %1;" ::"r"(8 + (l % nw)), "r"(64) : "memory");
    }
    t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) cyc[11] = (t1 - t0) / (N * nw);
    if (nw > 1 && warp == 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((N * nw - 1) % nw)), "r"(64) : "memory");
    // (12) the tiled kernel's protocol: every barrier B_l gets all 4 warps; the owner of level l syncs on
    // B_{l-1}, works, then arrives at B_l, B_{l+1}, B_{l+2}
    __syncthreads();
    if (nw == 4) {
        t0 = clock64();
        for (int i = 0; i < N; ++i) {
            const int l = i * 4 + warp;
            if (i == 0) {
                for (int q = 0; q <= l - 2; ++q) asm volatile("bar.arrive %0, %1;" ::"r"(8 + (q & 3)), "r"(128) : "memory");
            }
            if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(8 + ((l - 1) & 3)), "r"(128) : "memory");
            const double x0 = sm[(lane + 1) & 31], x1 = sm[(lane + 5) & 31], x2 = sm[(lane + 9) & 31];
            v = v - a * x0;
            v = v - a * x1;
            v = v - a * x2;
            sm[lane] = v;
            asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(g + lane + 32 * (l & 1023)), "d"(v) : "memory");
            const int last = (i == N - 1) ? N * 4 - 1 : l + 2;
            for (int q = l; q <= last; ++q) asm volatile("bar.arrive %0, %1;" ::"r"(8 + (q & 3)), "r"(128) : "memory");
        }
        t1 = clock64();
        if (tid == 0 && blockIdx.x == 0) cyc[12] = (t1 - t0) / (N * 4);
    }
    __syncthreads();
    out[tid] = s + s1 + s2 + p + v;
}

int main() {
    double *out, *g;
    long long *cyc, h[13];
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&g, 1024 * 8 * 64);
    cudaMalloc(&cyc, 104);
    const char *names[13] = {"dmul+dadd pair", "dadd", "ddiv(+dadd)", "lds chase", "bar.sync all warps",
                             "ring handoff arrive->sync", "st.volatile + bar", "level: sts,bar,3 lds,3 mul/sub,bar",
                             "st.volatile fresh line + bar", "ring level + st.volatile", "ring level + weak st",
                             "ring level, no global st", "4-warp protocol level"};
    const int grids[3] = {1, 148 * 4, 148 * 8};
    for (int gi = 0; gi < 3; ++gi)
    for (int threads = 32; threads <= 128; threads *= 2) {
        if (gi > 0 && threads != 128) continue;
        printf("grid %d\n", grids[gi]);
        probe<<<grids[gi], threads>>>(out, cyc, 1.25, g);
        probe<<<grids[gi], threads>>>(out, cyc, 1.25, g);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("kernel failed: %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, 104, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 13; ++i) printf("threads %3d  %-40s %lld cycles\n", threads, names[i], h[i]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
