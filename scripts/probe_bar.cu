// Hand-over cost of the block sweep's level protocol (csrc/sweep.cu) in isolation, one CTA on a B200:
// NS sets of W warps take "levels" in turn -- bar.sync on the predecessor's barrier, a shared-memory store/load
// chain, bar.arrive on the set's own barrier.  Prints cycles per level for W = 1..12 and NS = 2, 3, with the
// barrier id / count as immediates or registers, with and without helper warps that spin (mbarrier try_wait,
// volatile shared-memory polls with nanosleep) the way the kernel's issuer / gate / writers do.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_bar probe_bar.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool SPIN>
__global__ void probe(int NS, int W, int levels, int work, long long *cyc, double *sink) {
    __shared__ double xs[2048];
    __shared__ unsigned long long mbar;
    __shared__ int flag;
    const int tid = threadIdx.x, nct = 32 * W, ncomp = NS * nct;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
        flag = 0;
    }
    for (int i = tid; i < 2048; i += blockDim.x) xs[i] = 1.0 + i;
    __syncthreads();
    if (tid < ncomp) {
        const int set = tid / nct, t = tid - set * nct;
        const int bar_out = 1 + set, bar_in = 1 + (set == 0 ? NS - 1 : set - 1), pair = 2 * nct;
        long long t0 = clock64();
        double acc = 0.0;
        for (int l = set; l < levels; l += NS) {
            if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(bar_in), "r"(pair) : "memory");
            if (work) {
                double v = xs[(t + 37 * l) & 2047];
                v = v * 1.0000001 - 0.5;
                xs[(t + 37 * (l + 1) + 1) & 2047] = v;
                acc += v;
            }
            if (l + 1 < levels) asm volatile("bar.arrive %0, %1;" ::"r"(bar_out), "r"(pair) : "memory");
        }
        asm volatile("bar.sync 8, %0;" ::"r"(ncomp) : "memory");
        if (tid == 0) cyc[0] = clock64() - t0;
        if (acc == 12345.678) sink[0] = acc;
        if (tid == 0) {
            asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_u32(&flag)), "r"(1) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mbar)) : "memory");
        }
    } else if (SPIN) {
        const int h = (tid - ncomp) >> 5;
        if (h < 2) {          // issuer / gate: one lane spins on an mbarrier
            if ((tid & 31) == 0) {
                uint32_t done;
                do {
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                        : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0) : "memory");
                } while (!done);
            }
        } else {              // writers: poll a shared-memory word with nanosleep
            int v;
            do {
                asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&flag)) : "memory");
                if (!v) __nanosleep(20);
            } while (!v);
        }
    }
}

int main() {
    long long *cyc;
    double *sink;
    cudaMalloc(&cyc, 64);
    cudaMalloc(&sink, 64);
    const int levels = 4096;
    for (int spin = 0; spin < 2; ++spin)
        for (int work = 0; work < 2; ++work)
            for (int NS = 2; NS <= 3; ++NS)
                for (int W : {1, 2, 3, 4, 6, 8, 12}) {
                    const int threads = NS * W * 32 + (spin ? 8 * 32 : 0);
                    if (threads > 1024) continue;
                    for (int rep = 0; rep < 2; ++rep) {
                        if (spin) probe<true><<<1, threads>>>(NS, W, levels, work, cyc, sink);
                        else probe<false><<<1, threads>>>(NS, W, levels, work, cyc, sink);
                        cudaDeviceSynchronize();
                    }
                    long long c = 0;
                    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                    printf("{\"spin_helpers\": %d, \"work\": %d, \"sets\": %d, \"warps_per_set\": %d, \"cycles_per_level\": %.1f}\n",
                           spin, work, NS, W, (double)c / levels);
                }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
