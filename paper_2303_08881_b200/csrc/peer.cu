// Node-local exchanges over PEER MEMORY (NVLink / NVSwitch P2P stores, CUDA IPC mappings) instead of NCCL
// collectives -- the two exchanges of the multi-GPU path (halo of interface values
// before a product, sum of dot / norm scalars):
//
//   * every rank owns a MAILBOX in its own HBM that all ranks of the node map (paper_2303_08881_b200/dist.py
//     PeerComm): reduction slots red[2][size][kmax], halo buffers data[2][size][cap], and 64-bit sequence flags;
//   * a producer writes straight into the consumer's mailbox (remote stores), fences (system scope) and publishes a
//     sequence number with st.release.sys; the consumer's kernel polls its OWN memory (ld.acquire.sys) -- no
//     collective library call, no host synchronisation, one launch per reduction, two per halo exchange (send /
//     receive, so that the interior rows of the SpMV run in between);
//   * the scalar reduction sums the ranks' partials in RANK ORDER on every rank: bitwise the same result everywhere,
//     independent of the transport's algorithm;
//   * buffers alternate with the parity of the sequence number; a rank cannot be two exchanges ahead of a peer
//     (the next reduction needs that peer's partial), halo buffers are additionally acknowledged.
//
// Every wait is bounded (spin_cycles): a peer that never arrives sets *err instead of hanging the GPU.
#include <stdint.h>

#include "common.cuh"
#include "ddilu_b200.h"

namespace ddilu {

__device__ __forceinline__ long long peer_ld_acquire(const long long *p) {
    long long v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void peer_st_release(long long *p, long long v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double peer_ld_l2(const double *p) {      // written by a peer: not through this SM's L1
    double v;
    asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
// poll *flag until it reaches seq; false (and *err = code) when spin_cycles pass first
__device__ __forceinline__ bool peer_wait(const long long *flag, long long seq, long long spin_cycles, int *err, int code) {
    const long long t0 = clock64();
    while (peer_ld_acquire(flag) < seq) {
        if (clock64() - t0 > spin_cycles) {
            atomicExch(err, code);
            return false;
        }
        __nanosleep(64);
    }
    return true;
}

// out[i] = sum over ranks r (in rank order) of partial_r[i], i < k.  slots[r] / flags[r]: rank r's reduction slots
// red[2][size][kmax] and its flag array red_seq[size] as mapped in THIS process.  One CTA.
__global__ void peer_allreduce_kernel(int k, int kmax, const double *__restrict__ partial, double *out,
                                      const unsigned long long *__restrict__ slots,
                                      const unsigned long long *__restrict__ flags, int rank, int size, long long seq,
                                      long long spin_cycles, int *err) {
    const int buf = (int)(seq & 1);
    for (int idx = threadIdx.x; idx < size * k; idx += blockDim.x) {
        const int r = idx / k, i = idx - r * k;
        ((double *)slots[r])[((size_t)buf * size + rank) * kmax + i] = partial[i];
    }
    __threadfence_system();
    __syncthreads();
    if ((int)threadIdx.x < size) {
        peer_st_release((long long *)flags[threadIdx.x] + rank, seq);                     // my partial is in your slots
        peer_wait((const long long *)flags[rank] + threadIdx.x, seq, spin_cycles, err, 1);   // yours is in mine
    }
    __syncthreads();
    const double *mine = (const double *)slots[rank] + (size_t)buf * size * kmax;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < size; ++r) s += peer_ld_l2(mine + (size_t)r * kmax + i);
        out[i] = s;
    }
}

// value j of the message = send[j], or send[idx[j]] when idx is given (the pack of the interface values fused into
// the send).  Values off[d] .. off[d + 1] -> rank d's halo buffer data[buf][rank][0 ..), then data_seq_d[rank] = seq.
// ack[d]: my flag that rank d raises when it has consumed a message (seq - 2 used the same buffer).
__global__ void peer_send_kernel(int size, int rank, const double *__restrict__ send, const int *__restrict__ idx,
                                 const int *__restrict__ off,
                                 const unsigned long long *__restrict__ data, const unsigned long long *__restrict__ flags,
                                 const long long *ack, long long cap, long long seq, long long spin_cycles,
                                 unsigned int *counter, int *err) {
    __shared__ int ok;
    if (threadIdx.x == 0) ok = 1;
    __syncthreads();
    if ((int)threadIdx.x < size && (int)threadIdx.x != rank && off[threadIdx.x + 1] > off[threadIdx.x] && seq > 2)
        if (!peer_wait(ack + threadIdx.x, seq - 2, spin_cycles, err, 2)) ok = 0;
    __syncthreads();
    const int buf = (int)(seq & 1);
    if (ok) {
        const int total = off[size];
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += gridDim.x * blockDim.x) {
            int d = 0;
            while (off[d + 1] <= j) ++d;          // a handful of ranks
            if (d == rank) continue;
            ((double *)data[d])[((size_t)buf * size + rank) * cap + (j - off[d])] = send[idx ? idx[j] : j];
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(counter, 1u);
        if (done == gridDim.x - 1) {              // the last CTA publishes
            *counter = 0;
            __threadfence_system();
            for (int d = 0; d < size; ++d)
                if (d != rank && off[d + 1] > off[d]) peer_st_release((long long *)flags[d] + rank, seq);
        }
    }
}

// recv[off[s] .. off[s + 1]) <- my halo buffer data[buf][s][0 ..) once data_seq[s] >= seq; then rank s's ack[rank] = seq
__global__ void peer_recv_kernel(int size, int rank, double *__restrict__ recv, const int *__restrict__ off,
                                 const double *__restrict__ mydata, const long long *myflags,
                                 const unsigned long long *__restrict__ acks, const double *__restrict__ self_send,
                                 const int *__restrict__ self_idx, int self_off, long long cap, long long seq,
                                 long long spin_cycles, unsigned int *counter, int *err) {
    __shared__ int ok;
    if (threadIdx.x == 0) ok = 1;
    __syncthreads();
    if ((int)threadIdx.x < size && (int)threadIdx.x != rank && off[threadIdx.x + 1] > off[threadIdx.x])
        if (!peer_wait(myflags + threadIdx.x, seq, spin_cycles, err, 3)) ok = 0;
    __syncthreads();
    const int buf = (int)(seq & 1);
    if (ok) {
        const int total = off[size];
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += gridDim.x * blockDim.x) {
            int s = 0;
            while (off[s + 1] <= j) ++s;
            const int q = self_off + (j - off[s]);
            recv[j] = s == rank ? self_send[self_idx ? self_idx[q] : q]
                                : peer_ld_l2(mydata + ((size_t)buf * size + s) * cap + (j - off[s]));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(counter, 1u);
        if (done == gridDim.x - 1) {
            *counter = 0;
            __threadfence_system();
            for (int s = 0; s < size; ++s)
                if (s != rank && off[s + 1] > off[s]) peer_st_release((long long *)acks[s] + rank, seq);
        }
    }
}

}  // namespace ddilu

using namespace ddilu;

#define ST(s) ((cudaStream_t)(s))

extern "C" int ddilu_peer_allreduce(int k, int kmax, const double *partial, double *out,
                                    const unsigned long long *slots, const unsigned long long *flags, int rank,
                                    int size, long long seq, long long spin_cycles, int *err, void *stream) {
    if (k <= 0) return DDILU_OK;
    if (k > kmax || size < 1 || size > 64 || rank < 0 || rank >= size) return DDILU_ERR_ARG;
    peer_allreduce_kernel<<<1, 256, 0, ST(stream)>>>(k, kmax, partial, out, slots, flags, rank, size, seq, spin_cycles, err);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_peer_send(int size, int rank, int total, const double *send, const int *idx, const int *off,
                               const unsigned long long *data, const unsigned long long *flags, const long long *ack,
                               long long cap, long long seq, long long spin_cycles, unsigned int *counter, int *err,
                               void *stream) {
    if (size < 1 || size > 64 || rank < 0 || rank >= size) return DDILU_ERR_ARG;
    const int threads = 256;
    int grid = div_up(total > 0 ? total : 1, threads * 4);
    if (grid > 64) grid = 64;
    peer_send_kernel<<<grid, threads, 0, ST(stream)>>>(size, rank, send, idx, off, data, flags, ack, cap, seq,
                                                       spin_cycles, counter, err);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}

extern "C" int ddilu_peer_recv(int size, int rank, int total, double *recv, const int *off, const double *mydata,
                               const long long *myflags, const unsigned long long *acks, const double *self_send,
                               const int *self_idx, int self_off, long long cap, long long seq, long long spin_cycles,
                               unsigned int *counter, int *err, void *stream) {
    if (size < 1 || size > 64 || rank < 0 || rank >= size) return DDILU_ERR_ARG;
    const int threads = 256;
    int grid = div_up(total > 0 ? total : 1, threads * 4);
    if (grid > 64) grid = 64;
    peer_recv_kernel<<<grid, threads, 0, ST(stream)>>>(size, rank, recv, off, mydata, myflags, acks, self_send, self_idx,
                                                       self_off, cap, seq, spin_cycles, counter, err);
    DDILU_LAUNCH_CHECK();
    return DDILU_OK;
}
