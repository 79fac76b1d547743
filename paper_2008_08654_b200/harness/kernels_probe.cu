// kernels_probe.cu -- microbenchmarks that measure the roofline denominators
// this path needs and MEASURED_PEAKS.json does not carry ("measured
// peak IMAD.WIDE.U32 rate ... microbenchmark it on the same box"), plus the
// atomic throughputs that decide the Count Sketch privatisation strategy.
#include <cooperative_groups.h>

#include "../csrc/mb200_device.cuh"
#include "harness_internal.h"
#include "../csrc/mb200_mem.cuh"

namespace mb200 {

namespace {

constexpr int kChains = 8;

// kChains independent IMAD.WIDE.U32 chains per thread: acc = hi32(acc) * b.
// The next multiplicand is the product's own high word, so the products
// cannot be hoisted, and there is no accumulate: a mad.wide with a register
// addend is split by ptxas into IMAD.WIDE + IADD3/IADD3.X, and with
// loop-invariant operands the product is hoisted and only the 64-bit add is
// left (the round-1/2 form of this probe up to r02e measured that add rate,
// 1.72e13/s).  The SASS of this loop is IMAD.WIDE.U32 only.
__global__ void probe_imad_kernel(int iters, u64* sink) {
    u64 acc[kChains];
    const u32 b = blockIdx.x * 2654435761u + 12345u;
#pragma unroll
    for (int j = 0; j < kChains; ++j) acc[j] = threadIdx.x * 0x9E3779B97F4A7C15ull + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile("{\n\t.reg .u32 l, h;\n\tmov.b64 {l, h}, %0;\n\tmul.wide.u32 %0, h, %1;\n\t}"
                         : "+l"(acc[j])
                         : "r"(b));
    }
    u64 s = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s ^= acc[j];
    if (s == 0x123456789ull) sink[0] = s;
}

__device__ __forceinline__ u32 scramble(u32 x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// mode 0: shared red.u64 on random cells of a 4096-entry table
// mode 1: shared red.u32 on random cells
// mode 2: global red.u64 on random cells of [0, span)
// mode 3: global red.u64, every thread the same cell (worst-case hot key)
// mode 4: global red.u64, warp-aggregated hot cell (one red per warp)
__global__ void probe_atomics_kernel(int mode, int iters, u64* buf, u64 span) {
    __shared__ unsigned long long t64[4096];
    __shared__ unsigned t32[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        t64[i] = 0;
        t32[i] = 0;
    }
    __syncthreads();
    u32 h = scramble(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        h = scramble(h + i);
        switch (mode) {
            case 0: atomicAdd(&t64[h & 4095], 1ull); break;
            case 1: atomicAdd(&t32[h & 4095], 1u); break;
            case 2: red_add_u64(buf + (h % span), 1); break;
            case 3: red_add_u64(buf, 1); break;
            case 5: {  // global red.u32 on random cells
                unsigned* b32 = reinterpret_cast<unsigned*>(buf);
                asm volatile("red.global.add.u32 [%0], %1;" ::"l"(b32 + (h % span)), "r"(1u) : "memory");
                break;
            }
            case 6: atomicCAS(&t32[h & 4095], 0u, h); break;  // shared CAS, random cells
            case 7: {  // shared u64 atomic on 2 u32 halves (carry via returned old value)
                const unsigned old = atomicAdd(&t32[h & 4095], 1u);
                if (old == 0xffffffffu) atomicAdd(&t32[(h + 1) & 4095], 1u);
                break;
            }
            default:
                if ((threadIdx.x & 31) == 0) red_add_u64(buf, 32);
                break;
        }
    }
    __syncthreads();
    if (mode <= 1 && threadIdx.x == 0) buf[blockIdx.x % span] += t64[0] + t32[0];
}

// Distributed-shared-memory reductions inside a cluster of CS CTAs, each CTA
// owning `words` u32 counters: mode 0 random (rank, cell) -- (CS-1)/CS remote;
// mode 1 random cell of the own CTA; mode 2 one hot cell in rank 0.
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) probe_dsmem_kernel(int mode, int iters, u32 words, u64* out) {
    extern __shared__ u32 tab[];
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    for (u32 i = threadIdx.x; i < words; i += blockDim.x) tab[i] = 0;
    cl.sync();
    u32 h = scramble(blockIdx.x * blockDim.x + threadIdx.x);
    const u32 me = cl.block_rank();
    for (int i = 0; i < iters; ++i) {
        h = scramble(h + i);
        u32 rank = mode == 0 ? (h >> 24) % CS : (mode == 1 ? me : 0);
        u32 off = mode == 2 ? 0 : (h & 0xFFFFFF) % words;
        u32* remote = cl.map_shared_rank(tab, rank);
        atomicAdd(remote + off, 1u);
    }
    cl.sync();
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)tab[0]);
}

}  // namespace

cudaError_t launch_probe_dsmem(int cluster, int mode, int blocks, int threads, int iters, uint32_t words,
                               uint64_t* out, cudaStream_t s) {
    const size_t smem = (size_t)words * 4;
    cudaError_t e = cudaSuccess;
    switch (cluster) {
#define MB200_DS(CS)                                                                                    \
    case CS:                                                                                            \
        e = cudaFuncSetAttribute(probe_dsmem_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem);                                                           \
        if (e != cudaSuccess) return e;                                                                \
        probe_dsmem_kernel<CS><<<blocks, threads, smem, s>>>(mode, iters, words, out);                 \
        break;
        MB200_DS(1)
        MB200_DS(2)
        MB200_DS(4)
        MB200_DS(8)
#undef MB200_DS
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_probe_imad(int blocks, int threads, int iters, uint64_t* sink, cudaStream_t s) {
    probe_imad_kernel<<<blocks, threads, 0, s>>>(iters, sink);
    return cudaGetLastError();
}

cudaError_t launch_probe_atomics(int mode, int blocks, int threads, int iters, uint64_t* buf, uint64_t span,
                                 cudaStream_t s) {
    probe_atomics_kernel<<<blocks, threads, 0, s>>>(mode, iters, buf, span ? span : 1);
    return cudaGetLastError();
}

}  // namespace mb200
