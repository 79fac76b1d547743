// kernels_gen.cu -- synthetic workload generators (bench harness, not the hot
// path).  Every stream is counter-addressable SplitMix64 (prng.hpp:10-38:
// the i-th next() of SplitMix64(seed) is mix(seed + (i+1) golden)), so any
// shard [start, start+n) of a stream can be generated independently on any
// rank and is bit-identical to the sequential stream.  Streams follow the
// reference benchmark's convention of salting the seed for keys
// (bench.cpp:23, kKeyStreamSalt).  DESIGN.md "Inputs" defines each stream.
#include "../csrc/mb200_device.cuh"
#include "harness_internal.h"

namespace mb200 {

namespace {

constexpr int kThreads = 256;
constexpr u64 kSaltTail = 0x9E6C63D0676A9A99ull;
constexpr u64 kSaltW = 0xD1B54A32D192ED03ull;
constexpr u64 kSaltPerm = 0x2545F4914F6CDD1Dull;
constexpr u64 kSaltKeys = 0x7b5bad595e238e31ull;

int grid_for(uint64_t n) {
    const uint64_t need = (n + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sm_count() * 16;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

__global__ void gen_u32_kernel(u64 seed, uint64_t start, uint64_t n, u32* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (u32)splitmix_at(seed, start + i);
}

__global__ void gen_u64_kernel(u64 seed, uint64_t start, uint64_t n, u64* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = splitmix_at(seed, start + i);
}

// SplitMix64::below(2^61 - 1): shift = 3, reject v == p (prng.hpp:22-34)
__global__ void gen_below_p61_kernel(u64 seed, uint64_t start, uint64_t n, u64* out, unsigned long long* bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned nb = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 v = splitmix_at(seed, start + i) >> 3;
        nb += (v >= kP61);
        out[i] = v;
    }
    if (nb) atomicAdd(bad, (unsigned long long)nb);
}

// u128 uniform in [0, p^2), p = 2^64 - c: hi = next_{2i}, lo = next_{2i+1}
__global__ void gen_pm_kernel(u64 seed, u64 c, uint64_t start, uint64_t n, u64* out, unsigned long long* bad) {
    // p^2 = 2^128 - 2c 2^64 + c^2
    const u64 sq_lo = c * c;
    const u64 sq_hi = (0ull - 2 * c) + __umul64hi(c, c);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned nb = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 hi = splitmix_at(seed, 2 * (start + i));
        const u64 lo = splitmix_at(seed, 2 * (start + i) + 1);
        nb += (hi > sq_hi) || (hi == sq_hi && lo >= sq_lo);
        out[2 * i] = lo;
        out[2 * i + 1] = hi;
    }
    if (nb) atomicAdd(bad, (unsigned long long)nb);
}

__device__ __forceinline__ u32 feistel32(u64 key, u32 x) {
    u32 L = x >> 16, R = x & 0xFFFF;
#pragma unroll
    for (u32 round = 0; round < 4; ++round) {
        const u32 F = (u32)(mix64(key ^ (((u64)round << 16) | R)) >> 48);
        const u32 nl = R;
        R = (L ^ F) & 0xFFFF;
        L = nl;
    }
    return (L << 16) | R;
}

// Zipf(1.2) over [1, universe]: exact-CDF head (ranks 1..T, table computed on
// the host) + continuous Pareto tail with only correctly rounded IEEE
// operations (__d*_rn, no FMA contraction) so it is bit-reproducible on CPU.
__global__ void gen_zipf_kernel(u64 master, const u64* __restrict__ cdf, u32 T, double c1, double universe,
                                uint64_t start, uint64_t n, u32* keys, i32* weights) {
    const u64 sk = master ^ kSaltKeys, st = sk ^ kSaltTail, sw = sk ^ kSaltW, spm = master ^ kSaltPerm;
    const u64 head_total = cdf[T - 1];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t gi = start + i;
        const u64 u = splitmix_at(sk, gi);
        u64 rank;
        if (u < head_total) {
            u32 lo = 0, hi = T - 1;
            while (lo < hi) {
                const u32 mid = (lo + hi) >> 1;
                if (cdf[mid] > u) hi = mid;
                else lo = mid + 1;
            }
            rank = (u64)lo + 1;
        } else {
            const u64 v = splitmix_at(st, gi);
            const double w = __dmul_rn((double)(v >> 11), 0x1p-53);
            const double s = __dsub_rn(1.0, __dmul_rn(w, c1));
            const double s2 = __dmul_rn(s, s);
            const double s4 = __dmul_rn(s2, s2);
            const double s5 = __dmul_rn(s4, s);
            const double xr = __ddiv_rn(__dadd_rn((double)T, 0.5), s5);
            double xf = __dadd_rn(xr, 0.5);
            if (xf > universe) xf = universe;
            rank = __double2ull_rz(xf);
            if (rank < (u64)T + 1) rank = (u64)T + 1;
        }
        keys[i] = feistel32(spm, (u32)(rank - 1));
        if (weights) {
            const u64 z = splitmix_at(sw, gi);
            weights[i] = (i32)(((z >> 32) * 201ull) >> 32) - 100;
        }
    }
}

}  // namespace

cudaError_t launch_gen_u32(uint64_t seed, uint64_t start, uint64_t n, uint32_t* out, cudaStream_t s) {
    if (!n) return cudaSuccess;
    gen_u32_kernel<<<grid_for(n), kThreads, 0, s>>>(seed, start, n, out);
    return cudaGetLastError();
}
cudaError_t launch_gen_u64(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out, cudaStream_t s) {
    if (!n) return cudaSuccess;
    gen_u64_kernel<<<grid_for(n), kThreads, 0, s>>>(seed, start, n, out);
    return cudaGetLastError();
}
cudaError_t launch_gen_below_p61(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out,
                                 unsigned long long* d_bad, cudaStream_t s) {
    if (!n) return cudaSuccess;
    gen_below_p61_kernel<<<grid_for(n), kThreads, 0, s>>>(seed, start, n, out, d_bad);
    return cudaGetLastError();
}
cudaError_t launch_gen_pm_inputs(uint64_t seed, uint64_t c, uint64_t start, uint64_t n, uint64_t* out,
                                 unsigned long long* d_bad, cudaStream_t s) {
    if (!n) return cudaSuccess;
    gen_pm_kernel<<<grid_for(n), kThreads, 0, s>>>(seed, c, start, n, out, d_bad);
    return cudaGetLastError();
}
cudaError_t launch_gen_zipf(uint64_t master, const uint64_t* cdf, uint32_t T, double c1, double universe,
                            uint64_t start, uint64_t n, uint32_t* keys, int32_t* weights, cudaStream_t s) {
    if (!n) return cudaSuccess;
    gen_zipf_kernel<<<grid_for(n), kThreads, 0, s>>>(master, cdf, T, c1, universe, start, n, keys, weights);
    return cudaGetLastError();
}

}  // namespace mb200
