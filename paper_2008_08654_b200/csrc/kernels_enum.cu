// kernels_enum.cu -- exhaustive sketch second-moment enumeration on the GPU
// (reference enum_moment_sums_serial / _parallel, verify.cpp:505-603, the
// paper's exact-moment checks).
//
// Over every degree-3 coefficient vector (a0, a1, a2, a3) in Z_p^4,
// p = 2^b - 1, hash each stream key x_j to h_j = a0 x^3 + a1 x^2 + a2 x + a3
// (mod p), split it (idx_j, s_j) with the sketch's splitter, and accumulate
// X = sum_i C_i^2 (C_i = sum_{idx_j = i} s_j w_j) and X^2 exactly.
//
// GPU formulation: signs are +-1, so X = sum_j w_j^2 + 2 sum_{j<l} [idx_j == idx_l]
// s_j w_j s_l w_l -- no counter array per family.  One thread owns a triple
// (a0, a1, a2) and walks a3 over Z_p: h_j(a3 + 1) = h_j(a3) + 1 (mod p), so a
// family costs N shared-memory table lookups, N increments and N(N-1)/2
// compares.  The split table (index | sign << 15 for every h < p, p < 2^15)
// sits in shared memory.  Sums are exact: per-thread u64 (X <= 2^20, p
// families per triple), folded into u128 with carries, warp-reduced, then
// added into the global u128 pair with carry-propagating atomics.
#include "mb200_sketch_dev.cuh"

namespace mb200 {

namespace {

constexpr int kEnumThreads = 256;

__global__ void enum_table_kernel(const SketchParams sp, u32 p, uint16_t* tab) {
    for (u32 h = blockIdx.x * blockDim.x + threadIdx.x; h < p; h += gridDim.x * blockDim.x) {
        bool neg;
        const u64 idx = sk::split_small(sp, h, 0, neg);
        tab[h] = (uint16_t)(idx | (neg ? 0x8000u : 0u));
    }
}

__device__ __forceinline__ void add128(u64& lo, u64& hi, u64 v_lo, u64 v_hi) {
    asm("add.cc.u64  %0, %0, %2;\n\t"
        "addc.u64    %1, %1, %3;"
        : "+l"(lo), "+l"(hi)
        : "l"(v_lo), "l"(v_hi));
}

__device__ __forceinline__ void atomic_add128(unsigned long long* dst, u64 lo, u64 hi) {
    const unsigned long long old = atomicAdd(dst, (unsigned long long)lo);
    const u64 carry = (u64)old + lo < lo ? 1 : 0;
    if (hi + carry) atomicAdd(dst + 1, (unsigned long long)(hi + carry));
}

// N = capacity (>= number of non-zero stream entries; padding has w = 0).
// The stream (x, x^2, x^3, w) lives in shared memory next to the split table;
// weights are held in registers for N <= 8 (the reference suites' streams).
template <int N>
__global__ void __launch_bounds__(kEnumThreads) enum_moments_kernel(u32 p, u32 n, u64 triples, u32 w2,
                                                                    const u32* __restrict__ xs,
                                                                    const int32_t* __restrict__ ws,
                                                                    const uint16_t* __restrict__ tab_g,
                                                                    unsigned long long* out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    u32* sx = reinterpret_cast<u32*>(smem_raw);  // [3][N]
    int32_t* sw_s = reinterpret_cast<int32_t*>(sx + 3 * N);
    uint16_t* tab = reinterpret_cast<uint16_t*>(sw_s + N);
    for (u32 j = threadIdx.x; j < (u32)N; j += blockDim.x) {
        const bool v = j < n;
        sx[j] = v ? xs[j] : 0;
        sx[N + j] = v ? xs[n + j] : 0;
        sx[2 * N + j] = v ? xs[2 * n + j] : 0;
        sw_s[j] = v ? ws[j] : 0;
    }
    for (u32 h = threadIdx.x; h < p; h += blockDim.x) tab[h] = tab_g[h];
    __syncthreads();
    constexpr bool kRegW = N <= 8;
    int32_t wr[kRegW ? N : 1];
#pragma unroll
    for (int j = 0; j < (kRegW ? N : 1); ++j) wr[j] = sw_s[j];
    u64 sx_lo = 0, sx_hi = 0, sq_lo = 0, sq_hi = 0;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < triples; t += stride) {
        const u32 a2 = (u32)(t % p);
        const u64 t1 = t / p;
        const u32 a1 = (u32)(t1 % p), a0 = (u32)(t1 / p);
        u32 cur[N];
#pragma unroll
        for (int j = 0; j < N; ++j)  // a0 x^3 + a1 x^2 + a2 x < 3 p^2 < 2^32 for p < 2^15
            cur[j] = (a0 * sx[2 * N + j] + a1 * sx[N + j] + a2 * sx[j]) % p;
        u64 fx = 0, fxx = 0;
#pragma unroll 1
        for (u32 a3 = 0; a3 < p; ++a3) {
            int32_t e[N];  // (index << 16) | (s w & 0xffff), |w| <= 1024
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const u32 t2 = tab[cur[j]];
                const int32_t wj = kRegW ? wr[kRegW ? j : 0] : sw_s[j];
                const int32_t sgw = (t2 & 0x8000u) ? -wj : wj;
                e[j] = (int32_t)((t2 & 0x7fffu) << 16) | (sgw & 0xffff);
                cur[j] = cur[j] + 1 == p ? 0 : cur[j] + 1;
            }
            int32_t cross = 0;  // |cross| <= (sum |w|)^2 / 2 <= 2^19
#pragma unroll
            for (int j = 0; j < N; ++j)
#pragma unroll
                for (int l = j + 1; l < N; ++l)
                    cross += ((e[j] ^ e[l]) >> 16) == 0 ? (int32_t)(int16_t)e[j] * (int32_t)(int16_t)e[l] : 0;
            const u64 X = (u64)(int64_t)((int32_t)w2 + 2 * cross);
            fx += X;
            fxx += X * X;  // <= p 2^40 < 2^55
        }
        add128(sx_lo, sx_hi, fx, 0);
        add128(sq_lo, sq_hi, fxx, 0);
    }
    // warp reduction of the two u128 sums
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const u64 a = __shfl_down_sync(0xffffffffu, sx_lo, off), b = __shfl_down_sync(0xffffffffu, sx_hi, off);
        const u64 c = __shfl_down_sync(0xffffffffu, sq_lo, off), d = __shfl_down_sync(0xffffffffu, sq_hi, off);
        add128(sx_lo, sx_hi, a, b);
        add128(sq_lo, sq_hi, c, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_add128(out, sx_lo, sx_hi);
        atomic_add128(out + 2, sq_lo, sq_hi);
    }
}

template <int N>
cudaError_t launch_n(u32 p, u32 n, u32 w2, const u32* xs, const int32_t* ws, const uint16_t* tab,
                     unsigned long long* out, cudaStream_t s) {
    const u64 triples = (u64)p * p * p;
    u64 grid = (triples + kEnumThreads - 1) / kEnumThreads;
    const u64 cap = (u64)sm_count() * 8;
    if (grid > cap) grid = cap;
    const size_t smem = (size_t)N * 16 + (size_t)p * sizeof(uint16_t);
    auto fn = enum_moments_kernel<N>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    fn<<<(unsigned)grid, kEnumThreads, smem, s>>>(p, n, triples, w2, xs, ws, tab, out);
    return cudaGetLastError();
}

}  // namespace

// xs: 3n u32 (x, x^2, x^3 mod p, SoA); ws: n i32 (non-zero weights);
// sp: splitter geometry (b, splitter, width = buckets, lw); out: 4 u64 (accumulated)
cudaError_t launch_enum_moments(const SketchParams& sp, uint32_t n, uint32_t w2, const uint32_t* xs,
                                const int32_t* ws, uint16_t* tab, unsigned long long* out, cudaStream_t s) {
    const u32 p = (u32)sp.p;
    enum_table_kernel<<<(p + 255) / 256, 256, 0, s>>>(sp, p, tab);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (n <= 2) return launch_n<2>(p, n, w2, xs, ws, tab, out, s);
    if (n <= 4) return launch_n<4>(p, n, w2, xs, ws, tab, out, s);
    if (n <= 8) return launch_n<8>(p, n, w2, xs, ws, tab, out, s);
    if (n <= 16) return launch_n<16>(p, n, w2, xs, ws, tab, out, s);
    if (n <= 32) return launch_n<32>(p, n, w2, xs, ws, tab, out, s);
    return launch_n<64>(p, n, w2, xs, ws, tab, out, s);
}

}  // namespace mb200
