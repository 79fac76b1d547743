// kernels_divmod.cu -- K6: branch-free division and remainder by a
// pseudo-Mersenne number p = 2^b - c (Alg 4 + Alg 5; reference
// PseudoMersenneModulus::div_unchecked field.cpp:246-258, pseudo_mersenne_div
// :260-265, pseudo_mersenne_mod :267-273).
//
//   v' = v + c;  z = v' >> b;  repeat m-1 times: z = (z c + v') >> b
//   q = z;  r = (v + z c) & (2^b - 1)
//
// Layout: inputs are u128 stored as interleaved (lo, hi) u64 pairs (16 B per
// unit), outputs two dense u64 arrays q[] and r[] (SoA) -- 32 B of HBM
// traffic per unit, which bounds this kernel (HBM-bound).
// Intermediates are held in three 64-bit words (z c + v' < 2^130 for every
// b <= 64, c < 2^(b-1), v < 2^128).
#include "mb200_device.cuh"
#include "mb200_internal.h"
#include "mb200_mem.cuh"

namespace mb200 {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

struct W3 {
    u64 w0, w1, w2;
};

template <int B>
__device__ __forceinline__ W3 shr3(W3 a, u32 b_rt) {
    if (B == 64) return {a.w1, a.w2, 0};
    const u32 b = b_rt;
    if (b == 64) return {a.w1, a.w2, 0};
    return {(a.w0 >> b) | (a.w1 << (64 - b)), (a.w1 >> b) | (a.w2 << (64 - b)), a.w2 >> b};
}

// (z c + vp) with z, vp three words, c < 2^63; exact while the true value < 2^192
__device__ __forceinline__ W3 mul_add3(W3 z, u64 c, W3 vp) {
    W3 r;
    const u64 p0l = z.w0 * c, p0h = __umul64hi(z.w0, c);
    const u64 p1l = z.w1 * c, p1h = __umul64hi(z.w1, c);
    const u64 p2l = z.w2 * c;
    // r = vp + (p0l, p0h + p1l, p1h + p2l)
    asm("add.cc.u64  %0, %3, %6;\n\t"
        "addc.cc.u64 %1, %4, %7;\n\t"
        "addc.u64    %2, %5, %8;"
        : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2)
        : "l"(vp.w0), "l"(vp.w1), "l"(vp.w2), "l"(p0l), "l"(p0h), "l"(p2l + p1h));
    u64 c1;
    asm("add.cc.u64  %0, %0, %2;\n\t"
        "addc.u64    %1, 0, 0;"
        : "+l"(r.w1), "=l"(c1)
        : "l"(p1l));
    r.w2 += c1;
    return r;
}

template <int B, int M>
__device__ __forceinline__ void divmod_one(u64 vlo, u64 vhi, u32 b_rt, u64 c, u32 m_rt, u64& q, u64& r,
                                           unsigned& overflow) {
    W3 vp;
    asm("add.cc.u64  %0, %3, %4;\n\t"
        "addc.cc.u64 %1, %5, 0;\n\t"
        "addc.u64    %2, 0, 0;"
        : "=l"(vp.w0), "=l"(vp.w1), "=l"(vp.w2)
        : "l"(vlo), "l"(c), "l"(vhi));
    W3 z = shr3<B>(vp, b_rt);
    if (M > 0) {
#pragma unroll
        for (int i = 1; i < M; ++i) z = shr3<B>(mul_add3(z, c, vp), b_rt);
    } else {
#pragma unroll 1
        for (u32 i = 1; i < m_rt; ++i) z = shr3<B>(mul_add3(z, c, vp), b_rt);
    }
    overflow |= (z.w1 | z.w2) != 0;
    q = z.w0;
    const u32 b = B ? (u32)B : b_rt;
    const u64 low = vlo + z.w0 * c;  // (v + z c) mod 2^64; b <= 64 keeps only these bits
    r = b == 64 ? low : (low & ((1ull << b) - 1));
}

template <int B, int M>
__global__ void __launch_bounds__(kThreads) pm_divmod_kernel(const u64* __restrict__ v, uint64_t n, u32 b, u64 c,
                                                             u32 m, u64* __restrict__ q, u64* __restrict__ r,
                                                             unsigned long long* flags) {
    const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(v);
    ulonglong2* q2 = reinterpret_cast<ulonglong2*>(q);
    ulonglong2* r2 = reinterpret_cast<ulonglong2*>(r);
    const uint64_t npairs = n >> 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned overflow = 0;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < npairs; i += kUnroll * stride) {
        ulonglong2 a[kUnroll], bb[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            a[u] = ld_stream(v2 + 2 * (i + u * stride));
            bb[u] = ld_stream(v2 + 2 * (i + u * stride) + 1);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            u64 q0, r0, q1, r1;
            divmod_one<B, M>(a[u].x, a[u].y, b, c, m, q0, r0, overflow);
            divmod_one<B, M>(bb[u].x, bb[u].y, b, c, m, q1, r1, overflow);
            st_stream(q2 + i + u * stride, make_ulonglong2(q0, q1));
            st_stream(r2 + i + u * stride, make_ulonglong2(r0, r1));
        }
    }
    for (; i < npairs; i += stride) {
        const ulonglong2 a = ld_stream(v2 + 2 * i), bb = ld_stream(v2 + 2 * i + 1);
        u64 q0, r0, q1, r1;
        divmod_one<B, M>(a.x, a.y, b, c, m, q0, r0, overflow);
        divmod_one<B, M>(bb.x, bb.y, b, c, m, q1, r1, overflow);
        st_stream(q2 + i, make_ulonglong2(q0, q1));
        st_stream(r2 + i, make_ulonglong2(r0, r1));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        u64 q0, r0;
        divmod_one<B, M>(v[2 * (n - 1)], v[2 * (n - 1) + 1], b, c, m, q0, r0, overflow);
        q[n - 1] = q0;
        r[n - 1] = r0;
    }
    if (__any_sync(0xffffffffu, overflow) && (threadIdx.x & 31) == 0) atomicAdd(flags, 1ull);
}

template <int B, int M>
__global__ void __launch_bounds__(kThreads) pm_divmod_scalar(const u64* __restrict__ v, uint64_t n, u32 b, u64 c,
                                                             u32 m, u64* __restrict__ q, u64* __restrict__ r,
                                                             unsigned long long* flags) {
    unsigned overflow = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        divmod_one<B, M>(v[2 * i], v[2 * i + 1], b, c, m, q[i], r[i], overflow);
    if (__any_sync(0xffffffffu, overflow) && (threadIdx.x & 31) == 0) atomicAdd(flags, 1ull);
}

__global__ void count_above_kernel(const u64* __restrict__ v, uint64_t n, u64 max_lo, u64 max_hi,
                                   unsigned long long* count) {
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 lo = v[2 * i], hi = v[2 * i + 1];
        bad += (hi > max_hi) || (hi == max_hi && lo > max_lo);
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

int grid_for(uint64_t items, int per_sm) {
    const uint64_t need = (items + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_pm_divmod(const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t iters, uint64_t* q,
                             uint64_t* r, unsigned long long* d_flags, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)v | (uintptr_t)q | (uintptr_t)r) & 15) == 0;
    if (!vec) {
        const int g = grid_for(n, 8);
        if (b == 64) pm_divmod_scalar<64, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
        else pm_divmod_scalar<0, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
        return cudaGetLastError();
    }
    const int g = grid_for((n / 2 + kUnroll - 1) / kUnroll, 8);
    if (b == 64 && iters == 3) pm_divmod_kernel<64, 3><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else if (b == 64 && iters == 2) pm_divmod_kernel<64, 2><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else if (b == 64) pm_divmod_kernel<64, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else pm_divmod_kernel<0, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    return cudaGetLastError();
}

cudaError_t launch_count_above(const uint64_t* v, uint64_t n, uint64_t max_lo, uint64_t max_hi,
                               unsigned long long* d_count, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    count_above_kernel<<<grid_for(n, 8), kThreads, 0, s>>>(v, n, max_lo, max_hi, d_count);
    return cudaGetLastError();
}

}  // namespace mb200
