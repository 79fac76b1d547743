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
// input pairs per thread per round, with the next round's in flight (the
// kernels were HBM-latency bound without the prefetch: config 3 1.55 -> 1.38 ms,
// the exact division map 0.80 -> 0.70 ms; 4 pairs in flight measured slower)
constexpr int kUnroll = 2;
constexpr int kMapUnroll = kUnroll;

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
    // software pipeline: the next round's kUnroll input pairs are in flight while
    // the current round is divided (the kernel is HBM-latency bound otherwise)
    ulonglong2 a[kUnroll], bb[kUnroll];
    if (i + (kUnroll - 1) * stride < npairs) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            a[u] = ld_stream(v2 + 2 * (i + u * stride));
            bb[u] = ld_stream(v2 + 2 * (i + u * stride) + 1);
        }
    }
    for (; i + (kUnroll - 1) * stride < npairs; i += kUnroll * stride) {
        ulonglong2 na[kUnroll], nb[kUnroll];
        const uint64_t j = i + kUnroll * stride;
        const bool more = j + (kUnroll - 1) * stride < npairs;
        if (more) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                na[u] = ld_stream(v2 + 2 * (j + u * stride));
                nb[u] = ld_stream(v2 + 2 * (j + u * stride) + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            u64 q0, r0, q1, r1;
            divmod_one<B, M>(a[u].x, a[u].y, b, c, m, q0, r0, overflow);
            divmod_one<B, M>(bb[u].x, bb[u].y, b, c, m, q1, r1, overflow);
            st_stream(q2 + i + u * stride, make_ulonglong2(q0, q1));
            if (r2) st_stream(r2 + i + u * stride, make_ulonglong2(r0, r1));  // null: quotient only
        }
        if (more) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                a[u] = na[u];
                bb[u] = nb[u];
            }
        }
    }
    for (; i < npairs; i += stride) {
        const ulonglong2 a = ld_stream(v2 + 2 * i), bb = ld_stream(v2 + 2 * i + 1);
        u64 q0, r0, q1, r1;
        divmod_one<B, M>(a.x, a.y, b, c, m, q0, r0, overflow);
        divmod_one<B, M>(bb.x, bb.y, b, c, m, q1, r1, overflow);
        st_stream(q2 + i, make_ulonglong2(q0, q1));
        if (r2) st_stream(r2 + i, make_ulonglong2(r0, r1));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        u64 q0, r0;
        divmod_one<B, M>(v[2 * (n - 1)], v[2 * (n - 1) + 1], b, c, m, q0, r0, overflow);
        q[n - 1] = q0;
        if (r) r[n - 1] = r0;
    }
    if (__any_sync(0xffffffffu, overflow) && (threadIdx.x & 31) == 0) atomicAdd(flags, 1ull);
}

template <int B, int M>
__global__ void __launch_bounds__(kThreads) pm_divmod_scalar(const u64* __restrict__ v, uint64_t n, u32 b, u64 c,
                                                             u32 m, u64* __restrict__ q, u64* __restrict__ r,
                                                             unsigned long long* flags) {
    unsigned overflow = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        u64 q0, r0;
        divmod_one<B, M>(v[2 * i], v[2 * i + 1], b, c, m, q0, r0, overflow);
        q[i] = q0;
        if (r) r[i] = r0;
    }
    if (__any_sync(0xffffffffu, overflow) && (threadIdx.x & 31) == 0) atomicAdd(flags, 1ull);
}

// Alg 5 alone (pseudo_mersenne_mod, field.cpp:267-273) from a given quotient:
// r = (v + z c) & (2^b - 1); b <= 64 keeps only the low 64 bits of v + z c.
__global__ void __launch_bounds__(kThreads) pm_mod_kernel(const u64* __restrict__ v, const u64* __restrict__ z,
                                                          uint64_t n, u32 b, u64 c, u64* __restrict__ r) {
    const u64 mask = b == 64 ? ~0ull : ((1ull << b) - 1);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        r[i] = (__ldg(v + 2 * i) + __ldg(z + i) * c) & mask;
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

// Bucket maps (bucketing.cpp:61-95) on u64 values, b <= 64:
//   KIND 0 map_pow2      (v r) >> b
//   KIND 1 map_mersenne  ((v + 1) r) >> b
//   KIND 2 ExactDivisionMap  floor(v r / p) by Alg 4 with the constructor's m
// The product is formed in registers (u128), so one launch reads 8 B and
// writes 8 B per value (HBM-bound, like K6).  Values >= `bound` (the map's
// domain; 0 = every u64 is in the domain) are counted into flags[0].
template <int KIND, int B, int M>
__device__ __forceinline__ u64 bucket_one(u64 v, u32 b_rt, u64 c, u32 m_rt, u64 r, u64 bound, unsigned& bad) {
    bad += bound != 0 && v >= bound;
    if (KIND == 2) {
        u64 q, rem;
        unsigned overflow = 0;  // impossible inside the domain ((p-1) r <= max_input by construction)
        divmod_one<B, M>(v * r, __umul64hi(v, r), b_rt, c, m_rt, q, rem, overflow);
        return q;
    }
    const u64 x = KIND == 1 ? v + 1 : v;  // v < 2^b - 1, so no wrap for b = 64
    const u64 lo = x * r, hi = __umul64hi(x, r);
    const u32 b = B ? (u32)B : b_rt;
    return b == 64 ? hi : (lo >> b) | (hi << (64 - b));
}

template <int KIND, int B, int M>
__global__ void __launch_bounds__(kThreads) bucket_map_kernel(const u64* __restrict__ v, uint64_t n, u32 b, u64 c,
                                                              u32 m, u64 r, u64 bound, u64* __restrict__ out,
                                                              unsigned long long* flags) {
    const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(v);
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
    const uint64_t npairs = n >> 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned bad = 0;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // software pipeline as pm_divmod_kernel: the next round's pairs in flight
    ulonglong2 a[kMapUnroll];
    if (i + (kMapUnroll - 1) * stride < npairs) {
#pragma unroll
        for (int u = 0; u < kMapUnroll; ++u) a[u] = ld_stream(v2 + i + u * stride);
    }
    for (; i + (kMapUnroll - 1) * stride < npairs; i += kMapUnroll * stride) {
        ulonglong2 na[kMapUnroll];
        const uint64_t j = i + kMapUnroll * stride;
        const bool more = j + (kMapUnroll - 1) * stride < npairs;
        if (more) {
#pragma unroll
            for (int u = 0; u < kMapUnroll; ++u) na[u] = ld_stream(v2 + j + u * stride);
        }
#pragma unroll
        for (int u = 0; u < kMapUnroll; ++u)
            st_stream(o2 + i + u * stride,
                      make_ulonglong2(bucket_one<KIND, B, M>(a[u].x, b, c, m, r, bound, bad),
                                      bucket_one<KIND, B, M>(a[u].y, b, c, m, r, bound, bad)));
        if (more) {
#pragma unroll
            for (int u = 0; u < kMapUnroll; ++u) a[u] = na[u];
        }
    }
    for (; i < npairs; i += stride) {
        const ulonglong2 a = ld_stream(v2 + i);
        st_stream(o2 + i, make_ulonglong2(bucket_one<KIND, B, M>(a.x, b, c, m, r, bound, bad),
                                          bucket_one<KIND, B, M>(a.y, b, c, m, r, bound, bad)));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        out[n - 1] = bucket_one<KIND, B, M>(v[n - 1], b, c, m, r, bound, bad);
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicAdd(flags, (unsigned long long)bad);
}

template <int KIND, int B, int M>
__global__ void __launch_bounds__(kThreads) bucket_map_scalar(const u64* __restrict__ v, uint64_t n, u32 b, u64 c,
                                                              u32 m, u64 r, u64 bound, u64* __restrict__ out,
                                                              unsigned long long* flags) {
    unsigned bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = bucket_one<KIND, B, M>(v[i], b, c, m, r, bound, bad);
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicAdd(flags, (unsigned long long)bad);
}

constexpr int kStreamCtasPerSm = 256;
int grid_for(uint64_t items, int per_sm) {
    const uint64_t need = (items + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_pm_divmod(const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t iters, uint64_t* q,
                             uint64_t* r, unsigned long long* d_flags, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)v | (uintptr_t)q | (uintptr_t)r) & 15) == 0;  // r may be null
    if (!vec) {
        const int g = grid_for(n, 8);
        if (b == 64) pm_divmod_scalar<64, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
        else pm_divmod_scalar<0, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
        return cudaGetLastError();
    }
    // Grid: 256 CTAs per SM's worth (each CTA ~3.5 pipelined rounds on config 3), not one
    // resident wave: with 8 per SM the grid-stride puts the concurrently touched
    // addresses ~77 MB apart and config 3 ran 1.415 ms; 32 per SM 1.36 ms, 256 per SM
    // 1.294 ms (6.6 TB/s of algorithmic traffic), 512 per SM 1.33 ms, one round per CTA
    // 1.53 ms.
    const int g = grid_for((n / 2 + kUnroll - 1) / kUnroll, kStreamCtasPerSm);
    if (b == 64 && iters == 3) pm_divmod_kernel<64, 3><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else if (b == 64 && iters == 2) pm_divmod_kernel<64, 2><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else if (b == 64) pm_divmod_kernel<64, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    else pm_divmod_kernel<0, 0><<<g, kThreads, 0, s>>>(v, n, b, c, iters, q, r, d_flags);
    return cudaGetLastError();
}

namespace {
template <int KIND, int B, int M>
void bucket_launch(bool vec, const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t m, uint64_t r,
                   uint64_t bound, uint64_t* out, unsigned long long* flags, cudaStream_t s) {
    if (vec)
        bucket_map_kernel<KIND, B, M>
            <<<grid_for((n / 2 + kUnroll - 1) / kUnroll, kStreamCtasPerSm), kThreads, 0, s>>>(v, n, b, c, m, r, bound, out, flags);
    else
        bucket_map_scalar<KIND, B, M><<<grid_for(n, 8), kThreads, 0, s>>>(v, n, b, c, m, r, bound, out, flags);
}
}  // namespace

cudaError_t launch_bucket_map(int kind, const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t m,
                              uint64_t r, uint64_t bound, uint64_t* out, unsigned long long* d_flags, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)v | (uintptr_t)out) & 15) == 0;
    if (kind == 0) bucket_launch<0, 0, 0>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    else if (kind == 1) bucket_launch<1, 0, 0>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    else if (b == 64 && m == 2) bucket_launch<2, 64, 2>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    else if (b == 64 && m == 3) bucket_launch<2, 64, 3>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    else if (b == 64) bucket_launch<2, 64, 0>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    else bucket_launch<2, 0, 0>(vec, v, n, b, c, m, r, bound, out, d_flags, s);
    return cudaGetLastError();
}

cudaError_t launch_pm_mod(const uint64_t* v, const uint64_t* z, uint64_t n, uint32_t b, uint64_t c, uint64_t* r,
                          cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    pm_mod_kernel<<<grid_for(n, 8), kThreads, 0, s>>>(v, z, n, b, c, r);
    return cudaGetLastError();
}

cudaError_t launch_count_above(const uint64_t* v, uint64_t n, uint64_t max_lo, uint64_t max_hi,
                               unsigned long long* d_count, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    count_above_kernel<<<grid_for(n, 8), kThreads, 0, s>>>(v, n, max_lo, max_hi, d_count);
    return cudaGetLastError();
}

}  // namespace mb200
