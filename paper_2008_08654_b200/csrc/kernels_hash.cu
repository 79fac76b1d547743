// kernels_hash.cu -- K1 / K2: batched Horner evaluation of degree-(k-1)
// polynomials over Z_p (Alg 1; reference PolyHashFamily::operator(),
// polyhash.cpp:59-89).
//
// Data layout: keys are a dense u32 or u64 array in HBM, outputs a dense u64
// array (K2: two dense u64 arrays, low and high 64 bits of the 89-bit hash).
// Each thread streams 16-byte vectors with UNROLL loads in flight; the grid is
// a whole number of waves over the 148 SMs (grid-stride, persistent).
#include "mb200_device.cuh"
#include "mb200_internal.h"
#include "mb200_mem.cuh"

namespace mb200 {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

int grid_for(uint64_t work_items, int per_sm) {
    const int sms = sm_count();
    const uint64_t need = (work_items + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sms * per_sm;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

template <int K>
__device__ __forceinline__ u64 eval61_key64(const u64 (&a)[K], u64 x) {
    return h61_finish(h61_eval64<K>(a, h61_key64(x)));
}

// Degree 7 with adapted coefficients (host/precond61.cpp; Knuth 4.6.4): five
// modular products instead of Horner's seven, the same value mod p.
//   u(x) = a7 (x + s) U(x) + r0,  U = (w + z + al4) w + al5,
//   w = (x + al2) z + al3,  z = (x + al0) x + al1,    c = {al0..al5, s, a7, r0}, all < p.
// Bounds for h61_step64(y, x, a) = fold(y x) + a (needs y0 x1 + y1 x0 < 2^64 and
// y x < 2^125; result < 2^61 + (y x >> 61) + a), with x0 <= 2^61 + 6 the folded key:
//   z: y = x0 + al0 < 2^62 + 6, x = x0              -> < 2^63 + 2^36, folded to < 2^61 + 8
//   w: y = x0 + al2 < 2^62 + 6, x = z               -> likewise
//   U: y = w + z + al4 < 3 * 2^61 + 16, x = w       -> < 5 * 2^61 + 2^36
//   V = (x + s) U: SHIFT: y = fold(U) < 2^61 + 8, x = x0 + s < 2^62 + 6  -> < 3 * 2^61 + 2^36;
//                  s = 0: y = U, x = x0 (y0 x1 + y1 x0 < 2^61.1 + 5 * 2^61.1)  -> < 6 * 2^61 + 2^36
//   out: y = fold(V) < 2^61 + 8, x = a7 < 2^61      -> < 3 * 2^61, finished by h61_finish.
template <bool SHIFT>
__device__ __forceinline__ u64 eval61_pre8(const u64 (&c)[9], u64 key) {
    const u64 x0 = h61_key64(key);
    const u64 z = h61_fold(h61_step64(x0 + c[0], x0, c[1]));
    const u64 w = h61_fold(h61_step64(x0 + c[2], z, c[3]));
    const u64 U = h61_step64(w + z + c[4], w, c[5]);
    const u64 V = SHIFT ? h61_step64(h61_fold(U), x0 + c[6], 0) : h61_step64(U, x0, 0);
    return h61_finish(h61_step64(h61_fold(V), c[7], c[8]));
}

// K = 8 evaluators of hash61_key64_kernel: Horner, or the adapted form
template <int K, int PRE>
struct Eval61 {
    u64 a[K];
    __device__ __forceinline__ explicit Eval61(const HashParams& hp) {
#pragma unroll
        for (int i = 0; i < K; ++i) a[i] = hp.lo[i];
    }
    __device__ __forceinline__ u64 operator()(u64 x) const { return eval61_key64<K>(a, x); }
};
template <int PRE>
struct Eval61<8, PRE> {
    static constexpr int kN = PRE ? 9 : 8;
    u64 c[kN];
    __device__ __forceinline__ explicit Eval61(const HashParams& hp) {
#pragma unroll
        for (int i = 0; i < kN; ++i) c[i] = PRE ? hp.hi[i] : hp.lo[i];
    }
    __device__ __forceinline__ u64 operator()(u64 x) const {
        if constexpr (PRE == 0) return eval61_key64<8>(c, x);
        else return eval61_pre8<PRE == 2>(c, x);
    }
};

template <int K>
__device__ __forceinline__ u64 eval61_key32(const u64 (&a)[K], u32 x) {
    u64 y = a[K - 1];
#pragma unroll
    for (int i = K - 2; i >= 0; --i) y = h61_step32(y, x, a[i]);
    return h61_finish(y);
}

// ---- K1, 64-bit keys: config 2 ---------------------------------------------
template <int K, int PRE>
__global__ void __launch_bounds__(kThreads) hash61_key64_kernel(const u64* __restrict__ keys,
                                                                uint64_t n, HashParams hp,
                                                                u64* __restrict__ out) {
    const Eval61<K, PRE> ev(hp);
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
    const uint64_t npairs = n >> 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // software pipeline: the next round's kUnroll vectors are in flight while
    // the current round is hashed
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    ulonglong2 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
        if (i + u * stride < npairs) v[u] = ld_stream(k2 + i + u * stride);
    for (; i < npairs; i += kUnroll * stride) {
        ulonglong2 nx[kUnroll];
        const uint64_t j = i + kUnroll * stride;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (j + u * stride < npairs) nx[u] = ld_stream(k2 + j + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (i + u * stride < npairs) {
                ulonglong2 h;
                h.x = ev(v[u].x);
                h.y = ev(v[u].y);
                st_stream(o2 + i + u * stride, h);
            }
            v[u] = nx[u];
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[n - 1] = ev(keys[n - 1]);
}

// ---- K1, 32-bit keys (reference bench setup) ---------------------------------
template <int K>
__global__ void __launch_bounds__(kThreads) hash61_key32_kernel(const u32* __restrict__ keys,
                                                                uint64_t n, HashParams hp,
                                                                u64* __restrict__ out) {
    u64 a[K];
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = hp.lo[i];
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
    const uint64_t nquads = n >> 2;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nquads; i += stride) {
        const uint4 v = ld_stream(k4 + i);
        ulonglong2 h0, h1;
        h0.x = eval61_key32<K>(a, v.x);
        h0.y = eval61_key32<K>(a, v.y);
        h1.x = eval61_key32<K>(a, v.z);
        h1.y = eval61_key32<K>(a, v.w);
        st_stream(o2 + 2 * i, h0);
        st_stream(o2 + 2 * i + 1, h1);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        const uint64_t j = (n & ~3ull) + threadIdx.x;
        out[j] = eval61_key32<K>(a, keys[j]);
    }
}

// ---- scalar variants for pointers that are not 16-byte aligned ---------------
template <int K, int PRE>
__global__ void __launch_bounds__(kThreads) hash61_key64_scalar(const u64* __restrict__ keys,
                                                                uint64_t n, HashParams hp,
                                                                u64* __restrict__ out) {
    const Eval61<K, PRE> ev(hp);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = ev(keys[i]);
}

template <int K>
__global__ void __launch_bounds__(kThreads) hash61_key32_scalar(const u32* __restrict__ keys,
                                                                uint64_t n, HashParams hp,
                                                                u64* __restrict__ out) {
    u64 a[K];
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = hp.lo[i];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = eval61_key32<K>(a, keys[i]);
}

// ---- generic b <= 61, runtime k, reference domain (small fields, KATs) -------
template <typename KeyT>
__global__ void __launch_bounds__(kThreads) hash_generic_kernel(const KeyT* __restrict__ keys,
                                                                uint64_t n, HashParams hp,
                                                                u64* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 x = (u64)keys[i];
        u64 y = hp.lo[hp.k - 1];
        for (int j = (int)hp.k - 2; j >= 0; --j) y = hgen_step(y, x, hp.lo[j], hp.b, hp.p);
        out[i] = hgen_finish(y, hp.b, hp.p);
    }
}

// ---- K2: p = 2^89 - 1, 64-bit keys -----------------------------------------------
template <int K>
__device__ __forceinline__ void eval89(const u32 (&c)[K][3], u64 x, u64& lo, u64& hi) {
    u32 y0 = c[K - 1][0], y1 = c[K - 1][1], y2 = c[K - 1][2];
    const u32 x0 = lo32(x), x1 = hi32(x);
#pragma unroll
    for (int i = K - 2; i >= 0; --i) h89_step(y0, y1, y2, x0, x1, c[i][0], c[i][1], c[i][2]);
    h89_finish(y0, y1, y2);
    lo = ((u64)y1 << 32) | y0;
    hi = y2;
}

template <int K>
__global__ void __launch_bounds__(kThreads) hash89_kernel(const u64* __restrict__ keys, uint64_t n,
                                                          HashParams hp, u64* __restrict__ out_lo,
                                                          u64* __restrict__ out_hi) {
    u32 c[K][3];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        c[i][0] = lo32(hp.lo[i]);
        c[i][1] = hi32(hp.lo[i]);
        c[i][2] = lo32(hp.hi[i]);
    }
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
    ulonglong2* l2 = reinterpret_cast<ulonglong2*>(out_lo);
    ulonglong2* h2 = reinterpret_cast<ulonglong2*>(out_hi);
    const uint64_t npairs = n >> 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
        const ulonglong2 v = ld_stream(k2 + i);
        u64 l0, h0, l1, h1;
        eval89<K>(c, v.x, l0, h0);
        eval89<K>(c, v.y, l1, h1);
        const ulonglong2 lo = make_ulonglong2(l0, l1), hi = make_ulonglong2(h0, h1);
        st_stream(l2 + i, lo);
        st_stream(h2 + i, hi);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        u64 lo, hi;
        eval89<K>(c, keys[n - 1], lo, hi);
        out_lo[n - 1] = lo;
        out_hi[n - 1] = hi;
    }
}

template <typename KeyT>
__global__ void count_out_of_domain_kernel(const KeyT* __restrict__ keys, uint64_t n, u64 limit,
                                           unsigned long long* count) {
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        bad += ((u64)keys[i] >= limit);
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace

#define MB200_K_DISPATCH(KV, CALL)                 \
    switch (KV) {                                   \
        case 1: { constexpr int K = 1; CALL; } break;  \
        case 2: { constexpr int K = 2; CALL; } break;  \
        case 3: { constexpr int K = 3; CALL; } break;  \
        case 4: { constexpr int K = 4; CALL; } break;  \
        case 5: { constexpr int K = 5; CALL; } break;  \
        case 6: { constexpr int K = 6; CALL; } break;  \
        case 7: { constexpr int K = 7; CALL; } break;  \
        case 8: { constexpr int K = 8; CALL; } break;  \
        case 9: { constexpr int K = 9; CALL; } break;  \
        case 10: { constexpr int K = 10; CALL; } break; \
        case 11: { constexpr int K = 11; CALL; } break; \
        case 12: { constexpr int K = 12; CALL; } break; \
        case 13: { constexpr int K = 13; CALL; } break; \
        case 14: { constexpr int K = 14; CALL; } break; \
        case 15: { constexpr int K = 15; CALL; } break; \
        case 16: { constexpr int K = 16; CALL; } break; \
        default: return cudaErrorInvalidValue;      \
    }

cudaError_t launch_hash61_key64(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(keys) && aligned16(out);
    // 24 CTAs per SM's worth for the pipelined vector kernel (config 2: 0.751 / 1.250 ms
    // at k = 4 / 8, against 0.762 / 1.266 ms with one resident wave's 8 and 0.79 / 1.29 ms
    // with 256)
    const int grid = vec ? grid_for((n / 2 + kUnroll - 1) / kUnroll, 24) : grid_for(n, 8);
    if (hp.k == 8 && hp.pre) {  // adapted coefficients in hp.hi (capi.cu)
        if (hp.pre == 2) {
            if (vec) hash61_key64_kernel<8, 2><<<grid, kThreads, 0, s>>>(keys, n, hp, out);
            else hash61_key64_scalar<8, 2><<<grid, kThreads, 0, s>>>(keys, n, hp, out);
        } else {
            if (vec) hash61_key64_kernel<8, 1><<<grid, kThreads, 0, s>>>(keys, n, hp, out);
            else hash61_key64_scalar<8, 1><<<grid, kThreads, 0, s>>>(keys, n, hp, out);
        }
        return cudaGetLastError();
    }
    if (!vec) {
        MB200_K_DISPATCH(hp.k, (hash61_key64_scalar<K, 0><<<grid, kThreads, 0, s>>>(keys, n, hp, out)));
        return cudaGetLastError();
    }
    MB200_K_DISPATCH(hp.k, (hash61_key64_kernel<K, 0><<<grid, kThreads, 0, s>>>(keys, n, hp, out)));
    return cudaGetLastError();
}

cudaError_t launch_hash61_key32(const uint32_t* keys, uint64_t n, const HashParams& hp, uint64_t* out,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (!aligned16(keys) || !aligned16(out)) {
        const int g = grid_for(n, 8);
        MB200_K_DISPATCH(hp.k, (hash61_key32_scalar<K><<<g, kThreads, 0, s>>>(keys, n, hp, out)));
        return cudaGetLastError();
    }
    // 64 CTAs per SM's worth (2^28 keys: 0.525 / 0.955 ms at k = 4 / 8, against 0.576 / 1.006 ms
    // with one resident wave's 8; tools/key32_probe.py)
    const int grid = grid_for(n / 4 + 1, 64);
    MB200_K_DISPATCH(hp.k, (hash61_key32_kernel<K><<<grid, kThreads, 0, s>>>(keys, n, hp, out)));
    return cudaGetLastError();
}

cudaError_t launch_hash_generic(const void* keys, int key_width, uint64_t n, const HashParams& hp,
                                uint64_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int grid = grid_for(n, 8);
    if (key_width == 32)
        hash_generic_kernel<u32><<<grid, kThreads, 0, s>>>((const u32*)keys, n, hp, out);
    else
        hash_generic_kernel<u64><<<grid, kThreads, 0, s>>>((const u64*)keys, n, hp, out);
    return cudaGetLastError();
}

// 62 <= b <= 127: the generic four-limb Horner (polyhash.cpp:78-88), scalar
// per key (no BASELINE config uses these moduli)
__global__ void __launch_bounds__(kThreads) hash_wide_kernel(const u64* __restrict__ keys, uint64_t n,
                                                             const HashParams hp, u64* __restrict__ out_lo,
                                                             u64* __restrict__ out_hi) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        u64 lo, hi;
        hash_wide(hp.lo, hp.hi, (int)hp.k, hp.b, keys[i], lo, hi);
        out_lo[i] = lo;
        out_hi[i] = hi;
    }
}

cudaError_t launch_hash_wide(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out_lo,
                             uint64_t* out_hi, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + kThreads - 1) / kThreads;
    if (grid > (uint64_t)sm_count() * 8) grid = (uint64_t)sm_count() * 8;
    hash_wide_kernel<<<(unsigned)grid, kThreads, 0, s>>>(keys, n, hp, out_lo, out_hi);
    return cudaGetLastError();
}

cudaError_t launch_hash89(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out_lo,
                          uint64_t* out_hi, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (!aligned16(keys) || !aligned16(out_lo) || !aligned16(out_hi)) return cudaErrorMisalignedAddress;
    const int grid = grid_for(n / 2 + 1, 32);  // (2^27 keys, k = 4: 0.685 ms with 8 per SM, 0.656 ms with 24-64)
    MB200_K_DISPATCH(hp.k, (hash89_kernel<K><<<grid, kThreads, 0, s>>>(keys, n, hp, out_lo, out_hi)));
    return cudaGetLastError();
}

cudaError_t launch_count_out_of_domain(const void* keys, int key_width, uint64_t n, uint32_t key_bits,
                                       unsigned long long* d_count, cudaStream_t s) {
    if (n == 0 || key_bits >= (uint32_t)key_width) return cudaSuccess;
    const int grid = grid_for(n, 8);
    const u64 limit = 1ull << key_bits;
    if (key_width == 32)
        count_out_of_domain_kernel<u32><<<grid, kThreads, 0, s>>>((const u32*)keys, n, limit, d_count);
    else
        count_out_of_domain_kernel<u64><<<grid, kThreads, 0, s>>>((const u64*)keys, n, limit, d_count);
    return cudaGetLastError();
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

int device_id() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

}  // namespace mb200
