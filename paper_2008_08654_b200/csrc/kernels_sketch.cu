// kernels_sketch.cu -- K3 + K4 (fused hash -> two-for-one split -> Count
// Sketch scatter-add), K5 (exact 128-bit second-moment estimator), merge and
// point query.
//
// Reference: CountSketch::process sketch.cpp:133-140 (per row: h = family(x);
// (i, s) = split(h); c[row][i] += s * delta, wrapping u64), split_pow2
// sketch.cpp:13-19, row_second_moment sketch.cpp:142-158, merge :182-193,
// point_query :170-180.
//
// HBM layout: counters i64 [rows][width] row-major, exactly the reference's
// counters_ vector (sketch.hpp:75), so a D2H copy is byte-identical to it.
//
// Strategies (chosen by the launcher from the table size):
//   SMEM32 / SMEM64 : the whole table privatised per CTA in shared memory
//                     (config 1: 1 x 1024), shared atomics, one merge of the
//                     non-zero counters into HBM per CTA at the end.
//   GLOBAL          : tables larger than shared memory (configs 4, 5: 1 MiB,
//                     2.5 MiB, L2-resident): fire-and-forget red.global.add.u64,
//                     optionally preceded by warp-level aggregation of equal
//                     keys (__match_any_sync) so heavy hitters of a skewed
//                     stream cost one hash + one red per warp, not per item.
// Integer addition is associative and commutative, so every strategy and every
// grid produces bit-identical tables (the reference's merge-equals-
// concatenation property, test_sketch.cpp:239-261).
#include <type_traits>

#include "mb200_device.cuh"
#include "mb200_internal.h"
#include "mb200_mem.cuh"
#include "mb200_sketch_dev.cuh"

namespace mb200 {

namespace {

using namespace sk;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <int MODE, int K, typename KeyT, int WK, int STRAT, int FAM>
__global__ void __launch_bounds__(kThreads) cs_update_kernel(const SketchParams sp,
                                                             const KeyT* __restrict__ keys,
                                                             const void* __restrict__ w, uint64_t n,
                                                             i64* __restrict__ table, int aggregate) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ i64 scratch[kWarps][32];
    void* smem = smem_raw;
    const uint64_t cells = (uint64_t)sp.rows * sp.width;
    if (STRAT == SMEM_LOHI) {  // 2^31-biased low words + wrap counters (see table_add)
        for (uint64_t i = threadIdx.x; i < 2 * kLohiCells; i += kThreads)
            reinterpret_cast<u32*>(smem)[i] = i < kLohiCells ? 0x80000000u : 0u;
        __syncthreads();
    } else if (STRAT != GLOBAL) {
        const uint64_t words = STRAT == SMEM32 ? cells : 2 * cells;
        for (uint64_t i = threadIdx.x; i < words; i += kThreads) reinterpret_cast<u32*>(smem)[i] = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t warps_total = (uint64_t)gridDim.x * kWarps;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp;
    const uint64_t tile = 32ull * kSlots;
    if (STRAT != GLOBAL || !aggregate) {
        // independent items: the slots' Horner chains interleave, and the next
        // tile's loads are in flight while this one is hashed
        KeyT kx[kSlots];
        i64 dx[kSlots];
        uint64_t base = gw * tile;
#pragma unroll
        for (int u = 0; u < kSlots; ++u) {
            const uint64_t i = base + u * 32 + lane;
            kx[u] = i < n ? ld_nc(keys + i) : KeyT(0);
            dx[u] = i < n ? load_weight<WK>(w, i) : 0;
        }
        for (; base < n; base += warps_total * tile) {
            const uint64_t nb = base + warps_total * tile;
            KeyT kn[kSlots];
            i64 dn[kSlots];
#pragma unroll
            for (int u = 0; u < kSlots; ++u) {
                const uint64_t i = nb + u * 32 + lane;
                kn[u] = i < n ? ld_nc(keys + i) : KeyT(0);
                dn[u] = i < n ? load_weight<WK>(w, i) : 0;
            }
            unsigned valid = 0;
#pragma unroll
            for (int u = 0; u < kSlots; ++u) valid |= (base + u * 32 + lane < n ? 1u : 0u) << u;
            process_items<MODE, K, STRAT, kSlots, FAM>(sp, kx, dx, valid, smem, table);
#pragma unroll
            for (int u = 0; u < kSlots; ++u) {
                kx[u] = kn[u];
                dx[u] = dn[u];
            }
        }
    } else {
    for (uint64_t base = gw * tile; base < n; base += warps_total * tile) {
        KeyT kx[kSlots];
        i64 dx[kSlots];
#pragma unroll
        for (int u = 0; u < kSlots; ++u) {
            const uint64_t i = base + u * 32 + lane;
            kx[u] = i < n ? ld_nc(keys + i) : KeyT(0);
            dx[u] = i < n ? load_weight<WK>(w, i) : 0;
        }
#pragma unroll 1
        for (int u = 0; u < kSlots; ++u) {
            const uint64_t i = base + u * 32 + lane;
            const bool valid = i < n;
            if (STRAT == GLOBAL && aggregate) {
                const unsigned vmask = __ballot_sync(kFull, valid);
                if (valid) {
                    const unsigned peers = __match_any_sync(vmask, kx[u]);
                    const int leader = __ffs(peers) - 1;
                    i64 d = dx[u];
                    if (__popc(peers) > 1) {
                        scratch[warp][lane] = d;
                        __syncwarp(peers);
                        if (lane == leader) {
                            u64 s = 0;
                            for (unsigned m = peers; m; m &= m - 1) s += (u64)scratch[warp][__ffs(m) - 1];
                            d = (i64)s;
                        }
                        __syncwarp(peers);
                    }
                    if (lane == leader) process_item<MODE, K, STRAT>(sp, (u64)kx[u], d, smem, table);
                }
            } else if (valid) {
                process_item<MODE, K, STRAT>(sp, (u64)kx[u], dx[u], smem, table);
            }
        }
    }
    }
    if (STRAT != GLOBAL) {
        __syncthreads();
        for (uint64_t c = threadIdx.x; c < cells; c += kThreads) {
            u64 v;
            if (STRAT == SMEM32) v = (u64)(i64)(i32)reinterpret_cast<u32*>(smem)[c];
            else if (STRAT == SMEM_LOHI)
                v = (((u64)reinterpret_cast<u32*>(smem)[kLohiCells + c] << 32) | reinterpret_cast<u32*>(smem)[c]) -
                    0x80000000ull;
            else v = reinterpret_cast<u64*>(smem)[c];
            if (v) red_add_u64(reinterpret_cast<uint64_t*>(table) + c, v);
        }
    }
}

// ---- one row, Pow2 split, 32-bit keys, b = 61 (config 1's shape) ------------
// Whole 16-byte vectors of 4 keys (and 4 weights) per lane, two in flight, no
// per-item bounds checks; 1024-thread CTAs so the per-CTA merge of the private
// table into HBM (one red.global per non-zero cell) stays small.
constexpr int kSmallThreads = 1024;

template <int K, int WK, int STRAT>
__device__ __forceinline__ void small_vec(const SketchParams& sp, const u64* c, uint4 kv, const int4& wv,
                                          void* smem) {
    const u32 kk[4] = {kv.x, kv.y, kv.z, kv.w};
    const i32 ww[4] = {wv.x, wv.y, wv.z, wv.w};
    u64 y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = c[K - 1];
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = h61_step32_first(y[u], kk[u], c[K - 2]);
#pragma unroll
    for (int i = K - 3; i >= 0; --i)
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = h61_step32(y[u], kk[u], c[i]);
    const u32 mask = (u32)(sp.width - 1);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        bool neg;  // index = low bits, sign = bit 60 of y mod p (sketch.cpp:13-19)
        const u32 idx = h61_pow2_split(y[u], mask, neg);
        const u64 d = WK == W_NONE ? 1ull : (u64)(i64)ww[u];
        table_add<STRAT>(smem, nullptr, idx, neg ? 0ull - d : d);
    }
}

template <int K, int WK, int STRAT>
__global__ void __launch_bounds__(kSmallThreads, 1) cs_small_k32_kernel(const SketchParams sp,
                                                                      const u32* __restrict__ keys,
                                                                      const void* __restrict__ w, uint64_t n,
                                                                      i64* __restrict__ table) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    void* smem = smem_raw;
    const uint64_t cells = sp.width;
    if (STRAT == SMEM_LOHI) {
        for (uint64_t i = threadIdx.x; i < 2 * kLohiCells; i += kSmallThreads)
            reinterpret_cast<u32*>(smem)[i] = i < kLohiCells ? 0x80000000u : 0u;
    } else {
        for (uint64_t i = threadIdx.x; i < cells; i += kSmallThreads) reinterpret_cast<u32*>(smem)[i] = 0;
    }
    u64 c[K];
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = sp.lo[i];
    __syncthreads();
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    const int4* w4 = reinterpret_cast<const int4*>(w);
    const uint64_t nv = n / 4, stride = (uint64_t)gridDim.x * kSmallThreads;
    const int4 ones = make_int4(1, 1, 1, 1);
    uint64_t i = (uint64_t)blockIdx.x * kSmallThreads + threadIdx.x;
    // four vectors (16 keys) per lane in flight: the loop is otherwise bound by
    // the load latency
    for (; i + 3 * stride < nv; i += 4 * stride) {
        uint4 kv[4];
        int4 wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            kv[u] = ld_stream(k4 + i + u * stride);
            wv[u] = WK == W_NONE ? ones : ld_stream(w4 + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) small_vec<K, WK, STRAT>(sp, c, kv[u], wv[u], smem);
    }
    for (; i + stride < nv; i += 2 * stride) {
        const uint4 ka = ld_stream(k4 + i), kb = ld_stream(k4 + i + stride);
        const int4 wa = WK == W_NONE ? ones : ld_stream(w4 + i);
        const int4 wb = WK == W_NONE ? ones : ld_stream(w4 + i + stride);
        small_vec<K, WK, STRAT>(sp, c, ka, wa, smem);
        small_vec<K, WK, STRAT>(sp, c, kb, wb, smem);
    }
    if (i < nv) small_vec<K, WK, STRAT>(sp, c, ld_stream(k4 + i), WK == W_NONE ? ones : ld_stream(w4 + i), smem);
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // the last n % 4 items
        const uint64_t j = (n & ~3ull) + threadIdx.x;
        u64 y = c[K - 1];
#pragma unroll
        for (int t = K - 2; t >= 0; --t) y = h61_step32(y, keys[j], c[t]);
        const u64 h = h61_finish(y);
        const u64 d = WK == W_NONE ? 1ull : (u64)(i64)reinterpret_cast<const i32*>(w)[j];
        table_add<STRAT>(smem, nullptr, lo32(h) & (u32)(sp.width - 1), ((hi32(h) >> 28) & 1) ? 0ull - d : d);
    }
    __syncthreads();
    for (uint64_t cc = threadIdx.x; cc < cells; cc += kSmallThreads) {
        u64 v;
        if (STRAT == SMEM32) v = (u64)(i64)(i32)reinterpret_cast<u32*>(smem)[cc];
        else
            v = (((u64)reinterpret_cast<u32*>(smem)[kLohiCells + cc] << 32) | reinterpret_cast<u32*>(smem)[cc]) -
                0x80000000ull;
        if (v) red_add_u64(reinterpret_cast<uint64_t*>(table) + cc, v);
    }
}

// ---- K5: exact sum of squares per row, 192-bit accumulation ------------------
struct U192 {
    u64 w0, w1, w2;
};
__device__ __forceinline__ void add192(U192& a, u64 b0, u64 b1, u64 b2) {
    asm("add.cc.u64  %0, %0, %3;\n\t"
        "addc.cc.u64 %1, %1, %4;\n\t"
        "addc.u64    %2, %2, %5;"
        : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
        : "l"(b0), "l"(b1), "l"(b2));
}

// One row is split over gridDim.y CTAs (span cells each); each CTA adds
// its exact 192-bit partial into the row's out[0..2] with carry-propagating
// u64 atomics (integer addition commutes, so the total is exact in any order),
// and the last CTA of the row -- ticket in out[3], zeroed by the launcher --
// applies the reference's saturation and clears the ticket.
constexpr uint32_t kMomThreads = 256, kMomCells = 4096;

__device__ __forceinline__ void atomic_add192(unsigned long long* o, u64 w0, u64 w1, u64 w2) {
    const u64 o0 = atomicAdd(o, (unsigned long long)w0);
    const u64 c0 = o0 + w0 < o0 ? 1 : 0;
    const u64 o1 = atomicAdd(o + 1, (unsigned long long)w1);
    u64 c1 = o1 + w1 < o1 ? 1 : 0;
    if (c0) {
        const u64 o1b = atomicAdd(o + 1, 1ull);
        c1 += o1b + 1 == 0 ? 1 : 0;
    }
    if (w2 + c1) atomicAdd(o + 2, (unsigned long long)(w2 + c1));
}

__global__ void __launch_bounds__(kMomThreads) cs_moments_kernel(const i64* __restrict__ table, uint64_t width,
                                                                 uint64_t span, u64* __restrict__ out) {
    const uint32_t row = blockIdx.x;
    const i64* base = table + (uint64_t)row * width;
    const uint64_t lo = (uint64_t)blockIdx.y * span;
    const uint64_t hi = lo + span < width ? lo + span : width;
    U192 acc = {0, 0, 0};
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kMomThreads) {
        const i64 c = base[i];
        const u64 mag = c < 0 ? 0ull - (u64)c : (u64)c;  // sketch.cpp:149 (INT64_MIN-safe)
        add192(acc, mag * mag, __umul64hi(mag, mag), 0);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const u64 b0 = __shfl_xor_sync(kFull, acc.w0, off);
        const u64 b1 = __shfl_xor_sync(kFull, acc.w1, off);
        const u64 b2 = __shfl_xor_sync(kFull, acc.w2, off);
        add192(acc, b0, b1, b2);
    }
    __shared__ U192 part[kMomThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    U192 t = {0, 0, 0};
    for (int wdx = 0; wdx < (int)(kMomThreads / 32); ++wdx) add192(t, part[wdx].w0, part[wdx].w1, part[wdx].w2);
    u64 s0 = t.w0, s1 = t.w1, s2 = t.w2;
    if (gridDim.y > 1) {  // (one CTA per row: out is written directly, not zeroed first)
        unsigned long long* o = reinterpret_cast<unsigned long long*>(out + 4 * row);
        atomic_add192(o, t.w0, t.w1, t.w2);
        __threadfence();
        if (atomicAdd(o + 3, 1ull) != gridDim.y - 1) return;
        __threadfence();  // the last CTA of the row: every partial is in
        s0 = atomicAdd(o, 0ull);
        s1 = atomicAdd(o + 1, 0ull);
        s2 = atomicAdd(o + 2, 0ull);
    }
    // sketch.cpp:150-154: saturate at 2^128 - 1 and flag it
    const bool sat = s2 != 0;
    out[4 * row + 0] = sat ? ~0ull : s0;
    out[4 * row + 1] = sat ? ~0ull : s1;
    out[4 * row + 2] = sat ? 1 : 0;
    out[4 * row + 3] = 0;
}

__global__ void cs_merge_kernel(u64* __restrict__ dst, const u64* __restrict__ src, uint64_t count) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        dst[i] += src[i];  // sketch.cpp:189-191, wrapping
}

// point_query: lower median over rows of sign * counter (sketch.cpp:170-180)
template <int MODE, typename KeyT>
__global__ void cs_point_query_kernel(const SketchParams sp, const i64* __restrict__ table,
                                      const KeyT* __restrict__ keys, uint64_t n, i64* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 x = (u64)keys[i];
        i64 est[kMaxFamilies * 2];
        uint32_t ne = 0;
        for (uint32_t f = 0; f < sp.families; ++f) {
            const uint32_t subs = sp.splitter == SPLIT_TWO_FOR_ONE ? 2 : 1;
            u64 hlo = 0, hhi = 0;
            if (MODE == M89) hash89<0>(sp, f, x, hlo, hhi);
            else if (MODE == MWIDE) hash_wide_f(sp, f, x, hlo, hhi);
            else hlo = hash_small<MODE, 0>(sp, f, x);
            for (uint32_t s = 0; s < subs; ++s) {
                const uint32_t row = subs * f + s;
                if (row >= sp.rows) break;
                bool neg;
                const u64 idx = MODE == M89     ? split89(sp, hlo, hhi, s, neg)
                                : MODE == MWIDE ? split_wide(sp, hlo, hhi, s, neg)
                                                : split_small(sp, hlo, s, neg);
                const i64 c = table[(u64)row * sp.width + idx];
                est[ne++] = neg ? (i64)(0ull - (u64)c) : c;
            }
        }
        for (uint32_t a = 1; a < ne; ++a) {  // insertion sort, ne <= 32
            const i64 v = est[a];
            int j = (int)a - 1;
            while (j >= 0 && est[j] > v) {
                est[j + 1] = est[j];
                --j;
            }
            est[j + 1] = v;
        }
        out[i] = est[(ne - 1) / 2];
    }
}

int blocks_per_sm_cache(const void* fn, size_t smem) {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, kThreads, smem);
    return v > 0 ? v : 1;
}

template <int K, int WK, int STRAT>
cudaError_t launch_small_k32(const SketchParams& sp, const void* keys, const void* w, uint64_t n, int64_t* table,
                             cudaStream_t s) {
    auto fn = cs_small_k32_kernel<K, WK, STRAT>;
    const size_t smem = STRAT == SMEM_LOHI ? (size_t)kLohiCells * 8 : (size_t)sp.width * 4;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    // one 1024-thread CTA per SM (two when the batch is large): the merge costs
    // one red.global per cell per CTA
    const uint64_t nv = n / 4;
    uint64_t grid = (nv + 4 * kSmallThreads - 1) / (4 * kSmallThreads);
    const uint64_t cap = (uint64_t)sm_count();
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    fn<<<(unsigned)grid, kSmallThreads, smem, s>>>(sp, (const u32*)keys, w, n, table);
    return cudaGetLastError();
}

template <int MODE, int K, typename KeyT, int WK, int STRAT, int FAM = 0>
cudaError_t launch_strat(const SketchParams& sp, const void* keys, const void* w, uint64_t n, int64_t* table,
                         cudaStream_t s, bool aggregate) {
    // one row, Pow2, 32-bit keys, b = 61, k = 4, 16-byte aligned buffers: the vector kernel
    if (MODE == M61_K32 && K == 4 && (STRAT == SMEM32 || STRAT == SMEM_LOHI) && WK != W_I64 &&
        sp.families == 1 && sp.rows == 1 && sp.splitter == SPLIT_POW2 && sp.width <= kLohiCells &&
        ((uintptr_t)keys & 15) == 0 && ((uintptr_t)w & 15) == 0)
        return launch_small_k32<4, WK, STRAT == SMEM32 ? SMEM32 : SMEM_LOHI>(sp, keys, w, n, table, s);
    // one family with the Pow2 splitter (config 1's shape) gets a loop-free body
    if (FAM == 0 && STRAT != GLOBAL && sp.families == 1 && sp.rows == 1 && sp.splitter == SPLIT_POW2)
        return launch_strat<MODE, K, KeyT, WK, STRAT, 1>(sp, keys, w, n, table, s, aggregate);
    auto fn = cs_update_kernel<MODE, K, KeyT, WK, STRAT, FAM>;
    const uint64_t cells = (uint64_t)sp.rows * sp.width;
    const size_t smem = STRAT == GLOBAL      ? 0
                        : STRAT == SMEM_LOHI ? (size_t)kLohiCells * 8
                                             : (size_t)cells * (STRAT == SMEM32 ? 4 : 8);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int per_sm = blocks_per_sm_cache((const void*)fn, smem);
    const uint64_t tile = 32ull * kSlots * kWarps;
    uint64_t grid = (n + tile - 1) / tile;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    fn<<<(unsigned)grid, kThreads, smem, s>>>(sp, (const KeyT*)keys, w, n, table, aggregate ? 1 : 0);
    return cudaGetLastError();
}

template <int MODE, int K, typename KeyT, int WK>
cudaError_t launch_w(const SketchParams& sp, const void* keys, const void* w, uint64_t n, int64_t* table,
                     cudaStream_t s) {
    const uint64_t cells = (uint64_t)sp.rows * sp.width;
    // 32-bit private counters are exact when every increment is +-1 and a CTA
    // sees fewer than 2^31 items; 64-bit otherwise.
    if (WK == W_NONE && cells * 4 <= 64 * 1024 && n < (1ull << 31))
        return launch_strat<MODE, K, KeyT, WK, SMEM32>(sp, keys, w, n, table, s, false);
    // |delta| <= 2^31: exact two-word shared counters on native 32-bit atomics
    if (WK != W_I64 && cells <= kLohiCells)
        return launch_strat<MODE, K, KeyT, WK, SMEM_LOHI>(sp, keys, w, n, table, s, false);
    // 64-bit shared atomics are CAS loops on sm_100: only for int64 weights
    if (cells * 8 <= 64 * 1024) return launch_strat<MODE, K, KeyT, WK, SMEM64>(sp, keys, w, n, table, s, false);
    // large batches: heavy-hitter accumulation in shared memory (|delta| < 2^31 for the
    // exact two-word accumulator), everything else straight to L2
    if (MODE != MWIDE && WK != W_I64 && n >= (1ull << 22))
        return launch_cs_hot(sp, keys, (int)(sizeof(KeyT) * 8), w, WK, n, table, s);
    return launch_strat<MODE, K, KeyT, WK, GLOBAL>(sp, keys, w, n, table, s, WK != W_NONE);
}

template <int MODE, int K, typename KeyT>
cudaError_t launch_k(const SketchParams& sp, const void* keys, const void* w, int w_kind, uint64_t n,
                     int64_t* table, cudaStream_t s) {
    switch (w_kind) {
        case W_NONE: return launch_w<MODE, K, KeyT, W_NONE>(sp, keys, w, n, table, s);
        case W_I32: return launch_w<MODE, K, KeyT, W_I32>(sp, keys, w, n, table, s);
        case W_I64: return launch_w<MODE, K, KeyT, W_I64>(sp, keys, w, n, table, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int MODE, typename KeyT>
cudaError_t launch_mode(const SketchParams& sp, const void* keys, const void* w, int w_kind, uint64_t n,
                        int64_t* table, cudaStream_t s) {
    if (MODE != MGEN && sp.k == 4) return launch_k<MODE, 4, KeyT>(sp, keys, w, w_kind, n, table, s);
    return launch_k<MODE, 0, KeyT>(sp, keys, w, w_kind, n, table, s);
}

}  // namespace

cudaError_t launch_cs_update(const SketchParams& sp, const void* keys, int key_width, const void* w,
                             int w_kind, uint64_t n, int64_t* table, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    // 62 <= b <= 127 (and b = 89 with the arbitrary-width splitters): the generic
    // four-limb Horner and 128-bit splitters
    if ((sp.b > 61 && sp.b != 89) ||
        (sp.b == 89 && sp.splitter != SPLIT_POW2 && sp.splitter != SPLIT_TWO_FOR_ONE)) {
        if (key_width == 32) return launch_mode<MWIDE, u32>(sp, keys, w, w_kind, n, table, s);
        return launch_mode<MWIDE, u64>(sp, keys, w, w_kind, n, table, s);
    }
    if (sp.b == 89) {
        if (key_width == 32) return launch_mode<M89, u32>(sp, keys, w, w_kind, n, table, s);
        return launch_mode<M89, u64>(sp, keys, w, w_kind, n, table, s);
    }
    if (sp.b == 61) {
        if (key_width == 32) return launch_mode<M61_K32, u32>(sp, keys, w, w_kind, n, table, s);
        return launch_mode<M61_K64, u64>(sp, keys, w, w_kind, n, table, s);
    }
    if (sp.b > 61) return cudaErrorInvalidValue;
    if (key_width == 32) return launch_mode<MGEN, u32>(sp, keys, w, w_kind, n, table, s);
    return launch_mode<MGEN, u64>(sp, keys, w, w_kind, n, table, s);
}

cudaError_t launch_cs_moments(const int64_t* table, uint32_t rows, uint64_t width, uint64_t* out,
                              cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    uint64_t span = kMomCells, parts = width ? (width + span - 1) / span : 1;
    if (parts > 65535) {  // huge rows: fewer, longer CTAs (gridDim.y <= 65535)
        span = (width + 65534) / 65535;
        parts = (width + span - 1) / span;
    }
    if (parts > 1) {  // the partials are accumulated in out (the ticket in out[3])
        const cudaError_t e = cudaMemsetAsync(out, 0, (size_t)rows * 4 * sizeof(uint64_t), s);
        if (e != cudaSuccess) return e;
    }
    cs_moments_kernel<<<dim3(rows, (unsigned)parts), kMomThreads, 0, s>>>(table, width, span, out);
    return cudaGetLastError();
}

cudaError_t launch_cs_merge(int64_t* dst, const int64_t* src, uint64_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    uint64_t grid = (count + 255) / 256;
    if (grid > (uint64_t)sm_count() * 8) grid = (uint64_t)sm_count() * 8;
    cs_merge_kernel<<<(unsigned)grid, 256, 0, s>>>((u64*)dst, (const u64*)src, count);
    return cudaGetLastError();
}

cudaError_t launch_cs_point_query(const SketchParams& sp, const int64_t* table, const void* keys, int key_width,
                                  uint64_t n, int64_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + 255) / 256;
    if (grid > (uint64_t)sm_count() * 8) grid = (uint64_t)sm_count() * 8;
    const unsigned g = (unsigned)grid;
    if ((sp.b > 61 && sp.b != 89) ||
        (sp.b == 89 && sp.splitter != SPLIT_POW2 && sp.splitter != SPLIT_TWO_FOR_ONE)) {
        if (key_width == 32) cs_point_query_kernel<MWIDE, u32><<<g, 256, 0, s>>>(sp, table, (const u32*)keys, n, out);
        else cs_point_query_kernel<MWIDE, u64><<<g, 256, 0, s>>>(sp, table, (const u64*)keys, n, out);
    } else if (sp.b == 89) {
        if (key_width == 32) cs_point_query_kernel<M89, u32><<<g, 256, 0, s>>>(sp, table, (const u32*)keys, n, out);
        else cs_point_query_kernel<M89, u64><<<g, 256, 0, s>>>(sp, table, (const u64*)keys, n, out);
    } else if (sp.b == 61) {
        if (key_width == 32) cs_point_query_kernel<M61_K32, u32><<<g, 256, 0, s>>>(sp, table, (const u32*)keys, n, out);
        else cs_point_query_kernel<M61_K64, u64><<<g, 256, 0, s>>>(sp, table, (const u64*)keys, n, out);
    } else {
        if (key_width == 32) cs_point_query_kernel<MGEN, u32><<<g, 256, 0, s>>>(sp, table, (const u32*)keys, n, out);
        else cs_point_query_kernel<MGEN, u64><<<g, 256, 0, s>>>(sp, table, (const u64*)keys, n, out);
    }
    return cudaGetLastError();
}

// ---- batched splitters (sketch.cpp:13-34) ---------------------------------------
// The rule every sketch kernel applies in registers (split_small), exposed on a
// batch of u64 hash values: index into d_index, sign (+1 / -1) into d_sign.
__global__ void split_batch_kernel(const SketchParams sp, const u64* __restrict__ h, uint64_t n,
                                   u64* __restrict__ index, int32_t* __restrict__ sign,
                                   unsigned long long* flags) {
    // domain: h < 2^b (h < 2^b - 1 for the Mersenne splitter, sketch.cpp:32)
    const u64 top = sp.b == 64 ? ~0ull : ((1ull << sp.b) - 1);
    const u64 last = sp.splitter == SPLIT_MERSENNE_ARB ? top - 1 : top;
    unsigned bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 x = ld_nc(h + i);
        bad += x > last;
        bool neg;
        index[i] = split_small(sp, x, 0, neg);
        sign[i] = neg ? -1 : 1;
    }
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicAdd(flags, (unsigned long long)bad);
}

cudaError_t launch_split_batch(const SketchParams& sp, const uint64_t* h, uint64_t n, uint64_t* index,
                               int32_t* sign, unsigned long long* d_flags, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + 255) / 256;
    if (grid > (uint64_t)sm_count() * 8) grid = (uint64_t)sm_count() * 8;
    split_batch_kernel<<<(unsigned)grid, 256, 0, s>>>(sp, h, n, index, sign, d_flags);
    return cudaGetLastError();
}

// ---- delta widening (host API transport) --------------------------------------
// mb200_sketch_process ships deltas over PCIe in the narrowest of i8 / i16 that
// holds every delta of a chunk; this sign-extends them back to the API's weight
// kind before the scatter.  Four deltas per thread, stores coalesced.
template <typename Src, typename Dst>
__global__ void widen_deltas_kernel(const Src* __restrict__ src, Dst* __restrict__ dst, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (i + e < n) dst[i + e] = (Dst)ld_nc(src + i + e);
    }
}

cudaError_t launch_widen_deltas(const void* src, int src_bits, void* dst, int dst_bits, uint64_t n,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t need = (n + 1023) / 1024;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    const int grid = (int)(need < cap ? need : cap);
    if (src_bits == 8 && dst_bits == 32)
        widen_deltas_kernel<<<grid, 256, 0, s>>>((const int8_t*)src, (int32_t*)dst, n);
    else if (src_bits == 8 && dst_bits == 64)
        widen_deltas_kernel<<<grid, 256, 0, s>>>((const int8_t*)src, (int64_t*)dst, n);
    else if (src_bits == 16 && dst_bits == 32)
        widen_deltas_kernel<<<grid, 256, 0, s>>>((const int16_t*)src, (int32_t*)dst, n);
    else if (src_bits == 16 && dst_bits == 64)
        widen_deltas_kernel<<<grid, 256, 0, s>>>((const int16_t*)src, (int64_t*)dst, n);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace mb200
