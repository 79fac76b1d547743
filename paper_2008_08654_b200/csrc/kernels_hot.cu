// kernels_hot.cu -- Count Sketch update for tables larger than shared memory
// (configs 4 and 5: 1 MiB / 2.5 MiB of int64 counters).
//
// Measured on B200 (tools/probe.py): L2 reductions run at ~1.9e11/s whatever
// their width, shared-memory u32 atomics at ~9e11/s, and remote
// (distributed shared memory) atomics at only ~5e10/s -- so the table stays in
// L2 and the lever is the NUMBER of L2 reductions.  Count Sketch is linear:
// the updates of one key can be summed anywhere and applied once.
//
//   1. hh_count  : exact key counts over a sample (the batch's first 2^18 items)
//                  in an open-addressing table in global memory;
//   2. hh_hist /
//      hh_select : the most frequent sampled keys (count >= a threshold picked
//                  from the count histogram so that at most H qualify) form the
//                  hot list, with their sample counts;
//   3. cs_hot    : one 1024-thread CTA per SM keeps the hot keys in a shared-
//                  memory table with an exact 64-bit accumulator per key.  A hit
//                  costs one shared reduction and no hashing.  Misses are
//                  compacted per warp into full-warp batches that run the fused
//                  hash -> split -> red.global path.  Warps pull 128-item tiles
//                  of their CTA's contiguous range from a shared counter, so
//                  they finish together.  Finally each CTA applies every hot key
//                  once (hash -> split -> red).
// The table is bit-identical to the per-item path for ANY hot set (integer
// addition commutes); the hot set only decides how much L2 traffic is saved.
#include <type_traits>

#include "mb200_sketch_dev.cuh"

namespace mb200 {

// per-process counters of the heavy-hitter kernel: items, misses (items sent to
// the fused L2 path), hot keys applied at the end, hot-set size (summed over CTAs)
__device__ unsigned long long g_hot_stats[8];  // [4..7] reserved (always 0)

namespace {

using namespace sk;

constexpr int kHotThreads = 1024;
constexpr int kHotWarps = kHotThreads / 32;
constexpr uint32_t kHotSample = 1u << 18;
constexpr uint32_t kCountLog2 = 20;
constexpr uint32_t kCountSlots = 1u << kCountLog2;
constexpr int kQueue = 64;     // < 32 queued + one slot of 32 misses
constexpr int kTileSlots = 4;  // items per lane per tile
constexpr uint64_t kTile = 32ull * kTileSlots;

template <typename KeyT>
struct HotGeom;
template <>
struct HotGeom<u32> {
    static constexpr uint32_t kLog2 = 14;  // 16384 slots x (4 B key + 8 B sum) = 192 KiB
    static constexpr uint32_t kCap = 8192;
    static constexpr u32 kEmpty = 0xffffffffu;
    using Cas = unsigned;
};
template <>
struct HotGeom<u64> {
    static constexpr uint32_t kLog2 = 13;  // 8192 slots x (8 B key + 8 B sum) = 128 KiB
    static constexpr uint32_t kCap = 4096;
    static constexpr u64 kEmpty = ~0ull;
    using Cas = unsigned long long;
};

__device__ __forceinline__ u32 fmix32(u32 h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    return h ^ (h >> 16);
}
// two independent slot choices from the HIGH bits of multiplicative / mixing hashes
template <uint32_t LOG2>
__device__ __forceinline__ u32 slot1(u32 key) {
    return (key * 0x9E3779B1u) >> (32 - LOG2);
}
template <uint32_t LOG2>
__device__ __forceinline__ u32 slot2(u32 key) {
    return fmix32(key) >> (32 - LOG2);
}
template <uint32_t LOG2>
__device__ __forceinline__ u32 slot1(u64 key) {
    return (u32)(mix64(key) >> (64 - LOG2));
}
template <uint32_t LOG2>
__device__ __forceinline__ u32 slot2(u64 key) {
    return (u32)(mix64(key) >> 20) & ((1u << LOG2) - 1);
}

template <typename KeyT>
__global__ void hh_count_kernel(const KeyT* __restrict__ keys, uint64_t n, KeyT* tk, u32* tc) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const KeyT key = ld_nc(keys + i);
        if (key == G::kEmpty) continue;
        u32 h = slot1<kCountLog2>(key);
        for (;;) {
            KeyT cur = tk[h];
            if (cur == G::kEmpty) cur = (KeyT)atomicCAS(reinterpret_cast<C*>(tk + h), (C)G::kEmpty, (C)key);
            if (cur == G::kEmpty || cur == key) {
                atomicAdd(tc + h, 1u);
                break;
            }
            h = (h + 1) & (kCountSlots - 1);
        }
    }
}

__global__ void hh_hist_kernel(const u32* __restrict__ tc, u32* hist) {
    __shared__ u32 sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < kCountSlots; s += gridDim.x * blockDim.x) {
        const u32 c = tc[s];
        if (c) atomicAdd(&sh[c < 255 ? c : 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

template <typename KeyT>
__global__ void hh_select_kernel(const KeyT* __restrict__ tk, const u32* __restrict__ tc, const u32* __restrict__ hist,
                                 u32 cap, KeyT* hot, u32* hot_cnt, u32* hot_count) {
    __shared__ u32 thr;
    if (threadIdx.x == 0) {  // smallest threshold >= 2 whose tail fits the shared table
        u32 tail = 0, c = 255;
        for (; c >= 2; --c) {
            if (tail + hist[c] > cap) break;
            tail += hist[c];
        }
        thr = c + 1;
    }
    __syncthreads();
    const u32 t = thr;
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < kCountSlots; s += gridDim.x * blockDim.x) {
        const u32 c = tc[s];
        if (c >= t) {
            const u32 idx = atomicAdd(hot_count, 1u);
            if (idx < cap) {
                hot[idx] = tk[s];
                hot_cnt[idx] = c;
            }
        }
    }
}

// Exact 64-bit accumulation in two u32 words (|d| <= 2^31).  sm_100 has no
// native 64-bit shared-memory add (atomicAdd on u64 in shared memory compiles
// to an ATOMS.CAST.SPIN.64 loop, which serialises on hot keys: 101 ms instead
// of 13 ms on config 5), so: the low word carries a 2^31 bias, so a sum hovering
// around zero never wraps, and the high word counts the wraps.
__device__ __forceinline__ void hot_accumulate(u32* lo, u32* hi, u32 h, i32 d) {
    const u32 dd = (u32)d;
    const u32 old = atomicAdd(lo + h, dd);
    const u32 nw = old + dd;
    const int carry = d >= 0 ? (int)(nw < old) : -(int)(nw > old);
    if (carry) atomicAdd(hi + h, (u32)carry);
}

template <int WK>
__device__ __forceinline__ i32 load_w32(const void* w, uint64_t i) {
    if (WK == W_NONE) return 1;
    return ld_nc(reinterpret_cast<const i32*>(w) + i);
}

template <int MODE, int K, typename KeyT, int WK>
__global__ void __launch_bounds__(kHotThreads, 1)
    cs_hot_kernel(const SketchParams sp, const KeyT* __restrict__ keys, const void* __restrict__ w, uint64_t n,
                  i64* __restrict__ table, const KeyT* __restrict__ hot, const u32* __restrict__ hot_cnt,
                  const u32* __restrict__ hot_count) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    constexpr uint32_t S = 1u << G::kLog2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KeyT* hk = reinterpret_cast<KeyT*>(smem_raw);
    u32* lo = reinterpret_cast<u32*>(hk + S);
    u32* hi = lo + S;
    KeyT* qk = reinterpret_cast<KeyT*>(hi + S);
    i32* qd = reinterpret_cast<i32*>(qk + kHotWarps * kQueue);
    __shared__ u32 s_next;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    KeyT* wqk = qk + warp * kQueue;
    i32* wqd = qd + warp * kQueue;

    for (uint32_t s = threadIdx.x; s < S; s += kHotThreads) {
        hk[s] = G::kEmpty;
        lo[s] = 0x80000000u;
        hi[s] = 0;
    }
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    // Two-choice table, one key per slot: a key goes to slot1 if free, else to
    // slot2 if free, else it stays cold (exactness never depends on the hot set).
    // Slots are never freed, so a lookup whose slot1 is empty is a miss without
    // touching slot2.  Hottest keys are placed first so they own their slot1.
    const u32 nhot = min(*hot_count, G::kCap);
    const u32 bands[3] = {64u, 8u, 0u};
    u32 upper = 0xffffffffu;
    for (int r = 0; r < 3; ++r) {
        for (u32 j = threadIdx.x; j < nhot; j += kHotThreads) {
            const u32 c = hot_cnt[j];
            if (c < bands[r] || c >= upper) continue;
            const KeyT key = hot[j];
            if ((KeyT)atomicCAS(reinterpret_cast<C*>(hk + slot1<G::kLog2>(key)), (C)G::kEmpty, (C)key) != G::kEmpty)
                atomicCAS(reinterpret_cast<C*>(hk + slot2<G::kLog2>(key)), (C)G::kEmpty, (C)key);
        }
        upper = bands[r];
        __syncthreads();
    }

    const uint64_t lo_item = n * blockIdx.x / gridDim.x, hi_item = n * (blockIdx.x + 1) / gridDim.x;
    const uint64_t ntiles = (hi_item - lo_item + kTile - 1) / kTile;
    int qn = 0;
    unsigned misses = 0;
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(&s_next, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= ntiles) break;
        const uint64_t base = lo_item + (uint64_t)t * kTile;
        KeyT kx[kTileSlots];
        i32 dx[kTileSlots];
#pragma unroll
        for (int u = 0; u < kTileSlots; ++u) {
            const uint64_t i = base + u * 32 + lane;
            const bool v = i < hi_item;
            kx[u] = v ? ld_nc(keys + i) : G::kEmpty;
            dx[u] = v ? load_w32<WK>(w, i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kTileSlots; ++u) {
            const bool valid = base + u * 32 + lane < hi_item;
            const KeyT key = kx[u];
            u32 h = slot1<G::kLog2>(key);
            KeyT cur = hk[h];
            if (cur != key && cur != G::kEmpty) {
                h = slot2<G::kLog2>(key);
                cur = hk[h];
            }
            const bool hit = cur == key && key != G::kEmpty;
            if (hit) hot_accumulate(lo, hi, h, dx[u]);
            const bool miss = valid && !hit;
            const unsigned m = __ballot_sync(kFull, miss);
            if (miss) {
                const int pos = qn + __popc(m & ((1u << lane) - 1));
                wqk[pos] = key;
                wqd[pos] = dx[u];
            }
            qn += __popc(m);
            misses += __popc(m);
            __syncwarp();
            if (qn >= 32) {  // a full warp of misses
                process_item<MODE, K, GLOBAL>(sp, (u64)wqk[lane], (i64)wqd[lane], nullptr, table);
                __syncwarp();
                if (lane < qn - 32) {
                    wqk[lane] = wqk[32 + lane];
                    wqd[lane] = wqd[32 + lane];
                }
                __syncwarp();
                qn -= 32;
            }
        }
    }
    if (lane < qn) process_item<MODE, K, GLOBAL>(sp, (u64)wqk[lane], (i64)wqd[lane], nullptr, table);
    __syncthreads();
    unsigned flushed = 0;
    for (uint32_t s = threadIdx.x; s < S; s += kHotThreads) {
        if (hk[s] == G::kEmpty) continue;
        const u64 v = (((u64)hi[s] << 32) | lo[s]) - 0x80000000ull;
        if (v) {
            process_item<MODE, K, GLOBAL>(sp, (u64)hk[s], (i64)v, nullptr, table);
            ++flushed;
        }
    }
    // instrumentation for the L2-reduction roofline (mb200_hot_stats)
    if (lane == 0) atomicAdd(&g_hot_stats[1], (unsigned long long)misses);
    flushed = __reduce_add_sync(kFull, flushed);
    if (lane == 0) atomicAdd(&g_hot_stats[2], (unsigned long long)flushed);
    if (threadIdx.x == 0) {
        atomicAdd(&g_hot_stats[0], (unsigned long long)(hi_item - lo_item));
        atomicAdd(&g_hot_stats[3], (unsigned long long)nhot);
    }
}

template <int MODE, int K, typename KeyT, int WK>
cudaError_t launch_hot(const SketchParams& sp, const void* keys, const void* w, uint64_t n, int64_t* table,
                       cudaStream_t s) {
    using G = HotGeom<KeyT>;
    const uint64_t m = n < kHotSample ? n : kHotSample;
    const size_t tk_bytes = (size_t)kCountSlots * sizeof(KeyT), tc_bytes = (size_t)kCountSlots * 4;
    const size_t misc = 256 * 4 + 16;
    const size_t hot_bytes = (size_t)G::kCap * (sizeof(KeyT) + 4);
    unsigned char* ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, tk_bytes + tc_bytes + misc + hot_bytes, s);
    if (e != cudaSuccess) return e;
    KeyT* tk = reinterpret_cast<KeyT*>(ws);
    u32* tc = reinterpret_cast<u32*>(ws + tk_bytes);
    u32* hist = tc + kCountSlots;
    u32* hot_count = hist + 256;
    KeyT* hot = reinterpret_cast<KeyT*>(ws + tk_bytes + tc_bytes + misc);
    u32* hot_cnt = reinterpret_cast<u32*>(hot + G::kCap);
    cudaMemsetAsync(tk, 0xff, tk_bytes, s);
    cudaMemsetAsync(tc, 0, tc_bytes + misc, s);
    const int sms = sm_count();
    hh_count_kernel<KeyT><<<sms * 4, 256, 0, s>>>(reinterpret_cast<const KeyT*>(keys), m, tk, tc);
    hh_hist_kernel<<<sms, 256, 0, s>>>(tc, hist);
    hh_select_kernel<KeyT><<<sms, 256, 0, s>>>(tk, tc, hist, G::kCap, hot, hot_cnt, hot_count);
    auto fn = cs_hot_kernel<MODE, K, KeyT, WK>;
    const size_t smem = ((size_t)sizeof(KeyT) + 8) << G::kLog2;
    const size_t qbytes = (size_t)kHotWarps * kQueue * (sizeof(KeyT) + 4);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + qbytes));
    if (e == cudaSuccess) {
        uint64_t grid = (n + kTile * kHotWarps - 1) / (kTile * kHotWarps);
        if (grid > (uint64_t)sms) grid = sms;
        fn<<<(unsigned)grid, kHotThreads, smem + qbytes, s>>>(sp, reinterpret_cast<const KeyT*>(keys), w, n, table,
                                                              hot, hot_cnt, hot_count);
        e = cudaGetLastError();
    }
    cudaFreeAsync(ws, s);
    return e;
}

template <int MODE, typename KeyT>
cudaError_t launch_mode(const SketchParams& sp, const void* keys, const void* w, int w_kind, uint64_t n,
                        int64_t* table, cudaStream_t s) {
    const bool k4 = MODE != MGEN && sp.k == 4;
    if (w_kind == W_NONE)
        return k4 ? launch_hot<MODE, 4, KeyT, W_NONE>(sp, keys, w, n, table, s)
                  : launch_hot<MODE, 0, KeyT, W_NONE>(sp, keys, w, n, table, s);
    if (w_kind == W_I32)
        return k4 ? launch_hot<MODE, 4, KeyT, W_I32>(sp, keys, w, n, table, s)
                  : launch_hot<MODE, 0, KeyT, W_I32>(sp, keys, w, n, table, s);
    return cudaErrorInvalidValue;
}

// Keep the default stream-ordered pool's memory between calls: the hot path
// allocates its ~12 MiB workspace per call with cudaMallocAsync.
void retain_pool() {
    static bool done[64] = {false};
    const int dev = device_id();
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

}  // namespace

cudaError_t hot_stats(uint64_t out[8], bool reset) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && out) e = cudaMemcpyFromSymbol(out, g_hot_stats, sizeof(g_hot_stats));
    if (e == cudaSuccess && reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        e = cudaMemcpyToSymbol(g_hot_stats, z, sizeof(z));
    }
    return e;
}

cudaError_t launch_cs_hot(const SketchParams& sp, const void* keys, int key_width, const void* w, int w_kind,
                          uint64_t n, int64_t* table, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    retain_pool();
    if (sp.b == 89) {
        if (key_width == 32) return launch_mode<M89, u32>(sp, keys, w, w_kind, n, table, s);
        return launch_mode<M89, u64>(sp, keys, w, w_kind, n, table, s);
    }
    if (sp.b == 61) {
        if (key_width == 32) return launch_mode<M61_K32, u32>(sp, keys, w, w_kind, n, table, s);
        return launch_mode<M61_K64, u64>(sp, keys, w, w_kind, n, table, s);
    }
    if (key_width == 32) return launch_mode<MGEN, u32>(sp, keys, w, w_kind, n, table, s);
    return launch_mode<MGEN, u64>(sp, keys, w, w_kind, n, table, s);
}

}  // namespace mb200
