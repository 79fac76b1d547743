// kernels_hot.cu -- Count Sketch update for tables larger than shared memory
// (configs 4 and 5: 1 MiB / 2.5 MiB of int64 counters).
//
// Measured on B200 (tools/probe.py): L2 reductions run at ~1.9e11/s whatever
// their width, shared-memory u32 atomics at ~9e11/s, and remote
// (distributed shared memory) atomics at only ~5e10/s -- so the table stays in
// L2 and the lever is the NUMBER of L2 reductions.  Count Sketch is linear:
// the updates of one key can be summed anywhere and applied once.
//
//   1. hh_count  : exact key counts over a sample (the batch's first n/128
//                  items, clamped to [2^18, 2^22]) in an open-addressing table
//                  in global memory;
//   2. hh_hist /
//      hh_select : the most frequent sampled keys (count >= a threshold picked
//                  from the count histogram so that at most H qualify) form the
//                  hot list, written in count order, hottest first;
//      hh_layout : one CTA places the hot list in that order in the two-choice
//                  shared table layout every CTA copies (one level of cuckoo
//                  displacement; ~46K of 61440 candidates in 53248 slots);
//                  hh_slots writes the slot words (tags) the CTAs copy.
//                  (1-2: kernels_hotprep.cu)
//   3. cs_hot    : one 1024-thread CTA per SM keeps the hot keys in a shared-
//                  memory table with an exact 64-bit accumulator per key (a
//                  16-bit shared cell + a wrap counter in HBM).  A hit costs one
//                  shared atomic and no hashing.  Misses are compacted per warp
//                  into full-warp batches of 32 (key, delta) pairs that are
//                  hashed, split and sent to L2 as red.global (or, binned
//                  strategy, appended to a miss buffer in HBM).  Warps pull
//                  256-item tiles of their CTA's contiguous range from a shared
//                  counter, so they finish together.  Each CTA adds its slot
//                  sums into per-slot totals, and hh_merge applies every hot
//                  key once (hash -> split -> red).
//   4. cs_bin    : (opt-in binned strategy) the misses (or, when the sample
//                  shows no heavy hitters, the raw stream -- pass 3 is then
//                  skipped) are hashed, split and turned into 4-byte entries
//                  (16-bit cell | 16-bit signed delta) that are staged per
//                  (row, 65536-cell bin) in shared memory and written to per-bin
//                  buffers in HBM in 16-byte groups (one global atomic per bin
//                  per round).
//   5. cs_accum  : one CTA per (bin, part) sums its bin's entries into an exact
//                  shared-memory table of packed 16-bit cells and merges it into
//                  the L2 table with one red.global per non-zero cell.
// Passes 4-5 replace ~rows L2 reductions per missed item by 8 bytes of
// streaming HBM traffic per row update (measured slower than the direct path
// on config 5).  Anything that does not fit a staging buffer, a bin,
// the miss buffer or the 16-bit delta field takes the direct red.global path.
// Streams without heavy hitters whose table fits shared memory as bytes (unit
// deltas) take the private byte tables instead (cs_private_kernel, and config
// 4's shape cs_private89_kernel, mb200_private89.cuh).
// The table is bit-identical to the per-item path for ANY hot set (integer
// addition commutes); the hot set only decides how much L2 traffic is saved.
#include <type_traits>
#include <utility>
#include <vector>

#include "mb200_hot_geom.cuh"
#include "mb200_hotprep.h"
#include "mb200_sketch_dev.cuh"

namespace mb200 {

// per-process counters of the heavy-hitter pipeline: [0] items, [1] misses (items
// not accumulated in a hot table), [2] hot keys applied (once per call, by
// hh_merge_kernel), [3] hot keys placed in the shared table, [4] entries written
// to HBM bins, [5] row updates that took the direct red.global path,
// [6] red.global merges (per-slot sums of every CTA, bin tables), [7] batches
// that ran in raw mode (no hot pass)
__device__ unsigned long long g_hot_stats[8];

}  // namespace mb200

#include "mb200_private89.cuh"

namespace mb200 {
namespace {

using namespace sk;



constexpr int kHotThreads = 1024;
constexpr int kHotWarps = kHotThreads / 32;
// sample = n / 128 items, clamped to [2^18, 2^22] (a shard of a multi-GPU run
// gets a 2^21-item sample from 2^28 items); count table = 1 slot per sampled item
constexpr uint32_t kMinSample = 1u << 18, kMaxSample = 1u << 22;
constexpr int kQueue = 64;     // < 32 queued + one slot of 32 misses
constexpr uint32_t kMissChunk = 1024;  // miss-buffer slots a warp reserves at once

// a queued miss: key and delta side by side (one 8-byte shared store for u32 keys)
template <typename KeyT>
struct alignas(sizeof(KeyT) * 2) QEnt {
    KeyT k;
    i32 d;
};
// words of a CTA's cell storage (what it hands to hh_merge_kernel through its
// scratch area): the tagged table's slot words, else the packed 16-bit cells
template <typename KeyT>
struct HotCells {
    static constexpr u32 kWords = HotGeom<KeyT>::kTagged ? HotGeom<KeyT>::kSlots : HotGeom<KeyT>::kSlots / 2;
    static_assert(kWords % 4 == 0, "16-byte copies");
};

// Exact 64-bit accumulation in a 16-bit shared cell; the cell's wraps (units of
// 2^16) go straight into its slot's total in HBM.  sm_100 has no 16-bit (or
// native 64-bit) shared atomic add, so two cells share a 32-bit word: cell h is
// bits 16 (h & 1) of word h >> 1, biased by 2^15 so a sum hovering around zero
// rarely leaves [0, 2^16).  The delta is added to the word shifted to its cell.
// Every atomic change x of a cell whose value was c adds 2^16 floor((c + x) /
// 2^16) to the slot's total slot_sum[h] (shared by all CTAs: every CTA holds
// the same layout, and the totals are sums anyway), which keeps
//   sum over CTAs of (cell - bias) + slot_sum = sum of the slot's deltas
// exactly, under any interleaving: a low-cell add that leaves [0, 2^16) also
// carries w into the high cell (recorded against the high cell's value at that
// same atomic), and w is then taken back out of the high cell by a second
// atomic (recorded against its value then).  The range test is a 32-bit
// compare: c + x as a mathematical value lies in [-2^31, 2^31 + 2^16), so its
// u32 image exceeds 0xFFFF exactly when it is outside [0, 2^16).  Halving the
// cell width fits 35840 instead of 24576 slots into shared memory.
__device__ __forceinline__ void hot_accumulate(u32* cells, u64* slot_sum, u32 h, i32 d) {
    typedef unsigned long long ull;
    const u32 sh = (h & 1u) << 4;
    u32* word = cells + (h >> 1);
    const u32 old = atomicAdd(word, (u32)d << sh);
    if (((old >> sh) & 0xFFFFu) + (u32)d > 0xFFFFu) {  // rare: the cell left [0, 2^16)
        const i64 t = (i64)((old >> sh) & 0xFFFFu) + d;
        const i64 w = t >> 16;
        atomicAdd(reinterpret_cast<ull*>(slot_sum + h), (ull)(w << 16));
        if (sh == 0) {  // w also entered the high cell (slot h + 1): take it back
            const i64 w1 = ((i64)(old >> 16) + w) >> 16;
            const u32 old2 = atomicAdd(word, (u32)(-(i32)w) << 16);
            const i64 w2 = ((i64)(old2 >> 16) - w) >> 16;
            if (w1 + w2) atomicAdd(reinterpret_cast<ull*>(slot_sum + h + 1), (ull)((w1 + w2) << 16));
        }
    }
}

// The tagged table's cell (bits 18-31 of the slot word, 2^13-biased): one
// shared atomic; a cell that leaves [0, 2^14) records 2^14 floor((c + d) / 2^14)
// into the slot's total (its carry left the word; the tag below is untouched).
// The range test is the 32-bit compare of hot_accumulate.
__device__ __forceinline__ void tag_accumulate(u32* words, u64* slot_sum, u32 h, i32 d) {
    typedef unsigned long long ull;
    const u32 old = atomicAdd(words + h, (u32)d << kCellShift);
    const u32 c = old >> kCellShift;
    if (c + (u32)d > 0x3fffu) {  // rare
        const i64 t = (i64)c + d;
        atomicAdd(reinterpret_cast<ull*>(slot_sum + h), (ull)((t >> 14) << 14));
    }
}

// Raw mode: the hot set covers under 30% of the sample, so the hot pass would
// mostly copy the stream into the miss buffer; the binning pass then reads the
// stream itself.  Every kernel of the pipeline evaluates this on the same inputs.
__device__ __forceinline__ bool raw_mode(const u32* hot_sum, uint32_t sample) {
    return (uint64_t)*hot_sum * 10 < (uint64_t)sample * 3;
}

// where a missed item goes: the HBM miss buffer (binned later) or, when the
// buffer is full, the direct hash -> split -> red.global path
template <typename KeyT>
struct MissBuf {
    KeyT* keys;
    i32* deltas;
    unsigned long long* count;  // items stored (multiple of 32; may exceed cap)
    uint64_t cap;               // capacity, multiple of 32
};

template <int WK>
__device__ __forceinline__ i32 load_w32(const void* w, uint64_t i) {
    if (WK == W_NONE) return 1;
    return ld_nc(reinterpret_cast<const i32*>(w) + i);
}

enum SplitC { SPC_POW2 = 0, SPC_TFO = 1, SPC_ANY = 2 };  // compile-time splitter (Pow2 / two-for-one / other)

// bucket index (< 2^32) and sign of sub-row s, splitter known
// at compile time where it is Pow2 / two-for-one (sketch.cpp:13-19)
template <int MODE, int SPL>
__device__ __forceinline__ u32 split_c(const SketchParams& sp, u64 hlo, u64 hhi, uint32_t s, bool& neg) {
    if (MODE == M89) return (u32)split89(sp, hlo, hhi, s, neg);
    if (MODE != MGEN && SPL == SPC_POW2) {  // b = 61: sign = bit 60, index = low bits
        neg = (hi32(hlo) >> 28) & 1;
        return lo32(hlo) & (u32)(sp.width - 1);
    }
    if (MODE != MGEN && SPL == SPC_TFO) {
        neg = (hlo >> (60 - s)) & 1;
        return (u32)(hlo >> (sp.lw * s)) & (u32)(sp.width - 1);
    }
    return (u32)split_small(sp, hlo, s, neg);
}

// One item straight to L2: every family, every sub-row, hash -> split ->
// red.global (process_item with the splitter fixed at compile time where it is
// Pow2 or two-for-one; sketch.cpp:133-140).
template <int MODE, int K, int SPL>
__device__ __forceinline__ void rows_direct(const SketchParams& sp, u64 x, i64 delta, i64* table) {
    if (SPL == SPC_ANY) {
        process_item<MODE, K, GLOBAL>(sp, x, delta, nullptr, table);
        return;
    }
    const u64 dp = (u64)delta, dn = 0ull - dp;
    constexpr uint32_t subs = SPL == SPC_TFO ? 2 : 1;
    uint64_t* base = reinterpret_cast<uint64_t*>(table);
#pragma unroll 1
    for (uint32_t f = 0; f < sp.families; ++f) {
        if constexpr ((MODE == M61_K32 || MODE == M61_K64) && K > 0 && SPL == SPC_POW2) {
            // Pow2 split straight from the lazily reduced Horner value
            bool neg;
            const u32 idx = h61_pow2_split(hash61_lazy<MODE, K>(sp, f, x), (u32)(sp.width - 1), neg);
            red_add_u64(base + (u64)f * sp.width + idx, neg ? dn : dp);
            continue;
        }
        u64 hlo, hhi = 0;
        if (MODE == M89) hash89<K>(sp, f, x, hlo, hhi);
        else hlo = hash_small<MODE, K>(sp, f, x);
#pragma unroll
        for (uint32_t s = 0; s < subs; ++s) {
            const uint32_t row = subs * f + s;
            if (row >= sp.rows) break;
            bool neg;
            const u32 idx = split_c<MODE, SPL>(sp, hlo, hhi, s, neg);
            red_add_u64(base + (u64)row * sp.width + idx, neg ? dn : dp);
        }
    }
}

// a full warp of misses: the direct path
template <int MODE, int K, int SPL, typename KeyT>
__device__ __forceinline__ void misses_direct(const SketchParams& sp, KeyT key, i32 d, bool valid, i64* table) {
    if (valid) rows_direct<MODE, K, SPL>(sp, (u64)key, (i64)d, table);
}

// 16-byte vector of keys / weights (4 u32 or 2 u64 keys per vector)
template <typename KeyT>
struct KeyVec;
template <>
struct KeyVec<u32> {
    static constexpr int N = 4;
    uint4 v;
    __device__ __forceinline__ void load(const u32* p) { v = ld_stream(reinterpret_cast<const uint4*>(p)); }
    __device__ __forceinline__ u32 operator[](int e) const { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
};
template <>
struct KeyVec<u64> {
    static constexpr int N = 2;
    ulonglong2 v;
    __device__ __forceinline__ void load(const u64* p) { v = ld_stream(reinterpret_cast<const ulonglong2*>(p)); }
    __device__ __forceinline__ u64 operator[](int e) const { return e == 0 ? v.x : v.y; }
};
template <int N, int WK>
struct WVec {
    i32 d[N];
    __device__ __forceinline__ void load(const void* w, uint64_t i) {
        if (WK == W_NONE) {
#pragma unroll
            for (int e = 0; e < N; ++e) d[e] = 1;
        } else if (N == 4) {
            const int4 v = ld_stream(reinterpret_cast<const int4*>(reinterpret_cast<const i32*>(w) + i));
            d[0] = v.x;
            d[1] = v.y;
            d[2] = v.z;
            d[3] = v.w;
        } else {
            const long long v = __ldcs(reinterpret_cast<const long long*>(reinterpret_cast<const i32*>(w) + i));
            d[0] = (i32)(u32)v;
            d[1] = (i32)(u32)((u64)v >> 32);
        }
    }
};

template <int MODE, int K, int SPL, typename KeyT, int WK, bool BUF>
__global__ void __launch_bounds__(kHotThreads, 1)
    cs_hot_kernel(const SketchParams sp, const KeyT* __restrict__ keys, const void* __restrict__ w, uint64_t n,
                  i64* __restrict__ table, const KeyT* __restrict__ layout, const u32* __restrict__ tags,
                  u64* __restrict__ slot_sum, const u32* __restrict__ hot_sum, uint32_t sample,
                  const MissBuf<KeyT> mb, bool vec_ok, const u32* __restrict__ priv_go, u32* __restrict__ scratch) {
    if (priv_go && *priv_go == 0) return;  // cs_private_kernel took this stream
    using G = HotGeom<KeyT>;
    using KV = KeyVec<KeyT>;
    // keys hh_layout_kernel placed (its word follows hot_sum's; instrumentation)
    if (blockIdx.x == 0 && threadIdx.x == 0 && hot_sum[7]) atomicAdd(&g_hot_stats[3], (unsigned long long)hot_sum[7]);
    constexpr int kV = KV::N;          // items per vector
    constexpr int kVT = 8 / kV;        // vectors per lane per tile
    constexpr int kIt = kV * kVT;      // items per lane per tile (8 u32 / 4 u64)
    constexpr uint64_t kT = 32ull * kIt;
    constexpr uint32_t S = G::kSlots;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // tagged (u32 keys): S slot words; else S keys + S 16-bit cells
    KeyT* hk = reinterpret_cast<KeyT*>(smem_raw);
    u32* tw = reinterpret_cast<u32*>(smem_raw);
    static_assert(S % 2 == 0, "two cells per word");
    u32* cells = reinterpret_cast<u32*>(hk + S);  // S 16-bit cells (untagged)
    QEnt<KeyT>* q = reinterpret_cast<QEnt<KeyT>*>(G::kTagged ? reinterpret_cast<unsigned char*>(tw + S)
                                                             : reinterpret_cast<unsigned char*>(cells + S / 2));
    __shared__ u32 s_next;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 lanes_below;  // evaluated once (a volatile read is never rematerialised)
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(lanes_below));
    u32 wq_off;  // this warp's queue offset, held in a register (not re-derived from tid per item)
    asm volatile("mov.u32 %0, %1;" : "=r"(wq_off) : "r"((u32)warp * kQueue));
    QEnt<KeyT>* wq = q + wq_off;
    // CTAs own whole tiles (16-byte vector loads) and a share of the < kT tail
    // items (scalar loads; everything, when the buffers are not 16-byte aligned)
    const uint64_t ntiles_all = vec_ok ? n / kT : 0;
    const uint64_t t_lo = ntiles_all * blockIdx.x / gridDim.x, t_hi = ntiles_all * (blockIdx.x + 1) / gridDim.x;
    const uint64_t rest = n - ntiles_all * kT;
    const uint64_t tail_lo = ntiles_all * kT + rest * blockIdx.x / gridDim.x;
    const uint64_t tail_hi = ntiles_all * kT + rest * (blockIdx.x + 1) / gridDim.x;
    if (BUF && raw_mode(hot_sum, sample)) {  // the binning pass reads the stream itself
        if (threadIdx.x == 0) {
            const uint64_t cnt = (t_hi - t_lo) * kT + (tail_hi - tail_lo);
            atomicAdd(&g_hot_stats[0], (unsigned long long)cnt);
            atomicAdd(&g_hot_stats[1], (unsigned long long)cnt);
            if (blockIdx.x == 0) atomicAdd(&g_hot_stats[7], 1ull);
        }
        return;
    }

    // every CTA holds the same table layout (hh_layout_kernel), so the slot sums
    // of all CTAs can be merged per slot before the keys are hashed
    // (16-byte loads, kCopyB of a thread in flight at once: the copy costs a few L2
    // latencies, not one per slot -- it is a fixed cost of every call)
    constexpr u32 kCopyB = 7;
    if constexpr (G::kTagged) {
        static_assert(S % 4 == 0, "16-byte copies");
        const uint4* src = reinterpret_cast<const uint4*>(tags);
        uint4* dst = reinterpret_cast<uint4*>(tw);
        constexpr u32 kBias = kCellBias << kCellShift;
        for (u32 j0 = threadIdx.x; j0 < S / 4; j0 += kCopyB * kHotThreads) {
            uint4 v[kCopyB];
#pragma unroll
            for (u32 u = 0; u < kCopyB; ++u)
                if (j0 + u * kHotThreads < S / 4) v[u] = __ldg(src + j0 + u * kHotThreads);
#pragma unroll
            for (u32 u = 0; u < kCopyB; ++u)
                if (j0 + u * kHotThreads < S / 4)
                    dst[j0 + u * kHotThreads] = make_uint4(v[u].x | kBias, v[u].y | kBias, v[u].z | kBias, v[u].w | kBias);
        }
    } else {
        static_assert((S * sizeof(KeyT)) % 16 == 0, "16-byte copies");
        constexpr u32 kVecs = S * sizeof(KeyT) / 16;
        const uint4* src = reinterpret_cast<const uint4*>(layout);
        uint4* dst = reinterpret_cast<uint4*>(hk);
        for (u32 j0 = threadIdx.x; j0 < kVecs; j0 += kCopyB * kHotThreads) {
            uint4 v[kCopyB];
#pragma unroll
            for (u32 u = 0; u < kCopyB; ++u)
                if (j0 + u * kHotThreads < kVecs) v[u] = __ldg(src + j0 + u * kHotThreads);
#pragma unroll
            for (u32 u = 0; u < kCopyB; ++u)
                if (j0 + u * kHotThreads < kVecs) dst[j0 + u * kHotThreads] = v[u];
        }
        for (uint32_t s = threadIdx.x; s < S / 2; s += kHotThreads) cells[s] = 0x80008000u;
    }
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();

    int qn = 0;
    unsigned misses = 0, direct = 0;
    unsigned long long wbase = 0;  // this warp's reserved miss-buffer slots [wbase + wfill, wbase + kMissChunk)
    uint32_t wfill = kMissChunk;
    // one item: hot-table hit -> shared accumulation; miss -> the warp's queue,
    // and a full queue of 32 -> the miss buffer (warp-uniform call)
    auto item = [&](KeyT key, i32 d, bool valid) {
        // both slots probed speculatively (no divergent second probe); a key never
        // sits in its slot2 unless its slot1 was taken first, so this is exact
        bool hit;
        if constexpr (G::kTagged) {  // (slot, choice, tag) is the key; empty slots hold a marker
            // the two choices' products give both the slots (high bits) and the tags
            // (low 17 bits); the chosen slot is selected as a shared-memory address
            const u32 p1 = (u32)key * 0x9E3779B1u, p2 = ((u32)key ^ ((u32)key >> 15)) * 0x2C1B3C6Du;
            u32* a1 = tw + slot_of<S>(p1);
            u32* a2 = tw + slot_of<S>(p2);
            const bool m1 = (*a1 & kTagMask) == (p1 & 0x1ffffu);
            const bool m2 = (*a2 & kTagMask) == ((p2 & 0x1ffffu) | 0x20000u);
            hit = valid && (m1 || m2);
            if (hit) {
                u32* a = m1 ? a1 : a2;
                tag_accumulate(tw, slot_sum, (u32)(a - tw), d);
            }
        } else {  // empty slots hold foreign keys
            const u32 h1 = slot1<S>(key), h2 = slot2<S>(key);
            const bool m1 = hk[h1] == key, m2 = hk[h2] == key;
            hit = valid && (m1 || m2);
            if (hit) hot_accumulate(cells, slot_sum, m1 ? h1 : h2, d);
        }
        const bool miss = valid && !hit;
        const unsigned m = __ballot_sync(kFull, miss);
        if (miss) {
            const int pos = qn + __popc(m & lanes_below);
            wq[pos] = QEnt<KeyT>{key, d};  // one 8-byte store (u32 keys)
        }
        qn += __popc(m);
        misses += __popc(m);
        if (!BUF && qn >= 32) {  // a full warp of misses -> hash, split, red.global
            __syncwarp();
            misses_direct<MODE, K, SPL, KeyT>(sp, wq[lane].k, wq[lane].d, true, table);
            direct += sp.rows;
            __syncwarp();
            if (lane < qn - 32) {
                wq[lane] = wq[32 + lane];
            }
            __syncwarp();
            qn -= 32;
        } else if (BUF && qn >= 32) {  // a full warp of misses -> 32 slots of the miss buffer
            __syncwarp();
            if (wfill == kMissChunk) {
                if (lane == 0) wbase = atomicAdd(mb.count, (unsigned long long)kMissChunk);
                wbase = __shfl_sync(kFull, wbase, 0);
                wfill = 0;
            }
            const unsigned long long pos = wbase + wfill;
            wfill += 32;
            if (pos + 32 <= mb.cap) {
                mb.keys[pos + lane] = wq[lane].k;
                mb.deltas[pos + lane] = wq[lane].d;
            } else {
                misses_direct<MODE, K, SPL, KeyT>(sp, wq[lane].k, wq[lane].d, true, table);
                direct += sp.rows;
            }
            __syncwarp();
            if (lane < qn - 32) {
                wq[lane] = wq[32 + lane];
            }
            __syncwarp();
            qn -= 32;
        }
    };

    // full tiles, pulled dynamically from a shared counter; the next tile's
    // vectors are in flight while the current one is processed
    const uint64_t ntiles = t_hi - t_lo;
    KV kv[kVT];
    WVec<kV, WK> wv[kVT];
    u32 t = 0;
    if (lane == 0) t = atomicAdd(&s_next, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t < ntiles) {
        const uint64_t b = (t_lo + t) * kT;
#pragma unroll
        for (int v = 0; v < kVT; ++v) {
            const uint64_t i = b + (uint64_t)v * 32 * kV + lane * kV;
            kv[v].load(keys + i);
            wv[v].load(w, i);
        }
    }
    while (t < ntiles) {
        u32 tn = 0;
        if (lane == 0) tn = atomicAdd(&s_next, 1u);
        tn = __shfl_sync(kFull, tn, 0);
        KV kn[kVT];
        WVec<kV, WK> wn[kVT];
        if (tn < ntiles) {
            const uint64_t b = (t_lo + tn) * kT;
#pragma unroll
            for (int v = 0; v < kVT; ++v) {
                const uint64_t i = b + (uint64_t)v * 32 * kV + lane * kV;
                kn[v].load(keys + i);
                wn[v].load(w, i);
            }
        }
#pragma unroll
        for (int v = 0; v < kVT; ++v)
#pragma unroll
            for (int e = 0; e < kV; ++e) item(kv[v][e], wv[v].d[e], true);
#pragma unroll
        for (int v = 0; v < kVT; ++v) {
            kv[v] = kn[v];
            wv[v] = wn[v];
        }
        t = tn;
    }
    // this CTA's tail share: scalar loads
    for (uint64_t b = tail_lo + (uint64_t)warp * 32; b < tail_hi; b += (uint64_t)kHotWarps * 32) {
        const uint64_t i = b + lane;
        const bool v = i < tail_hi;
        item(v ? ld_nc(keys + i) : G::kEmpty, v ? load_w32<WK>(w, i) : 0, v);
    }
    if (lane < qn) {
        misses_direct<MODE, K, SPL, KeyT>(sp, wq[lane].k, wq[lane].d, true, table);
        direct += sp.rows;
    }
    // unused reserved slots become no-op items (delta 0)
    for (unsigned long long p = wbase + wfill + lane; BUF && p < wbase + kMissChunk && p < mb.cap; p += 32) {
        mb.keys[p] = 0;
        mb.deltas[p] = 0;
    }
    __syncthreads();
    // this CTA's cells go to its scratch area as they are (16-byte stores);
    // hh_merge_kernel sums the CTAs' cells per slot, adds the slot's wrap total and
    // hashes each hot key once.  (One L2 reduction per CTA and slot instead -- 6.9M
    // on config 5 -- took ~38 us at the end of every call.)
    {
        constexpr u32 kVecs = HotCells<KeyT>::kWords / 4;
        const uint4* src = reinterpret_cast<const uint4*>(G::kTagged ? tw : cells);
        uint4* dst = reinterpret_cast<uint4*>(scratch) + (size_t)blockIdx.x * kVecs;
        for (u32 j = threadIdx.x; j < kVecs; j += kHotThreads) dst[j] = src[j];
    }
    // instrumentation for the L2-reduction roofline (mb200_hot_stats)
    if (lane == 0) atomicAdd(&g_hot_stats[1], (unsigned long long)misses);
    direct = __reduce_add_sync(kFull, direct);
    if (lane == 0 && direct) atomicAdd(&g_hot_stats[5], (unsigned long long)direct);
    if (threadIdx.x == 0) atomicAdd(&g_hot_stats[0], (unsigned long long)((t_hi - t_lo) * kT + (tail_hi - tail_lo)));
}

// Each hot key once: its total = the slot's wrap total + the CTAs' cells (read from
// their scratch areas, coalesced over the slots), then hash -> split -> red.global.
// Skipped, like cs_hot_kernel, when the private byte tables or raw mode took the batch.
template <int MODE, int K, int SPL, typename KeyT>
__global__ void __launch_bounds__(256)
    hh_merge_kernel(const SketchParams sp, const KeyT* __restrict__ layout, const u64* __restrict__ slot_sum,
                    const u32* __restrict__ scratch, u32 nctas, const u32* __restrict__ hot_sum, uint32_t sample,
                    const u32* __restrict__ priv_go, i64* __restrict__ table) {
    using G = HotGeom<KeyT>;
    if (priv_go && *priv_go == 0) return;
    if (sample && raw_mode(hot_sum, sample)) return;
    constexpr u32 kW = HotCells<KeyT>::kWords;
    unsigned applied = 0;
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < G::kSlots) {
        const u32 idx = G::kTagged ? s : s >> 1, sh = G::kTagged ? kCellShift : (s & 1u) << 4;
        const u32 mask = G::kTagged ? 0x3fffu : 0xffffu;
        u32 acc = 0;  // <= nctas * 2^16
        constexpr u32 kB = 8;
        for (u32 c0 = 0; c0 < nctas; c0 += kB) {
            u32 wv[kB];
#pragma unroll
            for (u32 u = 0; u < kB; ++u) wv[u] = c0 + u < nctas ? __ldcg(scratch + (size_t)(c0 + u) * kW + idx) : 0u;
#pragma unroll
            for (u32 u = 0; u < kB; ++u) acc += c0 + u < nctas ? (wv[u] >> sh) & mask : 0u;
        }
        const u64 bias = G::kTagged ? (u64)kCellBias : 0x8000ull;
        const u64 v = slot_sum[s] + (u64)acc - (u64)nctas * bias;  // 0 in empty slots
        if (v) {
            rows_direct<MODE, K, SPL>(sp, (u64)layout[s], (i64)v, table);
            ++applied;
        }
    }
    applied = __reduce_add_sync(kFull, applied);
    if ((threadIdx.x & 31) == 0 && applied) atomicAdd(&g_hot_stats[2], (unsigned long long)applied);
}

// ---- passes 4 and 5: binned row updates ------------------------------------
// A bin is one row (or a 65536-cell slice of a wider row).  Entry = cell
// (16 bits) | signed delta (16 bits) << 16; 0 is a no-op (padding).
constexpr uint32_t kCellLog2 = 16;
constexpr i32 kDeltaLim = 1 << 15;
constexpr int kBinThreads = 1024;
constexpr uint32_t kMaxBins = 64;
constexpr size_t kStageBytes = 200 * 1024;
constexpr uint64_t kMinBinChunk = 1ull << 26;  // items binned per (pass 4, pass 5) round trip
constexpr uint32_t kMaxChunks = 8;
constexpr int kAccThreads = 1024;

struct BinGeom {
    u32* bins;                 // [nb][cap] 4-byte entries
    unsigned long long* gcnt;  // [chunks][nb] entries appended (may exceed cap)
    uint64_t cap;              // entries per bin, multiple of 4
    uint64_t width;
    uint32_t nb, bpr;          // bins, bins per row
    uint32_t cell_log2;        // log2 cells per bin (<= 16)
    uint32_t cap_s;            // staged entries per bin per round, multiple of 4
    uint32_t groups;           // 4-item groups per thread per round
};

__device__ __forceinline__ u32 make_entry(u32 cell, i32 d) { return cell | ((u32)d << kCellLog2); }
__device__ __forceinline__ void apply_entry_direct(const BinGeom& g, i64* table, u32 bin, u32 e) {
    if (!e) return;
    const u32 row = bin / g.bpr;
    const u64 idx = ((u64)(bin % g.bpr) << g.cell_log2) | (e & 0xffffu);
    red_add_u64(reinterpret_cast<uint64_t*>(table) + (u64)row * g.width + idx, (u64)(i64)((i32)e >> kCellLog2));
}

// Appends one row update per lane (warp-uniform call).  Lanes that target the
// same bin form one group (one ballot per bin-index bit; none when a row is
// one bin, ONEBIN) and one lane reserves the group's staging slots with ONE
// shared atomic -- per-lane atomics on a handful of counters serialise.
template <bool ONEBIN>
struct BinSink {
    const BinGeom& g;
    u32* stage;
    u32* scnt;
    i64* table;
    unsigned& direct;
    uint32_t sub_bits;  // ceil(log2(bins per row))
    __device__ __forceinline__ void operator()(u32 row, u32 idx, bool neg, i32 d, bool active) {
        active = active && d != 0;  // delta 0 adds nothing (sketch.cpp:136-138)
        const bool fits = active && (u32)(d + (kDeltaLim - 1)) < (u32)(2 * kDeltaLim - 1);  // |d| < 2^15
        const int lane = threadIdx.x & 31;
        unsigned peers = __ballot_sync(kFull, fits);
        u32 bin, base = 0;
        if (ONEBIN) {
            bin = row;
            if (lane == 0 && peers) base = atomicAdd(scnt + bin, (u32)__popc(peers));
            base = __shfl_sync(kFull, base, 0);
        } else {
            const u32 sub = idx >> g.cell_log2;
            for (uint32_t bit = 0; bit < sub_bits; ++bit) {
                const bool set = (sub >> bit) & 1;
                const unsigned m = __ballot_sync(kFull, set);
                peers &= set ? m : ~m;
            }
            bin = row * g.bpr + sub;
            const int leader = __ffs(peers) - 1;
            if (fits && lane == leader) base = atomicAdd(scnt + bin, (u32)__popc(peers));
            base = __shfl_sync(kFull, base, fits ? leader : lane);
        }
        const u32 slot = base + __popc(peers & ((1u << lane) - 1));
        if (fits && slot < g.cap_s) {
            stage[bin * g.cap_s + slot] = make_entry(idx & ((1u << g.cell_log2) - 1), neg ? -d : d);
        } else if (active) {
            const u64 sd = (u64)(i64)d;
            red_add_u64(reinterpret_cast<uint64_t*>(table) + (u64)row * g.width + idx, neg ? 0ull - sd : sd);
            ++direct;
        }
    }
};

// U items: per family the U Horner chains are interleaved, then every sub-row
// of every item goes to the sink (same arithmetic as process_item); warp-uniform.
template <int MODE, int K, int SPL, int U, typename Sink>
__device__ __forceinline__ void emit_items(const SketchParams& sp, const u64 (&x)[U], const i32 (&d)[U],
                                           unsigned valid, Sink& sink) {
    const uint32_t subs = (SPL == SPC_TFO || (SPL == SPC_ANY && sp.splitter == SPLIT_TWO_FOR_ONE)) ? 2 : 1;
#pragma unroll 1
    for (uint32_t f = 0; f < sp.families; ++f) {
        u64 hlo[U], hhi[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (MODE == M89) hash89<K>(sp, f, x[u], hlo[u], hhi[u]);
            else hlo[u] = hash_small<MODE, K>(sp, f, x[u]);
        }
        for (uint32_t s = 0; s < subs; ++s) {
            const uint32_t row = subs * f + s;
            if (row >= sp.rows) break;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                bool neg;
                const u32 idx = split_c<MODE, SPL>(sp, hlo[u], hhi[u], s, neg);
                sink(row, idx, neg, d[u], (valid >> u) & 1);
            }
        }
    }
}

// Pass 4.  RAW: the batch itself (raw mode); else the miss buffer.  Chunk c
// covers items [c * chunk_items, (c + 1) * chunk_items) of that source.
template <int MODE, int K, int SPL, typename KeyT, int WK, bool RAW, bool ONEBIN>
__global__ void __launch_bounds__(kBinThreads, 1)
    cs_bin_kernel(const SketchParams sp, const BinGeom g, const KeyT* __restrict__ keys, const void* __restrict__ w,
                  uint64_t n, const MissBuf<KeyT> mb, const u32* __restrict__ hot_sum, uint32_t sample,
                  uint32_t chunk, uint64_t chunk_items, i64* __restrict__ table) {
    if (raw_mode(hot_sum, sample) != RAW) return;
    const uint64_t total = RAW ? n : min((uint64_t)*mb.count, mb.cap);
    const uint64_t c0 = (uint64_t)chunk * chunk_items;
    if (c0 >= total) return;
    const uint64_t len = min(total - c0, chunk_items);
    const uint64_t lo = c0 + len * blockIdx.x / gridDim.x, hi = c0 + len * (blockIdx.x + 1) / gridDim.x;
    extern __shared__ __align__(16) u32 stage[];
    __shared__ u32 scnt[kMaxBins], sc4[kMaxBins];
    __shared__ unsigned long long spos[kMaxBins];
    for (u32 b = threadIdx.x; b < g.nb; b += kBinThreads) scnt[b] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned direct = 0, written = 0;
    uint32_t sub_bits = 0;
    while ((1u << sub_bits) < g.bpr) ++sub_bits;
    BinSink<ONEBIN> sink{g, stage, scnt, table, direct, sub_bits};
    const uint64_t per_round = (uint64_t)kBinThreads * 4 * g.groups;
    for (uint64_t base = lo; base < hi; base += per_round) {
#pragma unroll 1
        for (uint32_t gi = 0; gi < g.groups; ++gi) {
            u64 kx[4];
            i32 dx[4];
            unsigned valid = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = base + (uint64_t)(gi * 4 + u) * kBinThreads + threadIdx.x;
                const bool v = i < hi;
                valid |= (v ? 1u : 0u) << u;
                if (RAW) {
                    kx[u] = v ? (u64)ld_nc(keys + i) : 0;
                    dx[u] = v ? load_w32<WK>(w, i) : 0;
                } else {
                    kx[u] = v ? (u64)ld_nc(mb.keys + i) : 0;
                    dx[u] = v ? ld_nc(mb.deltas + i) : 0;
                }
            }
            emit_items<MODE, K, SPL, 4>(sp, kx, dx, valid, sink);
        }
        __syncthreads();
        // flush: pad each bin to whole 16-byte groups, reserve its HBM range with
        // one atomic, then all threads copy every bin in 16-byte groups
        if ((u32)warp < g.nb) {
            u32* st = stage + warp * g.cap_s;
            const u32 c = min(scnt[warp], g.cap_s);
            const u32 c4 = (c + 3) & ~3u;
            if ((u32)lane < c4 - c) st[c + lane] = 0;
            if (lane == 0) {
                sc4[warp] = c4;
                spos[warp] = c4 ? atomicAdd(g.gcnt + (uint64_t)chunk * g.nb + warp, (unsigned long long)c4) : 0;
            }
        }
        __syncthreads();
        for (u32 bin = 0; bin < g.nb; ++bin) {
            const u32 c4 = sc4[bin];
            const unsigned long long pos = spos[bin];
            const u32* st = stage + bin * g.cap_s;
            u32* dst = g.bins + (uint64_t)bin * g.cap;
            for (u32 j = threadIdx.x * 4; j < c4; j += 4 * kBinThreads) {
                const uint4 v = *reinterpret_cast<const uint4*>(st + j);
                if (pos + j + 4 <= g.cap) {
                    *reinterpret_cast<uint4*>(dst + pos + j) = v;
                    written += 4;
                } else {
                    apply_entry_direct(g, table, bin, v.x);
                    apply_entry_direct(g, table, bin, v.y);
                    apply_entry_direct(g, table, bin, v.z);
                    apply_entry_direct(g, table, bin, v.w);
                    direct += 4;
                }
            }
        }
        __syncthreads();
        for (u32 b = threadIdx.x; b < g.nb; b += kBinThreads) scnt[b] = 0;
        __syncthreads();
    }
    direct = __reduce_add_sync(kFull, direct);
    written = __reduce_add_sync(kFull, written);
    if (lane == 0 && direct) atomicAdd(&g_hot_stats[5], (unsigned long long)direct);
    if (lane == 0 && written) atomicAdd(&g_hot_stats[4], (unsigned long long)written);
}

// Exact accumulation into two 16-bit cells per 32-bit word (each 2^15-biased).
// The 32-bit atomic returns the word before the add, so every add knows the
// cell's 16-bit value before and after it: a value that leaves [0, 2^16) is
// recorded as +-2^16 straight into the L2 table (rare for small signed
// deltas).  A low-cell carry/borrow into the high cell is undone by a second
// atomic whose own wrap is recorded the same way; per cell, displayed value +
// 2^16 * (recorded wraps) = bias + sum of its deltas, exactly.
__device__ __forceinline__ void wrap16(uint64_t* row, u32 cell, i32 nv) {
    if (nv < 0 || nv > 0xffff) red_add_u64(row + cell, nv < 0 ? 0ull - 65536ull : 65536ull);
}
__device__ __forceinline__ void packed_add(u32* words, uint64_t* row, u32 cell, i32 d) {
    u32* w = words + (cell >> 1);
    if (cell & 1) {
        const u32 old = atomicAdd(w, (u32)d << 16);
        wrap16(row, cell, (i32)(old >> 16) + d);
    } else {
        const u32 old = atomicAdd(w, (u32)d);  // sign-extended: carries/borrows into the high cell
        const i32 nl = (i32)(old & 0xffffu) + d;
        if (nl < 0 || nl > 0xffff) {
            const i32 c = nl < 0 ? -1 : 1;
            red_add_u64(row + cell, (u64)(i64)(c * 65536));
            wrap16(row, cell + 1, (i32)(old >> 16) + c);      // the carry's effect on the high cell
            const u32 o2 = atomicAdd(w, (u32)(-c) << 16);     // ...undone
            wrap16(row, cell + 1, (i32)(o2 >> 16) - c);
        }
    }
}

// Pass 5: CTA (bin, part) sums a slice of its bin's entries in the packed
// shared table and merges the cells into the L2 table.
__global__ void __launch_bounds__(kAccThreads)
    cs_accum_kernel(const BinGeom g, uint32_t chunk, uint32_t parts, i64* __restrict__ table) {
    const u32 bin = blockIdx.x / parts, part = blockIdx.x % parts;
    const uint64_t cnt = min((uint64_t)g.gcnt[(uint64_t)chunk * g.nb + bin], g.cap);
    const uint64_t q = cnt / 4, q0 = q * part / parts, q1 = q * (part + 1) / parts;
    if (q0 == q1) return;
    extern __shared__ __align__(16) u32 words[];
    const u32 cells = 1u << g.cell_log2, nw = (cells + 1) / 2;
    for (u32 c = threadIdx.x; c < nw; c += kAccThreads) words[c] = 0x80008000u;
    __syncthreads();
    const u32 row = bin / g.bpr;
    const u64 col0 = (u64)(bin % g.bpr) << g.cell_log2;
    uint64_t* dst = reinterpret_cast<uint64_t*>(table) + (u64)row * g.width + col0;
    const uint4* src = reinterpret_cast<const uint4*>(g.bins + (uint64_t)bin * g.cap);
    uint64_t i = q0 + threadIdx.x;
    for (; i + 3 * kAccThreads < q1; i += 4 * kAccThreads) {  // four 16-byte loads in flight
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = ld_stream(src + i + k * kAccThreads);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u32 e[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (e[t]) packed_add(words, dst, e[t] & 0xffffu, (i32)e[t] >> kCellLog2);
        }
    }
    for (; i < q1; i += kAccThreads) {
        const uint4 v = ld_stream(src + i);
        const u32 e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (e[t]) packed_add(words, dst, e[t] & 0xffffu, (i32)e[t] >> kCellLog2);
    }
    __syncthreads();
    unsigned merged = 0;
    for (u32 c = threadIdx.x; c < cells; c += kAccThreads) {
        const i64 v = (i64)((words[c >> 1] >> ((c & 1) * 16)) & 0xffffu) - 0x8000;
        if (v) {  // cells past the row end never receive entries
            red_add_u64(dst + c, (u64)v);
            ++merged;
        }
    }
    merged = __reduce_add_sync(kFull, merged);
    if ((threadIdx.x & 31) == 0 && merged) atomicAdd(&g_hot_stats[6], (unsigned long long)merged);
}

// Private byte tables (streams without heavy hitters, unit deltas, rows x width
// <= 200 KiB cells): every CTA keeps the WHOLE table in shared memory as 8-bit
// cells (2^7-biased, four per 32-bit word), hashes each item once and adds +-1
// to one cell per row with one shared atomic.  The atomic returns the word
// before the add, so when the cell leaves [0, 2^8) every byte the carry or
// borrow reached is compared before/after and the difference between intended
// and displayed change goes to L2 (cell j receives intended_j - displayed_j):
// per cell, displayed - bias + recorded = sum of its deltas, exactly, under any
// interleaving and with no undo atomic.  The table is merged once per CTA.
// Runs only when the probe found no heavy hitters (go[0] == 0); cs_hot_kernel
// then returns at once.
constexpr int kPrivThreads = 1024;

__device__ __forceinline__ void byte_add(u32* words, uint64_t* cells_l2, u32 cell, i32 d) {
    const u32 q = cell & 3u, sh = q * 8;
    const u32 old = atomicAdd(words + (cell >> 2), (u32)d << sh);
    const i32 nb = (i32)((old >> sh) & 0xffu) + d;
    if ((u32)nb > 0xffu) {  // rare: the carry / borrow reached the bytes above
        const u32 nw = old + ((u32)d << sh);
        const u32 base = cell & ~3u;
        for (u32 j = q; j < 4; ++j) {
            const i32 disp = (i32)((nw >> (8 * j)) & 0xffu) - (i32)((old >> (8 * j)) & 0xffu);
            const i32 rec = (j == q ? d : 0) - disp;
            if (rec) red_add_u64(cells_l2 + base + j, (u64)(i64)rec);
        }
    }
}

template <int MODE, int K, int SPL, typename KeyT>
__global__ void __launch_bounds__(kPrivThreads, 1)
    cs_private_kernel(const SketchParams sp, const KeyT* __restrict__ keys, uint64_t n, i64* __restrict__ table,
                      const u32* __restrict__ go) {
    if (*go) return;
    extern __shared__ __align__(16) u32 pwords[];
    const u32 ncells = (u32)(sp.rows * sp.width), nw = ncells / 4;
    for (u32 c = threadIdx.x; c < nw; c += kPrivThreads) pwords[c] = 0x80808080u;
    __syncthreads();
    constexpr uint32_t subs = SPL == SPC_TFO ? 2 : 1;
    uint64_t* l2 = reinterpret_cast<uint64_t*>(table);
    const u32 width = (u32)sp.width;
    const uint64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    auto item = [&](u64 x) {
#pragma unroll 1
        for (uint32_t f = 0; f < sp.families; ++f) {
            if constexpr ((MODE == M61_K32 || MODE == M61_K64) && K > 0 && SPL == SPC_POW2) {
                bool neg;
                const u32 idx = h61_pow2_split(hash61_lazy<MODE, K>(sp, f, x), width - 1, neg);
                byte_add(pwords, l2, f * width + idx, neg ? -1 : 1);
                continue;
            }
            u64 hlo, hhi = 0;
            if (MODE == M89) hash89<K>(sp, f, x, hlo, hhi);
            else hlo = hash_small<MODE, K>(sp, f, x);
#pragma unroll
            for (uint32_t sub = 0; sub < subs; ++sub) {
                const uint32_t row = subs * f + sub;
                if (row >= sp.rows) break;
                bool neg;
                const u32 idx = split_c<MODE, SPL>(sp, hlo, hhi, sub, neg);
                byte_add(pwords, l2, row * width + idx, neg ? -1 : 1);
            }
        }
    };
    // eight keys per thread in flight (the loop is otherwise load-latency bound)
    constexpr int kU = 8;
    uint64_t i = lo + threadIdx.x;
    for (; i + (kU - 1) * kPrivThreads < hi; i += kU * kPrivThreads) {
        u64 xs[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) xs[u] = (u64)ld_nc(keys + i + u * kPrivThreads);
#pragma unroll
        for (int u = 0; u < kU; ++u) item(xs[u]);
    }
    for (; i < hi; i += kPrivThreads) item((u64)ld_nc(keys + i));
    __syncthreads();
    unsigned merged = 0;
    for (u32 c = threadIdx.x; c < ncells; c += kPrivThreads) {
        const i64 v = (i64)((pwords[c >> 2] >> ((c & 3) * 8)) & 0xffu) - 0x80;
        if (v) {
            red_add_u64(l2 + c, (u64)v);
            ++merged;
        }
    }
    merged = __reduce_add_sync(kFull, merged);
    if ((threadIdx.x & 31) == 0 && merged) atomicAdd(&g_hot_stats[6], (unsigned long long)merged);
    if (threadIdx.x == 0) atomicAdd(&g_hot_stats[0], (unsigned long long)(hi - lo));
}

// ---------------------------------------------------------------------------
// Row passes over the miss buffer (strategy STRAT_ROWS).  The hot pass leaves
// every missed item in the HBM miss buffer instead of sending rows L2
// reductions; then each CTA takes ONE row r = blockIdx % rows and a slice of the
// buffer, keeps that whole row in shared memory as 2^15-biased 16-bit cells
// (two per word, 2^16 cells = 128 KiB), hashes its slice for row r only and
// adds with one shared atomic per item.  The CTAs of one slice (blockIdx / rows)
// read it at the same time, so it comes from HBM once and from L2 rows - 1
// times.  A cell leaving [0, 2^16) (any i32 delta) records, per 16-bit cell the
// carry / borrow reached, (intended - displayed) change to L2 -- byte_add's
// exact accounting on 16-bit cells.  The rows' tables go to scratch and
// rows_fold_kernel sums each row's CTAs per cell: 148 x 2^16 cells instead of
// rows L2 reductions per missed item.
constexpr int kRowThreads = 1024;

__device__ __noinline__ void cell16_fix(uint64_t* l2row, u32 cell, i64 d, u32 old, u32 dw) {
    const u32 q = cell & 1u, base = cell & ~1u;
    const u32 nw = old + dw;
    for (u32 j = q; j < 2; ++j) {
        const i32 disp = (i32)((nw >> (16 * j)) & 0xffffu) - (i32)((old >> (16 * j)) & 0xffffu);
        const i64 rec = (j == q ? d : 0) - disp;
        if (rec) red_add_u64(l2row + base + j, (u64)rec);
    }
}

template <int MODE, int K, int SPL, typename KeyT>
__device__ __forceinline__ u32 row_cell(const SketchParams& sp, u32 f, u32 sub, KeyT key, bool& neg) {
    if constexpr ((MODE == M61_K32 || MODE == M61_K64) && K > 0 && SPL == SPC_POW2) {
        return h61_pow2_split(hash61_lazy<MODE, K>(sp, f, (u64)key), (u32)(sp.width - 1), neg);
    } else {
        u64 hlo, hhi = 0;
        if (MODE == M89) hash89<K>(sp, f, (u64)key, hlo, hhi);
        else hlo = hash_small<MODE, K>(sp, f, (u64)key);
        return split_c<MODE, SPL>(sp, hlo, hhi, sub, neg);
    }
}

template <int MODE, int K, int SPL, typename KeyT>
__global__ void __launch_bounds__(kRowThreads, 1)
    cs_rowpass_kernel(const SketchParams sp, const MissBuf<KeyT> mb, u32* __restrict__ scratch, i64* __restrict__ table) {
    extern __shared__ __align__(16) u32 rw[];
    const u32 W = (u32)sp.width, nw = W / 2;
    for (u32 i = threadIdx.x; i < nw; i += kRowThreads) rw[i] = 0x80008000u;
    __syncthreads();
    const u32 row = blockIdx.x % sp.rows, part = blockIdx.x / sp.rows;
    const u32 nparts = (gridDim.x - row + sp.rows - 1) / sp.rows;
    const u32 f = SPL == SPC_TFO ? row / 2 : row, sub = SPL == SPC_TFO ? row % 2 : 0;
    uint64_t* l2row = reinterpret_cast<uint64_t*>(table) + (size_t)row * W;
    const uint64_t stored = *mb.count;
    const uint64_t n = stored < mb.cap ? stored : mb.cap;
    const uint64_t lo = n * part / nparts, hi = n * (part + 1) / nparts;
    constexpr int kU = 4;  // items per thread in flight
    auto one = [&](KeyT key, i32 d) {
        bool neg;
        const u32 cell = row_cell<MODE, K, SPL, KeyT>(sp, f, sub, key, neg);
        const i64 dd = neg ? -(i64)d : (i64)d;  // (-INT32_MIN = 2^31: the reference's wrapping negation)
        const u32 sh = (cell & 1u) << 4;
        const u32 dw = (u32)dd << sh;
        const u32 old = atomicAdd(rw + (cell >> 1), dw);
        const i64 nb = (i64)((old >> sh) & 0xffffu) + dd;
        if (__builtin_expect((u64)nb > 0xffffu, 0)) cell16_fix(l2row, cell, dd, old, dw);
    };
    uint64_t i = lo + threadIdx.x;
    for (; i + (kU - 1) * kRowThreads < hi; i += kU * kRowThreads) {
        KeyT k[kU];
        i32 d[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            k[u] = __ldcg(mb.keys + i + u * kRowThreads);
            d[u] = __ldcg(mb.deltas + i + u * kRowThreads);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) one(k[u], d[u]);
    }
    for (; i < hi; i += kRowThreads) one(__ldcg(mb.keys + i), __ldcg(mb.deltas + i));
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(scratch + (size_t)blockIdx.x * nw);
    const uint4* src = reinterpret_cast<const uint4*>(rw);
    for (u32 j = threadIdx.x; j < nw / 4; j += kRowThreads) dst[j] = src[j];
    if (threadIdx.x == 0) atomicAdd(&g_hot_stats[4], (unsigned long long)(hi - lo));
}

// table[row][cell] += sum over the row's CTAs of (cell - 2^15); one thread per
// word (two cells) of one row
__global__ void __launch_bounds__(256)
    rows_fold_kernel(const u32* __restrict__ scratch, u32 rows, u32 width, u32 ctas, i64* __restrict__ table) {
    const u32 nw = width / 2;
    const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (u64)rows * nw) return;
    const u32 row = (u32)(gid / nw), w = (u32)(gid % nw);
    const u32 nparts = (ctas - row + rows - 1) / rows;
    i32 lo = 0, hi = 0;
    u32 p = 0;
    for (; p + 8 <= nparts; p += 8) {
        u32 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(scratch + (size_t)(row + (p + u) * rows) * nw + w);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            lo += (i32)(v[u] & 0xffffu);
            hi += (i32)(v[u] >> 16);
        }
    }
    for (; p < nparts; ++p) {
        const u32 v = __ldcg(scratch + (size_t)(row + p * rows) * nw + w);
        lo += (i32)(v & 0xffffu);
        hi += (i32)(v >> 16);
    }
    const i32 bias = 0x8000 * (i32)nparts;
    i64* t = table + (size_t)row * width + 2 * w;
    if (lo != bias) t[0] = (i64)((u64)t[0] + (u64)(i64)(lo - bias));
    if (hi != bias) t[1] = (i64)((u64)t[1] + (u64)(i64)(hi - bias));
}

inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Bench hook (mb200_kernel_timer): CUDA events around the dominant scatter
// kernel of every launch_cs_hot call (cs_hot / cs_private / cs_private89), on
// the stream it runs on, so the roofline divides by that kernel's own time.
struct KernelTimer {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
};
KernelTimer g_ktimer;
inline void ktimer_mark(cudaStream_t s, bool start) {
    KernelTimer& t = g_ktimer;
    if (!t.on) return;
    if (start) {
        if (t.used == t.ev.size()) {
            std::pair<cudaEvent_t, cudaEvent_t> p{};
            if (cudaEventCreate(&p.first) != cudaSuccess || cudaEventCreate(&p.second) != cudaSuccess) return;
            t.ev.push_back(p);
        }
        cudaEventRecord(t.ev[t.used].first, s);
    } else if (t.used < t.ev.size()) {
        cudaEventRecord(t.ev[t.used++].second, s);
    }
}

// large-table strategy (mb200_set_large_table_strategy): misses either go
// straight to L2 (fire-and-forget reductions, overlapped with the hot-key work;
// measured fastest on configs 4 and 5) or through the binned passes 4-5
int g_strategy = STRAT_DIRECT;

// Buffers of one call, carved from one stream-ordered allocation (the pool keeps
// its memory between calls, retain_pool).
template <typename KeyT>
struct HotPlan {
    BinGeom g{};
    uint32_t m = 0;            // sample size
    uint32_t slots = 0;        // sample count table slots (power of two >= m)
    uint32_t chunks = 0;       // (pass 4, pass 5) round trips
    uint64_t chunk_items = 0;  // items per round trip
    uint64_t cap_m = 0;        // miss-buffer capacity
    size_t tk_bytes = 0, tc_bytes = 0, misc = 0, gcnt_bytes = 0, sum_bytes = 0, hot_bytes = 0,
           layout_bytes = 0, mk_bytes = 0, md_bytes = 0, bin_bytes = 0;
    size_t tags_bytes = 0;   // tagged hot table (u32 keys): the slot words hh_slots writes
    size_t scr_bytes = 0;    // the scatter CTAs' cells (one area per CTA), summed by hh_merge
    bool rows_mode = false;  // STRAT_ROWS: misses to the buffer, then the row passes
    size_t rows_bytes = 0;   // row passes' per-CTA tables
    // tc .. slot sums are contiguous and zeroed per call
    size_t zero_bytes() const { return tc_bytes + misc + gcnt_bytes + sum_bytes; }
    size_t total() const {
        return tk_bytes + zero_bytes() + hot_bytes + layout_bytes + tags_bytes + scr_bytes + mk_bytes + md_bytes +
               bin_bytes + rows_bytes;
    }
};

template <typename KeyT>
HotPlan<KeyT> plan_hot(const SketchParams& sp, uint64_t n) {
    using G = HotGeom<KeyT>;
    HotPlan<KeyT> P;
    // sample = n / 128 items, clamped to [2^18, 2^22]: measured on config 5's stream,
    // a 2^28-item shard takes 1.119 ms with n / 256 and 1.092 ms with n / 128 (misses
    // 11.9% -> 10.7%), 2^29 items 2.01 -> 1.99 ms; the full 2^31 items sit at the
    // clamp either way (2^23 sampled items: misses 10.1% -> 9.9%, but the call only
    // 7.265 -> 7.245 ms and twice the workspace)
    uint64_t m = n / 128;
    m = m < kMinSample ? kMinSample : m > kMaxSample ? kMaxSample : m;
    P.m = (uint32_t)(n < m ? n : m);
    P.slots = 64;
    while (P.slots < P.m) P.slots *= 2;  // one slot per sampled item (bounded probing, hh_count)
    BinGeom& g = P.g;
    // bin geometry: rows x ceil(width / 8192) bins of <= 8192 cells
    g.width = sp.width;
    uint32_t cl = 0;
    while ((1ull << cl) < sp.width && cl < kCellLog2) ++cl;
    g.cell_log2 = cl;
    const uint64_t bpr = (sp.width + (1ull << cl) - 1) >> cl;
    const bool binned = g_strategy == STRAT_BINNED && (uint64_t)sp.rows * bpr <= kMaxBins;
    g.bpr = (uint32_t)bpr;
    g.nb = binned ? sp.rows * g.bpr : 0;
    if (binned) {
        // miss buffer: half the batch (the rest, if ever, goes straight to L2)
        P.cap_m = (n / 2 + 31) & ~31ull;
        const uint64_t src_max = n > P.cap_m ? n : P.cap_m;
        P.chunk_items = (src_max + kMaxChunks - 1) / kMaxChunks;
        if (P.chunk_items < kMinBinChunk) P.chunk_items = kMinBinChunk;
        P.chunks = (uint32_t)((src_max + P.chunk_items - 1) / P.chunk_items);
        const uint64_t per_chunk = src_max < P.chunk_items ? src_max : P.chunk_items;
        // a bin receives ~rows * per_chunk / nb entries per chunk (hash bits are
        // uniform); 25% margin + round padding, overflow goes straight to L2
        g.cap = (((uint64_t)sp.rows * per_chunk / g.nb) * 5 / 4 + 4 * (uint64_t)kBinThreads + 4096) & ~3ull;
        g.cap_s = (uint32_t)(kStageBytes / 4 / g.nb) & ~3u;
        // 4-item groups per round so that a bin's expected share (4096 rows / nb
        // entries per group) stays under ~85% of its staging buffer
        const uint64_t grp = (uint64_t)g.cap_s * 17 / 20 * g.nb / ((uint64_t)kBinThreads * 4 * sp.rows);
        g.groups = (uint32_t)(grp < 1 ? 1 : grp > 16 ? 16 : grp);
    }
    P.tk_bytes = align256((size_t)P.slots * sizeof(KeyT));
    P.tc_bytes = (size_t)P.slots * 4;
    P.misc = 256 * 4 + 64 + 256 * 4;  // hist[256], hot_count, hot_sum, miss count (u64), go words, fill[256]
    P.gcnt_bytes = align256((size_t)P.chunks * g.nb * 8 + 8);
    P.sum_bytes = align256((size_t)G::kSlots * 8);
    P.layout_bytes = align256((size_t)G::kSlots * sizeof(KeyT));
    P.tags_bytes = G::kTagged ? align256((size_t)G::kSlots * 4) : 0;
    P.scr_bytes = align256((size_t)sm_count() * HotCells<KeyT>::kWords * 4);
    P.hot_bytes = align256((size_t)G::kCap * sizeof(KeyT));  // the hot list, ordered by sample count
    // row passes: Pow2 / two-for-one splitters of power-of-two rows <= 2^16 cells
    P.rows_mode = g_strategy == STRAT_ROWS && !binned && (sp.b == 61 || sp.b == 89) &&
                  (sp.splitter == SPLIT_POW2 || sp.splitter == SPLIT_TWO_FOR_ONE) && sp.width >= 8 &&
                  sp.width <= 65536 && (sp.width & (sp.width - 1)) == 0 && sp.rows <= (uint32_t)sm_count();
    if (P.rows_mode) {
        P.cap_m = (n / 2 + 31) & ~31ull;  // the rest, if ever, goes straight to L2
        P.rows_bytes = align256((size_t)sm_count() * sp.width * 2);
    }
    P.mk_bytes = align256((size_t)P.cap_m * sizeof(KeyT));
    P.md_bytes = align256((size_t)P.cap_m * 4);
    P.bin_bytes = (size_t)g.nb * g.cap * 4;
    return P;
}

template <int MODE, int K, int SPL, typename KeyT, int WK>
cudaError_t run_hot(const SketchParams& sp, const KeyT* keys, const void* w, uint64_t n, int64_t* table,
                    cudaStream_t s, unsigned char* ws, HotPlan<KeyT> P) {
    using G = HotGeom<KeyT>;
    const int sms = sm_count();
    BinGeom& g = P.g;
    const bool binned = g.nb != 0;
    KeyT* tk = reinterpret_cast<KeyT*>(ws);
    u32* tc = reinterpret_cast<u32*>(ws + P.tk_bytes);
    u32* hist = tc + P.slots;
    u32* hot_count = hist + 256;
    u32* hot_sum = hot_count + 1;
    unsigned long long* mcount = reinterpret_cast<unsigned long long*>(hot_count + 2);
    g.gcnt = reinterpret_cast<unsigned long long*>(ws + P.tk_bytes + P.tc_bytes + P.misc);
    // zeroed per call: tc | misc | gcnt | slot sums
    u64* slot_sum = reinterpret_cast<u64*>(ws + P.tk_bytes + P.tc_bytes + P.misc + P.gcnt_bytes);
    unsigned char* p = ws + P.tk_bytes + P.zero_bytes();
    KeyT* hot = reinterpret_cast<KeyT*>(p);
    p += P.hot_bytes;
    KeyT* layout = reinterpret_cast<KeyT*>(p);
    p += P.layout_bytes;
    u32* tags = P.tags_bytes ? reinterpret_cast<u32*>(p) : nullptr;
    p += P.tags_bytes;
    u32* scratch = reinterpret_cast<u32*>(p);
    p += P.scr_bytes;
    const MissBuf<KeyT> mb{reinterpret_cast<KeyT*>(p), reinterpret_cast<i32*>(p + P.mk_bytes), mcount, P.cap_m};
    p += P.mk_bytes + P.md_bytes;
    g.bins = reinterpret_cast<u32*>(p);
    cudaMemsetAsync(tk, 0xff, P.tk_bytes, s);
    cudaMemsetAsync(tc, 0, P.zero_bytes(), s);
    u32* go = hot_count + 4;  // misc words after the miss count: go, covered, ticket
    u32* fill = hot_count + 16;  // per-level fill counters of the ordered selection
    const HotPrepWs<KeyT> pw{tk, tc, P.slots, hist, hot_count, hot_sum, fill, go, hot_count + 8, hot};
    cudaError_t e = launch_hot_select<KeyT>(keys, n, P.m, pw, s);
    if (e != cudaSuccess) return e;
    const bool rows_mode = P.rows_mode && SPL != SPC_ANY;
    auto fn = binned || rows_mode ? cs_hot_kernel<MODE, K, SPL, KeyT, WK, true>
                                  : cs_hot_kernel<MODE, K, SPL, KeyT, WK, false>;
    const size_t smem = G::kTagged ? (size_t)4 * G::kSlots : ((size_t)sizeof(KeyT) + 2) * G::kSlots;
    const size_t qbytes = (size_t)kHotWarps * kQueue * sizeof(QEnt<KeyT>);
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + qbytes))) != cudaSuccess)
        return e;
    uint64_t grid = (n + 256 * kHotWarps - 1) / (256 * kHotWarps);
    if (grid > (uint64_t)sms) grid = sms;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(keys) & 15) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0;
    // without bins (cap 0) every miss takes the direct path and raw mode is off
    // streams without heavy hitters and unit deltas whose whole table fits
    // shared memory as bytes: private byte tables instead of one L2 reduction
    // per row update
    const uint64_t pcells = (uint64_t)sp.rows * sp.width;
    const bool priv = !binned && WK == W_NONE && SPL != SPC_ANY && pcells <= 200u * 1024 && pcells % 4 == 0 &&
                      sp.width % 4 == 0 && n >= (1u << 20);
    if ((e = launch_hot_layout<KeyT>(pw, layout, tags, priv ? go : nullptr, s)) != cudaSuccess) return e;
    if (priv) {
        auto fp = cs_private_kernel<MODE, K, SPL, KeyT>;
        if ((e = cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcells)) != cudaSuccess)
            return e;
        ktimer_mark(s, true);
        fp<<<sms, kPrivThreads, pcells, s>>>(sp, keys, n, table, go);
        ktimer_mark(s, false);
    }
    if (!priv) ktimer_mark(s, true);
    fn<<<(unsigned)grid, kHotThreads, smem + qbytes, s>>>(sp, keys, w, n, table, layout, tags, slot_sum, hot_sum,
                                                          binned ? P.m : 0, mb, vec_ok,
                                                          priv ? go : nullptr, scratch);
    if (!priv) ktimer_mark(s, false);
    hh_merge_kernel<MODE, K, SPL, KeyT><<<(G::kSlots + 255) / 256, 256, 0, s>>>(
        sp, layout, slot_sum, scratch, (u32)grid, hot_sum, binned ? P.m : 0, priv ? go : nullptr, table);
    if (rows_mode) {
        if constexpr (SPL != SPC_ANY) {
            auto fr = cs_rowpass_kernel<MODE, K, SPL, KeyT>;
            const size_t rbytes = (size_t)sp.width * 2;
            if ((e = cudaFuncSetAttribute(fr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rbytes)) != cudaSuccess)
                return e;
            u32* rscratch = reinterpret_cast<u32*>(ws + P.total() - P.rows_bytes);
            fr<<<sms, kRowThreads, rbytes, s>>>(sp, mb, rscratch, table);
            const uint64_t words = (uint64_t)sp.rows * (sp.width / 2);
            rows_fold_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(rscratch, sp.rows, (u32)sp.width,
                                                                          (u32)sms, table);
        }
    }
    if ((e = cudaGetLastError()) != cudaSuccess || !binned) return e;
    auto fb_raw = g.bpr == 1 ? cs_bin_kernel<MODE, K, SPL, KeyT, WK, true, true>
                             : cs_bin_kernel<MODE, K, SPL, KeyT, WK, true, false>;
    auto fb_miss = g.bpr == 1 ? cs_bin_kernel<MODE, K, SPL, KeyT, W_I32, false, true>
                              : cs_bin_kernel<MODE, K, SPL, KeyT, W_I32, false, false>;
    const size_t sbytes = (size_t)g.nb * g.cap_s * 4;
    if ((e = cudaFuncSetAttribute(fb_raw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(fb_miss, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes)) != cudaSuccess)
        return e;
    const size_t abytes = (size_t)4 * (((1u << g.cell_log2) + 1) / 2);
    if ((e = cudaFuncSetAttribute(cs_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 << kCellLog2)) !=
        cudaSuccess)
        return e;
    // one wave: 1024-thread CTAs, up to 2 per SM when the cell table is small
    const uint32_t per_sm = abytes <= 96 * 1024 ? 2 : 1;
    const uint32_t parts = (uint32_t)(per_sm * sms / g.nb > 0 ? per_sm * sms / g.nb : 1);
    for (uint32_t c = 0; c < P.chunks; ++c) {
        if ((uint64_t)c * P.chunk_items < n)
            fb_raw<<<sms, kBinThreads, sbytes, s>>>(sp, g, keys, w, n, mb, hot_sum, P.m, c, P.chunk_items, table);
        if ((uint64_t)c * P.chunk_items < P.cap_m)
            fb_miss<<<sms, kBinThreads, sbytes, s>>>(sp, g, keys, w, n, mb, hot_sum, P.m, c, P.chunk_items, table);
        cs_accum_kernel<<<g.nb * parts, kAccThreads, abytes, s>>>(g, c, parts, table);
    }
    return cudaGetLastError();
}

// config 4's shape: cs_private89_kernel + private_fold_kernel, one CTA per SM,
// per-CTA byte tables (128 KiB each) in a scratch area of the stream-ordered pool
cudaError_t run_private89(const SketchParams& sp, const u64* keys, uint64_t n, int64_t* table, cudaStream_t s) {
    constexpr int LW = 16;
    constexpr size_t tbytes = 2u << LW;
    const int sms = sm_count();
    Coef89 c89;
    for (int j = 0; j < 4; ++j) {
        c89.a[j][0] = (u32)sp.lo[j];
        c89.a[j][1] = (u32)(sp.lo[j] >> 32);
        c89.a[j][2] = (u32)sp.hi[j];
    }
    auto fp = cs_private89_kernel<LW, false>;
    auto ff = cs_private89_kernel<LW, true>;
    cudaError_t e = cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tbytes);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ff, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tbytes)) != cudaSuccess)
        return e;
    uint4* scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), (size_t)sms * tbytes, s)) != cudaSuccess) return e;
    const ulonglong2* kv = reinterpret_cast<const ulonglong2*>(keys);
    uint64_t np = n / 2;
    const u64* odd = (n & 1) ? keys + n - 1 : nullptr;
    uint64_t* l2 = reinterpret_cast<uint64_t*>(table);
    const u32* nogo = nullptr;
    // one cooperative launch (grid barrier, then every CTA folds its share of the
    // columns) where the device supports it; else the kernel + private_fold_kernel
    static const bool coop = [] {
        int v = 0, dev = 0;
        cudaGetDevice(&dev);
        return cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && v != 0;
    }();
    ktimer_mark(s, true);
    if (coop) {
        void* args[] = {(void*)&c89, (void*)&kv, (void*)&np, (void*)&odd, (void*)&scratch, (void*)&l2, (void*)&nogo};
        e = cudaLaunchCooperativeKernel((const void*)ff, dim3(sms), dim3(kP89Threads), args, tbytes, s);
        ktimer_mark(s, false);
    } else {
        fp<<<sms, kP89Threads, tbytes, s>>>(c89, kv, np, odd, scratch, l2, nogo);
        ktimer_mark(s, false);
        const u32 cols = (u32)(tbytes / 16);
        private_fold_kernel<<<(cols + kFoldCols - 1) / kFoldCols, kFoldThreads, 0, s>>>(scratch, cols, (u32)sms,
                                                                                        table, nullptr);
        e = cudaGetLastError();
    }
    const cudaError_t e2 = cudaFreeAsync(scratch, s);
    return e != cudaSuccess ? e : e2;
}

template <int MODE, int K, typename KeyT, int WK>
cudaError_t launch_hot(const SketchParams& sp, const void* keys, const void* w, uint64_t n, int64_t* table,
                       cudaStream_t s) {
    // config 4's shape (cs_private89_kernel): 2^89-1, k = 4, u64 keys (16-byte
    // aligned), unit deltas, one family split two-for-one into 2 x 2^16 counters.
    // Byte tables are exact for any stream and their cost does not depend on its
    // skew (a hot cell leaves [0, 2^8) once per 2^8 updates of one CTA), so this
    // shape skips the heavy-hitter probe and its chain of kernels altogether.
    if (MODE == M89 && K == 4 && std::is_same<KeyT, u64>::value && WK == W_NONE &&
        sp.splitter == SPLIT_TWO_FOR_ONE && sp.families == 1 && sp.rows == 2 && sp.width == 65536 &&
        g_strategy == STRAT_DIRECT && n >= (1u << 20) && (reinterpret_cast<uintptr_t>(keys) & 15) == 0)
        return run_private89(sp, reinterpret_cast<const u64*>(keys), n, table, s);
    HotPlan<KeyT> P = plan_hot<KeyT>(sp, n);
    unsigned char* ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, P.total(), s);
    if (e != cudaSuccess) return e;
    const KeyT* kk = reinterpret_cast<const KeyT*>(keys);
    const bool narrow = sp.width <= (1ull << 32);  // compile-time splitters return u32 indices
    if (MODE != MGEN && narrow && sp.splitter == SPLIT_POW2)
        e = run_hot<MODE, K, SPC_POW2, KeyT, WK>(sp, kk, w, n, table, s, ws, P);
    else if (MODE != MGEN && narrow && sp.splitter == SPLIT_TWO_FOR_ONE)
        e = run_hot<MODE, K, SPC_TFO, KeyT, WK>(sp, kk, w, n, table, s, ws, P);
    else
        e = run_hot<MODE, K, SPC_ANY, KeyT, WK>(sp, kk, w, n, table, s, ws, P);
    const cudaError_t e2 = cudaFreeAsync(ws, s);
    return e != cudaSuccess ? e : e2;
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
// allocates its workspace per call with cudaMallocAsync (sample tables, hot
// list and layout, and for the binned / rows strategies the miss buffer, bins or
// row tables; config 4's shape: 148 x 128 KiB byte tables).
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

int set_large_table_strategy(int s) {
    if (s != STRAT_DIRECT && s != STRAT_BINNED && s != STRAT_ROWS) return -1;
    const int old = g_strategy;
    g_strategy = s;
    return old;
}

void kernel_timer(bool enable) {
    g_ktimer.on = enable;
    g_ktimer.used = 0;
}

cudaError_t kernel_timer_read(double* total_ms, uint64_t* launches) {
    double tot = 0;
    for (size_t i = 0; i < g_ktimer.used; ++i) {
        cudaError_t e = cudaEventSynchronize(g_ktimer.ev[i].second);
        if (e != cudaSuccess) return e;
        float ms = 0;
        if ((e = cudaEventElapsedTime(&ms, g_ktimer.ev[i].first, g_ktimer.ev[i].second)) != cudaSuccess) return e;
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = g_ktimer.used;
    g_ktimer.used = 0;
    return cudaSuccess;
}

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
