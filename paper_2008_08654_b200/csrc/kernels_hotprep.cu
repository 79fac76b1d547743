// kernels_hotprep.cu -- the heavy-hitter selection in front of cs_hot_kernel
// (kernels_hot.cu): a quick probe of the batch's head, exact counts of a sample,
// the count histogram, the ordered selection of the most frequent keys and
// their placement in the two-choice shared-memory table every scatter CTA
// copies.  None of this depends on the hash family or the splitter, and none of
// it affects the table's contents (integer addition commutes: the hot set only
// decides how many L2 reductions a call needs); it is a FIXED cost of every
// call, ~0.1 ms on a 2^28-item shard, which is why it is its own translation
// unit with latency-minded kernels.
#include "mb200_hot_geom.cuh"
#include "mb200_hotprep.h"
#include "mb200_internal.h"

namespace mb200 {
namespace {

template <typename T>
__device__ __forceinline__ T ld_key(const T* p) {  // read-once stream data
    return __ldg(p);
}

// Exact key counts of the sample in a global open-addressing table.  Each CTA
// first counts its share in a shared-memory table (so the hottest keys of a
// skewed stream cost one global atomic per CTA, not one per warp: 32K warps
// incrementing one counter serialise at L2), then merges its distinct keys.
constexpr int kCountThreads = 512;
constexpr uint32_t kLocalSlots = 4096;
constexpr uint32_t kCountProbes = 64;

template <typename KeyT>
__device__ __forceinline__ void count_global(KeyT* tk, u32* tc, u32 slots, KeyT key, u32 cnt) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    u32 h = (u32)(((u64)((u32)(mix64((u64)key) >> 32)) * slots) >> 32);
    // bounded: the table has as many slots as the sample has items (a Zipf sample
    // fills ~10% of it); a sample of (nearly) all distinct keys fills it, and
    // a key that finds no slot within kCountProbes is left uncounted -- the counts
    // only rank candidates
    for (u32 probe = 0; probe < kCountProbes; ++probe) {
        KeyT cur = tk[h];
        if (cur == G::kEmpty) cur = (KeyT)atomicCAS(reinterpret_cast<C*>(tk + h), (C)G::kEmpty, (C)key);
        if (cur == G::kEmpty || cur == key) {
            atomicAdd(tc + h, cnt);
            return;
        }
        h = h + 1 == slots ? 0 : h + 1;
    }
}

// Quick look at the batch's first kProbeItems items (kProbeCtas CTAs, each
// counting its contiguous share in a shared table): if keys seen at least twice
// within a share cover under 1/32 of the items (a stream without heavy
// hitters, like config 4's uniform 64-bit keys), the sample / selection kernels
// are skipped (go[0] = 0) and every item takes the direct path.  go[1] sums the
// covered items, go[2] is the ticket of the last CTA, which decides.
// Performance only.
constexpr uint32_t kProbeItems = 1u << 14;
constexpr int kProbeCtas = 8;

template <typename KeyT>
__global__ void __launch_bounds__(1024) hh_probe_kernel(const KeyT* __restrict__ keys, uint64_t n, u32* go) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    constexpr u32 kProbeSlots = kLocalSlots / 2;  // a share of 2^11 items fits
    __shared__ KeyT lk[kProbeSlots];
    __shared__ u32 lc[kProbeSlots];
    __shared__ u32 covered;
    for (u32 i = threadIdx.x; i < kProbeSlots; i += blockDim.x) {
        lk[i] = G::kEmpty;
        lc[i] = 0;
    }
    if (threadIdx.x == 0) covered = 0;
    __syncthreads();
    const u32 m = (u32)(n < kProbeItems ? n : kProbeItems);
    const u32 lo = m * blockIdx.x / gridDim.x, hi = m * (blockIdx.x + 1) / gridDim.x;
    for (u32 i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const KeyT key = ld_key(keys + i);
        if (key == G::kEmpty) continue;
        u32 h = (u32)mix64((u64)key) & (kProbeSlots - 1);
        for (int probe = 0; probe < 8; ++probe) {  // a crowded table just drops the item
            KeyT cur = lk[h];
            if (cur == G::kEmpty) cur = (KeyT)atomicCAS(reinterpret_cast<C*>(lk + h), (C)G::kEmpty, (C)key);
            if (cur == G::kEmpty || cur == key) {
                atomicAdd(lc + h, 1u);
                break;
            }
            h = (h + 1) & (kProbeSlots - 1);
        }
    }
    __syncthreads();
    u32 mine = 0;
    for (u32 i = threadIdx.x; i < kProbeSlots; i += blockDim.x) mine += lc[i] >= 2 ? lc[i] : 0;
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&covered, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (covered) atomicAdd(go + 1, covered);
        __threadfence();
        if (atomicAdd(go + 2, 1u) == gridDim.x - 1) {  // the last CTA: every share is counted
            __threadfence();
            go[0] = atomicAdd(go + 1, 0u) * 32 >= m ? 1u : 0u;
        }
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(kCountThreads) hh_count_kernel(const KeyT* __restrict__ keys, uint64_t n, KeyT* tk,
                                                                 u32* tc, u32 slots, const u32* __restrict__ go) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    if (!*go) return;
    __shared__ KeyT lk[kLocalSlots];
    __shared__ u32 lc[kLocalSlots];
    for (u32 i = threadIdx.x; i < kLocalSlots; i += kCountThreads) {
        lk[i] = G::kEmpty;
        lc[i] = 0;
    }
    __syncthreads();
    const uint64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    constexpr int kLd = 8;  // keys of a thread loaded together (a share is ~7 per thread at 2^20 sampled items)
    for (uint64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (uint64_t)kLd * kCountThreads) {
        KeyT kk[kLd];
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
            const uint64_t i = i0 + (uint64_t)u * kCountThreads;
            kk[u] = i < hi ? ld_key(keys + i) : G::kEmpty;
        }
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
            const KeyT key = kk[u];
            if (key == G::kEmpty) continue;  // the sentinel key is never hot
            u32 h = (u32)mix64((u64)key) & (kLocalSlots - 1);
            bool done = false;
            for (int probe = 0; probe < 8 && !done; ++probe) {
                KeyT cur = lk[h];
                if (cur == G::kEmpty) cur = (KeyT)atomicCAS(reinterpret_cast<C*>(lk + h), (C)G::kEmpty, (C)key);
                if (cur == G::kEmpty || cur == key) {
                    atomicAdd(lc + h, 1u);
                    done = true;
                }
                h = (h + 1) & (kLocalSlots - 1);
            }
            if (!done) count_global(tk, tc, slots, key, 1u);  // local table crowded
        }
    }
    __syncthreads();
    // the CTA's distinct keys into the global table, kLocalSlots / kCountThreads of
    // a thread at once: home slots read together, then the claims, then the adds
    // (three global latencies per thread instead of three per key); a key whose
    // home slot holds another key takes the probing path
    constexpr u32 kPerT = kLocalSlots / kCountThreads;
    static_assert(kLocalSlots % kCountThreads == 0, "whole batches");
    KeyT key[kPerT], cur[kPerT];
    u32 cnt[kPerT], h[kPerT];
#pragma unroll
    for (u32 j = 0; j < kPerT; ++j) {
        const u32 i = threadIdx.x + j * kCountThreads;
        cnt[j] = lc[i];
        key[j] = lk[i];
        h[j] = (u32)(((u64)((u32)(mix64((u64)key[j]) >> 32)) * slots) >> 32);
    }
#pragma unroll
    for (u32 j = 0; j < kPerT; ++j)
        if (cnt[j]) cur[j] = tk[h[j]];
#pragma unroll
    for (u32 j = 0; j < kPerT; ++j)
        if (cnt[j] && cur[j] == G::kEmpty) cur[j] = (KeyT)atomicCAS(reinterpret_cast<C*>(tk + h[j]), (C)G::kEmpty, (C)key[j]);
#pragma unroll
    for (u32 j = 0; j < kPerT; ++j) {
        if (!cnt[j]) continue;
        if (cur[j] == G::kEmpty || cur[j] == key[j]) atomicAdd(tc + h[j], cnt[j]);
        else count_global(tk, tc, slots, key[j], cnt[j]);
    }
}

__global__ void hh_hist_kernel(const u32* __restrict__ tc, u32* hist, u32 slots, const u32* __restrict__ go) {
    if (!*go) return;
    __shared__ u32 sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    // (8 loads of a thread in flight: the table is 2-32 MB, the kernel latency-bound)
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t s0 = blockIdx.x * blockDim.x + threadIdx.x; s0 < slots; s0 += 8 * stride) {
        u32 c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = s0 + u * stride < slots ? tc[s0 + u * stride] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c[u]) atomicAdd(&sh[c[u] < 255 ? c[u] : 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// One pass over the count table that also ORDERS the selection: the count
// histogram (levels min(count, 255)) gives, for every level, how many selected
// keys have a higher one, so a key of level L goes to hot[above(L) + its rank
// within L] -- a counting sort by sample count, hottest first, done by the
// CTAs that scan the table (hh_layout_kernel places the list in this order).
// thr = the smallest level >= 2 whose keys and everything above fit the
// candidate list; level thr - 1 (when >= 2) fills what capacity is left, first
// come first served.  Ranks within a level: one shared atomic per key, one
// global atomic per (CTA, level present).  hot_count[0] = keys listed.
constexpr int kSelThreads = 256;
constexpr int kSelPer = 8;
constexpr u32 kSelChunks = 4;
template <typename KeyT>
__global__ void __launch_bounds__(kSelThreads)
    hh_select_kernel(const KeyT* __restrict__ tk, const u32* __restrict__ tc, const u32* __restrict__ hist, u32 cap,
                     KeyT* hot, u32* hot_count, u32* hot_sum, u32* fill, u32 slots, const u32* __restrict__ go) {
    if (!*go) return;
    static_assert(kSelThreads == 256, "one histogram level per thread");
    __shared__ u32 sc[256], above[256], cnt[256], gbase[256], thr_s, cta_sum;
    const u32 t = threadIdx.x;
    const u32 mine = hist[255 - t];  // index t ascending = level descending
    sc[t] = mine;
    cnt[t] = 0;
    if (t == 0) {
        thr_s = 256;
        cta_sum = 0;
    }
    __syncthreads();
    for (u32 o = 1; o < 256; o <<= 1) {  // inclusive scan: sc[t] = keys of level >= 255 - t
        const u32 x = t >= o ? sc[t - o] : 0;
        __syncthreads();
        sc[t] += x;
        __syncthreads();
    }
    above[255 - t] = sc[t] - mine;
    if (255 - t >= 2 && sc[t] <= cap) atomicMin(&thr_s, 255 - t);
    __syncthreads();
    const u32 thr = thr_s;
    const u32 lmin = thr - 1 >= 2 ? thr - 1 : thr;  // lowest level listed
    if (blockIdx.x == 0 && t == 0) {
        const u32 listed = lmin < 256 ? above[lmin] + hist[lmin] : 0;
        hot_count[0] = listed < cap ? listed : cap;
    }
    // kSelChunks chunks of kSelThreads * kSelPer slots per CTA (the level scan above is
    // a fixed cost per CTA; the table has up to 2^23 slots)
    u32 covered = 0;
#pragma unroll 1
    for (u32 ch = 0; ch < kSelChunks; ++ch) {
        const uint32_t s0 = ((blockIdx.x * kSelChunks + ch) * kSelThreads + t) * kSelPer;
        if ((blockIdx.x * kSelChunks + ch) * kSelThreads * kSelPer >= slots) break;  // (uniform)
        u32 lev[kSelPer], rank[kSelPer], cs[kSelPer];
#pragma unroll
        for (int k = 0; k < kSelPer; ++k) {
            const u32 c = s0 + k < slots ? tc[s0 + k] : 0;
            const u32 l = c < 255 ? c : 255;
            cs[k] = c;
            lev[k] = l >= lmin ? l : 0;  // 0: not selected (lmin >= 2)
        }
#pragma unroll
        for (int k = 0; k < kSelPer; ++k)
            if (lev[k]) rank[k] = atomicAdd(&cnt[lev[k]], 1u);
        __syncthreads();
        if (cnt[t]) gbase[t] = above[t] + atomicAdd(fill + t, cnt[t]);
        __syncthreads();
        cnt[t] = 0;  // (read again only after the next chunk's barrier)
#pragma unroll
        for (int k = 0; k < kSelPer; ++k) {
            if (!lev[k]) continue;
            const u32 idx = gbase[lev[k]] + rank[k];
            if (idx < cap) {
                hot[idx] = tk[s0 + k];
                covered += cs[k];
            }
        }
        __syncthreads();
    }
    if (covered) atomicAdd(&cta_sum, covered);
    __syncthreads();
    if (t == 0 && cta_sum) atomicAdd(hot_sum, cta_sum);  // sampled items the hot set covers
}

// One CTA lays out the hot set in the two-choice table once for every CTA.
// The list arrives ordered by sample count, hottest first (hh_select_kernel),
// and is placed in that order, in rounds of growing
// size: a key goes to slot1 if free, else
// to slot2 if free; if both are taken, one level of cuckoo displacement moves
// the occupant of either slot to ITS other slot when that one is free.  Keys
// that still find no slot stay cold.  Exactness never depends on the layout:
// a lookup picks slot1 if it holds the key, else slot2, else the item is a miss,
// and hh_merge credits each slot's sum to the key stored there.
template <typename KeyT>
__device__ __forceinline__ u32 other_slot(KeyT k, u32 s) {
    using G = HotGeom<KeyT>;
    const u32 s1 = slot1<G::kSlots>(k);
    return s1 == s ? slot2<G::kSlots>(k) : s1;
}

// one placement round: N keys per thread, sorted[(r0 + i) * 1024 + tid] for r0 + i < r1
// (r1 - r0 <= N; the early rounds are small, and a round's cost on the one SM is
// mostly the instructions of its unrolled key slots, hence the sizes)
template <typename KeyT, u32 N>
__device__ __forceinline__ void place_round(KeyT* hk, const KeyT* __restrict__ sorted, u32 r0, u32 r1, u32 nhot) {
    using G = HotGeom<KeyT>;
    using C = typename G::Cas;
    constexpr uint32_t S = G::kSlots;
    KeyT rk[N];
#pragma unroll
    for (u32 i = 0; i < N; ++i) {
        const u32 j = (r0 + i) * 1024 + threadIdx.x;
        rk[i] = (r0 + i < r1 && j < nhot) ? sorted[j] : G::kEmpty;
    }
    // a claim is preceded by a plain load and skipped when the slot is seen taken
    // (slots never become free again); the claims of a thread's keys are
    // independent: first choices of all keys, then the second choices of those
    // that lost
    auto claim = [&](u32 slot, KeyT key) {
        return hk[slot] == G::kEmpty &&
               (KeyT)atomicCAS(reinterpret_cast<C*>(hk + slot), (C)G::kEmpty, (C)key) == G::kEmpty;
    };
    u32 left = 0;  // bit i: key rk[i] still has no slot
#pragma unroll
    for (u32 i = 0; i < N; ++i) {
        const KeyT key = rk[i];
        if (key == G::kEmpty) continue;
        if (!claim(slot1<S>(key), key)) left |= 1u << i;
    }
#pragma unroll
    for (u32 i = 0; i < N; ++i) {
        if (!((left >> i) & 1u)) continue;
        if (claim(slot2<S>(rk[i]), rk[i])) left &= ~(1u << i);
    }
    __syncthreads();
#pragma unroll
    for (u32 i = 0; i < N; ++i) {
        if (!((left >> i) & 1u)) continue;
        // one level of displacement (races only cost a slot, never exactness: a key
        // left in both its slots is always found in its slot1, and the copy never
        // collects a sum)
        const KeyT key = rk[i];
        const u32 s1 = slot1<S>(key), s2 = slot2<S>(key);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const u32 sl = t == 0 ? s1 : s2;
            const KeyT occ = hk[sl];
            if (occ == G::kEmpty || occ == key) break;
            const u32 alt = other_slot<KeyT>(occ, sl);
            if (alt == sl || !claim(alt, occ)) continue;
            atomicCAS(reinterpret_cast<C*>(hk + sl), (C)occ, (C)key);
            break;
        }
    }
    __syncthreads();
}

template <typename KeyT>
__global__ void __launch_bounds__(1024) hh_layout_kernel(const KeyT* __restrict__ sorted,
                                                         const u32* __restrict__ hot_count, u32 cap,
                                                         KeyT* __restrict__ layout,
                                                         const u32* __restrict__ priv_go) {
    if (priv_go && *priv_go == 0) return;  // the private byte tables took this stream: no hot set
    using G = HotGeom<KeyT>;
    constexpr uint32_t S = G::kSlots;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KeyT* hk = reinterpret_cast<KeyT*>(smem_raw);
    for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) hk[s] = G::kEmpty;
    const u32 nhot = min(hot_count[0], cap);
    __syncthreads();
    // placement rounds of doubling size (1, 1, 2, 4, 8, 16, ... keys per thread,
    // read coalesced from the count-sorted list): priority is fine-grained where
    // counts differ (the hottest keys) and coarse where they are nearly equal
    // (the many keys seen twice or three times); launched with 1024 threads
    constexpr u32 kRounds = G::kCap / 1024;
    constexpr u32 kMaxPer = 16;
#pragma unroll 1
    for (u32 r0 = 0, r1 = 1; r0 < kRounds && r0 * 1024 < nhot; r0 = r1, r1 = min(2 * r1, min(r1 + kMaxPer, kRounds))) {
        const u32 per = r1 - r0;
        if (per <= 1) place_round<KeyT, 1>(hk, sorted, r0, r1, nhot);
        else if (per <= 2) place_round<KeyT, 2>(hk, sorted, r0, r1, nhot);
        else if (per <= 4) place_round<KeyT, 4>(hk, sorted, r0, r1, nhot);
        else if (per <= 8) place_round<KeyT, 8>(hk, sorted, r0, r1, nhot);
        else place_round<KeyT, kMaxPer>(hk, sorted, r0, r1, nhot);
    }
    // the table as placed (empty slots hold the empty key), 16 bytes per store;
    // hh_slots_kernel turns it into what the scatter kernels copy
    static_assert((S * sizeof(KeyT)) % 16 == 0, "16-byte copies");
    const uint4* src = reinterpret_cast<const uint4*>(hk);
    uint4* dst = reinterpret_cast<uint4*>(layout);
    for (u32 j = threadIdx.x; j < S * sizeof(KeyT) / 16; j += blockDim.x) dst[j] = src[j];
}

// The slot contents the scatter kernels copy, one thread per slot (on the one
// layout SM this pass alone took ~13 us).  Tagged table (u32 keys): tags[s] =
// the placed key's tag for the slot it sits in (choice 1 only when it is not its
// slot1), else the empty marker; layout[] keeps the keys for hh_merge_kernel
// (empty slots never have a sum).  Untagged: an empty slot s gets a FOREIGN key,
// one with slot1 != s and slot2 != s: no lookup can match it, so the hot kernel
// needs no empty-slot test.
template <typename KeyT>
__global__ void __launch_bounds__(256) hh_slots_kernel(KeyT* __restrict__ layout, u32* __restrict__ tags,
                                                       u32* __restrict__ placed_out,
                                                       const u32* __restrict__ priv_go) {
    if (priv_go && *priv_go == 0) return;
    using G = HotGeom<KeyT>;
    constexpr uint32_t S = G::kSlots;
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned placed = 0;
    if (s < S) {
        KeyT k = layout[s];
        if constexpr (G::kTagged) {
            u32 t;
            if (k == G::kEmpty) {
                t = empty_tag<S>(s);
            } else {
                t = slot1<S>(k) == s ? tag1((u32)k) : tag2((u32)k);
                placed = 1;
            }
            tags[s] = t;
        } else {
            if (k == G::kEmpty) {
                for (KeyT t = 0;; ++t) {
                    k = G::kEmpty - t;
                    if (slot1<S>(k) != s && slot2<S>(k) != s) break;
                }
                layout[s] = k;
            } else {
                placed = 1;
            }
        }
    }
    placed = __reduce_add_sync(0xffffffffu, placed);
    if ((threadIdx.x & 31) == 0 && placed) atomicAdd(placed_out, placed);  // keys in the table (hot stats)
}

}  // namespace

template <typename KeyT>
cudaError_t launch_hot_select(const KeyT* keys, uint64_t n, uint32_t sample, const HotPrepWs<KeyT>& w, cudaStream_t s) {
    using G = HotGeom<KeyT>;
    const int sms = sm_count();
    hh_probe_kernel<KeyT><<<kProbeCtas, 1024, 0, s>>>(keys, n, w.go);
    // a share of kLocalSlots sampled items per CTA (its distinct keys fit the local
    // table: with 2 CTAs per SM a 2^22-item sample crowded it, 128 us against 50 us)
    uint32_t cgrid = (uint32_t)sms * 2;
    if ((sample + kLocalSlots - 1) / kLocalSlots > cgrid) cgrid = (sample + kLocalSlots - 1) / kLocalSlots;
    hh_count_kernel<KeyT><<<cgrid, kCountThreads, 0, s>>>(keys, sample, w.tk, w.tc, w.slots, w.go);
    hh_hist_kernel<<<sms * 8, 256, 0, s>>>(w.tc, w.hist, w.slots, w.go);
    constexpr u32 kSelCta = kSelThreads * kSelPer * kSelChunks;  // slots per CTA
    hh_select_kernel<KeyT><<<(w.slots + kSelCta - 1) / kSelCta, kSelThreads, 0, s>>>(
        w.tk, w.tc, w.hist, G::kCap, w.hot, w.hot_count, w.hot_sum, w.fill, w.slots, w.go);
    return cudaGetLastError();
}

template <typename KeyT>
cudaError_t launch_hot_layout(const HotPrepWs<KeyT>& w, KeyT* layout, uint32_t* tags, const uint32_t* priv_go,
                              cudaStream_t s) {
    using G = HotGeom<KeyT>;
    auto fl = hh_layout_kernel<KeyT>;
    const size_t lbytes = sizeof(KeyT) * G::kSlots;
    cudaError_t e = cudaFuncSetAttribute(fl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lbytes);
    if (e != cudaSuccess) return e;
    fl<<<1, 1024, lbytes, s>>>(w.hot, w.hot_count, G::kCap, layout, priv_go);
    hh_slots_kernel<KeyT><<<(G::kSlots + 255) / 256, 256, 0, s>>>(layout, tags, w.placed, priv_go);
    return cudaGetLastError();
}

template cudaError_t launch_hot_select<u32>(const u32*, uint64_t, uint32_t, const HotPrepWs<u32>&, cudaStream_t);
template cudaError_t launch_hot_select<u64>(const u64*, uint64_t, uint32_t, const HotPrepWs<u64>&, cudaStream_t);
template cudaError_t launch_hot_layout<u32>(const HotPrepWs<u32>&, u32*, uint32_t*, const uint32_t*, cudaStream_t);
template cudaError_t launch_hot_layout<u64>(const HotPrepWs<u64>&, u64*, uint32_t*, const uint32_t*, cudaStream_t);

}  // namespace mb200
