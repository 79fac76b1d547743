// mb200_sketch_dev.cuh -- device building blocks shared by the Count Sketch
// kernels (kernels_sketch.cu, kernels_hot.cu): per-family Horner hashing,
// the two-for-one / arbitrary-width splitters and the fused per-item update.
// Reference: CountSketch::process sketch.cpp:133-140, split_pow2 :13-19,
// split_arb_* :21-34.
#pragma once
#include <cstdint>

#include "mb200_device.cuh"
#include "mb200_internal.h"
#include "mb200_mem.cuh"

namespace mb200 {
namespace sk {

constexpr int kSlots = 4;  // items per lane per warp-iteration (loads in flight)
constexpr unsigned kFull = 0xffffffffu;

enum Mode { M61_K32 = 0, M61_K64 = 1, M89 = 2, MGEN = 3, MWIDE = 4 };  // MWIDE: 62 <= b <= 127
enum Strat { SMEM32 = 0, SMEM64 = 1, GLOBAL = 2, SMEM_LOHI = 3 };
constexpr uint32_t kLohiCells = 8192;  // SMEM_LOHI table capacity (2 x 32 KiB)

template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) {
    return __ldcs(p);
}

// 61-bit (or <= 61-bit generic) hash of family f, fully reduced.
template <int MODE, int K>
__device__ __forceinline__ u64 hash_small(const SketchParams& sp, uint32_t f, u64 x) {
    const u64* c = sp.lo + (size_t)f * sp.k;
    if (MODE == M61_K32) {
        const u32 xs = (u32)x;
        if (K > 0) {
            u64 y = c[K - 1];
#pragma unroll
            for (int i = K - 2; i >= 0; --i) y = h61_step32(y, xs, c[i]);
            return h61_finish(y);
        }
        u64 y = c[sp.k - 1];
#pragma unroll 1
        for (int i = (int)sp.k - 2; i >= 0; --i) y = h61_step32(y, xs, c[i]);
        return h61_finish(y);
    } else if (MODE == M61_K64) {
        const u64 xr = h61_key64(x);
        if (K > 0) return h61_finish(h61_eval64<K>(c, xr));
        return h61_finish(h61_eval64_rt(c, (int)sp.k, xr));
    } else {
        u64 y = c[sp.k - 1];
#pragma unroll 1
        for (int i = (int)sp.k - 2; i >= 0; --i) y = hgen_step(y, x, c[i], sp.b, sp.p);
        return hgen_finish(y, sp.b, sp.p);
    }
}

// 2^61-1 hash of family f before the final reduction (any value < 2^64 that is
// congruent to the hash mod p): for splitters that reduce on their own.
template <int MODE, int K>
__device__ __forceinline__ u64 hash61_lazy(const SketchParams& sp, uint32_t f, u64 x) {
    static_assert(MODE == M61_K32 || MODE == M61_K64, "2^61-1 modes only");
    const u64* c = sp.lo + (size_t)f * sp.k;
    if (MODE == M61_K32) {
        const u32 xs = (u32)x;
        if (K < 2) return c[0];
        u64 y = h61_step32_first(c[K - 1], xs, c[K - 2]);
#pragma unroll
        for (int i = K - 3; i >= 0; --i) y = h61_step32(y, xs, c[i]);
        return y;
    }
    return h61_eval64<K>(c, h61_key64(x));
}

// 89-bit hash of family f as (lo 64 bits, hi 25 bits).
template <int K>
__device__ __forceinline__ void hash89(const SketchParams& sp, uint32_t f, u64 x, u64& lo, u64& hi) {
    const u64* cl = sp.lo + (size_t)f * sp.k;
    const u64* ch = sp.hi + (size_t)f * sp.k;
    const int k = K > 0 ? K : (int)sp.k;
    u32 y0 = lo32(cl[k - 1]), y1 = hi32(cl[k - 1]), y2 = lo32(ch[k - 1]);
    const u32 x0 = lo32(x), x1 = hi32(x);
    if (K > 0) {
#pragma unroll
        for (int i = K - 2; i >= 0; --i)
            h89_step(y0, y1, y2, x0, x1, lo32(cl[i]), hi32(cl[i]), lo32(ch[i]));
    } else {
#pragma unroll 1
        for (int i = k - 2; i >= 0; --i)
            h89_step(y0, y1, y2, x0, x1, lo32(cl[i]), hi32(cl[i]), lo32(ch[i]));
    }
    h89_finish(y0, y1, y2);
    lo = ((u64)y1 << 32) | y0;
    hi = y2;
}

// Alg 2 and the arbitrary-width splitters on a hash h < 2^b (b <= 64 path).
// Returns the counter index within the row and writes the sign bit
// (1 means "subtract delta").
__device__ __forceinline__ u64 split_small(const SketchParams& sp, u64 h, uint32_t sub, bool& neg) {
    const u32 b = sp.b;
    switch (sp.splitter) {
        case SPLIT_POW2:  // sketch.cpp:13-19: index = low l bits, sign = 1 - 2 * top bit
            neg = (h >> (b - 1)) & 1;
            return h & (sp.width - 1);
        case SPLIT_TWO_FOR_ONE:  // bits [l sub, l sub + l), sign bit b-1-sub
            neg = (h >> (b - 1 - sub)) & 1;
            return (h >> (sp.lw * sub)) & (sp.width - 1);
        default: {  // sketch.cpp:21-34: j = low b-1 bits (+1 for Mersenne), (j r) >> (b-1)
            u64 hh = h + (sp.splitter == SPLIT_MERSENNE_ARB ? 1 : 0);
            neg = !((hh >> (b - 1)) & 1);  // sign = 2a - 1: top bit set -> +1
            const u64 j = hh & ((1ull << (b - 1)) - 1);
            const u64 plo = j * sp.width, phi = __umul64hi(j, sp.width);
            const u32 s = b - 1;
            return (phi << (64 - s)) | (plo >> s);
        }
    }
}

__device__ __forceinline__ u64 split89(const SketchParams& sp, u64 lo, u64 hi, uint32_t sub, bool& neg) {
    // b = 89: sign bit 88 - sub lives in the high word (bits 64..88)
    if (sp.splitter == SPLIT_POW2) {
        neg = (hi >> 24) & 1;
        return lo & (sp.width - 1);
    }
    neg = (hi >> (24 - sub)) & 1;
    return (lo >> (sp.lw * sub)) & (sp.width - 1);
}

// hash of family f for 62 <= b <= 127 (any splitter), as (lo 64 bits, hi bits)
__device__ __forceinline__ void hash_wide_f(const SketchParams& sp, uint32_t f, u64 x, u64& lo, u64& hi) {
    hash_wide(sp.lo + (size_t)f * sp.k, sp.hi + (size_t)f * sp.k, (int)sp.k, sp.b, x, lo, hi);
}

// Every splitter on a 128-bit hash h < 2^b, 62 <= b <= 127 (sketch.cpp:13-34;
// map_pow2 bucketing.cpp:61-66 = (j r) >> (b - 1)); index < width < 2^34.
__device__ __forceinline__ u64 split_wide(const SketchParams& sp, u64 lo, u64 hi, uint32_t sub, bool& neg) {
    const u32 b = sp.b;
    auto bit = [&](u64 l, u64 h, u32 pos) -> bool { return pos >= 64 ? (h >> (pos - 64)) & 1 : (l >> pos) & 1; };
    if (sp.splitter == SPLIT_POW2) {  // index = low l bits, sign = 1 - 2 * bit b-1
        neg = bit(lo, hi, b - 1);
        return lo & (sp.width - 1);
    }
    if (sp.splitter == SPLIT_TWO_FOR_ONE) {  // bits [l sub, l sub + l) (2 l <= 64), sign bit b-1-sub
        neg = bit(lo, hi, b - 1 - sub);
        return (lo >> (sp.lw * sub)) & (sp.width - 1);
    }
    u64 l2 = lo, h2 = hi;
    if (sp.splitter == SPLIT_MERSENNE_ARB) {  // split_arb_uniform(h + 1, ...), h < p
        l2 = lo + 1;
        h2 = hi + (l2 == 0);
    }
    const u32 s = b - 1;        // >= 61
    neg = !bit(l2, h2, s);      // sign = 2 a - 1
    const u64 jl = s >= 64 ? l2 : l2 & ((1ull << s) - 1);
    const u64 jh = s > 64 ? h2 & ((1ull << (s - 64)) - 1) : 0;
    const u64 r = sp.width;     // < 2^34
    const u64 p1l = jl * r, p1h = __umul64hi(jl, r);
    const u64 p2l = jh * r, p2h = __umul64hi(jh, r);
    const u64 mid = p1h + p2l;
    const u64 top = p2h + (mid < p1h);
    if (s < 64) return (p1l >> s) | (mid << (64 - s));
    if (s == 64) return mid;
    return (mid >> (s - 64)) | (top << (128 - s));
}

template <int WK>
__device__ __forceinline__ i64 load_weight(const void* w, uint64_t i) {
    if (WK == W_NONE) return 1;
    if (WK == W_I32) return (i64)ld_nc(reinterpret_cast<const i32*>(w) + i);
    return ld_nc(reinterpret_cast<const i64*>(w) + i);
}

template <int STRAT>
__device__ __forceinline__ void table_add(void* smem, i64* table, u64 cell, u64 sd) {
    if (STRAT == SMEM32) {
        atomicAdd(reinterpret_cast<unsigned*>(smem) + cell, (unsigned)sd);
    } else if (STRAT == SMEM_LOHI) {
        // exact 64-bit counter as a 2^31-biased low word + wrap counter, on native
        // 32-bit shared atomics (|sd| <= 2^31; sm_100 has no 64-bit shared add)
        u32* lo = reinterpret_cast<u32*>(smem);
        const u32 dd = (u32)sd;
        const u32 old = atomicAdd(lo + cell, dd);
        const u32 nw = old + dd;
        const int carry = (i64)sd >= 0 ? (int)(nw < old) : -(int)(nw > old);
        if (carry) atomicAdd(lo + kLohiCells + cell, (u32)carry);
    } else if (STRAT == SMEM64) {
        red_add_shared_u64(reinterpret_cast<uint64_t*>(smem) + cell, sd);
    } else {
        red_add_u64(reinterpret_cast<uint64_t*>(table) + cell, sd);
    }
}

// One item: every family, every sub-row.  delta is applied with the
// reference's wrapping sign convention (sketch.cpp:136-138).
template <int MODE, int K, int STRAT>
__device__ __forceinline__ void process_item(const SketchParams& sp, u64 x, i64 delta, void* smem,
                                             i64* table) {
    const u64 d = (u64)delta;
    if (MODE == M89 || MODE == MWIDE) {
        const uint32_t subs = sp.splitter == SPLIT_TWO_FOR_ONE ? 2 : 1;
#pragma unroll 1
        for (uint32_t f = 0; f < sp.families; ++f) {
            u64 hlo, hhi;
            if (MODE == M89) hash89<K>(sp, f, x, hlo, hhi);
            else hash_wide_f(sp, f, x, hlo, hhi);
            for (uint32_t s = 0; s < subs; ++s) {
                const uint32_t row = subs * f + s;
                if (row >= sp.rows) break;
                bool neg;
                const u64 idx = MODE == M89 ? split89(sp, hlo, hhi, s, neg) : split_wide(sp, hlo, hhi, s, neg);
                table_add<STRAT>(smem, table, (u64)row * sp.width + idx, neg ? (0ull - d) : d);
            }
        }
    } else {
        if (sp.splitter == SPLIT_TWO_FOR_ONE) {
#pragma unroll 1
            for (uint32_t f = 0; f < sp.families; ++f) {
                const u64 h = hash_small<MODE, K>(sp, f, x);
                for (uint32_t s = 0; s < 2; ++s) {
                    const uint32_t row = 2 * f + s;
                    if (row >= sp.rows) break;
                    bool neg;
                    const u64 idx = split_small(sp, h, s, neg);
                    table_add<STRAT>(smem, table, (u64)row * sp.width + idx, neg ? (0ull - d) : d);
                }
            }
        } else {
#pragma unroll 1
            for (uint32_t f = 0; f < sp.families; ++f) {
                const u64 h = hash_small<MODE, K>(sp, f, x);
                bool neg;
                const u64 idx = split_small(sp, h, 0, neg);
                table_add<STRAT>(smem, table, (u64)f * sp.width + idx, neg ? (0ull - d) : d);
            }
        }
    }
}

// U independent items at once: for each family the U Horner chains are issued
// back to back (instruction-level parallelism across items), then split and
// scattered.  Same arithmetic and update order per item as process_item.
template <int MODE, int K, int STRAT, int U, int FAM = 0, typename KeyT>
__device__ __forceinline__ void process_items(const SketchParams& sp, const KeyT (&x)[U], const i64 (&delta)[U],
                                              unsigned valid, void* smem, i64* table) {
    if (FAM == 1 && MODE != M89 && MODE != MWIDE) {
        // one family, Pow2 splitter (the caller checked): no loops, no splitter switch
        u64 h[U];
#pragma unroll
        for (int u = 0; u < U; ++u) h[u] = hash_small<MODE, K>(sp, 0, (u64)x[u]);
        const u32 top = sp.b - 1;
        const u64 mask = sp.width - 1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!((valid >> u) & 1)) continue;
            const u64 d = (u64)delta[u];
            table_add<STRAT>(smem, table, h[u] & mask, ((h[u] >> top) & 1) ? (0ull - d) : d);
        }
        return;
    }
    if (MODE == M89 || MODE == MWIDE) {
        const uint32_t subs = sp.splitter == SPLIT_TWO_FOR_ONE ? 2 : 1;
#pragma unroll 1
        for (uint32_t f = 0; f < sp.families; ++f) {
            u64 hlo[U], hhi[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (MODE == M89) hash89<K>(sp, f, (u64)x[u], hlo[u], hhi[u]);
                else hash_wide_f(sp, f, (u64)x[u], hlo[u], hhi[u]);
            }
            for (uint32_t s = 0; s < subs; ++s) {
                const uint32_t row = subs * f + s;
                if (row >= sp.rows) break;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!((valid >> u) & 1)) continue;
                    bool neg;
                    const u64 idx = MODE == M89 ? split89(sp, hlo[u], hhi[u], s, neg)
                                                : split_wide(sp, hlo[u], hhi[u], s, neg);
                    const u64 d = (u64)delta[u];
                    table_add<STRAT>(smem, table, (u64)row * sp.width + idx, neg ? (0ull - d) : d);
                }
            }
        }
    } else {
        const uint32_t subs = sp.splitter == SPLIT_TWO_FOR_ONE ? 2 : 1;
#pragma unroll 1
        for (uint32_t f = 0; f < sp.families; ++f) {
            u64 h[U];
#pragma unroll
            for (int u = 0; u < U; ++u) h[u] = hash_small<MODE, K>(sp, f, (u64)x[u]);
            for (uint32_t s = 0; s < subs; ++s) {
                const uint32_t row = subs * f + s;
                if (row >= sp.rows) break;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!((valid >> u) & 1)) continue;
                    bool neg;
                    const u64 idx = split_small(sp, h[u], s, neg);
                    const u64 d = (u64)delta[u];
                    table_add<STRAT>(smem, table, (u64)row * sp.width + idx, neg ? (0ull - d) : d);
                }
            }
        }
    }
}

}  // namespace sk
}  // namespace mb200
