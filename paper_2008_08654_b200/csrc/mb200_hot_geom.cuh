// mb200_hot_geom.cuh -- the heavy-hitter table's geometry: slot choices, tags
// and sizes shared by the selection / layout kernels (kernels_hotprep.cu) and
// the scatter kernels (kernels_hot.cu).
#pragma once
#include "mb200_device.cuh"

namespace mb200 {
namespace {

template <typename KeyT>
struct HotGeom;
// u32 keys: a TAGGED slot, one 32-bit word = 14-bit cell (bits 18-31, the low
// 14 bits of the slot's sum, 2^13-biased) | choice bit (17) | 17-bit tag.  A
// key's two choices are the bijections pi1(K) = K c1 and pi2(K) = (K ^ K >> 15)
// c2 of the u32 key; slot_i = floor(pi_i S / 2^32) and tag_i = pi_i mod 2^17.
// The pi values of one slot form an interval of ceil(2^32 / S) = 80660 < 2^17
// values, so (slot, choice, tag) identifies the key exactly, and the value
// just below a slot's interval (mod 2^17) with choice 0 is a tag no key can
// have there: the empty-slot marker.  The cell sits in the word's top bits, so
// an add's carry leaves the word instead of touching the tag.  4 bytes per slot:
// 53248 slots in 208 KiB (35840 in the 6-byte key + 16-bit cell layout before;
// misses 10.8% -> ~9.7% on config 5).
// u64 keys: slot = 8-byte key + a 16-bit cell (two per 32-bit word).
// Slot counts need not be powers of 2.  The wraps of either cell go straight
// into the slot's shared total in HBM (hot_accumulate / tag_accumulate).
template <>
struct HotGeom<u32> {
    static constexpr bool kTagged = true;
    static constexpr uint32_t kSlots = 53248;  // x 4 B = 208 KiB
    static constexpr uint32_t kCap = 61440;    // selected candidates (the layout places ~46K)
    static constexpr u32 kEmpty = 0xffffffffu;
    using Cas = unsigned;
};
template <>
struct HotGeom<u64> {
    static constexpr bool kTagged = false;
    static constexpr uint32_t kSlots = 19456;  // x (8 B key + 2 B cell) = 190 KiB
    static constexpr uint32_t kCap = 16384;
    static constexpr u64 kEmpty = ~0ull;
    using Cas = unsigned long long;
};
constexpr u32 kTagMask = 0x3ffffu;  // choice bit + 17-bit tag
constexpr u32 kCellShift = 18;      // 14-bit cell in bits 18-31
constexpr u32 kCellBias = 0x2000u;

// two independent slot choices in [0, S): multiply-high range reduction of two
// independent 32-bit mixes (any S, not only powers of two)
template <uint32_t S>
__device__ __forceinline__ u32 slot_of(u32 h) {
    return (u32)(((u64)h * S) >> 32);
}
template <uint32_t S>
__device__ __forceinline__ u32 slot1(u32 key) {
    return slot_of<S>(key * 0x9E3779B1u);
}
template <uint32_t S>
__device__ __forceinline__ u32 slot2(u32 key) {
    return slot_of<S>((key ^ (key >> 15)) * 0x2C1B3C6Du);
}
// the tagged table's identity of key K in slot_i(K): tag_i(K) (choice bit i)
__device__ __forceinline__ u32 tag1(u32 key) { return (key * 0x9E3779B1u) & 0x1ffffu; }
__device__ __forceinline__ u32 tag2(u32 key) { return (((key ^ (key >> 15)) * 0x2C1B3C6Du) & 0x1ffffu) | 0x20000u; }
// empty-slot marker of slot s: choice 0, tag = (first pi1 value of the slot) - 1 mod 2^17
template <uint32_t S>
__device__ __forceinline__ u32 empty_tag(u32 s) {
    const u64 lo = (((u64)s << 32) + S - 1) / S;  // ceil(s 2^32 / S)
    return (u32)(lo - 1) & 0x1ffffu;
}
template <uint32_t S>
__device__ __forceinline__ u32 slot1(u64 key) {
    return slot_of<S>((u32)(mix64(key) >> 32));
}
template <uint32_t S>
__device__ __forceinline__ u32 slot2(u64 key) {
    return slot_of<S>((u32)mix64(key));
}

}  // namespace
}  // namespace mb200
