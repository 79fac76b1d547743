// mb200_private89.cuh -- config 4's shape as its own kernel: one 2^89-1
// degree-3 family, two-for-one split into two rows of 2^LW counters, unit
// deltas, a stream without heavy hitters (reference hash
// polyhash.cpp:78-88 + field.hpp:66-73, split sketch.cpp:13-19 applied to h and
// to (h >> l) & (2^72 - 1), process sketch.cpp:133-140).
//
// Included by kernels_hot.cu (it shares the heavy-hitter probe's go flag and
// the g_hot_stats counters).  Everything the generic private kernel decides at
// run time is fixed here: the coefficients are 12 words of the parameter bank
// (uniform-register operands, no loads), the family loop and row checks are
// gone, keys arrive two per 16-byte load, and
//
//   * the 89-bit Horner step is schoolbook over 32-bit limbs written as
//     mad.wide chains (y_i x_j + hi + lo <= 2^64 - 1 never overflows), which
//     ptxas turns into 6 IMAD.WIDE + 3-input IADD3 carry pairs (12 separate
//     IMAD / IMAD.HI and their carry materialisation before), with the work
//     split between the FMA-heavy and ALU pipes that bind it;
//   * the final reduction produces only what the two splits read: the low 32
//     bits of h = y mod p and its bits 87, 88 (if y >= p then h < 2^65 and both
//     sign bits are 0);
//   * the byte cells (2^7-biased, four per word, one shared atomic per row
//     update, exact carry accounting to L2 exactly as byte_add) take ONE
//     out-of-line branch per four keys, after their hashes and atomics;
//   * the per-CTA tables are NOT merged with one L2 reduction per cell (148 x
//     2^17 = 19.4M reductions, ~0.1 ms at the L2 atomic rate): each CTA writes
//     its table to a scratch area (128 KiB per CTA, L2-resident) with 16-byte
//     stores and private_fold_kernel sums the 148 tables per cell.
#pragma once

#include <cooperative_groups.h>

namespace mb200 {
namespace {

static __constant__ u32 kFma128 = 128;
static __constant__ u32 kFmaM3 = 0xfffffffdu;   // -3
static __constant__ u32 kFma512 = 512;
static __constant__ u32 kFma8 = 8;
static __constant__ u32 kFma64K = 65536;
static __constant__ u32 kFmaM2 = 0xfffffffeu;   // -2

struct Coef89 {
    u32 a[4][3];  // coefficient j = a[j][0] + a[j][1] 2^32 + a[j][2] 2^64 (a[j][2] < 2^25)
};

// y <- y x + a (mod 2^89 - 1), lazily reduced: y < 2^90 in and out
// (y2 < 2^26), x < 2^64, a < 2^89.  t = y x + a < 2^154 + 2^89 as five words
// w0..w4, then the reference's single partial fold (t & p) + (t >> 89)
// < 2^89 + 2^65 (field.hpp:66-73).  Row x0: r_i = y_i x0 + hi(r_{i-1}) + a_i;
// row x1: s_i = y_i x1 + hi(s_{i-1}) + w_{i+1}; every r_i, s_i is a product of
// two words plus at most two words (<= 2^64 - 1, never overflows).
//
// Pipe balance (measured, tools/kvariants/c4_variants.py): the kernel is bound
// by the FMA-heavy pipe (every IMAD; an IMAD.WIDE takes two of its slots) and
// the ALU pipe together.  The three coefficient words enter on the FMA pipe
// (mad.wide by a runtime 1), the other carries and the fold stay on the ALU
// pipe.  Measured alternatives at config 4: all carries on the ALU 338 us, all
// on the FMA pipe 445-515 us, the fold's shifts as IMAD.HI / IMAD 360 us,
// against 325 us for this form.
__device__ __forceinline__ void h89_step_w(u32& y0, u32& y1, u32& y2, u32 x0, u32 x1, u32 a0, u32 a1, u32 a2) {
    u32 w0, w1, w2, w3, w4;
    asm("{\n\t"
        ".reg .u32 r0h, r1l, r1h, r2l, r2h, s0h, s1h;\n\t"
        ".reg .u64 R0, R1, R2, S0, S1, S2, Z;\n\t"
        "mul.wide.u32 R0, %5, %8;\n\t"
        "mad.wide.u32 R0, %10, %13, R0;\n\t"  // y0 x0 + a0
        "mov.b64 {%0, r0h}, R0;\n\t"
        "mov.b64 Z, {r0h, 0};\n\t"
        "mad.wide.u32 R1, %6, %8, Z;\n\t"
        "mad.wide.u32 R1, %11, %13, R1;\n\t"  // y1 x0 + hi + a1
        "mov.b64 {r1l, r1h}, R1;\n\t"
        "mov.b64 Z, {r1h, 0};\n\t"
        "mad.wide.u32 R2, %7, %8, Z;\n\t"
        "mad.wide.u32 R2, %12, %13, R2;\n\t"  // y2 x0 + hi + a2
        "mov.b64 {r2l, r2h}, R2;\n\t"
        "mov.b64 Z, {r1l, 0};\n\t"
        "mad.wide.u32 S0, %5, %9, Z;\n\t"  // y0 x1 + w1
        "mov.b64 {%1, s0h}, S0;\n\t"
        "mov.b64 Z, {s0h, 0};\n\t"
        "mad.wide.u32 S1, %6, %9, Z;\n\t"  // y1 x1 + hi + w2
        "mov.b64 Z, {r2l, 0};\n\t"
        "add.u64 S1, S1, Z;\n\t"
        "mov.b64 {%2, s1h}, S1;\n\t"
        "mov.b64 Z, {s1h, 0};\n\t"
        "mad.wide.u32 S2, %7, %9, Z;\n\t"  // y2 x1 + hi + w3
        "mov.b64 Z, {r2h, 0};\n\t"
        "add.u64 S2, S2, Z;\n\t"
        "mov.b64 {%3, %4}, S2;\n\t"
        "}"
        : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3), "=r"(w4)
        : "r"(y0), "r"(y1), "r"(y2), "r"(x0), "r"(x1), "r"(a0), "r"(a1), "r"(a2), "r"(kFmaOne));
    const u32 l2 = w2 & kP89Top;
    const u32 h0 = __funnelshift_r(w2, w3, 25);
    const u32 h1 = __funnelshift_r(w3, w4, 25);
    const u32 h2 = w4 >> 25;
    asm("add.cc.u32  %0, %3, %6;\n\t"
        "addc.cc.u32 %1, %4, %7;\n\t"
        "addc.u32    %2, %5, %8;"
        : "=r"(y0), "=r"(y1), "=r"(y2)
        : "r"(w0), "r"(w1), "r"(l2), "r"(h0), "r"(h1), "r"(h2));
}

// h = (sum_j a_j x^j) mod p, reduced to the bits the two-for-one split reads:
// lo = h mod 2^32 and top = (h >> 87) & 3 (bit 1 = bit 88, bit 0 = bit 87).
// The last fold leaves y < 2^89 + 2^65: z = (y + 1) >> 89 is 1 exactly when
// y >= p, and then h = y + 1 - 2^89 < 2^65 + 1 (low word y0 + 1, bits 87 and
// 88 clear) -- the reference's branch-free finish (polyhash.cpp:74-75) cut
// down to the bits the splits read.
__device__ __forceinline__ void hash89_c4(const Coef89& c, u64 x, u32& lo, u32& top) {
    const u32 x0 = lo32(x), x1 = hi32(x);
    u32 y0 = c.a[3][0], y1 = c.a[3][1], y2 = c.a[3][2];
    h89_step_w(y0, y1, y2, x0, x1, c.a[2][0], c.a[2][1], c.a[2][2]);
    h89_step_w(y0, y1, y2, x0, x1, c.a[1][0], c.a[1][1], c.a[1][2]);
    h89_step_w(y0, y1, y2, x0, x1, c.a[0][0], c.a[0][1], c.a[0][2]);
    // z = (y + 1) >> 89 exactly (one carry chain), the rest on the FMA pipe:
    // lo = y0 + z, top = (y2 >> 23) & (3 - 3 z)
    asm("{\n\t.reg .u32 t0, t1, s2, z, m;\n\t"
        "add.cc.u32  t0, %2, 1;\n\t"
        "addc.cc.u32 t1, %3, 0;\n\t"
        "addc.u32    s2, %4, 0;\n\t"
        "mul.hi.u32  z, s2, %5;\n\t"      // s2 >> 25 (s2 < 2^26)
        "mad.lo.u32  %0, z, %6, %2;\n\t"  // y0 + z
        "mad.lo.u32  m, z, %7, 3;\n\t"    // 3 - 3 z
        "mul.hi.u32  t1, %4, %8;\n\t"     // y2 >> 23
        "and.b32     %1, t1, m;\n\t}"
        : "=r"(lo), "=r"(top)
        : "r"(y0), "r"(y1), "r"(y2), "r"(kFma128), "r"(kFmaOne), "r"(kFmaM3), "r"(kFma512));
}

// One +-1 row update of a byte cell (2^7-biased, four per word).  The word
// before the add comes back from the atomic; the cell left [0, 2^8) exactly
// when bit 8 of (b + d) differs from bit 8 of b, b = old >> 8q.
struct CellUpd {
    u32 cell, old, dw;
    i32 d;
    // bit 8 set: the cell left [0, 2^8)
    __device__ __forceinline__ u32 left_bit() const {
        const u32 b = old >> ((cell & 3u) << 3);
        return (b + (u32)d) ^ b;
    }
};
__device__ __forceinline__ CellUpd cell_add(u32* words, u32 cell, bool neg) {
    CellUpd u;
    u.cell = cell;
    u.d = neg ? -1 : 1;
    u.dw = (u32)u.d << ((cell & 3u) << 3);
    u.old = atomicAdd(words + (cell >> 2), u.dw);
    return u;
}
// the cell left [0, 2^8): record (intended - displayed) change of every byte
// the carry / borrow reached (byte_add's accounting)
__device__ __noinline__ void cell_fix(uint64_t* l2, u32 cell, i32 d, u32 old, u32 dw) {
    const u32 q = cell & 3u, base = cell & ~3u;
    const u32 nw = old + dw;
    for (u32 j = q; j < 4; ++j) {
        const i32 disp = (i32)((nw >> (8 * j)) & 0xffu) - (i32)((old >> (8 * j)) & 0xffu);
        const i32 rec = (j == q ? d : 0) - disp;
        if (rec) red_add_u64(l2 + base + j, (u64)(i64)rec);
    }
}

constexpr int kP89Threads = 1024;
#ifndef C4PAIRS
#define C4PAIRS 4
#endif
#ifndef C4KP
#define C4KP 8
#endif
// 16-byte key pairs in flight per thread and keys per branch-free phase, measured
// with the final scatter (tools/kvariants/c4_variants.py): 4 pairs in one phase of
// 8 keys 310 us, 8 pairs in phases of 4 keys 318 us (the choice before the
// scatter lost its shifts), 6 / 12 310 us, 3 / 6 319 us, 2 / 4 331 us
constexpr int kP89Pairs = C4PAIRS;
constexpr int kC4KP = C4KP;

template <int LW>
__device__ __forceinline__ void key_c4(const Coef89& c, u64 x, u32* words, uint64_t* l2) {
    constexpr u32 W = 1u << LW;
    u32 lo, top;
    hash89_c4(c, x, lo, top);
    const CellUpd u0 = cell_add(words, lo & (W - 1), top >> 1);
    const CellUpd u1 = cell_add(words, W + ((lo >> LW) & (W - 1)), top & 1u);
    const u32 l0 = u0.left_bit(), l1 = u1.left_bit();
    if (__builtin_expect(((l0 | l1) & 0x100u) != 0, 0)) {
        if (l0 & 0x100u) cell_fix(l2, u0.cell, u0.d, u0.old, u0.dw);
        if (l1 & 0x100u) cell_fix(l2, u1.cell, u1.d, u1.old, u1.dw);
    }
}

// KP keys at once, in phases with no branch between them: KP independent
// Horner chains (the scheduler interleaves them), then 2 KP shared atomics,
// then ONE test of every cell for leaving [0, 2^8) (almost never true; the
// words before the adds are kept for the fix-up).  A branch after every key
// would stop the chains of the next keys from starting before it.
template <int LW, int KP>
__device__ __forceinline__ void keys_c4(const Coef89& c, const u64 (&x)[KP], u32* words, uint64_t* l2) {
    constexpr u32 W = 1u << LW;
    u32 lo[KP], top[KP];
#pragma unroll
    for (int u = 0; u < KP; ++u) hash89_c4(c, x[u], lo[u], top[u]);
    // Trigger of the out-of-line fix-up: conservative and shift-free.  A byte within
    // 2^6 of a wrap has bit 7 == bit 6, i.e. bit 7 of o ^ 2o clear; the AND over both
    // words of every key keeps bit 7 of each byte lane set while no byte of any touched
    // word is that close (two ALU ops per update instead of three; 332 -> 325 us).  The
    // exact per-update test below then decides which cells really left [0, 2^8).
    u32 old[2 * KP], safe = 0xffffffffu;
#pragma unroll
    for (int u = 0; u < KP; ++u) {
        static_assert(LW == 16, "cell arithmetic below is for 2^16-cell rows");
        // shifts by constants and the +-1 on the FMA pipe (runtime multipliers)
        // the byte shift 8 (cell & 3) is the low 5 bits of 8 cell: a wrap-mode funnel
        // shift takes them itself (no mask; 325 -> 321 us)
        u32 hi16, s0, s1, d0, d1;
        asm("{\n\t.reg .u32 t;\n\t"
            "mul.hi.u32 %0, %5, %7;\n\t"       // lo >> 16
            "mul.lo.u32 %1, %5, %8;\n\t"       // 8 lo
            "mul.lo.u32 %2, %0, %8;\n\t"       // 8 (lo >> 16)
            "mul.hi.u32 t, %6, %9;\n\t"        // top >> 1
            "mad.lo.u32 %3, t, %10, 1;\n\t"    // 1 - 2 (top >> 1)
            "and.b32    t, %6, 1;\n\t"
            "mad.lo.u32 %4, t, %10, 1;\n\t}"   // 1 - 2 (top & 1)
            : "=r"(hi16), "=r"(s0), "=r"(s1), "=r"(d0), "=r"(d1)
            : "r"(lo[u]), "r"(top[u]), "r"(kFma64K), "r"(kFma8), "r"(0x80000000u), "r"(kFmaM2));
        const u32 dw0 = __funnelshift_l(0u, d0, s0), dw1 = __funnelshift_l(0u, d1, s1);
        const u32 o0 = atomicAdd(words + ((lo[u] & 0xfffcu) >> 2), dw0);
        const u32 o1 = atomicAdd(words + W / 4 + ((hi16 & 0xfffcu) >> 2), dw1);
        old[2 * u] = o0;
        old[2 * u + 1] = o1;
        safe &= (o0 ^ (o0 + o0)) & (o1 ^ (o1 + o1));
    }
    if (__builtin_expect((safe & 0x80808080u) != 0x80808080u, 0)) {  // (unrolled: the arrays stay in registers)
#pragma unroll
        for (int u = 0; u < KP; ++u) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                CellUpd v;
                v.cell = r ? W + ((lo[u] >> LW) & (W - 1)) : lo[u] & (W - 1);
                v.d = ((r ? top[u] : top[u] >> 1) & 1u) ? -1 : 1;
                v.dw = (u32)v.d << ((v.cell & 3u) << 3);
                v.old = old[2 * u + r];
                if (v.left_bit() & 0x100u) cell_fix(l2, v.cell, v.d, v.old, v.dw);
            }
        }
    }
}

// keys as 16-byte pairs [0, npairs) (+ one odd last key, taken by CTA 0);
// each CTA a contiguous share.  The CTA's byte table goes to scratch[blockIdx]
// (2^(LW+1) bytes), summed by private_fold_kernel.
template <int LW, bool FUSED>
__global__ void __launch_bounds__(kP89Threads, 1)
    cs_private89_kernel(const Coef89 c, const ulonglong2* __restrict__ kv, uint64_t npairs, const u64* __restrict__ odd,
                        uint4* __restrict__ scratch, uint64_t* __restrict__ l2, const u32* __restrict__ go) {
    if (go && *go) return;
    extern __shared__ __align__(16) u32 pwords[];
    constexpr u32 kWords = (2u << LW) / 4;
    uint4* pw4 = reinterpret_cast<uint4*>(pwords);
    for (u32 i = threadIdx.x; i < kWords / 4; i += kP89Threads) pw4[i] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    __syncthreads();
    const uint64_t lo = npairs * blockIdx.x / gridDim.x, hi = npairs * (blockIdx.x + 1) / gridDim.x;
    uint64_t i = lo + threadIdx.x;
    for (; i + (kP89Pairs - 1) * kP89Threads < hi; i += kP89Pairs * kP89Threads) {
        ulonglong2 v[kP89Pairs];
#pragma unroll
        for (int u = 0; u < kP89Pairs; ++u) v[u] = __ldcs(kv + i + u * kP89Threads);
#pragma unroll
        for (int h = 0; h < kP89Pairs; h += kC4KP / 2) {
            u64 x[kC4KP];
#pragma unroll
            for (int u = 0; u < kC4KP / 2; ++u) {
                x[2 * u] = v[h + u].x;
                x[2 * u + 1] = v[h + u].y;
            }
            keys_c4<LW, kC4KP>(c, x, pwords, l2);
        }
    }
    for (; i < hi; i += kP89Threads) {
        const ulonglong2 v = __ldcs(kv + i);
        key_c4<LW>(c, v.x, pwords, l2);
        key_c4<LW>(c, v.y, pwords, l2);
    }
    if (odd && blockIdx.x == 0 && threadIdx.x == 0) key_c4<LW>(c, *odd, pwords, l2);
    __syncthreads();
    uint4* dst = scratch + (size_t)blockIdx.x * (kWords / 4);
    for (u32 j = threadIdx.x; j < kWords / 4; j += kP89Threads) dst[j] = pw4[j];
    if (threadIdx.x == 0) atomicAdd(&g_hot_stats[0], (unsigned long long)(2 * (hi - lo) + (odd && blockIdx.x == 0)));
    if constexpr (FUSED) {
        // cooperative launch: every CTA's table is in scratch after the grid barrier;
        // CTA b then folds its share of the 16-byte columns (64 columns x 16 groups
        // of CTAs per pass, partial sums in the freed shared table)
        cooperative_groups::this_grid().sync();
        constexpr u32 cols = kWords / 4, kC = 64, kG = kP89Threads / kC;
        const u32 per = (cols + gridDim.x - 1) / gridDim.x;
        const u32 ci = threadIdx.x % kC, grp = threadIdx.x / kC;
        i32(*part)[kC][17] = reinterpret_cast<i32(*)[kC][17]>(pwords);
        for (u32 c0 = blockIdx.x * per; c0 < min((blockIdx.x + 1) * per, cols); c0 += kC) {
            const u32 col = c0 + ci;
            const bool live = ci < per && col < min((blockIdx.x + 1) * per, cols);
            i32 acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0;
            if (live) {
                for (u32 cta = grp; cta < gridDim.x; cta += kG) {
                    const uint4 v = __ldcg(scratch + (size_t)cta * cols + col);
                    const u32 wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int w = 0; w < 4; ++w)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[4 * w + b] += (i32)((wv[w] >> (8 * b)) & 0xffu);
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 16; ++j) part[grp][ci][j] = acc[j];
            __syncthreads();
            if (live) {  // thread (ci, grp) finishes cell grp of column ci
                i32 v = -0x80 * (i32)gridDim.x;
#pragma unroll
                for (int g = 0; g < (int)kG; ++g) v += part[g][ci][grp];
                if (v) {
                    i64* t = reinterpret_cast<i64*>(l2) + (size_t)col * 16 + grp;
                    *t = (i64)((u64)*t + (u64)(i64)v);
                }
            }
        }
    }
}

// table[cell] += sum over the CTAs' byte tables of (byte - 2^7).  A block of
// 256 threads = 16 columns of 16 bytes x 16 groups of CTAs (up to 10 loads of
// a thread in flight at once: the 148 x 128 KiB tables are read from L2 once);
// the groups' partial sums meet in shared memory and 16 threads per column
// update its 16 cells.
constexpr int kFoldThreads = 256;
constexpr int kFoldCols = 16;
constexpr int kFoldGroups = kFoldThreads / kFoldCols;
constexpr int kFoldMaxPer = 10;  // CTAs per group handled in one unrolled batch
__global__ void __launch_bounds__(kFoldThreads)
    private_fold_kernel(const uint4* __restrict__ scratch, u32 cols, u32 ctas, i64* __restrict__ table,
                        const u32* __restrict__ go) {
    if (go && *go) return;
    __shared__ i32 part[kFoldGroups][kFoldCols][17];
    const u32 ci = threadIdx.x % kFoldCols, grp = threadIdx.x / kFoldCols;
    const u32 col = blockIdx.x * kFoldCols + ci;
    i32 s[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j] = 0;
    if (col < cols) {
        for (u32 c0 = grp; c0 < ctas; c0 += kFoldGroups * kFoldMaxPer) {
            uint4 v[kFoldMaxPer];
#pragma unroll
            for (int u = 0; u < kFoldMaxPer; ++u) {
                const u32 cta = c0 + u * kFoldGroups;
                v[u] = cta < ctas ? __ldcg(scratch + (size_t)cta * cols + col) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kFoldMaxPer; ++u) {
                const u32 wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int b = 0; b < 4; ++b) s[4 * w + b] += (i32)((wv[w] >> (8 * b)) & 0xffu);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) part[grp][ci][j] = s[j];
    __syncthreads();
    // thread (ci, j = grp) finishes cell j of column ci
    if (col < cols) {
        i32 v = -0x80 * (i32)ctas;
#pragma unroll
        for (int g = 0; g < kFoldGroups; ++g) v += part[g][ci][grp];
        if (v) {
            i64* t = table + (size_t)col * 16 + grp;
            *t = (i64)((u64)*t + (u64)(i64)v);
        }
    }
}

}  // namespace
}  // namespace mb200
