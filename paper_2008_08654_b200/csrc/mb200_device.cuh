// mb200_device.cuh -- register-level integer arithmetic for sm_100a.
//
// Every multi-word product is built from 32x32->64 limb products
// (mul.wide.u32 -> IMAD.WIDE.U32) and every reduction is a branch-free
// shift/mask/add fold.  No u128 emulation from the compiler, no division.
//
// Reference semantics being reproduced (file:line under /root/reference/proj):
//   Alg 1 Horner mod 2^61-1   polyhash.cpp:64-76
//   Alg 1 Horner mod 2^89-1   polyhash.cpp:78-88, field.hpp:66-73
//   Alg 2 two-for-one split   sketch.cpp:13-19
//   Alg 4/5 pseudo-Mersenne   field.cpp:246-273
#pragma once
#include <cstdint>

namespace mb200 {

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;
typedef int32_t i32;

constexpr u64 kP61 = (1ull << 61) - 1;
constexpr u32 kP89Top = (1u << 25) - 1;  // limb 2 of 2^89-1 (bits 64..88)

__device__ __forceinline__ u64 mulw(u32 a, u32 b) { return (u64)a * (u64)b; }
__device__ __forceinline__ u32 lo32(u64 v) { return (u32)v; }
__device__ __forceinline__ u32 hi32(u64 v) { return (u32)(v >> 32); }

// ---------------------------------------------------------------------------
// p = 2^61 - 1, 32-bit keys (the reference's classic setup, bench.cpp:54-58).
// One Horner step y <- y x + a, lazily reduced:
//   in  y < 2^63, x < 2^32, a < p
//   out (yx & p) + (yx >> 61) + a  <  2^61 + 2^34 + 2^61  <  2^63   (closed)
// Two limb products A = y0 x, B = y1 x; y x = A + B 2^32, and (y x) >> 32 =
// B + A1 < 2^63 + 2^32 is ONE mad.wide (no carry chain).  The fold takes the
// shift (t1, t2) >> 29 and the mask of t1, the three-term sum is one 3-input
// add pair (IADD3, IADD3.X).  Per step: 3 IMAD.WIDE + 1 IMAD.HI on the FMA
// pipe, 4 ops on the ALU pipe (was 3 + 6: the carry chain and the t2 >> 29
// shift ran on the ALU pipe, the binding one of the hash kernels).
// The two multipliers 1 (B + A1 as mad.wide A1 * 1 + y1 x) and 8
// (t2 >> 29 = hi32(8 t2)) are runtime values from constant memory, so ptxas
// cannot strength-reduce them back into ALU adds and shifts.
static __constant__ u32 kFmaOne = 1;
static __constant__ u32 kFmaEight = 8;

__device__ __forceinline__ u64 h61_step32(u64 y, u32 x, u64 a) {
    u64 lo, hi;
    asm("{\n\t"
        ".reg .u32 y0, y1, A0, A1, t1, t2, h0, h1;\n\t"
        ".reg .u64 A, B;\n\t"
        "mov.b64 {y0, y1}, %2;\n\t"
        "mul.wide.u32 A, y0, %3;\n\t"
        "mov.b64 {A0, A1}, A;\n\t"
        "mul.wide.u32 B, A1, %4;\n\t"      // A1 (times the runtime 1)
        "mad.wide.u32 B, y1, %3, B;\n\t"   // (y x) >> 32 = (t1, t2) < 2^63 + 2^32
        "mov.b64 {t1, t2}, B;\n\t"
        "shf.r.clamp.b32 h0, t1, t2, 29;\n\t"  // (y x) >> 61
        "mul.hi.u32 h1, t2, %5;\n\t"           // t2 >> 29 = hi32(8 t2)
        "and.b32 t1, t1, 0x1FFFFFFF;\n\t"      // (y x) & p, high word
        "mov.b64 %0, {A0, t1};\n\t"
        "mov.b64 %1, {h0, h1};\n\t"
        "}"
        : "=l"(lo), "=l"(hi)
        : "l"(y), "r"(x), "r"(kFmaOne), "r"(kFmaEight));
    return lo + hi + a;
}

// The first step of a chain, y = a_{k-1} < 2^61: y1 x + A1 <= (2^29 - 1)(2^32 - 1)
// + 2^32 - 1 < 2^61, so t2 < 2^29 and (y x) >> 61 fits one word (no IMAD.HI).
__device__ __forceinline__ u64 h61_step32_first(u64 y, u32 x, u64 a) {
    u64 lo, hi;
    asm("{\n\t"
        ".reg .u32 y0, y1, A0, A1, t1, t2, h0;\n\t"
        ".reg .u64 A, B;\n\t"
        "mov.b64 {y0, y1}, %2;\n\t"
        "mul.wide.u32 A, y0, %3;\n\t"
        "mov.b64 {A0, A1}, A;\n\t"
        "mul.wide.u32 B, A1, %4;\n\t"
        "mad.wide.u32 B, y1, %3, B;\n\t"
        "mov.b64 {t1, t2}, B;\n\t"
        "shf.r.clamp.b32 h0, t1, t2, 29;\n\t"
        "and.b32 t1, t1, 0x1FFFFFFF;\n\t"
        "mov.b64 %0, {A0, t1};\n\t"
        "mov.b64 %1, {h0, 0};\n\t"
        "}"
        : "=l"(lo), "=l"(hi)
        : "l"(y), "r"(x), "r"(kFmaOne));
    return lo + hi + a;
}

// Full reduction of a lazily reduced value y < 2^64 to [0, p): one fold to
// < 2^61 + 8 < 2p, then the reference's branch-free finish
// z = (y + 1) >> b; (y + z) & p   (polyhash.cpp:74-75).
__device__ __forceinline__ u64 h61_fold(u64 y) { return (y & kP61) + (y >> 61); }
__device__ __forceinline__ u64 h61_finish(u64 y) {
    y = h61_fold(y);
    const u64 z = (y + 1) >> 61;
    return (y + z) & kP61;
}

// Alg 2 with b = 61 and a power-of-two width straight from a lazily reduced
// y < 2^64 (sketch.cpp:13-19 on h = y mod p): after one fold y < 2^61 + 8, and
// z = (y + 1) >> 61 is 1 exactly when y >= p, in which case h = y - p < 8 (its
// low word is lo32(y) + 1, its bit 60 is 0).  Returns the bucket (mask < 2^32)
// and sets neg = bit 60 of h.  Two ALU ops fewer than h61_finish + split.
__device__ __forceinline__ u32 h61_pow2_split(u64 y, u32 mask, bool& neg) {
    y = h61_fold(y);
    const u32 z = (u32)((y + 1) >> 61);
    neg = ((hi32(y) >> 28) & ~z) & 1u;
    return (lo32(y) + z) & mask;
}

// ---------------------------------------------------------------------------
// p = 2^61 - 1, any 64-bit key (config 2 draws keys from [0, p), beyond the
// reference's u <= 2^60 domain; SURVEY 7.3 hard part 2).  Keys are folded once
// to x <= 2^61 + 6 (x1 = x >> 32 <= 2^29).  One step, bound B on the input y:
//   t = y x = P00 + M 2^32 + P11 2^64 with M = y0 x1 + y1 x0 < 2^61 + B (one
//   64-bit mad.wide chain, valid while B < 7 * 2^61), P11 = y1 x1 <= 2^61;
//   out s = (t & p) + (t >> 61) + a < B + 2^62 + 43.
// So from y < 2^61 + 8 up to THREE steps run without the second fold (bound
// after j steps: (2j + 1) 2^61 + 43 j < 7 * 2^61); h61_eval64 folds y before
// every fourth.  Four limb products per step.
__device__ __forceinline__ u64 h61_key64(u64 x) { return (x & kP61) + (x >> 61); }
constexpr int kLazySteps = 3;

__device__ __forceinline__ u64 h61_step64(u64 y, u64 x, u64 a) {
    u64 lo, hi;
    asm("{\n\t"
        ".reg .u32 y0, y1, x0, x1, t0, t1, t2, t3, m0, m1, p0, p1, h0, h1;\n\t"
        ".reg .u64 P00, M, P11;\n\t"
        "mov.b64 {y0, y1}, %2;\n\t"
        "mov.b64 {x0, x1}, %3;\n\t"
        "mul.wide.u32 P00, y0, x0;\n\t"
        "mul.wide.u32 M, y0, x1;\n\t"
        "mad.wide.u32 M, y1, x0, M;\n\t"
        "mul.wide.u32 P11, y1, x1;\n\t"
        "mov.b64 {t0, p0}, P00;\n\t"
        "mov.b64 {m0, m1}, M;\n\t"
        "mov.b64 {p1, t3}, P11;\n\t"
        "add.cc.u32 t1, p0, m0;\n\t"       // t = (t0, t1, t2, t3)
        "addc.cc.u32 t2, p1, m1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        "shf.r.clamp.b32 h0, t1, t2, 29;\n\t"  // t >> 61
        "shf.r.clamp.b32 h1, t2, t3, 29;\n\t"
        "and.b32 t1, t1, 0x1FFFFFFF;\n\t"      // t & p
        "mov.b64 %0, {t0, t1};\n\t"
        "mov.b64 %1, {h0, h1};\n\t"
        "}"
        : "=l"(lo), "=l"(hi)
        : "l"(y), "l"(x));
    return lo + hi + a;
}

// Horner over K (compile-time) coefficients, lowest first in c[]: leading
// coefficient c[K-1] (polyhash.cpp:67-69), key already folded by h61_key64.
template <int K>
__device__ __forceinline__ u64 h61_eval64(const u64* c, u64 x) {
    u64 y = c[K - 1];
#pragma unroll
    for (int i = K - 2; i >= 0; --i) {
        if ((K - 2 - i) > 0 && (K - 2 - i) % kLazySteps == 0) y = h61_fold(y);
        y = h61_step64(y, x, c[i]);
    }
    return y;
}
// runtime k
__device__ __forceinline__ u64 h61_eval64_rt(const u64* c, int k, u64 x) {
    u64 y = c[k - 1];
    int lazy = 0;
#pragma unroll 1
    for (int i = k - 2; i >= 0; --i) {
        if (lazy == kLazySteps) {
            y = h61_fold(y);
            lazy = 0;
        }
        y = h61_step64(y, x, c[i]);
        ++lazy;
    }
    return y;
}

// ---------------------------------------------------------------------------
// Generic Mersenne p = 2^b - 1 with b <= 61 and runtime b, valid on the
// reference's domain x < u <= 2^(b-1) (polyhash.cpp:48-57): exactly the
// reference's native Horner (u128 t = y x + a; y = (t & p) + (t >> b);
// invariant y < 2p), the u128 built from two 64-bit halves.
__device__ __forceinline__ u64 hgen_step(u64 y, u64 x, u64 a, u32 b, u64 p) {
    const u64 lo = y * x;
    u64 hi = __umul64hi(y, x);
    const u64 tl = lo + a;
    hi += (tl < lo);
    return (tl & p) + ((hi << (64 - b)) | (tl >> b));
}
__device__ __forceinline__ u64 hgen_finish(u64 y, u32 b, u64 p) {
    const u64 z = (y + 1) >> b;  // y < 2p: the carry is the top bit
    return (y + z) & p;
}

// ---------------------------------------------------------------------------
// p = 2^89 - 1 on 32-bit limbs (y0,y1,y2), y < 2p (y2 < 2^26), x < 2^64,
// a < p.  t = y x + a < 2^154 + 2^89 in five limbs via a PTX carry chain
// (six limb products, each a mad.lo/mad.hi pair), then the reference's single
// partial fold (t & p) + (t >> 89) < 2^89 + 2^65 < 2p (field.hpp:66-73).
__device__ __forceinline__ void h89_step(u32& y0, u32& y1, u32& y2, u32 x0, u32 x1, u32 a0,
                                         u32 a1, u32 a2) {
    u32 t0, t1, t2, t3, t4;
    asm("mad.lo.cc.u32  %0, %5, %8, %10;\n\t"
        "madc.lo.cc.u32 %1, %6, %8, %11;\n\t"
        "madc.lo.cc.u32 %2, %7, %8, %12;\n\t"
        "addc.u32       %3, 0, 0;\n\t"
        "mad.hi.cc.u32  %1, %5, %8, %1;\n\t"
        "madc.hi.cc.u32 %2, %6, %8, %2;\n\t"
        "madc.hi.u32    %3, %7, %8, %3;\n\t"
        "mad.lo.cc.u32  %1, %5, %9, %1;\n\t"
        "madc.lo.cc.u32 %2, %6, %9, %2;\n\t"
        "madc.lo.cc.u32 %3, %7, %9, %3;\n\t"
        "addc.u32       %4, 0, 0;\n\t"
        "mad.hi.cc.u32  %2, %5, %9, %2;\n\t"
        "madc.hi.cc.u32 %3, %6, %9, %3;\n\t"
        "madc.hi.u32    %4, %7, %9, %4;"
        : "=&r"(t0), "=&r"(t1), "=&r"(t2), "=&r"(t3), "=&r"(t4)
        : "r"(y0), "r"(y1), "r"(y2), "r"(x0), "r"(x1), "r"(a0), "r"(a1), "r"(a2));
    const u32 l2 = t2 & kP89Top;
    const u32 h0 = __funnelshift_r(t2, t3, 25);
    const u32 h1 = __funnelshift_r(t3, t4, 25);
    const u32 h2 = t4 >> 25;
    asm("add.cc.u32  %0, %3, %6;\n\t"
        "addc.cc.u32 %1, %4, %7;\n\t"
        "addc.u32    %2, %5, %8;"
        : "=r"(y0), "=r"(y1), "=r"(y2)
        : "r"(t0), "r"(t1), "r"(l2), "r"(h0), "r"(h1), "r"(h2));
}

// Branch-free finish for y < 2p: z = (y + 1) >> 89; (y + z) & p.
__device__ __forceinline__ void h89_finish(u32& y0, u32& y1, u32& y2) {
    u32 s2;
    asm("{\n\t.reg .u32 t0, t1;\n\t"
        "add.cc.u32  t0, %1, 1;\n\t"
        "addc.cc.u32 t1, %2, 0;\n\t"
        "addc.u32    %0, %3, 0;\n\t}"
        : "=r"(s2)
        : "r"(y0), "r"(y1), "r"(y2));
    const u32 z = s2 >> 25;
    asm("add.cc.u32  %0, %0, %3;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.u32    %2, %2, 0;"
        : "+r"(y0), "+r"(y1), "+r"(y2)
        : "r"(z));
    y2 &= kP89Top;
}

// ---------------------------------------------------------------------------
// Generic Mersenne p = 2^b - 1 for 62 <= b <= 127 (polyhash.cpp:78-88 on
// UWide, field.hpp:66-73): y < 2p in four 32-bit limbs, x < 2^64 (two limbs),
// a < p.  On the key domain x < 2^(b-1) the reference's invariant y < 2p
// holds after every partial fold.  t = y x + a < 2^192 as six words, each row
// term a product of two words plus at most two words (<= 2^64 - 1); then
// (t & p) + (t >> b) with b = 32 Q + R: Q = b / 32 is a template parameter (the
// word indices are static), R runtime.  t >> b < 2^65 fits three words.
// Performance is not the point here (no BASELINE config uses these moduli;
// b = 89's config runs h89_step / the config-4 kernel): exactness is.
template <int Q>
__device__ __forceinline__ void hw_step(u32 (&y)[4], u32 x0, u32 x1, const u32 (&a)[4], u32 R) {
    u32 w[7];
    u64 r = (u64)y[0] * x0 + a[0];
    w[0] = (u32)r;
    u32 c0, c1, c2, c3;  // row x0, words 1..4
    r = (u64)y[1] * x0 + (r >> 32) + a[1];
    c0 = (u32)r;
    r = (u64)y[2] * x0 + (r >> 32) + a[2];
    c1 = (u32)r;
    r = (u64)y[3] * x0 + (r >> 32) + a[3];
    c2 = (u32)r;
    c3 = (u32)(r >> 32);
    u64 q = (u64)y[0] * x1 + c0;
    w[1] = (u32)q;
    q = (u64)y[1] * x1 + (q >> 32) + c1;
    w[2] = (u32)q;
    q = (u64)y[2] * x1 + (q >> 32) + c2;
    w[3] = (u32)q;
    q = (u64)y[3] * x1 + (q >> 32) + c3;
    w[4] = (u32)q;
    w[5] = (u32)(q >> 32);
    w[6] = 0;
    const u32 mask = R ? (0xffffffffu >> (32 - R)) : 0u;
    u32 L[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) L[j] = j < Q ? w[j] : (j == Q ? w[j] & mask : 0u);
    u32 H[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) H[j] = __funnelshift_r(w[Q + j], w[Q + j + 1], R);
    u64 acc = (u64)L[0] + H[0];
    y[0] = (u32)acc;
    acc = (u64)L[1] + H[1] + (acc >> 32);
    y[1] = (u32)acc;
    acc = (u64)L[2] + H[2] + (acc >> 32);
    y[2] = (u32)acc;
    y[3] = L[3] + (u32)(acc >> 32);
}

// The reference's branch-free finish for y < 2p: z = (y + 1) >> b; (y + z) & p
template <int Q>
__device__ __forceinline__ void hw_finish(u32 (&y)[4], u32 R) {
    u64 acc = (u64)y[0] + 1;
    u32 t[4];
    t[0] = (u32)acc;
#pragma unroll
    for (int j = 1; j < 4; ++j) {
        acc = (u64)y[j] + (acc >> 32);
        t[j] = (u32)acc;
    }
    const u32 z = (t[Q] >> R) & 1u;  // y + 1 < 2^(b+1): bit b is the whole quotient
    acc = (u64)y[0] + z;
    y[0] = (u32)acc;
#pragma unroll
    for (int j = 1; j < 4; ++j) {
        acc = (u64)y[j] + (acc >> 32);
        y[j] = (u32)acc;
    }
    const u32 mask = R ? (0xffffffffu >> (32 - R)) : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = j < Q ? y[j] : (j == Q ? y[j] & mask : 0u);
}

template <int Q>
__device__ __forceinline__ void hash_wide_q(const u64* clo, const u64* chi, int k, u32 R, u64 x, u64& lo, u64& hi) {
    u32 y[4] = {lo32(clo[k - 1]), hi32(clo[k - 1]), lo32(chi[k - 1]), hi32(chi[k - 1])};
    const u32 x0 = lo32(x), x1 = hi32(x);
#pragma unroll 1
    for (int i = k - 2; i >= 0; --i) {
        const u32 a[4] = {lo32(clo[i]), hi32(clo[i]), lo32(chi[i]), hi32(chi[i])};
        hw_step<Q>(y, x0, x1, a, R);
    }
    hw_finish<Q>(y, R);
    lo = ((u64)y[1] << 32) | y[0];
    hi = ((u64)y[3] << 32) | y[2];
}

// h = (sum_i a_i x^i) mod (2^b - 1) as (low 64 bits, high bits), 62 <= b <= 127;
// coefficients lowest first as (lo, hi) 64-bit halves
__device__ __forceinline__ void hash_wide(const u64* clo, const u64* chi, int k, u32 b, u64 x, u64& lo, u64& hi) {
    const u32 R = b & 31u;
    switch (b >> 5) {
        case 1: hash_wide_q<1>(clo, chi, k, R, x, lo, hi); break;
        case 2: hash_wide_q<2>(clo, chi, k, R, x, lo, hi); break;
        default: hash_wide_q<3>(clo, chi, k, R, x, lo, hi); break;
    }
}

// ---------------------------------------------------------------------------
// SplitMix64 (prng.hpp:10-38) in counter form: the i-th next() of
// SplitMix64(seed) is mix(seed + (i+1) * golden).
constexpr u64 kGolden = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 splitmix_at(u64 seed, u64 i) {
    return mix64(seed + (i + 1) * kGolden);
}

}  // namespace mb200
