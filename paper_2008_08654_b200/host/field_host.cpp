// field_host.cpp -- construction-time host logic of the C-ABI: the
// pseudo-Mersenne iteration count and exact division domain of
// PseudoMersenneModulus (reference field.cpp:156-193 and ctor :224-244), the
// ExactDivisionMap iteration search (bucketing.cpp:75-89), the seeded
// coefficient draw (polyhash.cpp:12-35) and CountSketch row seeds
// (sketch.cpp:72-77).  Runs once per object, never per key; every per-key
// computation is on the GPU.
//
// The domain threshold is stated here in closed form and evaluated without a
// general long division.  For p = q - c (q = 2^b) and n iterations the
// reference admits every dividend up to
//     T(n) = floor(N / C),  N = q^n - d,  C = c^(n-1),
// with d = c^n when c is a power of two (then T = 2^(bn - s(n-1)) - c exactly
// for c = 2^s) and d = c q^(n-1) otherwise, and clamps T below
// 2^255 - 2^127 so every iteration intermediate fits 256 bits.  Because the
// clamp caps the answer at 255 bits, T is found by deciding its bits from the
// top: start from the clamp test (clamp * C <= N ?), then for bit 254 .. 0 keep
// the bit when (T + 2^bit) * C <= N.  Each test is one 4-limb x |C| product
// and a comparison, so the whole search is ~255 short products on
// arbitrarily long N and C (n up to ~2b iterations, i.e. ~32k-bit numbers).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/mersenne_b200.h"
#include "../csrc/mb200_capi_util.h"

namespace {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

constexpr u64 kGolden = 0x9E3779B97F4A7C15ull;
// SplitMix64::next (prng.hpp:14-19)
u64 splitmix_next(u64& state) {
    u64 z = (state += kGolden);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Natural number as little-endian 64-bit limbs; normalised (no high zero limbs).
using Nat = std::vector<u64>;

void normalise(Nat& a) {
    while (!a.empty() && a.back() == 0) a.pop_back();
}

Nat nat_of(u128 v) {
    Nat a{u64(v), u64(v >> 64)};
    normalise(a);
    return a;
}

// 2^e
Nat nat_pow2(size_t e) {
    Nat a(e / 64 + 1, 0);
    a.back() = u64(1) << (e % 64);
    return a;
}

size_t nat_bits(const Nat& a) { return a.empty() ? 0 : 64 * a.size() - size_t(__builtin_clzll(a.back())); }

// three-way compare
int nat_cmp(const Nat& a, const Nat& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

// schoolbook product
Nat nat_mul(const Nat& a, const Nat& b) {
    if (a.empty() || b.empty()) return {};
    Nat r(a.size() + b.size(), 0);
    for (size_t i = 0; i < a.size(); ++i) {
        u64 carry = 0;
        for (size_t j = 0; j < b.size(); ++j) {
            const u128 t = u128(a[i]) * b[j] + r[i + j] + carry;
            r[i + j] = u64(t);
            carry = u64(t >> 64);
        }
        r[i + b.size()] = carry;
    }
    normalise(r);
    return r;
}

// a - b for a >= b
Nat nat_sub(Nat a, const Nat& b) {
    unsigned borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const u128 sub = u128(i < b.size() ? b[i] : 0) + borrow;
        borrow = u128(a[i]) < sub;
        a[i] = u64(u128(a[i]) - sub);
    }
    normalise(a);
    return a;
}

// a * 2^e
Nat nat_shl(const Nat& a, size_t e) {
    if (a.empty()) return {};
    Nat r(a.size() + e / 64 + 1, 0);
    const unsigned s = unsigned(e % 64);
    for (size_t i = 0; i < a.size(); ++i) {
        r[i + e / 64] |= a[i] << s;
        if (s) r[i + e / 64 + 1] |= a[i] >> (64 - s);
    }
    normalise(r);
    return r;
}

Nat nat_pow(u128 base, unsigned e) {
    Nat r = nat_of(1), x = nat_of(base);
    for (; e; e >>= 1) {  // square and multiply
        if (e & 1) r = nat_mul(r, x);
        if (e > 1) x = nat_mul(x, x);
    }
    return r;
}

bool is_pow2(u128 c) { return (c & (c - 1)) == 0; }

// Iteration count (field.cpp:156-171).  The comment there states the bound as
// c^m <= 2^(b(m-2)); the reference's test is bit_length(c^m) <= b(m-2), i.e. the
// STRICT c^m < 2^(b(m-2)), which differs exactly when c is a power of two and
// c^m lands on the bound (b = 5, c = 8: m = 6, not 5).  Restated as executed:
// c = 1 gives 2, otherwise the smallest m >= 3 with bits(c^m) <= b(m-2).
unsigned default_iterations(unsigned b, u128 c) {
    if (c == 1) return 2;
    Nat cm = nat_pow(c, 3);
    for (unsigned m = 3;; ++m, cm = nat_mul(cm, nat_of(c)))
        if (nat_bits(cm) <= size_t(b) * (m - 2)) return m;
}

// T(n) of the header comment, clamped to 2^255 - 2^127; out = 4 little-endian limbs.
void domain_threshold(unsigned b, u128 c, unsigned n, u64 out[4]) {
    const Nat d = is_pow2(c) ? nat_pow(c, n) : nat_shl(nat_of(c), size_t(b) * (n - 1));
    const Nat N = nat_sub(nat_pow2(size_t(b) * n), d);
    const Nat C = nat_pow(c, n - 1);
    const Nat clamp = nat_sub(nat_pow2(255), nat_pow2(127));
    Nat t;
    if (nat_cmp(nat_mul(clamp, C), N) <= 0) {
        t = clamp;
    } else {
        Nat cand(4, 0);  // T < clamp < 2^255: decide bits 254..0
        for (int bit = 254; bit >= 0; --bit) {
            cand[size_t(bit) / 64] |= u64(1) << (bit % 64);
            Nat trial = cand;
            normalise(trial);
            if (nat_cmp(nat_mul(trial, C), N) > 0) cand[size_t(bit) / 64] &= ~(u64(1) << (bit % 64));
        }
        t = cand;
        normalise(t);
    }
    for (size_t i = 0; i < 4; ++i) out[i] = i < t.size() ? t[i] : 0;
}

}  // namespace

extern "C" {

int mb200_pm_modulus(unsigned b, uint64_t c_lo, uint64_t c_hi, unsigned m_iters, unsigned* iterations,
                     uint64_t max_input[4]) {
    using mb200::fail;
    const u128 c = (u128(c_hi) << 64) | c_lo;
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 127]");  // field.cpp:225
    if (c == 0 || c >= (u128(1) << (b - 1)))
        return fail(MB200_INVALID_ARGUMENT, "offset must satisfy 1 <= c < 2^(b-1)");  // field.cpp:226-228
    const unsigned m = m_iters ? m_iters : default_iterations(b, c);
    if (iterations) *iterations = m;
    u64 tmp[4];
    domain_threshold(b, c, m, max_input ? max_input : tmp);
    return MB200_OK;
}

int mb200_exact_division_iterations(unsigned b, uint64_t c, uint64_t r, unsigned* iterations) {
    using mb200::fail;
    if (int rc = mb200_pm_modulus(b, c, 0, 0, nullptr, nullptr)) return rc;  // PseudoMersenneModulus(b, c)
    const u128 p = (u128(1) << b) - c;
    if (r == 0 || u128(r) > p) return fail(MB200_INVALID_ARGUMENT, "bucket count must be in [1, p]");
    // bucketing.cpp:80-88: the first m whose domain admits the largest product (p-1) r
    const Nat largest = nat_mul(nat_of(p - 1), nat_of(r));
    for (unsigned m = 1;; ++m) {
        u64 thr[4];
        domain_threshold(b, c, m, thr);
        Nat t(thr, thr + 4);
        normalise(t);
        if (nat_cmp(largest, t) <= 0) {
            if (iterations) *iterations = m;
            return MB200_OK;
        }
    }
}

int mb200_draw_coeffs(unsigned b, unsigned k, uint64_t seed, uint64_t* lo, uint64_t* hi) {
    using mb200::fail;
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "exponent must be in [2, 127]");
    if (k == 0) return fail(MB200_INVALID_ARGUMENT, "independence degree must be at least 1");
    if (!lo || (b > 64 && !hi)) return fail(MB200_INVALID_ARGUMENT, "null output");
    const u128 p = (u128(1) << b) - 1;
    u64 state = seed;
    for (unsigned i = 0; i < k; ++i) {
        u128 v;
        do {  // draw_residue: mask to b bits, reject the single value p
            if (b <= 64) {
                v = splitmix_next(state) & u64(p);
            } else {
                // polyhash.cpp:19 `(u128(g.next()) << 64) | g.next()` as compiled by the
                // reference toolchain (g++ 13.3): the first draw is the high limb.
                const u64 h = splitmix_next(state);
                v = ((u128(h) << 64) | splitmix_next(state)) & p;
            }
        } while (v == p);
        lo[i] = u64(v);
        if (hi) hi[i] = u64(v >> 64);
    }
    return MB200_OK;
}

int mb200_row_seeds(uint64_t master, unsigned rows, uint64_t* out) {
    u64 state = master;
    for (unsigned r = 0; r < rows; ++r) out[r] = splitmix_next(state);
    return MB200_OK;
}

}  // extern "C"
