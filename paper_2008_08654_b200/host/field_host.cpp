// field_host.cpp -- construction-time host logic of the C-ABI: the
// pseudo-Mersenne iteration count and exact division domain (reference
// field.cpp:158-193 and PseudoMersenneModulus ctor :224-244, restated on a
// small vector bignum), the seeded coefficient draw (polyhash.cpp:12-35) and
// CountSketch row seeds (sketch.cpp:72-77).  Runs once per object, never per
// key; every per-key computation is on the GPU.
#include <cstdint>
#include <string>
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

struct Big {
    std::vector<u64> w;  // little endian, trimmed
    void trim() {
        while (!w.empty() && w.back() == 0) w.pop_back();
    }
    static Big of(u64 v) {
        Big b;
        if (v) b.w = {v};
        return b;
    }
    static Big pow2(size_t bits) {
        Big b;
        b.w.assign(bits / 64 + 1, 0);
        b.w[bits / 64] = u64(1) << (bits % 64);
        return b;
    }
    size_t bitlen() const { return w.empty() ? 0 : 64 * (w.size() - 1) + (64 - __builtin_clzll(w.back())); }
    void mul(u64 m) {
        u64 carry = 0;
        for (auto& x : w) {
            u128 t = u128(x) * m + carry;
            x = u64(t);
            carry = u64(t >> 64);
        }
        if (carry) w.push_back(carry);
        trim();
    }
    void shl(size_t bits) {
        if (w.empty() || !bits) return;
        const size_t words = bits / 64, rem = bits % 64;
        std::vector<u64> out(w.size() + words + 1, 0);
        for (size_t i = 0; i < w.size(); ++i) {
            out[i + words] |= rem ? (w[i] << rem) : w[i];
            if (rem) out[i + words + 1] |= w[i] >> (64 - rem);
        }
        w.swap(out);
        trim();
    }
    void shr1() {
        for (size_t i = 0; i < w.size(); ++i) {
            w[i] >>= 1;
            if (i + 1 < w.size()) w[i] |= w[i + 1] << 63;
        }
        trim();
    }
};

int cmp(const Big& a, const Big& b) {
    if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
    for (size_t i = a.w.size(); i-- > 0;)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

void sub(Big& a, const Big& b) {
    u64 borrow = 0;
    for (size_t i = 0; i < a.w.size(); ++i) {
        const u64 bi = i < b.w.size() ? b.w[i] : 0;
        const u64 d = a.w[i] - bi;
        const u64 bo = (a.w[i] < bi) | (d < borrow);
        a.w[i] = d - borrow;
        borrow = bo;
    }
    a.trim();
}

Big divide(Big t, const Big& d) {
    Big q;
    if (d.w.empty() || cmp(t, d) < 0) return q;
    const long shift = long(t.bitlen()) - long(d.bitlen());
    Big cur = d;
    cur.shl(size_t(shift));
    q.w.assign(size_t(shift) / 64 + 1, 0);
    for (long s = shift; s >= 0; --s) {
        if (cmp(cur, t) <= 0) {
            sub(t, cur);
            q.w[size_t(s) / 64] |= u64(1) << (size_t(s) % 64);
        }
        cur.shr1();
    }
    q.trim();
    return q;
}

// field.cpp:158-171: smallest m with c^m <= 2^(b(m-2))
unsigned default_iterations(unsigned b, u64 c) {
    if (c == 1) return 2;
    Big cm = Big::of(c);
    cm.mul(c);
    unsigned m = 2;
    for (;;) {
        ++m;
        cm.mul(c);
        if (cm.bitlen() <= size_t(b) * (m - 2) && cmp(cm, Big::pow2(size_t(b) * (m - 2))) <= 0) return m;
    }
}

// field.cpp:176-193
void domain_threshold(unsigned b, u64 c, unsigned n, u64 out[4]) {
    Big qn = Big::pow2(size_t(b) * n);
    Big d;
    if ((c & (c - 1)) == 0) {
        d = Big::of(1);
        for (unsigned i = 0; i < n; ++i) d.mul(c);
    } else {
        d = Big::of(c);
        d.shl(size_t(b) * (n - 1));
    }
    sub(qn, d);
    Big cn1 = Big::of(1);
    for (unsigned i = 0; i + 1 < n; ++i) cn1.mul(c);
    Big v = divide(std::move(qn), cn1);
    Big clamp = Big::pow2(255);
    sub(clamp, Big::pow2(127));
    const Big& r = cmp(v, clamp) < 0 ? v : clamp;
    for (int i = 0; i < 4; ++i) out[i] = size_t(i) < r.w.size() ? r.w[size_t(i)] : 0;
}

}  // namespace

extern "C" {

int mb200_pm_modulus(unsigned b, uint64_t c, unsigned m_iters, unsigned* iterations, uint64_t max_input[4]) {
    using mb200::fail;
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 127]");
    if (c == 0 || (b - 1 < 64 && c >= (u64(1) << (b - 1))))
        return fail(MB200_INVALID_ARGUMENT, "offset must satisfy 1 <= c < 2^(b-1)");
    const unsigned m = m_iters ? m_iters : default_iterations(b, c);
    if (iterations) *iterations = m;
    u64 tmp[4];
    domain_threshold(b, c, m, max_input ? max_input : tmp);
    return MB200_OK;
}

int mb200_exact_division_iterations(unsigned b, uint64_t c, uint64_t r, unsigned* iterations) {
    using mb200::fail;
    if (int rc = mb200_pm_modulus(b, c, 0, nullptr, nullptr)) return rc;  // PseudoMersenneModulus(b, c)
    const u128 p = (u128(1) << b) - c;
    if (r == 0 || u128(r) > p) return fail(MB200_INVALID_ARGUMENT, "bucket count must be in [1, p]");
    // bucketing.cpp:80-88: grow m until the largest product (p-1) r is admissible
    Big largest;
    largest.w = {u64(p - 1), u64((p - 1) >> 64)};
    largest.trim();
    largest.mul(r);
    for (unsigned m = 1;; ++m) {
        u64 thr[4];
        domain_threshold(b, c, m, thr);
        Big t;
        t.w.assign(thr, thr + 4);
        t.trim();
        if (cmp(largest, t) <= 0) {
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
    auto next = [&state] { return splitmix_next(state); };
    for (unsigned i = 0; i < k; ++i) {
        u128 v;
        for (;;) {
            if (b <= 64) {
                v = next() & u64(p);
            } else {
                // polyhash.cpp:19 `(u128(g.next()) << 64) | g.next()` as compiled by the
                // reference toolchain (g++ 13.3): the first draw is the high limb.
                const u64 h = next();
                const u64 l = next();
                v = ((u128(h) << 64) | l) & p;
            }
            if (v != p) break;
        }
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
