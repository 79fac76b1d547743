/*
 * oracle.c -- CPU restatement of the reference's hashing and sketching path
 * (arXiv 2008.08654 reference, /root/reference/proj).  TEST INFRASTRUCTURE:
 * see oracle.h for who may use it.  Parity pinned against the reference's
 * frozen unit-test values and against golden vectors produced by the compiled
 * reference itself (tests/golden/, tests/test_oracle.py).
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef int64_t i64;

#define GOLDEN 0x9E3779B97F4A7C15ULL

/* ======================= prng.hpp:10-38 ================================= */
static inline u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

u64 orc_splitmix_next(u64* state) { return mix64(*state += GOLDEN); }

u64 orc_splitmix_at(u64 seed, u64 i) { return mix64(seed + (i + 1) * GOLDEN); }

u64 orc_splitmix_below(u64* state, u64 bound) {
    if (bound <= 1) return 0;
    int shift = 64;
    u64 b = bound - 1;
    while (b) {
        --shift;
        b >>= 1;
    }
    for (;;) {
        u64 v = orc_splitmix_next(state) >> shift;
        if (v < bound) return v;
    }
}

/* ======================= 256-bit helper (uwide.hpp:34-163) =============== */
typedef struct { u64 l[4]; } u256;

static inline u256 w_of(u128 v) {
    u256 r = {{(u64)v, (u64)(v >> 64), 0, 0}};
    return r;
}
static inline u128 w_low128(u256 a) { return ((u128)a.l[1] << 64) | a.l[0]; }
static inline u256 w_add(u256 a, u256 b) {
    u256 r;
    u128 c = 0;
    for (int i = 0; i < 4; ++i) {
        u128 t = (u128)a.l[i] + b.l[i] + c;
        r.l[i] = (u64)t;
        c = t >> 64;
    }
    return r;
}
static inline u256 w_sub(u256 a, u256 b) { /* a >= b */
    u256 r;
    u64 borrow = 0;
    for (int i = 0; i < 4; ++i) {
        u64 d = a.l[i] - b.l[i];
        u64 bo = (a.l[i] < b.l[i]) | (d < borrow);
        r.l[i] = d - borrow;
        borrow = bo;
    }
    return r;
}
static inline int w_cmp(u256 a, u256 b) {
    for (int i = 3; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}
static inline u256 w_shr(u256 v, unsigned s) {
    u256 r = {{0, 0, 0, 0}};
    if (s >= 256) return r;
    unsigned ls = s >> 6, bs = s & 63;
    for (unsigned i = 0; i + ls < 4; ++i) {
        u64 w = v.l[i + ls] >> bs;
        if (bs && i + ls + 1 < 4) w |= v.l[i + ls + 1] << (64 - bs);
        r.l[i] = w;
    }
    return r;
}
static inline u256 w_mask(u256 v, unsigned bits) {
    for (unsigned i = 0; i < 4; ++i) {
        if (bits >= 64 * (i + 1)) continue;
        if (bits > 64 * i) v.l[i] &= (((u64)1) << (bits - 64 * i)) - 1;
        else v.l[i] = 0;
    }
    return v;
}
/* exact product, caller guarantees it fits (uwide.hpp:148-163) */
static inline u256 w_mul(u256 a, u256 b) {
    u256 r = {{0, 0, 0, 0}};
    for (int i = 0; i < 4; ++i) {
        if (!a.l[i]) continue;
        u64 carry = 0;
        for (int j = 0; i + j < 4; ++j) {
            u128 t = (u128)a.l[i] * b.l[j] + r.l[i + j] + carry;
            r.l[i + j] = (u64)t;
            carry = (u64)(t >> 64);
        }
    }
    return r;
}
static inline int w_bitlen(u256 a) {
    for (int i = 3; i >= 0; --i)
        if (a.l[i]) return 64 * (i + 1) - __builtin_clzll(a.l[i]);
    return 0;
}

/* ======================= polyhash.cpp:12-35 ============================= */
void orc_draw_coeffs(unsigned b, unsigned k, u64 seed, u64* lo, u64* hi) {
    const u128 p = (((u128)1) << b) - 1;
    u64 state = seed;
    for (unsigned i = 0; i < k; ++i) {
        u128 v;
        for (;;) {
            if (b <= 64) {
                v = orc_splitmix_next(&state) & (u64)p;
            } else {
                /* polyhash.cpp:19 has unsequenced operands; g++ 13.3 evaluates the
                 * first next() as the HIGH limb (pinned against the compiled reference
                 * in tests/test_oracle.py::test_coeffs_match_reference). */
                u64 h = orc_splitmix_next(&state);
                u64 l = orc_splitmix_next(&state);
                v = (((u128)h << 64) | l) & p;
            }
            if (v != p) break;
        }
        lo[i] = (u64)v;
        hi[i] = (u64)(v >> 64);
    }
}

void orc_row_seeds(u64 master, unsigned rows, u64* out) {
    u64 state = master;
    for (unsigned r = 0; r < rows; ++r) out[r] = orc_splitmix_next(&state);
}

/* ======================= polyhash.cpp:59-89 (Alg 1) ===================== */
static int hash_one(unsigned b, const u64* clo, const u64* chi, unsigned k, unsigned key_bits,
                    u128 x, int finish, u128* out) {
    if (key_bits < 128 && x >= (((u128)1) << key_bits)) return 1; /* polyhash.cpp:60 */
    const u128 p = (((u128)1) << b) - 1;
    if (b <= 61) { /* native path, polyhash.cpp:64-76 */
        const u64 pp = (u64)p;
        const u64 xs = (u64)x;
        u64 y = clo[k - 1];
        for (unsigned i = k - 1; i-- > 0;) {
            u128 t = (u128)y * xs + clo[i];
            y = (u64)(t & pp) + (u64)(t >> b);
            if (!(y < 2 * pp)) return 2; /* polyhash.cpp:71 */
        }
        if (finish == 0) {
            *out = y >= pp ? y - pp : y;
        } else {
            u64 z = (y + 1) >> b;
            *out = (y + z) & pp;
        }
        return 0;
    }
    /* generic path, polyhash.cpp:78-88 (wide_mul + mersenne_reduce_partial) */
    const u256 xw = w_of(x);
    u128 y = ((u128)chi[k - 1] << 64) | clo[k - 1];
    const u256 psq = w_mul(w_of(p), w_of(p));
    const u256 bound = w_add(psq, w_of(p));
    for (unsigned i = k - 1; i-- > 0;) {
        u256 t = w_add(w_mul(w_of(y), xw), w_of(((u128)chi[i] << 64) | clo[i]));
        if (!(w_cmp(t, bound) < 0)) return 2; /* field.hpp:69 */
        u128 lo = w_low128(w_mask(t, b));
        u128 hi = w_low128(w_shr(t, b));
        y = lo + hi;
        if (!(y < 2 * p)) return 2; /* polyhash.cpp:87 */
    }
    if (finish == 0) {
        *out = y >= p ? y - p : y;
    } else {
        u128 z = (y + 1) >> b;
        *out = (y + z) & p;
    }
    return 0;
}

int orc_hash(unsigned b, const u64* clo, const u64* chi, unsigned k, unsigned key_bits, u64 x_lo,
             u64 x_hi, int finish, u64* out_lo, u64* out_hi) {
    u128 h = 0;
    int rc = hash_one(b, clo, chi, k, key_bits, ((u128)x_hi << 64) | x_lo, finish, &h);
    *out_lo = (u64)h;
    *out_hi = (u64)(h >> 64);
    return rc;
}

u64 orc_hash_batch(unsigned b, const u64* clo, const u64* chi, unsigned k, unsigned key_bits,
                   const u64* keys, u64 n, u64* out_lo, u64* out_hi) {
    u64 rejected = 0;
#pragma omp parallel for schedule(static) reduction(+ : rejected)
    for (u64 i = 0; i < n; ++i) {
        u128 h = 0;
        int rc = hash_one(b, clo, chi, k, key_bits, keys[i], 0, &h);
        if (rc) {
            ++rejected;
            h = 0;
        }
        out_lo[i] = (u64)h;
        if (out_hi) out_hi[i] = (u64)(h >> 64);
    }
    return rejected;
}

/* ======================= field.cpp:208-222 (Alg 3) ===================== */
static inline void divmod_mersenne_w(unsigned b, u256 v, u256* q, u256* r) {
    u256 one = {{1, 0, 0, 0}};
    u256 vp = w_add(v, one);
    u256 z = w_shr(w_add(w_shr(vp, b), vp), b);
    *q = z;
    *r = w_mask(w_add(v, z), b);
}

int orc_mersenne_divmod(unsigned b, u64 v_lo, u64 v_hi, u64* q_lo, u64* q_hi, u64* r_lo,
                        u64* r_hi) {
    u256 v = w_of(((u128)v_hi << 64) | v_lo);
    if (w_bitlen(v) > (int)(2 * b)) return 1; /* field.cpp:210 */
    u256 q, r;
    divmod_mersenne_w(b, v, &q, &r);
    *q_lo = q.l[0];
    *q_hi = q.l[1];
    *r_lo = r.l[0];
    *r_hi = r.l[1];
    return 0;
}

void orc_mersenne_reduce_partial(unsigned b, u64 y_lo, u64 y_hi, u64* lo, u64* hi) {
    u256 y = w_of(((u128)y_hi << 64) | y_lo);
    u128 s = w_low128(w_mask(y, b)) + w_low128(w_shr(y, b));
    *lo = (u64)s;
    *hi = (u64)(s >> 64);
}

/* SURVEY 7.4 config-2 oracle: full Alg-3 reduction per Horner step */
static inline u64 mod_full61(unsigned b, u128 v) {
    u256 q, r;
    divmod_mersenne_w(b, w_of(v), &q, &r);
    return r.l[0];
}

void orc_hash_full_batch(unsigned b, const u64* coeffs, unsigned k, const u64* keys, u64 n,
                         u64* out) {
#pragma omp parallel for schedule(static)
    for (u64 i = 0; i < n; ++i) {
        u64 x = mod_full61(b, keys[i]); /* key < 2^64 < 2^(2b) */
        u64 y = coeffs[k - 1];
        for (unsigned j = k - 1; j-- > 0;) y = mod_full61(b, (u128)y * x + coeffs[j]);
        out[i] = y;
    }
}

/* ======================= field.cpp:15-193 (construction-time bignum) ==== */
#define BIGW 640
typedef struct {
    u64 w[BIGW];
    int n; /* words in use, no leading zero words */
} big;

static void big_trim(big* a) {
    while (a->n > 0 && a->w[a->n - 1] == 0) --a->n;
}
static void big_set_u128(big* a, u128 v) {
    memset(a, 0, sizeof(*a));
    a->w[0] = (u64)v;
    a->w[1] = (u64)(v >> 64);
    a->n = 2;
    big_trim(a);
}
static void big_pow2(big* a, size_t bits) {
    memset(a, 0, sizeof(*a));
    a->w[bits / 64] = ((u64)1) << (bits % 64);
    a->n = (int)(bits / 64) + 1;
}
static size_t big_bitlen(const big* a) {
    if (!a->n) return 0;
    return 64 * (size_t)(a->n - 1) + (64 - __builtin_clzll(a->w[a->n - 1]));
}
static void big_mul_u64(big* a, u64 m) {
    u64 carry = 0;
    for (int i = 0; i < a->n; ++i) {
        u128 t = (u128)a->w[i] * m + carry;
        a->w[i] = (u64)t;
        carry = (u64)(t >> 64);
    }
    if (carry) a->w[a->n++] = carry;
    big_trim(a);
}
static int big_cmp(const big* a, const big* b) {
    if (a->n != b->n) return a->n < b->n ? -1 : 1;
    for (int i = a->n - 1; i >= 0; --i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}
static void big_sub(big* a, const big* b) { /* a -= b, a >= b */
    u64 borrow = 0;
    for (int i = 0; i < a->n; ++i) {
        u64 bi = i < b->n ? b->w[i] : 0;
        u64 d = a->w[i] - bi;
        u64 bo = (a->w[i] < bi) | (d < borrow);
        a->w[i] = d - borrow;
        borrow = bo;
    }
    big_trim(a);
}
static void big_shl(big* a, size_t bits) {
    if (!a->n || !bits) return;
    size_t words = bits / 64, rem = bits % 64;
    big out;
    memset(&out, 0, sizeof(out));
    for (int i = 0; i < a->n; ++i) {
        out.w[i + words] |= rem ? (a->w[i] << rem) : a->w[i];
        if (rem) out.w[i + words + 1] |= a->w[i] >> (64 - rem);
    }
    out.n = a->n + (int)words + 1;
    big_trim(&out);
    *a = out;
}
static void big_shr1(big* a) {
    for (int i = 0; i < a->n; ++i) {
        a->w[i] >>= 1;
        if (i + 1 < a->n) a->w[i] |= a->w[i + 1] << 63;
    }
    big_trim(a);
}
static void big_divide(big* t, const big* d, big* q) { /* q = t / d (t destroyed) */
    memset(q, 0, sizeof(*q));
    if (!d->n || big_cmp(t, d) < 0) return;
    long shift = (long)big_bitlen(t) - (long)big_bitlen(d);
    big* cur = (big*)malloc(sizeof(big));
    *cur = *d;
    big_shl(cur, (size_t)shift);
    q->n = (int)(shift / 64) + 1;
    for (long s = shift; s >= 0; --s) {
        if (big_cmp(cur, t) <= 0) {
            big_sub(t, cur);
            q->w[s / 64] |= ((u64)1) << (s % 64);
        }
        big_shr1(cur);
    }
    free(cur);
    big_trim(q);
}

/* field.cpp:158-171 */
static unsigned default_iterations(unsigned b, u64 c) {
    if (c == 1) return 2;
    big* cm = (big*)malloc(sizeof(big));
    big* p2 = (big*)malloc(sizeof(big));
    big_set_u128(cm, c);
    big_mul_u64(cm, c);
    unsigned m = 2;
    for (;;) {
        ++m;
        big_mul_u64(cm, c);
        big_pow2(p2, (size_t)b * (m - 2));
        if (big_bitlen(cm) <= (size_t)b * (m - 2) && big_cmp(cm, p2) <= 0) break;
    }
    free(cm);
    free(p2);
    return m;
}

/* field.cpp:176-193 */
static void domain_threshold(unsigned b, u64 c, unsigned n, u64 out[4]) {
    big* qn = (big*)malloc(sizeof(big));
    big* d = (big*)malloc(sizeof(big));
    big* cn1 = (big*)malloc(sizeof(big));
    big* v = (big*)malloc(sizeof(big));
    big* clamp = (big*)malloc(sizeof(big));
    big* t = (big*)malloc(sizeof(big));
    big_pow2(qn, (size_t)b * n);
    if ((c & (c - 1)) == 0) {
        big_set_u128(d, 1);
        for (unsigned i = 0; i < n; ++i) big_mul_u64(d, c);
    } else {
        big_set_u128(d, c);
        big_shl(d, (size_t)b * (n - 1));
    }
    big_sub(qn, d);
    big_set_u128(cn1, 1);
    for (unsigned i = 0; i + 1 < n; ++i) big_mul_u64(cn1, c);
    big_divide(qn, cn1, v);
    big_pow2(clamp, 255);
    big_pow2(t, 127);
    big_sub(clamp, t);
    const big* r = big_cmp(v, clamp) < 0 ? v : clamp;
    for (int i = 0; i < 4; ++i) out[i] = i < r->n ? r->w[i] : 0;
    free(qn);
    free(d);
    free(cn1);
    free(v);
    free(clamp);
    free(t);
}

unsigned orc_pm_setup(unsigned b, u64 c, unsigned m_iters, u64 max_input[4]) {
    /* field.cpp:224-244 */
    if (b < 2 || b > 127) return 0;
    if (c == 0 || (b - 1 < 64 && c >= (((u64)1) << (b - 1)))) return 0;
    unsigned m = m_iters ? m_iters : default_iterations(b, c);
    domain_threshold(b, c, m, max_input);
    return m;
}

/* field.cpp:246-258 (generic engine arithmetic; for b <= 61 the native engine
 * computes the same integers) */
static u256 pm_div_w(unsigned b, u64 c, unsigned iters, u256 v) {
    u256 cw = w_of(c);
    u256 vp = w_add(v, cw);
    u256 z = w_shr(vp, b);
    for (unsigned i = 1; i < iters; ++i) z = w_shr(w_add(w_mul(z, cw), vp), b);
    return z;
}

void orc_pm_div_iters(unsigned b, u64 c, unsigned iters, u64 v_lo, u64 v_hi, u64* q_lo,
                      u64* q_hi) {
    u256 z = pm_div_w(b, c, iters, w_of(((u128)v_hi << 64) | v_lo));
    *q_lo = z.l[0];
    *q_hi = z.l[1];
}

int orc_pm_divmod(unsigned b, u64 c, unsigned m, const u64 max_input[4], u64 v_lo, u64 v_hi,
                  u64* q_lo, u64* q_hi, u64* r_lo, u64* r_hi) {
    u256 v = w_of(((u128)v_hi << 64) | v_lo);
    u256 mx = {{max_input[0], max_input[1], max_input[2], max_input[3]}};
    if (w_cmp(v, mx) > 0) return 1; /* field.cpp:261-263 */
    u256 z = pm_div_w(b, c, m, v);
    /* field.cpp:267-273: (v + z c) & (2^b - 1) */
    u256 r = w_mask(w_add(w_mul(z, w_of(c)), v), b);
    *q_lo = z.l[0];
    *q_hi = z.l[1];
    *r_lo = r.l[0];
    *r_hi = r.l[1];
    return 0;
}

u64 orc_pm_divmod_batch(unsigned b, u64 c, unsigned m, const u64 max_input[4], const u64* v,
                        u64 n, u64* q, u64* r) {
    u64 rejected = 0;
#pragma omp parallel for schedule(static) reduction(+ : rejected)
    for (u64 i = 0; i < n; ++i) {
        u64 ql, qh, rl, rh;
        if (orc_pm_divmod(b, c, m, max_input, v[2 * i], v[2 * i + 1], &ql, &qh, &rl, &rh)) {
            ++rejected;
            ql = rl = 0;
        }
        q[i] = ql;
        r[i] = rl;
    }
    return rejected;
}

/* field.cpp:275-311 (Alg 8) */
void orc_cch_divmod(unsigned b, u64 c, u64 v_lo, u64 v_hi, u64* q_lo, u64* q_hi, u64* r_lo,
                    u64* r_hi) {
    u256 x = w_of(((u128)v_hi << 64) | v_lo);
    u256 cw = w_of(c);
    u256 q = w_shr(x, b), r = w_mask(x, b);
    u256 quot = q, rem = r;
    u256 zero = {{0, 0, 0, 0}};
    while (w_cmp(q, zero) != 0) {
        u256 t = w_mul(q, cw);
        q = w_shr(t, b);
        quot = w_add(quot, q);
        rem = w_add(rem, w_mask(t, b));
    }
    u256 one = {{1, 0, 0, 0}};
    u256 p = w_of((((u128)1) << b) - c);
    while (w_cmp(rem, p) >= 0) {
        rem = w_sub(rem, p);
        quot = w_add(quot, one);
    }
    *q_lo = quot.l[0];
    *q_hi = quot.l[1];
    *r_lo = rem.l[0];
    *r_hi = rem.l[1];
}

/* ======================= sketch.cpp:13-34 (Alg 2, Alg 6/7) ============== */
void orc_split_pow2(u64 h_lo, u64 h_hi, unsigned b, unsigned l, u64* index, int* sign) {
    u128 h = ((u128)h_hi << 64) | h_lo;
    u128 i = h & ((((u128)1) << l) - 1);
    int a = (int)(h >> (b - 1));
    *index = (u64)i;
    *sign = 1 - 2 * a;
}

/* bucketing.cpp:61-66 map_pow2: (v * r) >> b at full width */
static u128 scaled_shift(u128 v, u128 r, unsigned b) {
    return w_low128(w_shr(w_mul(w_of(v), w_of(r)), b));
}

void orc_split_arb_uniform(u64 h_lo, u64 h_hi, unsigned b, u64 r, u64* index, int* sign) {
    u128 h = ((u128)h_hi << 64) | h_lo;
    u128 j = h & ((((u128)1) << (b - 1)) - 1);
    *index = (u64)scaled_shift(j, r, b - 1);
    int a = (int)(h >> (b - 1));
    *sign = 2 * a - 1;
}

void orc_split_arb_mersenne(u64 h_lo, u64 h_hi, unsigned b, u64 r, u64* index, int* sign) {
    u128 h = (((u128)h_hi << 64) | h_lo) + 1;
    orc_split_arb_uniform((u64)h, (u64)(h >> 64), b, r, index, sign);
}

/* ---- bucket maps (bucketing.cpp:61-95) ---- */

/* bucketing.cpp:75-89: the iteration count grows from 1 until the largest
 * product (p-1) r lies inside domain_threshold(b, c, m).  0 = invalid r. */
unsigned orc_exact_div_iterations(unsigned b, u64 c, u64 r) {
    const u128 p = (((u128)1) << b) - c;
    if (r == 0 || (u128)r > p) return 0; /* "bucket count must be in [1, p]" */
    u256 largest = w_mul(w_of(p - 1), w_of(r));
    for (unsigned m = 1;; ++m) {
        u64 mx[4];
        domain_threshold(b, c, m, mx);
        u256 t = {{mx[0], mx[1], mx[2], mx[3]}};
        if (w_cmp(largest, t) <= 0) return m;
    }
}

/* kind 0 = map_pow2 (:61-66), 1 = map_mersenne (:68-73),
 * 2 = ExactDivisionMap::operator() (:91-95) with m from orc_exact_div_iterations */
u64 orc_bucket_map(int kind, unsigned b, u64 c, unsigned m, u64 r, u64 v) {
    switch (kind) {
        case 0: return (u64)scaled_shift(v, r, b);
        case 1: return (u64)scaled_shift((u128)v + 1, r, b);
        default: return pm_div_w(b, c, m, w_mul(w_of(v), w_of(r))).l[0];
    }
}

void orc_bucket_map_batch(int kind, unsigned b, u64 c, unsigned m, u64 r, const u64* v, u64 n, u64* out) {
#pragma omp parallel for schedule(static)
    for (u64 i = 0; i < n; ++i) out[i] = orc_bucket_map(kind, b, c, m, r, v[i]);
}

/* ======================= sketch.cpp:121-193 (Count Sketch) ============== */
static inline void split_dispatch(int splitter, unsigned b, u64 width, unsigned lw, u128 h,
                                  unsigned sub, u64* idx, int* sign) {
    switch (splitter) {
        case 0: orc_split_pow2((u64)h, (u64)(h >> 64), b, lw, idx, sign); break;
        case 1: orc_split_arb_uniform((u64)h, (u64)(h >> 64), b, width, idx, sign); break;
        case 2: orc_split_arb_mersenne((u64)h, (u64)(h >> 64), b, width, idx, sign); break;
        default: {
            /* TwoForOne: row `sub` = split_pow2 of the substring
             * bits [l sub, b - sub) of h, i.e. (h >> l sub) & (2^bs - 1) with
             * bs = b - (l + 1) sub: index bits [l sub, l sub + l), sign bit b-1-sub.
             * For b = 89, l = 16: row 0 = split_pow2(h, 89, 16), row 1 =
             * split_pow2((h >> 16) & (2^72 - 1), 72, 16). */
            u128 hs = h >> (lw * sub);
            unsigned bs = b - (lw + 1) * sub;
            hs &= (((u128)1) << bs) - 1;
            orc_split_pow2((u64)hs, (u64)(hs >> 64), bs, lw, idx, sign);
            break;
        }
    }
}

static inline unsigned ctz64(u64 v) { return (unsigned)__builtin_ctzll(v); }

u64 orc_cs_process(unsigned rows, u64 width, unsigned b, unsigned k, const u64* clo,
                   const u64* chi, unsigned key_bits, int splitter, const u64* keys64,
                   const uint32_t* keys32, const int32_t* w32, const int64_t* w64, u64 n,
                   i64* counters) {
    /* all-or-nothing domain validation (the batch API's documented delta from
     * the reference's throw-mid-stream, sketch.cpp:133 -> polyhash.cpp:60) */
    u64 rejected = 0;
    if (key_bits < 64) {
        const u64 lim = ((u64)1) << key_bits;
#pragma omp parallel for schedule(static) reduction(+ : rejected)
        for (u64 i = 0; i < n; ++i) {
            u64 x = keys64 ? keys64[i] : keys32[i];
            rejected += (x >= lim);
        }
    }
    if (rejected) return rejected;
    const unsigned lw = ctz64(width);
    const unsigned fams = splitter == 3 ? (rows + 1) / 2 : rows;
    const size_t cells = (size_t)rows * width;
#pragma omp parallel
    {
        i64* local = (i64*)calloc(cells, sizeof(i64));
#pragma omp for schedule(static)
        for (u64 i = 0; i < n; ++i) {
            u128 x = keys64 ? keys64[i] : keys32[i];
            i64 delta = w64 ? w64[i] : (w32 ? (i64)w32[i] : 1);
            for (unsigned f = 0; f < fams; ++f) {
                u128 h = 0;
                if (b <= 61 && key_bits > b - 1) {
                    /* beyond the reference domain (u > 2^(b-1)): the GPU path reduces keys
                     * exactly; restated as Horner with Alg-3 full reduction per step */
                    u64 xr = mod_full61(b, x), y = clo[(size_t)f * k + k - 1];
                    for (unsigned j = k - 1; j-- > 0;) y = mod_full61(b, (u128)y * xr + clo[(size_t)f * k + j]);
                    h = y;
                } else {
                    hash_one(b, clo + (size_t)f * k, chi + (size_t)f * k, k, 128, x, 0, &h);
                }
                unsigned subs = splitter == 3 ? 2 : 1;
                for (unsigned s = 0; s < subs; ++s) {
                    unsigned row = splitter == 3 ? 2 * f + s : f;
                    if (row >= rows) break;
                    u64 idx;
                    int sign;
                    split_dispatch(splitter, b, width, lw, h, s, &idx, &sign);
                    u64 sd = sign > 0 ? (u64)delta : (u64)0 - (u64)delta;
                    i64* c = &local[(size_t)row * width + idx];
                    *c = (i64)((u64)*c + sd); /* sketch.cpp:138, wrapping */
                }
            }
        }
#pragma omp critical
        orc_cs_merge(counters, local, cells);
        free(local);
    }
    return 0;
}

void orc_cs_merge(i64* dst, const i64* src, u64 count) {
    for (u64 i = 0; i < count; ++i) dst[i] = (i64)((u64)dst[i] + (u64)src[i]); /* :189-191 */
}

void orc_cs_row_moment(const i64* base, u64 width, u64* lo, u64* hi, int* saturated) {
    /* sketch.cpp:142-158 */
    u128 sum = 0;
    int sat = 0;
    for (u64 i = 0; i < width; ++i) {
        u64 mag = base[i] < 0 ? (u64)0 - (u64)base[i] : (u64)base[i];
        u128 sq = (u128)mag * mag;
        if (sum > ~(u128)0 - sq) {
            sat = 1;
            sum = ~(u128)0;
            break;
        }
        sum += sq;
    }
    *lo = (u64)sum;
    *hi = (u64)(sum >> 64);
    *saturated = sat;
}

void orc_cs_second_moment(const i64* counters, unsigned rows, u64 width, int median, u64* lo,
                          u64* hi, int* saturated) {
    /* sketch.cpp:160-168: lower median [(t-1)/2] of rows sorted by value */
    if (!median || rows == 1) {
        orc_cs_row_moment(counters, width, lo, hi, saturated);
        return;
    }
    u128 v[256];
    int s[256];
    for (unsigned r = 0; r < rows && r < 256; ++r) {
        u64 l, h;
        orc_cs_row_moment(counters + (size_t)r * width, width, &l, &h, &s[r]);
        v[r] = ((u128)h << 64) | l;
    }
    /* stable insertion sort by value (std::sort ties carry equal values, so the
     * returned value is order-independent; the flag of equal values can differ
     * only when both saturated, i.e. value == 2^128-1 in both) */
    for (unsigned i = 1; i < rows; ++i) {
        u128 kv = v[i];
        int ks = s[i];
        int j = (int)i - 1;
        while (j >= 0 && v[j] > kv) {
            v[j + 1] = v[j];
            s[j + 1] = s[j];
            --j;
        }
        v[j + 1] = kv;
        s[j + 1] = ks;
    }
    unsigned m = (rows - 1) / 2;
    *lo = (u64)v[m];
    *hi = (u64)(v[m] >> 64);
    *saturated = s[m];
}

static int cmp_i64(const void* a, const void* b) {
    i64 x = *(const i64*)a, y = *(const i64*)b;
    return x < y ? -1 : x > y;
}

u64 orc_cs_point_query(unsigned rows, u64 width, unsigned b, unsigned k, const u64* clo,
                       const u64* chi, unsigned key_bits, int splitter, const i64* counters,
                       const u64* keys, u64 n, i64* out) {
    u64 rejected = 0;
    const unsigned lw = ctz64(width);
    for (u64 i = 0; i < n; ++i) {
        i64 est[256];
        unsigned ne = 0;
        int bad = 0;
        const unsigned fams = splitter == 3 ? (rows + 1) / 2 : rows;
        for (unsigned f = 0; f < fams && !bad; ++f) {
            u128 h = 0;
            if (hash_one(b, clo + (size_t)f * k, chi + (size_t)f * k, k, key_bits, keys[i], 0,
                         &h)) {
                bad = 1;
                break;
            }
            unsigned subs = splitter == 3 ? 2 : 1;
            for (unsigned s = 0; s < subs; ++s) {
                unsigned row = splitter == 3 ? 2 * f + s : f;
                if (row >= rows) break;
                u64 idx;
                int sign;
                split_dispatch(splitter, b, width, lw, h, s, &idx, &sign);
                i64 c = counters[(size_t)row * width + idx];
                est[ne++] = sign > 0 ? c : (i64)((u64)0 - (u64)c);
            }
        }
        if (bad) {
            ++rejected;
            out[i] = 0;
            continue;
        }
        qsort(est, ne, sizeof(i64), cmp_i64);
        out[i] = est[(ne - 1) / 2];
    }
    return rejected;
}

/* ======================= synthetic workload generators ================== */
#define SALT_KEYS 0x7b5bad595e238e31ULL /* bench.cpp:23 */
#define SALT_TAIL 0x9E6C63D0676A9A99ULL
#define SALT_W 0xD1B54A32D192ED03ULL
#define SALT_PERM 0x2545F4914F6CDD1DULL

void orc_gen_u32_keys(u64 key_seed, u64 start, u64 n, uint32_t* out) {
#pragma omp parallel for schedule(static)
    for (u64 i = 0; i < n; ++i) out[i] = (uint32_t)orc_splitmix_at(key_seed, start + i);
}

void orc_gen_u64_keys(u64 key_seed, u64 start, u64 n, u64* out) {
#pragma omp parallel for schedule(static)
    for (u64 i = 0; i < n; ++i) out[i] = orc_splitmix_at(key_seed, start + i);
}

u64 orc_gen_below_p61(u64 key_seed, u64 start, u64 n, u64* out) {
    const u64 p = (((u64)1) << 61) - 1;
    u64 bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (u64 i = 0; i < n; ++i) {
        u64 v = orc_splitmix_at(key_seed, start + i) >> 3; /* below(p): shift = 3 */
        bad += (v >= p);
        out[i] = v;
    }
    return bad;
}

u64 orc_gen_pm_inputs(u64 key_seed, u64 c, u64 start, u64 n, u64* out) {
    const u128 p = ~(u128)0 >> 64; /* 2^64 - 1 */
    const u128 pp = p + 1 - c;     /* 2^64 - c */
    u256 psq = w_mul(w_of(pp), w_of(pp));
    u64 bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (u64 i = 0; i < n; ++i) {
        u64 hi = orc_splitmix_at(key_seed, 2 * (start + i));
        u64 lo = orc_splitmix_at(key_seed, 2 * (start + i) + 1);
        u256 v = w_of(((u128)hi << 64) | lo);
        bad += (w_cmp(v, psq) >= 0);
        out[2 * i] = lo;
        out[2 * i + 1] = hi;
    }
    return bad;
}

static u64 to_fixed64(double x) {
    double s = x * 18446744073709551616.0;
    if (s >= 18446744073709551615.0) return ~(u64)0;
    if (s <= 0) return 0;
    return (u64)s;
}

void orc_zipf_table(double alpha, uint32_t T, double universe, u64* cdf, double* tail_c1) {
    double head = 0;
    for (uint32_t r = 1; r <= T; ++r) head += pow((double)r, -alpha);
    double tail = (pow(T + 0.5, 1 - alpha) - pow(universe + 0.5, 1 - alpha)) / (alpha - 1);
    double total = head + tail;
    double acc = 0;
    for (uint32_t r = 1; r <= T; ++r) {
        acc += pow((double)r, -alpha);
        cdf[r - 1] = to_fixed64(acc / total);
    }
    *tail_c1 = 1.0 - pow((universe + 0.5) / (T + 0.5), 1 - alpha);
}

uint32_t orc_feistel32(u64 key, uint32_t x) {
    uint32_t L = x >> 16, R = x & 0xFFFF;
    for (uint32_t round = 0; round < 4; ++round) {
        uint32_t F = (uint32_t)(mix64(key ^ (((u64)round << 16) | R)) >> 48);
        uint32_t nl = R;
        R = (L ^ F) & 0xFFFF;
        L = nl;
    }
    return (L << 16) | R;
}

void orc_gen_zipf_items(u64 master_seed, const u64* cdf, uint32_t T, double tail_c1,
                        double universe, u64 start, u64 n, uint32_t* keys, int32_t* weights) {
    const u64 sk = master_seed ^ SALT_KEYS;
    const u64 st = sk ^ SALT_TAIL;
    const u64 sw = sk ^ SALT_W;
    const u64 sp = master_seed ^ SALT_PERM;
    const u64 head_total = cdf[T - 1];
#pragma omp parallel for schedule(static)
    for (u64 i = 0; i < n; ++i) {
        const u64 gi = start + i;
        u64 u = orc_splitmix_at(sk, gi);
        u64 rank;
        if (u < head_total) {
            uint32_t lo = 0, hi = T - 1; /* smallest j with cdf[j] > u */
            while (lo < hi) {
                uint32_t mid = (lo + hi) >> 1;
                if (cdf[mid] > u) hi = mid;
                else lo = mid + 1;
            }
            rank = (u64)lo + 1;
        } else {
            u64 v = orc_splitmix_at(st, gi);
            double w = (double)(v >> 11) * 0x1p-53;
            double s = 1.0 - w * tail_c1;
            double s2 = s * s;
            double s4 = s2 * s2;
            double s5 = s4 * s;
            double xr = ((double)T + 0.5) / s5;
            double xf = xr + 0.5;
            if (xf > universe) xf = universe;
            rank = (u64)xf;
            if (rank < (u64)T + 1) rank = (u64)T + 1;
        }
        keys[i] = orc_feistel32(sp, (uint32_t)(rank - 1));
        if (weights) {
            u64 z = orc_splitmix_at(sw, gi);
            weights[i] = (int32_t)(((z >> 32) * 201ULL) >> 32) - 100;
        }
    }
}

/* ======================= exact enumeration (verify.cpp:508-546 style) ===== */
/* Sum over ALL p^k coefficient vectors of a one-row sketch's second moment and
 * of the row point-query estimate at `qkey` (test_sketch.cpp:119-178 frozen
 * values).  Small fields only. */
void orc_enum_sums(unsigned b, unsigned k, unsigned key_bits, u64 width, int splitter,
                   const u64* keys, const int64_t* deltas, u64 n, u64 qkey, u64* sum_f2,
                   int64_t* sum_pq) {
    const u64 p = (((u64)1) << b) - 1;
    u64 total = 1;
    for (unsigned i = 0; i < k; ++i) total *= p;
    u64 s2 = 0;
    int64_t spq = 0;
#pragma omp parallel for schedule(static) reduction(+ : s2, spq)
    for (u64 idx = 0; idx < total; ++idx) {
        u64 lo[16], hi[16];
        u64 t = idx;
        for (unsigned i = 0; i < k; ++i) {
            lo[i] = t % p;
            hi[i] = 0;
            t /= p;
        }
        int64_t c[64];
        for (u64 j = 0; j < width; ++j) c[j] = 0;
        for (u64 j = 0; j < n; ++j) {
            u128 h;
            hash_one(b, lo, hi, k, key_bits, keys[j], 0, &h);
            u64 ix;
            int sg;
            split_dispatch(splitter, b, width, ctz64(width), h, 0, &ix, &sg);
            c[ix] = (int64_t)((u64)c[ix] + (sg > 0 ? (u64)deltas[j] : (u64)0 - (u64)deltas[j]));
        }
        u64 l2, h2;
        int sat;
        orc_cs_row_moment(c, width, &l2, &h2, &sat);
        s2 += l2;
        u128 h;
        hash_one(b, lo, hi, k, key_bits, qkey, 0, &h);
        u64 ix;
        int sg;
        split_dispatch(splitter, b, width, ctz64(width), h, 0, &ix, &sg);
        spq += sg > 0 ? c[ix] : -c[ix];
    }
    *sum_f2 = s2;
    *sum_pq = spq;
}

/* verify.cpp:505-546 moment_range + 555-603 enum_moment_sums_{serial,parallel}:
 * for every (a0, a1, a2, a3) in Z_p^4 (p = 2^b - 1, a0 the x^3 coefficient)
 * fill the one-row sketch of the stream, then X = sum c^2 (u64) and accumulate
 * sum_x += X, sum_x_sq += X^2 (u128).  Restated loop for loop, counters
 * included; the split tables are apply_splitter (verify.cpp:389-399), which
 * is split_pow2 with l = bit_width(r) - 1 or the arbitrary-width splitters.
 * out: sum_x lo/hi, sum_x_sq lo/hi.  Parallel over a0 like the reference's
 * parallel kernel (integer sums: identical for any thread count). */
void orc_enum_moment_sums(unsigned b, u64 buckets, int splitter, const u64* keys,
                          const int64_t* deltas, u64 n, u64 out[4]) {
    const u64 p = (((u64)1) << b) - 1;
    unsigned* idx = (unsigned*)malloc(sizeof(unsigned) * p);
    int* sgn = (int*)malloc(sizeof(int) * p);
    unsigned lw = 0;
    while ((((u64)1) << (lw + 1)) <= buckets) ++lw; /* bit_width(r) - 1 */
    for (u64 h = 0; h < p; ++h) {
        u64 ix;
        int sg;
        split_dispatch(splitter, b, buckets, lw, (u128)h, 0, &ix, &sg);
        idx[h] = (unsigned)ix;
        sgn[h] = sg;
    }
    u64 *x1 = (u64*)malloc(8 * (n + 1)), *x2 = (u64*)malloc(8 * (n + 1)), *x3 = (u64*)malloc(8 * (n + 1));
    for (u64 j = 0; j < n; ++j) {
        x1[j] = keys[j] % p;
        x2[j] = x1[j] * x1[j] % p;
        x3[j] = x2[j] * x1[j] % p;
    }
    u128 sum_x = 0, sum_xx = 0;
#pragma omp parallel
    {
        u128 lx = 0, lxx = 0;
        u64* t0 = (u64*)malloc(8 * (n + 1));
        u64* t1 = (u64*)malloc(8 * (n + 1));
        u64* t2 = (u64*)malloc(8 * (n + 1));
        int64_t* counters = (int64_t*)malloc(8 * buckets);
#pragma omp for schedule(static)
        for (u64 a0 = 0; a0 < p; ++a0) {
            for (u64 j = 0; j < n; ++j) t0[j] = a0 * x3[j] % p;
            for (u64 a1 = 0; a1 < p; ++a1) {
                for (u64 j = 0; j < n; ++j) t1[j] = (t0[j] + a1 * x2[j]) % p;
                for (u64 a2 = 0; a2 < p; ++a2) {
                    for (u64 j = 0; j < n; ++j) t2[j] = (t1[j] + a2 * x1[j]) % p;
                    for (u64 a3 = 0; a3 < p; ++a3) {
                        memset(counters, 0, 8 * buckets);
                        for (u64 j = 0; j < n; ++j) {
                            u64 h = t2[j] + a3;
                            if (h >= p) h -= p;
                            counters[idx[h]] += sgn[h] * deltas[j];
                        }
                        u64 x_val = 0;
                        for (u64 i = 0; i < buckets; ++i) x_val += (u64)(counters[i] * counters[i]);
                        lx += x_val;
                        lxx += (u128)x_val * x_val;
                    }
                }
            }
        }
#pragma omp critical
        {
            sum_x += lx;
            sum_xx += lxx;
        }
        free(t0);
        free(t1);
        free(t2);
        free(counters);
    }
    out[0] = (u64)sum_x;
    out[1] = (u64)(sum_x >> 64);
    out[2] = (u64)sum_xx;
    out[3] = (u64)(sum_xx >> 64);
    free(idx);
    free(sgn);
    free(x1);
    free(x2);
    free(x3);
}
