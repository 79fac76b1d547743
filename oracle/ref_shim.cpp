// ref_shim.cpp -- extern "C" bridge onto the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE.  Compiled by oracle/Makefile together with
// the reference sources where they lie (/root/reference/proj/src/{field,
// polyhash,bucketing,sketch}.cpp and src/cli/bench.cpp) into
// oracle/_ref/libmersenne_ref.so, at the reference's own Release flags
// (-std=c++20 -O3, NDEBUG stripped so assert() stays live; CMakeLists.txt:11-15).
// Used (a) by tests/golden/make_golden.py to freeze golden vectors, (b) by the
// parity tests to cross-check the oracle restatement, and (c) by bench.py
// --impl reference / cpu_baseline as the reference CPU path.  This file only
// calls the reference's public API; it restates nothing.
#include <omp.h>

#include <cstring>
#include <stdexcept>
#include <vector>

#include "mersenne/bucketing.hpp"
#include "mersenne/cli.hpp"
#include "mersenne/field.hpp"
#include "mersenne/polyhash.hpp"
#include "mersenne/sketch.hpp"

using namespace mersenne;

namespace {

u128 mk(uint64_t lo, uint64_t hi) { return (u128(hi) << 64) | lo; }

std::vector<u128> coeff_vec(const uint64_t* lo, const uint64_t* hi, unsigned k) {
    std::vector<u128> v(k);
    for (unsigned i = 0; i < k; ++i) v[i] = mk(lo[i], hi ? hi[i] : 0);
    return v;
}

}  // namespace

extern "C" {

// PolyHashFamily(MersenneModulus(b,true), k, 2^key_bits, seed).coefficients()
int ref_coeffs(unsigned b, unsigned k, unsigned key_bits, uint64_t seed, uint64_t* lo,
               uint64_t* hi) {
    try {
        PolyHashFamily f(MersenneModulus(b, true), k, u128(1) << key_bits, seed);
        for (unsigned i = 0; i < k; ++i) {
            lo[i] = uint64_t(f.coefficients()[i]);
            hi[i] = uint64_t(f.coefficients()[i] >> 64);
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// row seeds of CountSketch(rows, ..., seed)
int ref_row_seeds(unsigned rows, uint64_t seed, uint64_t* out) {
    CountSketch sk(rows, 2, MersenneModulus(61, true), u128(1) << 32, Splitter::Pow2, seed);
    for (unsigned r = 0; r < rows; ++r) out[r] = sk.seeds()[r];
    return 0;
}

// PolyHashFamily::operator() on a batch; rc per key: 0 ok, 1 domain_error.
uint64_t ref_hash_batch(unsigned b, const uint64_t* clo, const uint64_t* chi, unsigned k,
                        unsigned key_bits, int finish, const uint64_t* keys, uint64_t n,
                        uint64_t* out_lo, uint64_t* out_hi, int threads) {
    PolyHashFamily f(MersenneModulus(b, true), coeff_vec(clo, chi, k), u128(1) << key_bits,
                     finish ? HashFinish::BranchFree : HashFinish::ConditionalSubtract);
    uint64_t rejected = 0;
#pragma omp parallel for schedule(static) num_threads(threads) reduction(+ : rejected)
    for (uint64_t i = 0; i < n; ++i) {
        u128 h = 0;
        try {
            h = f(keys[i]);
        } catch (const std::domain_error&) {
            ++rejected;
        }
        out_lo[i] = uint64_t(h);
        if (out_hi) out_hi[i] = uint64_t(h >> 64);
    }
    return rejected;
}

// Config-2 restatement over keys in [0,2^64) using the reference's own Alg 3
// (mersenne_divmod, field.cpp:208-222) as a full reduction per Horner step.
void ref_hash_full_batch(unsigned b, const uint64_t* coeffs, unsigned k, const uint64_t* keys,
                         uint64_t n, uint64_t* out, int threads) {
    const MersenneModulus mod(b, true);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (uint64_t i = 0; i < n; ++i) {
        u64 x = mersenne_divmod(UWide(keys[i]), mod).remainder.low_u64();
        u64 y = coeffs[k - 1];
        for (unsigned j = k - 1; j-- > 0;) {
            y = mersenne_divmod(UWide::of_u128(u128(y) * x + coeffs[j]), mod)
                    .remainder.low_u64();
        }
        out[i] = y;
    }
}

int ref_mersenne_divmod(unsigned b, uint64_t v_lo, uint64_t v_hi, uint64_t* q_lo,
                        uint64_t* q_hi, uint64_t* r_lo, uint64_t* r_hi) {
    try {
        DivMod d = mersenne_divmod(UWide::of_u128(mk(v_lo, v_hi)), MersenneModulus(b));
        *q_lo = d.quotient.limb[0];
        *q_hi = d.quotient.limb[1];
        *r_lo = d.remainder.limb[0];
        *r_hi = d.remainder.limb[1];
        return 0;
    } catch (const std::domain_error&) {
        return 1;
    }
}

// PseudoMersenneModulus(b, c, m_iters, engine) for u128 c = (c_hi << 64) | c_lo:
// returns iterations, 0 on invalid_argument
unsigned ref_pm_setup(unsigned b, uint64_t c_lo, uint64_t c_hi, unsigned m_iters, int engine,
                      uint64_t max_input[4]) {
    try {
        PseudoMersenneModulus m(b, mk(c_lo, c_hi), m_iters, Engine(engine));
        for (int i = 0; i < 4; ++i) max_input[i] = m.max_input().limb[i];
        return m.iterations();
    } catch (const std::invalid_argument&) {
        return 0;
    }
}

// pseudo_mersenne_div + pseudo_mersenne_mod (bench.cpp:165-175's pair) on a batch
uint64_t ref_pm_divmod_batch(unsigned b, uint64_t c, unsigned m_iters, const uint64_t* v,
                             uint64_t n, uint64_t* q, uint64_t* r, int threads) {
    const PseudoMersenneModulus mod(b, c, m_iters);
    uint64_t rejected = 0;
#pragma omp parallel for schedule(static) num_threads(threads) reduction(+ : rejected)
    for (uint64_t i = 0; i < n; ++i) {
        try {
            const UWide vw = UWide::of_u128(mk(v[2 * i], v[2 * i + 1]));
            const UWide z = pseudo_mersenne_div(vw, mod);
            const UWide y = pseudo_mersenne_mod(vw, z, mod);
            q[i] = z.limb[0];
            r[i] = y.limb[0];
        } catch (const std::domain_error&) {
            ++rejected;
            q[i] = r[i] = 0;
        }
    }
    return rejected;
}

int ref_pm_divmod(unsigned b, uint64_t c, unsigned m_iters, uint64_t v_lo, uint64_t v_hi,
                  uint64_t* q_lo, uint64_t* q_hi, uint64_t* r_lo, uint64_t* r_hi) {
    try {
        const PseudoMersenneModulus mod(b, c, m_iters);
        const UWide vw = UWide::of_u128(mk(v_lo, v_hi));
        const UWide z = pseudo_mersenne_div(vw, mod);
        const UWide y = pseudo_mersenne_mod(vw, z, mod);
        *q_lo = z.limb[0];
        *q_hi = z.limb[1];
        *r_lo = y.limb[0];
        *r_hi = y.limb[1];
        return 0;
    } catch (const std::domain_error&) {
        return 1;
    }
}

void ref_cch_divmod(unsigned b, uint64_t c, uint64_t v_lo, uint64_t v_hi, uint64_t* q_lo,
                    uint64_t* q_hi, uint64_t* r_lo, uint64_t* r_hi) {
    const PseudoMersenneModulus mod(b, c);
    DivMod d = cch_divmod(UWide::of_u128(mk(v_lo, v_hi)), mod);
    *q_lo = d.quotient.limb[0];
    *q_hi = d.quotient.limb[1];
    *r_lo = d.remainder.limb[0];
    *r_hi = d.remainder.limb[1];
}

void ref_split(int which, uint64_t h_lo, uint64_t h_hi, unsigned b, uint64_t l_or_r,
               uint64_t* index, int* sign) {
    SignIndexPair s = which == 0   ? split_pow2(mk(h_lo, h_hi), b, unsigned(l_or_r))
                      : which == 1 ? split_arb_uniform(mk(h_lo, h_hi), b, l_or_r)
                                   : split_arb_mersenne(mk(h_lo, h_hi), b, l_or_r);
    *index = uint64_t(s.index);
    *sign = s.sign;
}

// bucketing.cpp:61-95 on a batch: kind 0 map_pow2(v, b, r), 1 map_mersenne(v, b, r),
// 2 ExactDivisionMap(PseudoMersenneModulus(b, c), r)(v).  Returns the divider's
// iteration count for kind 2 (1 otherwise), 0 if the constructor threw.
unsigned ref_bucket_map(int kind, unsigned b, uint64_t c, uint64_t r, const uint64_t* v,
                        uint64_t n, uint64_t* out) {
    if (kind == 2) {
        try {
            const ExactDivisionMap map(PseudoMersenneModulus(b, c), r);
            for (uint64_t i = 0; i < n; ++i) out[i] = uint64_t(map(v[i]));
            return map.divider().iterations();
        } catch (const std::invalid_argument&) {
            return 0;
        }
    }
    for (uint64_t i = 0; i < n; ++i)
        out[i] = uint64_t(kind == 0 ? map_pow2(v[i], b, r) : map_mersenne(v[i], b, r));
    return 1;
}

// Seeded CountSketch(rows, width, MersenneModulus(b,true), 2^key_bits, splitter, seed);
// process(key, w) over the batch, sharded over `threads` sketches + merge()
// (bit-identical to one serial pass: test_sketch.cpp:239-261).
// Returns 0, or 1 if a key was rejected (domain_error) -- mid-stream, as the reference.
int ref_cs_run(unsigned rows, uint64_t width, unsigned b, unsigned key_bits, int splitter,
               uint64_t seed, const uint64_t* keys64, const uint32_t* keys32,
               const int32_t* w32, const int64_t* w64, uint64_t n, int threads,
               int64_t* counters, uint64_t* moments /* rows x (lo,hi,sat) + median (lo,hi,sat) */) {
    const MersenneModulus mod(b, true);
    auto fresh = [&] {
        return CountSketch(rows, width, mod, u128(1) << key_bits, Splitter(splitter), seed);
    };
    std::vector<CountSketch> parts;
    for (int t = 0; t < threads; ++t) parts.push_back(fresh());
    int bad = 0;
#pragma omp parallel num_threads(threads) reduction(| : bad)
    {
        const int t = omp_get_thread_num();
        const int nt = omp_get_num_threads();
        const uint64_t lo = n * uint64_t(t) / uint64_t(nt), hi = n * uint64_t(t + 1) / uint64_t(nt);
        CountSketch& sk = parts[size_t(t)];
        try {
            for (uint64_t i = lo; i < hi; ++i) {
                const u128 x = keys64 ? u128(keys64[i]) : u128(keys32[i]);
                const i64 d = w64 ? w64[i] : (w32 ? i64(w32[i]) : 1);
                sk.process(x, d);
            }
        } catch (const std::domain_error&) {
            bad = 1;
        }
    }
    for (int t = 1; t < threads; ++t) parts[0].merge(parts[size_t(t)]);
    const CountSketch& sk = parts[0];
    std::memcpy(counters, sk.counters().data(), sk.counters().size() * sizeof(int64_t));
    if (moments) {
        for (unsigned r = 0; r < rows; ++r) {
            auto m = sk.row_second_moment(r);
            moments[3 * r] = uint64_t(m.value);
            moments[3 * r + 1] = uint64_t(m.value >> 64);
            moments[3 * r + 2] = m.saturated;
        }
        auto m = sk.second_moment(true);
        moments[3 * rows] = uint64_t(m.value);
        moments[3 * rows + 1] = uint64_t(m.value >> 64);
        moments[3 * rows + 2] = m.saturated;
    }
    return bad;
}

// Injected-family CountSketch(width, splitter, {families}) (sketch.cpp:84-95),
// serial; coefficients row-major rows x k.
int ref_cs_run_families(unsigned rows, uint64_t width, unsigned b, unsigned key_bits,
                        int splitter, unsigned k, const uint64_t* clo, const uint64_t* chi,
                        const uint64_t* keys64, const int64_t* w64, uint64_t n,
                        int64_t* counters, uint64_t* moments) {
    const MersenneModulus mod(b, true);
    std::vector<PolyHashFamily> fams;
    for (unsigned r = 0; r < rows; ++r) {
        fams.emplace_back(mod, coeff_vec(clo + size_t(r) * k, chi ? chi + size_t(r) * k : nullptr, k),
                          u128(1) << key_bits);
    }
    CountSketch sk(width, Splitter(splitter), std::move(fams));
    try {
        for (uint64_t i = 0; i < n; ++i) sk.process(keys64[i], w64 ? w64[i] : 1);
    } catch (const std::domain_error&) {
        return 1;
    }
    std::memcpy(counters, sk.counters().data(), sk.counters().size() * sizeof(int64_t));
    if (moments) {
        for (unsigned r = 0; r < rows; ++r) {
            auto m = sk.row_second_moment(r);
            moments[3 * r] = uint64_t(m.value);
            moments[3 * r + 1] = uint64_t(m.value >> 64);
            moments[3 * r + 2] = m.saturated;
        }
        auto m = sk.second_moment(true);
        moments[3 * rows] = uint64_t(m.value);
        moments[3 * rows + 1] = uint64_t(m.value >> 64);
        moments[3 * rows + 2] = m.saturated;
    }
    return 0;
}

// point_query of a seeded sketch after processing a stream
int ref_cs_point_query(unsigned rows, uint64_t width, unsigned b, unsigned key_bits, int splitter,
                       uint64_t seed, const uint64_t* keys, const int64_t* w, uint64_t n,
                       const uint64_t* qkeys, uint64_t nq, int64_t* out) {
    CountSketch sk(rows, width, MersenneModulus(b, true), u128(1) << key_bits,
                   Splitter(splitter), seed);
    try {
        for (uint64_t i = 0; i < n; ++i) sk.process(keys[i], w ? w[i] : 1);
        for (uint64_t i = 0; i < nq; ++i) out[i] = sk.point_query(qkeys[i]);
    } catch (const std::domain_error&) {
        return 1;
    }
    return 0;
}

// MCSK1 serialization of a seeded sketch after a stream (sketch.cpp:195-211)
uint64_t ref_cs_serialize(unsigned rows, uint64_t width, unsigned b, unsigned key_bits,
                          int splitter, uint64_t seed, const uint64_t* keys, const int64_t* w,
                          uint64_t n, uint8_t* out, uint64_t cap) {
    CountSketch sk(rows, width, MersenneModulus(b, true), u128(1) << key_bits,
                   Splitter(splitter), seed);
    for (uint64_t i = 0; i < n; ++i) sk.process(keys[i], w ? w[i] : 1);
    auto bytes = sk.serialize();
    if (bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return bytes.size();
}

// Resume a serialized sketch in the reference (sketch.cpp:213-244): deserialize the
// MCSK1 bytes, process (keys, w) serially, serialize again.  Returns the new size
// (bytes written only when cap suffices); 0 when deserialize throws.
uint64_t ref_cs_resume(const uint8_t* bytes, uint64_t len, const uint64_t* keys, const int64_t* w,
                       uint64_t n, uint8_t* out, uint64_t cap, uint64_t* f2_lo, uint64_t* f2_hi) {
    try {
        CountSketch sk = CountSketch::deserialize(std::vector<uint8_t>(bytes, bytes + len));
        for (uint64_t i = 0; i < n; ++i) sk.process(keys[i], w ? w[i] : 1);
        const auto m = sk.second_moment(true);
        *f2_lo = uint64_t(m.value);
        *f2_hi = uint64_t(m.value >> 64);
        auto b = sk.serialize();
        if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
        return b.size();
    } catch (const std::invalid_argument&) {
        return 0;
    }
}

// Config 4's two-for-one table from the reference's own pieces: the
// 89-bit PolyHashFamily::operator() and split_pow2 applied to the two substrings
// (row 0: split_pow2(h, 89, 16); row 1: split_pow2((h >> 16) & (2^72 - 1), 72, 16)),
// unit deltas, wrapping adds like CountSketch::process.  Serial.
void ref_two_for_one_run(const uint64_t* clo, const uint64_t* chi, unsigned k, const uint64_t* keys, uint64_t n,
                         int64_t* table, int threads) {
    const PolyHashFamily fam(MersenneModulus(89, true), coeff_vec(clo, chi, k), u128(1) << 64);
    // contiguous shards over host threads, per-thread tables summed after (the
    // table is linear, like CountSketch::merge); threads = 1 is one serial pass
    const int t = threads > 0 ? threads : 1;
    std::vector<std::vector<uint64_t>> part(size_t(t), std::vector<uint64_t>(2 * 65536, 0));
#pragma omp parallel num_threads(t)
    {
        const int id = omp_get_thread_num();
        std::vector<uint64_t>& tab = part[size_t(id)];
        const uint64_t lo = n * uint64_t(id) / uint64_t(t), hi = n * uint64_t(id + 1) / uint64_t(t);
        for (uint64_t i = lo; i < hi; ++i) {
            const u128 h = fam(keys[i]);
            const auto a = split_pow2(h, 89, 16);
            const auto b = split_pow2((h >> 16) & ((u128(1) << 72) - 1), 72, 16);
            tab[size_t(a.index)] += uint64_t(int64_t(a.sign));
            tab[65536 + size_t(b.index)] += uint64_t(int64_t(b.sign));
        }
    }
    for (const auto& tab : part)
        for (size_t j = 0; j < tab.size(); ++j) table[j] = int64_t(uint64_t(table[j]) + tab[j]);
}

// The reference's own benchmark loops (bench.cpp:96-189): median of 5 after 3 warm-ups.
double ref_bench_hash(unsigned b, unsigned k, uint64_t n, uint64_t seed, uint64_t* checksum) {
    auto rows = cli::bench_hash(b, k, n, seed);
    *checksum = rows[0].checksum;
    return rows[0].ops_per_sec;
}

double ref_bench_div(unsigned b, uint64_t c, uint64_t n, uint64_t seed, double* cascade_ops,
                     uint64_t* checksum) {
    auto res = cli::bench_div(b, c, n, seed);
    *cascade_ops = res.cascade.ops_per_sec;
    *checksum = res.branch_free.checksum;
    return res.branch_free.ops_per_sec;
}

int ref_max_threads() { return omp_get_max_threads(); }

}  // extern "C"
