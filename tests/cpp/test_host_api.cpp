// C++ host-API tests: the reference's own unit-test cases (tests/unit/
// test_{field,polyhash,sketch}.cpp under /root/reference/proj), re-run against
// mersenne::b200 (include/mersenne_b200/mersenne_b200.hpp) on the GPU, plus
// batch parity against the C oracle (oracle/liboracle.so, test infrastructure).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mersenne_b200/mersenne_b200.hpp"
#include "../../oracle/oracle.h"

using namespace mersenne::b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (cond) {                                                            \
            ++g_pass;                                                          \
        } else {                                                               \
            ++g_fail;                                                          \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ex)                                                          \
    do {                                                                                   \
        bool thrown = false;                                                               \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const ex&) {                                                              \
            thrown = true;                                                                 \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (thrown) {                                                                      \
            ++g_pass;                                                                      \
        } else {                                                                           \
            ++g_fail;                                                                      \
            std::fprintf(stderr, "FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #ex); \
        }                                                                                  \
    } while (0)

static void test_field() {  // test_field.cpp:56-158
    CHECK(MersenneModulus(3).p() == 7);
    CHECK_THROWS_AS(MersenneModulus(1), std::invalid_argument);
    CHECK_THROWS_AS(MersenneModulus(128), std::invalid_argument);
    CHECK_THROWS_AS(MersenneModulus(11, true), std::invalid_argument);
    MersenneModulus m13(13, true);
    CHECK(m13.prime_exponent());
    CHECK_THROWS_AS(PseudoMersenneModulus(4, 8), std::invalid_argument);
    CHECK_THROWS_AS(PseudoMersenneModulus(4, 0), std::invalid_argument);
    PseudoMersenneModulus m(4, 3, 2);
    CHECK(m.p() == 13 && m.iterations() == 2 && m.max_input()[0] == 69 && m.max_input() == UWide(69));
    u64 v[4] = {27, 0, 69, 0}, q[2], r[2];
    m.divmod(v, 2, q, r);
    CHECK(q[0] == 2 && r[0] == 1 && q[1] == 5 && r[1] == 4);
    u64 bad[2] = {70, 0};
    CHECK_THROWS_AS(m.divmod(bad, 1, q, r), std::domain_error);
    CHECK(PseudoMersenneModulus(64, 59).iterations() == 3);
    CHECK(PseudoMersenneModulus(61, 1).iterations() == 2);
}

static void test_polyhash() {  // test_polyhash.cpp:57-88
    MersenneModulus m7(3, true);
    PolyHashFamily f(m7, std::vector<u128>{3, 5}, 4);
    CHECK(f(2) == 6 && f(0) == 3 && f(1) == 1 && f(3) == 4);
    CHECK_THROWS_AS(f(4), std::domain_error);
    MersenneModulus m31(5, true);
    PolyHashFamily ident(m31, std::vector<u128>{0, 1, 0, 0}, 16);
    PolyHashFamily constant(m31, std::vector<u128>{23, 0, 0, 0}, 16);
    bool ok = true;
    for (u128 x = 0; x < 16; ++x) ok &= ident(x) == x && constant(x) == 23;
    CHECK(ok);
    CHECK_THROWS_AS(PolyHashFamily(m31, 4, 32, 1), std::invalid_argument);
    CHECK_THROWS_AS(PolyHashFamily(m31, 0, 16, 1), std::invalid_argument);
    CHECK_THROWS_AS(PolyHashFamily(m31, std::vector<u128>{31}, 16), std::invalid_argument);
    // seeded draws and a 61-bit batch vs the oracle
    MersenneModulus m61(61, true);
    PolyHashFamily g(m61, 4, u128(1) << 32, 0xABCDEF);
    std::vector<u64> lo(4), hi(4);
    orc_draw_coeffs(61, 4, 0xABCDEF, lo.data(), hi.data());
    for (unsigned i = 0; i < 4; ++i) CHECK(g.coefficients()[i] == lo[i]);
    std::vector<u64> keys(10000);
    orc_gen_u64_keys(7, 0, keys.size(), keys.data());
    for (auto& k : keys) k &= 0xFFFFFFFFull;
    auto h = g.hash(keys);
    std::vector<u64> out(keys.size());
    CHECK(orc_hash_batch(61, lo.data(), hi.data(), 4, 32, keys.data(), keys.size(), out.data(), nullptr) == 0);
    bool same = true;
    for (size_t i = 0; i < keys.size(); ++i) same &= h[i] == out[i];
    CHECK(same);
    // 89-bit family
    MersenneModulus m89(89, true);
    PolyHashFamily g89(m89, 4, u128(1) << 64, 3);
    orc_draw_coeffs(89, 4, 3, lo.data(), hi.data());
    orc_gen_u64_keys(8, 0, keys.size(), keys.data());
    auto h89 = g89.hash(keys);
    std::vector<u64> oh(keys.size());
    orc_hash_batch(89, lo.data(), hi.data(), 4, 64, keys.data(), keys.size(), out.data(), oh.data());
    same = true;
    for (size_t i = 0; i < keys.size(); ++i) same &= h89[i] == ((u128(oh[i]) << 64) | out[i]);
    CHECK(same);
    // generic wide moduli (62 <= b <= 127) through mb200_hash_wide
    for (unsigned b : {62u, 107u, 127u}) {
        MersenneModulus mb(b, b != 62);  // 2^62-1 is composite: unchecked modulus
        for (unsigned k : {1u, 3u, 8u}) {
            PolyHashFamily gb(mb, k, u128(1) << 60, 11 + b + k);
            std::vector<u64> wl(k), wh(k);
            orc_draw_coeffs(b, k, 11 + b + k, wl.data(), wh.data());
            for (auto& x : keys) x &= (u64(1) << 60) - 1;
            auto hb = gb.hash(keys);
            CHECK(orc_hash_batch(b, wl.data(), wh.data(), k, 60, keys.data(), keys.size(), out.data(), oh.data()) == 0);
            same = true;
            for (size_t i = 0; i < keys.size(); ++i) same &= hb[i] == ((u128(oh[i]) << 64) | out[i]);
            CHECK(same);
        }
    }
}

static void test_bucketing() {  // test_bucketing.cpp:101-127
    PseudoMersenneModulus m13(4, 3);
    ExactDivisionMap map4(m13, 4);
    long counts[4] = {0, 0, 0, 0};
    for (u64 v = 0; v < 13; ++v) ++counts[map4(v)];
    CHECK(counts[0] == 4 && counts[1] == 3 && counts[2] == 3 && counts[3] == 3);
    ExactDivisionMap ident(m13, 13);
    bool id = true;
    for (u64 v = 0; v < 13; ++v) id &= ident(v) == v;
    CHECK(id);
    CHECK(map4.buckets() == 4 && map4.divider().iterations() >= 1);
    CHECK_THROWS_AS(ExactDivisionMap(m13, 0), std::invalid_argument);
    CHECK_THROWS_AS(ExactDivisionMap(m13, 14), std::invalid_argument);
    CHECK_THROWS_AS(map4(13), std::domain_error);
    // batch vs oracle at b = 64
    const PseudoMersenneModulus big(64, 59);
    const ExactDivisionMap dmap(big, 1000003);
    const u64 n = 4099;
    std::vector<u64> v(n), got(n);
    orc_gen_u64_keys(5, 0, n, v.data());
    for (auto& x : v) x %= u64(big.p());
    u64 *d_v = nullptr, *d_o = nullptr;
    cudaMalloc(&d_v, n * 8);
    cudaMalloc(&d_o, n * 8);
    cudaMemcpy(d_v, v.data(), n * 8, cudaMemcpyHostToDevice);
    dmap.map_device(d_v, n, d_o);
    cudaMemcpy(got.data(), d_o, n * 8, cudaMemcpyDeviceToHost);
    bool same = true;
    const unsigned m = orc_exact_div_iterations(64, 59, 1000003);
    for (u64 i = 0; i < n; ++i) same &= got[i] == orc_bucket_map(2, 64, 59, m, 1000003, v[i]);
    CHECK(same && m == dmap.divider().iterations());
    map_pow2_device(d_v, n, 64, 77, d_o);
    cudaMemcpy(got.data(), d_o, n * 8, cudaMemcpyDeviceToHost);
    same = true;
    for (u64 i = 0; i < n; ++i) same &= got[i] == orc_bucket_map(0, 64, 0, 0, 77, v[i]);
    CHECK(same);
    cudaFree(d_v);
    cudaFree(d_o);
}

static void test_sketch() {  // test_sketch.cpp
    CHECK((split_pow2(0b110, 3, 2) == SignIndexPair{2, -1}));
    CHECK((split_pow2(0, 3, 2) == SignIndexPair{0, +1}));
    CHECK((split_pow2(0b011, 3, 2) == SignIndexPair{3, +1}));
    MersenneModulus m61(61, true);
    {
        CountSketch sk(3, 8, m61, u128(1) << 32, Splitter::Pow2, 0xF00D);
        CHECK(sk.second_moment().value == 0);
        sk.process(123, -7);
        for (unsigned r = 0; r < 3; ++r) CHECK(sk.row_second_moment(r).value == 49);
        CHECK(sk.second_moment(true).value == 49);
    }
    {
        CountSketch sk(3, 8, m61, u128(1) << 32, Splitter::MersenneArb, 0xCAFE);
        sk.process(17, 5);
        sk.process(17, -5);
        bool zero = true;
        for (i64 c : sk.counters()) zero &= c == 0;
        CHECK(zero);
    }
    {
        CountSketch sk(5, 16, m61, u128(1) << 32, Splitter::MersenneArb, 0xBEEF);
        CHECK(sk.point_query(42) == 0);
        sk.process(42, 1234);
        CHECK(sk.point_query(42) == 1234);
        sk.process(42, -234);
        CHECK(sk.point_query(42) == 1000);
    }
    {  // merge equals the concatenated stream (test_sketch.cpp:239-261)
        auto fresh = [&] { return CountSketch(3, 32, m61, u128(1) << 32, Splitter::MersenneArb, 0x5EED); };
        CountSketch a = fresh(), b = fresh(), both = fresh();
        std::vector<u64> k(600);
        std::vector<i64> d(600);
        for (size_t i = 0; i < k.size(); ++i) {
            k[i] = orc_splitmix_at(0xAB, 2 * i) & 0xFFFF;
            d[i] = i64(orc_splitmix_at(0xAB, 2 * i + 1) % 200) - 100;
        }
        a.process_batch(k.data(), 64, d.data(), MB200_W_I64, 300);
        b.process_batch(k.data() + 300, 64, d.data() + 300, MB200_W_I64, 300);
        both.process_batch(k.data(), 64, d.data(), MB200_W_I64, 600);
        a.merge(b);
        CHECK(a.counters() == both.counters());
        CHECK_THROWS_AS(a.merge(CountSketch(3, 32, m61, u128(1) << 32, Splitter::MersenneArb, 1)),
                        std::invalid_argument);
    }
    // construction validation (test_sketch.cpp:278-298)
    MersenneModulus m31(5, true);
    CHECK_THROWS_AS(CountSketch(1, 1, m61, 16, Splitter::MersenneArb, 1), std::invalid_argument);
    CHECK_THROWS_AS(CountSketch(0, 8, m61, 16, Splitter::Pow2, 1), std::invalid_argument);
    CHECK_THROWS_AS(CountSketch(1, 24, m61, 16, Splitter::Pow2, 1), std::invalid_argument);
    CHECK_THROWS_AS(CountSketch(1, 32, m31, 16, Splitter::Pow2, 1), std::invalid_argument);
    CHECK_THROWS_AS(CountSketch(1, 17, m31, 16, Splitter::MersenneArb, 1), std::invalid_argument);
    CHECK_THROWS_AS(CountSketch(1, 4, m31, 32, Splitter::Pow2, 1), std::invalid_argument);
    {
        CountSketch sk(1, 4, m31, 16, Splitter::Pow2, 1);
        CHECK_THROWS_AS(sk.process(16, 1), std::domain_error);
        CHECK_THROWS_AS(sk.point_query(16), std::domain_error);
    }
    {  // config-1 slice through the host-buffer batch API vs the oracle
        CountSketch sk(1, 1024, m61, u128(1) << 32, Splitter::Pow2, 1);
        std::vector<uint32_t> keys(1 << 20);
        orc_gen_u32_keys(1 ^ 0x7b5bad595e238e31ull, 0, keys.size(), keys.data());
        sk.process_batch(keys.data(), 32, nullptr, MB200_W_NONE, keys.size());
        std::vector<u64> lo(4), hi(4);
        orc_draw_coeffs(61, 4, sk.seeds()[0], lo.data(), hi.data());
        std::vector<int64_t> exp(1024, 0);
        orc_cs_process(1, 1024, 61, 4, lo.data(), hi.data(), 32, 0, nullptr, keys.data(), nullptr, nullptr,
                       keys.size(), exp.data());
        CHECK(sk.counters() == exp);
        u64 vlo, vhi;
        int sat;
        orc_cs_row_moment(exp.data(), 1024, &vlo, &vhi, &sat);
        CHECK(sk.second_moment().value == ((u128(vhi) << 64) | vlo));
    }
}

static void test_reference_free_functions() {  // test_field.cpp:104-158, 250-277; test_sketch.cpp:14-52
    // mersenne_divmod (Alg 3)
    MersenneModulus m3(3);
    DivMod d = mersenne_divmod(UWide(30), m3);
    CHECK(d.quotient == UWide(4) && d.remainder == UWide(2));
    d = mersenne_divmod(UWide(63), m3);
    CHECK(d.quotient == UWide(9) && d.remainder == UWide(0));
    CHECK_THROWS_AS(mersenne_divmod(UWide(64), m3), std::domain_error);
    bool exact = true;
    for (u64 v = 0; v < 64; ++v) {
        const DivMod e = mersenne_divmod(UWide(v), m3);
        exact &= e.quotient == UWide(v / 7) && e.remainder == UWide(v % 7);
    }
    CHECK(exact);
    // pseudo_mersenne_div / pseudo_mersenne_mod (Alg 4, 5)
    PseudoMersenneModulus m(4, 3, 2);
    CHECK(pseudo_mersenne_div(UWide(27), m) == UWide(2));
    CHECK(pseudo_mersenne_div(UWide(69), m) == UWide(5));
    CHECK_THROWS_AS(pseudo_mersenne_div(UWide(70), m), std::domain_error);
    CHECK(pseudo_mersenne_mod(UWide(27), UWide(2), m) == UWide(1));
    CHECK(pseudo_mersenne_mod(UWide(0), UWide(0), m) == UWide(0));
    PseudoMersenneModulus m31(3, 1);
    CHECK(pseudo_mersenne_div(UWide(30), m31) == mersenne_divmod(UWide(30), m3).quotient);
    CHECK(pseudo_mersenne_mod(UWide(48), UWide(6), m31) == UWide(6));
    // Engine selection and u128 offsets (field.cpp:224-244)
    CHECK(PseudoMersenneModulus(89, 1).engine() == Engine::Generic);
    CHECK(PseudoMersenneModulus(61, 1).engine() == Engine::Native);
    CHECK(PseudoMersenneModulus(13, 5, 0, Engine::Generic).engine() == Engine::Generic);
    CHECK_THROWS_AS(PseudoMersenneModulus(89, 1, 0, Engine::Native), std::invalid_argument);
    const PseudoMersenneModulus wide(127, (u128(1) << 100) + 12345);
    CHECK(wide.c() == (u128(1) << 100) + 12345 && wide.iterations() >= 3);
    CHECK_THROWS_AS(pseudo_mersenne_div(UWide(5), wide), std::runtime_error);  // GPU division: b <= 64
    CHECK_THROWS_AS(PseudoMersenneModulus(100, u128(1) << 99), std::invalid_argument);
    // splitters
    CHECK(split_pow2(0b110, 3, 2) == (SignIndexPair{2, -1}));
    CHECK(split_arb_uniform(0b1011, 4, 3) == (SignIndexPair{1, +1}));
    CHECK(split_arb_uniform(0, 4, 3) == (SignIndexPair{0, -1}));
    CHECK(split_arb_mersenne(3, 3, 3) == (SignIndexPair{0, +1}));
    CHECK(split_arb_mersenne(6, 3, 3) == (SignIndexPair{2, +1}));
    int zero_hits = 0;
    for (u128 h = 0; h < 7; ++h) zero_hits += split_arb_mersenne(h, 3, 3).index == 0;
    CHECK(zero_hits == 3);
    // the batched device splitter against the host rule
    std::vector<u64> hs(4096);
    for (size_t i = 0; i < hs.size(); ++i) hs[i] = (i * 0x9E3779B97F4A7C15ull) >> 3;  // < 2^61
    u64* dh = nullptr;
    u64* di = nullptr;
    int32_t* ds = nullptr;
    cudaMalloc(&dh, hs.size() * 8);
    cudaMalloc(&di, hs.size() * 8);
    cudaMalloc(&ds, hs.size() * 4);
    cudaMemcpy(dh, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice);
    bool same = true;
    for (Splitter sp : {Splitter::Pow2, Splitter::UniformArb, Splitter::MersenneArb}) {
        const u64 lr = sp == Splitter::Pow2 ? 16 : 1000003;
        split_device(sp, dh, hs.size(), 61, lr, di, ds);
        std::vector<u64> idx(hs.size());
        std::vector<int32_t> sg(hs.size());
        cudaMemcpy(idx.data(), di, idx.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(sg.data(), ds, sg.size() * 4, cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < hs.size(); ++i) {
            const SignIndexPair e = sp == Splitter::Pow2       ? split_pow2(hs[i], 61, 16)
                                    : sp == Splitter::UniformArb ? split_arb_uniform(hs[i], 61, lr)
                                                                 : split_arb_mersenne(hs[i], 61, lr);
            same &= e.index == idx[i] && e.sign == sg[i];
        }
    }
    CHECK(same);
    cudaFree(dh);
    cudaFree(di);
    cudaFree(ds);
}

static void test_sketch_value_semantics() {  // sketch.hpp:72-82: counter(), operator==, copies
    MersenneModulus m61(61, true);
    CountSketch a(3, 8, m61, u128(1) << 32, Splitter::Pow2, 0xCAFE);
    a.process(99, 2);
    a.process(99, 2);
    CountSketch once(3, 8, m61, u128(1) << 32, Splitter::Pow2, 0xCAFE);
    once.process(99, 4);
    CHECK(a == once);  // test_sketch.cpp:56-72
    CountSketch copy(a);
    CHECK(copy == a);
    copy.process(7, 1);
    CHECK(!(copy == a));  // independent HBM tables
    const std::vector<int64_t> c = a.counters();
    bool cells = true;
    for (unsigned r = 0; r < 3; ++r)
        for (u64 i = 0; i < 8; ++i) cells &= a.counter(r, i) == c[r * 8 + i];
    CHECK(cells);
    CountSketch other(3, 8, m61, u128(1) << 32, Splitter::Pow2, 0xBEEF);
    other = a;
    CHECK(other == a && other.seeds() == a.seeds());
}

static void test_allreduce() {  // SURVEY 8b entry 6: CountSketch::allreduce over NCCL
    MersenneModulus m61(61, true);
    NcclCommunicator comm(1, NcclCommunicator::unique_id(), 0);  // one GPU: a one-rank job
    CHECK(comm.size() == 1 && comm.get() != nullptr);
    CountSketch a(5, 4096, m61, u128(1) << 32, Splitter::Pow2, 7);
    CountSketch b(5, 4096, m61, u128(1) << 32, Splitter::Pow2, 7);
    std::vector<uint32_t> keys(1 << 16);
    std::vector<int32_t> w(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        keys[i] = uint32_t(i * 2654435761u);
        w[i] = int32_t(i % 201) - 100;
    }
    a.process_batch(keys.data(), 32, w.data(), MB200_W_I32, keys.size() / 2);
    b.process_batch(keys.data() + keys.size() / 2, 32, w.data() + keys.size() / 2, MB200_W_I32, keys.size() / 2);
    a.merge(b);                                  // the single-process merge
    const std::vector<int64_t> merged = a.counters();
    a.allreduce(comm.get());                     // one rank: the sum over ranks is the table itself
    CHECK(a.counters() == merged);
    CHECK_THROWS_AS(a.allreduce(nullptr), std::invalid_argument);
}

int main() {
    try {
        test_field();
        test_polyhash();
        test_bucketing();
        test_sketch();
        test_reference_free_functions();
        test_sketch_value_semantics();
        test_allreduce();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
