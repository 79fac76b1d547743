"""Pin the CPU oracle (oracle/oracle.c) before trusting it.

(a) known-answer values frozen in the reference's own unit tests
    (/root/reference/proj/tests/unit/*.cpp, acceptance.cpp);
(b) golden vectors produced by executing the compiled reference
    (tests/golden/golden.json, tests/golden/make_golden.py);
(c) when oracle/_ref is built (this container), randomized cross-checks
    against the reference itself.
"""
import ctypes as C
from fractions import Fraction

import numpy as np
import pytest

from oracle_bind import ptr

P61 = (1 << 61) - 1
P89 = (1 << 89) - 1


# ------------------------------------------------------------------ (a) KATs
def test_hash_known_answers(orc):
    # test_polyhash.cpp:68-81
    assert [orc.hash(3, [3, 5], x, key_bits=2) for x in (2, 0, 1, 3)] == [6, 3, 1, 4]
    for x in range(16):
        assert orc.hash(5, [0, 1, 0, 0], x, key_bits=4) == x
        assert orc.hash(5, [23, 0, 0, 0], x, key_bits=4) == 23
    with pytest.raises(ValueError, match="key outside domain"):
        orc.hash(3, [3, 5], 4, key_bits=2)


def test_branch_free_finish_matches_conditional_subtract(orc):
    # test_polyhash.cpp:157-191 (b = 3 exhaustive)
    for a0 in range(7):
        for a1 in range(7):
            for x in range(4):
                assert orc.hash(3, [a0, a1], x, 2, 0) == orc.hash(3, [a0, a1], x, 2, 1)


def test_split_known_answers(orc):
    # test_sketch.cpp:14-54
    assert orc.split(0, 0b110, 3, 2) == (2, -1)
    assert orc.split(0, 0, 3, 2) == (0, 1)
    assert orc.split(0, 0b011, 3, 2) == (3, 1)
    for h in range(8):
        assert orc.split(0, h, 3, 1) == (h & 1, -1 if h >= 4 else 1)
    assert orc.split(1, 0b1011, 4, 3) == (1, 1)
    assert orc.split(1, 0, 4, 3) == (0, -1)
    assert orc.split(2, 3, 3, 3) == (0, 1)
    assert orc.split(2, 6, 3, 3) == (2, 1)
    assert sum(orc.split(2, h, 3, 3)[0] == 0 for h in range(7)) == 3


def test_field_known_answers(orc):
    # test_field.cpp:79-158
    assert orc.reduce_partial(3, 13) == 6
    assert orc.reduce_partial(3, 0) == 0
    assert orc.reduce_partial(3, 48) == 6
    assert orc.mersenne_divmod(3, 30) == (4, 2)
    assert orc.mersenne_divmod(3, 63) == (9, 0)
    assert orc.mersenne_divmod(3, 0) == (0, 0)
    with pytest.raises(ValueError, match="exceeds 2"):
        orc.mersenne_divmod(3, 64)
    m, mx, _ = orc.pm_setup(4, 3, 2)
    assert (m, mx) == (2, 69)
    assert orc.pm_divmod(4, 3, 27, 2)[0] == 2
    assert orc.pm_divmod(4, 3, 69, 2)[0] == 5
    with pytest.raises(ValueError, match="division domain"):
        orc.pm_divmod(4, 3, 70, 2)
    assert orc.pm_divmod(4, 3, 27, 2)[1] == 1
    assert orc.pm_divmod(3, 1, 30, 2)[0] == 4
    assert orc.pm_divmod(3, 1, 48, 2)[1] == 6
    assert orc.cch_divmod(4, 3, 27) == (2, 1)
    assert orc.cch_divmod(3, 1, 63) == (9, 0)
    # default iteration count (test_field.cpp:174-188)
    assert orc.pm_setup(3, 1)[0] == 2
    assert orc.pm_setup(61, 1)[0] == 2
    assert orc.pm_setup(127, 1)[0] == 2
    # config 3: 2^64 - 59 needs 3 rounds and admits all of [0, 2^128) (181-bit bound)
    m, mx, _ = orc.pm_setup(64, 59)
    assert m == 3 and mx.bit_length() == 181


def test_divmod_exhaustive_small_widths(orc):
    # test_field.cpp:120-134 (subset of widths; exhaustive per width)
    for b in (2, 3, 5, 7):
        p = (1 << b) - 1
        for v in range(1 << (2 * b)):
            assert orc.mersenne_divmod(b, v) == (v // p, v % p)


def test_sketch_known_answers(orc):
    # test_sketch.cpp:106-117: one key with delta -7 gives 49 in every row and the median
    seeds = orc.row_seeds(0xF00D, 3)
    fams = [orc.coeffs(61, 4, s) for s in seeds]
    c = orc.cs_process(3, 8, 61, fams, 32, 0, np.array([123], np.uint64), np.array([-7], np.int64))
    for r in range(3):
        assert orc.row_moment(c[8 * r:8 * r + 8], 8) == (49, False)
    assert orc.second_moment(c, 3, 8, True) == (49, False)
    # cancellation (test_sketch.cpp:56-73)
    c = orc.cs_process(3, 8, 61, fams, 32, 0, np.array([17, 17], np.uint64), np.array([5, -5], np.int64))
    assert not c.any()


@pytest.mark.parametrize("splitter", [0, 2])
def test_exact_enumeration_values(orc, splitter):
    # test_sketch.cpp:119-178: sums over all 31^4 degree-3 families
    f = orc.lib.orc_enum_sums
    f.restype = None
    f.argtypes = [C.c_uint, C.c_uint, C.c_uint, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                  C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    keys = np.array([1, 3, 7], np.uint64)
    d = np.array([2, -1, 3], np.int64)
    s2, pq = C.c_uint64(), C.c_int64()
    f(5, 4, 4, 4, splitter, ptr(keys), ptr(d), 3, 1, C.byref(s2), C.byref(pq))
    assert s2.value == 12931216
    assert pq.value == 1848964


def test_saturation_semantics(orc):
    # sketch.cpp:142-158: INT64_MIN squares via its magnitude; overflow saturates
    c = np.array([np.iinfo(np.int64).min] * 4, np.int64)
    v, sat = orc.row_moment(c, 4)
    assert sat and v == (1 << 128) - 1
    c = np.array([np.iinfo(np.int64).min, 0], np.int64)
    assert orc.row_moment(c, 2) == (1 << 126, False)


# ------------------------------------------------------------------ (b) golden
def test_golden_coefficients(orc, golden):
    S = golden["seed"]
    assert orc.coeffs(61, 4, S) == golden["coeffs"]["61_4"]
    assert orc.coeffs(61, 8, S) == golden["coeffs"]["61_8"]
    assert orc.coeffs(89, 4, S) == [int(c) for c in golden["coeffs"]["89_4"]]
    assert orc.row_seeds(S, 5) == [int(s) for s in golden["row_seeds_5"]]


def test_golden_hashes(orc, golden):
    g = golden["hash61_u32"]
    lo, _, rej = orc.hash_batch(61, g["coeffs"], np.array(g["keys"], np.uint64), 32)
    assert rej == 0 and [int(x) for x in lo] == g["out"]
    g = golden["hash61_full"]
    for k in (4, 8):
        out = orc.hash_full(61, g[f"k{k}"]["coeffs"], np.array(g["keys"], np.uint64))
        assert [int(x) for x in out] == g[f"k{k}"]["out"]
        # and against exact big-integer arithmetic
        for x, h in zip(g["keys"][:16], out[:16]):
            y = 0
            for a in reversed(g[f"k{k}"]["coeffs"]):
                y = (y * x + a) % P61
            assert y == int(h)
    g = golden["hash89"]
    coeffs = [int(c) for c in g["coeffs"]]
    lo, hi, rej = orc.hash_batch(89, coeffs, np.array(g["keys"], np.uint64), 64)
    assert [int(l) | (int(h) << 64) for l, h in zip(lo, hi)] == [int(v) for v in g["out"]]
    for x, h in zip(g["keys"][:16], g["out"][:16]):
        y = 0
        for a in reversed(coeffs):
            y = (y * x + a) % P89
        assert y == int(h)


def test_golden_divmod(orc, golden):
    g = golden["pm_divmod"]
    m, mx, _ = orc.pm_setup(g["b"], g["c"])
    assert m == g["iterations"] and mx == int(g["max_input"])
    v = [int(x) for x in g["v"]]
    flat = np.array([w for x in v for w in (x & (2**64 - 1), x >> 64)], np.uint64)
    q, r, rej = orc.pm_divmod_batch(64, 59, flat)
    assert rej == 0
    assert [int(x) for x in q] == g["q"] and [int(x) for x in r] == g["r"]
    p = (1 << 64) - 59
    assert all(int(q[i]) == v[i] // p and int(r[i]) == v[i] % p for i in range(len(v)))


def test_golden_sketches(orc, golden):
    S, SK = golden["seed"], golden["key_seed"]
    g = golden["c1_sketch"]
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, 1)]
    keys = orc.gen_u32_keys(SK, 0, g["n"])
    c = orc.cs_process(1, 1024, 61, fams, 32, 0, keys)
    assert [int(x) for x in c] == g["counters"]
    assert orc.row_moment(c, 1024)[0] == int(g["f2"])

    g = golden["c5_sketch"]
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, 5)]
    k, w = orc.gen_zipf_items(S, 0, g["n"])
    assert [int(x) for x in k[:64]] == g["keys_head"] and [int(x) for x in w[:64]] == g["weights_head"]
    c = orc.cs_process(5, 65536, 61, fams, 32, 0, k, w)
    nz = np.nonzero(c)[0]
    assert [int(x) for x in nz] == g["nonzero_index"]
    assert [int(x) for x in c[nz]] == g["nonzero_value"]
    assert [orc.row_moment(c[r * 65536:(r + 1) * 65536], 65536)[0] for r in range(5)] == \
        [int(x) for x in g["row_f2"]]
    assert orc.second_moment(c, 5, 65536, True)[0] == int(g["median_f2"])

    g = golden["c4_sketch"]
    c89 = orc.coeffs(89, 4, S)
    keys = orc.gen_u64_keys(SK, 0, g["n"])
    c = orc.cs_process(2, 65536, 89, [c89], 64, 3, keys)
    nz = np.nonzero(c)[0]
    assert [int(x) for x in nz] == g["nonzero_index"]
    assert [int(x) for x in c[nz]] == g["nonzero_value"]


def test_golden_point_query(orc, golden):
    g = golden["point_query"]
    S = golden["seed"]
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, g["rows"])]
    c = orc.cs_process(g["rows"], g["width"], 61, fams, 32, 0, np.array(g["keys"], np.uint64),
                       np.array(g["weights"], np.int64))
    out = orc.point_query(g["rows"], g["width"], 61, fams, 32, 0, c, np.array(g["query"], np.uint64))
    assert [int(x) for x in out] == g["out"]


# ------------------------------------------------------------------ generators
def test_counter_form_equals_sequential_stream(orc):
    seed = 0x1234
    st = C.c_uint64(seed)
    seq = [orc.lib.orc_splitmix_next(C.byref(st)) for _ in range(64)]
    assert [orc.lib.orc_splitmix_at(seed, i) for i in range(64)] == seq
    assert [int(x) for x in orc.gen_u64_keys(seed, 0, 64)] == seq
    assert [int(x) for x in orc.gen_u64_keys(seed, 10, 5)] == seq[10:15]
    assert [int(x) for x in orc.gen_u32_keys(seed, 0, 64)] == [s & 0xFFFFFFFF for s in seq]
    # below(p) for p = 2^61 - 1 (prng.hpp:22-34): shift 3, rejection probability 2^-61
    st = C.c_uint64(seed)
    below = [orc.lib.orc_splitmix_below(C.byref(st), P61) for _ in range(64)]
    assert [int(x) for x in orc.gen_below_p61(seed, 0, 64)] == below


def test_zipf_stream_shape(orc):
    keys, w = orc.gen_zipf_items(1, 0, 1 << 18)
    _, counts = np.unique(keys, return_counts=True)
    top = counts.max() / len(keys)
    # Zipf(1.2) over 2^32: P(rank 1) = 1 / H(2^32, 1.2) ~ 0.180
    assert 0.17 < top < 0.19
    assert w.min() == -100 and w.max() == 100
    # shards are independent windows of one stream
    k2, w2 = orc.gen_zipf_items(1, 1000, 100)
    assert (k2 == keys[1000:1100]).all() and (w2 == w[1000:1100]).all()
    # the Feistel rank->key map is a bijection on a sample
    xs = np.arange(0, 1 << 16, dtype=np.uint64)
    ys = {orc.lib.orc_feistel32(77, int(x)) for x in xs}
    assert len(ys) == len(xs)


# ------------------------------------------------------------------ (c) vs reference
def test_oracle_matches_reference_random(orc, ref):
    rng = np.random.default_rng(5)
    for b, k in [(61, 4), (61, 8), (89, 4), (31, 4), (13, 2), (127, 4)]:
        seed = int(rng.integers(0, 2**63))
        assert orc.coeffs(b, k, seed) == ref.coeffs(b, k, seed, key_bits=min(b - 1, 32) if b < 64 else 64)
    for b, kb in [(61, 32), (61, 60), (31, 20), (89, 64), (89, 88)]:
        c = orc.coeffs(b, 4, 99)
        keys = rng.integers(0, 2**min(kb, 63), size=4096, dtype=np.uint64)
        if kb == 64:
            keys = orc.gen_u64_keys(3, 0, 4096)
        a = orc.hash_batch(b, c, keys, kb)
        r = ref.hash_batch(b, c, keys, kb)
        assert (a[0] == r[0]).all() and (a[1] == r[1]).all()


def test_pm_setup_matches_reference(orc, ref):
    # test_field.cpp "domain threshold matches reference" style sweep, c < 2^64
    rng = np.random.default_rng(0xD0)
    for _ in range(200):
        b = int(rng.integers(2, 128))
        bits = int(rng.integers(1, min(b - 1, 63) + 1))
        c = int(rng.integers(1, 2**bits))
        if b - 1 < 64 and c >= 1 << (b - 1):
            c >>= 1
        c = max(c, 1)
        n = int(rng.integers(1, 7))
        assert orc.pm_setup(b, c, n)[:2] == ref.pm_setup(b, c, n)
    for b, c in [(64, 59), (61, 1), (4, 3), (32, 5), (64, 1)]:
        assert orc.pm_setup(b, c)[:2] == ref.pm_setup(b, c)


def test_divmod_matches_reference_random(orc, ref):
    v = orc.gen_pm_inputs(11, 59, 0, 20000)
    q1, r1, _ = orc.pm_divmod_batch(64, 59, v)
    q2, r2, _ = ref.pm_divmod_batch(64, 59, v)
    assert (q1 == q2).all() and (r1 == r2).all()
    for b, c in [(33, 7), (48, 1), (61, 1), (64, 1), (40, 1000)]:
        m, mx = ref.pm_setup(b, c)
        rng = np.random.default_rng(b)
        vals = [int(x) % min(mx + 1, 1 << 128) for x in rng.integers(0, 2**63, 64, dtype=np.uint64)]
        for x in vals:
            x = (x * 0x9E3779B97F4A7C15) % min(mx + 1, 1 << 128)
            assert orc.pm_divmod(b, c, x) == ref.pm_divmod(b, c, x)


def test_sketch_matches_reference_all_splitters(orc, ref):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 20, size=3000, dtype=np.uint64)
    w = rng.integers(-1000, 1000, size=3000).astype(np.int64)
    for splitter, width in [(0, 64), (1, 48), (2, 48)]:
        fams = [orc.coeffs(31, 4, s) for s in orc.row_seeds(0xC0FFEE, 3)]
        a = orc.cs_process(3, width, 31, fams, 20, splitter, keys, w)
        r, moms, med = ref.cs_run(3, width, 31, 20, splitter, 0xC0FFEE, keys, w)
        assert (a == r).all()
        assert orc.second_moment(a, 3, width, True) == med


# ------------------------------------------------------------------ bucket maps
def _counts(vals, r):
    return np.bincount(np.asarray(vals, np.int64), minlength=r).tolist()


def test_bucket_map_known_answers(orc):
    # test_bucketing.cpp:101-127 (ExactDivisionMap over p = 13 and p = 7)
    m, out = orc.bucket_map(2, 4, 4, np.arange(13), c=3)
    assert _counts(out, 4) == [4, 3, 3, 3]
    _, ident = orc.bucket_map(2, 4, 13, np.arange(13), c=3)
    assert ident.tolist() == list(range(13))
    _, div3 = orc.bucket_map(2, 3, 3, np.arange(7), c=1)
    _, mer3 = orc.bucket_map(1, 3, 3, np.arange(7))
    assert sorted(_counts(div3, 3)) == sorted(_counts(mer3, 3))
    assert _counts(div3, 3) != _counts(mer3, 3)
    assert div3.tolist() != mer3.tolist()
    assert orc.lib.orc_exact_div_iterations(4, 3, 0) == 0
    assert orc.lib.orc_exact_div_iterations(4, 3, 14) == 0
    assert orc.lib.orc_exact_div_iterations(4, 3, 13) > 0
    # test_bucketing.cpp:83-98 (map_pow2 / map_mersenne)
    _, pw = orc.bucket_map(0, 3, 3, np.arange(8))
    assert sorted(_counts(pw, 3)) == [2, 3, 3]
    assert orc.bucket_map(0, 5, 32, np.arange(32))[1].tolist() == list(range(32))
    assert orc.bucket_map(0, 5, 1, np.arange(32))[1].tolist() == [0] * 32
    assert orc.bucket_map(1, 3, 1, np.arange(7))[1].tolist() == [0] * 7
    assert _counts(orc.bucket_map(1, 3, 7, np.arange(7))[1], 7) == [1] * 7


def test_bucket_maps_most_uniform(orc):
    # test_bucketing.cpp:129-150: every map keeps preimage sizes within one
    for b in (4, 6, 9, 11):
        q = 1 << b
        for r in (1, 2, 3, 5, 8, 17, 33, 64):
            if r > q - 1:
                continue
            for kind, dom, c in ((0, q, 0), (1, q - 1, 0), (2, q - 3, 3)):
                _, out = orc.bucket_map(kind, b, r, np.arange(dom), c=c)
                cnt = _counts(out, r)
                assert max(cnt) - min(cnt) <= 1 and sum(cnt) == dom


def test_bucket_maps_match_reference(orc, ref):
    rng = np.random.default_rng(0xB0C)
    cases = [(0, 64, 0, 1000003), (0, 17, 0, 5), (1, 64, 0, 2**63 + 12345), (1, 40, 0, 77),
             (2, 64, 59, 2**64 - 59), (2, 64, 59, 1000), (2, 64, 2**62 + 1, 12345), (2, 33, 7, 2**32),
             (2, 20, 1, 3), (2, 61, 1, 2**61 - 1), (2, 48, 2**40 + 3, 2**47)]
    for kind, b, c, r in cases:
        dom = (1 << b) - (c if kind == 2 else kind)
        v = (rng.integers(0, 2**63, 4096, dtype=np.uint64) * np.uint64(3)) % np.uint64(dom) \
            if dom < 2**64 else rng.integers(0, 2**63, 4096, dtype=np.uint64) * np.uint64(2)
        v[:3] = [0, 1, dom - 1]
        mo, out_o = orc.bucket_map(kind, b, r, v, c=c)
        mr, out_r = ref.bucket_map(kind, b, r, v, c=c)
        assert mo == mr, (kind, b, c, r)
        assert (out_o == out_r).all(), (kind, b, c, r)
    assert ref.bucket_map(2, 4, 14, np.arange(3), c=3)[0] == 0  # invalid_argument


def test_golden_bucket_maps(orc, golden):
    for case in golden["bucket_maps"]:
        m, out = orc.bucket_map(case["kind"], case["b"], int(case["r"]), np.array(case["v"], np.uint64),
                                c=int(case["c"]))
        assert m == case["iterations"]
        assert out.tolist() == case["out"]


# ------------------------------------------------------------------ moment enumeration
ENUM_STREAM = [(1, 2), (3, -1), (7, 3)]


def test_enum_moment_sums_known_answers(orc):
    # test_verify.cpp:205-216 (frozen values), :227-243 (variance 45352128/923521 for
    # Pow2 r=4), :245-256 (variance 60396800/923521 for MersenneArb r=3): with
    # F = 923521 families, sum_x_sq = F var + sum_x^2 / F.
    F = 31 ** 4
    sx, sxx = orc.enum_moment_sums(5, 4, 0, ENUM_STREAM)
    assert (sx, sxx) == (12931216, 226416064)
    assert F * Fraction(sxx, F) - Fraction(sx * sx, F) == 45352128
    assert orc.enum_moment_sums(5, 4, 2, ENUM_STREAM)[0] == 12931216
    sx3, sxx3 = orc.enum_moment_sums(5, 3, 2, ENUM_STREAM)
    assert F * Fraction(sxx3, F) - Fraction(sx3 * sx3, F) == 60396800
    # single key: X = 81 for every family, variance exactly zero (:258-265)
    assert orc.enum_moment_sums(5, 4, 0, [(5, 9)]) == (81 * F, 6561 * F)


@pytest.mark.parametrize("b,r,splitter", [(3, 2, 0), (3, 3, 1), (5, 3, 1), (5, 5, 2), (5, 8, 0)])
def test_enum_moment_mean_is_exact(orc, b, r, splitter):
    # size-independent property (verify.cpp:621-625, p prime): E[X] = (F2 p^2 + F1^2 - F2) / p^2
    p = (1 << b) - 1
    stream = [(0, 3), (2, -2), (5, 1), (p - 1, 4)][: 3 if b == 3 else 4]
    sx, sxx = orc.enum_moment_sums(b, r, splitter, stream)
    f1 = sum(d for _, d in stream)
    f2 = sum(d * d for _, d in stream)
    assert Fraction(sx, p ** 4) == Fraction(f2 * p * p + f1 * f1 - f2, p * p)
    assert sxx >= sx * sx // p ** 4


def _digest(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_matches_reference_large_goldens(orc, golden):
    """The restated oracle reproduces the reference-executed >= 2^22-unit digests
    (tests/golden/make_golden.py large_prefixes), so the GPU's large-batch kernels and
    the oracle are pinned to the same reference outputs."""
    L = golden["large"]
    S, SK = golden["seed"], golden["key_seed"]
    fams5 = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, 5)]
    for name in ("c5_head", "c5_window"):
        g = L[name]
        zk, zw = orc.gen_zipf_items(S, g["start"], g["n"])
        t = orc.cs_process(5, 65536, 61, fams5, 32, 0, zk, zw)
        assert _digest(t) == g["sha256"]
        assert [str(orc.row_moment(t[r * 65536:(r + 1) * 65536], 65536)[0]) for r in range(5)] == g["row_f2"]
        assert str(orc.second_moment(t, 5, 65536, True)[0]) == g["median_f2"]
    g = L["c4_head"]
    t = orc.cs_process(2, 65536, 89, [orc.coeffs(89, 4, S)], 64, 3, orc.gen_u64_keys(SK, 0, g["n"]))
    assert _digest(t) == g["sha256"]
    g = L["c1_full"]
    t = orc.cs_process(1, 1024, 61, [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, 1)], 32, 0,
                       orc.gen_u32_keys(SK, 0, g["n"]))
    assert _digest(t) == g["sha256"] and str(orc.row_moment(t, 1024)[0]) == g["f2"]
    kp = orc.gen_below_p61(SK, 0, L["c2_k4_head"]["n"])
    for k in (4, 8):
        assert _digest(orc.hash_full(61, orc.coeffs(61, k, S), kp)) == L[f"c2_k{k}_head"]["sha256"]
    v = orc.gen_pm_inputs(SK, 59, 0, L["c3_head"]["n"])
    q, r, _ = orc.pm_divmod_batch(64, 59, v)
    assert _digest(q) == L["c3_head"]["q_sha256"] and _digest(r) == L["c3_head"]["r_sha256"]
