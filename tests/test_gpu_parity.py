"""Parity of the sm_100a path with the CPU oracle, through the C-ABI.

Bit-exact for every kernel (integer work).  Sizes: golden fixtures, seeded
oracle comparisons at sizes the oracle finishes in seconds, and BASELINE
full sizes through exact sampled comparisons plus size-independent properties.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P61 = (1 << 61) - 1
P89 = (1 << 89) - 1
M64 = (1 << 64) - 1


def dev(a):
    import torch

    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def host_u64(t):
    return t.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- hashing
def test_small_field_known_answers(cuda, mb):
    # test_polyhash.cpp:68-81 through the generic-b kernel
    out = mb.hash61(dev(np.array([2, 0, 1, 3], np.uint64)), [3, 5], b=3, key_bits=2)
    assert list(host_u64(out)) == [6, 3, 1, 4]
    x = dev(np.arange(16, dtype=np.uint32))
    assert list(host_u64(mb.hash61(x, [0, 1, 0, 0], b=5, key_bits=4))) == list(range(16))
    assert list(host_u64(mb.hash61(x, [23, 0, 0, 0], b=5, key_bits=4))) == [23] * 16


def test_pairwise_and_fourwise_exhaustive(cuda, mb, orc):
    # every family of p = 31, k = 4 on keys 0..15 equals the oracle
    import itertools

    x = dev(np.arange(16, dtype=np.uint64))
    rng = np.random.default_rng(0)
    for a in itertools.islice(itertools.product(range(31), repeat=4), 0, 923521, 9001):
        got = host_u64(mb.hash61(x, list(a), b=5, key_bits=4))
        exp = orc.hash_batch(5, list(a), np.arange(16, dtype=np.uint64), 4)[0]
        assert (got == exp).all()
    del rng


def test_golden_hash61_u32(cuda, mb, golden):
    g = golden["hash61_u32"]
    out = mb.hash61(dev(np.array(g["keys"], np.uint32)), g["coeffs"], key_bits=32)
    assert [int(v) for v in host_u64(out)] == g["out"]


@pytest.mark.parametrize("k", [4, 8])
def test_golden_hash61_full(cuda, mb, golden, k):
    g = golden["hash61_full"]
    out = mb.hash61(dev(np.array(g["keys"], np.uint64)), g[f"k{k}"]["coeffs"], key_bits=64)
    assert [int(v) for v in host_u64(out)] == g[f"k{k}"]["out"]


def test_golden_hash89(cuda, mb, golden):
    g = golden["hash89"]
    lo, hi = mb.hash89(dev(np.array(g["keys"], np.uint64)), [int(c) for c in g["coeffs"]])
    got = [int(l) | (int(h) << 64) for l, h in zip(host_u64(lo), host_u64(hi))]
    assert got == [int(v) for v in g["out"]]


@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 1023, 100003])
def test_hash61_sizes_and_tails(cuda, mb, orc, n):
    c = orc.coeffs(61, 4, 17)
    k32 = orc.gen_u32_keys(9, 0, n)
    k64 = orc.gen_u64_keys(9, 0, n)
    if n == 0:
        assert mb.hash61(dev(k32), c).numel() == 0
        return
    exp32 = orc.hash_batch(61, c, k32.astype(np.uint64), 32)[0]
    assert (host_u64(mb.hash61(dev(k32), c, key_bits=32)) == exp32).all()
    exp64 = orc.hash_full(61, c, k64)
    assert (host_u64(mb.hash61(dev(k64), c, key_bits=64)) == exp64).all()


def test_hash61_extreme_keys(cuda, mb, orc):
    # keys at the edges of every reduction step: 0, p-1, p, p+1, 2^61.., 2^64-1
    keys = np.array([0, 1, P61 - 1, P61, P61 + 1, 1 << 61, (1 << 62) - 1, (1 << 63), M64, M64 - 1,
                     (1 << 32) - 1, 1 << 32], np.uint64)
    for k in range(1, 17):
        for coeffs in (orc.coeffs(61, k, k), [P61 - 1] * k, [0] * k):
            got = host_u64(mb.hash61(dev(keys), coeffs, key_bits=64))
            for x, h in zip(keys, got):
                y = 0
                for a in reversed(coeffs):
                    y = (y * int(x) + a) % P61
                assert y == int(h), (k, int(x))
    k32 = np.array([0, 1, 0xFFFFFFFF, 0x80000000], np.uint32)
    c = [P61 - 1] * 4
    got = host_u64(mb.hash61(dev(k32), c, key_bits=32))
    exp = orc.hash_batch(61, c, k32.astype(np.uint64), 32)[0]
    assert (got == exp).all()


def test_hash61_k8_adapted_coefficients(cuda, mb, orc):
    """k = 8 with 64-bit keys runs the five-product adapted form (host/precond61.cpp,
    eval61_pre8): families with shift 0 and with a shift, both kernel forms (16-byte
    vectors, scalar for unaligned views), odd sizes, a leading coefficient of 0 (Horner),
    against the oracle's Horner with a full reduction per step."""
    rng = np.random.default_rng(8)
    edge = np.array([0, 1, P61 - 1, P61, P61 + 1, 1 << 61, (1 << 62) - 1, 1 << 63, M64, M64 - 1], np.uint64)
    keys = np.concatenate([edge, rng.integers(0, 1 << 63, 100_003, dtype=np.uint64) * 2 + 1,
                           rng.integers(0, P61, 50_000, dtype=np.uint64)])
    t = dev(keys)
    seen = {}
    seed = 0
    while len(seen) < 3 and seed < 400:  # shift 0, two different non-zero shifts
        seed += 1
        c = orc.coeffs(61, 8, 1000 + seed)
        s = mb.precondition61(c)["s"]
        if s in seen or (s == 0 and seed > 1 and 0 in seen):
            continue
        seen[s] = c
    assert 0 in seen and len(seen) == 3
    fams = list(seen.values()) + [[P61 - 1] * 8, [0] * 7 + [1], [5, 4, 3, 2, 1, 0, 7, 0]]
    for c in fams:
        exp = orc.hash_full(61, c, keys)
        assert (host_u64(mb.hash61(t, c, key_bits=64)) == exp).all()
        assert (host_u64(mb.hash61(t[1:], c, key_bits=64)) == exp[1:]).all()  # scalar kernel
        assert (host_u64(mb.hash61(t[:7], c, key_bits=64)) == exp[:7]).all()


def test_hash61_unaligned_views(cuda, mb, orc):
    c = orc.coeffs(61, 8, 3)
    k64 = orc.gen_u64_keys(4, 0, 4097)
    t = dev(k64)
    out = mb.hash61(t[1:], c, key_bits=64)  # keys 8-byte but not 16-byte aligned
    assert (host_u64(out) == orc.hash_full(61, c, k64[1:])).all()


def test_hash61_domain_all_or_nothing(cuda, mb):
    import torch

    keys = dev(np.array([1, 2, 1 << 40, 3], np.uint64))
    out = torch.full((4,), -1, dtype=torch.int64, device="cuda")
    with pytest.raises(mb.DomainError, match="key outside domain"):
        mb.hash61(keys, [1, 2, 3, 4], key_bits=32, out=out)
    assert (out.cpu() == -1).all()


@pytest.mark.parametrize("k", [2, 4, 8])
def test_hash89_random(cuda, mb, orc, k):
    c = orc.coeffs(89, k, 5 + k)
    keys = orc.gen_u64_keys(k, 0, 50001)
    keys[:4] = [0, 1, M64, M64 - 1]
    lo, hi = mb.hash89(dev(keys), c)
    el, eh, _ = orc.hash_batch(89, c, keys, 64)
    assert (host_u64(lo) == el).all() and (host_u64(hi) == eh).all()


# ---------------------------------------------------------------- division
def test_golden_divmod(cuda, mb, golden):
    g = golden["pm_divmod"]
    v = [int(x) for x in g["v"]]
    flat = np.array([w for x in v for w in (x & M64, x >> 64)], np.uint64)
    q, r = mb.pm_divmod(dev(flat), 64, 59)
    assert [int(x) for x in host_u64(q)] == g["q"]
    assert [int(x) for x in host_u64(r)] == g["r"]


def test_divmod_known_answers_and_domain(cuda, mb):
    def run(b, c, vals, m=0):
        flat = np.array([w for x in vals for w in (x & M64, x >> 64)], np.uint64)
        q, r = mb.pm_divmod(dev(flat), b, c, m)
        return [int(x) for x in host_u64(q)], [int(x) for x in host_u64(r)]

    assert run(4, 3, [27, 69], 2) == ([2, 5], [1, 4])  # test_field.cpp:136-146
    assert run(3, 1, [30, 48], 2) == ([4, 6], [2, 6])
    with pytest.raises(mb.DomainError, match="division domain"):
        run(4, 3, [27, 70], 2)


@pytest.mark.parametrize("b,c", [(64, 59), (64, 1), (63, 25), (61, 1), (40, 3), (33, 1 << 20)])
def test_divmod_random(cuda, mb, orc, b, c):
    m, mx, _ = orc.pm_setup(b, c)
    p = (1 << b) - c
    n = 20001
    v = orc.gen_pm_inputs(b * 1000 + c, 59, 0, n)
    vals = [int(v[2 * i]) | (int(v[2 * i + 1]) << 64) for i in range(n)]
    lim = min(mx, p * p - 1, (p << 64) - 1)  # keep q < 2^64 and inside the domain
    vals = [x % (lim + 1) for x in vals]
    vals[:6] = [0, 1, p - 1, p, p * p - 1 if p * p - 1 <= lim else lim, lim]
    flat = np.array([w for x in vals for w in (x & M64, x >> 64)], np.uint64)
    q, r = mb.pm_divmod(dev(flat), b, c)
    eq, er, rej = orc.pm_divmod_batch(b, c, flat)
    assert rej == 0
    assert (host_u64(q) == eq).all() and (host_u64(r) == er).all()
    assert all(int(host_u64(q)[i]) == vals[i] // p for i in range(64))


# ---------------------------------------------------------------- bucket maps
def test_golden_bucket_maps(cuda, mb, golden):
    for case in golden["bucket_maps"]:
        b, c, r = case["b"], int(case["c"]), int(case["r"])
        if case["kind"] == mb.MAP_EXACT_DIV:
            assert mb.exact_division_iterations(b, c, r) == case["iterations"]
        out = mb.bucket_map(case["kind"], dev(np.array(case["v"], np.uint64)), b, r, c)
        assert [int(x) for x in host_u64(out)] == case["out"]


def test_bucket_map_known_answers(cuda, mb):
    # test_bucketing.cpp:101-127
    m13 = mb.ExactDivisionMap(4, 3, 4)
    out = host_u64(m13(dev(np.arange(13, dtype=np.uint64)))).astype(np.int64)
    assert np.bincount(out, minlength=4).tolist() == [4, 3, 3, 3]
    ident = mb.ExactDivisionMap(4, 3, 13)
    assert host_u64(ident(dev(np.arange(13, dtype=np.uint64)))).tolist() == list(range(13))
    for r in (0, 14):
        with pytest.raises(mb.InvalidArgument, match=r"bucket count must be in \[1, p\]"):
            mb.ExactDivisionMap(4, 3, r)
    x = dev(np.arange(32, dtype=np.uint64))
    assert host_u64(mb.bucket_map(mb.MAP_POW2, x, 5, 32)).tolist() == list(range(32))
    assert host_u64(mb.bucket_map(mb.MAP_POW2, x, 5, 1)).tolist() == [0] * 32


@pytest.mark.parametrize("kind,b,c,r", [(0, 64, 0, 1000003), (0, 61, 0, 1 << 61), (0, 17, 0, 5),
                                         (1, 64, 0, (1 << 63) + 12345), (1, 40, 0, 77),
                                         (2, 64, 59, (1 << 64) - 59), (2, 64, 59, 1000),
                                         (2, 64, (1 << 62) + 1, 12345), (2, 33, 7, 1 << 32),
                                         (2, 61, 1, (1 << 61) - 1), (2, 48, (1 << 40) + 3, 1 << 47)])
def test_bucket_map_random(cuda, mb, orc, kind, b, c, r):
    dom = (1 << b) - (c if kind == 2 else kind)
    n = (1 << 20) + 3  # odd: exercises the vector body and the scalar tail
    v = orc.gen_u64_keys(kind * 1000 + b, 0, n)
    if dom < (1 << 64):
        v = v % np.uint64(dom)
    v[:3] = [0, 1, dom - 1]
    got = host_u64(mb.bucket_map(kind, dev(v), b, r, c))
    m, exp = orc.bucket_map(kind, b, r, v, c=c)
    assert (got == exp).all()
    # unaligned views take the scalar kernel
    got1 = host_u64(mb.bucket_map(kind, dev(v)[1:], b, r, c))
    assert (got1 == exp[1:]).all()


def test_bucket_map_domain(cuda, mb):
    import torch

    v = dev(np.array([0, 5, 12, 13, 40], np.uint64))
    with pytest.raises(mb.DomainError, match="outside the map's domain"):
        mb.bucket_map(mb.MAP_EXACT_DIV, v, 4, 4, 3)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mb.bucket_map(mb.MAP_EXACT_DIV, v, 4, 4, 3, out_of_domain=cnt)
    assert int(cnt.item()) == 2
    with pytest.raises(mb.DomainError):
        mb.bucket_map(mb.MAP_MERSENNE, dev(np.array([7], np.uint64)), 3, 3)
    assert mb.bucket_map(mb.MAP_POW2, dev(np.zeros(0, np.uint64)), 5, 3).numel() == 0
    with pytest.raises(mb.Unsupported):
        mb.bucket_map(mb.MAP_EXACT_DIV, v, 89, 4, 1)


# ---------------------------------------------------------------- sketches
def make_spec(mb, orc, rows, width, b, key_bits, splitter, seed):
    if splitter == mb.SPLIT_TWO_FOR_ONE:
        fams = [orc.coeffs(b, 4, s) for s in orc.row_seeds(seed, (rows + 1) // 2)]
    else:
        fams = [orc.coeffs(b, 4, s) for s in orc.row_seeds(seed, rows)]
    return mb.SketchSpec(rows, width, b, fams, key_bits, splitter), fams


def test_golden_c1_sketch(cuda, mb, orc, golden):
    import torch

    g = golden["c1_sketch"]
    spec, _ = make_spec(mb, orc, 1, 1024, 61, 32, 0, golden["seed"])
    keys = orc.gen_u32_keys(golden["key_seed"], 0, g["n"])
    cnt = torch.zeros(1024, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), cnt)
    assert [int(x) for x in cnt.cpu()] == g["counters"]
    m = mb.moments_to_python(mb.cs_moments(cnt, 1, 1024))
    assert m[0] == (int(g["f2"]), False)


def test_golden_c5_sketch(cuda, mb, orc, golden):
    import torch

    g = golden["c5_sketch"]
    spec, _ = make_spec(mb, orc, 5, 65536, 61, 32, 0, golden["seed"])
    zs = mb.ZipfStream(golden["seed"])
    k, w = zs.generate(0, g["n"])
    assert [int(x) for x in k[:64].cpu().numpy().view(np.uint32)] == g["keys_head"]
    assert [int(x) for x in w[:64].cpu()] == g["weights_head"]
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, k, cnt, w)
    c = cnt.cpu().numpy()
    nz = np.nonzero(c)[0]
    assert [int(x) for x in nz] == g["nonzero_index"]
    assert [int(x) for x in c[nz]] == g["nonzero_value"]
    m = mb.moments_to_python(mb.cs_moments(cnt, 5, 65536))
    assert [v for v, _ in m] == [int(x) for x in g["row_f2"]]
    assert mb.lower_median(m)[0] == int(g["median_f2"])


def test_golden_c4_sketch(cuda, mb, orc, golden):
    import torch

    g = golden["c4_sketch"]
    spec, _ = make_spec(mb, orc, 2, 65536, 89, 64, mb.SPLIT_TWO_FOR_ONE, golden["seed"])
    # config 4 uses PolyHashFamily(m89, 4, 2^64, S) directly as the single family
    spec = mb.SketchSpec(2, 65536, 89, [orc.coeffs(89, 4, golden["seed"])], 64, mb.SPLIT_TWO_FOR_ONE)
    keys = orc.gen_u64_keys(golden["key_seed"], 0, g["n"])
    cnt = torch.zeros(2 * 65536, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), cnt)
    c = cnt.cpu().numpy()
    nz = np.nonzero(c)[0]
    assert [int(x) for x in nz] == g["nonzero_index"]
    assert [int(x) for x in c[nz]] == g["nonzero_value"]


CASES = [
    # rows, width, b, key_bits, splitter, key dtype, weights
    (1, 1024, 61, 32, 0, np.uint32, None),          # config 1 (smem32 strategy)
    (1, 1024, 61, 32, 0, np.uint32, np.int32),      # smem64 strategy
    (3, 64, 61, 20, 0, np.uint64, np.int64),        # reference-domain u64 keys
    (5, 65536, 61, 32, 0, np.uint32, np.int32),     # config 5 geometry (global + aggregation)
    (5, 65536, 61, 32, 0, np.uint32, None),         # global without aggregation
    (2, 65536, 89, 64, 3, np.uint64, None),         # config 4
    (4, 4096, 89, 64, 0, np.uint64, np.int64),      # 89-bit pow2
    (3, 48, 61, 32, 1, np.uint32, np.int64),        # UniformArb
    (3, 48, 61, 32, 2, np.uint32, np.int64),        # MersenneArb
    (4, 256, 61, 32, 3, np.uint32, np.int32),       # two-for-one with b = 61
    (3, 16, 31, 20, 0, np.uint64, np.int64),        # generic b
    (3, 12, 31, 20, 2, np.uint64, np.int64),        # generic b, arbitrary width
]


@pytest.mark.parametrize("case", CASES, ids=[f"r{c[0]}w{c[1]}b{c[2]}s{c[4]}" for c in CASES])
def test_sketch_random_vs_oracle(cuda, mb, orc, case):
    import torch

    rows, width, b, kb, sp, kdt, wdt = case
    spec, fams = make_spec(mb, orc, rows, width, b, kb, sp, 0xABC + rows)
    n = 200003
    rng = np.random.default_rng(rows * 7 + width)
    keys = rng.integers(0, 2**kb if kb < 64 else 2**63, size=n, dtype=np.uint64)
    if kb == 64:
        keys = orc.gen_u64_keys(width, 0, n)
    keys[: n // 3] = keys[: n // 3] % 97  # heavy duplicates: exercises aggregation
    keys = keys.astype(kdt)
    w = None
    if wdt is not None:
        w = rng.integers(-1000, 1000, size=n).astype(wdt)
        w[:5] = np.iinfo(wdt).min if wdt == np.int64 else w[:5]
    cnt = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), cnt, None if w is None else dev(w))
    exp = orc.cs_process(rows, width, b, fams, kb, sp, keys, w)
    assert (cnt.cpu().numpy() == exp).all()
    m = mb.moments_to_python(mb.cs_moments(cnt, rows, width))
    for r in range(rows):
        assert m[r] == orc.row_moment(exp[r * width:(r + 1) * width], width)
    assert mb.lower_median(m) == orc.second_moment(exp, rows, width, True)


@pytest.mark.parametrize("width", [2, 4, 1024, 8192])
@pytest.mark.parametrize("weights", [None, "small", "extreme"])
@pytest.mark.parametrize("n,offset", [(0, 0), (1, 0), (3, 0), (5, 0), (4099, 0), (1000003, 0), (1000003, 1)])
def test_one_row_vector_kernel(cuda, mb, orc, width, weights, n, offset):
    """Config 1's shape (one row, Pow2, 32-bit keys, b = 61, k = 4) runs the 16-byte
    vector kernel when the buffers are aligned (offset 0) and the generic one when
    not; both equal the oracle for every tail length, width and weight range (the
    extreme weights drive the exact two-word shared counters across 2^32)."""
    import torch

    spec, fams = make_spec(mb, orc, 1, width, 61, 32, 0, 0xC1 + width)
    rng = np.random.default_rng(n + width)
    keys = rng.integers(0, 2**32, size=n + offset, dtype=np.uint64).astype(np.uint32)
    w = None
    if weights == "small":
        w = rng.integers(-100, 101, size=n + offset).astype(np.int32)
    elif weights == "extreme":
        w = rng.choice(np.array([np.iinfo(np.int32).max, np.iinfo(np.int32).min, 2**30], np.int32),
                       size=n + offset)
    cnt = torch.zeros(width, dtype=torch.int64, device="cuda")
    dk = dev(keys)[offset:]
    dw = None if w is None else dev(w)[offset:]
    mb.cs_update(spec, dk, cnt, dw)
    exp = orc.cs_process(1, width, 61, fams, 32, 0, keys[offset:], None if w is None else w[offset:])
    assert (cnt.cpu().numpy() == exp).all()


HOT_CASES = [
    # rows, width, b, key_bits, splitter, key kind, weights: batches >= 2^22 take the
    # heavy-hitter path (shared-memory accumulation of sampled hot keys)
    (5, 65536, 61, 32, 0, "zipf", np.int32),
    (5, 65536, 61, 32, 0, "zipf", None),
    (5, 65536, 61, 32, 0, "uniform32", np.int32),
    (2, 65536, 89, 64, 3, "zipf64", None),
    (3, 4096, 61, 64, 0, "zipf64", np.int32),
    (16, 8192, 61, 32, 2, "zipf", np.int32),
    (3, 65536, 61, 32, 3, "zipf", np.int32),        # two-for-one, odd rows (last family one sub-row)
    (3, 16384, 89, 64, 0, "zipf64", np.int32),      # 89-bit Pow2
    (2, 65536, 31, 20, 0, "zipf20", np.int32),      # generic b (runtime splitter)
]


STRATEGIES = {"direct": 0, "binned": 1, "rows": 2}


@pytest.mark.parametrize("strategy", ["direct", "binned", "rows"])
@pytest.mark.parametrize("case", HOT_CASES, ids=[f"r{c[0]}b{c[2]}{c[5]}" for c in HOT_CASES])
def test_hot_path_large_batches(cuda, mb, orc, case, strategy):
    """Every large-table strategy (misses -> L2 reductions, misses -> HBM bins summed
    in shared memory, misses -> miss buffer summed by per-row passes) gives the
    oracle's table bit for bit."""
    import torch

    rows, width, b, kb, sp, kind, wdt = case
    prev = mb.set_large_table_strategy(STRATEGIES[strategy])
    spec, fams = make_spec(mb, orc, rows, width, b, kb, sp, 0xB16 + rows)
    n = (1 << 22) + 12345
    zk, zw = orc.gen_zipf_items(7, 0, n)
    if kind == "uniform32":
        zk = orc.gen_u32_keys(7, 0, n)
    keys = zk if kind != "zipf64" else (zk.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    if kind == "zipf64" and kb < 64:
        keys = keys >> np.uint64(64 - kb)
    if kind == "zipf20":  # the generic-b domain: keys < 2^20
        keys = (zk.astype(np.uint64) & np.uint64((1 << 20) - 1)).astype(np.uint64)
    keys[:3] = [0, np.iinfo(keys.dtype).max if kb >= 32 else 1, 0]  # the empty-slot sentinel key
    w = None if wdt is None else zw.astype(wdt)
    if w is not None:
        w[:4] = [np.iinfo(np.int32).min, np.iinfo(np.int32).max, -1, 1]
    cnt = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    try:
        mb.cs_update(spec, dev(keys), cnt, None if w is None else dev(w))
    finally:
        mb.set_large_table_strategy(prev)
    st = mb.hot_stats(reset=True)
    exp = orc.cs_process(rows, width, b, fams, kb, sp, keys, w)
    assert (cnt.cpu().numpy() == exp).all()
    assert st["items"] == n
    if strategy == "binned" and rows * -(-width // 65536) <= 64:
        assert st["binned"] > 0  # the binned passes really ran
    if strategy == "rows" and sp in (0, 3) and b in (61, 89) and width <= 65536:
        assert st["binned"] > 0  # the row passes really ran (entries they summed)


@pytest.mark.parametrize("shape,strategy", [("overflow", "binned"), ("wide", "binned"), ("bigdelta", "binned"),
                                            ("overflow", "rows"), ("bigdelta", "rows")])
def test_binned_strategy_edge_paths(cuda, mb, orc, shape, strategy):
    """The binned strategy's fall-backs stay exact: more misses than the miss buffer
    holds (35% one key, 65% distinct keys: not raw mode, misses > n/2), rows wider
    than one 65536-cell bin (several bins per row, ballot grouping), and deltas
    outside the 16-bit entry field (direct reductions from the sink)."""
    import torch

    n = (1 << 22) + 333
    rng = np.random.default_rng({"overflow": 1, "wide": 2, "bigdelta": 3}[shape])
    rows, width = (3, 1 << 18) if shape == "wide" else (5, 65536)
    spec, fams = make_spec(mb, orc, rows, width, 61, 32, 0, 0x5EED)
    if shape == "overflow":
        keys = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        keys[rng.random(n) < 0.35] = 12345
    else:
        keys, _ = orc.gen_zipf_items(11, 0, n)
    w = rng.integers(-100, 101, size=n).astype(np.int32)
    if shape == "bigdelta":
        big = rng.random(n) < 0.1
        w[big] = rng.integers(-(2**31), 2**31, size=int(big.sum())).astype(np.int32)
    cnt = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    prev = mb.set_large_table_strategy(STRATEGIES[strategy])
    mb.hot_stats(reset=True)
    try:
        mb.cs_update(spec, dev(keys), cnt, dev(w))
    finally:
        mb.set_large_table_strategy(prev)
    st = mb.hot_stats(reset=True)
    exp = orc.cs_process(rows, width, 61, fams, 32, 0, keys, w)
    assert (cnt.cpu().numpy() == exp).all()
    if strategy == "binned":
        assert st["binned"] > 0 and st["direct"] > 0  # both the bins and a fall-back path ran
    else:
        assert st["binned"] > 0  # the row passes ran (and, for "overflow", the direct fall-back)
        assert shape != "overflow" or st["direct"] > 0


def test_large_table_strategy_rejects_unknown(cuda, mb):
    with pytest.raises(mb.InvalidArgument):
        mb.set_large_table_strategy(7)


@pytest.mark.parametrize("weight", [np.iinfo(np.int32).max, np.iinfo(np.int32).min])
def test_hot_path_accumulator_wraps(cuda, mb, orc, weight):
    """One key with extreme weights: every CTA's 32-bit hot accumulator wraps many
    times (sum = 2^22 x +-2^31); the wrap counters keep the table exact."""
    import torch

    n = (1 << 22) + 7
    keys = np.full(n, 7, np.uint32)
    keys[::1000] = np.arange(len(keys[::1000]), dtype=np.uint32) + 100  # some cold keys
    w = np.full(n, weight, np.int32)
    spec, fams = make_spec(mb, orc, 5, 65536, 61, 32, 0, 0xAA)
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, dev(keys), cnt, dev(w))
    st = mb.hot_stats(reset=True)
    assert st["items"] == n and st["misses"] < n // 100  # key 7 was accumulated in shared memory
    exp = orc.cs_process(5, 65536, 61, fams, 32, 0, keys, w)
    assert (cnt.cpu().numpy() == exp).all()


@pytest.mark.parametrize("wset", ["extreme", "cell_edges"])
def test_hot_path_cells_wrap_under_contention(cuda, mb, orc, wset):
    """Hot sums live in 16-bit shared cells, two per 32-bit word, with wraps
    recorded in HBM: a Zipf stream (thousands of hot keys, so both cells of
    most words are busy) whose weights make nearly every add leave the cell
    range -- the full i32 extremes, or values around the 2^15 / 2^16 cell
    edges -- still gives the oracle's table bit for bit."""
    import torch

    n = (1 << 22) + 77
    zk, _ = orc.gen_zipf_items(13, 0, n)
    rng = np.random.default_rng(17 if wset == "extreme" else 19)
    if wset == "extreme":
        vals = np.array([np.iinfo(np.int32).max, np.iinfo(np.int32).min, 1 << 30, -(1 << 30), 65537, -65537], np.int64)
    else:
        vals = np.array([32767, -32768, 32768, -32769, 65535, -65535, 65536, -65536, 1, -1], np.int64)
    w = rng.choice(vals, size=n).astype(np.int32)
    spec, fams = make_spec(mb, orc, 5, 65536, 61, 32, 0, 0xCE11)
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, dev(zk), cnt, dev(w))
    st = mb.hot_stats(reset=True)
    assert st["items"] == n and st["hot_keys"] > 1000
    exp = orc.cs_process(5, 65536, 61, fams, 32, 0, zk, w)
    assert (cnt.cpu().numpy() == exp).all()


@pytest.mark.parametrize("kb", [32, 64])
def test_hot_path_sentinel_keys_heavy(cuda, mb, orc, kb):
    """Empty hot-table slots hold foreign keys (keys whose two slot choices are
    elsewhere), so the lookup has no empty-slot test: the all-ones key (the
    empty marker, never selected as hot) and its neighbours -- the foreign-key
    candidates -- are frequent here, next to a few genuinely hot keys, with most
    slots empty.  The table equals the oracle's."""
    import torch

    n = (1 << 22) + 101
    rng = np.random.default_rng(kb)
    top = (1 << kb) - 1
    keys = rng.integers(0, 1 << min(kb, 62), size=n, dtype=np.uint64)
    u = rng.random(n)
    keys[u < 0.25] = top
    keys[(u >= 0.25) & (u < 0.40)] = top - 1
    keys[(u >= 0.40) & (u < 0.50)] = top - 2
    keys[(u >= 0.50) & (u < 0.60)] = 12345
    if kb == 32:
        keys = keys.astype(np.uint32)
    w = rng.integers(-100, 101, size=n).astype(np.int32)
    spec, fams = make_spec(mb, orc, 5, 65536, 61, kb, 0, 0xFEE)
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, dev(keys), cnt, dev(w))
    st = mb.hot_stats(reset=True)
    assert st["items"] == n and 0 < st["hot_keys"] < 100  # a nearly empty hot table
    exp = orc.cs_process(5, 65536, 61, fams, kb, 0, keys, w)
    assert (cnt.cpu().numpy() == exp).all()


@pytest.mark.parametrize("kb", [32, 64])
def test_hot_path_sample_fills_count_table(cuda, mb, orc, kb):
    """A batch whose head is skewed (the probe sees heavy hitters) and whose sample is
    otherwise all distinct keys: the sample's count table (one slot per sampled item)
    fills up, probing is bounded and keys without a slot go uncounted -- which only
    changes the hot set, never the table: it equals the oracle's."""
    import torch

    n = (1 << 23) + 13
    rng = np.random.default_rng(100 + kb)
    mult = np.uint64(0x9E3779B97F4A7C15 if kb == 64 else 2654435761)
    keys = (np.arange(n, dtype=np.uint64) * mult) % np.uint64(1 << min(kb, 62))  # distinct
    keys[:16384] = rng.choice(np.array([7, 11, 13, 17, 19, 23, 29, 31], np.uint64), 16384)
    keys[16384::97] = 7  # one genuinely hot key through the rest of the stream
    if kb == 32:
        keys = keys.astype(np.uint32)
    w = rng.integers(-100, 101, size=n).astype(np.int32)
    spec, fams = make_spec(mb, orc, 5, 65536, 61, kb, 0, 0xC0DE)
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, dev(keys), cnt, dev(w))
    st = mb.hot_stats(reset=True)
    assert st["items"] == n and st["hot_keys"] >= 1
    exp = orc.cs_process(5, 65536, 61, fams, kb, 0, keys, w)
    assert (cnt.cpu().numpy() == exp).all()


def test_sketch_empty_and_single(cuda, mb, orc):
    import torch

    spec, fams = make_spec(mb, orc, 3, 8, 61, 32, 0, 0xF00D)
    cnt = torch.zeros(24, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(np.zeros(0, np.uint32)), cnt)
    assert not cnt.any()
    mb.cs_update(spec, dev(np.array([123], np.uint32)), cnt, dev(np.array([-7], np.int64)))
    m = mb.moments_to_python(mb.cs_moments(cnt, 3, 8))
    assert m == [(49, False)] * 3  # test_sketch.cpp:106-117


def test_sketch_domain_all_or_nothing(cuda, mb, orc):
    import torch

    spec, _ = make_spec(mb, orc, 3, 64, 61, 20, 0, 1)
    cnt = torch.zeros(3 * 64, dtype=torch.int64, device="cuda")
    with pytest.raises(mb.DomainError, match="key outside domain"):
        mb.cs_update(spec, dev(np.array([1, 2, 1 << 20], np.uint64)), cnt)
    assert not cnt.any()


def test_estimator_saturation(cuda, mb, orc):
    import torch

    for vals in ([np.iinfo(np.int64).min] * 4, [np.iinfo(np.int64).min, 0],
                 [np.iinfo(np.int64).max] * 3, [-5, 7, 0, 1]):
        c = np.array(vals, np.int64)
        m = mb.moments_to_python(mb.cs_moments(torch.from_numpy(c).cuda(), 1, len(vals)))
        assert m[0] == orc.row_moment(c, len(vals))


def test_estimator_rows_over_many_ctas(cuda, mb, orc):
    """The estimator splits each row over CTAs of 4096 cells and adds the
    192-bit partials with carry-propagating atomics: rows whose partial sums
    carry across words between CTAs, just below and exactly at the 2^128
    saturation boundary, and a width that is not a multiple of 4096."""
    import torch

    width = 20000
    rng = np.random.default_rng(5)
    rows = [rng.integers(-(2**40), 2**40, size=width, dtype=np.int64),
            rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, size=width, dtype=np.int64),
            rng.integers(-(2**20), 2**20, size=width, dtype=np.int64),
            np.zeros(width, np.int64)]
    rows[2][[0, 8000, 16000]] = np.iinfo(np.int64).min  # 3 * 2^126 + small: below 2^128
    rows[3][[1, 5000, 9000, 19999]] = np.iinfo(np.int64).min  # exactly 2^128: saturated
    c = np.concatenate(rows)
    m = mb.moments_to_python(mb.cs_moments(torch.from_numpy(c).cuda(), len(rows), width))
    for r in range(len(rows)):
        assert m[r] == orc.row_moment(rows[r], width), r
    assert m[3][1] and not m[2][1]


def test_merge_equals_concatenation(cuda, mb, orc):
    import torch

    spec, fams = make_spec(mb, orc, 5, 65536, 61, 32, 0, 77)
    zs = mb.ZipfStream(3)
    k, w = zs.generate(0, 1 << 20)
    a = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    bb = torch.zeros_like(a)
    full = torch.zeros_like(a)
    mb.cs_update(spec, k[: 1 << 19], a, w[: 1 << 19])
    mb.cs_update(spec, k[1 << 19:], bb, w[1 << 19:])
    mb.cs_update(spec, k, full, w)
    mb.cs_merge(a, bb)
    assert torch.equal(a, full)


def test_point_query_golden(cuda, mb, orc, golden):
    import torch

    g = golden["point_query"]
    spec, _ = make_spec(mb, orc, g["rows"], g["width"], 61, 32, 0, golden["seed"])
    cnt = torch.zeros(g["rows"] * g["width"], dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(np.array(g["keys"], np.uint64)), cnt, dev(np.array(g["weights"], np.int64)))
    out = mb.cs_point_query(spec, cnt, dev(np.array(g["query"], np.uint64)))
    assert [int(x) for x in out.cpu()] == g["out"]


# ---------------------------------------------------------------- host object API
def test_count_sketch_object_matches_reference_semantics(cuda, mb, orc):
    # seeded ctor, process on host buffers, moments, point query, merge (sketch.cpp:68-193)
    sk = mb.CountSketch(5, 16, 61, 32, mb.SPLIT_MERSENNE_ARB, 0xBEEF)
    assert sk.point_query(np.array([42], np.uint64))[0] == 0
    sk.process_one(42, 1234)
    assert sk.point_query(np.array([42], np.uint64))[0] == 1234
    sk.process_one(42, -234)
    assert sk.point_query(np.array([42], np.uint64))[0] == 1000  # test_sketch.cpp:145-153

    a = mb.CountSketch(3, 32, 61, 32, mb.SPLIT_MERSENNE_ARB, 0x5EED)
    b = mb.CountSketch(3, 32, 61, 32, mb.SPLIT_MERSENNE_ARB, 0x5EED)
    both = mb.CountSketch(3, 32, 61, 32, mb.SPLIT_MERSENNE_ARB, 0x5EED)
    rng = np.random.default_rng(0xAB)
    k1 = rng.integers(0, 1 << 16, 300, dtype=np.uint64)
    d1 = rng.integers(-100, 100, 300).astype(np.int64)
    k2 = rng.integers(0, 1 << 16, 300, dtype=np.uint64)
    d2 = rng.integers(-100, 100, 300).astype(np.int64)
    a.process(k1, d1)
    b.process(k2, d2)
    both.process(np.concatenate([k1, k2]), np.concatenate([d1, d2]))
    a.merge(b)
    assert (a.counters() == both.counters()).all()  # test_sketch.cpp:239-261
    with pytest.raises(mb.InvalidArgument, match="geometry or seeds"):
        a.merge(mb.CountSketch(3, 32, 61, 32, mb.SPLIT_MERSENNE_ARB, 0x5EEE))
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(0x5EED, 3)]
    assert a.coefficients() == fams
    exp = orc.cs_process(3, 32, 61, fams, 32, 2, np.concatenate([k1, k2]), np.concatenate([d1, d2]))
    assert (a.counters() == exp).all()
    with pytest.raises(mb.DomainError, match="key outside domain"):
        a.process(np.array([1 << 33], np.uint64))
    assert (a.counters() == exp).all()


def test_mcsk1_serialization_matches_reference(cuda, mb, golden):
    """A GPU table serializes byte-identically to the reference (sketch.cpp:195-211),
    round-trips, and keeps hashing identically after deserialize (test_sketch.cpp:180-205)."""
    g = golden["mcsk1"]
    sk = mb.CountSketch(3, 16, 61, 32, mb.SPLIT_MERSENNE_ARB, 0xABCD)
    sk.process(np.array(g["keys"], np.uint64), np.array(g["weights"], np.int64))
    payload = sk.serialize()
    assert payload == bytes.fromhex(g["bytes"])
    assert len(payload) == 33 + 8 * 3 + 8 * 3 * 16 and payload[:5] == b"MCSK1"
    back = mb.CountSketch.deserialize(payload)
    assert back.serialize() == payload
    back.process_one(7, 3)
    sk.process_one(7, 3)
    assert back.serialize() == sk.serialize()
    for bad in (b"", b"XCSK1" + payload[5:], payload[:-1], payload + b"\0",
                payload[:25] + b"\x09" + payload[26:]):
        with pytest.raises(mb.InvalidArgument, match="malformed sketch payload"):
            mb.CountSketch.deserialize(bad)
    inj = mb.CountSketch.from_families(4, mb.SPLIT_POW2, 5, 4, [[1, 2, 3, 4]])
    with pytest.raises(mb.LogicError):
        inj.serialize()


def test_count_sketch_injected_families(cuda, mb):
    sk = mb.CountSketch.from_families(4, mb.SPLIT_POW2, 5, 4, [[1, 2, 3, 4]])
    with pytest.raises(mb.LogicError):
        sk.seeds()
    keys, deltas = np.array([1, 3, 7], np.uint64), np.array([2, -1, 3], np.int64)
    sk.process(keys, deltas)
    exp = orc_cs(mb, [[1, 2, 3, 4]], keys, deltas)
    assert (sk.counters() == exp).all() and exp.any()


def orc_cs(mb, fams, keys, deltas):
    from oracle_bind import oracle

    return oracle().cs_process(1, 4, 5, fams, 4, mb.SPLIT_POW2, keys, deltas)


# ---------------------------------------------------------------- multi-GPU merge
def test_nccl_allreduce_one_rank(cuda, mb, orc):
    """mb200_cs_allreduce over a one-rank communicator made by the product: the merge
    of one table is that table (N > 1 is covered by the gloo tests of bench's step
    logic; one box has one GPU).  Exercises the dlopen'd NCCL, the comm lifecycle
    and the uint64 in-place reduction on a table holding wrap-around values."""
    import torch

    comm = mb.NcclComm(1, mb.nccl_unique_id(), 0)
    assert comm.size() == 1 and mb.nccl_version() >= 21800
    vals = np.array([0, 1, -1, 2**63 - 1, -(2**63), 12345, -987654321] * 1000, np.int64)
    t = torch.from_numpy(vals.copy()).cuda()
    mb.cs_allreduce(t, comm)
    torch.cuda.synchronize()
    assert (t.cpu().numpy() == vals).all()
    # the object path: CountSketch.allreduce leaves the (one-rank) merged table in HBM
    sk = mb.CountSketch(5, 1 << 10, 61, 32, mb.SPLIT_POW2, 1)
    keys, w = orc.gen_zipf_items(1, 0, 50_000)
    sk.process(keys, w)
    before = sk.counters()
    sk.allreduce(comm)
    assert (sk.counters() == before).all()
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(1, 5)]
    assert (before == orc.cs_process(5, 1 << 10, 61, fams, 32, 0, keys, w)).all()
    comm.close()


# ---------------------------------------------------------------- generators
def test_generators_match_oracle(cuda, mb, orc):
    SK = 1 ^ mb.SALT_KEYS
    for start, n in [(0, 4097), (123456789, 1000)]:
        assert (mb.gen_u32_keys(SK, start, n).cpu().numpy().view(np.uint32)
                == orc.gen_u32_keys(SK, start, n)).all()
        assert (host_u64(mb.gen_u64_keys(SK, start, n)) == orc.gen_u64_keys(SK, start, n)).all()
        out, bad = mb.gen_below_p61(SK, start, n)
        assert int(bad.item()) == 0 and (host_u64(out) == orc.gen_below_p61(SK, start, n)).all()
        v, bad = mb.gen_pm_inputs(SK, 59, start, n)
        assert int(bad.item()) == 0
        assert (v.cpu().numpy().reshape(-1).view(np.uint64) == orc.gen_pm_inputs(SK, 59, start, n)).all()
    zs = mb.ZipfStream(1)
    cdf, c1 = orc.zipf_table()
    assert (zs.cdf_host == cdf).all() and zs.c1 == c1
    for start, n in [(0, 1 << 18), ((1 << 31) - 5000, 5000)]:
        k, w = zs.generate(start, n)
        ek, ew = orc.gen_zipf_items(1, start, n)
        assert (k.cpu().numpy().view(np.uint32) == ek).all()
        assert (w.cpu().numpy() == ew).all()


# ---------------------------------------------------------------- full BASELINE sizes
@pytest.mark.slow
def test_full_size_c2(cuda, mb, orc):
    import torch

    n = 1 << 28
    keys, bad = mb.gen_below_p61(1 ^ mb.SALT_KEYS, 0, n)
    assert int(bad.item()) == 0
    for k in (4, 8):
        c = orc.coeffs(61, k, 1)
        out = mb.hash61(keys, c, key_bits=64)
        assert bool((out >= 0).all()) and bool((out < P61).all())  # fully reduced
        # every one of the 2^28 hashes against the (OpenMP) oracle, in 2^26 chunks
        for s0 in range(0, n, 1 << 26):
            exp = orc.hash_full(61, c, host_u64(keys[s0:s0 + (1 << 26)]))
            assert (host_u64(out[s0:s0 + (1 << 26)]) == exp).all()
        del out
    del keys


@pytest.mark.slow
def test_full_size_c3(cuda, mb, orc):
    import torch

    n = 1 << 28
    v, bad = mb.gen_pm_inputs(1 ^ mb.SALT_KEYS, 59, 0, n)
    assert int(bad.item()) == 0
    q, r = mb.pm_divmod(v, 64, 59)
    # every one of the 2^28 quotients and remainders against the oracle, in 2^26 chunks
    for s0 in range(0, n, 1 << 26):
        flat = v[s0:s0 + (1 << 26)].cpu().numpy().reshape(-1).view(np.uint64)
        eq, er, _ = orc.pm_divmod_batch(64, 59, flat)
        assert (host_u64(q[s0:s0 + (1 << 26)]) == eq).all() and (host_u64(r[s0:s0 + (1 << 26)]) == er).all()
    # size-independent property on every unit: r < p (u64 compare via sign flip)
    p = (1 << 64) - 59
    rr = r ^ (-(1 << 63))
    assert bool((rr < (p - (1 << 64)) ^ (-(1 << 63))).all())


@pytest.mark.slow
def test_full_size_c1_and_c5(cuda, mb, orc):
    import os

    import torch

    # config 1 in full: 2^24 keys vs the oracle
    spec, fams = make_spec(mb, orc, 1, 1024, 61, 32, 0, 1)
    keys = mb.gen_u32_keys(1 ^ mb.SALT_KEYS, 0, 1 << 24)
    cnt = torch.zeros(1024, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, keys, cnt)
    exp = orc.cs_process(1, 1024, 61, fams, 32, 0, keys.cpu().numpy().view(np.uint32))
    assert (cnt.cpu().numpy() == exp).all()
    # config 5: the full 2^31-item stream in ONE call (the bench's call) when the host has
    # the cores for the oracle (~20 s on 16), else a 2^27 prefix; equality of the whole
    # table, row moments and the median estimate
    n = 1 << 31 if (os.cpu_count() or 1) >= 16 else 1 << 27
    spec, fams = make_spec(mb, orc, 5, 65536, 61, 32, 0, 1)
    zs = mb.ZipfStream(1)
    keys, wts = zs.generate(0, n)
    cnt = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, keys, cnt, wts)
    exp = np.zeros(5 * 65536, np.int64)
    chunk = 1 << 26
    for s in range(0, n, chunk):
        orc.cs_process(5, 65536, 61, fams, 32, 0, keys[s:s + chunk].cpu().numpy().view(np.uint32),
                       wts[s:s + chunk].cpu().numpy(), counters=exp)
    del keys, wts
    assert (cnt.cpu().numpy() == exp).all()
    m = mb.moments_to_python(mb.cs_moments(cnt, 5, 65536))
    assert mb.lower_median(m) == orc.second_moment(exp, 5, 65536, True)


@pytest.mark.slow
def test_full_size_c4(cuda, mb, orc):
    """Config 4 in full: 2^26 u64 keys through one 89-bit family split two-for-one into
    two rows of 2^16 counters, one call, against the oracle; both row moments."""
    import torch

    n = 1 << 26
    keys = mb.gen_u64_keys(1 ^ mb.SALT_KEYS, 0, n)
    c = orc.coeffs(89, 4, 1)
    spec = mb.SketchSpec(2, 1 << 16, 89, [c], 64, mb.SPLIT_TWO_FOR_ONE)
    cnt = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, keys, cnt)
    exp = orc.cs_process(2, 1 << 16, 89, [c], 64, 3, host_u64(keys))
    assert (cnt.cpu().numpy() == exp).all()
    m = mb.moments_to_python(mb.cs_moments(cnt, 2, 1 << 16))
    for r in range(2):
        assert m[r] == orc.row_moment(exp[r << 16:(r + 1) << 16], 1 << 16)


# ---------------------------------------------------------------- moment enumeration
ENUM_STREAM = [(1, 2), (3, -1), (7, 3)]


def test_enum_moment_sums_known_answers(cuda, mb):
    # test_verify.cpp:205-265 frozen values (see tests/test_oracle.py for the derivation)
    from fractions import Fraction

    F = 31 ** 4
    s = mb.enum_moment_sums(5, 4, mb.SPLIT_POW2, ENUM_STREAM, key_domain=16)
    assert (s["sum_x"], s["sum_x_sq"], s["families"]) == (12931216, 226416064, F)
    assert mb.enum_moment_sums(5, 4, mb.SPLIT_MERSENNE_ARB, ENUM_STREAM, 16)["sum_x"] == 12931216
    assert mb.enum_moment_sums(5, 4, mb.SPLIT_POW2, [(5, 9)], 16)["sum_x_sq"] == 6561 * F
    rep = mb.enum_sketch_moments(5, 4, mb.SPLIT_POW2, ENUM_STREAM, 16)
    c = {x["name"]: x for x in rep["checks"]}
    assert all(x["pass"] for x in rep["checks"])
    assert c["mean matches exact formula"]["value"] == Fraction(13456, 961)
    assert c["variance below bound"]["value"] == Fraction(45352128, 923521)
    assert c["variance below bound"]["bound"] == Fraction(2 * 14 * 14, 4)
    mrep = mb.enum_sketch_moments(5, 3, mb.SPLIT_MERSENNE_ARB, ENUM_STREAM, 16)
    mv = [x for x in mrep["checks"] if x["name"] == "variance below bound"][0]
    assert mv["value"] == Fraction(60396800, 923521)
    assert mv["bound"] == Fraction(2 * 14 * 14 * (1024 + 9), 3 * 1024)
    assert all(x["pass"] for x in mrep["checks"])


@pytest.mark.parametrize("b,r,splitter,n", [(5, 4, 0, 3), (5, 3, 1, 5), (5, 16, 2, 9), (5, 1, 0, 17),
                                             (4, 8, 0, 15), (6, 5, 2, 31), (6, 32, 0, 40), (3, 2, 1, 7)])
def test_enum_moment_sums_vs_oracle(cuda, mb, orc, b, r, splitter, n):
    p = (1 << b) - 1
    rng = np.random.default_rng(b * 100 + n)
    keys = rng.choice(p, size=n, replace=False)
    budget = 1024 // n
    deltas = rng.integers(-min(budget, 50), min(budget, 50) + 1, size=n)
    deltas[0] = 0 if n > 3 else deltas[0]  # zero weights are skipped by the kernel
    stream = [(int(k), int(d)) for k, d in zip(keys, deltas)]
    got = mb.enum_moment_sums(b, r, splitter, stream)
    exp = orc.enum_moment_sums(b, r, splitter, stream)
    assert (got["sum_x"], got["sum_x_sq"]) == exp
    assert got["families"] == p ** 4


def test_enum_moment_mean_exact_b7(cuda, mb):
    # p = 127 (2.6e8 families): the exact-mean identity holds on the GPU sums
    from fractions import Fraction

    stream = [(3, 5), (10, -7), (126, 2), (64, 1)]
    for splitter, r in ((mb.SPLIT_POW2, 16), (mb.SPLIT_UNIFORM_ARB, 10), (mb.SPLIT_MERSENNE_ARB, 6)):
        rep = mb.enum_sketch_moments(7, r, splitter, stream)
        assert rep["sums"]["families"] == 127 ** 4
        assert all(x["pass"] for x in rep["checks"]), rep["checks"]
        f1, f2 = 1, 25 + 49 + 4 + 1
        assert Fraction(rep["sums"]["sum_x"], 127 ** 4) == Fraction(f2 * 127 ** 2 + f1 * f1 - f2, 127 ** 2)


# ------------------------------------------------- host API delta transport
@pytest.mark.parametrize("wdtype", [np.int32, np.int64])
@pytest.mark.parametrize("mag,nbytes", [(100, 1), (128, 2), (30000, 2), (1 << 20, None)])
def test_host_process_narrowed_deltas(cuda, mb, orc, wdtype, mag, nbytes):
    """mb200_sketch_process ships each chunk's deltas in the narrowest of i8 / i16
    that holds them (else as given) and widens them on the device: counters equal
    the oracle's for deltas at and just past each width's edge, and the reported
    H2D bytes show which width crossed."""
    mb.set_host_threads(8)
    rng = np.random.default_rng(mag)
    n = 5000
    keys = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(-mag, mag + 1, n).astype(wdtype)
    d[:4] = [mag, -mag, mag - 1, -mag - 1 if mag < 1 << 20 else -mag]
    sk = mb.CountSketch(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 0x5EED)
    b0 = sk.h2d_bytes()
    sk.process(keys, d)
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(0x5EED, 5)]
    exp = orc.cs_process(5, 1 << 16, 61, fams, 32, mb.SPLIT_POW2, keys.astype(np.uint64), d.astype(np.int64))
    assert (sk.counters() == exp).all()
    wb = nbytes if nbytes else np.dtype(wdtype).itemsize
    if mag == 128:  # -129 is in the stream: i8 fails, i16 holds it
        wb = 2
    assert sk.h2d_bytes() - b0 == n * 4 + n * wb


def test_host_process_mixed_width_chunks(cuda, mb):
    """Three 2^24-item chunks in one call: i8-sized deltas, a chunk with one i32
    extreme (ships at full width), then small deltas again; equal to the device
    entry on the same items (itself pinned to the oracle above)."""
    import torch

    mb.set_host_threads(8)
    C = 1 << 24
    n = 2 * C + 1000
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(-100, 101, n).astype(np.int32)
    d[C + 12345] = np.iinfo(np.int32).max
    d[C + 99] = np.iinfo(np.int32).min
    sk = mb.CountSketch(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 3)
    sk.process(keys, d)
    assert sk.h2d_bytes() == n * 4 + C * 1 + (C + 1000) * 4
    spec = mb.SketchSpec.seeded(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 3)
    table = torch.zeros(5 << 16, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), table, torch.from_numpy(d).cuda())
    assert (sk.counters() == table.cpu().numpy()).all()
    # a second call starts narrow again
    sk.process(keys[:1000], d[:1000])
    assert sk.h2d_bytes() == n * 4 + C * 1 + (C + 1000) * 4 + 1000 * 5


@pytest.mark.parametrize("key_bits", [32, 64])
def test_host_process_u64_keys(cuda, mb, orc, key_bits):
    """u64 keys of a 32-bit domain cross PCIe as u32 after the (parallel)
    all-or-nothing domain check; a 64-bit domain ships them whole.  Counters
    equal the oracle's either way."""
    mb.set_host_threads(8)
    rng = np.random.default_rng(key_bits)
    n = (1 << 17) + 3  # the parallel check and packing paths
    keys = rng.integers(0, 1 << key_bits, n, dtype=np.uint64)
    keys[:3] = [0, (1 << key_bits) - 1, 1 << (key_bits - 1)]
    d = rng.integers(-100, 101, n).astype(np.int64)
    b = 61 if key_bits == 32 else 89
    sk = mb.CountSketch(2, 1 << 16, b, key_bits, mb.SPLIT_POW2, 11)
    sk.process(keys, d)
    assert sk.h2d_bytes() == n * (4 if key_bits == 32 else 8) + n * 1
    fams = [orc.coeffs(b, 4, s) for s in orc.row_seeds(11, 2)]
    exp = orc.cs_process(2, 1 << 16, b, fams, key_bits, mb.SPLIT_POW2, keys, d)
    assert (sk.counters() == exp).all()
    if key_bits == 32:
        bad = keys.copy()
        bad[n - 1] = 1 << 32  # last item out of domain: nothing may be applied
        with pytest.raises(mb.DomainError, match="key outside domain"):
            sk.process(bad, d)
        assert (sk.counters() == exp).all()


def test_host_process_unnarrowed_with_few_threads(cuda, mb, orc):
    """Below 6 host threads the inputs ship as given (packing would not outrun
    PCIe); the counters are the same."""
    rng = np.random.default_rng(5)
    n = (1 << 17) + 1
    keys = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    d = rng.integers(-100, 101, n).astype(np.int64)
    try:
        mb.set_host_threads(2)
        assert mb.host_threads() == 2
        sk = mb.CountSketch(2, 1 << 16, 61, 32, mb.SPLIT_POW2, 9)
        sk.process(keys, d)
        assert sk.h2d_bytes() == n * 16
    finally:
        mb.set_host_threads(0)
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(9, 2)]
    exp = orc.cs_process(2, 1 << 16, 61, fams, 32, mb.SPLIT_POW2, keys, d)
    assert (sk.counters() == exp).all()
    assert mb.host_threads() >= 1


@pytest.mark.parametrize("c0", [0x0123456789ABCDE, (1 << 61) - 2, 12345])
def test_private_byte_tables_wrap_exactly(cuda, mb, orc, c0):
    """Streams without heavy hitters, unit deltas and a table that fits shared
    memory as bytes take the private byte tables (8-bit cells, four per word).
    A constant polynomial sends all 2^23 distinct keys to one cell per row, so
    every CTA's cell wraps hundreds of times (carry or borrow, any byte of the
    word): the table still equals the oracle's, and no item went to L2
    directly."""
    import torch

    n = 1 << 23
    keys = (np.arange(n, dtype=np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)  # distinct
    fam = [[c0, 0, 0, 0]]
    spec = mb.SketchSpec(2, 1 << 16, 61, fam, 32, mb.SPLIT_TWO_FOR_ONE)
    table = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, dev(keys), table)
    hs = mb.hot_stats(reset=True)
    exp = orc.cs_process(2, 1 << 16, 61, fam, 32, mb.SPLIT_TWO_FOR_ONE, keys)
    got = table.cpu().numpy()
    assert (got == exp).all()
    assert np.count_nonzero(got) == 2 and abs(got).sum() == 2 * n
    assert hs["direct"] == 0 and hs["bin_merges"] > 0


# --- config 4's specialised kernel (cs_private89_kernel + private_fold_kernel) ---


def _c4_run(mb, orc, fam, keys):
    import torch

    spec = mb.SketchSpec(2, 1 << 16, 89, [fam], 64, mb.SPLIT_TWO_FOR_ONE)
    table = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, keys if not isinstance(keys, np.ndarray) else dev(keys), table)
    hs = mb.hot_stats(reset=True)
    kh = keys if isinstance(keys, np.ndarray) else host_u64(keys)
    exp = orc.cs_process(2, 1 << 16, 89, [fam], 64, mb.SPLIT_TWO_FOR_ONE, kh)
    return table.cpu().numpy(), exp, hs


@pytest.mark.parametrize("c0", [0x0123456789ABCDEF01234 & P89, P89 - 1, 12345, (1 << 87) | 0xFF])
def test_c4_kernel_byte_cells_wrap_exactly(cuda, mb, orc, c0):
    """A constant 89-bit polynomial sends 2^23 distinct keys to one cell per row
    (both signs, every byte position of the word): each CTA's byte cell wraps
    hundreds of times; the table equals the oracle's and nothing went to L2
    directly."""
    n = 1 << 23
    keys = (np.arange(n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    got, exp, hs = _c4_run(mb, orc, [c0, 0, 0, 0], keys)
    assert (got == exp).all()
    assert np.count_nonzero(got) == 2 and abs(got).sum() == 2 * n
    assert hs["direct"] == 0 and hs["items"] == n


def test_c4_kernel_hash_equal_to_p(cuda, mb, orc):
    """h(x) = x - 12345 mod p: for x = 12345 the last fold leaves y = p exactly
    (h = 0), the one value the kernel's shortcut reduction patches."""
    rng = np.random.default_rng(3)
    n = (1 << 21) + 1  # odd: the last key takes the odd-key path
    keys = rng.integers(0, 1 << 64, n, dtype=np.uint64)
    keys[[0, 1000, n // 2, n - 1]] = 12345
    keys[[5, 6]] = [12344, 12346]
    got, exp, _ = _c4_run(mb, orc, [P89 - 12345, 1, 0, 0], keys)
    assert (got == exp).all()


def test_c4_kernel_unaligned_and_random(cuda, mb, orc):
    """Random 89-bit families on random keys: the specialised kernel (16-byte
    aligned keys) and, for a view 8 bytes off, the generic private kernel."""
    import torch

    rng = np.random.default_rng(9)
    n = (1 << 21) + 7
    keys = rng.integers(0, 1 << 64, n + 1, dtype=np.uint64)
    fam = orc.coeffs(89, 4, 77)
    d = torch.from_numpy(keys.view(np.int64)).cuda()
    got, exp, _ = _c4_run(mb, orc, fam, d[:n])
    assert (got == exp).all()
    got, exp, _ = _c4_run(mb, orc, fam, d[1:])
    assert (got == exp).all()


# --- 62 <= b <= 127: the generic four-limb path (polyhash.cpp:78-88) ---

WIDE_BS = [62, 63, 64, 65, 89, 96, 100, 107, 127]


@pytest.mark.parametrize("b", WIDE_BS)
@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_hash_wide_random(cuda, mb, orc, b, k):
    """mb200_hash_wide (any 62 <= b <= 127, including composite exponents) against
    the oracle's generic Horner, which is pinned to the reference at b <= 127."""
    rng = np.random.default_rng(b * 31 + k)
    kb = min(b - 1, 64)
    n = 40000
    keys = rng.integers(0, 1 << 64, n, dtype=np.uint64)
    if kb < 64:
        keys &= np.uint64((1 << kb) - 1)
    keys[:3] = [0, (1 << kb) - 1, 1]
    c = orc.coeffs(b, k, 1000 + b + k)
    lo, hi = mb.hash_wide(dev(keys), b, c, key_bits=kb)
    el, eh, _ = orc.hash_batch(b, c, keys, kb)
    assert (host_u64(lo) == el).all() and (host_u64(hi) == eh).all()


def test_hash_wide_extreme_coefficients(cuda, mb, orc):
    """Coefficients at p - 1 and 0, keys at the domain edge: every partial fold and the
    finish's y >= p branch (h = y - p) get exercised."""
    for b in (64, 107, 127):
        p = (1 << b) - 1
        kb = min(b - 1, 64)
        keys = np.array([0, 1, 2, (1 << kb) - 1, (1 << kb) - 2, 12345], np.uint64)
        for c in ([p - 1] * 4, [0, 0, 0, p - 1], [p - 1, 0, 0, 1], [1, p - 1, 1, p - 1]):
            lo, hi = mb.hash_wide(dev(keys), b, c, key_bits=kb)
            el, eh, _ = orc.hash_batch(b, c, keys, kb)
            assert (host_u64(lo) == el).all() and (host_u64(hi) == eh).all(), (b, c)


WIDE_SKETCH = [
    # rows, width, b, splitter, weights
    (3, 1024, 107, 0, np.int32),
    (4, 1000, 107, 1, np.int64),
    (2, 777, 127, 2, np.int32),
    (5, 4096, 127, 3, None),
    (2, 65536, 64, 0, np.int32),
    (3, 3000, 89, 1, np.int32),      # b = 89 with an arbitrary-width splitter
    (2, 1 << 20, 89, 2, None),       # ... and a table larger than shared memory (L2 path)
    (6, 8192, 62, 3, np.int64),
]


@pytest.mark.parametrize("case", WIDE_SKETCH, ids=[f"b{c[2]}s{c[3]}w{c[1]}" for c in WIDE_SKETCH])
def test_sketch_wide_moduli(cuda, mb, orc, case):
    """Count Sketch updates and point queries for 62 <= b <= 127 (and b = 89 with the
    arbitrary-width splitters) equal the oracle's per-item process, every splitter."""
    import torch

    rows, width, b, sp, wdt = case
    kb = min(b - 1, 64)
    spec, fams = make_spec(mb, orc, rows, width, b, kb, sp, 0x51DE + b)
    rng = np.random.default_rng(b + sp)
    n = 300_000
    keys = rng.integers(0, 1 << 64, n, dtype=np.uint64)
    if kb < 64:
        keys &= np.uint64((1 << kb) - 1)
    keys[: n // 3] = keys[n // 3: 2 * (n // 3)] % np.uint64(777)  # repeats
    w = None if wdt is None else rng.integers(-(2**31), 2**31, n).astype(wdt)
    cnt = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), cnt, None if w is None else dev(w))
    exp = orc.cs_process(rows, width, b, fams, kb, sp, keys, w)
    assert (cnt.cpu().numpy() == exp).all()
    q = keys[:2000]
    got = mb.cs_point_query(spec, cnt, dev(q)).cpu().numpy()
    want = orc.point_query(rows, width, b, fams, kb, sp, exp, q)
    assert (got == want).all()
