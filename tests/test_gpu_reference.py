"""GPU kernels pinned to the REFERENCE ITSELF (not only to the restated oracle).

- Large-batch kernels against reference-executed digests of >= 2^22-unit slices
  (tests/golden/make_golden.py large_prefixes): the heavy-hitter scatter
  (cs_hot_kernel, config 5 stream head and a shard window), the private
  byte-table scatter (cs_private_kernel, config 4), config 1 at full size, and
  2^22-unit slices of configs 2 and 3.
- Drop-in round trip with the compiled reference (oracle/_ref, unmodified
  sources): a sketch the reference built and serialized is loaded by the GPU
  library, continued on the GPU, serialized, and read back by the reference's
  CountSketch::deserialize -- equal to the reference's serial pass.
- The reference API names this round added to the boundary: mersenne_divmod,
  pseudo_mersenne_div / pseudo_mersenne_mod, the batched splitters.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dev(a):
    import torch

    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).cuda()


def host_u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name", ["c5_head", "c5_window"])
def test_hot_kernel_matches_reference_digest(cuda, mb, golden, name):
    torch = cuda
    g = golden["large"][name]
    keys, w = mb.ZipfStream(golden["seed"]).generate(g["start"], g["n"])
    spec = mb.SketchSpec.seeded(5, 65536, 61, 32, mb.SPLIT_POW2, golden["seed"])
    table = torch.zeros(5 * 65536, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, keys, table, w)
    st = mb.hot_stats(reset=True)
    assert st["items"] == g["n"] and st["hot_keys"] > 0, st  # the heavy-hitter path ran
    assert digest(table.cpu().numpy()) == g["sha256"]
    mom = mb.moments_to_python(mb.cs_moments(table, 5, 65536))
    assert [str(v) for v, _ in mom] == g["row_f2"]
    assert str(mb.lower_median(mom)[0]) == g["median_f2"]


def test_private_kernel_matches_reference_digest(cuda, mb, golden):
    torch = cuda
    g = golden["large"]["c4_head"]
    keys = mb.gen_u64_keys(golden["key_seed"], 0, g["n"])
    spec = mb.SketchSpec(2, 1 << 16, 89, [mb.draw_coeffs(89, 4, golden["seed"])], 64, mb.SPLIT_TWO_FOR_ONE)
    table = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
    mb.hot_stats(reset=True)
    mb.cs_update(spec, keys, table)
    st = mb.hot_stats(reset=True)
    assert st["items"] == g["n"] and st["hot_keys"] == 0 and st["misses"] == 0, st  # private byte tables
    assert digest(table.cpu().numpy()) == g["sha256"]
    mom = mb.moments_to_python(mb.cs_moments(table, 2, 1 << 16))
    assert [str(v) for v, _ in mom] == g["row_f2"]


def test_config1_full_matches_reference_digest(cuda, mb, golden):
    torch = cuda
    g = golden["large"]["c1_full"]
    keys = mb.gen_u32_keys(golden["key_seed"], 0, g["n"])
    table = torch.zeros(1024, dtype=torch.int64, device="cuda")
    mb.cs_update(mb.SketchSpec.seeded(1, 1024, 61, 32, mb.SPLIT_POW2, golden["seed"]), keys, table)
    assert digest(table.cpu().numpy()) == g["sha256"]
    assert str(mb.moments_to_python(mb.cs_moments(table, 1, 1024))[0][0]) == g["f2"]


def test_config2_config3_heads_match_reference_digest(cuda, mb, golden):
    L, S, SK = golden["large"], golden["seed"], golden["key_seed"]
    keys, bad = mb.gen_below_p61(SK, 0, L["c2_k4_head"]["n"])
    assert int(bad.item()) == 0
    for k in (4, 8):
        assert digest(host_u64(mb.hash61(keys, mb.draw_coeffs(61, k, S), key_bits=64))) == L[f"c2_k{k}_head"]["sha256"]
    v, bad = mb.gen_pm_inputs(SK, 59, 0, L["c3_head"]["n"])
    q, r = mb.pm_divmod(v, 64, 59)
    assert digest(host_u64(q)) == L["c3_head"]["q_sha256"] and digest(host_u64(r)) == L["c3_head"]["r_sha256"]


@pytest.mark.parametrize("splitter,width", [(0, 65536), (1, 1000), (2, 77777)])
def test_reference_sketch_round_trips_through_the_gpu(cuda, mb, ref, orc, splitter, width):
    """MCSK1 is the wire format either side of the path: the
    reference's own CountSketch -> serialize -> mb200_sketch_deserialize -> GPU
    process (>= 2^22 items: the large-table kernels) -> mb200_sketch_serialize ->
    the reference's CountSketch::deserialize.  Bytes and median F2 equal the
    reference's single serial pass over the whole stream."""
    n1, n2 = 10_000, (1 << 22) + 333
    zk, zw = orc.gen_zipf_items(1, 0, n1 + n2)
    head = ref.serialize(5, width, 61, 32, splitter, 0xC0FFEE, zk[:n1], zw[:n1].astype(np.int64))
    gpu = mb.CountSketch.deserialize(head)
    gpu.process(zk[n1:], zw[n1:])            # int32 deltas, host buffers
    payload = gpu.serialize()
    back, f2_ref = ref.resume(payload)        # the reference reads the GPU's bytes
    assert back == payload
    whole = ref.serialize(5, width, 61, 32, splitter, 0xC0FFEE, zk, zw.astype(np.int64))
    assert payload == whole
    assert gpu.second_moment(True)[0] == f2_ref
    # and the reference can keep going from the GPU's state
    more_k, more_w = orc.gen_zipf_items(1, n1 + n2, 5000)
    cont, _ = ref.resume(payload, more_k, more_w.astype(np.int64))
    gpu.process(more_k, more_w)
    assert gpu.serialize() == cont


def test_mersenne_divmod_batch(cuda, mb, orc, ref):
    """mersenne_divmod (Alg 3, field.cpp:208-222) as a device batch: KATs of
    test_field.cpp:104-126, random v < 2^(2b) against the reference, and the
    all-or-nothing domain error."""
    torch = cuda
    v = dev(np.array([30, 0, 63, 0, 0, 0], np.uint64))
    q, r = mb.mersenne_divmod(v, 3)
    assert list(host_u64(q)) == [4, 9, 0] and list(host_u64(r)) == [2, 0, 0]
    rng = np.random.default_rng(3)
    for b in (2, 5, 13, 31, 32, 33, 61, 63):
        n = 3001
        lo = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
        hi = rng.integers(0, 2**63, n, dtype=np.uint64)
        vals = [((int(h) << 64) | int(lo_)) % (1 << (2 * b)) for lo_, h in zip(lo, hi)]
        vals[:3] = [0, (1 << (2 * b)) - 1, (1 << b) - 1]
        arr = np.array([[x & (2**64 - 1), x >> 64] for x in vals], np.uint64)
        q, r = mb.mersenne_divmod(dev(arr), b)
        p = (1 << b) - 1
        exp = [ref.mersenne_divmod(b, x) for x in vals[:200]]
        assert [(int(a), int(c)) for a, c in zip(host_u64(q)[:200], host_u64(r)[:200])] == exp
        assert [int(a) for a in host_u64(q)] == [x // p for x in vals]  # Alg 3 is exact on [0, 2^(2b))
        assert [int(c) for c in host_u64(r)] == [x % p for x in vals]
    out = torch.full((2,), 7, dtype=torch.int64, device="cuda")
    with pytest.raises(mb.DomainError, match=r"input exceeds 2\^\(2b\)"):
        mb.mersenne_divmod(dev(np.array([1, 0, 64, 0], np.uint64)), 3, q=out[:1].clone(), r=out[1:].clone())
    with pytest.raises(mb.Unsupported):
        mb.mersenne_divmod(dev(np.array([1, 0], np.uint64)), 89)


def test_pseudo_mersenne_div_and_mod_separately(cuda, mb, orc):
    """pseudo_mersenne_div / pseudo_mersenne_mod as separate batches (field.cpp:260-273):
    KATs of test_field.cpp:136-158 and random inputs against the oracle's pair."""
    v = dev(np.array([27, 0, 69, 0, 0, 0], np.uint64))
    q = mb.pm_div(v, 4, 3, 2)  # PseudoMersenneModulus(4, 3, 2): max_input 69
    assert list(host_u64(q)) == [2, 5, 0]
    assert list(host_u64(mb.pm_mod(v, q, 4, 3))) == [1, 4, 0]
    with pytest.raises(mb.DomainError, match="input exceeds division domain for m iterations"):
        mb.pm_div(dev(np.array([70, 0], np.uint64)), 4, 3, 2)
    z = dev(np.array([2, 6], np.uint64))
    assert list(host_u64(mb.pm_mod(dev(np.array([27, 0, 48, 0], np.uint64)), z, 4, 3)))[0] == 1
    assert list(host_u64(mb.pm_mod(dev(np.array([48, 0], np.uint64)), dev(np.array([6], np.uint64)), 3, 1))) == [6]
    SK = 1 ^ mb.SALT_KEYS
    vin, _ = mb.gen_pm_inputs(SK, 59, 0, 100_001)
    q = mb.pm_div(vin, 64, 59)
    r = mb.pm_mod(vin, q, 64, 59)
    eq, er, _ = orc.pm_divmod_batch(64, 59, vin.cpu().numpy().reshape(-1).view(np.uint64))
    assert (host_u64(q) == eq).all() and (host_u64(r) == er).all()


@pytest.mark.parametrize("splitter", [0, 1, 2])
def test_split_batch_matches_reference(cuda, mb, ref, splitter):
    """split_pow2 / split_arb_uniform / split_arb_mersenne over device batches against the
    reference's own functions, including the KATs of test_sketch.cpp:14-52."""
    kats = {0: [((0b110, 3, 2), (2, -1)), ((0, 3, 2), (0, 1)), ((0b011, 3, 2), (3, 1))],
            1: [((0b1011, 4, 3), (1, 1)), ((0, 4, 3), (0, -1))],
            2: [((3, 3, 3), (0, 1)), ((6, 3, 3), (2, 1))]}
    for (h, b, lr), exp in kats[splitter]:
        i, s = mb.split_batch(splitter, dev(np.array([h], np.uint64)), b, lr)
        assert (int(i.item()), int(s.item())) == exp
    rng = np.random.default_rng(splitter)
    for b in (3, 17, 61, 64):
        top = (1 << b) - (2 if splitter == 2 else 1)
        h = (rng.integers(0, 2**64 - 1, 20_000, dtype=np.uint64) % np.uint64(top + 1)) if b < 64 else \
            rng.integers(0, 2**64 - 1, 20_000, dtype=np.uint64)
        if splitter == 2:
            h = np.minimum(h, np.uint64(top))
        for lr in ([1, b // 2, b - 1] if splitter == 0 else [x for x in (1, 3, 1000, 1 << (b - 1)) if x <= 1 << (b - 1)]):
            i, s = mb.split_batch(splitter, dev(h), b, lr)
            got = list(zip(host_u64(i)[:300].tolist(), s.cpu().numpy()[:300].tolist()))
            assert got == [ref.split(splitter, int(x), b, lr) for x in h[:300]], (b, lr)
    with pytest.raises(mb.DomainError):
        mb.split_batch(splitter, dev(np.array([1 << 5], np.uint64)), 5, 2)
