"""CPU-side checks of the product boundary (no GPU compute):

- the C-ABI library loads and exports every symbol include/mersenne_b200.h declares;
- host-side logic (coefficient draw, row seeds, pseudo-Mersenne setup, argument
  validation with the reference's exception classes and messages) matches the oracle;
- with no sm_100 device the device entries fail loudly (no CPU fallback).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "mersenne_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mb200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(mb):
    syms = header_symbols()
    assert len(syms) >= 30
    lib = C.CDLL(mb.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers exactly the declared surface
    assert sorted(n for n, _, _ in mb.SIGNATURES) == syms


def test_harness_library_exports_its_header(mb):
    """Generators and probes live in a separate harness library, outside the drop-in ABI."""
    with open(os.path.join(ROOT, "include", "mersenne_b200_harness.h")) as f:
        syms = sorted(set(re.findall(r"\b(mb200_[a-z0-9_]+)\s*\(", f.read())))
    h = C.CDLL(mb._lib.HARNESS_PATH)
    assert all(hasattr(h, s) for s in syms)
    assert sorted(n for n, _, _ in mb._lib.HARNESS_SIGNATURES) == syms
    assert not set(syms) & set(header_symbols())
    prod = C.CDLL(mb.LIB_PATH)
    assert not any(hasattr(prod, s) for s in syms), "harness entries leaked into the product library"


def test_nccl_entries_validate_without_gpu(mb):
    """The multi-GPU merge entry rejects a null communicator before touching NCCL state."""
    import numpy as np
    with pytest.raises(mb.InvalidArgument, match="null communicator"):
        mb.check(mb.lib.mb200_cs_allreduce(None, 8, None, None))
    assert len(mb.nccl_unique_id()) == 128  # libnccl.so.2 resolved at run time


def test_abi_version(mb):
    assert mb.lib.mb200_abi_version() == 2


def test_host_coefficients_match_oracle(mb, orc, golden):
    S = golden["seed"]
    assert mb.draw_coeffs(61, 4, S) == golden["coeffs"]["61_4"]
    assert mb.draw_coeffs(89, 4, S) == [int(c) for c in golden["coeffs"]["89_4"]]
    assert mb.row_seeds(S, 5) == [int(s) for s in golden["row_seeds_5"]]
    rng = np.random.default_rng(1)
    for b in (3, 5, 13, 31, 61, 89, 107, 127):
        for _ in range(5):
            s = int(rng.integers(0, 2**63))
            assert mb.draw_coeffs(b, 8, s) == orc.coeffs(b, 8, s)


def test_host_pm_modulus_matches_oracle(mb, orc):
    rng = np.random.default_rng(7)
    for _ in range(100):
        b = int(rng.integers(2, 128))
        c = int(rng.integers(1, 2**min(b - 1, 63)))
        n = int(rng.integers(0, 6))
        assert mb.pm_modulus(b, c, n) == orc.pm_setup(b, c, n)[:2]
    assert mb.pm_modulus(64, 59) == orc.pm_setup(64, 59)[:2]


def _threshold_bigint(b, c, n):
    """field.cpp:173-193 in Python integers (an independent third statement)."""
    q = 1 << b
    d = c ** n if c & (c - 1) == 0 else c * q ** (n - 1)
    return min((q ** n - d) // c ** (n - 1), (1 << 255) - (1 << 127))


def test_host_pm_modulus_matches_reference_wide_c(mb, ref):
    """PseudoMersenneModulus(b, c, m) setup for u128 c (field.hpp:45) against the compiled
    reference over 200 random (b, c, m) -- including the default iteration count, which
    reaches ~2b rounds (~32k-bit intermediates) when c is close to 2^(b-1)."""
    rng = np.random.default_rng(0x5EED)
    cases = [(127, (1 << 126) - 1, 0), (127, 1, 0), (89, 1 << 70, 0), (127, (1 << 126) - 3, 0), (65, 2**64 - 1, 0),
             (2, 1, 0), (3, 3, 0), (128 - 1, 3, 7)]
    for _ in range(200):
        b = int(rng.integers(2, 128))
        c = int.from_bytes(rng.bytes(16), "little") % ((1 << (b - 1)) - 1) + 1
        if rng.random() < 0.3:
            c = max(1, (1 << (b - 1)) - 1 - int(rng.integers(0, 1000)))
        n = int(rng.integers(0, 8)) if rng.random() < 0.5 else 0
        cases.append((b, c, n))
    for b, c, n in cases:
        got = mb.pm_modulus(b, c, n)
        assert got == ref.pm_setup(b, c, n), (b, c, n)
        assert got[1] == _threshold_bigint(b, c, got[0]), (b, c, n)


def test_host_exact_division_iterations(mb, orc, ref):
    """ExactDivisionMap ctor (bucketing.cpp:75-89) on the host vs oracle and compiled reference."""
    rng = np.random.default_rng(0xE)
    cases = [(4, 3, 4), (4, 3, 13), (3, 1, 3), (64, 59, (1 << 64) - 59), (64, (1 << 62) + 1, 12345)]
    for _ in range(150):
        b = int(rng.integers(3, 65))
        c = int(rng.integers(1, 2 ** min(b - 1, 63)))
        p = (1 << b) - c
        r = int(rng.integers(1, min(p, 2**63 - 1) + 1)) if rng.random() < 0.7 else p if p < 2**64 else 1
        cases.append((b, c, r))
    for b, c, r in cases:
        m = mb.exact_division_iterations(b, c, r)
        assert m == orc.lib.orc_exact_div_iterations(b, c, r)
        assert m == ref.bucket_map(2, b, r, np.zeros(1, np.uint64), c=c)[0], (b, c, r)
    with pytest.raises(mb.InvalidArgument, match=r"bucket count must be in \[1, p\]"):
        mb.exact_division_iterations(4, 3, 14)
    with pytest.raises(mb.InvalidArgument, match="offset"):
        mb.exact_division_iterations(4, 8, 1)


def test_validation_messages(mb):
    with pytest.raises(mb.InvalidArgument, match=r"offset must satisfy 1 <= c < 2\^\(b-1\)"):
        mb.pm_modulus(4, 8)
    with pytest.raises(mb.InvalidArgument, match="offset"):
        mb.pm_modulus(4, 0)
    with pytest.raises(mb.InvalidArgument, match="exponent must be in"):
        mb.mersenne_modulus_check(1)
    with pytest.raises(mb.InvalidArgument, match="not prime"):
        mb.mersenne_modulus_check(11, True)
    mb.mersenne_modulus_check(11)
    mb.mersenne_modulus_check(127, True)
    with pytest.raises(mb.InvalidArgument, match="independence degree"):
        mb.draw_coeffs(61, 0, 1)


def test_sketch_descriptor_validation_without_gpu(mb):
    """Construction-time checks of sketch.cpp:97-119 run on the host before any launch."""
    import torch

    coeffs = mb.draw_coeffs(61, 4, 1)
    keys = torch.zeros(4, dtype=torch.int32)
    counters = torch.zeros(16, dtype=torch.int64)
    bad = [
        (mb.SketchSpec(1, 24, 61, [coeffs], 32), "power of two"),
        (mb.SketchSpec(1, 1, 61, [coeffs], 32, mb.SPLIT_MERSENNE_ARB), "width must be at least 2"),
        (mb.SketchSpec(1, 32, 5, [[1, 2, 3, 4]], 4), "strictly inside"),
        (mb.SketchSpec(1, 4, 5, [[1, 2, 3, 4]], 5), "modulus too small for key domain"),
        (mb.SketchSpec(1, 17, 5, [[1, 2, 3, 4]], 4, mb.SPLIT_MERSENNE_ARB), "half the hash range"),
        (mb.SketchSpec(1, 16, 61, [[mb.MASK64 >> 3] + coeffs[1:]], 32), "coefficient not reduced"),
    ]
    for spec, msg in bad:
        with pytest.raises(mb.InvalidArgument, match=msg):
            mb.lib.mb200_cs_update(C.byref(spec.desc), None, 32, None, 0, 0, None, None) and \
                mb.check(mb.lib.mb200_cs_update(C.byref(spec.desc), None, 32, None, 0, 0, None, None))
    del keys, counters


def test_no_cpu_fallback(mb):
    if mb.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(mb.CudaError):
        mb.CountSketch(1, 1024)
    import torch

    with pytest.raises(mb.InvalidArgument, match="CUDA tensors"):
        mb.hash61(torch.zeros(8, dtype=torch.int32), mb.draw_coeffs(61, 4, 1))


def test_enum_moment_validation_without_gpu(mb):
    """validate_moment_spec / exact_family_count messages (verify.cpp:480-503, 566-573):
    all checked on the host before any device work."""
    s = [(1, 2), (3, -1), (7, 3)]
    bad = [
        (dict(b=1, buckets=4, splitter=0, stream=s), "width must be in \\[2, 31\\]"),
        (dict(b=5, buckets=0, splitter=0, stream=s), "bucket count must be at least 1"),
        (dict(b=5, buckets=3, splitter=0, stream=s), "power of two for this splitter"),
        (dict(b=5, buckets=17, splitter=2, stream=s), "exceeds half the hash range"),
        (dict(b=5, buckets=4, splitter=0, stream=s, key_domain=32), "modulus too small for key domain"),
        (dict(b=5, buckets=4, splitter=0, stream=[]), "stream must not be empty"),
        (dict(b=5, buckets=4, splitter=0, stream=s, key_domain=5), "key outside domain"),
        (dict(b=5, buckets=4, splitter=0, stream=[(1, 1000), (2, 25)]), "too large for exact enumeration"),
        (dict(b=5, buckets=4, splitter=0, stream=[(1, 1), (1, 2)]), "distinct modulo the modulus"),
        (dict(b=16, buckets=4, splitter=0, stream=s), "\\[2, 15\\] to enumerate exactly"),
        (dict(b=5, buckets=4, splitter=3, stream=s), "unknown splitter"),
    ]
    for kw, msg in bad:
        with pytest.raises(mb.InvalidArgument, match=msg):
            mb.enum_moment_sums(**kw)
    big = [(i, 1) for i in range(70)]
    with pytest.raises(mb.Unsupported, match="64 non-zero"):
        mb.enum_moment_sums(7, 4, 0, big)


def test_host_threads_setting(mb):
    """Packing threads of the host-buffer entry: explicit, then automatic (this
    process's CPUs per local rank, one left free, at most 8)."""
    try:
        mb.set_host_threads(3)
        assert mb.host_threads() == 3
        mb.set_host_threads(0)
        auto = mb.host_threads()
        cpus = len(os.sched_getaffinity(0)) // int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1)
        assert auto == max(1, min(cpus - 1 if cpus >= 8 else cpus, 8))
    finally:
        mb.set_host_threads(0)


P61 = (1 << 61) - 1


def _horner61(coeffs, x):
    y = 0
    for a in reversed(coeffs):
        y = (y * x + a) % P61
    return y


def _eval_plan(pl, x):
    al = pl["al"]
    x %= P61
    z = ((x + al[0]) * x + al[1]) % P61
    w = ((x + al[2]) * z + al[3]) % P61
    u = ((w + z + al[4]) * w + al[5]) % P61
    return (pl["a7"] * ((x + pl["s"]) * u % P61) + pl["r0"]) % P61


def test_precondition61_equals_horner(mb, orc):
    """The adapted coefficients of the k = 8 hash (host/precond61.cpp) define the same
    polynomial function as Horner's rule over Z_(2^61-1): seeded families, the oracle's
    config-2 family, coefficient extremes, families that need a shift (cubic without a
    root at shift 0), and the degenerate leading coefficient."""
    rng = np.random.default_rng(61)
    fams = [[int(v) for v in orc.coeffs(61, 8, seed)] for seed in range(1, 65)]
    fams += [[int(rng.integers(0, P61)) for _ in range(8)] for _ in range(64)]
    fams += [[0] * 7 + [1], [P61 - 1] * 8, [0, 0, 0, 0, 0, 0, 0, P61 - 1], [1] * 8, [P61 - 1] * 7 + [1]]
    keys = [0, 1, 2, P61 - 1, P61, P61 + 1, (1 << 64) - 1] + [int(v) for v in rng.integers(0, 1 << 63, 24)]
    shifts = set()
    for c in fams:
        pl = mb.precondition61(c)
        assert pl is not None and all(0 <= v < P61 for v in pl["al"] + [pl["a7"], pl["r0"]]) and pl["s"] < 64
        shifts.add(pl["s"])
        for x in keys:
            assert _eval_plan(pl, x) == _horner61(c, x % P61), (c, x)
    assert 0 in shifts and len(shifts) > 1  # both kernel variants are reachable
    assert mb.precondition61([1, 2, 3, 4, 5, 6, 7, 0]) is None  # degree < 7: Horner
    with pytest.raises(ValueError):
        mb.precondition61([P61] + [1] * 7)  # unreduced coefficient
