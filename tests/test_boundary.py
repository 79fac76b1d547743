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


def test_abi_version(mb):
    assert mb.lib.mb200_abi_version() == 1


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
