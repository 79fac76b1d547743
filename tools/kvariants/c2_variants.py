"""A/B timing of config-2 hash kernel variants (tools/kvariants/c2_bench.cu -D
flags), checked bit for bit against the product kernel (mb200_hash61).
Usage (GPU box): python tools/kvariants/c2_variants.py 8 "-DKU=8 -DLOCK=1" ..."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2008_08654_b200 as mb  # noqa: E402


def main():
    k = int(sys.argv[1])
    n = 1 << 28
    keys, _ = mb.gen_below_p61(1 ^ mb.SALT_KEYS, 0, n)
    coeffs = mb.draw_coeffs(61, k, 1)
    ref = mb.hash61(keys, coeffs, key_bits=64)
    dc = torch.tensor([c if c < 2**63 else c - 2**64 for c in coeffs], dtype=torch.int64, device="cuda")
    out = torch.empty_like(ref)
    for i, flags in enumerate(sys.argv[2:] or [""]):
        so = f"/tmp/c2v{i}.so"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                               "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "paper_2008_08654_b200", "csrc")]
                              + flags.split() + [os.path.join(ROOT, "tools", "kvariants", "c2_bench.cu"), "-o", so])
        lib = ctypes.CDLL(so)
        lib.c2_run.restype = ctypes.c_float
        lib.c2_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                               ctypes.c_void_p]
        out.zero_()
        ms = lib.c2_run(keys.data_ptr(), n, dc.data_ptr(), k, 6, out.data_ptr())
        ok = bool((out == ref).all().item())
        print(f"{flags or '(default)':34s} {ms * 1000:8.1f} us  {n / ms / 1e6:.3e} hashes/s  exact={ok}", flush=True)


if __name__ == "__main__":
    main()
