"""Config 2, k = 8: Horner against the preconditioned (adapted-coefficient)
evaluation, both from tools/kvariants/c2_bench.cu, checked bit for bit against
the product kernel.  Usage (GPU box): python tools/kvariants/c2_pre.py "-DKU=4" ..."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2008_08654_b200 as mb  # noqa: E402
import precond_proto as pp  # noqa: E402


def i64(v):
    return v if v < 2**63 else v - 2**64


def main():
    n = 1 << 28
    keys, _ = mb.gen_below_p61(1 ^ mb.SALT_KEYS, 0, n)
    coeffs = [int(c) for c in mb.draw_coeffs(61, 8, 1)]
    ref = mb.hash61(keys, coeffs, key_bits=64)
    plan = pp.precondition(coeffs)
    for force_shift in (0, 1):
        if force_shift and plan["s"] == 0:
            # a shifted plan for the same polynomial (the SHIFT = true code path)
            plan = pp.precondition(coeffs, first_shift=1)
        dp = torch.tensor([i64(v) for v in plan["al"] + [plan["s"], plan["a7"], plan["r0"]]], dtype=torch.int64,
                          device="cuda")
        dc = torch.tensor([i64(c) for c in coeffs], dtype=torch.int64, device="cuda")
        out = torch.empty_like(ref)
        for i, flags in enumerate(sys.argv[1:] or [""]):
            so = f"/tmp/c2p{i}.so"
            subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                                   "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "paper_2008_08654_b200", "csrc")]
                                  + flags.split() + [os.path.join(ROOT, "tools", "kvariants", "c2_bench.cu"), "-o", so])
            lib = ctypes.CDLL(so)
            for f in (lib.c2_run, lib.c2_run_pre):
                f.restype = ctypes.c_float
                f.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p]
            out.zero_()
            ms = lib.c2_run(keys.data_ptr(), n, dc.data_ptr(), 8, 6, out.data_ptr())
            ok = bool((out == ref).all().item())
            print(f"horner {flags:30s} {ms * 1000:8.1f} us exact={ok}", flush=True)
            out.zero_()
            ms = lib.c2_run_pre(keys.data_ptr(), n, dp.data_ptr(), 1 if plan["s"] else 0, 6, out.data_ptr())
            ok = bool((out == ref).all().item())
            print(f"precond s={plan['s']} {flags:26s} {ms * 1000:8.1f} us exact={ok}", flush=True)


if __name__ == "__main__":
    main()
