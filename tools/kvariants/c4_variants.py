"""A/B timing of cs_private89_kernel source variants (-D flags of
mb200_private89.cuh) on config 4's input, one nvcc build per variant.
Usage (GPU box): python tools/kvariants/c4_variants.py "-DH89V=1" "-DH89V=3" ..."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2008_08654_b200 as mb  # noqa: E402


def build(flags, out):
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
           "-fPIC", "-I" + os.path.join(ROOT, "paper_2008_08654_b200", "csrc")] + flags.split() + [
        os.path.join(ROOT, "tools", "kvariants", "c4_bench.cu"), "-o", out]
    subprocess.check_call(cmd)


def main():
    n = 1 << 26
    keys = mb.gen_u64_keys(1 ^ mb.SALT_KEYS, 0, n)
    c = mb.draw_coeffs(89, 4, 1)
    coef = (ctypes.c_uint32 * 12)(*[(v >> (32 * l)) & 0xffffffff for v in c for l in range(3)])
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    scratch = torch.empty(sms * (2 << 16), dtype=torch.uint8, device="cuda")
    table = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
    go = torch.zeros(1, dtype=torch.int32, device="cuda")
    for i, flags in enumerate(sys.argv[1:] or [""]):
        so = f"/tmp/c4v{i}.so"
        build(flags, so)
        lib = ctypes.CDLL(so)
        lib.c4_run.restype = ctypes.c_float
        lib.c4_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p]
        ms = lib.c4_run(keys.data_ptr(), n, coef, 6, scratch.data_ptr(), table.data_ptr(), go.data_ptr())
        print(f"{flags or '(default)':40s} {ms * 1000:8.1f} us  ({n / ms / 1e6:.3e} keys/s)", flush=True)


if __name__ == "__main__":
    main()
