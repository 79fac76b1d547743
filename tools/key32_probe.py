"""hash61 on 32-bit keys (the reference bench_hash setup, bench.cpp:96-144): per-launch CUDA-event times."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402

n = 1 << 28
keys = mb.gen_u32_keys(1 ^ mb.SALT_KEYS, 0, n)
out = torch.empty(n, dtype=torch.int64, device="cuda")
for k in (4, 8):
    c = mb.draw_coeffs(61, k, 1)
    ts = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mb.hash61(keys, c, key_bits=32, out=out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"key32 k={k}: {min(ts[1:]):.3f} ms  {n / min(ts[1:]) / 1e6:.3e} hashes/s", flush=True)
