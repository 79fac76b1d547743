"""Host-buffer (end-to-end) throughput of the CountSketch object API vs raw H2D copies."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 31
zs = mb.ZipfStream(1)
dk = torch.empty(n, dtype=torch.int32, device="cuda")
dw = torch.empty(n, dtype=torch.int32, device="cuda")
zs.generate(0, n, dk, dw)
hk = torch.empty(n, dtype=torch.int32, pin_memory=True)
hw = torch.empty(n, dtype=torch.int32, pin_memory=True)
hk.copy_(dk)
hw.copy_(dw)
torch.cuda.synchronize()
# raw H2D bandwidth of the same bytes
for _ in range(4):
    t0 = time.perf_counter()
    dk.copy_(hk, non_blocking=True)
    dw.copy_(hw, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"raw H2D: {2 * 4 * n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
sk = mb.CountSketch(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 1)
hk_np, hw_np = hk.numpy(), hw.numpy()
for rep in range(8):
    t0 = time.perf_counter()
    sk.process(hk_np, hw_np)
    dt = time.perf_counter() - t0
    print(f"process(): {n / dt / 1e9:.2f} G items/s, {2 * 4 * n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
