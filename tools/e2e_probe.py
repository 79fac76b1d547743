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
import statistics  # noqa: E402
import subprocess  # noqa: E402
import threading  # noqa: E402

# a background nvidia-smi sampler like bench.py's clocks thread (contention check)
stop = threading.Event()


def sampler():
    while not stop.is_set():
        subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True)
        time.sleep(0.2)


threads = [int(t) for t in os.environ.get("THREADS", "0").split(",")]
for with_sampler in (False, True):
    if with_sampler:
        th = threading.Thread(target=sampler, daemon=True)
        th.start()
    for t in threads:
        mb.set_host_threads(t)
        ms = []
        for rep in range(8):
            t0 = time.perf_counter()
            sk.process(hk_np, hw_np)
            ms.append((time.perf_counter() - t0) * 1e3)
        ms = ms[2:]
        print(f"threads={mb.host_threads():3d} sampler={with_sampler}: process() ms min {min(ms):.1f} "
              f"median {statistics.median(ms):.1f} max {max(ms):.1f} -> {n / statistics.median(ms) / 1e6:.2f} G items/s")
stop.set()
