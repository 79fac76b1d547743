"""L2 reduction rate (red.global.add on random cells) against the footprint of the cell array:
does spreading the counters over more L2 lines raise the rate config 5 is bound by?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402

sms = torch.cuda.get_device_properties(0).multi_processor_count
blocks, threads, iters = sms * 8, 256, 256
for mode, name, esz in ((2, "u64", 8), (5, "u32", 4)):
    for lg in (15, 17, 18, 19, 20, 21, 22, 23, 24, 26):
        span = 1 << lg
        buf = torch.zeros(span * esz // 8 + 1, dtype=torch.int64, device="cuda")
        best = 1e9
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mb.probe_atomics(mode, blocks, threads, iters, buf, span)
            e1.record()
            e1.synchronize()
            if rep:
                best = min(best, e0.elapsed_time(e1) / 1e3)
        print(f"red.{name} span 2^{lg} cells ({span * esz / 2**20:.2f} MiB): {blocks * threads * iters / best / 1e9:.1f} G red/s",
              flush=True)
