"""Direct vs binned large-table strategy on a few stream shapes (event timing)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402


def run(name, spec, keys, w, rows, width):
    table = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    out = {}
    for strat, sname in ((mb.LARGE_DIRECT, "direct"), (mb.LARGE_BINNED, "binned")):
        prev = mb.set_large_table_strategy(strat)
        best = 1e9
        for _ in range(4):
            table.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            mb.cs_update(spec, keys, table, w)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        mb.set_large_table_strategy(prev)
        out[sname] = best
    print(f"{name:40s} direct {out['direct']:8.3f} ms  binned {out['binned']:8.3f} ms", flush=True)


n = 1 << 26
ku = mb.gen_u32_keys(5, 0, n)
w = torch.randint(-100, 101, (n,), dtype=torch.int32, device="cuda")
for rows in (2, 5, 10):
    spec = mb.SketchSpec.seeded(rows, 1 << 16, 61, 32, mb.SPLIT_POW2, 1)
    run(f"uniform u32, {rows} rows x 2^16", spec, ku, w, rows, 1 << 16)
zs = mb.ZipfStream(1)
zk, zw = zs.generate(0, n)
spec = mb.SketchSpec.seeded(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 1)
run("zipf1.2 u32, 5 rows x 2^16", spec, zk, zw, 5, 1 << 16)
k64 = mb.gen_u64_keys(7, 0, n)
spec = mb.SketchSpec(2, 1 << 16, 89, [mb.draw_coeffs(89, 4, 1)], 64, mb.SPLIT_TWO_FOR_ONE)
run("config-4 shape (89-bit, 2 rows)", spec, k64, None, 2, 1 << 16)
