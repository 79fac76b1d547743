"""One config's hot kernel, launched `--reps` times on BASELINE-sized inputs: the
command profiled by ncu (tools/ncu_round.sh).  Prints the per-launch CUDA-event
time so the same command also gives an un-profiled reference number."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402

S = 1
SK = S ^ mb.SALT_KEYS


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c1", "c2k4", "c2k8", "c3", "c4", "c5"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--binned", action="store_true", help="large tables: binned strategy")
    ap.add_argument("--rows", action="store_true", help="large tables: miss buffer + row passes")
    ap.add_argument("--items", type=int, default=1 << 31, help="config-5 stream length (one shard of N GPUs)")
    a = ap.parse_args()
    w = a.which
    if a.binned:
        mb.set_large_table_strategy(mb.LARGE_BINNED)
    if a.rows:
        mb.set_large_table_strategy(mb.LARGE_ROWS)
    if w == "c5":
        zs = mb.ZipfStream(S)
        keys, wts = zs.generate(0, a.items)
        spec = mb.SketchSpec.seeded(5, 1 << 16, 61, 32, mb.SPLIT_POW2, S)
        table = torch.zeros(5 << 16, dtype=torch.int64, device="cuda")
        fn = lambda: mb.cs_update(spec, keys, table, wts)  # noqa: E731
    elif w == "c1":
        keys = mb.gen_u32_keys(SK, 0, 1 << 24)
        spec = mb.SketchSpec.seeded(1, 1024, 61, 32, mb.SPLIT_POW2, S)
        table = torch.zeros(1024, dtype=torch.int64, device="cuda")
        fn = lambda: mb.cs_update(spec, keys, table)  # noqa: E731
    elif w in ("c2k4", "c2k8"):
        keys, _ = mb.gen_below_p61(SK, 0, 1 << 28)
        out = torch.empty(1 << 28, dtype=torch.int64, device="cuda")
        coeffs = mb.draw_coeffs(61, 4 if w == "c2k4" else 8, S)
        fn = lambda: mb.hash61(keys, coeffs, key_bits=64, out=out)  # noqa: E731
    elif w == "c3":
        v, _ = mb.gen_pm_inputs(SK, 59, 0, 1 << 28)
        q = torch.empty(1 << 28, dtype=torch.int64, device="cuda")
        r = torch.empty(1 << 28, dtype=torch.int64, device="cuda")
        ovf = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: mb.pm_divmod(v, 64, 59, 3, q, r, ovf)  # noqa: E731
    else:
        keys = mb.gen_u64_keys(SK, 0, 1 << 26)
        spec = mb.SketchSpec(2, 1 << 16, 89, [mb.draw_coeffs(89, 4, S)], 64, mb.SPLIT_TWO_FOR_ONE)
        table = torch.zeros(2 << 16, dtype=torch.int64, device="cuda")
        fn = lambda: mb.cs_update(spec, keys, table)  # noqa: E731
    torch.cuda.synchronize()
    for i in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        print(f"{w} launch {i}: {e0.elapsed_time(e1):.3f} ms", flush=True)
    if w == "c5":
        hs = mb.hot_stats(reset=True)
        print(f"c5 hot set: {hs['hot_keys'] / a.reps:.0f} keys placed, miss fraction "
              f"{hs['misses'] / max(1, hs['items']):.4f}", flush=True)


if __name__ == "__main__":
    main()
