"""Microbenchmarks that size the design (run on a B200): IMAD.WIDE.U32 peak and the
throughput of the atomic flavours the Count Sketch update can use."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"sms": sms}
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    for bps, thr in [(8, 256), (4, 256), (16, 128)]:
        blocks, iters = sms * bps, 4096
        t = timeit(lambda: mb.probe_imad(blocks, thr, iters, sink))
        res[f"imad_wide_per_s_{bps}x{thr}"] = blocks * thr * 8 * iters / t
    buf = torch.zeros(1 << 22, dtype=torch.int64, device="cuda")
    names = {0: "smem_u64_random4096", 1: "smem_u32_random4096", 2: "global_red_u64_random",
             3: "global_red_u64_same_addr", 4: "global_red_u64_warp_aggregated_same_addr",
             5: "global_red_u32_random", 6: "smem_cas_u32_random4096", 7: "smem_u32_add_with_return"}
    for mode, name in names.items():
        for span in ([1 << 14, 327680, 1 << 22] if mode in (2, 5) else [1]):
            blocks, thr, iters = sms * 8, 256, 256 if mode != 3 else 16
            t = timeit(lambda: mb.probe_atomics(mode, blocks, thr, iters, buf, span))
            ops = blocks * thr * iters / (32 if mode == 4 else 1)
            res[f"{name}_span{span}_ops_per_s"] = ops / t
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for cs, words in [(1, 40960), (2, 40960), (4, 32768), (8, 40960), (8, 16384)]:
        for mode in (0, 1, 2):
            blocks = (sms // cs) * cs
            iters = 256 if mode != 2 else 32
            try:
                t = timeit(lambda: mb.probe_dsmem(cs, mode, blocks, 512, iters, words, out))
                res[f"dsmem_cs{cs}_w{words}_mode{mode}_ops_per_s"] = blocks * 512 * iters / t
            except Exception as e:  # noqa: BLE001
                res[f"dsmem_cs{cs}_w{words}_mode{mode}"] = str(e)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
