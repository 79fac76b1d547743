"""Config 5: hot-set sample size vs miss fraction and step time (event timing)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("EXPDIR") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402

n = int(os.environ.get("ITEMS", 1 << 31))
zs = mb.ZipfStream(1)
keys, wts = zs.generate(0, n)
spec = mb.SketchSpec.seeded(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 1)
table = torch.zeros(5 << 16, dtype=torch.int64, device="cuda")
ref = None
for lg, cap in [(int(x.split(":")[0]), x.split(":")[1]) for x in os.environ.get("LOGS", "20:20480").split()]:
    os.environ["MB200_HH_SAMPLE_LOG2"] = str(lg)
    os.environ["MB200_HH_CAP"] = cap
    ts = []
    for r in range(4):
        table.zero_()
        mb.hot_stats(reset=True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mb.cs_update(spec, keys, table, wts)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
        hs = mb.hot_stats()
    t = table.cpu()
    if ref is None:
        ref = t
    assert torch.equal(t, ref)
    print(f"sample 2^{lg} cap {cap}: {sorted(ts)[1]:.3f} ms  miss {hs['misses'] / hs['items']:.4f}  hot_keys {hs['hot_keys']}", flush=True)
