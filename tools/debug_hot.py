import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2008_08654_b200 as mb  # noqa: E402
from oracle_bind import oracle  # noqa: E402

orc = oracle()


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def run(rows, width, b, kb, sp, keys, w, tag):
    fams = [orc.coeffs(b, 4, s) for s in orc.row_seeds(0xB16 + rows, rows)]
    spec = mb.SketchSpec(rows, width, b, fams, kb, sp)
    cnt = torch.zeros(rows * width, dtype=torch.int64, device="cuda")
    mb.cs_update(spec, dev(keys), cnt, None if w is None else dev(w))
    exp = orc.cs_process(rows, width, b, fams, kb, sp, keys, w)
    got = cnt.cpu().numpy()
    bad = np.nonzero(got != exp)[0]
    print(tag, "mismatches", len(bad), "of", len(exp), "sum diff", int((got - exp).sum()),
          [(int(i), int(got[i]), int(exp[i])) for i in bad[:4]])


n = (1 << 22) + 12345
zk, zw = orc.gen_zipf_items(7, 0, n)
k64 = zk.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
w = zw.astype(np.int32)
run(3, 4096, 61, 64, 0, k64, w, "base")
run(3, 4096, 61, 64, 0, k64, None, "noweights")
run(3, 4096, 61, 64, 0, zk.astype(np.uint64), w, "small u64 keys")
run(3, 4096, 61, 32, 0, zk, w, "u32 keys")
k2 = k64.copy()
k2[:3] = [0, np.iinfo(np.uint64).max, 0]
run(3, 4096, 61, 64, 0, k2, w, "sentinel")
w2 = w.copy()
w2[:4] = [np.iinfo(np.int32).min, np.iinfo(np.int32).max, -1, 1]
run(3, 4096, 61, 64, 0, k64, w2, "extreme w")
run(3, 4096, 61, 64, 0, k64[: 1 << 20], w[: 1 << 20], "small n")
