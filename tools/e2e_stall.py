"""e2e stall probe: host-buffer CountSketch::process steps of config 5, each with
the host's CPU accounting (/proc/stat deltas: user, system, iowait, steal) and
this process's context switches, to tell a host-side stall from a device one."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_08654_b200 as mb  # noqa: E402


def cpu():
    f = open("/proc/stat").readline().split()[1:]
    return np.array([int(x) for x in f[:8]])


def ctx():
    d = {}
    for line in open(f"/proc/{os.getpid()}/status"):
        if "ctxt_switches" in line:
            k, v = line.split(":")
            d[k.strip()] = int(v)
    return d["voluntary_ctxt_switches"], d["nonvoluntary_ctxt_switches"]


n = 1 << 31
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mb.set_host_threads(threads)
zs = mb.ZipfStream(1)
dk = torch.empty(n, dtype=torch.int32, device="cuda")
dw = torch.empty(n, dtype=torch.int32, device="cuda")
zs.generate(0, n, dk, dw)
hk = torch.empty(n, dtype=torch.int32, pin_memory=True)
hw = torch.empty(n, dtype=torch.int32, pin_memory=True)
hk.copy_(dk)
hw.copy_(dw)
del dk, dw
torch.cuda.synchronize()
sk = mb.CountSketch(5, 1 << 16, 61, 32, mb.SPLIT_POW2, 1)
hk_np, hw_np = hk.numpy(), hw.numpy()
zeros = np.zeros(5 << 16, np.int64)
print(f"host threads {mb.host_threads()}", flush=True)
for i in range(steps):
    c0, x0 = cpu(), ctx()
    t0 = time.perf_counter()
    sk.set_counters(zeros)
    sk.process(hk_np, hw_np)
    f2 = sk.second_moment(True)
    dt = (time.perf_counter() - t0) * 1e3
    c1, x1 = cpu(), ctx()
    d = c1 - c0
    tot = d.sum()
    print(f"step {i:2d} {dt:7.1f} ms  user {d[0] / tot:.2f} sys {d[2] / tot:.2f} idle {d[3] / tot:.2f} "
          f"iowait {d[4] / tot:.2f} steal {d[7] / tot:.2f}  ctx vol {x1[0] - x0[0]} invol {x1[1] - x0[1]}",
          flush=True)
