import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2008_08654_b200 as mb
dev = torch.device("cuda:0")
sink = torch.zeros(1, dtype=torch.int64, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
for blocks_per_sm, threads in [(8, 256), (4, 256), (8, 128), (16, 128), (2, 1024)]:
    blocks, iters = sms * blocks_per_sm, 4096
    for _ in range(2): mb.probe_imad(blocks, threads, iters, sink)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); mb.probe_imad(blocks, threads, iters, sink); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    r = blocks * threads * 8 * iters / best
    print(f"blocks/SM {blocks_per_sm} threads {threads}: {r:.4e} IMAD.WIDE/s = {r/sms/1.965e9:.1f} per SM per clk @1965MHz")
