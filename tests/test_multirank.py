"""The N > 1 path on CPU: world_size-2 gloo ranks run bench.py's sharding and
table merge with the CPU oracle standing in for the per-GPU scatter kernel.

Count Sketch is linear (sketch.cpp:182-193, merge-equals-concatenation,
test_sketch.cpp:239-261): the allreduce-summed per-rank tables must equal the
single-pass table bit for bit, and so must the median-of-rows F2 estimate.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS, WIDTH, N, S = 5, 1 << 12, 200_003, 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from bench import shard
    from oracle_bind import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle()
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, ROWS)]
    lo, hi = shard(N, rank, world)
    keys, w = orc.gen_zipf_items(S, lo, hi - lo)  # counter-addressable: this rank's window only
    table = orc.cs_process(ROWS, WIDTH, 61, fams, 32, 0, keys, w)
    t = torch.from_numpy(table)
    dist.all_reduce(t)  # the NCCL allreduce of bench.py, here over gloo
    elapsed = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)  # max-over-ranks timing
    if rank == 0:
        np.save(os.path.join(out_dir, "merged.npy"), t.numpy())
        np.save(os.path.join(out_dir, "max.npy"), elapsed.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_merge_equals_single_pass(tmp_path, orc, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    merged = np.load(tmp_path / "merged.npy")
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, ROWS)]
    keys, w = orc.gen_zipf_items(S, 0, N)
    full = orc.cs_process(ROWS, WIDTH, 61, fams, 32, 0, keys, w)
    assert (merged == full).all()
    assert orc.second_moment(merged, ROWS, WIDTH, True) == orc.second_moment(full, ROWS, WIDTH, True)
    assert float(np.load(tmp_path / "max.npy")[0]) == float(world)


def test_shards_cover_every_item_once():
    sys.path.insert(0, ROOT)
    from bench import shard

    for n in (0, 1, 7, 1 << 31, 2**31 + 5):
        for world in (1, 2, 3, 4, 8):
            bounds = [shard(n, r, world) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in bounds) - min(b - a for a, b in bounds) <= 1
