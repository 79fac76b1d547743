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


class _OracleOps:
    """The CPU oracle standing in for the two KERNELS only (cs_update, cs_moments);
    sharding, zeroing, the merge and the estimator are bench.py's own code."""

    def __init__(self, orc):
        self.orc = orc

    def cs_update(self, spec, keys, table, wts=None):
        part = self.orc.cs_process(spec.rows, spec.width, spec.b, spec.families, spec.key_bits,
                                   spec.splitter, keys.numpy(), None if wts is None else wts.numpy())
        table += torch.from_numpy(part)  # int64 add wraps like the kernels' red.global

    def cs_moments(self, table, rows, width, mom):
        c = table.numpy()
        for r in range(rows):
            v, sat = self.orc.row_moment(c[r * width:(r + 1) * width], width)
            mom[r, 0] = np.int64(np.uint64(v & (2**64 - 1)).view(np.int64))
            mom[r, 1] = np.int64(np.uint64(v >> 64).view(np.int64))
            mom[r, 2] = int(sat)
            mom[r, 3] = 0


class _OracleSketch:
    """Host-API stand-in for bench.e2e_step (set_counters / process / counters /
    second_moment of mb.CountSketch), backed by the oracle."""

    def __init__(self, orc, spec):
        self.orc, self.spec = orc, spec
        self.c = np.zeros(spec.rows * spec.width, np.int64)

    def set_counters(self, c):
        self.c = np.array(c, np.int64)

    def counters(self):
        return self.c.copy()

    def process(self, keys, w):
        sp = self.spec
        self.orc.cs_process(sp.rows, sp.width, sp.b, sp.families, sp.key_bits, sp.splitter, keys, w,
                            counters=self.c)

    def second_moment(self, median=True):
        return self.orc.second_moment(self.c, self.spec.rows, self.spec.width, median)


def _bench_step_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import bench
    import paper_2008_08654_b200 as mb
    from oracle_bind import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle()
    merge = bench.TableMerge(mb, dist, world)
    assert "gloo" in merge.kind
    spec = mb.SketchSpec.seeded(ROWS, WIDTH, 61, 32, mb.SPLIT_POW2, S)
    lo, hi = bench.shard(N, rank, world)
    keys, w = orc.gen_zipf_items(S, lo, hi - lo)
    table = torch.full((ROWS * WIDTH,), 12345, dtype=torch.int64)  # stale: the step must zero it
    mom = torch.empty((ROWS, 4), dtype=torch.int64)
    ops = _OracleOps(orc)
    for _ in range(2):  # steps are idempotent
        bench.sketch_step(ops, spec, torch.from_numpy(keys), torch.from_numpy(w), table, mom, merge)
    f2 = mb.lower_median(mb.moments_to_python(mom))
    # the end-to-end step of the host API, twice (the counter reset makes it idempotent)
    sk = _OracleSketch(orc, spec)
    zeros = np.zeros(ROWS * WIDTH, np.int64)
    e2e = [bench.e2e_step(sk, keys, w, merge, zeros) for _ in range(2)]
    np.save(os.path.join(out_dir, f"table{rank}.npy"), table.numpy())
    np.save(os.path.join(out_dir, f"e2e{rank}.npy"), sk.counters())
    with open(os.path.join(out_dir, f"f2_{rank}.txt"), "w") as f:
        f.write(f"{f2[0]} {int(f2[1])} {e2e[0][0]} {e2e[1][0]}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_step_logic_merged_equals_single_pass(tmp_path, orc, world):
    """bench.py's own N > 1 step functions (sketch_step for configs 1/4/5, e2e_step for
    the host-API line, TableMerge): every rank ends with the merged table, and its
    median F2 equals the single-pass estimate."""
    mp.spawn(_bench_step_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, ROWS)]
    keys, w = orc.gen_zipf_items(S, 0, N)
    full = orc.cs_process(ROWS, WIDTH, 61, fams, 32, 0, keys, w)
    f2 = orc.second_moment(full, ROWS, WIDTH, True)[0]
    for r in range(world):
        assert (np.load(tmp_path / f"table{r}.npy") == full).all()
        assert (np.load(tmp_path / f"e2e{r}.npy") == full).all()
        got = open(tmp_path / f"f2_{r}.txt").read().split()
        assert [int(got[0]), int(got[2]), int(got[3])] == [f2, f2, f2] and got[1] == "0"


def test_shards_cover_every_item_once():
    sys.path.insert(0, ROOT)
    from bench import shard

    for n in (0, 1, 7, 1 << 31, 2**31 + 5):
        for world in (1, 2, 3, 4, 8):
            bounds = [shard(n, r, world) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in bounds) - min(b - a for a, b in bounds) <= 1
