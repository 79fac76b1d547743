#!/usr/bin/env python3
"""Benchmark of the B200 hashing / Count Sketch path (BASELINE.json metric:
"4-universal hashes/s and Count Sketch updates/s per B200, at 1/2/4/8 GPUs").

Headline workload: config 5 (BASELINE.json configs[4]) -- Count Sketch with
t = 5 rows x 2^16 int64 counters, degree-3 mod 2^61-1 families, two-for-one
bucket/sign split, 2^31 Zipf(1.2) items with int32 weights in [-100, 100],
sharded over the ranks, tables merged by NCCL allreduce, median-of-rows F2.
One step = zero table + fused hash/split/scatter over the rank's shard +
allreduce + estimator.  value = items (Count Sketch updates) per second over
the whole job; each item is t = 5 four-universal hash evaluations.

Configs 1-4 are measured in the same run and reported under "configs".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S = 1  # master seed (the reference CLI default, commands.cpp:31)
C5_ITEMS = 1 << 31
C5_ROWS, C5_WIDTH = 5, 1 << 16
C1_ITEMS, C2_KEYS, C3_UNITS, C4_KEYS = 1 << 24, 1 << 28, 1 << 28, 1 << 26
# algorithmic work per unit: bytes of HBM traffic and 32x32->64 limb products
WORK = {
    "c1": (4, 6), "c2_k4": (16, 12), "c2_k8": (16, 28), "c3": (32, 6), "c4": (8, 18), "c5": (8, 30),
    # SURVEY 8f rank 4 (not BASELINE configs): ExactDivisionMap over u64 values --
    # 8 B in + 8 B out; v r (4 limb products) + 2 Alg-4 rounds by a 6-bit c (2 x 2)
    "exact_div": (16, 8),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip configs 1-4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--items", type=int, default=C5_ITEMS, help="config-5 stream length (tests only)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(n, rank, world):
    """Contiguous shard [lo, hi) of n units for `rank` (every unit exactly once)."""
    return n * rank // world, n * (rank + 1) // world


class TableMerge:
    """The N > 1 exchange step: ONE in-place allreduce of the rank-local
    t x m counter table -- the distributed CountSketch::merge (sketch.cpp:182-193).
    On GPUs it is the product's own entry, mb200_cs_allreduce, over an NCCL
    communicator the product library made (mb.NcclComm); the table never leaves HBM.
    Under gloo (the CPU tests) torch.distributed sums the CPU table instead."""

    def __init__(self, mb, dist, world):
        self.mb, self.dist, self.world, self.comm = mb, dist, world, None
        self.kind = "none (one rank)"
        if world > 1:
            if dist.get_backend() == "nccl":
                self.comm = mb.NcclComm.from_process_group()
                self.kind = "mb200_cs_allreduce (NCCL uint64 sum, in place in HBM)"
            else:
                self.kind = f"torch.distributed.all_reduce ({dist.get_backend()}, CPU tables)"

    def table(self, t, stream=None):
        if self.world == 1:
            return
        if self.comm is not None:
            self.mb.cs_allreduce(t, self.comm, stream)
        else:
            self.dist.all_reduce(t)

    def sketch(self, sk):
        """CountSketch.allreduce: the sketch object's HBM table summed in place."""
        if self.world == 1:
            return
        if self.comm is not None:
            sk.allreduce(self.comm)
        else:
            import torch
            t = torch.from_numpy(sk.counters())
            self.dist.all_reduce(t)
            sk.set_counters(t.numpy())


def sketch_step(ops, spec, keys, wts, table, mom, merge, ev=None):
    """One step of a sharded Count Sketch config on one rank: zero the rank's table,
    fused hash -> split -> scatter of its shard, merge over the ranks, estimator.
    `ev` = (start, stop) events around the scatter kernel(s)."""
    table.zero_()
    if ev is not None:
        ev[0].record()
    ops.cs_update(spec, keys, table, wts)
    if ev is not None:
        ev[1].record()
    merge.table(table)
    ops.cs_moments(table, spec.rows, spec.width, mom)


def e2e_step(sk, h_keys, h_wts, merge, zeros):
    """The same step through the public host API: counters reset, process() of HOST
    buffers (H2D inside), merge of the replicas' HBM tables, median F2 read back.
    BENCH_TRACE_E2E=1 prints the parts' wall times to stderr."""
    t = [time.perf_counter()]
    sk.set_counters(zeros)
    t.append(time.perf_counter())
    sk.process(h_keys, h_wts)
    t.append(time.perf_counter())
    merge.sketch(sk)
    t.append(time.perf_counter())
    m = sk.second_moment(True)
    t.append(time.perf_counter())
    if os.environ.get("BENCH_TRACE_E2E"):
        parts = ", ".join(f"{k} {1e3 * (b - a):.1f}" for k, a, b in zip(("reset", "process", "merge", "moment"), t, t[1:]))
        print(f"[e2e step] {parts} ms", file=sys.stderr, flush=True)
    return m


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- reference arm / CPU baselines
def cpu_info():
    """Host CPU of this run (nproc + lscpu model + threads per core)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k == "Thread(s) per core":
                info["threads_per_core"] = int(v)
            elif k == "Core(s) per socket":
                info["cores_per_socket"] = int(v)
            elif k == "Socket(s)":
                info["sockets"] = int(v)
    except Exception:  # noqa: BLE001
        pass
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        pass
    return info


def _median_rate(fn, units, reps):
    """Units per second: median of `reps` timed calls after one warm-up."""
    fn()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return units / statistics.median(times), statistics.median(times)


def cpu_baselines(threads=None, reps=3):
    """The reference's own CPU path (oracle/_ref = the unmodified reference sources
    compiled by oracle/Makefile; the oracle port if it is absent) on every config,
    single-thread and all-core, on bounded samples of each config's own inputs,
    plus the reference's own benchmark loops (cli::bench_hash / bench_div,
    bench.cpp:96-189: 3 warm-ups + median of 5).  Reported baselines, not targets."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import oracle, reference

    ref, orc = reference(), oracle()
    kind = "reference" if ref is not None else "port"
    allc = threads or (os.cpu_count() or 1)
    SK = S ^ 0x7B5BAD595E238E31
    out = {"_cpu": cpu_info()}

    def lines(name, unit, sample, run1, runN, n1, nN, note):
        ent = {"unit": unit, "kind": kind, "note": note}
        for tag, fn, n, cores in (("single_thread", run1, n1, 1), ("all_core", runN, nN, allc)):
            v, sec = _median_rate(fn, n, reps)
            ent[tag] = {"value": v, "cores": cores, "sample": f"{n} {sample}", "median_s": sec}
        ent["value"], ent["cores"] = ent["all_core"]["value"], allc
        ent["sample"] = ent["all_core"]["sample"] + f"; median of {reps} after 1 warm-up"
        out[name] = ent

    fams5 = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, 5)]
    if ref is not None:
        # config 1: CountSketch(1, 1024)::process over u32 keys (shard + merge() on all cores)
        k1 = orc.gen_u32_keys(SK, 0, 1 << 23)
        lines("c1", "updates/s", "config-1 keys", lambda: ref.cs_run(1, 1024, 61, 32, 0, S, k1[:1 << 21]),
              lambda: ref.cs_run(1, 1024, 61, 32, 0, S, k1, threads=allc), 1 << 21, 1 << 23,
              "CountSketch::process (sketch.cpp:133-140)")
        # config 2: keys in [0, p) lie outside the reference API's domain: Horner with the
        # reference's own Alg 3 per step (the route make_golden.py pins)
        kp = orc.gen_below_p61(SK, 0, 1 << 23)
        for k in (4, 8):
            ck = ref.coeffs(61, k, S)
            lines(f"c2_k{k}", "hashes/s", "config-2 keys", lambda ck=ck: ref.hash_full(61, ck, kp[:1 << 21]),
                  lambda ck=ck: ref.hash_full(61, ck, kp, threads=allc), 1 << 21, 1 << 23,
                  "Horner on the reference's mersenne_divmod (field.cpp:208-222)")
            ops, _ = ref.bench_hash(61, k, 10_000_000, S)
            out[f"c2_k{k}"]["reference_bench_hash"] = {
                "value": ops, "unit": "hashes/s", "cores": 1,
                "sample": "cli::bench_hash(61, k, 1e7): PolyHashFamily::operator() on 32-bit keys incl. key "
                          "generation, median of 5 after 3 warm-ups (bench.cpp:96-144)"}
        # config 3: pseudo_mersenne_div + pseudo_mersenne_mod by 2^64 - 59
        v3 = orc.gen_pm_inputs(SK, 59, 0, 1 << 22)
        lines("c3", "divmod/s", "config-3 inputs", lambda: ref.pm_divmod_batch(64, 59, v3[:2 << 20]),
              lambda: ref.pm_divmod_batch(64, 59, v3, threads=allc), 1 << 20, 1 << 22,
              "pseudo_mersenne_div + pseudo_mersenne_mod (field.cpp:260-273), Generic engine")
        bops, casc, _ = ref.bench_div(64, 59, 2_000_000, S)
        out["c3"]["reference_bench_div"] = {
            "value": bops, "cascade_value": casc, "unit": "divmod/s", "cores": 1,
            "sample": "cli::bench_div(64, 59, 2e6): branch-free Alg 4+5 and the cch_divmod cascade, "
                      "median of 5 after 3 warm-ups (bench.cpp:146-189)"}
        # config 4: 89-bit hash -> two-for-one split -> two rows (reference hash + split_pow2)
        c89 = ref.coeffs(89, 4, S, key_bits=64)
        k4 = orc.gen_u64_keys(SK, 0, 1 << 23)
        lines("c4", "keys/s", "config-4 keys", lambda: ref.two_for_one(c89, k4[:1 << 21]),
              lambda: ref.two_for_one(c89, k4, threads=allc), 1 << 21, 1 << 23,
              "PolyHashFamily(m89)::operator() + split_pow2 twice (SURVEY 7.4)")
        # config 5: CountSketch(5, 65536)::process over the Zipf stream
        zk, zw = orc.gen_zipf_items(S, 0, 1 << 23)
        lines("c5", "updates/s", "config-5 Zipf items", lambda: ref.cs_run(5, 65536, 61, 32, 0, S, zk[:1 << 21], zw[:1 << 21]),
              lambda: ref.cs_run(5, 65536, 61, 32, 0, S, zk, zw, threads=allc), 1 << 21, 1 << 23,
              "CountSketch::process (sketch.cpp:133-140), all-core = contiguous shards + merge()")
    else:  # oracle port (oracle.c, OpenMP): config 5 only
        zk, zw = orc.gen_zipf_items(S, 0, 1 << 22)
        lines("c5", "updates/s", "config-5 Zipf items",
              lambda: orc.cs_process(5, 65536, 61, fams5, 32, 0, zk[:1 << 20], zw[:1 << 20]),
              lambda: orc.cs_process(5, 65536, 61, fams5, 32, 0, zk, zw), 1 << 20, 1 << 22, "oracle port")
    return out


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    per_step = 1 << 23
    cores = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import oracle, reference

    ref = reference()
    orc = oracle()
    keys, w = orc.gen_zipf_items(S, 0, per_step)
    kind = "reference" if ref is not None else "port"
    fams = [orc.coeffs(61, 4, s) for s in orc.row_seeds(S, C5_ROWS)]

    def step():
        if ref is not None:
            ref.cs_run(C5_ROWS, C5_WIDTH, 61, 32, 0, S, keys, w, threads=cores)
        else:
            orc.cs_process(C5_ROWS, C5_WIDTH, 61, fams, 32, 0, keys, w)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": metric_name(), "value": value, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "config5_countsketch_t5_m65536_zipf1.2", "sample_items_per_step": per_step,
                   "rows": C5_ROWS, "width": C5_WIDTH, "prime": "2^61-1", "k": 4},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} items of the config-5 stream per step, CountSketch::process "
                                   f"sharded over {cores} threads + merge()", "cpu": cpu_info()},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name():
    return "Count Sketch updates/s (config 5: t=5 rows of 4-universal 2^61-1 hashes, 2^31 Zipf items)"


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2008_08654_b200 as mb

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    merge = TableMerge(mb, dist, world)
    hbm_peak, peak_kind = load_peaks()
    traffic = load_traffic()

    # ---- integer-pipe peak: independent IMAD.WIDE.U32 product chains (
    # the SASS of the probe loop is IMAD.WIDE only, profiles/r02f/imad_probe.txt) ----
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    blocks, threads, iters = mb_sm_count(torch) * 8, 256, 4096
    for _ in range(2):
        mb.probe_imad(blocks, threads, iters, sink)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mb.probe_imad(blocks, threads, iters, sink)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    imad_peak = blocks * threads * 8 * iters / best  # IMAD.WIDE.U32 per second
    # L2 reduction peak: red.global.add.u64 on random cells of a config-5-sized table
    red_buf = torch.zeros(C5_ROWS * C5_WIDTH, dtype=torch.int64, device=dev)
    rblocks, rthreads, riters = mb_sm_count(torch) * 8, 256, 256
    best = 1e9
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mb.probe_atomics(2, rblocks, rthreads, riters, red_buf, C5_ROWS * C5_WIDTH)
        e1.record()
        e1.synchronize()
        if rep:
            best = min(best, e0.elapsed_time(e1) / 1e3)
    red_peak = rblocks * rthreads * riters / best
    del red_buf

    def roofline(cfg, units, kernel_s, kname, l2_reds=None):
        """SURVEY 8d roofline of one kernel: algorithmic bytes (HBM) and 32x32->64 limb
        products (integer pipe, against the IMAD.WIDE peak measured in this run) per
        launch over its CUDA-event time; `bound` is the larger of the two fractions,
        the roofline 8d defines.  `binding_unit` is the pipe the committed ncu capture
        of the same kernel shows busiest (what actually limits it), and for the
        scatter kernels the counted L2 reductions are reported against the measured
        red.global rate as a further view."""
        bpu, lpu = WORK[cfg]
        hbm = units * bpu / kernel_s / 1e9
        ints = units * lpu / kernel_s
        frac_h, frac_i = hbm / hbm_peak, ints / imad_peak
        ent = traffic.get(kname) or {}
        views = {"hbm": {"achieved": hbm, "peak": hbm_peak, "unit": "GB/s", "frac": frac_h, "peak_kind": peak_kind,
                         "frac_of_8TBs": hbm / 8000.0},
                 "int": {"achieved": ints / 1e12, "peak": imad_peak / 1e12, "unit": "T IMAD.WIDE/s", "frac": frac_i,
                         "peak_kind": "measured (probe_imad, this run)",
                         "note": "algorithmic limb products (SURVEY 8d) / measured IMAD.WIDE.U32 peak"}}
        bound = "hbm" if frac_h >= frac_i else "int"
        out = {"bound": bound, **{k: views[bound][k] for k in ("achieved", "peak", "unit", "frac")},
               "traffic": ent.get("dram_bytes_per_launch"), "peak_kind": views[bound]["peak_kind"]}
        out.update({k: v for k, v in views.items() if k != bound})
        if bound == "hbm" and frac_h > 1.0:
            out["note"] = ("algorithmic read+write traffic above the driver-measured copy bandwidth "
                           "(MEASURED_PEAKS.json); see frac_of_8TBs for the nominal figure")
            out["frac_of_8TBs"] = hbm / 8000.0
        if l2_reds is not None:
            out["l2_red"] = {"achieved": l2_reds / kernel_s / 1e9, "peak": red_peak / 1e9, "unit": "G red/s",
                             "frac": l2_reds / kernel_s / red_peak, "reds_per_launch": l2_reds,
                             "peak_kind": "measured (probe_atomics random red.global.add.u64, this run)"}
        wi = ent.get("warp_instructions_per_launch")
        if wi and world == 1:  # ncu's executed warp instructions of the same-size launch, per unit of work
            out["thread_instructions_per_unit"] = wi * 32 / units
        iw = ent.get("imad_wide_warp_per_launch")
        if iw and world == 1:  # the IMAD.WIDE the kernel executes (ncu SASS opcode counts), same peak
            out["int_executed"] = {"imad_wide_per_unit": iw * 32 / units, "achieved": iw * 32 / kernel_s / 1e12,
                                   "peak": imad_peak / 1e12, "unit": "T IMAD.WIDE/s",
                                   "frac": iw * 32 / kernel_s / imad_peak,
                                   "note": "executed IMAD.WIDE.U32 warp instructions x 32 (ncu SASS source page "
                                           "of the same-size launch) / measured peak"}
        pipes = ent.get("pipes")
        if pipes:
            busy = {k: v for k, v in pipes.items() if v is not None}
            out["binding_unit"] = max(busy, key=busy.get)
            out["ncu_pipes"] = {**pipes, "source": f"profiles/{traffic.get('round')}/ncu_{kname}.txt"}
        return out

    # ---------------------------------------------------------- config 5 headline
    n_total = args.items
    lo, hi = shard(n_total, rank, world)
    n_local = hi - lo
    zs = mb.ZipfStream(S)
    keys = torch.empty(n_local, dtype=torch.int32, device=dev)
    wts = torch.empty(n_local, dtype=torch.int32, device=dev)
    zs.generate(lo, n_local, keys, wts)
    spec = mb.SketchSpec.seeded(C5_ROWS, C5_WIDTH, 61, 32, mb.SPLIT_POW2, S)
    table = torch.zeros(C5_ROWS * C5_WIDTH, dtype=torch.int64, device=dev)
    mom = torch.empty((C5_ROWS, 4), dtype=torch.int64, device=dev)
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]

    def c5_step(i=None):
        sketch_step(mb, spec, keys, wts, table, mom, merge, None if i is None else k_ev[i])

    for _ in range(max(3, args.warmup)):
        c5_step()
    mb.hot_stats(reset=True)  # synchronizes; outside the timed region
    barrier_sync()
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mb.kernel_timer(True)  # events around cs_hot_kernel itself, recorded by the library
    with ClockSampler(local) as clk:
        t_start.record()
        for i in range(args.steps):
            c5_step(i)
        t_stop.record()
        barrier_sync()
    elapsed = max_over_ranks(t_start.elapsed_time(t_stop) / 1e3)
    # the whole scatter call (prepass + cs_hot + merge) and the dominant kernel alone
    kern = max_over_ranks(sum(a.elapsed_time(b) for a, b in k_ev) / 1e3 / args.steps)
    hot_total, hot_launches = mb.kernel_timer_read()
    mb.kernel_timer(False)
    assert hot_launches == args.steps
    hot_k = max_over_ranks(hot_total / hot_launches)
    hs = mb.hot_stats(reset=True)
    # L2 reductions per launch: every applied hot key touches the 5 rows, plus the
    # bin-table merges and the row updates that took the direct path
    c5_reds = (C5_ROWS * hs["hot_applied"] + hs["bin_merges"] + hs["direct"]) / args.steps
    moments = mb.moments_to_python(mom)
    f2 = mb.lower_median(moments)
    value = n_total * args.steps / elapsed
    clocks = clk.summary()

    line = {
        "metric": metric_name(), "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded Zipf(1.2) stream generated on device, DESIGN.md Inputs)",
        "config": {"workload": "config5_countsketch_t5_m65536_zipf1.2", "items": n_total,
                   "rows": C5_ROWS, "width": C5_WIDTH, "prime": "2^61-1", "k": 4, "split": "two-for-one pow2",
                   "weights": "int32 uniform [-100,100]", "parallelism": f"dp{world} (item shards + NCCL allreduce)",
                   "merge": merge.kind,
                   "l2": "inputs 16 GiB >> 126 MB L2 (no flush needed)"},
        # each item is C5_ROWS 4-universal hash evaluations in the reference's per-item
        # process(); here the ~89% of items that hit the shared hot-key table are summed
        # per key and hashed once per call, so this is a hash-EQUIVALENT rate (raw
        # hashing throughput: configs.c2_k4)
        "hash_equivalents_per_s": value * C5_ROWS,
        "f2_median": str(f2[0]),
        "roofline": roofline("c5", n_local, hot_k, "c5", l2_reds=c5_reds),
        "kernel_ms": hot_k * 1e3,
        "scatter_call_ms": kern * 1e3,
        "hot_path": {"miss_fraction": hs["misses"] / max(1, hs["items"]),
                     "hot_keys": hs["hot_keys"] / max(1, args.steps),
                     "l2_reds_per_item": c5_reds / max(1, n_local),
                     "binned_entries_per_item": hs["binned"] / max(1, hs["items"]),
                     "direct_row_updates": hs["direct"] / args.steps,
                     "raw_batches": hs["raw_batches"]},
        # per step: hh_probe, hh_count, hh_hist, hh_select, hh_layout, cs_hot, hh_merge, cs_moments
        # (the table zeroing is a torch fill)
        "gpu_launches": 8 * args.steps,
        "clocks": clocks,
        "peaks": {"imad_wide_per_s": imad_peak, "l2_red_per_s": red_peak, "hbm_gbs": hbm_peak,
                  "hbm_kind": peak_kind},
    }
    del keys, wts

    # ---------------------------------------------------------- e2e through the host API
    if not args.no_e2e:
        hk = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
        hw = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
        dk = torch.empty(n_local, dtype=torch.int32, device=dev)
        dw = torch.empty(n_local, dtype=torch.int32, device=dev)
        zs.generate(lo, n_local, dk, dw)
        hk.copy_(dk)
        hw.copy_(dw)
        del dk, dw
        torch.cuda.synchronize()
        sk = mb.CountSketch(C5_ROWS, C5_WIDTH, 61, 32, mb.SPLIT_POW2, S)
        hk_np, hw_np = hk.numpy(), hw.numpy()
        zeros = np.zeros(C5_ROWS * C5_WIDTH, np.int64)
        e2e_f2 = []

        def one_e2e():
            e2e_f2.append(e2e_step(sk, hk_np, hw_np, merge, zeros))

        # untimed warm-up until two consecutive steps agree within 3% (the first calls
        # size the pinned-copy pipeline; host-side transients settle), at most 8
        prev_ms = None
        for _ in range(8):
            ts = time.perf_counter()
            one_e2e()
            cur_ms = (time.perf_counter() - ts) * 1e3
            stable = prev_ms is not None and abs(cur_ms - prev_ms) <= 0.03 * prev_ms
            if world > 1:  # every rank leaves together (e2e_step holds a collective)
                flag = torch.tensor([1 if stable else 0], dtype=torch.int32, device=dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                stable = bool(flag.item())
            if stable:
                break
            prev_ms = cur_ms
        barrier_sync()
        t0 = time.perf_counter()
        # at least 10 timed host-API steps: a PCIe / host transient in one step (the
        # box's other tenants share the host) weighs less in the mean
        e2e_steps = max(10, args.steps)
        step_ms = []
        b0 = sk.h2d_bytes()
        for _ in range(e2e_steps):
            ts = time.perf_counter()
            one_e2e()
            step_ms.append((time.perf_counter() - ts) * 1e3)
        barrier_sync()
        dt = max_over_ranks(time.perf_counter() - t0)
        # bytes the library reports it moved (u32 keys + deltas narrowed to i8 when a
        # chunk fits) plus the counter reset
        h2d = (sk.h2d_bytes() - b0) // e2e_steps + C5_ROWS * C5_WIDTH * 8
        line["e2e"] = {"value": n_total * e2e_steps / dt, "unit": "updates/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": C5_ROWS * 32,
                       "h2d_bytes_api_input": n_local * 8,
                       "h2d_gbs": h2d * e2e_steps / dt / 1e9, "step_ms": step_ms,
                       "path": "mb200_sketch_process (host buffers, pinned; deltas narrowed to i8 on the host cores)"
                               + (" + mb200_sketch_allreduce" if world > 1 else "") + " + mb200_sketch_second_moment",
                       "f2_median": str(e2e_f2[-1][0]), "f2_matches_device_step": e2e_f2[-1][0] == f2[0],
                       "steps": e2e_steps}
        del sk, hk, hw

    # ---------------------------------------------------------- configs 1-4
    if not args.no_extras:
        line["configs"] = bench_extras(args, mb, torch, dist, rank, world, dev, roofline, max_over_ranks, merge)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baselines()
        cpu = cb.pop("_cpu")
        head = cb.pop("c5")
        line["cpu_baseline"] = {**head, "cpu": cpu}
        for name, ent in cb.items():
            if name in line.get("configs", {}):
                line["configs"][name]["cpu_baseline"] = ent
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def mb_sm_count(torch):
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def timed_steps(torch, steps, warmup, fn, flush=None):
    """Per-step CUDA-event timing; an L2 flush (outside the events) between steps when given."""
    for _ in range(max(3, warmup)):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b) / 1e3
    return tot / steps


def kernel_time(torch, mb, steps, warmup, fn, name=None):
    """Average duration of the dominant scatter kernel inside `fn` (a cs_update call):
    CUDA events the library records around that kernel on its own stream
    (mb200_kernel_timer), over `steps` calls after the warm-up."""
    for _ in range(max(3, warmup)):
        fn()
    torch.cuda.synchronize()
    mb.kernel_timer(True)
    for _ in range(steps):
        fn()
    total, launches = mb.kernel_timer_read()
    mb.kernel_timer(False)
    assert launches == steps, f"kernel timer saw {launches} launches of {name} for {steps} calls"
    return total / launches


def graph_step(torch, eager_fn, local_fn, tail_fn, world, name):
    """A short step replayed as one CUDA graph (launch gaps out): the rank-local part
    (zero + scatter (+ estimator at N = 1)) is captured; with N > 1 the merge and the
    estimator (`tail_fn`) follow the replay eagerly.  Eager launches if capture fails."""
    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            local_fn()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            local_fn()
        if world == 1:
            return graph.replay, True

        def step():
            graph.replay()
            tail_fn()
        return step, True
    except Exception as exc:  # eager launches when capture is unavailable
        print(f"{name}: graph capture failed ({exc}); eager", file=sys.stderr)
        return eager_fn, False


def bench_extras(args, mb, torch, dist, rank, world, dev, roofline, max_over_ranks, merge):
    out = {}
    SK = S ^ mb.SALT_KEYS
    steps = args.steps
    flushbuf = torch.empty(1 << 28, dtype=torch.uint8, device=dev)  # 256 MiB > 126 MB L2

    def flush():
        flushbuf.fill_(1)

    # config 1: CountSketch(1, 1024), 2^24 u32 keys (64 MiB < L2: flushed between steps)
    lo, hi = shard(C1_ITEMS, rank, world)
    keys = mb.gen_u32_keys(SK, lo, hi - lo)
    spec = mb.SketchSpec.seeded(1, 1024, 61, 32, mb.SPLIT_POW2, S)
    table = torch.zeros(1024, dtype=torch.int64, device=dev)
    mom = torch.empty((1, 4), dtype=torch.int64, device=dev)

    def c1():
        sketch_step(mb, spec, keys, None, table, mom, merge)

    # a ~50 us step of three launches: replayed as one CUDA graph (launch gaps out).
    # With N > 1 the graph holds the rank-local part (zero + scatter) and the merge
    # and estimator follow it eagerly.
    def c1_local():
        table.zero_()
        mb.cs_update(spec, keys, table)
        if world == 1:
            mb.cs_moments(table, 1, 1024, mom)

    step_fn, graphed = graph_step(torch, c1, c1_local, lambda: (merge.table(table), mb.cs_moments(table, 1, 1024, mom)),
                                  world, "config 1")
    t = max_over_ranks(timed_steps(torch, steps, args.warmup, step_fn, flush))
    tk = max_over_ranks(timed_steps(torch, steps, args.warmup, lambda: mb.cs_update(spec, keys, table), flush))
    out["c1"] = {"value": C1_ITEMS / t, "unit": "updates/s", "ms_per_step": t * 1e3,
                 "workload": "CountSketch(1,1024), 2^24 u32 keys, delta +1", "l2": "flushed between steps",
                 "cuda_graph": graphed, "roofline": roofline("c1", hi - lo, tk, "c1")}
    del keys

    # config 2: raw hashing, 2^28 u64 keys uniform in [0, p), k = 4 and 8
    lo, hi = shard(C2_KEYS, rank, world)
    keys, bad = mb.gen_below_p61(SK, lo, hi - lo)
    assert int(bad.item()) == 0
    outb = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    for k in (4, 8):
        coeffs = mb.draw_coeffs(61, k, S)
        t = max_over_ranks(timed_steps(torch, steps, args.warmup,
                                       lambda: mb.hash61(keys, coeffs, key_bits=64, out=outb)))
        out[f"c2_k{k}"] = {"value": C2_KEYS / t, "unit": "hashes/s", "ms_per_step": t * 1e3,
                           "workload": f"degree-{k-1} mod 2^61-1, 2^28 u64 keys in [0,p)",
                           "l2": "inputs 2 GiB > L2",
                           "evaluation": ("Horner" if k != 8 or mb.precondition61(coeffs) is None else
                                          "adapted coefficients: 5 modular products per key, same values as "
                                          "Horner's 7 (host/precond61.cpp)"),
                           "roofline": roofline(f"c2_k{k}", hi - lo, t, f"c2k{k}")}
    del keys
    # the reference's own hash benchmark setup (cli::bench_hash, bench.cpp:96-144: 32-bit keys): the
    # figure comparable with cpu_baseline.reference_bench_hash and the paper's Table 1
    keys32 = mb.gen_u32_keys(SK, lo, hi - lo)
    for k in (4, 8):
        coeffs = mb.draw_coeffs(61, k, S)
        t = max_over_ranks(timed_steps(torch, steps, args.warmup,
                                       lambda: mb.hash61(keys32, coeffs, key_bits=32, out=outb)))
        out[f"c2_k{k}"]["key32"] = {"value": C2_KEYS / t, "unit": "hashes/s", "ms_per_step": t * 1e3,
                                    "workload": f"degree-{k-1} mod 2^61-1, 2^28 u32 keys (reference bench_hash setup)",
                                    "hbm_gbs": (hi - lo) * 12 / t / 1e9}
    del keys32, outb

    # config 3: div/mod by 2^64 - 59 of 2^28 u128 inputs in [0, p^2)
    lo, hi = shard(C3_UNITS, rank, world)
    v, bad = mb.gen_pm_inputs(SK, 59, lo, hi - lo)
    assert int(bad.item()) == 0
    q = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    r = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    ovf = torch.zeros(1, dtype=torch.int64, device=dev)
    t = max_over_ranks(timed_steps(torch, steps, args.warmup, lambda: mb.pm_divmod(v, 64, 59, 3, q, r, ovf)))
    assert int(ovf.item()) == 0
    out["c3"] = {"value": C3_UNITS / t, "unit": "divmod/s", "ms_per_step": t * 1e3,
                 "workload": "Alg 4+5 by 2^64-59 (m=3), 2^28 u128 inputs in [0,p^2)", "l2": "inputs 4 GiB > L2",
                 "roofline": roofline("c3", hi - lo, t, "c3")}
    del v, q, r

    # config 4: 89-bit two-for-one, 2^26 u64 keys -> two rows of 2^16 counters
    lo, hi = shard(C4_KEYS, rank, world)
    keys = mb.gen_u64_keys(SK, lo, hi - lo)
    spec = mb.SketchSpec(2, 1 << 16, 89, [mb.draw_coeffs(89, 4, S)], 64, mb.SPLIT_TWO_FOR_ONE)
    table = torch.zeros(2 << 16, dtype=torch.int64, device=dev)
    mom = torch.empty((2, 4), dtype=torch.int64, device=dev)

    def c4():
        sketch_step(mb, spec, keys, None, table, mom, merge)

    # zero + scatter (kernel + fold) + estimator replayed as one CUDA graph, as config 1
    def c4_local():
        table.zero_()
        mb.cs_update(spec, keys, table)
        if world == 1:
            mb.cs_moments(table, 2, 1 << 16, mom)

    step_fn, graphed4 = graph_step(torch, c4, c4_local,
                                   lambda: (merge.table(table), mb.cs_moments(table, 2, 1 << 16, mom)), world,
                                   "config 4")
    t = max_over_ranks(timed_steps(torch, steps, args.warmup, step_fn))
    # the scatter kernel alone (cs_private89_kernel), on the stream it is launched on
    tk = max_over_ranks(kernel_time(torch, mb, steps, args.warmup, lambda: mb.cs_update(spec, keys, table),
                                    "cs_private89"))
    out["c4"] = {"value": C4_KEYS / t, "unit": "keys/s", "row_updates_per_s": 2 * C4_KEYS / t,
                 "ms_per_step": t * 1e3, "workload": "2^89-1 two-for-one, 2^26 u64 keys, 2 x 2^16 counters",
                 "l2": "inputs 512 MiB > L2", "kernel_ms": tk * 1e3, "cuda_graph": graphed4,
                 "roofline": roofline("c4", hi - lo, tk, "c4"),
                 "path": "cs_private89_kernel (config 4's shape: whole table per CTA in 8-bit shared cells, "
                         "per-CTA tables summed by private_fold_kernel); bound by the FMA-heavy + ALU pipes "
                         "(roofline.ncu_pipes)"}
    del keys

    # ExactDivisionMap(PseudoMersenneModulus(64, 59), r) (bucketing.cpp:75-95)
    # over 2^28 u64 values (uniform; P(v >= p) = 59 / 2^64, counted and asserted zero)
    lo, hi = shard(C2_KEYS, rank, world)
    vals = mb.gen_u64_keys(SK ^ 0xB0C, lo, hi - lo)
    outb = torch.empty_like(vals)
    ood = torch.zeros(1, dtype=torch.int64, device=dev)
    r_buckets = 1000003
    t = max_over_ranks(timed_steps(torch, steps, args.warmup, lambda: mb.bucket_map(
        mb.MAP_EXACT_DIV, vals, 64, r_buckets, 59, out=outb, out_of_domain=ood)))
    assert int(ood.item()) == 0
    out["exact_div_map"] = {"value": C2_KEYS / t, "unit": "maps/s", "ms_per_step": t * 1e3,
                            "workload": f"floor(v r / (2^64-59)), r = {r_buckets}, m = "
                                        f"{mb.exact_division_iterations(64, 59, r_buckets)}, 2^28 u64 values",
                            "l2": "inputs 2 GiB > L2", "roofline": roofline("exact_div", hi - lo, t, "exact_div")}
    del vals, outb, flushbuf

    # exhaustive moment enumeration (verify.cpp:505-603) over p^4 families,
    # the reference suite's stream {(1,2),(3,-1),(7,3)} at p = 2^8 - 1 (4.2e9 families)
    if rank == 0:
        stream = [(1, 2), (3, -1), (7, 3)]
        mb.enum_moment_sums(5, 4, mb.SPLIT_POW2, stream)  # warm-up (module load)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sums = mb.enum_moment_sums(8, 16, mb.SPLIT_POW2, stream)
        e1.record()
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3
        ent = {"value": sums["families"] / te, "unit": "families/s", "ms": te * 1e3,
               "workload": "enum_moment_sums b=8 (p=255, 255^4 families), r=16 Pow2, 3-key stream",
               "sum_x": str(sums["sum_x"]), "sum_x_sq": str(sums["sum_x_sq"])}
        try:  # cpu_baseline leg: the oracle restatement (all host threads) on p = 63 for scale
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_bind import oracle
            orc = oracle()
            t0 = time.perf_counter()
            orc.enum_moment_sums(6, 16, 0, stream)
            tc = time.perf_counter() - t0
            ent["cpu_baseline"] = {"value": 63 ** 4 / tc, "unit": "families/s", "cores": os.cpu_count(),
                                   "kind": "port", "sample": "b=6 (63^4 families), same stream, OpenMP over a0"}
        except Exception as exc:  # noqa: BLE001
            ent["cpu_baseline"] = {"unavailable": str(exc)[:200]}
        out["enum_moments"] = ent
    return out


if __name__ == "__main__":
    main()
