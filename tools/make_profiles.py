"""Copy the judged evidence of one ncu round (gpurun_out/ncu_<tag>) into profiles/<tag>/:
launch list (kernel, grid, block, duration), per-config `ncu --set full` summaries, and
profiles/ncu_traffic.json (DRAM bytes per launch of each top kernel, read by bench.py).

    python tools/make_profiles.py r01e
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

KERNEL_KEY = {"c5": "cs_hot_kernel", "c1": "cs_small_k32_kernel", "c4": "cs_private89_kernel",
              "c2k4": "hash61_key64_kernel", "c2k8": "hash61_key64_kernel", "c3": "pm_divmod_kernel"}


def main(tag):
    src = os.path.join(ROOT, "gpurun_out", f"ncu_{tag}")
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    # launch list
    launches = os.path.join(src, "launches.csv")
    if os.path.exists(launches):
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        h = rows[0]
        iN, iV, iU, iG, iB = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size",
                                                    "Block Size"))
        agg = collections.OrderedDict()
        with open(os.path.join(dst, "launches.csv"), "w") as f:
            f.write("id,kernel,grid,block,duration_us\n")
            for k, r in enumerate(rows[1:]):
                v = float(r[iV].replace(",", ""))
                us = v / 1e3 if r[iU] in ("ns", "nsecond") else (v * 1e3 if r[iU] in ("ms", "msecond") else v)
                name = r[iN].split("(")[0].replace(",", ";")
                f.write(f"{k},{name},{r[iG].replace(',', ' ')},{r[iB].replace(',', ' ')},{us:.3f}\n")
                a = agg.setdefault(name, [0, 0.0])
                a[0] += 1
                a[1] += us
        tot = sum(t for _, t in agg.values())
        with open(os.path.join(dst, "launches_summary.txt"), "w") as f:
            f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
            f.write("command: python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline\n\n")
            f.write(f"{'launches':>8} {'total_us':>12} {'share':>7}  kernel\n")
            for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{c:8d} {t:12.1f} {t / tot:7.1%}  {name}\n")
    traffic = {}
    for t in ("c5", "c1", "c2k4", "c2k8", "c3", "c4"):
        rep = os.path.join(src, f"prof_{t}.ncu-rep")
        if not os.path.exists(rep):
            continue
        buf = io.StringIO()
        old = sys.stdout
        sys.stdout = buf
        try:
            ncu_summary.main(rep, 14)
        finally:
            sys.stdout = old
        with open(os.path.join(dst, f"ncu_{t}.txt"), "w") as f:
            f.write(f"ncu --set full --clock-control none --import-source on, tools/prof_target.py {t}\n")
            f.write(buf.getvalue())
        h, u, vals = ncu_summary.raw(rep)
        v = vals[0]
        rd = float(v[h.index("dram__bytes_read.sum")]) * (1e9 if u[h.index("dram__bytes_read.sum")] == "Gbyte" else
                                                           1e6 if u[h.index("dram__bytes_read.sum")] == "Mbyte" else 1)
        wr = float(v[h.index("dram__bytes_write.sum")]) * (1e9 if u[h.index("dram__bytes_write.sum")] == "Gbyte" else
                                                            1e6 if u[h.index("dram__bytes_write.sum")] == "Mbyte" else 1)
        def pct(metric):
            return float(v[h.index(metric)]) / 100.0 if metric in h else None

        inst = float(v[h.index("smsp__inst_executed.sum")].replace(",", "")) if "smsp__inst_executed.sum" in h else None
        traffic[t] = {"kernel": v[h.index("Kernel Name")].split("(")[0], "dram_bytes_per_launch": rd + wr,
                      "warp_instructions_per_launch": inst,
                      "pipes": {"alu": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                                "fma": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                                "fmaheavy": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                                "issue": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                "dram": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                                "lts": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed")}}
        mix = ncu_summary.opcode_mix(rep)
        if mix:
            traffic[t]["imad_wide_warp_per_launch"] = sum(n for k, n in mix.items() if k.startswith("IMAD.WIDE"))
            traffic[t]["opcodes_per_launch"] = dict(sorted(mix.items(), key=lambda kv: -kv[1])[:16])
    with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump({"round": tag, **traffic}, f, indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main(sys.argv[1])
