"""Summarise an ncu --set full report: key throughput / pipe / stall metrics and the
source lines with the most executed instructions and stall samples."""
import csv
import io
import subprocess
import sys

WANT = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_requests_op_red.sum", "lts__t_requests_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def opcode_mix(rep):
    """Executed warp instructions per SASS mnemonic (predicate stripped), from the
    SASS source page of the report."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = next((x for x in r if x and x[0] == "Address"), None)
    if not hdr:
        return {}
    iS, iI = hdr.index("Source"), hdr.index("Instructions Executed")
    mix = {}
    for x in r:
        if len(x) <= iI or not x[0].startswith("0x"):
            continue
        toks = x[iS].split()
        if toks and toks[0].startswith("@"):
            toks = toks[1:]
        if not toks:
            continue
        try:
            n = float(x[iI])
        except ValueError:
            continue
        mix[toks[0]] = mix.get(toks[0], 0.0) + n
    return mix


def main(rep, top=12):
    h, u, rows = raw(rep)
    for v in rows:
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w} = {v[i]} {u[i]}")
        stalls = sorted(((float(v[i] or 0), h[i]) for i in range(len(h))
                         if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")),
                        reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        print("  stall mix:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {s / tot:.0%}"
                                         for s, n in stalls[:8]))
    mix = opcode_mix(rep)
    if mix:
        tot = sum(mix.values()) or 1
        print("  SASS opcode mix (warp instructions):", ", ".join(
            f"{k} {v / tot:.1%}" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:12]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = next((x for x in r if x and x[0] == "Line No"), None)
    if not hdr:
        return
    iI = hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    lines = [x for x in r if len(x) > iI and x[0].isdigit()]
    def f(s):
        try:
            return float(s)
        except ValueError:
            return 0.0
    ti = sum(f(x[iI]) for x in lines) or 1
    ts = sum(f(x[iS]) for x in lines) or 1
    print(f"  top source lines (of {ti:.3g} warp instructions):")
    for x in sorted(lines, key=lambda x: -f(x[iI]) - f(x[iS]) * ti / ts)[:top]:
        print(f"    L{x[0]:>4} inst {f(x[iI]) / ti:6.1%} stall {f(x[iS]) / ts:6.1%}  {x[1].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
