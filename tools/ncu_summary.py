"""Summarise one-kernel ncu --set full captures for profiles/ (developer tool).

    python tools/ncu_summary.py OUT_PREFIX BINS:REPORT.ncu-rep [...]

Writes OUT_PREFIX_<name>.txt per report (the metrics the roofline cites) and
prints a JSON dict {name: {...}} for profiles/roofline_traffic.json.
"""
import csv, io, json, subprocess, sys
from pathlib import Path

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "gpc__cycles_elapsed.max",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "not_selected",
          "barrier", "dispatch_stall", "mio_throttle", "branch_resolving", "no_instruction"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    return {k: (v, u) for k, u, v in zip(h, units, vals)}, vals[h.index("Kernel Name")]


def num(d, k):
    v = d[k][0].replace(",", "")
    return float(v) if v not in ("", "n/a", "no data") else float("nan")


def main():
    prefix = sys.argv[1]
    summary = {}
    for spec in sys.argv[2:]:
        bins_s, rep = spec.split(":", 1)
        bins = int(bins_s)
        d, kname = raw(rep)
        name = Path(rep).stem
        cyc = num(d, "gpc__cycles_elapsed.max")
        fp64_thr = sum(num(d, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                       for op in ("dadd", "dmul", "dfma")) * cyc
        # units: ncu reports time in us/ms/ns and bytes in Kbyte/Mbyte/Gbyte
        t, tu = num(d, "gpu__time_duration.sum"), d["gpu__time_duration.sum"][1]
        t_us = t * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(tu, 1.0)
        def byt(k):
            v, u = num(d, k), d[k][1]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rd, wr = byt("dram__bytes_read.sum"), byt("dram__bytes_write.sum")
        s = {"kernel": kname, "bins": bins, "time_us": t_us, "dram_read_bytes": rd,
             "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
             "dram_bytes_per_bin": (rd + wr) / bins,
             "fp64_thread_inst_per_bin": fp64_thr / bins,
             "inst_per_bin_warp_level": num(d, "smsp__inst_executed.sum") * 32 / bins,
             "fp64_pipe_active_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
             "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "registers": num(d, "launch__registers_per_thread"),
             "grid": num(d, "launch__grid_size"), "block": num(d, "launch__block_size"),
             "source": f"{Path(prefix).name}_{name}.txt"}
        stalls = {}
        for st in STALLS:
            k = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            if k in d:
                stalls[st] = num(d, k)
        s["stalls_per_issue"] = stalls
        summary[name] = s
        lines = [f"# ncu --set full --clock-control none --import-source on, one launch of {kname}",
                 f"# report: {rep}   bins per launch: {bins}"]
        for k in WANT:
            if k in d:
                lines.append(f"{k:78s} {d[k][0]:>18s} {d[k][1]}")
        # every per-pipe utilisation the capture holds (XU = MUFU / conversions,
        # FP64, FMA, ALU, LSU, ...): the roofline's "which unit is busy" evidence
        pipes = {k: num(d, k) for k in d
                 if (k.startswith("sm__inst_executed_pipe_") or k.startswith("sm__pipe_"))
                 and ".avg." in k and k.endswith("pct_of_peak_sustained_active")}
        s["pipes_pct"] = pipes
        for k in sorted(pipes):
            lines.append(f"{k:78s} {d[k][0]:>18s} {d[k][1]}")
        for st, v in stalls.items():
            lines.append(f"{'stall_' + st + ' (per issue)':78s} {v:18.3f}")
        lines.append("# derived")
        for k in ("dram_bytes_per_bin", "fp64_thread_inst_per_bin", "inst_per_bin_warp_level"):
            lines.append(f"{k:78s} {s[k]:18.3f}")
        Path(f"{prefix}_{name}.txt").write_text("\n".join(lines) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
