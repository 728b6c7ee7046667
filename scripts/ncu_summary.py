#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (committed evidence).

usage:
  scripts/ncu_summary.py full <prof.ncu-rep> [msgs_per_launch]   -> key counters of the captured kernel
  scripts/ncu_summary.py launches <launches.csv>                 -> per-kernel launch list and share
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__inst_executed.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_average_branch_targets_threads_uniform.pct",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed_pipe_cbu.sum", "sm__inst_executed_pipe_adu.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__cycles_active.sum",
]


def full(rep, msgs=None):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        name = v[hdr.index("Kernel Name")]
        out.append(f"kernel: {name}")
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = v[i]
                out.append(f"  {k:62s} {v[i]:>20s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
                try:
                    stalls.append((float(v[i].replace(",", "")), h))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            out.append("  top stall reasons (pc sampling):")
            tot = sum(s for s, _ in stalls if "pcsamp" in _) or 1
            for s, h in stalls[:10]:
                if "pcsamp" in h:
                    out.append(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):32s} {s / tot * 100:5.1f}%")
        if msgs:
            try:
                inst = float(d["smsp__inst_executed.sum"].replace(",", ""))
                out.append(f"  warp-instructions per message: {inst / msgs:.2f}")
                for pipe in ("alu", "fma", "lsu", "cbu", "adu"):
                    k = f"sm__inst_executed_pipe_{pipe}.sum"
                    if k in d:
                        out.append(f"  {pipe}-pipe warp-instructions per message: {float(d[k].replace(',', '')) / msgs:.2f}")
                rd = float(d["dram__bytes_read.sum"].replace(",", "")) * (1 if units[hdr.index("dram__bytes_read.sum")] == "byte" else 1)
                out.append(f"  (dram units: {units[hdr.index('dram__bytes_read.sum')]})")
            except (KeyError, ValueError):
                pass
    return "\n".join(out)


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) > vi:
            d.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = [f"{'kernel':70s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:70]:70s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot * 100:6.2f}%")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        print(full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None))
    else:
        print(launches(sys.argv[2]))
