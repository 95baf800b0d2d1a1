#!/usr/bin/env python
"""Summarise ncu outputs into markdown for profiles/.

  tools/ncu_summary.py launches <launches.csv>      # --metrics gpu__time_duration.sum launch list
  tools/ncu_summary.py full <report.ncu-rep>        # --set full capture (needs the ncu CLI)
"""
import collections
import csv
import io
import subprocess
import sys


def _table(text):
    rows = list(csv.reader(io.StringIO(text)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            return rows[i], rows[i + 1:]
    raise SystemExit("no ncu CSV header found")


def launches(path):
    hdr, rows = _table(open(path).read())
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows:
        if len(r) < len(hdr):
            continue
        name = r[ki].split("(")[0].replace("amppi_dev::<unnamed>::", "").replace("void ", "")
        v = float(r[vi].replace(",", "")) / 1e3  # ns -> us
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
    print(f"| kernel | launches | total µs | mean µs | share |\n|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / total:.1f}% |")


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-inst"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thread-inst"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thread-inst"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long scoreboard"),
    ("smsp__average_warp_latency_issue_stalled_wait", "stall wait"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0]
        print(f"### `{name}` grid {r[col['Grid Size']]} block {r[col['Block Size']]}\n")
        print("| metric | value |\n|---|---|")
        for m, label in METRICS:
            if m in col:
                print(f"| {label} (`{m}`) | {r[col[m]]} {units[col[m]]} |")
        def num(k):
            try:
                return float(r[col[k]].replace(",", ""))
            except (KeyError, ValueError):
                return float("nan")

        fl = (2 * num("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed")
              + num("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed")
              + num("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed"))
        hz = num("gpc__cycles_elapsed.avg.per_second")
        unit = units[col["gpc__cycles_elapsed.avg.per_second"]].lower() if "gpc__cycles_elapsed.avg.per_second" in col else ""
        hz *= 1e9 if "ghz" in unit else (1e6 if "mhz" in unit else 1.0)
        peak = 2 * num("sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained")
        if fl == fl and hz == hz:
            print(f"| executed FP32 flops (2 FFMA + FADD + FMUL) | {fl:.0f} /cycle = {fl * hz / 1e12:.2f} TFLOP/s "
                  f"= {100 * fl / peak:.1f}% of the {peak:.0f}/cycle FFMA peak |")
        scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
        def nbytes(m):  # ncu picks a unit per column
            return num(m) * scale.get(units[col[m]].lower(), float("nan")) if m in col else float("nan")
        dram = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
        print(f"| DRAM traffic read+write | {dram / 1e6:.1f} Mbyte |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
