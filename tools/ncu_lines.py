#!/usr/bin/env python
"""Per-source-line summary of an `ncu --import-source on` capture.

  tools/ncu_lines.py <report.ncu-rep> [top [kernel-regex]]  # per source line
  tools/ncu_lines.py <report.ncu-rep> --ops [kernel-regex]  # per SASS opcode + executed FP32 flops

Reads `ncu -i ... --page source --csv --print-source cuda,sass` and prints,
per CUDA source line (file:line), the share of warp-stall samples, of warp
instructions executed, the average active threads per executed instruction
and the two largest stall reasons -- the per-line view behind profiles/.
--ops reads the SASS page instead: the opcode mix and the FP32 flops the
kernel executed (FFMA 2, FADD/FMUL 1, packed FFMA2 4, FADD2/FMUL2 2 per
predicated-on thread instruction)."""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=40, kernel=None):
    flt = ["-k", f"regex:{kernel}"] if kernel else []
    out = subprocess.run(["ncu", "-i", path] + flt + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file, hdr = None, None
    agg = collections.OrderedDict()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit() or r[2] != "-":
            continue
        col = {h: i for i, h in enumerate(hdr) if h}
        key = (cur_file, int(r[0]))
        a = agg.setdefault(key, {"src": r[1].strip()[:80], "samp": 0, "inst": 0, "thr": 0, "stall": collections.Counter()})
        num = lambda k: float(r[col[k]]) if k in col and r[col[k]] not in ("", "-") else 0.0
        a["samp"] += num("Warp Stall Sampling (All Samples)")
        a["inst"] += num("Instructions Executed")
        a["thr"] += num("Thread Instructions Executed")
        for h, i in col.items():
            if h.startswith("stall_") and r[i] not in ("", "-"):
                a["stall"][h[6:]] += float(r[i])
    ts = sum(a["samp"] for a in agg.values()) or 1
    ti = sum(a["inst"] for a in agg.values()) or 1
    tt = sum(a["thr"] for a in agg.values())
    print(f"total: {ts:.0f} stall samples, {ti:.4g} warp instructions, {tt / ti:.1f} active threads per instruction\n")
    print("| file:line | stall samples | warp inst | threads/inst | top stalls | source |\n|---|---|---|---|---|---|")
    for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1]["samp"])[:top]:
        st = ", ".join(f"{k} {100 * v / max(a['samp'], 1):.0f}%" for k, v in a["stall"].most_common(2))
        tpi = a["thr"] / a["inst"] if a["inst"] else 0.0
        print(f"| {f}:{ln} | {100 * a['samp'] / ts:.1f}% | {100 * a['inst'] / ti:.1f}% | {tpi:.1f} | {st} | "
              f"`{a['src'].replace('|', '/')}` |")


def ops(path, top=30, kernel=None):
    import re

    flt = ["-k", f"regex:{kernel}"] if kernel else []
    out = subprocess.run(["ncu", "-i", path] + flt + ["--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    col = {h: i for i, h in enumerate(hdr)}
    warp, thread = collections.Counter(), collections.Counter()
    for r in rows:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[col["Source"]])
        if not m:
            continue
        warp[m.group(2)] += float(r[col["Instructions Executed"]] or 0)
        thread[m.group(2)] += float(r[col["Predicated-On Thread Instructions Executed"]] or 0)
    tot = sum(warp.values()) or 1
    print("| opcode | share of warp instructions | warp instructions | thread instructions |\n|---|---|---|---|")
    for op, n in warp.most_common(top):
        print(f"| {op} | {100 * n / tot:.1f}% | {n:.3g} | {thread[op]:.3g} |")
    flops = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2}
    f = sum(thread[o] * k for o, k in flops.items())
    print(f"\nexecuted FP32 flops per launch (FFMA 2, FADD/FMUL 1, FFMA2 4, FADD2/FMUL2 2): {f:.4g}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "--ops":  # [kernel regex]
        ops(sys.argv[1], kernel=sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)
