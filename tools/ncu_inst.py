#!/usr/bin/env python
"""Per-source-line instruction counts (share of warp instructions executed) and
stall samples from an ncu report.  usage: ncu_inst.py report [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, fname = [], None, None
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)))
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        rows.append((fname, int(r[0]), r[1], d))


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


ti = sum(num(d.get("Instructions Executed")) for *_, d in rows) or 1
ts = sum(num(d.get("Warp Stall Sampling (All Samples)")) for *_, d in rows) or 1
print(f"total warp inst {ti:.0f}, stall samples {ts:.0f}")
rows.sort(key=lambda x: -num(x[3].get("Instructions Executed")))
for f, l, src, d in rows[:top]:
    print(f"{100*num(d.get('Instructions Executed'))/ti:5.1f}%i {100*num(d.get('Warp Stall Sampling (All Samples)'))/ts:5.1f}%s "
          f"{f}:{l:4d} thr={d.get('Avg. Threads Executed')} | {src.strip()[:95]}")
