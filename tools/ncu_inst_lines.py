#!/usr/bin/env python
"""Warp instructions per source line of an ncu report, per unit (e.g. per
1024-start round): usage: python tools/ncu_inst_lines.py report.ncu-rep units [top_n] [scan.cu]
(the optional source file supplies each line's text for scan.cu lines, when
the report's copy is not the source the binary was built from)"""
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
src = open(sys.argv[4]).read().splitlines() if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
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
        try:
            n = float(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            n = 0
        if n:
            rows.append((n, fname, r[0], r[1].strip()))
tot = sum(n for n, *_ in rows)
print(f"total {tot:.4g} warp instructions = {tot / units:.1f} per unit")
rows.sort(reverse=True)
for n, f, ln, text in rows[:top]:
    if src and f == "scan.cu" and 0 < int(ln) <= len(src):
        text = src[int(ln) - 1].strip()
    print(f"{n / units:7.1f} {f}:{ln:>5} | {text[:100]}")
