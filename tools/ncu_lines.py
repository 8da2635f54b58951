#!/usr/bin/env python
"""Summarise an ncu report's source page per CUDA source line:
warp-stall samples, warp instructions executed, top stall reasons.
usage: python tools/ncu_lines.py report.ncu-rep [top_n] [scan.cu]
(the optional source file supplies the text of scan.cu lines, when the
report's copy is not the source the binary was built from)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
def num(x):
    try:
        return int(float(x))
    except (TypeError, ValueError):
        return 0


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
        # cuda,sass layout: Line No, Source, Address, Source(sass), metrics...
        d = dict(zip(hdr[4:], r[4:]))
        d["Line No"], d["Source"] = r[0], r[1]
        rows.append((fname, d))
tot = sum(num(d.get("Warp Stall Sampling (All Samples)")) for _, d in rows) or 1
rows.sort(key=lambda x: -num(x[1].get("Warp Stall Sampling (All Samples)")))
stalls = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
print(f"total samples {tot}")
for f, d in rows[:top]:
    s = num(d.get("Warp Stall Sampling (All Samples)"))
    if s == 0:
        break
    st = sorted(((num(d.get(h)), h[6:]) for h in stalls), reverse=True)[:3]
    text = d['Source'].strip()
    if src and f == "scan.cu" and 0 < int(d['Line No']) <= len(src):
        text = src[int(d['Line No']) - 1].strip()
    print(f"{100*s/tot:5.1f}% {f}:{d['Line No']:>4} inst={d.get('Instructions Executed','')} "
          f"thr={d.get('Avg. Threads Executed','')} {st} | {text[:90]}")
