#!/usr/bin/env python
"""Share of warp instructions / stall samples per code region of scan.cu.
usage: ncu_regions.py report  (regions from the '// ----' / '// ====' markers
and device-function boundaries in paper_1702_03657_b200/csrc/scan.cu)"""
import csv
import io
import re
import subprocess
import sys

src = open("paper_1702_03657_b200/csrc/scan.cu").read().splitlines()
marks = []
for i, l in enumerate(src, 1):
    m = re.match(r"\s*// (?:----|=+) (.*)", l)
    if m:
        marks.append((i, m.group(1).strip()[:40]))
    m = re.match(r"(?:template <.*>\s*)?__(?:device|global)__ .*?(\w+)\(", l)
    if m:
        marks.append((i, "fn " + m.group(1)))
marks.sort()


def region(line):
    r = "header"
    for i, name in marks:
        if i <= line:
            r = name
    return r


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname = None, None
agg = {}
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
        key = region(int(r[0])) if fname == "scan.cu" else fname
        a = agg.setdefault(key, [0.0, 0.0])
        try:
            a[0] += float(d.get("Instructions Executed") or 0)
            a[1] += float(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100*v[0]/ti:5.1f}% inst {100*v[1]/ts:5.1f}% stall  {k}")
