#!/usr/bin/env python
"""Per-warp phase timing of the scan kernel (instrumented build).
usage: PFAC_LIB=paper_1702_03657_b200/libpfac_timing.so python tools/timing.py [config]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = gen.config(cid)["text_len"] if cid != 5 else 2 << 30
n = min(n, 1 << 30)
if len(sys.argv) > 2:
    n = int(sys.argv[2])
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
t = pf.Trie(gen.patterns(cid))
sc = pf.Scanner(t, "cuda:0", capacity=n // 256 + 4096)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = pf._lib()
lib.pfac_debug_timing.argtypes = [C.c_void_p, C.c_uint64]
buf = np.zeros(8192 * 16, dtype=np.uint64)
for rep in range(4):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(rep)
    torch.cuda.synchronize()
    sc.launch(text)
    torch.cuda.synchronize()
lib.pfac_debug_timing(buf.ctypes.data, buf.size)
b = buf.reshape(8192, 16).astype(np.int64)
used = b[:, 0] > 0
b = b[used]
t0 = b[:, 0].min()
names = ["start", "tables staged", "phase1 end", "offsets known", "end", "tables arrived", "first text in",
         "local scan done", "filter copied", "after sync", "first issued", "mbar init synced",
         "table copies issued", "-", "last round done"]
print(f"config C{cid}, {n} bytes, {used.sum()} warps; times in us relative to the first warp start")
for k, nm in enumerate(names):
    if nm == "-":
        continue
    col = (b[:, k] - t0) / 1e3
    print(f"{nm:15s} min {col.min():8.2f} med {np.median(col):8.2f} p90 {np.percentile(col, 90):8.2f} max {col.max():8.2f}")
ph1 = (b[:, 2] - b[:, 1]) / 1e3
fl = (b[:, 2] - b[:, 13]) / 1e3
print(f"final queue flush per warp: med {np.median(fl):.2f} p90 {np.percentile(fl, 90):.2f} max {fl.max():.2f} us")
print(f"phase-1 duration per warp: min {ph1.min():.2f} med {np.median(ph1):.2f} max {ph1.max():.2f} us")
# per-CTA view: is the phase-1 end spread between SMs or between warps of one SM?
W = 32
nc = len(b) // W
e = ((b[:nc * W, 2] - t0) / 1e3).reshape(nc, W)
cta_max, cta_med = e.max(1), np.median(e, 1)
print(f"per-CTA phase-1 end: max-of-CTA min {cta_max.min():.2f} med {np.median(cta_max):.2f} max {cta_max.max():.2f};"
      f" median-of-CTA min {cta_med.min():.2f} max {cta_med.max():.2f}")
print("slowest 8 CTAs (id, median, max):",
      [(int(k), round(float(cta_med[k]), 1), round(float(cta_max[k]), 1)) for k in np.argsort(-cta_max)[:8]])
out = os.environ.get("TIMING_NPY")
if out:
    np.save(out, b)
