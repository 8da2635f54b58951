#!/usr/bin/env python
"""Kernel time vs text size on C2 patterns (CUDA events, L2 flushed between
launches): separates the fixed per-launch cost from the per-byte cost."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t = pf.Trie(gen.patterns(cid))
big = 256 << 20
text = torch.from_numpy(gen.text(cid, 0, big)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.zeros((), dtype=torch.int64, device="cuda")
CLEAN = os.environ.get("CLEAN_FLUSH") == "1"
sc = pf.Scanner(t, "cuda:0", capacity=big // 256 + 4096)
rows = []
for n in [1 << 10, 1 << 16, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 128 << 20, 256 << 20]:
    x = text[:n]
    ts, hs = [], []
    evs = []
    for rep in range(12):
        flush.fill_(rep)  # the GPU is busy flushing while the host enqueues the launch
        if CLEAN:
            sink.copy_(flush2.sum(dtype=torch.int64))  # read pass: the dirty lines are written back before the scan
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h0 = time.perf_counter()
        sc.launch(x)
        hs.append((time.perf_counter() - h0) * 1e6)
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1e3 for a, b in evs[2:]]
    print(f"   host launch call median {np.median(hs[2:]):.1f} us", end="")
    med = float(np.median(ts))
    rows.append((n, med))
    print(f"{n:>10d} B  {med:9.2f} us  {8 * n / med / 1e3:9.1f} Gbps", flush=True)
n = np.array([r[0] for r in rows[-4:]], float)
tt = np.array([r[1] for r in rows[-4:]])
k, c = np.polyfit(n, tt, 1)
print(f"fit over >=16 MiB: fixed {c:.2f} us + {k * (1 << 20):.3f} us/MiB -> asymptotic {8 / k / 1e3:.0f} Gbps")
