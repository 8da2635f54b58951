#!/usr/bin/env python
"""Quick timing of the scan per config (bench-style: CUDA events, L2 flushed
outside them, device-resident text) plus a 16 MiB oracle spot check.
usage: python tools/qt.py [C:MiB ...] [key=value plan options ...]
  e.g. python tools/qt.py 4:4096 2:64 3:1024 5:2048 stage2=1"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cfgs = [a for a in sys.argv[1:] if ":" in a] or ["2:64", "3:1024", "4:4096", "5:2048"]
opts = {k: (v if k == "placement" else int(v)) for k, v in (a.split("=") for a in sys.argv[1:] if "=" in a)}
BUILD = {"filter_kind", "pair_bits_per_key", "gram8_bits_per_key", "truncate_depth"}
build = {k: v for k, v in opts.items() if k in BUILD}
plan = {k: v for k, v in opts.items() if k not in BUILD}
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6450.0
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for c in cfgs:
    cid, mib = (int(x) for x in c.split(":"))
    n = mib << 20
    ps = gen.patterns(cid)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    gen.text(cid, 0, n, out=host.numpy())
    text = host.to("cuda")
    trie = pf.Trie(ps, **build)
    sc = pf.Scanner(trie, "cuda:0", capacity=max(1 << 20, n // 256), **plan)
    reps = 50 if n <= (256 << 20) else 10
    ts = []
    for i in range(reps + 3):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sc.launch(text)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) / 1e3)
    t = float(np.median(ts))
    cnt = int(sc.count.item())
    # spot parity: rows with start < 16 MiB against the oracle
    m = min(n, 16 << 20)
    gp = sc.pos[:cnt].cpu().numpy().astype(np.uint64)
    gq = sc.pid[:cnt].cpu().numpy().astype(np.uint32)
    sel = gp < m
    e = min(n, m + 127)
    wp, wq = oracle.Trie(ps).match(host.numpy()[:e], readable_len=e, lo=0, hi=m, engine="ac" if cid == 5 else "pfac")
    ok = bool(np.array_equal(gp[sel], wp) and np.array_equal(gq[sel], wq))
    print(json.dumps({"config": f"C{cid}", "mib": mib, "us": round(t * 1e6, 2), "gbps": round(8 * n / t / 1e9, 1),
                      "frac": round((n + 12 * cnt) / t / 1e9 / peak, 4), "matches": cnt, "spot_ok": ok,
                      "plan": {k: v for k, v in trie.plan(n, **plan).items() if k in ("stage2", "placement", "hot_nodes", "filter_copies", "kset", "entry")},
                      "opts": opts}), flush=True)
    del text, host, sc
    torch.cuda.empty_cache()
