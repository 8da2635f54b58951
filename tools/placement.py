#!/usr/bin/env python
"""NEXT-4: Fig. 6-style placement ablation on B200.  The paper
measured the same scan with the trie in global memory (12 Gbps) and in texture
memory with row_ptr in shared memory (22 Gbps) on a GTX 1080 (PAPER.md:121-125,
136).  Here, per config, the same kernel and inputs with each pfac_placement
(include/pfac.h; chosen through pfac_match_device_ex's plan options):
  global   - no trie level staged in shared memory (root table and level-1
             bitmaps only; nodes/labels/records via L1/L2)
  smem     - the whole trie, or its upper levels, in shared memory
  smem+L2p - smem plus the device image as an L2 persisting access window
  big_l1   - no trie level staged, 2-slot ring, one filter copy (largest L1)
  cluster2/4/8 - thread-block clusters of 2/4/8 CTAs: node records of the
             BFS prefix spread over the cluster's shared memories, read through
             distributed shared memory (kinds 1, 3, 4; C2 reports n/a)
  auto     - the planner's choice
Timing as bench.py (CUDA events, L2 flushed outside them).  One JSON line per
(config, variant), with the plan the library reports."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

VARIANTS = {"global": {"placement": "global"}, "smem": {"placement": "smem"},
            "smem+L2p": {"placement": "smem", "l2_persist": 1}, "big_l1": {"placement": "big_l1"},
            "cluster2": {"placement": "cluster", "cluster": 2}, "cluster4": {"placement": "cluster", "cluster": 4},
            "cluster8": {"placement": "cluster", "cluster": 8}, "auto": {}}
if os.environ.get("VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["VARIANTS"].split(",")}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cid in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    n = min(gen.config(cid)["text_len"], 1 << 30)
    text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
    trie = pf.Trie(gen.patterns(cid))
    reps = 100 if cid == 2 else 8
    for name, kw in VARIANTS.items():
        try:
            plan = trie.plan(n, **kw)
        except pf.PfacError as e:
            print(json.dumps({"config": f"C{cid}", "variant": name, "n": n, "unavailable": str(e)}), flush=True)
            continue
        sc = pf.Scanner(trie, "cuda:0", capacity=n // 64 + 4096, **kw)
        for _ in range(3):
            flush.fill_(1)
            sc.launch(text)
        torch.cuda.synchronize()
        ts = []
        for i in range(reps):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sc.launch(text)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = float(np.median(ts))
        print(json.dumps({"config": f"C{cid}", "variant": name, "n": n, "us": t * 1e6, "gbps": 8 * n / t / 1e9,
                          "count": int(sc.count.item()),
                          "plan": {k: plan[k] for k in ("placement", "hot_nodes", "image_nodes", "filter_copies",
                                                        "ring_slots", "smem_bytes", "grid", "cluster",
                                                        "dsm_nodes")}}), flush=True)
