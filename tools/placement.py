#!/usr/bin/env python
"""NEXT-4: Fig. 6-style placement ablation on B200.  The paper
measured the same scan with the trie in global memory (12 Gbps) and in texture
memory with row_ptr in shared memory (22 Gbps) on a GTX 1080 (PAPER.md:121-125,
136).  Here, per config, the same kernel and inputs with:
  global   - no trie level staged in shared memory (PFAC_HOT_BYTES=64: root
             table and level-1 bitmaps only; nodes/labels/records via L1/L2)
  smem     - the default plan (whole trie, or its upper levels, in shared memory)
  smem+L2p - default plus the device image as an L2 persisting access window
Timing as bench.py (CUDA events, L2 flushed outside them).  One JSON line per
(config, variant)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, torch, numpy as np
sys.path.insert(0, %r)
import gen, paper_1702_03657_b200 as pf
cid = int(sys.argv[1]); n = min(gen.config(cid)["text_len"], 1 << 30)
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
sc = pf.Scanner(pf.Trie(gen.patterns(cid)), "cuda:0", capacity=n // 64 + 4096)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.fill_(1); sc.launch(text)
torch.cuda.synchronize()
ts = []
for i in range(int(sys.argv[2])):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sc.launch(text); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
t = float(np.mean(ts))
print(json.dumps({"n": n, "us": t * 1e6, "gbps": 8 * n / t / 1e9}))
''' % ROOT

variants = {"global": {"PFAC_HOT_BYTES": "64"}, "smem": {}, "smem+L2p": {"PFAC_L2_PERSIST": "1"},
            "global+bigL1": {"PFAC_HOT_BYTES": "64", "PFAC_SLOTS2": "1", "PFAC_MAX_REP_LOG2": "0"},
            "global+L1mid": {"PFAC_HOT_BYTES": "64", "PFAC_SLOTS2": "1"}}
if os.environ.get("VARIANTS"):
    variants = {k: v for k, v in variants.items() if k in os.environ["VARIANTS"].split(",")}
for cid in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    reps = "100" if cid == 2 else "6"
    for name, env in variants.items():
        out = subprocess.run([sys.executable, "-c", CHILD, str(cid), reps], env=dict(os.environ, **env),
                             capture_output=True, text=True)
        if out.returncode:
            print(json.dumps({"config": f"C{cid}", "variant": name, "error": out.stderr[-300:]}), flush=True)
            continue
        r = json.loads(out.stdout.strip().splitlines()[-1])
        print(json.dumps({"config": f"C{cid}", "variant": name, **r}), flush=True)
