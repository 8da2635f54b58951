#!/usr/bin/env python
"""Per-CTA-range content of a config's text: match rows per CTA range and, for
the timing build, the per-CTA phase-1 end next to it (is a slow CTA's range
richer in matches?).  usage: python tools/cta_hist.py [config] [grid]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 148
n = min(gen.config(cid)["text_len"], 1 << 30)
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
sc = pf.Scanner(pf.Trie(gen.patterns(cid)), "cuda:0", capacity=n // 256 + 4096)
pos, pid = sc.match(text)
rounds = (n + 1023) // 1024
rpc = (rounds + grid - 1) // grid
cta = (pos.cpu().numpy() // 1024) // rpc
h = np.bincount(cta, minlength=grid)
print(f"C{cid}: {len(pos)} rows; per-CTA rows min {h.min()} med {int(np.median(h))} max {h.max()}")
print("first 12 CTAs:", h[:12].tolist())
print("top 8 CTAs:", [(int(k), int(h[k])) for k in np.argsort(-h)[:8]])
# distinct positions per CTA (walks that hit)
up = np.unique(pos.cpu().numpy())
hu = np.bincount((up // 1024) // rpc, minlength=grid)
print(f"distinct hit positions per CTA: min {hu.min()} med {int(np.median(hu))} max {hu.max()}; first 12: {hu[:12].tolist()}")
