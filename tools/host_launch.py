#!/usr/bin/env python
"""Host-side cost of one Scanner.launch (enqueue only, no sync): the plan +
the cooperative launch through the C ABI.  usage: python tools/host_launch.py [config]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = min(gen.config(cid)["text_len"], 1 << 26)
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
sc = pf.Scanner(pf.Trie(gen.patterns(cid)), "cuda:0", capacity=n // 256 + 4096)
sc.launch(text)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(200):
        sc.launch(text)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"C{cid}: {(t1 - t0) / 200 * 1e6:.1f} us host time per launch (enqueue)")
