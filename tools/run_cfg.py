#!/usr/bin/env python
"""Run the scan on one config (for ncu captures): python tools/run_cfg.py CID MiB [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

cid, mib = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = mib << 20
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
t = pf.Trie(gen.patterns(cid))
sc = pf.Scanner(t, "cuda:0", capacity=n // 128 + 4096)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(reps):
    ev[0].record()
    sc.launch(text)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"C{cid} {mib} MiB rep {r}: {ev[0].elapsed_time(ev[1]):.3f} ms, matches {int(sc.count.item())}")
