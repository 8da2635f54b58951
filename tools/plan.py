#!/usr/bin/env python
"""Print the kernel's shared-memory plan for each config (PFAC_DEBUG_PLAN)."""
import os
import sys

os.environ["PFAC_DEBUG_PLAN"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

for cid in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    n = min(gen.config(cid)["text_len"], 1 << 30)
    text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
    sc = pf.Scanner(pf.Trie(gen.patterns(cid)), "cuda:0", capacity=n // 256 + 4096)
    sys.stderr.write(f"C{cid}: ")
    sc.launch(text)
    torch.cuda.synchronize()
