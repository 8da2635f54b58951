#!/usr/bin/env python
"""Print the scan plan (pfac_plan_query) for each config at its bench size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

for cid in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    n = min(gen.config(cid)["text_len"], 4 << 30)
    print(json.dumps({"config": f"C{cid}", "n_starts": n, **pf.Trie(gen.patterns(cid)).plan(n)}))
