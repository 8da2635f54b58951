#!/usr/bin/env python
"""Small scans for compute-sanitizer (memcheck / racecheck / synccheck):
C1 and 1 MiB of C2..C5 through pfac_match_device (every filter kind, the
two-level probe/walk path, the pool and overflow re-scan), a truncated trie,
and the streaming pfac_match; each result checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

mib = int(os.environ.get("SAN_MIB", "1"))
ok = True
for cid, n, kw in [(1, 1024, {}), (2, mib << 20, {}), (3, mib << 20, {}), (4, mib << 20, {}), (5, mib << 20, {}),
                   (4, mib << 20, {"truncate_depth": 8}), (2, mib << 20, {"truncate_depth": 3})]:
    ps = gen.patterns(cid)
    text = gen.text(cid, 0, n)
    t = pf.Trie(ps, **kw)
    pos, pid = t.match(torch.from_numpy(text.copy()).cuda(), ctg64=32, pool64=8)
    want = oracle.Trie(ps).match(text)
    same = np.array_equal(pos.cpu().numpy().astype(np.uint64), want[0]) and \
        np.array_equal(pid.cpu().numpy().astype(np.uint32), want[1])
    print(f"C{cid} {n} {kw}: rows {len(want[0])} {'ok' if same else 'MISMATCH'}", flush=True)
    ok &= same
# dense matches: hit-list overflow -> re-scan fallback
ps = [b"a", b"aa"]
text = np.full(200000, ord("a"), np.uint8)
pos, pid = pf.Trie(ps).match(torch.from_numpy(text).cuda())
want = oracle.Trie(ps).match(text)
ok &= len(pos) == len(want[0])
print("dense overflow:", "ok" if len(pos) == len(want[0]) else "MISMATCH", flush=True)
# host streaming path (2 chunks)
ps = gen.patterns(2)
text = gen.text(2, 0, (64 << 20) + 4096)
got = pf.Trie(ps).match_host(text)
want = oracle.Trie(ps).match(text)
ok &= np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
print("streaming:", "ok" if np.array_equal(got[0], want[0]) else "MISMATCH", flush=True)
sys.exit(0 if ok else 1)
