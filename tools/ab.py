#!/usr/bin/env python
"""A/B kernel timing (ENVS: a library name may carry +VAR=value suffixes): alternates processes running the working-tree library
(libpfac.so) and a reference build (libpfac_ref.so, tools/ab_build.sh) on one
config; bench-style timing (L2 flush outside CUDA events).
usage: python tools/ab.py [config] [rounds]"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, torch, numpy as np
sys.path.insert(0, %r)
import gen, paper_1702_03657_b200 as pf
cid = int(sys.argv[1]); n = min(gen.config(cid)["text_len"], 1 << 30)
text = torch.from_numpy(gen.text(cid, 0, n)).cuda()
sc = pf.Scanner(pf.Trie(gen.patterns(cid)), "cuda:0", capacity=n // 256 + 4096)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    flush.fill_(1); sc.launch(text)
torch.cuda.synchronize()
ev = []
for i in range(int(sys.argv[2])):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sc.launch(text); b.record(); ev.append((a, b))
torch.cuda.synchronize()
print(" ".join("%%.2f" %% (a.elapsed_time(b) * 1e3) for a, b in ev))
''' % HERE

cid = sys.argv[1] if len(sys.argv) > 1 else "2"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
libs = sys.argv[3:] or ["libpfac_ref.so", "libpfac.so"]
reps = "100" if cid == "2" else "6"
res = {lib: [] for lib in libs}
for r in range(rounds):
    for lib in libs:
        name = lib
        env = dict(os.environ, PFAC_LIB=os.path.join(HERE, "paper_1702_03657_b200", lib.split("+")[0]))
        for kv in lib.split("+")[1:]:  # lib+VAR=value: an environment variant of a library
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD, cid, reps], env=env, capture_output=True, text=True)
        if out.returncode:
            print(out.stderr[-2000:])
            sys.exit(1)
        res[name] += [float(x) for x in out.stdout.split()]
# CUDA event timestamps are quantised (~2 us steps on this box): compare means
base = np.mean(res[libs[0]])
for k in libs:
    v = np.array(res[k])
    print(f"C{cid} {k:24s}: mean {np.mean(v):8.2f} us  median {np.median(v):8.2f}  p10 {np.percentile(v, 10):8.2f}"
          f"  p90 {np.percentile(v, 90):8.2f}  (n={len(v)})  x{np.mean(v) / base:.4f}")
