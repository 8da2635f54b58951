#!/usr/bin/env python
"""Per-config measurement for the BASELINE.md results table: scan throughput
(bench-style: CUDA events, L2 flushed outside them, device-resident text),
KB0 read stream on the same bytes, trie image ratio, and the oracle's
throughput on the host cores (bounded sample).  Prints one JSON line per config.
usage: python tools/config_table.py [configs...]"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03657_b200 as pf  # noqa: E402

SIZES = {2: 64 << 20, 3: 1 << 30, 4: 1 << 30, 5: 1 << 30}  # per-GPU text (C4/C5: 1 GiB slices)
ENGINE = {2: "pfac", 3: "pfac", 4: "pfac", 5: "ac"}


def timed(fn, flush, reps):
    ts = []
    for i in range(reps + 2):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) / 1e3)
    return float(np.mean(ts))


kb0 = C.CDLL(os.path.join(ROOT, "tools", "probe", "libkb0.so"))
kb0.kb0_launch.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.zeros(sms * 64, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cid in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    n = SIZES[cid]
    ps = gen.patterns(cid)
    host = gen.text(cid, 0, n)
    text = torch.from_numpy(host).cuda()
    t = pf.Trie(ps)
    sc = pf.Scanner(t, "cuda:0", capacity=n // 64 + 4096)
    sc.launch(text)
    torch.cuda.synchronize()
    count = int(sc.count.item())
    reps = 50 if n <= (64 << 20) else 8
    ts = timed(lambda: sc.launch(text), flush, reps)
    stream = torch.cuda.current_stream().cuda_stream
    tk = timed(lambda: kb0.kb0_launch(text.data_ptr(), n, sink.data_ptr(), sms, stream), flush, reps)
    # oracle on the host cores: bounded sample (~8 s)
    o = oracle.Trie(ps)
    cores = os.cpu_count()
    S = 1 << 20
    t0 = time.perf_counter()
    o.match(host[:S], engine=ENGINE[cid], threads=cores)
    est = time.perf_counter() - t0
    S = int(min(n, max(S, S * 8.0 / max(est, 1e-3)))) & ~4095
    t0 = time.perf_counter()
    o.match(host[:S], engine=ENGINE[cid], threads=cores)
    to = time.perf_counter() - t0
    print(json.dumps({
        "config": f"C{cid}", "text_bytes": n, "matches": count, "us": ts * 1e6,
        "gbps": 8 * n / ts / 1e9, "frac_hbm_6536": n / ts / 6536e9, "kb0_us": tk * 1e6, "frac_kb0": tk / ts,
        "image_vs_36N": t.nbytes("device_image") / t.nbytes("uncompressed"),
        "oracle": {"gbps": 8 * S / to / 1e9, "cores": cores, "engine": ENGINE[cid], "sample_bytes": S}}), flush=True)
