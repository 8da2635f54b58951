#!/usr/bin/env python
"""bench.py -- PFAC scan throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pfac|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload: BASELINE.json configs[3] = C4, the configuration the metric
"(1/2/4/8 B200)" is quoted on and the largest that fits one GPU: 100,000 byte
patterns of length 4-128 (uniform bytes) over 4 GiB of uniform text with
planted matches (2^32 start positions).  A step is one pass of the whole hot
path (text streaming, per-position walk, deterministic
compaction) over that text, plus, for N > 1, the gather of the sorted (pos,
pid) rows to rank 0 (a8).

N > 1 is STRONG scaling of the same 4 GiB: rank r owns a 4 KiB-aligned start
range and reads a (longest-1)-byte halo; the trie image is
NCCL-broadcast once (timed separately: `broadcast`); every step is scan +
gather (counts all-gathered, rows sent point-to-point to rank 0), timed with
CUDA events on each rank and maxed over ranks.  Rank 0 checks the count and
a 64-bit digest of the gathered rows against the CPU oracle (not timed).

Text is resident in HBM before timing and larger than L2 (4 GiB vs 126 MB);
L2 is also flushed (256 MiB write) before every step, outside the events.
Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the
test-infrastructure program under oracle/) on the box's host cores instead.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan throughput Gbps (1/2/4/8 B200) vs HBM roofline; trie bytes vs uncompressed"
CONFIG_ID = 4
WORKLOADS = {
    2: "C2: 1,000 random printable-ASCII patterns (len 4-32), 64 MiB printable-ASCII text",
    3: "C3: 10,000 Snort/ClamAV-shaped patterns (len 8-64), 1 GiB packet-like text",
    4: "C4: 100,000 random byte patterns (len 4-128), 4 GiB uniform-byte text with planted matches",
    5: "C5: 50,000 DNA k-mers (k=16-32), 2 GiB slice of the 16 GiB genome-like text (its 1-GPU share at G=8)",
    6: "C4's ASCII variant (reported, not gating): 100,000 printable patterns (len 4-128), 1 GiB slice of its "
       "4 GiB printable text",
    7: "C2's paper-shaped variant (reported): 1,000 substrings (len 4-32) of a Zipf(1.0) word text, 64 MiB",
    8: "C2's dense variant (reported): every 64-byte slot planted, 64 MiB",
}
EXTRA_BYTES = {2: 64 << 20, 3: 1 << 30, 5: 2 << 30, 6: 1 << 30, 7: 64 << 20, 8: 64 << 20}
EXTRA_NAMES = {6: "C4ascii", 7: "C2paper", 8: "C2dense"}
# --config: the headline workload (4: the metric's config; 5: C5's whole
# 16 GiB genome-like text, the SURVEY §8(e) 8-GPU configuration, strong
# scaling of the 16 GiB over --gpus N)
HEADLINE = {4: WORKLOADS[4],
            5: "C5: 50,000 DNA k-mers (k=16-32), 16 GiB genome-like text (the 8-GPU configuration)"}
ORACLE_ENGINE = {4: "pfac", 5: "ac"}  # C5: the AC engine (the bitmap-trie walk is ~4x slower on DNA)
PAPER_CONTEXT = {"gbps": 22, "hw": "GTX 1080", "patterns": 1000, "text": "King James Bible", "cite": "PAPER.md:136"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pfac", choices=["pfac", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[4, 5],
                    help="4: C4 4 GiB (default, the metric's config); 5: C5's whole 16 GiB")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip rank 0's oracle count/digest check")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2/C3/C5 side lines (N=1)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded oracle sample (wall seconds)")
    ap.add_argument("--ref-seconds", type=float, default=45.0,
                    help="--impl reference: oracle seconds over all steps (each step a bounded sample)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(cid):
    """dram bytes per launch of the scan kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        d = d.get(f"C{cid}", {})
        return d.get("bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


def digest(pos, pid):
    import numpy as np
    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(pos, np.uint64).tobytes())
    h.update(np.ascontiguousarray(pid, np.uint32).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """NVML samples of the SM clock and throttle reasons while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU oracle
def oracle_sample_gbps(otrie, cid, seconds, reps_cap=1000, engine="pfac"):
    """The oracle as it stands (PFAC bitmap-trie walk, all host threads) on a
    bounded prefix of config cid's text: (Gbps, bytes per pass, passes)."""
    import gen
    cores = os.cpu_count()
    n = gen.config(cid)["text_len"]
    probe = 16 << 20
    text = gen.text(cid, 0, probe + 4096)
    t0 = time.perf_counter()
    otrie.match(text[:probe + 127], readable_len=probe + 127, lo=0, hi=probe, engine=engine, threads=cores)
    est = (time.perf_counter() - t0) / probe  # s per byte
    S = int(min(n - 4096, max(probe, seconds / max(est, 1e-12))))
    S -= S % 4096
    if S > probe:
        text = gen.text(cid, 0, S + 4096)
    done, t_tot, reps = 0, 0.0, 0
    while t_tot < seconds and reps < reps_cap:
        t0 = time.perf_counter()
        otrie.match(text[:S + 127], readable_len=S + 127, lo=0, hi=S, engine=engine, threads=cores)
        t_tot += time.perf_counter() - t0
        done += S
        reps += 1
    return 8.0 * done / t_tot / 1e9, S, reps, t_tot


def oracle_engines(otrie_h, cid_h, seconds=2.0):
    """Context beside cpu_baseline (SURVEY §8(d) "oracle beside it"): both CPU
    engines -- "CPU PFAC" (the paper's walk over the uncompressed bitmap trie)
    and "CPU Aho-Corasick" (the textbook DFA, the best serial algorithm) -- on
    16 MiB of the headline config (otrie_h = its oracle trie) with every host
    thread, and single-threaded on C1 and on 4 MiB of C2.  Gbps over the sample; each timing repeats the match until
    about `seconds` have passed."""
    import gen
    import oracle
    cores = os.cpu_count()

    def rate(ot, text, n, engine, threads):
        ot.match(text[:1 << 16], readable_len=min(len(text), 1 << 16), lo=0, hi=min(n, 1 << 16), engine=engine,
                 threads=threads)  # (untimed: lazy per-engine tables)
        t_tot, done = 0.0, 0
        while t_tot < seconds:
            t0 = time.perf_counter()
            ot.match(text, readable_len=len(text), lo=0, hi=n, engine=engine, threads=threads)
            t_tot += time.perf_counter() - t0
            done += n
        return round(8.0 * done / t_tot / 1e9, 4)

    out = {}
    th = gen.text(cid_h, 0, 16 << 20)
    for eng in ("pfac", "ac"):
        try:
            out[f"C{cid_h}_16MiB_{eng}_{cores}t"] = rate(otrie_h, th, len(th), eng, cores)
        except oracle.OracleError as e:  # C4's DFA (6.4 M states x 256) exceeds the oracle's size limit
            out[f"C{cid_h}_16MiB_{eng}_{cores}t"] = f"unavailable ({e})"
    for cid, nbytes in ((1, None), (2, 4 << 20)):
        ot = oracle.Trie(gen.patterns(cid))
        tx = gen.text(cid, 0, nbytes or gen.config(cid)["text_len"])
        for eng in ("pfac", "ac"):
            out[f"C{cid}_{eng}_1t"] = rate(ot, tx, len(tx), eng, 1)
    out["unit"] = "Gbps"
    return out


def run_reference(args, rank):
    """`--impl reference`: the oracle as it stands (oracle/, test
    infrastructure) on the box's host cores, same metric and config; each step
    a bounded sample (a prefix of the C4 text) sized so the run takes about a
    minute.  Under torchrun only rank 0 runs it."""
    if rank != 0:
        return
    import gen
    import oracle
    cid = args.config
    eng = ORACLE_ENGINE[cid]
    ps = gen.patterns(cid)
    otrie = oracle.Trie(ps)
    cores = os.cpu_count()
    per_step = args.ref_seconds / max(1, args.steps + args.warmup)
    _, S, _, _ = oracle_sample_gbps(otrie, cid, per_step, reps_cap=1, engine=eng)
    text = gen.text(cid, 0, S + 4096)
    for _ in range(args.warmup):
        otrie.match(text[:S + 127], readable_len=S + 127, lo=0, hi=S, engine=eng, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        otrie.match(text[:S + 127], readable_len=S + 127, lo=0, hi=S, engine=eng, threads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    gbps = 8.0 * S * len(times) / tot / 1e9
    sample = (f"first {S} start positions of the C{cid} text per step "
              f"({'PFAC bitmap-trie walk' if eng == 'pfac' else 'Aho-Corasick DFA'}, {cores} threads)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": "Gbps", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": HEADLINE[cid], "text_bytes": S, "patterns": len(ps),
                   "parallelism": "cpu threads"},
        "cpu_baseline": {"value": gbps, "unit": "Gbps", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbps, "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------- probes
def read_stream_ceiling(dev, text, flush, scan_s):
    """KB0 (tools/probe/kb0.cu): a pure 16-byte read stream, timed like the scan
    (L2 flushed outside CUDA events), on the bench's own text buffer: the
    read-only ceiling next to the copy-based MEASURED_PEAKS figure.  Outside
    the scan's timed region; None if the probe is not built."""
    import ctypes as C

    import torch
    lib_path = os.path.join(ROOT, "tools", "probe", "libkb0.so")
    if not os.path.exists(lib_path):
        return None
    lib = C.CDLL(lib_path)
    lib.kb0_launch.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.zeros(sms * 4 * 16, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    n = text.numel() // 16 * 16
    ts = []
    for i in range(8):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lib.kb0_launch(text.data_ptr(), n, sink.data_ptr(), sms, stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) / 1e3)
    t = sum(ts) / len(ts)
    return {"bytes": n, "us": 1e6 * t, "GBs": n / t / 1e9, "scan_vs_kb0_same_bytes": t / scan_s}


def time_launches(sc, text, flush, n, reps, stream):
    """Median/mean device time of `reps` single-launch scans (L2 flushed)."""
    import torch
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sc.launch(text, readable_len=n)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts), sum(ts) / len(ts)


STAGE_KINDS = ["uncompressed", "pipe_trunc", "pipe_merged", "pipe_crs", "paper_crs", "merged", "merged_image",
               "csr_core", "device_image"]


def byte_stages(ps):
    """Fig. 5-style per-stage trie bytes (PAPER.md:80 steps I-V)
    from a build with merge_suffixes: the paper's pipeline (36 B/node trie ->
    cut at 8 levels -> merged -> N x 9 CRS) next to this library's exact forms."""
    import paper_1702_03657_b200 as pf
    t = pf.Trie(ps, merge_suffixes=1)
    b = {k: t.nbytes(k) for k in STAGE_KINDS if k != "device_image"}
    b["device_image"] = pf.Trie(ps).nbytes("device_image")  # the product build (no DAG sections)
    b["pipe_crs_vs_uncompressed"] = b["pipe_crs"] / b["uncompressed"]
    b["device_image_vs_uncompressed"] = b["device_image"] / b["uncompressed"]
    return b


def extra_configs(dev, flush, peak, stream):
    """C2, C3, C5 (1-GPU sizes) and the reported variants (C4 ASCII, C2
    paper-shaped and dense) timed like the headline: side lines only."""
    import torch

    import gen
    import paper_1702_03657_b200 as pf
    out = {}
    for cid, n in EXTRA_BYTES.items():
        ps = gen.patterns(cid)
        trie = pf.Trie(ps)
        host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        gen.text(cid, 0, n, out=host.numpy())
        text = host.to(dev)
        sc = pf.Scanner(trie, dev, capacity=max(1 << 16, n // 256))
        time_launches(sc, text, flush, n, 3, stream)
        med, mean = time_launches(sc, text, flush, n, 30 if n <= (64 << 20) else 10, stream)
        cnt = int(sc.count.item())
        out[EXTRA_NAMES.get(cid, f"C{cid}")] = {"workload": WORKLOADS[cid], "text_bytes": n, "us_median": 1e6 * med,
                          "gbps": 8.0 * n / med / 1e9, "hbm_frac": (n + 12 * cnt) / med / 1e9 / peak,
                          "matches": cnt,
                          "trie_image_vs_uncompressed": trie.nbytes("device_image") / trie.nbytes("uncompressed"),
                          "trie_bytes_stages": byte_stages(ps)}
        del text, host, sc
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- main
def main():
    args = parse()
    global CONFIG_ID
    CONFIG_ID = args.config
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    import paper_1702_03657_b200 as pf
    from paper_1702_03657_b200 import multigpu

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)

    cfg = gen.config(CONFIG_ID)
    n_total = cfg["text_len"]                   # 4 GiB, split across ranks (strong scaling)
    ps = gen.patterns(CONFIG_ID)
    broadcast = None
    if world > 1:
        trie0 = pf.Trie(ps) if rank == 0 else None
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        trie = multigpu.broadcast_trie(trie0, src=0, device=local_rank)
        torch.cuda.synchronize()
        bt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(bt, op=dist.ReduceOp.MAX)
        broadcast = {"us": 1e6 * float(bt.item()), "image_bytes": trie.nbytes("device_image"),
                     "what": "NCCL broadcast of the trie image + pfac_attach upload (one-time, not in value)"}
    else:
        trie = pf.Trie(ps)
    st = trie.stats()
    a, b = multigpu.shard_bounds(n_total, world, rank)
    r0, r1 = multigpu.read_range(a, b, n_total, st["max_len"])
    host = torch.empty(r1 - r0, dtype=torch.uint8, pin_memory=True)
    gen.text(CONFIG_ID, r0, r1 - r0, out=host.numpy())
    text = host.to(dev)
    n_starts = b - a

    sc = pf.Scanner(trie, dev, capacity=max(1 << 20, n_starts // 2048))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    gpos = gpid = None

    def scan():
        sc.launch(text, readable_len=r1 - r0, n_starts=n_starts, pos_base=a)

    def gather():
        nonlocal gpos, gpid
        n = int(sc.count.item())
        res = multigpu.gather_matches(sc.pos[:n], sc.pid[:n], dst=0, out=(gpos, gpid) if gpos is not None else None)
        if res is not None:
            gpos, gpid = res
        return res

    for _ in range(max(3, args.warmup)):
        flush.fill_(1)
        scan()
        if world > 1:
            gather()
    torch.cuda.synchronize()
    count = int(sc.count.item())
    assert count <= sc.cap, "capacity"

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        t_settle = time.perf_counter()
        while time.perf_counter() - t_settle < 0.2:  # let the clock sampler see load first
            flush.fill_(2)
            scan()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(args.steps):
            flush.fill_(1)                 # L2 flush, outside the events
            ev[i][0].record(stream)
            scan()
            ev[i][1].record(stream)
            if world > 1:
                gather()
            ev[i][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, _, e in ev]         # device time of each step
    kern_ms = [s.elapsed_time(k) for s, k, _ in ev]         # the scan launch alone
    t_rank = sum(step_ms) / 1e3
    t = torch.tensor([t_rank], dtype=torch.float64, device=dev)
    tot_count = torch.tensor([count], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_count, op=dist.ReduceOp.SUM)
    t_max = float(t.item())
    value = 8.0 * n_total * args.steps / t_max / 1e9       # whole-job Gbps (all ranks' starts)

    # roofline of the dominant (only) kernel of this rank: one scan launch
    kern_s = sum(kern_ms) / len(kern_ms) / 1e3
    alg_bytes = (r1 - r0) + 12 * count                     # text read once + 12 B per output row
    peak, peak_src = load_peaks()
    achieved = alg_bytes / kern_s / 1e9
    traffic, traffic_src = load_traffic(CONFIG_ID)
    if traffic is not None and world > 1:
        traffic = None  # the committed capture is of the 1-GPU launch
        traffic_src = None

    verify = None  # rank 0: count + digest of the rows (the last step's gather for N > 1) vs the oracle
    otrie = None
    if rank == 0 and not args.no_verify:
        import oracle
        otrie = oracle.Trie(ps)
        if world == 1:
            gp, gq = sc.pos[:count].cpu().numpy().astype(np.uint64), sc.pid[:count].cpu().numpy().astype(np.uint32)
        else:
            gp, gq = gpos.cpu().numpy().astype(np.uint64), gpid.cpu().numpy().astype(np.uint32)
        full = host.numpy() if world == 1 else gen.text(CONFIG_ID, 0, n_total)
        t0 = time.perf_counter()
        wp, wq = otrie.match(full, engine=ORACLE_ENGINE[CONFIG_ID], threads=os.cpu_count())
        verify = {"rows": int(len(gp)), "digest": digest(gp, gq), "oracle_rows": int(len(wp)),
                  "oracle_digest": digest(wp, wq),
                  "equal": bool(len(gp) == len(wp) and np.array_equal(gp, wp) and np.array_equal(gq, wq)),
                  "oracle_s": time.perf_counter() - t0}
        del full

    e2e = None
    if not args.no_e2e:
        # end to end through the C ABI's host call (pfac_match): pinned host
        # text -> H2D -> scan -> D2H of the sorted rows, every step (N > 1:
        # each rank's own shard; the rank-0 gather is not part of it)
        n_e2e = min(args.steps, 5)
        hv = host.numpy()
        trie.match_host(hv)                                   # warm the cached device buffers
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts, rows = [], 0
        for _ in range(n_e2e):
            t0 = time.perf_counter()
            pos, pid = trie.match_host(hv)
            ts.append(time.perf_counter() - t0)
            rows = len(pos)
        te = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": 8.0 * n_total * n_e2e / float(te.item()) / 1e9, "unit": "Gbps",
               "h2d_bytes_per_step": int(r1 - r0), "d2h_bytes_per_step": int(8 + 12 * rows),
               "api": "pfac_match (host buffers, pinned)" + (" per rank, no gather" if world > 1 else "")}

    kb0 = read_stream_ceiling(dev, text, flush, kern_s) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        otrie = otrie or oracle.Trie(ps)
        eng = ORACLE_ENGINE[CONFIG_ID]
        g, S, reps, tt = oracle_sample_gbps(otrie, CONFIG_ID, args.cpu_seconds, engine=eng)
        cpu = {"value": g, "unit": "Gbps", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{reps} pass(es) over the first {S} start positions of the C{CONFIG_ID} text "
                         f"({'PFAC bitmap-trie walk' if eng == 'pfac' else 'Aho-Corasick DFA'}, "
                         f"{os.cpu_count()} threads, {tt:.1f} s)",
               "engines": oracle_engines(otrie, CONFIG_ID)}

    variants = None  # the C4 launch with the trie cut at 8 levels (NEXT-1) and as the merged DAG (NEXT-2)
    if rank == 0 and world == 1 and not args.no_extras and CONFIG_ID == 4:
        variants = {}
        for name, bkw, pkw in [("truncated_depth8", {"truncate_depth": 8}, {}),
                               ("merged_dag", {"merge_suffixes": 1}, {"form": "merged_dag"})]:
            tv = pf.Trie(ps, **bkw)
            sv = pf.Scanner(tv, dev, capacity=max(1 << 20, n_starts // 2048), **pkw)
            med, _ = time_launches(sv, text, flush, r1 - r0, 5, stream)
            variants[name] = {"us_median": 1e6 * med, "gbps": 8.0 * n_starts / med / 1e9,
                              "matches": int(sv.count.item()), "equal_count": int(sv.count.item()) == count,
                              "trie_bytes": {k: tv.nbytes(k) for k in ("truncated", "device_image")
                                             if k != "truncated" or bkw.get("truncate_depth")}}
            del sv, tv
    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        del text
        torch.cuda.empty_cache()
        extras = extra_configs(dev, flush, peak, stream)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "Gbps", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": HEADLINE[CONFIG_ID], "text_bytes": int(n_total), "patterns": len(ps),
                       "parallelism": f"text-sharded x{world} (4 KiB-aligned starts, halo {st['max_len'] - 1} B)"
                                      + (", rank-0 gather in every step" if world > 1 else ""),
                       "l2": f"text {n_total >> 30} GiB > L2; also flushed before every step (256 MiB write, outside the events)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "pfac_scan_kernel", "alg_bytes_per_launch": int(alg_bytes),
                         "kernel_us": 1e6 * kern_s, "peak_source": peak_src, "traffic_source": traffic_src},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": sampler.summary(),
            "gpu_launches": args.steps * pf.launches_per_call(),
            "matches": int(tot_count.item()),
            "verify": verify,
            "broadcast": broadcast,
            "trie_bytes": {"device_image": trie.nbytes("device_image"), "uncompressed": trie.nbytes("uncompressed"),
                           "csr_core": trie.nbytes("csr_core"), "paper_crs": trie.nbytes("paper_crs"),
                           "dense_stt": trie.nbytes("dense_stt"),
                           "image_vs_uncompressed": trie.nbytes("device_image") / trie.nbytes("uncompressed"),
                           "stages": byte_stages(ps) if rank == 0 else None},
            "variants": variants,
            "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
            "plan": trie.plan(n_starts, local_rank),
            "paper_context": PAPER_CONTEXT,
            "kb0": kb0,
            "extra_configs": extras,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
