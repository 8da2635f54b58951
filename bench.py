#!/usr/bin/env python
"""bench.py -- PFAC scan throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pfac|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

A step is one pass of the whole hot path (text
streaming, per-position walk, deterministic compaction) over one batch of
synthetic input: the C2 workload (BASELINE.json configs[1]: 1,000 printable
ASCII patterns of length 4-32, 64 MiB of text) per GPU.  Multi-GPU is weak
scaling: rank r scans its own 64 MiB shard of one long text plus the
(longest-1)-byte halo of the next shard; the trie image is NCCL-broadcast once
(outside the timed region).  Text is resident in HBM before timing; L2 is
flushed (256 MiB write) before every step, outside the timed events.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the
test-infrastructure program under oracle/) on the box's host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan throughput Gbps (1/2/4/8 B200) vs HBM roofline; trie bytes vs uncompressed"
CONFIG_ID = 2
WORKLOAD = "C2: 1,000 random printable-ASCII patterns (len 4-32), 64 MiB synthetic printable-ASCII text with planted matches"
PAPER_CONTEXT = {"gbps": 22, "hw": "GTX 1080", "patterns": 1000, "text": "King James Bible", "cite": "PAPER.md:136"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="pfac", choices=["pfac", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded oracle sample (wall seconds)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    """dram bytes per launch of the scan kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get("bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


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


# ------------------------------------------------------------ reference
def run_reference(args, rank):
    """The oracle as it stands (oracle/, test infrastructure) on host cores."""
    if rank != 0:
        return
    import gen
    import oracle
    ps = gen.patterns(CONFIG_ID)
    n = gen.config(CONFIG_ID)["text_len"]
    text = gen.text(CONFIG_ID, 0, n)
    trie = oracle.Trie(ps)
    cores = os.cpu_count()
    # each step: a bounded sample of the workload (the first S bytes), sized
    # from a probe so the whole run takes about a minute
    t0 = time.perf_counter()
    trie.match(text[: 4 << 20], engine="pfac", threads=cores)
    probe = time.perf_counter() - t0
    budget = 60.0 / max(1, args.steps + args.warmup)
    S = int(min(n, max(1 << 20, (4 << 20) * budget / max(probe, 1e-6))))
    S -= S % 4096
    for _ in range(args.warmup):
        trie.match(text[:S], engine="pfac", threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        trie.match(text[:S], engine="pfac", threads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    gbps = 8.0 * S * len(times) / tot / 1e9
    sample = f"first {S} bytes of the C2 text per step (PFAC bitmap-trie walk, {cores} threads)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": "Gbps", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": WORKLOAD, "text_bytes": S, "patterns": len(ps), "parallelism": "cpu threads"},
        "cpu_baseline": {"value": gbps, "unit": "Gbps", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbps, "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def read_stream_ceiling(dev, text, flush, scan_s):
    """KB0 (tools/probe/kb0.cu): a pure 16-byte read stream, timed like the scan
    (L2 flushed outside CUDA events), on the bench's own text buffer and on a
    1 GiB buffer: the read-only ceiling next to the copy-based MEASURED_PEAKS
    figure.  Outside the scan's timed region; None if the probe is not built."""
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
    out = {}
    for name, buf in [("bench_text", text), ("1GiB", torch.ones(1 << 30, dtype=torch.uint8, device=dev))]:
        n = buf.numel() // 16 * 16
        ts = []
        for i in range(12):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            lib.kb0_launch(buf.data_ptr(), n, sink.data_ptr(), sms, stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b) / 1e3)
        t = sum(ts) / len(ts)
        out[name] = {"bytes": n, "us": 1e6 * t, "GBs": n / t / 1e9}
    out["scan_vs_kb0_same_bytes"] = out["bench_text"]["us"] / (1e6 * scan_s)
    return out


def cpu_baseline(seconds):
    """Oracle timed on a bounded sample of the same workload (rank 0, N=1)."""
    import gen
    import oracle
    ps = gen.patterns(CONFIG_ID)
    n = gen.config(CONFIG_ID)["text_len"]
    text = gen.text(CONFIG_ID, 0, n)
    trie = oracle.Trie(ps)
    cores = os.cpu_count()
    done, t_tot, reps = 0, 0.0, 0
    S = n
    t0 = time.perf_counter()
    trie.match(text[: 1 << 20], engine="pfac", threads=cores)
    est = (time.perf_counter() - t0) * (n >> 20)
    if est > seconds:
        S = max(1 << 20, int(n * seconds / est)) & ~4095
    while t_tot < seconds and reps < 1000:
        t0 = time.perf_counter()
        trie.match(text[:S], engine="pfac", threads=cores)
        t_tot += time.perf_counter() - t0
        done += S
        reps += 1
    return {"value": 8.0 * done / t_tot / 1e9, "unit": "Gbps", "cores": cores, "kind": "oracle",
            "sample": f"{reps} pass(es) over {S} bytes of the C2 text, PFAC bitmap-trie walk, {cores} threads"}


# ---------------------------------------------------------------- main
def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist

    import gen
    import paper_1702_03657_b200 as pf
    from paper_1702_03657_b200 import multigpu

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = gen.config(CONFIG_ID)
    shard = cfg["text_len"]                      # per-GPU bytes (weak scaling)
    n_total = shard * world
    ps = gen.patterns(CONFIG_ID)
    if world > 1:
        trie = multigpu.broadcast_trie(pf.Trie(ps) if rank == 0 else None, src=0, device=local_rank)
    else:
        trie = pf.Trie(ps)
    st = trie.stats()
    a, b = multigpu.shard_bounds(n_total, world, rank)
    r0, r1 = multigpu.read_range(a, b, n_total, st["max_len"])
    host = torch.empty(r1 - r0, dtype=torch.uint8, pin_memory=True)
    gen.text(CONFIG_ID, r0, r1 - r0, out=host.numpy())
    text = host.to(dev)
    n_starts = b - a

    sc = pf.Scanner(trie, dev, capacity=max(1 << 16, n_starts // 512))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        sc.launch(text, readable_len=r1 - r0, n_starts=n_starts, pos_base=a)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    count = int(sc.count.item())
    assert count <= sc.cap

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        # keep the clock sampler busy for a while before the timed steps
        t_settle = time.perf_counter()
        while time.perf_counter() - t_settle < 0.2:
            flush.fill_(2)
            step()
        for i in range(args.steps):
            flush.fill_(1)                 # L2 flush, outside the events
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [s.elapsed_time(e) for s, e in evs]          # ms, device time of each step
    t_rank = sum(per_step) / 1e3
    t = torch.tensor([t_rank], dtype=torch.float64, device=dev)
    tot_count = torch.tensor([count], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_count, op=dist.ReduceOp.SUM)
    t_max = float(t.item())
    value = 8.0 * n_total * args.steps / t_max / 1e9       # whole-job Gbps

    # roofline of the dominant (only) kernel: the step is exactly one launch
    # of pfac_scan_kernel, so its average duration is the mean step time
    kern_s = t_rank / args.steps
    alg_bytes = (r1 - r0) + 12 * count                     # text read once + output rows
    peak, peak_src = load_peaks()
    achieved = alg_bytes / kern_s / 1e9
    traffic, traffic_src = load_traffic()

    e2e = None
    if not args.no_e2e:
        # end to end through the C ABI's host call (pfac_match): pinned host
        # text -> H2D -> scan -> D2H of the sorted rows, every step
        n_e2e = min(args.steps, 20)
        trie.match_host(host.numpy()[: n_starts + 0])       # warm the cached device buffers
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(n_e2e):
            t0 = time.perf_counter()
            pos, pid = trie.match_host(host.numpy())
            ts.append(time.perf_counter() - t0)
        te = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": 8.0 * (r1 - r0) * world * n_e2e / float(te.item()) / 1e9, "unit": "Gbps",
               "h2d_bytes_per_step": int(r1 - r0), "d2h_bytes_per_step": int(8 + 12 * len(pos)),
               "api": "pfac_match (host buffers)"}

    kb0 = read_stream_ceiling(dev, text, flush, kern_s) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "Gbps", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "text_bytes_per_gpu": int(shard), "patterns": len(ps),
                       "parallelism": f"text-sharded x{world} (halo {st['max_len'] - 1} B)",
                       "l2": "flushed before every step (256 MiB write, outside the timed events)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "pfac_scan_kernel", "alg_bytes_per_launch": int(alg_bytes),
                         "peak_source": peak_src, "traffic_source": traffic_src},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": sampler.summary(),
            "gpu_launches": args.steps * pf.launches_per_call(),
            "matches": int(tot_count.item()),
            "trie_bytes": {"device_image": trie.nbytes("device_image"), "uncompressed": trie.nbytes("uncompressed"),
                           "csr_core": trie.nbytes("csr_core"), "paper_crs": trie.nbytes("paper_crs"),
                           "dense_stt": trie.nbytes("dense_stt"),
                           "image_vs_uncompressed": trie.nbytes("device_image") / trie.nbytes("uncompressed")},
            "step_ms": {"median": statistics.median(per_step), "min": min(per_step), "max": max(per_step)},
            "paper_context": PAPER_CONTEXT,
            "kb0": kb0,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
