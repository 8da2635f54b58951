"""Multi-GPU text sharding; one process per GPU.

Start positions are independent units: rank r owns the contiguous start range
[b_r, b_{r+1}) (4 KiB-aligned cuts) and reads a read-only halo of
(longest pattern - 1) bytes past it -- the overlap rule of PAPER.md:66 (§II-B:
"Each thread is required to overlap the next chunk of data by the length of
the longest pattern -1").  There is no exchange step in the scan itself; the
only collectives are the one-time trie-image broadcast and the gather of the
per-shard match lists, which concatenate in rank order into the globally
sorted (pos, pid) list because starts are owned exclusively.

Works with any torch.distributed backend: NCCL with CUDA tensors on the GPU
box, gloo with CPU tensors in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import Trie

ALIGN = 4096


def shard_bounds(n_text: int, world: int, rank: int, align: int = ALIGN):
    """[start, end) of the start positions rank `rank` owns (4 KiB-aligned cuts)."""
    units = (n_text + align - 1) // align
    a = min(n_text, (units * rank // world) * align)
    b = min(n_text, (units * (rank + 1) // world) * align)
    return a, b


def read_range(start: int, end: int, n_text: int, max_len: int):
    """Bytes a shard must read: its starts plus the (max_len - 1)-byte halo."""
    return start, min(n_text, end + max(0, max_len - 1))


def broadcast_trie(trie: Trie | None, src: int = 0, device: int = -1, group=None) -> Trie:
    """Rank `src` serialises its trie image; every rank returns a Trie attached
    to `device` (-1: host only).  Uses CUDA tensors when the backend is NCCL."""
    rank = dist.get_rank(group)
    use_cuda = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if use_cuda else torch.device("cpu")
    if rank == src:
        img = trie.image()
        size = torch.tensor([len(img)], dtype=torch.int64, device=dev)
    else:
        size = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.broadcast(size, src, group=group)
    n = int(size.item())
    if rank == src:
        buf = torch.frombuffer(bytearray(img), dtype=torch.uint8).to(dev)
    else:
        buf = torch.empty(n, dtype=torch.uint8, device=dev)
    dist.broadcast(buf, src, group=group)
    if rank == src and device < 0:
        return trie
    return Trie.attach(buf, device=device)


def gather_matches(pos: torch.Tensor, pid: torch.Tensor, dst: int = 0, group=None):
    """Concatenate per-rank (pos, pid) lists on `dst` in rank order (globally
    sorted because start ranges are disjoint and ordered).  Others get None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = pos.device
    n = torch.tensor([pos.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts) if counts else 0
    pad_pos = torch.zeros(m, dtype=torch.int64, device=dev)
    pad_pid = torch.zeros(m, dtype=torch.int32, device=dev)
    pad_pos[: pos.numel()] = pos
    pad_pid[: pid.numel()] = pid
    all_pos = [torch.empty(m, dtype=torch.int64, device=dev) for _ in range(world)]
    all_pid = [torch.empty(m, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(all_pos, pad_pos, group=group)
    dist.all_gather(all_pid, pad_pid, group=group)
    if rank != dst:
        return None
    return (torch.cat([p[:c] for p, c in zip(all_pos, counts)]),
            torch.cat([q[:c] for q, c in zip(all_pid, counts)]))
