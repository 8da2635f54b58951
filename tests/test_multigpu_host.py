"""N>1 host logic on CPU with gloo, world_size 2:
shard bounds, halo rule, trie-image broadcast + attach, rank-ordered gather.
The per-shard scan is stood in for, in this test only, by the oracle run on
exactly the bytes a shard reads (the GPU kernel's sharded behaviour is
covered by tests/test_gpu_parity.py::test_sharded_equals_unsharded)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_1702_03657_b200 import Trie, multigpu


def test_shard_bounds_partition():
    for n in [0, 1, 4095, 4096, 4097, 10 ** 6, 64 << 20]:
        for world in [1, 2, 3, 4, 8]:
            prev = 0
            for r in range(world):
                a, b = multigpu.shard_bounds(n, world, r)
                assert a == prev and a <= b <= n
                assert a % multigpu.ALIGN == 0 or a == n
                prev = b
            assert prev == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_text, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = gen.patterns(2)
        trie = Trie(ps) if rank == 0 else None
        t = multigpu.broadcast_trie(trie, src=0, device=-1)
        img_ok = t.image() == Trie(ps).image()
        text = gen.text(2, 0, n_text)
        a, b = multigpu.shard_bounds(n_text, world, rank)
        r0, r1 = multigpu.read_range(a, b, n_text, t.stats()["max_len"])
        # stand-in scan of exactly the bytes this shard reads (test only)
        p, k = oracle.Trie(ps).match(text[r0:r1], readable_len=r1 - r0, lo=0, hi=b - a)
        pos = torch.from_numpy(p.astype(np.int64)) + a
        pid = torch.from_numpy(k.astype(np.int32))
        out = multigpu.gather_matches(pos, pid, dst=0)
        if rank == 0:
            full = oracle.Trie(ps).match(text)
            same = np.array_equal(out[0].numpy().astype(np.uint64), full[0]) and \
                np.array_equal(out[1].numpy().astype(np.uint32), full[1])
            q.put(("r0", img_ok, same, len(full[0])))
        else:
            q.put((f"r{rank}", img_ok, out is None, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_text", [(2, 3 * 4096 + 17), (2, 2 << 20), (3, (2 << 20) + 999)])
def test_gloo_broadcast_shard_gather(world, n_text):
    """World 2 and 3 (uneven shards and counts): broadcast, shard + halo,
    point-to-point gather to rank 0 == the unsharded oracle result."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_text, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res), "broadcast image differs"
    r0 = [r for r in res if r[0] == "r0"][0]
    assert r0[2], "gathered shards != unsharded oracle result"
    assert all(r[2] for r in res if r[0] != "r0")
