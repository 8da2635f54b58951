"""GPU parity: the sm_100a scan (through the C ABI) against the CPU oracle,
element by element (bit-exact: this path is integer/byte/index work).

Small cases compare full outputs; full BASELINE.json sizes (C2..C5, in the
launch configuration bench.py times) compare every row's soundness, exact
rows on oracle-computed sample windows, completeness on planted occurrences,
and global (pos, pid) order."""
import numpy as np
import pytest

import gen
import oracle
import paper_1702_03657_b200 as pf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def gpu_rows(trie, text_np, readable=None, n_starts=None, pos_base=0, offset=0, **plan):
    """Scan via the C ABI; `offset` shifts the text start inside the buffer
    to exercise unaligned device pointers; `plan` = pfac_plan_options fields."""
    buf = torch.zeros(len(text_np) + offset + 16, dtype=torch.uint8)
    buf[offset:offset + len(text_np)] = torch.from_numpy(np.array(text_np, np.uint8))
    d = buf.to(DEV)[offset:offset + len(text_np)]
    pos, pid = trie.match(d, readable_len=readable, n_starts=n_starts, pos_base=pos_base, **plan)
    return pos.cpu().numpy().astype(np.uint64), pid.cpu().numpy().astype(np.uint32)


def assert_same(a, b, what=""):
    (p1, q1), (p2, q2) = a, b
    if len(p1) != len(p2) or not np.array_equal(p1, p2) or not np.array_equal(q1, q2):
        n = min(len(p1), len(p2))
        diff = np.nonzero((p1[:n] != p2[:n]) | (q1[:n] != q2[:n]))[0]
        first = int(diff[0]) if len(diff) else n
        raise AssertionError(f"{what}: counts {len(p1)} vs {len(p2)}, first difference at row {first}")


def test_worked_examples(golden):
    for ex in golden("examples.json")["matches"]:
        t = pf.Trie([p.encode() for p in ex["patterns"]])
        text = np.frombuffer(ex["text"].encode(), np.uint8)
        if len(text) == 0:
            continue
        p, q = gpu_rows(t, text)
        assert list(zip(p.tolist(), q.tolist())) == [tuple(r) for r in ex["expect"]], ex["cite"]


def test_host_api_pfac_match(golden):
    t = pf.Trie([b"he", b"she", b"his", b"hers"])
    p, q = t.match_host(b"ushers")
    assert list(zip(p.tolist(), q.tolist())) == [(1, 1), (2, 0), (2, 3)]
    p, q = t.match_host(b"")
    assert len(p) == 0


def test_random_tiny_cases():
    rng = np.random.default_rng(2024)
    for trial in range(300):
        sigma = int(rng.choice([2, 4, 256]))
        alpha = rng.choice(256, size=sigma, replace=False)
        m = int(rng.integers(1, 51))
        pats = [bytes(alpha[rng.integers(0, sigma, int(rng.integers(1, 13)))].astype(np.uint8)) for _ in range(m)]
        if trial % 4 == 0:
            pats += [pats[0], pats[-1][:1]]
        n = int(rng.choice([1, 3, 100, 4095, 4096, 4097, 9000, 70000]))
        text = alpha[rng.integers(0, sigma, n)].astype(np.uint8)
        for _ in range(min(20, n // 8)):
            p = pats[int(rng.integers(len(pats)))]
            if len(p) <= n:
                o = int(rng.integers(0, n - len(p) + 1))
                text[o:o + len(p)] = np.frombuffer(p, np.uint8)
        want = oracle.Trie(pats).match(text)
        got = gpu_rows(pf.Trie(pats), text, offset=int(rng.integers(0, 16)))
        assert_same(got, want, f"trial {trial} sigma {sigma} n {n}")


def test_halo_and_pos_base():
    rng = np.random.default_rng(5)
    pats = [b"ab", b"abab", b"b", b"bab", b"aaa", b"ba" * 20]
    text = rng.choice(np.frombuffer(b"ab", np.uint8), size=50000).astype(np.uint8)
    o = oracle.Trie(pats)
    t = pf.Trie(pats)
    for _ in range(20):
        L = int(rng.integers(1, 50001))
        ns = int(rng.integers(0, L + 1))
        base = int(rng.integers(0, 1 << 40))
        wp, wq = o.match(text, readable_len=L, lo=0, hi=ns)
        gp, gq = gpu_rows(t, text, readable=L, n_starts=ns, pos_base=base)
        assert_same((gp, gq), (wp + np.uint64(base), wq), f"L={L} ns={ns}")


def test_sharded_equals_unsharded():
    """Shards with a (max_len-1) halo, concatenated in order == one scan."""
    ps = gen.patterns(2)
    t = pf.Trie(ps)
    text = gen.text(2, 0, 8 << 20)
    full = gpu_rows(t, text)
    halo = t.stats()["max_len"] - 1
    rng = np.random.default_rng(9)
    for G in [2, 3, 8]:
        cuts = np.sort(rng.choice(np.arange(1, len(text)), size=G - 1, replace=False))
        bounds = [0] + cuts.tolist() + [len(text)]
        P, Q = [], []
        for a, b in zip(bounds[:-1], bounds[1:]):
            e = min(len(text), b + halo)
            p, q = gpu_rows(t, text[a:e], n_starts=b - a, pos_base=a)
            P.append(p)
            Q.append(q)
        assert_same((np.concatenate(P), np.concatenate(Q)), full, f"G={G}")


def test_capacity_overflow_and_count():
    ps = [b"a", b"aa", b"aaa"]
    t = pf.Trie(ps)
    text = torch.full((10000,), ord("a"), dtype=torch.uint8, device=DEV)
    sc = pf.Scanner(t, DEV, capacity=100)
    sc.launch(text)
    torch.cuda.synchronize()
    n = int(sc.count.item())
    assert n == 10000 + 9999 + 9998
    want_p, want_q = oracle.Trie(ps).match(text.cpu().numpy())
    assert np.array_equal(sc.pos[:100].cpu().numpy().astype(np.uint64), want_p[:100])
    assert np.array_equal(sc.pid[:100].cpu().numpy().astype(np.uint32), want_q[:100])


@pytest.mark.parametrize("plan", [{}, {"ctg64": 48}, {"ctg64": 32, "pool64": 8}], ids=["auto", "ctg48", "ctg32-pool8"])
def test_round_pool_and_overflow(plan):
    """A trie too large for shared memory (C4's 100,000 patterns) plans the
    shared round pool (the text's last 1/16) and, with ctg64 < 64, dynamic
    rounds; dense 'a' runs in a CTA range and in the pool overflow the warps'
    hit lists, so the re-scan fallback runs over block, dynamic and pool
    rounds."""
    ps = gen.patterns(4).to_list() + [b"a" * k for k in range(4, 9)]
    n = 4 << 20
    text = gen.text(4, 0, n).copy()
    text[n // 3:n // 3 + (64 << 10)] = ord("a")
    text[n - (256 << 10):n - 1000] = ord("a")
    t = pf.Trie(ps)
    p = t.plan(n, **plan)
    assert p["pool_rounds"] > 0
    want = oracle.Trie(ps).match(text)
    assert_same(gpu_rows(t, text, **plan), want, "pool + overflow")
    assert_same(gpu_rows(t, text, offset=3, **plan), want, "pool + overflow, unaligned")


@pytest.mark.parametrize("kind", ["nested", "zero_bytes", "long", "len1", "len2", "dups"])
def test_adversarial(kind):
    rng = np.random.default_rng(["nested", "zero_bytes", "long", "len1", "len2", "dups"].index(kind))
    if kind == "nested":
        pats = [b"a" * k for k in range(1, 200)]
        text = np.full(20000, ord("a"), np.uint8)
        text[rng.integers(0, 20000, 50)] = ord("b")
    elif kind == "zero_bytes":
        pats = [b"\x00", b"\x00\x00\x01", b"\x01\x00", bytes(7)]
        text = rng.integers(0, 2, 30000).astype(np.uint8)
    elif kind == "long":
        pats = [bytes(rng.integers(0, 256, 5000).astype(np.uint8)), b"xyz"]
        text = rng.integers(0, 256, 100000).astype(np.uint8)
        text[777:5777] = np.frombuffer(pats[0], np.uint8)
        text[-3:] = np.frombuffer(b"xyz", np.uint8)
    elif kind == "len1":
        pats = [bytes([c]) for c in range(0, 256, 3)] + [b"\x03\x06"]
        text = rng.integers(0, 256, 50000).astype(np.uint8)
    elif kind == "len2":
        pats = [bytes(rng.integers(0, 256, 2).astype(np.uint8)) for _ in range(500)] + [b"ab", b"abc"]
        text = rng.integers(0, 256, 200000).astype(np.uint8)
    else:
        pats = [b"needle", b"needle", b"need", b"needle", b"le"]
        text = np.frombuffer(b"xxneedlexxneedneedle" * 1000, np.uint8).copy()
    want = oracle.Trie(pats).match(text)
    assert_same(gpu_rows(pf.Trie(pats), text, offset=3), want, kind)


def test_attach_from_device_image():
    ps = gen.patterns(2)
    t = pf.Trie(ps)
    img = torch.frombuffer(bytearray(t.image()), dtype=torch.uint8).to(DEV)
    t2 = pf.Trie.attach(img, device=0)
    text = gen.text(2, 0, 1 << 20)
    assert_same(gpu_rows(t2, text), gpu_rows(t, text), "attach")


def test_repeated_calls_reuse_workspace():
    """The workspace is left ready for the next call (no per-call reset by the caller)."""
    ps = gen.patterns(2)
    t = pf.Trie(ps)
    sc = pf.Scanner(t, DEV, capacity=1 << 16)
    texts = [torch.from_numpy(gen.text(2, k << 20, (k + 1) * 300000)).to(DEV) for k in range(3)]
    ref = [oracle.Trie(ps).match(x.cpu().numpy()) for x in texts]
    for rep in range(3):
        for x, (wp, wq) in zip(texts, ref):
            sc.launch(x)
            torch.cuda.synchronize()
            n = int(sc.count.item())
            assert_same((sc.pos[:n].cpu().numpy().astype(np.uint64), sc.pid[:n].cpu().numpy().astype(np.uint32)),
                        (wp, wq), f"rep {rep}")


# ---------------------------------------------------------------- full sizes
def digest(pos, pid):
    """64-bit digest of a (pos, pid) row list (reported next to the count)."""
    import hashlib
    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(pos, np.uint64).tobytes())
    h.update(np.ascontiguousarray(pid, np.uint32).tobytes())
    return h.hexdigest()


def _plants_complete(cid, ps, pos, pid, lo, hi, readable_end):
    """Every planted occurrence whose start lies in [lo, hi) and that fits
    before readable_end is in the rows (independent of the oracle)."""
    pp, pq = gen.plants(cid, lo // gen.CHUNK, (hi + gen.CHUNK - 1) // gen.CHUNK)
    keep = (pp >= lo) & (pp < hi) & (pp + ps.lens[pq] <= readable_end)
    key = pos * np.uint64(1 << 20) + pid
    want = pp[keep] * np.uint64(1 << 20) + pq[keep]
    assert np.isin(want, key).all(), "a planted occurrence is missing"


def _full_size_exact(cid, n_bytes, engine):
    """The whole text at BASELINE.json's size, in bench.py's launch
    configuration (one pfac_match_device launch over the device-resident
    text): the (pos, pid) array, its count and its digest equal the oracle's
    element by element (PAPER.md:62 problem statement; SURVEY §8(d) "full
    array compare for every config")."""
    ps = gen.patterns(cid)
    t = pf.Trie(ps)
    host = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    gen.text(cid, 0, n_bytes, out=host.numpy())
    d = host.to(DEV, non_blocking=True)
    pos, pid = t.match(d)
    del d
    pos = pos.cpu().numpy().astype(np.uint64)
    pid = pid.cpu().numpy().astype(np.uint32)
    text = host.numpy()
    want = oracle.Trie(ps).match(text, engine=engine)
    assert len(pos) == len(want[0]) and digest(pos, pid) == digest(*want), \
        f"C{cid}: count {len(pos)} vs {len(want[0])}, digest {digest(pos, pid)} vs {digest(*want)}"
    assert_same((pos, pid), want, f"C{cid} full {n_bytes} B")
    _plants_complete(cid, ps, pos, pid, 0, n_bytes, n_bytes)
    return len(pos)


@pytest.mark.parametrize("cid", [2, 3, 4, 5, 6, 7, 8])
def test_configs_unaligned_exact(cid):
    """4 MiB of each config's text at a 16-byte-unaligned device address (the
    lane-copy ring path instead of TMA for every round), every filter kind
    and ring depth, compared with the oracle element by element."""
    ps = gen.patterns(cid)
    text = gen.text(cid, 0, 4 << 20)
    want = oracle.Trie(ps).match(text)
    assert_same(gpu_rows(pf.Trie(ps), text, offset=5), want, f"C{cid} unaligned 4 MiB")


def test_dna_filter_other_bytes():
    """Kind 3 (DNA k-mer filter): bytes outside {A,C,G,T} (N, lowercase, any
    byte) alias in the 2-bit code; they may only add filter survivors, never
    drop a match.  Text = C5 text with 2% of its bytes replaced."""
    ps = gen.patterns(5)
    text = gen.text(5, 0, 2 << 20).copy()
    rng = np.random.default_rng(55)
    idx = rng.choice(len(text), len(text) // 50, replace=False)
    text[idx] = rng.choice(np.frombuffer(b"NnacgtRYK\x00\xff", np.uint8), len(idx))
    t = pf.Trie(ps)
    assert t.stats()["filter_gram"] == 16  # kind 3 in use
    want = oracle.Trie(ps).match(text)
    assert len(want[0]) > 0
    assert_same(gpu_rows(t, text), want, "C5 text with non-ACGT bytes")


def test_dna_small_set_aliasing():
    """Kind 3 with a trie small enough for shared memory: 200 k-mers (16-24
    bases); the text plants them, plants copies whose bytes are aliases of
    A/C/G/T in the 2-bit code (lowercase: same key, no match), and sprinkles
    N.  The entry table may be entered only when the 16 bytes are A/C/G/T."""
    rng = np.random.default_rng(77)
    acgt = np.frombuffer(b"ACGT", np.uint8)
    ps = [rng.choice(acgt, int(rng.integers(16, 25))).tobytes() for _ in range(200)]
    text = rng.choice(acgt, 3 << 20).astype(np.uint8)
    for k in range(4000):
        p = ps[k % len(ps)]
        o = int(rng.integers(0, len(text) - 32))
        text[o:o + len(p)] = np.frombuffer(p.lower() if k % 3 == 0 else p, np.uint8)
    text[rng.choice(len(text), 20000, replace=False)] = ord("N")
    t = pf.Trie(ps)
    assert t.stats()["filter_gram"] == 16
    want = oracle.Trie(ps).match(text)
    assert len(want[0]) > 1000
    assert_same(gpu_rows(t, text), want, "small DNA set, aliasing bytes")
    assert_same(gpu_rows(t, text, offset=7), want, "small DNA set, unaligned")


def test_full_c2_exact():
    ps = gen.patterns(2)
    n = gen.config(2)["text_len"]
    text = gen.text(2, 0, n)
    want = oracle.Trie(ps).match(text)
    got = gpu_rows(pf.Trie(ps), text)
    assert_same(got, want, "C2 full 64 MiB")


@pytest.mark.parametrize("cid,n_bytes,engine", [(3, 1 << 30, "pfac"), (4, 4 << 30, "pfac"), (5, 2 << 30, "ac"),
                                                (6, 1 << 30, "pfac"), (7, 64 << 20, "pfac"), (8, 64 << 20, "pfac")],
                         ids=["C3-1GiB", "C4-4GiB", "C5-2GiB", "C4ascii-1GiB", "C2paper-64MiB", "C2dense-64MiB"])
def test_full_size_exact(cid, n_bytes, engine):
    """C3 1 GiB, C4 4 GiB (the metric's config: 2^32 start positions in one
    launch), C5 2 GiB (its per-GPU share at G=8), 1 GiB of C4's ASCII variant
    and C2's paper-shaped and dense variants: full-array exact parity.
    The oracle engine is the PFAC walk, or for C5 the textbook Aho-Corasick
    DFA (both engines are pinned in test_oracle.py)."""
    assert _full_size_exact(cid, n_bytes, engine) > 0


def test_launch_past_4gib():
    """One launch over more than 2^32 start positions (C4 patterns on 4.25
    GiB: the cross-CTA pool is planned only up to 2^32 starts, so this runs
    the pool-less plan with 64-bit positions past 4 GiB), full-array exact."""
    ps = gen.patterns(4)
    n = (4 << 30) + (256 << 20)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    gen.text(4, 0, n, out=host.numpy())
    t = pf.Trie(ps)
    assert t.plan(n)["pool_rounds"] == 0
    pos, pid = t.match(host.to(DEV))
    got = (pos.cpu().numpy().astype(np.uint64), pid.cpu().numpy().astype(np.uint32))
    want = oracle.Trie(ps).match(host.numpy())
    assert int(want[0][-1]) >= (4 << 30)  # rows past 2^32 are checked
    assert_same(got, want, "C4 text, 4.25 GiB, one launch")


def test_full_c5_16gib_sharded():
    """C5's whole 16 GiB text as the 8 halo'd shards of the 8-GPU layout
    (multigpu.shard_bounds / read_range; PAPER.md:66 overlap rule), each
    scanned on this GPU with pos_base = its first start and compared with the
    oracle (AC engine) on exactly the bytes that shard reads.  The shards
    concatenate, in order, into the sorted result of the whole text."""
    from paper_1702_03657_b200 import multigpu
    cid, G = 5, 8
    ps = gen.patterns(cid)
    n = gen.config(cid)["text_len"]
    assert n == 16 << 30
    t = pf.Trie(ps)
    o = oracle.Trie(ps)
    sc = pf.Scanner(t, DEV, capacity=1 << 22)
    halo = t.stats()["max_len"] - 1
    total, last = 0, -1
    for g in range(G):
        a, b = multigpu.shard_bounds(n, G, g)
        r0, r1 = multigpu.read_range(a, b, n, halo + 1)
        host = torch.empty(r1 - r0, dtype=torch.uint8, pin_memory=True)
        gen.text(cid, r0, r1 - r0, out=host.numpy())
        pos, pid = sc.match(host.to(DEV), readable_len=r1 - r0, n_starts=b - a, pos_base=a)
        pos = pos.cpu().numpy().astype(np.uint64)
        pid = pid.cpu().numpy().astype(np.uint32)
        wp, wq = o.match(host.numpy(), readable_len=r1 - r0, lo=0, hi=b - a, engine="ac")
        assert_same((pos, pid), (wp + np.uint64(a), wq), f"C5 shard {g}")
        assert len(pos) == 0 or int(pos[0]) > last  # shards concatenate in position order
        last = int(pos[-1]) if len(pos) else last
        _plants_complete(cid, ps, pos, pid, a, b, r1)
        total += len(pos)
        del host
    assert total > 0


# ------------------------------------------------ host streaming pipeline
@pytest.mark.parametrize("pinned", [True, False], ids=["pinned", "pageable"])
def test_pfac_match_streaming(pinned):
    """pfac_match (host buffers) streams the text in PFAC_STREAM_CHUNK-start
    chunks with their (max_len-1)-byte halos: 200 MiB
    of C2 text = 4 chunks, with planted occurrences straddling every chunk
    boundary; equal to the oracle element by element, page-locked or not."""
    ps = gen.patterns(2)
    n = 200 << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    text = host.numpy()
    gen.text(2, 0, n, out=text)
    C = 64 << 20
    pats = ps.to_list()
    longest = max(pats, key=len)
    for k, b in enumerate(range(C, n, C)):  # a pattern across a boundary, or one ending exactly at it
        if k % 2 == 0:
            text[b - 5:b - 5 + len(longest)] = np.frombuffer(longest, np.uint8)
        else:
            text[b - len(pats[0]):b] = np.frombuffer(pats[0], np.uint8)
    t = pf.Trie(ps)
    got = t.match_host(text)
    want = oracle.Trie(ps).match(text)
    assert_same(got, want, f"streamed pfac_match ({'pinned' if pinned else 'pageable'})")
    for k, b in enumerate(range(C, n, C)):
        p0, k0 = (b - 5, pats.index(longest)) if k % 2 == 0 else (b - len(pats[0]), 0)
        assert ((got[0] == p0) & (got[1] == k0)).any()


def test_pfac_match_streaming_chunk_overflow():
    """A chunk with more rows than its planned room (dense matches in the
    first chunk) is scanned again into buffers of its size."""
    ps = [b"a", b"aa", b"xyz"]
    n = (64 << 20) + 12345
    text = np.frombuffer(gen.text(2, 0, n).tobytes(), np.uint8).copy()
    text[: 2 << 20] = ord("a")
    t = pf.Trie(ps)
    got = t.match_host(text)
    want = oracle.Trie(ps).match(text)
    assert len(want[0]) > (4 << 20)
    assert_same(got, want, "chunk overflow")


# ------------------------------------------------ truncated trie (NEXT-1)
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_truncated_trie_exact(cid):
    """The trie cut at depth d (PAPER.md:80 step III) with on-device
    verification of the patterns below each depth-d node gives the oracle's
    rows exactly (4 MiB of each config, unaligned device text)."""
    ps = gen.patterns(cid)
    n = 1024 if cid == 1 else 4 << 20
    text = gen.text(cid, 0, n)
    want = oracle.Trie(ps).match(text, engine="ac" if cid == 5 else "pfac")
    for d in [1, 2, 4, 8, 16]:
        t = pf.Trie(ps, truncate_depth=d)
        assert_same(gpu_rows(t, text, offset=3), want, f"C{cid} depth {d}")


def test_truncated_random_tiny_gpu():
    rng = np.random.default_rng(32)
    for trial in range(120):
        sigma = int(rng.choice([2, 4, 256]))
        alpha = rng.choice(256, size=sigma, replace=False)
        m = int(rng.integers(1, 40))
        pats = [bytes(alpha[rng.integers(0, sigma, int(rng.integers(1, 14)))].astype(np.uint8)) for _ in range(m)]
        if trial % 3 == 0:
            pats += [pats[0], pats[0] + pats[-1]]
        n = int(rng.choice([1, 100, 4097, 70000]))
        text = alpha[rng.integers(0, sigma, n)].astype(np.uint8)
        d = int(rng.integers(1, 10))
        want = oracle.Trie(pats).match(text)
        assert_same(gpu_rows(pf.Trie(pats, truncate_depth=d), text), want, f"trial {trial} depth {d}")


def test_truncated_c4_full_exact():
    """C4 at its full 4 GiB with the trie cut at the paper's eight levels."""
    ps = gen.patterns(4)
    n = 4 << 30
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    gen.text(4, 0, n, out=host.numpy())
    pos, pid = pf.Trie(ps, truncate_depth=8).match(host.to(DEV))
    want = oracle.Trie(ps).match(host.numpy())
    assert_same((pos.cpu().numpy().astype(np.uint64), pid.cpu().numpy().astype(np.uint32)), want, "C4 depth 8")


# ------------------------------------------- merged DAG (NEXT-2) on the GPU
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_merged_dag_scan_exact(cid):
    """The id-preserving merged DAG (PAPER.md:80 steps IV-V) scanned on the
    device (plan form PFAC_FORM_MERGED_DAG: path-rank walks) gives the
    oracle's rows exactly; the main form of the same handle too."""
    ps = gen.patterns(cid)
    n = 1024 if cid == 1 else 2 << 20
    text = gen.text(cid, 0, n)
    want = oracle.Trie(ps).match(text, engine="ac" if cid == 5 else "pfac")
    t = pf.Trie(ps, merge_suffixes=1)
    assert_same(gpu_rows(t, text, offset=1, form="merged_dag"), want, f"C{cid} merged DAG")
    assert_same(gpu_rows(t, text), want, f"C{cid} CSR form of a merged build")


def test_merged_dag_random_tiny_gpu():
    rng = np.random.default_rng(33)
    for trial in range(120):
        sigma = int(rng.choice([2, 4, 256]))
        alpha = rng.choice(256, size=sigma, replace=False)
        m = int(rng.integers(1, 40))
        pats = [bytes(alpha[rng.integers(0, sigma, int(rng.integers(1, 14)))].astype(np.uint8)) for _ in range(m)]
        if trial % 3 == 0:
            pats += [pats[0], pats[0] + pats[-1]]
        n = int(rng.choice([1, 100, 20000, 70000]))
        text = alpha[rng.integers(0, sigma, n)].astype(np.uint8)
        L = int(rng.integers(0, n + 1))
        ns = int(rng.integers(0, L + 1))
        wp, wq = oracle.Trie(pats).match(text, readable_len=L, lo=0, hi=ns)
        got = gpu_rows(pf.Trie(pats, merge_suffixes=1), text, readable=L, n_starts=ns, pos_base=7, form="merged_dag")
        assert_same(got, (wp + np.uint64(7), wq), f"trial {trial}")


# ---------------------------------------------- placements (NEXT-4 parity)
@pytest.mark.parametrize("placement", [{"placement": "global"}, {"placement": "smem"}, {"placement": "big_l1"},
                                       {"placement": "smem", "l2_persist": 1}, {"placement": "smem", "hot_bytes_cap": 4096},
                                       {"max_filter_rep_log2": 0, "ring_slots": 2}, {"stage2": 0}, {"stage2": 1}],
                         ids=["global", "smem", "big_l1", "smem-l2persist", "smem-4KiB", "rep1-slots2", "stage2-off",
                              "stage2-on"])
@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_placement_variants_exact(cid, placement):
    """Every trie placement and plan knob of the Fig. 6-style ablation
    (tools/placement.py) gives the oracle's rows:
    placement changes speed only."""
    ps = gen.patterns(cid)
    text = gen.text(cid, 0, 2 << 20)
    want = oracle.Trie(ps).match(text, engine="ac" if cid == 5 else "pfac")
    t = pf.Trie(ps)
    if cid == 5 and placement.get("stage2") == 1:
        placement = {"stage2": 0}  # (no 2-gram stage for the DNA filter)
    if cid == 4 and placement.get("stage2") == 1:
        with pytest.raises(pf.PfacError) as e:  # the 2-gram table does not fit beside C4's 128 KiB filter
            t.plan(len(text), **placement)
        assert e.value.status == 2
        return
    p = t.plan(len(text), **placement)
    if "placement" in placement and "hot_bytes_cap" not in placement:
        assert p["placement"] == pf.PLACEMENTS[placement["placement"]], p
    assert_same(gpu_rows(t, text, offset=2, **placement), want, f"C{cid} {placement}")


@pytest.mark.parametrize("cluster", [2, 4, 8])
@pytest.mark.parametrize("cid", [3, 4, 5])
def test_cluster_placement_exact(cid, cluster):
    """The cluster/DSMEM tier of the placement ablation: node
    records spread over the shared memories of a thread-block cluster, read
    by the walks through distributed shared memory, give the oracle's rows
    (a multi-round scan with a ragged tail, and a scan smaller than one
    cluster's grid)."""
    ps = gen.patterns(cid)
    t = pf.Trie(ps)
    for n in (16 << 20 | 333, 5000):
        text = gen.text(cid, 1, n)
        want = oracle.Trie(ps).match(text, engine="ac" if cid == 5 else "pfac")
        p = t.plan(len(text), placement="cluster", cluster=cluster)
        assert p["placement"] == pf.PLACEMENTS["cluster"] and p["cluster"] == cluster, p
        assert p["dsm_nodes"] > 0 and p["grid"] % cluster == 0, p
        assert_same(gpu_rows(t, text, offset=2, placement="cluster", cluster=cluster), want,
                    f"C{cid} cluster {cluster} n={n}")


def test_cluster_placement_limits():
    """Cluster placement is for the filter kinds whose tries outgrow one SM
    (1, 3, 4): the pair-filter kind is refused with LIMIT, a bad cluster size
    with INVALID_ARG."""
    t = pf.Trie(gen.patterns(2))
    with pytest.raises(pf.PfacError) as e:
        t.plan(1 << 20, placement="cluster")
    assert e.value.status == 2
    t4 = pf.Trie(gen.patterns(4))
    with pytest.raises(pf.PfacError) as e:
        t4.plan(1 << 20, placement="cluster", cluster=3)
    assert e.value.status == 1


# ------------------------------------- launch hygiene (ADVICE r1 fixes)
def test_cuda_graph_replay():
    """The scan captured once in a CUDA graph and replayed many times gives
    the same exact rows every time: the grid barrier resets itself in device
    memory (no host-side per-launch state baked into the graph)."""
    ps = gen.patterns(4)
    text = gen.text(4, 0, 8 << 20)
    want = oracle.Trie(ps).match(text)
    t = pf.Trie(ps)
    d = torch.from_numpy(text.copy()).to(DEV)
    s = torch.cuda.Stream()
    sc = pf.Scanner(t, DEV, capacity=1 << 16)
    with torch.cuda.stream(s):
        sc.launch(d)  # warm-up (allocations happen outside the capture)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sc.launch(d)
    for rep in range(6):
        sc.count.zero_()
        g.replay()
        torch.cuda.synchronize()
        n = int(sc.count.item())
        got = (sc.pos[:n].cpu().numpy().astype(np.uint64), sc.pid[:n].cpu().numpy().astype(np.uint32))
        assert_same(got, want, f"graph replay {rep}")


def test_launch_on_foreign_stream():
    """Scanner.launch(stream=s) on a stream other than the current one: the
    workspace's allocation and zero-fill are ordered before the scan."""
    ps = gen.patterns(2)
    text = gen.text(2, 0, 4 << 20)
    want = oracle.Trie(ps).match(text)
    d = torch.from_numpy(text.copy()).to(DEV)
    for _ in range(3):
        sc = pf.Scanner(pf.Trie(ps), DEV, capacity=1 << 16)
        s = torch.cuda.Stream()
        sc.launch(d, stream=s)
        s.synchronize()
        n = int(sc.count.item())
        got = (sc.pos[:n].cpu().numpy().astype(np.uint64), sc.pid[:n].cpu().numpy().astype(np.uint32))
        assert_same(got, want, "foreign stream")


def test_device_must_be_current():
    """pfac_match_device refuses a `device` that is not the current device
    (INVALID_ARG) instead of mixing contexts."""
    import ctypes as C
    t = pf.Trie([b"abc"])
    d = torch.zeros(64, dtype=torch.uint8, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    pos = torch.zeros(16, dtype=torch.int64, device=DEV)
    pid = torch.zeros(16, dtype=torch.int32, device=DEV)
    ws = torch.zeros(t.workspace_bytes(64), dtype=torch.uint8, device=DEV)
    st = pf._lib().pfac_match_device(t._h, 5, d.data_ptr(), 64, 64, 0, pos.data_ptr(), pid.data_ptr(), 16,
                                     cnt.data_ptr(), ws.data_ptr(), ws.numel(), None)
    assert st == 1
    assert b"current" in pf._lib().pfac_last_error()
