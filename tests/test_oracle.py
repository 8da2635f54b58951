"""Pins for the CPU oracle -- no GPU needed.

The oracle (oracle/) is pinned here to things other than itself: hand-derived
arrays of the toy trie (P1), textbook / SPEC worked examples (P2-P4), closed
forms (P6), an independent numpy brute force on random tiny inputs (P7), and
invariants on generated full-shape inputs (P8).  Cross-engine agreement (PFAC
bitmap walk == own CSR walk == Aho-Corasick DFA == memcmp brute force) is the
"compressed == uncompressed" invariant of BASELINE.json's north star.
"""
import numpy as np
import pytest

import gen
import oracle


def numpy_brute(patterns, text, lo=0, hi=None, readable=None):
    """Plain definition M = {(i,k): T[i:i+|P_k|] == P_k}, numpy,
    independent of the C oracle."""
    t = np.frombuffer(bytes(text), np.uint8) if not isinstance(text, np.ndarray) else text
    L = len(t) if readable is None else readable
    t = t[:L]
    hi = L if hi is None else min(hi, L)
    rows = []
    for k, p in enumerate(patterns):
        p = np.frombuffer(bytes(p), np.uint8)
        if len(p) > L:
            continue
        w = np.lib.stride_tricks.sliding_window_view(t, len(p))
        hit = np.nonzero((w == p).all(axis=1))[0]
        hit = hit[(hit >= lo) & (hit < hi)]
        rows.extend((int(i), k) for i in hit)
    rows.sort()
    return rows


# ----------------------------------------------------------------- P9 RNG
def test_rng_pins(golden):
    g = golden("rng.json")
    assert gen.mt64_outputs(g["mt19937_64_seed"], 10000)[-1] == g["mt19937_64_10000th"]
    assert [hex(x) for x in gen.splitmix64_outputs(0, 2)] == g["splitmix64_state0"]


# ----------------------------------------------------------------- P1 toy
def test_toy_trie_arrays(golden):
    g = golden("toy_trie.json")
    t = oracle.Trie([p.encode() for p in g["patterns"]])
    st = t.stats()
    assert st["nodes"] == g["nodes"] and st["edges"] == g["edges"]
    for v in range(g["nodes"]):
        bm, off = t.node(v)
        assert bm[3] == g["node_bitmap_word3"][v], v
        assert [w for i, w in enumerate(bm) if i != 3] == [0] * 7
        assert off == g["node_offset"][v], v
        assert t.node_pids(v) == g["terminals"].get(str(v), [])
    row_ptr, labels, child = t.csr()
    assert row_ptr == g["csr_row_ptr"]
    assert labels == g["csr_labels"].encode()
    assert child == g["csr_child"]
    assert t.bytes("uncompressed") == g["bytes_uncompressed"]
    assert t.bytes("dense_stt") == g["bytes_dense_stt"]
    val, col, rp = t.paper_crs()
    assert val == g["paper_crs_val"] and col == g["paper_crs_col_ind"] and rp == g["paper_crs_row_ptr"]
    assert len(val) == g["paper_crs_nnz"]
    # P5: the CRS storage cost 2nnz+n+1 is the element count
    assert len(val) + len(col) + len(rp) == g["paper_crs_elements"]
    assert t.bytes("paper_crs") == 4 * g["paper_crs_elements"]


# ------------------------------------------------------------ P2/P3 examples
@pytest.mark.parametrize("engine", ["pfac", "csr", "brute", "ac"])
def test_worked_examples(golden, engine):
    for ex in golden("examples.json")["matches"]:
        t = oracle.Trie([p.encode() for p in ex["patterns"]])
        got = t.match_list(ex["text"].encode(), engine=engine)
        assert got == [tuple(r) for r in ex["expect"]], ex["cite"]


# ------------------------------------------------------------- P4 shapes
def test_shapes_and_rank(golden):
    g = golden("examples.json")
    for s in g["shapes"]:
        assert oracle.Trie([p.encode() for p in s["patterns"]]).stats()["nodes"] == s["nodes"], s["cite"]
    for r in g["rank"]:
        t = oracle.Trie([bytes.fromhex(h) for h in r["patterns_hex"]])
        bm, off = t.node(r["node"])
        bits = [32 * w + b for w in range(8) for b in range(32) if (bm[w] >> b) & 1]
        assert bits == r["bits"] and off == r["offset"], r["cite"]
        assert t.child(r["node"], r["c"]) == r["child"], r["cite"]


def test_invalid_inputs():
    with pytest.raises(oracle.OracleError):
        oracle.Trie([])
    with pytest.raises(oracle.OracleError):
        oracle.Trie([b"ab", b""])


# ------------------------------------------------------------ P6 closed forms
def _random_patterns(rng, m, lmin, lmax, sigma):
    alpha = rng.choice(256, size=sigma, replace=False) if sigma < 256 else np.arange(256)
    pats = []
    for _ in range(m):
        L = int(rng.integers(lmin, lmax + 1))
        pats.append(bytes(alpha[rng.integers(0, sigma, L)].astype(np.uint8)))
    if m > 2 and rng.random() < 0.5:  # duplicates and nested prefixes
        pats.append(pats[0])
        pats.append(pats[1][: max(1, len(pats[1]) // 2)])
    return pats, alpha


def test_closed_forms():
    rng = np.random.default_rng(6)
    for trial in range(200):
        pats, _ = _random_patterns(rng, int(rng.integers(1, 40)), 1, 10, int(rng.choice([2, 4, 256])))
        t = oracle.Trie(pats)
        st = t.stats()
        prefixes = {p[:j] for p in pats for j in range(1, len(p) + 1)}
        assert st["nodes"] == 1 + len(prefixes)                      # one node per distinct prefix
        assert st["edges"] == st["nodes"] - 1
        assert st["terminals"] == len(set(pats))
        assert sum(map(len, pats)) >= st["nodes"] - 1
        assert t.bytes("uncompressed") == 36 * st["nodes"]
        assert t.bytes("dense_stt") == 1024 * st["nodes"]
        # BFS/rank consistency: every set bit resolves to the next level, in order
        depth = {0: 0}
        for v in range(st["nodes"]):
            bm, off = t.node(v)
            bits = [32 * w + b for w in range(8) for b in range(32) if (bm[w] >> b) & 1]
            for r, c in enumerate(bits):
                ch = t.child(v, c)
                assert ch == off + r
                depth[ch] = depth[v] + 1
            if not bits:
                assert off == 0
        order = [depth[v] for v in range(st["nodes"])]
        assert order == sorted(order)                                # level by level (step I)
        # pid lists: node reached by P_k holds k
        for k, p in enumerate(pats):
            v = 0
            for c in p:
                v = t.child(v, c)
            assert k in t.node_pids(v)


# --------------------------------------------------------- P7 brute force
def test_random_tiny_vs_numpy_bruteforce():
    rng = np.random.default_rng(7)
    for trial in range(1000):
        sigma = int(rng.choice([2, 4, 256]))
        pats, alpha = _random_patterns(rng, int(rng.integers(1, 51)), 1, 12, sigma)
        n = int(rng.choice([0, 1, 7, 64, 500, 4096])) if trial % 50 else int(rng.integers(8192, 65536))
        text = bytes(alpha[rng.integers(0, sigma, n)].astype(np.uint8)) if n else b""
        # plant a few occurrences so matches exist on large alphabets
        tb = bytearray(text)
        for _ in range(min(5, n // 16)):
            p = pats[int(rng.integers(len(pats)))]
            if len(p) <= n:
                o = int(rng.integers(0, n - len(p) + 1))
                tb[o:o + len(p)] = p
        text = bytes(tb)
        want = numpy_brute(pats, text)
        t = oracle.Trie(pats)
        engines = ["pfac", "csr", "ac"] + (["brute"] if n <= 4096 else [])
        for e in engines:
            got = t.match_list(text, engine=e, threads=int(rng.integers(1, 9)))
            assert got == want, (trial, e, sigma, n)


def test_range_semantics():
    """Starts in [lo, hi), bytes readable up to L (shard + halo)."""
    rng = np.random.default_rng(8)
    pats = [b"ab", b"abab", b"b", b"bab", b"aaa"]
    text = bytes(rng.choice(list(b"ab"), size=3000).astype(np.uint8))
    t = oracle.Trie(pats)
    for _ in range(50):
        L = int(rng.integers(0, 3001))
        lo = int(rng.integers(0, L + 1))
        hi = int(rng.integers(lo, L + 1))
        want = numpy_brute(pats, text, lo, hi, readable=L)
        for e in ["pfac", "ac", "csr"]:
            assert t.match_list(text, readable_len=L, lo=lo, hi=hi, engine=e) == want


# ------------------------------------------------ P8 invariants, full shapes
@pytest.mark.parametrize("cid,nbytes", [(1, 1024), (2, 4 << 20), (3, 4 << 20), (5, 4 << 20)])
def test_generated_configs_invariants(cid, nbytes):
    ps = gen.patterns(cid)
    pats = ps.to_list()
    text = gen.text(cid, 0, nbytes)
    t = oracle.Trie(ps)
    pos, pid = t.match(text, engine="pfac")
    # (i) compressed == uncompressed == AC
    for e in ["csr", "ac"]:
        p2, q2 = t.match(text, engine=e)
        assert np.array_equal(pos, p2) and np.array_equal(pid, q2), e
    # (ii) thread-count invariance
    p3, q3 = t.match(text, engine="pfac", threads=3)
    assert np.array_equal(pos, p3) and np.array_equal(pid, q3)
    # sorted by (pos, pid), unique
    key = pos.astype(np.uint64) * np.uint64(1 << 32) + pid.astype(np.uint64)
    assert np.all(np.diff(key.astype(np.float64)) > 0) or len(key) < 2
    # (iii) soundness: every row is a real occurrence
    for i, k in zip(pos.tolist(), pid.tolist()):
        assert text[i:i + len(pats[k])].tobytes() == pats[k]
    # (iv) completeness on plants: every planted occurrence, and every pattern
    # that is a prefix of it, is reported at that position
    ppos, ppid = gen.plants(cid, 0, (nbytes + gen.CHUNK - 1) // gen.CHUNK)
    keep = ppos < nbytes
    rows = set(zip(pos.tolist(), pid.tolist()))
    assert keep.sum() > 0
    for i, k in zip(ppos[keep].tolist(), ppid[keep].tolist()):
        if i + len(pats[k]) <= nbytes:
            assert (i, k) in rows
            for k2, p2 in enumerate(pats) if cid == 1 else []:
                if pats[k].startswith(p2):
                    assert (i, k2) in rows


def test_toy_plants_imply_prefix_matches():
    """C1: a planted 'hers' at p implies (p,0),(p,3); 'she' at p implies (p,1),(p+1,0)."""
    ps = gen.patterns(1)
    text = gen.text(1, 0, 1024)
    rows = set(oracle.Trie(ps).match_list(text))
    ppos, ppid = gen.plants(1, 0, 1)
    keep = ppos < 1024
    ppos, ppid = ppos[keep], ppid[keep]
    implied = {0: [(0, 0)], 1: [(0, 1), (1, 0)], 2: [(0, 2)], 3: [(0, 0), (0, 3)]}
    assert len(ppos) == 16
    for i, k in zip(ppos.tolist(), ppid.tolist()):
        for d, k2 in implied[k]:
            if i + d + len(ps[k2]) <= 1024:
                assert (i + d, k2) in rows
