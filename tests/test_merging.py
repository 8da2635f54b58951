"""NEXT-2: suffix and end-node merging (PAPER.md:80 steps
IV-V) with pattern identity kept by path rank, and the Fig. 5-style byte
accounting of the paper's pipeline (uncompressed -> truncated at 8 levels ->
merged -> CRS).  CPU side: the merged DAG, interpreted
independently (tests/image_walker.py dag_match), equals the oracle; the DAG
is minimal and its counts obey closed forms."""
import numpy as np
import pytest

import gen
import oracle
import paper_1702_03657_b200 as pf
from tests import image_walker


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_merged_dag_equals_oracle(cid):
    ps = gen.patterns(cid)
    text = gen.text(cid, 0, 20000).tobytes()
    t = pf.Trie(ps, merge_suffixes=1)
    h = image_walker.parse(t.image())
    assert image_walker.dag_match(h, text) == oracle.Trie(ps).match_list(text)
    assert image_walker.match(h, text) == oracle.Trie(ps).match_list(text)  # the main image is unchanged


def _dag_strings(h):
    """Every string the DAG accepts, with the rank its walk computes."""
    node, lab, child, skip = h["dag_node"], h["dag_label"], h["dag_child"], h["dag_skip"]
    out, stack = [], [(0, b"", 0)]
    while stack:
        v, s, r = stack.pop()
        if int(node[v]) & image_walker.TERM:
            out.append((s, r))
        a, b = int(node[v]) & image_walker.MASK, int(node[v + 1]) & image_walker.MASK
        for e in range(a, b):
            stack.append((int(child[e]), s + bytes([int(lab[e])]), r + int(skip[e])))
    return out


def test_toy_dag_by_hand():
    """{he, she, his, hers}: trie of 10 nodes; merging gives 7 (the leaves
    'his', 'she', 'hers' become one node; 'he' and 'she' end nodes differ in
    children).  Ranks follow lexicographic order: he 0, hers 1, his 2, she 3."""
    t = pf.Trie([b"he", b"she", b"his", b"hers"], merge_suffixes=1)
    h = image_walker.parse(t.image())
    assert h["n_nodes_full"] == 10 and h["n_dag_nodes"] == 7
    assert sorted(_dag_strings(h)) == [(b"he", 0), (b"hers", 1), (b"his", 2), (b"she", 3)]
    assert t.nbytes("merged") == 36 * 7
    assert image_walker.dag_match(h, b"ushers") == [(1, 1), (2, 0), (2, 3)]


@pytest.mark.parametrize("cid", [2, 5])
def test_dag_language_and_ranks(cid):
    """The DAG accepts exactly the distinct pattern strings, each at its
    lexicographic rank (proper prefixes first)."""
    pats = sorted(set(gen.patterns(cid).to_list()))
    h = image_walker.parse(pf.Trie(gen.patterns(cid), merge_suffixes=1).image())
    got = sorted(_dag_strings(h))
    assert [s for s, _ in got] == pats
    assert [r for _, r in got] == list(range(len(pats)))


def test_dag_is_minimal_random():
    """Minimality (brute force on small sets): two DAG nodes never accept the
    same right language."""
    rng = np.random.default_rng(7)
    for _ in range(30):
        pats = [bytes(rng.choice(np.frombuffer(b"ab", np.uint8), int(rng.integers(1, 7)))) for _ in range(12)]
        h = image_walker.parse(pf.Trie(pats, merge_suffixes=1).image())
        node, lab, child = h["dag_node"], h["dag_label"], h["dag_child"]

        def lang(v, memo={}):
            key = (id(h), v)
            if key not in memo:
                s = {b""} if int(node[v]) & image_walker.TERM else set()
                a, b = int(node[v]) & image_walker.MASK, int(node[v + 1]) & image_walker.MASK
                for e in range(a, b):
                    s |= {bytes([int(lab[e])]) + x for x in lang(int(child[e]))}
                memo[key] = frozenset(s)
            return memo[key]
        langs = [lang(v) for v in range(h["n_dag_nodes"])]
        assert len(set(langs)) == len(langs)


def test_pipeline_accounting_toy():
    """Paper pipeline on the toy set (depth 8 cuts nothing): merged 7 nodes;
    CRS of the merged trie: val/col_ind entries = 2 per inner node with one
    bitmap word (root: h,s in word 3 -> 1 word + offset) ... = 2 nnz + n + 1."""
    t = pf.Trie([b"he", b"she", b"his", b"hers"], merge_suffixes=1)
    assert t.nbytes("pipe_trunc") == t.nbytes("uncompressed") == 360
    assert t.nbytes("pipe_merged") == 36 * 7
    # merged nodes with children: root(h,s), h(e,i), s(h), he(r), sh(e), her(s)... by hand:
    # classes: root, h, s, he, hi~(s->leaf), sh, her, leaf -> 7 nodes, 6 inner with one bitmap word each
    assert t.nbytes("pipe_crs") == 4 * (2 * (6 + 6) + 7 + 1)
    assert t.nbytes("merged_crs") == t.nbytes("pipe_crs")


def test_merge_requires_option():
    t = pf.Trie(gen.patterns(2))
    with pytest.raises(pf.PfacError):
        t.nbytes("merged")


def test_attach_rejects_bad_dag():
    t = pf.Trie(gen.patterns(2), merge_suffixes=1)
    img = t.image()
    pf.Trie.attach(img, device=-1)
    h = image_walker.parse(img)
    bad = bytearray(img)
    o = h["off_dag_child"]
    bad[o:o + 4] = int(h["n_dag_nodes"] + 3).to_bytes(4, "little")
    with pytest.raises(pf.PfacError):
        pf.Trie.attach(bytes(bad), device=-1)
