"""NEXT-1: the trie truncated at depth d (PAPER.md:80 step
III, "the trie is truncated at the appropriate level"; "in this case to
eight levels") with exact results kept by verifying, on the device, the
patterns below each depth-d node (verify leaves; image.h).  CPU side: the
exported image, interpreted independently (tests/image_walker.py), equals
the oracle at every depth; the paper's truncated-trie byte count equals its
closed form (36 B x (1 + distinct non-empty prefixes of length <= d), SURVEY
§8(c) P6); validation of verify records."""
import numpy as np
import pytest

import gen
import oracle
import paper_1702_03657_b200 as pf
from tests import image_walker

DEPTHS = [1, 2, 3, 4, 8, 16]


def prefixes_upto(pats, d):
    return len({p[:k] for p in pats for k in range(1, min(d, len(p)) + 1)})


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_truncated_image_equals_oracle(cid):
    ps = gen.patterns(cid)
    pats = ps.to_list()
    text = gen.text(cid, 0, 30000).tobytes()
    want = oracle.Trie(ps).match_list(text)
    full = pf.Trie(ps)
    for d in DEPTHS:
        t = pf.Trie(ps, truncate_depth=d)
        h = image_walker.parse(t.image())
        assert h["trunc_depth"] == d and t.stats()["truncate_depth"] == d
        assert image_walker.match(h, text) == want, f"C{cid} depth {d}"
        # the paper's 36-B-node trie cut at depth d (closed form)
        assert t.nbytes("truncated") == 36 * (1 + prefixes_upto(pats, d))
        assert t.nbytes("uncompressed") == full.nbytes("uncompressed")  # the untruncated reference
    assert full.nbytes("truncated") == full.nbytes("uncompressed")


def test_truncated_random_tiny():
    """Random small sets (nested, duplicated, Σ in {2, 4, 256}) at random
    depths: the image interpreter equals the oracle on random text."""
    rng = np.random.default_rng(31)
    for trial in range(200):
        sigma = int(rng.choice([2, 4, 256]))
        alpha = rng.choice(256, size=sigma, replace=False)
        m = int(rng.integers(1, 30))
        pats = [bytes(alpha[rng.integers(0, sigma, int(rng.integers(1, 14)))].astype(np.uint8)) for _ in range(m)]
        if trial % 3 == 0:
            pats += [pats[0], pats[0] + pats[-1]]
        text = bytes(alpha[rng.integers(0, sigma, int(rng.integers(0, 800)))].astype(np.uint8))
        d = int(rng.integers(1, 10))
        h = image_walker.parse(pf.Trie(pats, truncate_depth=d).image())
        assert image_walker.match(h, text) == oracle.Trie(pats).match_list(text), (trial, d)


def test_verify_records_layout():
    """{he, she, his, hers} cut at depth 1: the root's children h and s are
    verify leaves; h's candidates are "hers", "his", "he" (longest first: the
    bytes past depth 1 are "ers", "is", "e"), s's is "she" ("he")."""
    t = pf.Trie([b"he", b"she", b"his", b"hers"], truncate_depth=1)
    h = image_walker.parse(t.image())
    assert h["n_nodes"] == 3 and h["n_tails"] == 2 and h["n_cand"] == 4
    recs = [tuple(int(y) for y in r) for r in h["tails"]]
    assert [r[2] for r in recs[:2]] == [image_walker.VERIFY] * 2
    got = {}
    for (first, count, _, _) in recs[:2]:
        got[first] = [h["tail_bytes"][recs[c][0]:recs[c][0] + recs[c][1]].tobytes() for c in range(first, first + count)]
    assert sorted(got.values()) == [[b"ers", b"is", b"e"], [b"he"]]
    assert image_walker.match(h, b"ushers") == [(1, 1), (2, 0), (2, 3)]


def test_attach_rejects_bad_verify_record():
    t = pf.Trie(gen.patterns(2), truncate_depth=3)
    img = t.image()
    pf.Trie.attach(img, device=-1)
    h = image_walker.parse(img)
    i = int(np.nonzero(h["tails"][:h["n_tails"], 2] == image_walker.VERIFY)[0][0])
    bad = bytearray(img)
    off = h["off_tails"] + 16 * i + 4  # candidate count past the end
    bad[off:off + 4] = int(h["n_cand"] + 5).to_bytes(4, "little")
    with pytest.raises(pf.PfacError) as e:
        pf.Trie.attach(bytes(bad), device=-1)
    assert e.value.status == 1
