"""Generator checks (inputs only; SURVEY.md §8(d) recipe): determinism, chunk
independence (any shard/halo can be materialised alone), value ranges."""
import numpy as np
import pytest

import gen


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5, 6, 7, 8])
def test_patterns_shape(cid):
    c = gen.config(cid)
    ps = gen.patterns(cid)
    assert len(ps) == c["n_patterns"]
    assert ps.lens.min() >= c["min_len"] and ps.lens.max() <= c["max_len"]
    assert len(set(ps.to_list())) == len(ps)                 # deduplicated by resampling
    if cid in (2, 6, 8):
        assert ps.data.min() >= 0x20 and ps.data.max() <= 0x7E
    if cid == 7:  # substrings of the first 4 MiB of the word text
        head = gen.text(7, 0, 4 << 20).tobytes()
        assert all(p in head for p in ps.to_list()[:50])
    if cid == 5:
        assert set(np.unique(ps.data).tolist()) <= set(b"ACGT")


@pytest.mark.parametrize("cid", [2, 3, 4, 5, 6, 7, 8])
def test_text_chunk_independence(cid):
    full = gen.text(cid, 0, 3 * gen.CHUNK)
    for a, n in [(0, 100), (gen.CHUNK - 7, 20), (gen.CHUNK + 12345, gen.CHUNK), (2 * gen.CHUNK, gen.CHUNK)]:
        assert np.array_equal(gen.text(cid, a, n, threads=1), full[a:a + n])
    assert np.array_equal(gen.text(cid, 0, 3 * gen.CHUNK, threads=3), full)
    # chunks differ (no shifted copies)
    assert not np.array_equal(full[: gen.CHUNK - 64], full[gen.CHUNK + 1: 2 * gen.CHUNK - 63])


def test_text_value_ranges():
    for cid in (2, 6, 8):
        t2 = gen.text(cid, 0, gen.CHUNK)
        assert t2.min() >= 0x20 and t2.max() <= 0x7E
    t7 = gen.text(7, 0, gen.CHUNK)  # Zipf words: lowercase letters and single spaces
    assert set(np.unique(t7).tolist()) <= set(b" abcdefghijklmnopqrstuvwxyz")
    words = t7.tobytes().split(b" ")[1:-1]  # (plants, substrings of the text, cut a few words)
    assert sum(2 <= len(w) <= 10 for w in words) / len(words) > 0.99
    top = max(set(words), key=words.count)
    assert words.count(top) / len(words) > 0.05  # rank 1 of Zipf(1.0) over 20 K words: ~9%
    t5 = gen.text(5, 0, gen.CHUNK)
    assert set(np.unique(t5).tolist()) <= set(b"ACGT")
    freq = np.bincount(t5, minlength=256)[list(b"ACGT")] / t5.size
    assert abs(freq[0] - 0.295) < 0.02 and abs(freq[1] - 0.205) < 0.02
    t4 = gen.text(4, 0, gen.CHUNK)
    h = np.bincount(t4, minlength=256)
    assert h.min() > 0.8 * t4.size / 256


@pytest.mark.parametrize("cid", [1, 2, 5])
def test_plants_are_in_text(cid):
    ps = gen.patterns(cid)
    n = min(gen.config(cid)["text_len"], 2 * gen.CHUNK)
    t = gen.text(cid, 0, n)
    pos, pid = gen.plants(cid, 0, (n + gen.CHUNK - 1) // gen.CHUNK)
    keep = pos < n
    pos, pid = pos[keep], pid[keep]
    c = gen.config(cid)
    expect = (n // c["plant_slot"]) * c["plant_p_q20"] / (1 << 20)
    assert abs(len(pos) - expect) < 5 * np.sqrt(expect) + 1
    for i, k in zip(pos.tolist(), pid.tolist()):
        p = ps[k]
        assert t[i:i + len(p)].tobytes() == p
