"""Host-side hygiene of the product library (no GPU): build options replace
the environment knobs (no getenv in the product), pfac_attach validates every
index the kernel follows, the pid-list budget, and option validation."""
import os
import re

import numpy as np
import pytest

import gen
import paper_1702_03657_b200 as pf
from tests import image_walker

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_environment_reads_in_product():
    """Product behaviour never depends on the environment."""
    csrc = os.path.join(ROOT, "paper_1702_03657_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert not re.search(r"\bgetenv\b", src), f


def test_default_options_equal_plain_build():
    ps = gen.patterns(2)
    assert pf.Trie(ps).image() == pf.Trie(ps, filter_kind=-1).image()
    assert pf.Trie(ps).image() == pf.Trie(ps, pair_bits_per_key=512).image()


@pytest.mark.parametrize("cid,kind", [(2, 1), (2, 2), (3, 1), (3, 2), (3, 4), (4, 1), (4, 2), (5, 3), (5, 1), (5, 4)])
def test_forced_filter_kinds(cid, kind):
    ps = gen.patterns(cid)
    h = image_walker.parse(pf.Trie(ps, filter_kind=kind).image())
    assert h["filter_kind"] == kind
    d = h["filter_gram"]
    for k in range(0, len(ps), max(1, len(ps) // 500)):  # the filter stays complete
        key = image_walker.dna_key(ps[k]) if kind == 3 else int.from_bytes(ps[k][:d], "little")
        if kind == 4:
            continue  # checked through the interpreter below
        assert image_walker.filter_pass(h, key, 0) and image_walker.filter_pass(h, key, 1)
    text = gen.text(cid, 0, 20000).tobytes()
    import oracle
    assert image_walker.match(h, text) == oracle.Trie(ps).match_list(text)


@pytest.mark.parametrize("cid,kind", [(2, 3), (2, 4), (4, 4), (2, 0), (1, 1), (1, 3)])
def test_forced_filter_kind_rejected(cid, kind):
    with pytest.raises(pf.PfacError) as e:
        pf.Trie(gen.patterns(cid), filter_kind=kind)
    assert e.value.status == 1


def test_bad_build_options():
    with pytest.raises(pf.PfacError):
        pf.Trie([b"abc"], filter_kind=7)
    o = pf.build_options()
    o.reserved[0] = 1
    import ctypes as C
    h = C.c_void_p()
    data = np.frombuffer(b"abc", np.uint8).copy()
    lens = np.array([3], np.uint32)
    assert pf._lib().pfac_build_ex(data.ctypes.data, lens.ctypes.data, 1, C.byref(o), C.byref(h)) == 1
    o = pf.build_options()
    o.struct_bytes = 4
    assert pf._lib().pfac_build_ex(data.ctypes.data, lens.ctypes.data, 1, C.byref(o), C.byref(h)) == 1


def test_pid_list_budget():
    """Nested patterns make each terminal's list the union of its ancestors':
    quadratic growth is refused with PFAC_ERR_LIMIT (2^28 entries), not built."""
    pf.Trie([b"a" * k for k in range(1, 3000)])  # ~4.5 M entries: fine
    with pytest.raises(pf.PfacError) as e:
        pf.Trie([b"a" * k for k in range(1, 30000)])  # ~450 M entries
    assert e.value.status == 2


def _corrupt(img, mutate):
    b = bytearray(img)
    h = image_walker.parse(img)
    mutate(b, h)
    return bytes(b)


def _u32(b, off, v):
    b[off:off + 4] = int(v).to_bytes(4, "little")


def _aux_off(h):
    return (h["off_node"] + 4 * (h["n_nodes"] + 1) + 255) // 256 * 256


CORRUPTIONS = {
    "root_out_of_level1": lambda b, h: _u32(b, h["off_root"] + 4 * 7, h["n_level1"] + 3),
    "record_aux_index": lambda b, h: _u32(b, _aux_off(h) + 4 * int(np.nonzero(h["node"][:-1] & image_walker.TAIL)[0][0]),
                                          h["n_tails"] + 10),
    "term_node_wrong": lambda b, h: _u32(b, h["off_term_node"], int(h["term_node"][0]) + 1),
    "out_ptr_not_monotone": lambda b, h: _u32(b, h["off_out_ptr"] + 4, h["n_out"] + 1),
    "out_pid_range": lambda b, h: _u32(b, h["off_out_pid"], h["n_patterns"]),
    "record_misaligned": lambda b, h: _u32(b, h["off_tails"], int(h["tails"][0][0]) + 1),
    "level1_prefix": lambda b, h: _u32(b, h["off_level1"] + 4 * 8, int(h["level1"][0][8]) ^ 0x0100),
    "tail_rank": lambda b, h: _u32(b, h["off_tail_rank"] + 4, int(h["tail_rank"][1]) + 1),
    "tail_bits": lambda b, h: _u32(b, h["off_tail_bits"], int(h["tail_bits"][0]) ^ 1),
    "term_rank": lambda b, h: _u32(b, h["off_term_rk"] + 12, int(h["term_rk"][1][1]) + 1),
    "term_bits": lambda b, h: _u32(b, h["off_term_rk"], int(h["term_rk"][0][0]) ^ 2),
}


@pytest.mark.parametrize("name", sorted(CORRUPTIONS))
def test_attach_rejects_bounds_valid_corruption(name):
    """A corrupted image whose section bounds are intact is refused by
    pfac_attach (INVALID_ARG) instead of reaching the kernel."""
    img = pf.Trie(gen.patterns(2)).image()
    pf.Trie.attach(img, device=-1)  # the intact image is accepted
    with pytest.raises(pf.PfacError) as e:
        pf.Trie.attach(_corrupt(img, CORRUPTIONS[name]), device=-1)
    assert e.value.status == 1


def test_plan_options_validation():
    """Bad plan options are refused before any device is touched."""
    import torch
    t = pf.Trie([b"abcd", b"xyz0"])
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    for kw in [{"ring_slots": 4}, {"ctg64": 65}, {"pool64": 40}, {"placement": 9}, {"stage2": 2}]:
        with pytest.raises(pf.PfacError) as e:
            t.plan(1 << 20, **kw)
        assert e.value.status == 1, kw
    with pytest.raises(pf.PfacError) as e:  # valid options, no device
        t.plan(1 << 20)
    assert e.value.status == 4
