"""C-ABI boundary and host logic, no GPU: the library loads and exports every
symbol include/pfac.h declares; the host builder's trie and byte accounting
agree with the oracle; the exported image, interpreted on the CPU
(tests/image_walker.py), reaches the oracle's result; error codes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import gen
import oracle
import paper_1702_03657_b200 as pf
from tests import image_walker

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pfac.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pfac_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 15
    lib = C.CDLL(pf.lib_path)
    for s in syms:
        assert hasattr(lib, s), s
    assert pf._lib().pfac_version().decode().endswith("sm_100a")


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {pf.lib_path} 2>&1").read()
    assert "sm_100a" in out, out


def test_build_errors():
    with pytest.raises(pf.PfacError) as e:
        pf.Trie([])
    assert e.value.status == 1
    with pytest.raises(pf.PfacError) as e:
        pf.Trie([b"ok", b""])
    assert e.value.status == 1
    with pytest.raises(pf.PfacError) as e:
        pf.Trie([b"x" * 65536])
    assert e.value.status == 1
    pf.Trie([b"x" * 65535])  # library limit is inclusive


@pytest.mark.parametrize("cid", [1, 2, 3, 5])
def test_stats_and_bytes_match_oracle(cid):
    ps = gen.patterns(cid)
    t = pf.Trie(ps)
    o = oracle.Trie(ps)
    st, ost = t.stats(), o.stats()
    for k in ["nodes", "edges", "terminals", "n_patterns", "max_len", "min_len"]:
        assert st[k] == ost[k], k
    assert t.nbytes("uncompressed") == o.bytes("uncompressed") == 36 * st["nodes"]
    assert t.nbytes("dense_stt") == o.bytes("dense_stt")
    assert t.nbytes("paper_crs") == o.bytes("paper_crs")
    assert st["image_nodes"] <= st["nodes"]
    assert t.nbytes("csr_core") <= 4 * (st["nodes"] + 1) + st["edges"] or cid == 1
    assert t.nbytes("device_image") < t.nbytes("uncompressed") or cid == 1
    assert t.nbytes("device_image") == len(t.image())


def test_image_interpreter_toy(golden):
    ex = golden("examples.json")["matches"]
    for e in ex:
        t = pf.Trie([p.encode() for p in e["patterns"]])
        h = image_walker.parse(t.image())
        assert image_walker.match(h, e["text"].encode()) == [tuple(r) for r in e["expect"]], e["cite"]


def test_image_layout_toy():
    """Path-compressed image of {he, she, his, hers}, derived by hand from the
    layout documented in csrc/image.h: 's'->"he" and 'he'->"rs" are tails
    (single paths of 2 bytes ending at one terminal); 'hi'->'s' (1 byte) is not."""
    t = pf.Trie([b"he", b"she", b"his", b"hers"])
    h = image_walker.parse(t.image())
    M, TE, TA = image_walker.MASK, image_walker.TERM, image_walker.TAIL
    assert t.stats()["nodes"] == 10 and t.stats()["image_nodes"] == 6
    assert [int(x) & M for x in h["node"]] == [0, 2, 4, 4, 4, 5, 5]
    assert bytes(h["label"]) == b"hseis"
    flags = [(bool(int(x) & TE), bool(int(x) & TA)) for x in h["node"][:6]]
    assert flags == [(False, False), (False, False), (False, True), (True, True), (False, False), (True, False)]
    assert list(h["term_node"]) == [3, 5] and h["n_terminals"] == 4
    assert [tuple(int(y) for y in x[:3]) for x in h["tails"]] == [(0, 2, 2), (4, 2, 3)]
    assert h["tail_bytes"][:8].tobytes() == b"he\x00\x00rs\x00\x00"
    outs = [h["out_pid"][h["out_ptr"][k]:h["out_ptr"][k + 1]].tolist() for k in range(4)]
    assert outs == [[0], [2], [1], [0, 3]]  # he, his, she, hers (+ its prefix he)
    assert h["filter_gram"] == 2 and h["filter_exact"] == 1
    # aux words: labels of nodes with 1..4 children packed little-endian, the
    # record index of tail/chain starts, 0 for leaves
    assert [int(x) for x in h["aux"]] == [0x7368, 0x6965, 0, 1, 0x73, 0]


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_pair_table(cid):
    """2-gram prefix table = bit (b0, b1) set iff a pattern path continues
    with b1 after b0, or b0 alone reaches a terminal / tail / chain start."""
    h = image_walker.parse(pf.Trie(gen.patterns(cid)).image())
    node, root, l1 = h["node"], h["root"], h["level1"]
    for b0 in range(256):
        v = int(root[b0])
        want = [0] * 8 if v == 0 else ([0xFFFFFFFF] * 8 if int(node[v]) & (image_walker.TERM | image_walker.TAIL)
                                       else [int(x) for x in l1[v - 1][:8]])
        assert [int(x) for x in h["pair"][b0]] == want, b0


@pytest.mark.parametrize("cid", [3, 5])
def test_entry_table(cid):
    """Kinds 4 (C3: 8-byte prefixes) and 3 (C5: 16-base DNA keys): one entry
    per distinct D-byte pattern prefix; entering the walk at the entry's
    (node, depth) gives the root walk's result for every pattern, the entry
    node is the root walk's node after `depth` bytes, and keys that begin no
    pattern are absent."""
    ps = gen.patterns(cid).to_list()
    h = image_walker.parse(pf.Trie(ps).image())
    D = h["filter_gram"]
    assert (h["filter_kind"], D) in [(4, 8), (3, 16)] and h["off_entry"] and not h["off_kset"]

    def key(x):
        if h["filter_kind"] == 3:
            return image_walker.dna_key(x[:D]), 0
        return int.from_bytes(x[:4], "little"), int.from_bytes(x[4:8], "little")
    prefixes = {p[:D] for p in ps}
    assert int((h["entry"][:, 2] != 0xFFFFFFFF).sum()) == len(prefixes)
    rng = np.random.default_rng(3)
    for k in rng.choice(len(ps), 1500, replace=False):
        p = ps[int(k)]
        en = image_walker.entry_find(h, *key(p))
        assert en is not None and 1 <= en[1] <= D
        full = image_walker.walk(h, p, 0, len(p))
        assert full is not None and image_walker.walk(h, p, 0, len(p), *en) == full
        assert _node_after(h, p, en[1]) == en[0]
    alpha = np.frombuffer(b"ACGT", np.uint8) if cid == 5 else np.arange(256, dtype=np.uint8)
    for _ in range(2000):
        x = rng.choice(alpha, D).astype(np.uint8).tobytes()
        if x not in prefixes:
            assert image_walker.entry_find(h, *key(x)) is None


def _node_after(h, text, d):
    """Image node reached by consuming text[:d] from the root (a record's
    start when the path enters a record before depth d)."""
    node, label = h["node"], h["label"]
    v, j = int(h["root"][text[0]]), 1
    while j < d:
        if int(node[v]) & image_walker.TAIL:
            off, ln, ti, x = (int(y) for y in h["tails"][image_walker.tail_index(h, v)])
            if ti != 0xFFFFFFFF or j + ln > d:
                return v  # the record spans depth d: its start is the deepest image node
            v, j = x, j + ln
            continue
        s_, e_ = int(node[v]) & image_walker.MASK, int(node[v + 1]) & image_walker.MASK
        k = int(np.searchsorted(label[s_:e_], text[j]))
        assert k < e_ - s_ and label[s_ + k] == text[j]
        v, j = s_ + k + 1, j + 1
    return v


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_aux_words(cid):
    """aux[v] = record rank (tail/chain start) or packed labels (1..4 children;
    the first four of 5..8); the node record's last word = labels 4..7."""
    h = image_walker.parse(pf.Trie(gen.patterns(cid)).image())
    node, aux, label = h["node"].astype(np.int64), h["aux"], h["label"]
    rank = 0
    for v in range(len(aux)):
        e0, e1 = int(node[v]) & image_walker.MASK, int(node[v + 1]) & image_walker.MASK
        if node[v] & image_walker.TAIL:
            assert aux[v] == rank == image_walker.tail_index(h, v)
            rank += 1
        elif 1 <= e1 - e0 <= 8:  # (the first four labels of a node with 5..8 children)
            assert aux[v] == int.from_bytes(bytes(label[e0:min(e1, e0 + 4)]), "little"), v
        else:
            assert aux[v] == 0
        rec = [int(x) for x in h["rec"][v]]
        want4 = int.from_bytes(bytes(label[e0 + 4:e1]), "little") if 5 <= e1 - e0 <= 8 and not node[v] & image_walker.TAIL else 0
        assert rec == [int(node[v]), int(node[v + 1]), int(aux[v]), want4], v


def test_image_interpreter_random_vs_oracle():
    rng = np.random.default_rng(11)
    for trial in range(150):
        sigma = int(rng.choice([2, 4, 256]))
        alpha = rng.choice(256, size=sigma, replace=False)
        m = int(rng.integers(1, 30))
        pats = [bytes(alpha[rng.integers(0, sigma, int(rng.integers(1, 9)))].astype(np.uint8)) for _ in range(m)]
        if trial % 3 == 0:
            pats.append(pats[0])
        n = int(rng.integers(0, 600))
        text = bytes(alpha[rng.integers(0, sigma, n)].astype(np.uint8))
        h = image_walker.parse(pf.Trie(pats).image())
        L = int(rng.integers(0, n + 1))
        ns = int(rng.integers(0, L + 1))
        want = oracle.Trie(pats).match_list(text, readable_len=L, lo=0, hi=ns)
        assert image_walker.match(h, text, readable=L, n_starts=ns) == want, trial


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_image_interpreter_configs(cid):
    ps = gen.patterns(cid)
    t = pf.Trie(ps)
    h = image_walker.parse(t.image())
    text = gen.text(cid, 0, 40000).tobytes()
    want = oracle.Trie(ps).match_list(text)
    assert image_walker.match(h, text) == want


def test_filter_is_complete():
    """Every pattern's d-gram bit is set (a clear bit must imply no match)."""
    for cid in [2, 3, 4, 5]:
        ps = gen.patterns(cid)
        h = image_walker.parse(pf.Trie(ps).image())
        d = h["filter_gram"]
        assert h["filter_kind"] == {2: 2, 3: 4, 4: 1, 5: 3}[cid]  # pair / 8-gram / blocked / DNA k-mer filters
        for k in range(len(ps)):
            key = image_walker.dna_key(ps[k]) if h["filter_kind"] == 3 else int.from_bytes(ps[k][:d], "little")
            assert image_walker.filter_pass(h, key, 0) and image_walker.filter_pass(h, key, 1)


def test_attach_roundtrip_and_validation():
    t = pf.Trie(gen.patterns(2))
    img = t.image()
    t2 = pf.Trie.attach(img, device=-1)  # host only, no device upload
    assert t2.image() == img and t2.stats() == t.stats()
    bad = bytearray(img)
    bad[0] ^= 0xFF
    with pytest.raises(pf.PfacError):
        pf.Trie.attach(bytes(bad), device=-1)
    bad = bytearray(img)
    bad[image_walker.parse(img)["off_node"] + 4 * 3] = 0xFF  # corrupt row_ptr monotonicity
    with pytest.raises(pf.PfacError):
        pf.Trie.attach(bytes(bad), device=-1)
    with pytest.raises(pf.PfacError):
        pf.Trie.attach(img[:-256], device=-1)


def test_workspace_bytes_needs_device():
    """Workspace size depends on the device's SM count (launch geometry)."""
    import torch
    t = pf.Trie([b"abc"])
    if torch.cuda.is_available():
        a, b = t.workspace_bytes(1), t.workspace_bytes(1 << 30)
        assert 256 < a < b
    else:
        with pytest.raises(pf.PfacError) as e:
            t.workspace_bytes(1)
        assert e.value.status == 4


def test_no_cpu_fallback():
    """Without a usable device the product path fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = pf.Trie([b"he", b"she"])
    with pytest.raises(pf.PfacError) as e:
        t.match_host(b"ushers")
    assert e.value.status == 4


def test_option_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of pfac_build_options / pfac_plan_options /
    pfac_plan_info (argument marshalling only) have the header's size and
    field offsets: compiled from include/pfac.h with the host C compiler."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no host C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    structs = {"pfac_build_options": pf.BuildOptions, "pfac_plan_options": pf.PlanOptions,
               "pfac_plan_info": pf._PlanInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pfac.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, f, v = line.split()
        got[(cname, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_terminal_rank_matches_term_node(cid):
    """Image v22's kept-terminal rank (bits + per-32-node prefix counts) gives
    every kept terminal node its index in the ascending term_node list (the
    definition), and no other node has the terminal bit."""
    h = image_walker.parse(pf.Trie(gen.patterns(cid)).image())
    rk = h["term_rk"].astype(np.uint64)
    tn = h["term_node"].astype(np.int64)
    v = tn
    below = rk[v >> 5, 0] & ((np.uint64(1) << (v & 31).astype(np.uint64)) - np.uint64(1))
    popc = np.array([bin(int(x)).count("1") for x in below], np.uint64)
    assert np.array_equal(rk[v >> 5, 1] + popc, np.arange(len(tn), dtype=np.uint64))
    bits = np.unpackbits(h["term_rk"][:, 0].astype("<u4").view(np.uint8), bitorder="little")[: h["n_nodes"]]
    assert np.array_equal(np.nonzero(bits)[0], tn)
