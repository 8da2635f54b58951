"""A plain CPU interpreter of the product's exported device image (T2 in
SURVEY.md §4): walks the CSR image exactly as the layout documented in
paper_1702_03657_b200/csrc/image.h says, so that the layout is checked
against the oracle independently of the CUDA kernel.  Test code only."""
import struct

import numpy as np

TERM = 0x80000000
TAIL = 0x40000000
MASK = 0x3FFFFFFF

_HDR = struct.Struct("<8sII Q QQQQ IIII IIII QQQQQQQ QQQQ QQQQQQ QQ QQ Q II Q Q II Q II Q QQQQQQQ QQ QQQQ Q Q")
VERIFY = 0xFFFFFFFE


def parse(image: bytes) -> dict:
    f = _HDR.unpack_from(image, 0)
    keys = ["magic", "version", "header_bytes", "image_bytes", "n_nodes", "n_edges", "n_terminals", "n_out",
            "n_patterns", "max_len", "min_len", "filter_gram", "filter_log2_bits", "filter_exact", "filter_mul",
            "filter_kind", "off_node", "off_label", "off_term_node", "off_out_ptr", "off_out_pid", "off_root",
            "off_filter", "bytes_uncompressed", "bytes_dense_stt", "bytes_paper_crs", "bytes_csr_core",
            "n_tails", "n_tail_bytes", "off_tail_bits", "off_tail_rank", "off_tails", "off_tail_bytes",
            "n_level1", "off_level1", "n_kept_terminals", "n_nodes_full", "off_kset", "kset_log2", "kset_empty", "off_pair",
            "off_entry", "entry_log2", "entry_pad", "n_cand", "trunc_depth", "trunc_pad", "bytes_truncated",
            "n_dag_nodes", "n_dag_edges", "off_dag_node", "off_dag_label", "off_dag_child", "off_dag_skip",
            "off_rank_term", "bytes_merged", "bytes_merged_crs", "pipe_depth", "bytes_pipe_trunc",
            "bytes_pipe_merged", "bytes_pipe_crs", "off_rec", "off_term_rk"]
    h = dict(zip(keys, f))
    buf = np.frombuffer(image, np.uint8)
    N, E, T = h["n_nodes"], h["n_edges"], h["n_terminals"]
    h["node"] = buf[h["off_node"]:h["off_node"] + 4 * (N + 1)].view(np.uint32)
    off_aux = (h["off_node"] + 4 * (N + 1) + 255) // 256 * 256  # image.h: aux follows node
    h["aux"] = buf[off_aux:off_aux + 4 * N].view(np.uint32)
    h["label"] = buf[h["off_label"]:h["off_label"] + E]
    h["term_node"] = buf[h["off_term_node"]:h["off_term_node"] + 4 * h["n_kept_terminals"]].view(np.uint32)
    h["out_ptr"] = buf[h["off_out_ptr"]:h["off_out_ptr"] + 4 * (T + 1)].view(np.uint32)
    h["out_pid"] = buf[h["off_out_pid"]:h["off_out_pid"] + 4 * h["n_out"]].view(np.uint32)
    h["root"] = buf[h["off_root"]:h["off_root"] + 1024].view(np.uint32)
    nbits = 1 << h["filter_log2_bits"]
    h["filter"] = buf[h["off_filter"]:h["off_filter"] + max(4, nbits // 8)].view(np.uint32)
    nw = (N + 31) // 32
    h["tail_bits"] = buf[h["off_tail_bits"]:h["off_tail_bits"] + 4 * nw].view(np.uint32)
    h["tail_rank"] = buf[h["off_tail_rank"]:h["off_tail_rank"] + 4 * nw].view(np.uint32)
    h["tails"] = buf[h["off_tails"]:h["off_tails"] + 16 * (h["n_tails"] + h["n_cand"])].view(np.uint32).reshape(-1, 4)
    h["tail_bytes"] = buf[h["off_tail_bytes"]:h["off_tail_bytes"] + h["n_tail_bytes"]]
    h["level1"] = buf[h["off_level1"]:h["off_level1"] + 40 * h["n_level1"]].view(np.uint32).reshape(-1, 10)
    h["pair"] = buf[h["off_pair"]:h["off_pair"] + 8192].view(np.uint32).reshape(256, 8)
    if h["off_kset"]:
        h["kset"] = buf[h["off_kset"]:h["off_kset"] + (4 << h["kset_log2"])].view(np.uint32)
    h["rec"] = buf[h["off_rec"]:h["off_rec"] + 16 * N].view(np.uint32).reshape(-1, 4)
    h["term_rk"] = buf[h["off_term_rk"]:h["off_term_rk"] + 8 * ((N + 31) // 32)].view(np.uint32).reshape(-1, 2)
    if h["n_dag_nodes"]:
        ND, ED = h["n_dag_nodes"], h["n_dag_edges"]
        h["dag_node"] = buf[h["off_dag_node"]:h["off_dag_node"] + 4 * (ND + 1)].view(np.uint32)
        h["dag_label"] = buf[h["off_dag_label"]:h["off_dag_label"] + ED]
        h["dag_child"] = buf[h["off_dag_child"]:h["off_dag_child"] + 4 * ED].view(np.uint32)
        h["dag_skip"] = buf[h["off_dag_skip"]:h["off_dag_skip"] + 4 * ED].view(np.uint32)
        h["rank_term"] = buf[h["off_rank_term"]:h["off_rank_term"] + 4 * T].view(np.uint32)
    if h["off_entry"]:
        h["entry"] = buf[h["off_entry"]:h["off_entry"] + (16 << h["entry_log2"])].view(np.uint32).reshape(-1, 4)
    return h


def entry_find(h, x0, x1):
    """Depth-8 entry table probe (image.h): (node, depth) or None."""
    t, lg = h["entry"], h["entry_log2"]
    i = ((x0 * 0x9E3779B1 + x1 * 0x85EBCA6B) & 0xFFFFFFFF) >> (32 - lg)
    while int(t[i][2]) != 0xFFFFFFFF:
        if int(t[i][0]) == x0 and int(t[i][1]) == x1:
            return int(t[i][2]), int(t[i][3])
        i = (i + 1) & ((1 << lg) - 1)
    return None


def tail_index(h, v):
    w = int(h["tail_bits"][v >> 5])
    return int(h["tail_rank"][v >> 5]) + bin(w & ((1 << (v & 31)) - 1)).count("1")


def filter_bits(h, key):
    """Bit indices (word * 32 + bit) of the filter entries a d-gram key tests
    (all must be set for the start to survive)."""
    if h["filter_kind"] == 2:  # d = 4: pair filter, tested here as the first start of a pair
        raise ValueError("kind 2 tests depend on the start's parity; use filter_pass")
    if h["filter_kind"] == 1:  # d = 4: blocked three-bit filter in 32-bit words (image.h)
        mask = ((1 << (h["filter_log2_bits"] - 3)) - 1) & ~3
        w = (((key * h["filter_mul"]) >> 32) & mask) // 4
        return [w * 32 + (31 - ((key >> (8 * b)) & 31)) for b in (3, 2, 1)]
    return [filter_index(h, key)]


def _block(h, x3):
    return ((x3 * ((h["filter_mul"] << 8) & 0xFFFFFFFF)) & 0xFFFFFFFF) >> (32 - (h["filter_log2_bits"] - 6))


def _pair_word(h, x3):
    return ((x3 * ((h["filter_mul"] << 8) & 0xFFFFFFFF)) & 0xFFFFFFFF) >> (32 - (h["filter_log2_bits"] - 5))


def dna_key(window: bytes) -> int:
    """Kind 3: 2-bit codes (b >> 1) & 3 of the first 16 bytes, byte i at bits 2i."""
    return sum(((b >> 1) & 3) << (2 * i) for i, b in enumerate(window[:16]))


def filter_pass(h, key, start=0):
    """Does the start whose first d bytes are `key` pass the filter?  Kind 2
    (pair filter) depends on the start's parity (image.h).  Kind 3 takes the
    DNA key (dna_key of the start's 16 bytes)."""
    if h["filter_kind"] == 4:  # key = the 8 bytes, little-endian (an int)
        f = h["filter"]
        x0, x1 = key & 0xFFFFFFFF, key >> 32
        hh = (x0 * 0x9E3779B1 + x1 * 0x85EBCA6B) & 0xFFFFFFFF
        b = hh >> (32 - (h["filter_log2_bits"] - 6))
        return bool((int(f[2 * b]) >> (31 - (x0 & 31))) & 1) and bool((int(f[2 * b + 1]) >> (31 - (x1 & 31))) & 1)
    if h["filter_kind"] == 3:  # 32-bit words as kind 1; bits from bases 0-2, 8-10, 13-15 (image.h)
        mask = ((1 << (h["filter_log2_bits"] - 3)) - 1) & ~3
        w = int(h["filter"][(((key * 0x9E3779B1) >> 32) & mask) // 4])
        return all((w >> (31 - ((key >> s) & 31))) & 1 for s in (0, 16, 26))
    if h["filter_kind"] == 2:
        f = h["filter"]
        if start % 2 == 0:  # first of the pair: shared bytes 1..3, own byte 0
            w = int(f[_pair_word(h, key >> 8)])
            return bool((w >> (31 - (key & 31))) & 1)
        w = int(f[_pair_word(h, key & 0xFFFFFF)])  # second: shared bytes are the start's bytes 0..2, own byte 3
        return bool((w >> (31 - ((key >> 24) & 31))) & 1)
    return all((int(h["filter"][i >> 5]) >> (i & 31)) & 1 for i in filter_bits(h, key))


def filter_index(h, key):
    if h["filter_exact"]:
        return key
    return ((key * h["filter_mul"]) & 0xFFFFFFFF) >> (32 - h["filter_log2_bits"])


def term_of(h, last):
    if last is None:
        return None
    k = int(np.searchsorted(h["term_node"], last))
    assert h["term_node"][k] == last
    return k


def walk(h, text, i, L, v0=None, d0=1):
    """Terminal index of the deepest terminal passed by the walk from start i
    (entered at node v0 of depth d0 when given).  Bit 30 marks a tail start
    (record ends at a terminal: compare and stop) or a chain start (record
    ends at node x: compare, continue at x)."""
    node, label = h["node"], h["label"]
    v = int(h["root"][text[i]]) if v0 is None else v0
    if v == 0:
        return None
    last = v if node[v] & TERM else None
    j = i + d0
    l1 = d0 == 1
    while j < L:
        if node[v] & TAIL:
            off, ln, ti, x = (int(y) for y in h["tails"][tail_index(h, v)])
            if ti == VERIFY:  # verify leaf (truncated trie): the longest candidate the text matches
                for c in range(off, off + ln):
                    co, cl, ct, _ = (int(y) for y in h["tails"][c])
                    if j + cl <= L and bytes(text[j:j + cl]) == h["tail_bytes"][co:co + cl].tobytes():
                        return ct
                return term_of(h, last)
            if not (j + ln <= L and bytes(text[j:j + ln]) == h["tail_bytes"][off:off + ln].tobytes()):
                return term_of(h, last)
            if ti != 0xFFFFFFFF:  # tail: ends at its terminal
                return ti
            v, j = x, j + ln  # chain: continue at its end node
        else:
            s_, e_ = int(node[v]) & MASK, int(node[v + 1]) & MASK
            if l1:  # level 1: the bitmapped node
                bm = [int(y) for y in h["level1"][v - 1]]
                c = text[j]
                if not (bm[c >> 5] >> (c & 31)) & 1:
                    break
                pre = (bm[8 + (c >> 7)] >> (8 * ((c >> 5) & 3))) & 0xFF
                v = s_ + pre + bin(bm[c >> 5] & ((1 << (c & 31)) - 1)).count("1") + 1
            else:
                labs = label[s_:e_]
                k = np.searchsorted(labs, text[j])
                if k >= len(labs) or labs[k] != text[j]:
                    break
                v = s_ + int(k) + 1
            j += 1
        l1 = False
        if node[v] & TERM:
            last = v
    return term_of(h, last)


def kset_has(h, key):
    """Exact key set probe (image.h): buckets of 4 slots from the home bucket
    (key * M) >> (34 - log2) until the key (present) or an empty slot (absent)."""
    t, lg = h["kset"], h["kset_log2"]
    b = ((key * 0x9E3779B1) & 0xFFFFFFFF) >> (34 - lg)
    while True:
        q = [int(x) for x in t[4 * b:4 * b + 4]]
        if key in q:
            return True
        if h["kset_empty"] in q:
            return False
        b = (b + 1) & ((1 << (lg - 2)) - 1)


def match(h, text: bytes, readable=None, n_starts=None):
    """Rows (pos, pid) per the image: filter test, then walk to the deepest terminal."""
    L = len(text) if readable is None else readable
    ns = L if n_starts is None else n_starts
    d = h["filter_gram"]
    rows = []
    for i in range(ns):
        if i + d > L:
            continue
        key = dna_key(text[i:i + d]) if h["filter_kind"] == 3 else int.from_bytes(text[i:i + d], "little")
        if not filter_pass(h, key, i):
            continue
        if h["off_kset"] and not kset_has(h, key):  # the exact key set (image.h)
            continue
        if h["off_entry"]:  # kinds 4 and 3: enter through the entry table (image.h)
            if h["filter_kind"] == 3:
                ok = all(b in b"ACGT" for b in bytes(text[i:i + d]))  # the key aliases other bytes
                en = entry_find(h, key, 0) if ok else None
            else:
                en = entry_find(h, key & 0xFFFFFFFF, key >> 32)
            ti = walk(h, text, i, L, *en) if en else None
        else:
            ti = walk(h, text, i, L)
        if ti is not None:
            for r in range(int(h["out_ptr"][ti]), int(h["out_ptr"][ti + 1])):
                rows.append((i, int(h["out_pid"][r])))
    return rows


def dag_walk(h, text, i, L):
    """Merged DAG (image.h dag_*): walk from the root adding each edge's rank
    skip; the rank at the deepest terminal reached -> its terminal index."""
    node, lab, child, skip = h["dag_node"], h["dag_label"], h["dag_child"], h["dag_skip"]
    v, rank, last, j = 0, 0, None, i
    while j < L:
        a, b = int(node[v]) & MASK, int(node[v + 1]) & MASK
        k = int(np.searchsorted(lab[a:b], text[j]))
        if k >= b - a or lab[a + k] != text[j]:
            break
        rank += int(skip[a + k])
        v = int(child[a + k])
        j += 1
        if int(node[v]) & TERM:
            last = rank
    return None if last is None else int(h["rank_term"][last])


def dag_match(h, text, readable=None, n_starts=None):
    L = len(text) if readable is None else readable
    ns = L if n_starts is None else n_starts
    out = []
    for i in range(ns):
        t = dag_walk(h, text, i, L)
        if t is not None:
            out += [(i, int(p)) for p in h["out_pid"][h["out_ptr"][t]:h["out_ptr"][t + 1]]]
    return out
