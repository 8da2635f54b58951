"""A plain CPU interpreter of the product's exported device image (T2 in
SURVEY.md §4): walks the CSR image exactly as the layout documented in
paper_1702_03657_b200/csrc/image.h says, so that the layout is checked
against the oracle independently of the CUDA kernel.  Test code only."""
import struct

import numpy as np

TERM = 0x80000000
MASK = 0x7FFFFFFF

_HDR = struct.Struct("<8sII Q QQQQ IIII IIII QQQQQQQ QQQQ")


def parse(image: bytes) -> dict:
    f = _HDR.unpack_from(image, 0)
    keys = ["magic", "version", "header_bytes", "image_bytes", "n_nodes", "n_edges", "n_terminals", "n_out",
            "n_patterns", "max_len", "min_len", "filter_gram", "filter_log2_bits", "filter_exact", "filter_mul",
            "filter_kind", "off_node", "off_label", "off_term_node", "off_out_ptr", "off_out_pid", "off_root",
            "off_filter", "bytes_uncompressed", "bytes_dense_stt", "bytes_paper_crs", "bytes_csr_core"]
    h = dict(zip(keys, f))
    buf = np.frombuffer(image, np.uint8)
    N, E, T = h["n_nodes"], h["n_edges"], h["n_terminals"]
    h["node"] = buf[h["off_node"]:h["off_node"] + 4 * (N + 1)].view(np.uint32)
    h["label"] = buf[h["off_label"]:h["off_label"] + E]
    h["term_node"] = buf[h["off_term_node"]:h["off_term_node"] + 4 * T].view(np.uint32)
    h["out_ptr"] = buf[h["off_out_ptr"]:h["off_out_ptr"] + 4 * (T + 1)].view(np.uint32)
    h["out_pid"] = buf[h["off_out_pid"]:h["off_out_pid"] + 4 * h["n_out"]].view(np.uint32)
    h["root"] = buf[h["off_root"]:h["off_root"] + 1024].view(np.uint32)
    nbits = 1 << h["filter_log2_bits"]
    h["filter"] = buf[h["off_filter"]:h["off_filter"] + max(4, nbits // 8)].view(np.uint32)
    return h


def filter_bits(h, key):
    """Bit indices (word * 32 + bit) of the filter entries a d-gram key tests
    (all must be set for the start to survive)."""
    if h["filter_kind"] == 1:  # d = 4: blocked two-bit filter (image.h)
        b = ((key * ((h["filter_mul"] << 8) & 0xFFFFFFFF)) & 0xFFFFFFFF) >> (32 - (h["filter_log2_bits"] - 6))
        return [2 * b * 32 + (31 - ((key >> 24) & 31)), (2 * b + 1) * 32 + (31 - ((key >> 16) & 31))]
    return [filter_index(h, key)]


def filter_pass(h, key):
    return all((int(h["filter"][i >> 5]) >> (i & 31)) & 1 for i in filter_bits(h, key))


def filter_index(h, key):
    if h["filter_exact"]:
        return key
    return ((key * h["filter_mul"]) & 0xFFFFFFFF) >> (32 - h["filter_log2_bits"])


def match(h, text: bytes, readable=None, n_starts=None):
    """Rows (pos, pid) per the image: filter test, then walk to the deepest terminal."""
    L = len(text) if readable is None else readable
    ns = L if n_starts is None else n_starts
    node, label = h["node"], h["label"]
    term = {int(v): i for i, v in enumerate(h["term_node"])}
    d = h["filter_gram"]
    rows = []
    for i in range(ns):
        if i + d > L:
            continue
        if not filter_pass(h, int.from_bytes(text[i:i + d], "little")):
            continue
        v = int(h["root"][text[i]])
        if v == 0:
            continue
        last = v if node[v] & TERM else None
        j = i + 1
        while j < L:
            s, e = int(node[v]) & MASK, int(node[v + 1]) & MASK
            labs = label[s:e]
            k = np.searchsorted(labs, text[j])
            if k >= len(labs) or labs[k] != text[j]:
                break
            v = s + int(k) + 1
            if node[v] & TERM:
                last = v
            j += 1
        if last is not None:
            t = term[last]
            for r in range(int(h["out_ptr"][t]), int(h["out_ptr"][t + 1])):
                rows.append((i, int(h["out_pid"][r])))
    return rows
