"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and its
`--impl reference` arm) may import this package.  The product path
(paper_1702_03657_b200/) never imports it and shares no code with it.

ctypes over oracle/liboracle.so (plain C, oracle/oracle.c).  What it computes
is the plain definition of multi-pattern matching (§II-B), reached
by four independent engines -- see oracle/oracle.h and DESIGN.md "Oracle".
Pins: tests/test_oracle.py.  Parity unpinned: none (every function has a pin).
"""
from __future__ import annotations

import ctypes as C
import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

PFAC_BITMAP, PFAC_CSR, BRUTE, AC = 0, 1, 2, 3
ENGINES = {"pfac": PFAC_BITMAP, "csr": PFAC_CSR, "brute": BRUTE, "ac": AC}


class _Matches(C.Structure):
    _fields_ = [("n", C.c_uint64), ("pos", C.POINTER(C.c_uint64)), ("pid", C.POINTER(C.c_uint32))]


@functools.lru_cache(None)
def _lib():
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} missing: run `make`")
    L = C.CDLL(_LIB_PATH)
    L.or_build.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]
    L.or_free.argtypes = [C.c_void_p]
    L.or_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    L.or_node.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    L.or_node_pids.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.POINTER(C.c_uint32)),
                               C.POINTER(C.c_uint32)]
    L.or_child.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
    L.or_child.restype = C.c_int64
    L.or_bytes.argtypes = [C.c_void_p, C.c_int]
    L.or_bytes.restype = C.c_uint64
    L.or_paper_crs.argtypes = [C.c_void_p] + [C.POINTER(C.POINTER(C.c_uint32))] * 3 + \
        [C.POINTER(C.c_uint64)] * 2
    L.or_csr.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_uint8)),
                         C.POINTER(C.POINTER(C.c_uint32))]
    L.or_match.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                           C.c_int, C.POINTER(_Matches)]
    L.or_matches_free.argtypes = [C.POINTER(_Matches)]
    return L


def _as_patset(patterns):
    if hasattr(patterns, "data") and hasattr(patterns, "lens"):
        return np.ascontiguousarray(patterns.data, np.uint8), np.ascontiguousarray(patterns.lens, np.uint32)
    pats = [bytes(p) for p in patterns]
    data = np.frombuffer(b"".join(pats), dtype=np.uint8).copy() if pats else np.zeros(0, np.uint8)
    return data, np.array([len(p) for p in pats], dtype=np.uint32)


class OracleError(RuntimeError):
    pass


class Trie:
    """The paper's uncompressed trie (36-byte bitmap nodes, BFS order)."""

    def __init__(self, patterns):
        data, lens = _as_patset(patterns)
        self._data, self._lens = data, lens  # keep alive
        h = C.c_void_p()
        rc = _lib().or_build(data.ctypes.data if data.size else None, lens.ctypes.data if lens.size else None,
                             int(lens.size), C.byref(h))
        if rc != 0:
            raise OracleError(f"or_build failed: {rc}")
        self._h = h

    def __del__(self):
        # at interpreter exit the module globals (_lib) may already be gone
        if getattr(self, "_h", None) and _lib is not None:
            _lib().or_free(self._h)
            self._h = None

    def stats(self) -> dict:
        a = (C.c_uint64 * 6)()
        _lib().or_stats(self._h, a)
        return dict(zip(["nodes", "edges", "terminals", "n_patterns", "max_len", "min_len"], list(a)))

    def node(self, v: int):
        bm = (C.c_uint32 * 8)()
        off = C.c_uint32()
        if _lib().or_node(self._h, v, bm, C.byref(off)) != 0:
            raise IndexError(v)
        return list(bm), off.value

    def node_pids(self, v: int):
        p = C.POINTER(C.c_uint32)()
        n = C.c_uint32()
        if _lib().or_node_pids(self._h, v, C.byref(p), C.byref(n)) != 0:
            raise IndexError(v)
        return [p[i] for i in range(n.value)]

    def child(self, v: int, c: int):
        r = _lib().or_child(self._h, v, c)
        return None if r < 0 else int(r)

    def bytes(self, kind: str) -> int:
        return int(_lib().or_bytes(self._h, {"uncompressed": 0, "dense_stt": 1, "paper_crs": 2}[kind]))

    def paper_crs(self):
        v, c, r = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
        nnz, n = C.c_uint64(), C.c_uint64()
        if _lib().or_paper_crs(self._h, C.byref(v), C.byref(c), C.byref(r), C.byref(nnz), C.byref(n)) != 0:
            raise OracleError("or_paper_crs")
        z, nr = nnz.value, n.value
        out = ([v[i] for i in range(z)], [c[i] for i in range(z)], [r[i] for i in range(nr + 1)])
        libc = C.CDLL(None)
        libc.free.argtypes = [C.c_void_p]
        for p in (v, c, r):
            libc.free(C.cast(p, C.c_void_p))
        return out

    def csr(self):
        r, l, ch = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint8)(), C.POINTER(C.c_uint32)()
        _lib().or_csr(self._h, C.byref(r), C.byref(l), C.byref(ch))
        st = self.stats()
        N, E = st["nodes"], st["edges"]
        return ([r[i] for i in range(N + 1)], bytes(l[i] for i in range(E)), [ch[i] for i in range(E)])

    def match(self, text, readable_len=None, lo=0, hi=None, engine="pfac", threads=0):
        """Rows (pos uint64[], pid uint32[]) sorted by (pos, pid), starts in [lo, hi)."""
        t = np.ascontiguousarray(np.frombuffer(text, np.uint8) if isinstance(text, (bytes, bytearray))
                                 else text, dtype=np.uint8)
        L = t.size if readable_len is None else readable_len
        hi = L if hi is None else hi
        m = _Matches()
        rc = _lib().or_match(self._h, t.ctypes.data if t.size else None, L, lo, hi,
                             ENGINES[engine] if isinstance(engine, str) else engine, threads, C.byref(m))
        if rc != 0:
            raise OracleError(f"or_match failed: {rc}")
        n = m.n
        pos = np.ctypeslib.as_array(m.pos, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
        pid = np.ctypeslib.as_array(m.pid, shape=(n,)).copy() if n else np.zeros(0, np.uint32)
        _lib().or_matches_free(C.byref(m))
        return pos, pid

    def match_list(self, text, **kw):
        pos, pid = self.match(text, **kw)
        return list(zip(pos.tolist(), pid.tolist()))
