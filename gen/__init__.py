"""Seeded synthetic input generators (ctypes over gen/libpfacgen.so).

Holds none of the method's arithmetic: it only draws the pattern sets and
text bytes of BASELINE.json's five configurations (SURVEY.md §8(d) recipe,
restated in DESIGN.md "Input recipe").  Both the oracle side and the CUDA side
of every test and of bench.py take their inputs from here.
"""
from __future__ import annotations

import ctypes as C
import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpfacgen.so")

CHUNK = 1 << 20
CONFIG_NAMES = {
    1: "C1 toy {he,she,his,hers} / 1 KiB printable ASCII",
    2: "C2 1,000 ASCII patterns len 4-32 / 64 MiB",
    3: "C3 10,000 Snort/ClamAV-shaped patterns len 8-64 / 1 GiB packets",
    4: "C4 100,000 byte patterns len 4-128 / 4 GiB",
    5: "C5 DNA 50,000 k-mers k=16-32 / 16 GiB",
    6: "C4 ASCII variant: 100,000 printable patterns len 4-128 / 4 GiB printable text (reported, not gating)",
    7: "C2 paper-shaped variant: 1,000 substrings (len 4-32) of a Zipf(1.0) word text / 64 MiB (reported)",
    8: "C2 dense variant: C2's distribution (its own seeds) with every 64-byte slot planted / 64 MiB (reported)",
}


class _Cfg(C.Structure):
    _fields_ = [
        ("id", C.c_int),
        ("text_len", C.c_uint64),
        ("n_patterns", C.c_uint32),
        ("min_len", C.c_uint32),
        ("max_len", C.c_uint32),
        ("seed_pat", C.c_uint64),
        ("seed_text", C.c_uint64),
        ("seed_plant", C.c_uint64),
        ("plant_slot", C.c_uint32),
        ("plant_p_q20", C.c_uint32),
    ]


class _MT(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int)]


@functools.lru_cache(None)
def _lib():
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
    L = C.CDLL(_LIB_PATH)
    L.pg_config_get.argtypes = [C.c_int, C.POINTER(_Cfg)]
    L.pg_make_patterns.argtypes = [C.POINTER(_Cfg), C.POINTER(C.POINTER(C.c_uint8)),
                                   C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint32)]
    L.pg_make_text.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_void_p, C.c_uint32,
                               C.c_uint64, C.c_uint64, C.c_void_p, C.c_int]
    L.pg_plants.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                            C.c_uint64, C.POINTER(C.POINTER(C.c_uint64)),
                            C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]
    L.pg_free.argtypes = [C.c_void_p]
    L.pg_mt64_seed.argtypes = [C.POINTER(_MT), C.c_uint64]
    L.pg_mt64_next.argtypes = [C.POINTER(_MT)]
    L.pg_mt64_next.restype = C.c_uint64
    L.pg_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
    L.pg_splitmix64_next.restype = C.c_uint64
    return L


def config(cid: int) -> dict:
    c = _Cfg()
    if _lib().pg_config_get(cid, C.byref(c)) != 0:
        raise ValueError(f"unknown config {cid}")
    return {f: getattr(c, f) for f, _ in _Cfg._fields_}


def _cfg(cid: int) -> _Cfg:
    c = _Cfg()
    if _lib().pg_config_get(cid, C.byref(c)) != 0:
        raise ValueError(f"unknown config {cid}")
    return c


class PatternSet:
    """Concatenated pattern bytes + lengths (binary-safe), pid = index."""

    def __init__(self, data: np.ndarray, lens: np.ndarray):
        self.data = np.ascontiguousarray(data, dtype=np.uint8)
        self.lens = np.ascontiguousarray(lens, dtype=np.uint32)
        self.offs = np.concatenate([[0], np.cumsum(self.lens, dtype=np.uint64)[:-1]]).astype(np.uint64)

    @classmethod
    def from_list(cls, pats):
        pats = [bytes(p) for p in pats]
        data = np.frombuffer(b"".join(pats), dtype=np.uint8) if pats else np.zeros(0, np.uint8)
        return cls(data.copy(), np.array([len(p) for p in pats], dtype=np.uint32))

    def __len__(self):
        return int(self.lens.shape[0])

    def __getitem__(self, k) -> bytes:
        o = int(self.offs[k])
        return self.data[o:o + int(self.lens[k])].tobytes()

    def to_list(self):
        return [self[k] for k in range(len(self))]

    @property
    def max_len(self):
        return int(self.lens.max()) if len(self) else 0


@functools.lru_cache(None)
def patterns(cid: int) -> PatternSet:
    c = _cfg(cid)
    d = C.POINTER(C.c_uint8)()
    l = C.POINTER(C.c_uint32)()
    n = C.c_uint32()
    if _lib().pg_make_patterns(C.byref(c), C.byref(d), C.byref(l), C.byref(n)) != 0:
        raise RuntimeError("pg_make_patterns failed")
    lens = np.ctypeslib.as_array(l, shape=(n.value,)).copy()
    total = int(lens.sum(dtype=np.uint64))
    data = np.ctypeslib.as_array(d, shape=(max(total, 1),))[:total].copy()
    _lib().pg_free(C.cast(d, C.c_void_p))
    _lib().pg_free(C.cast(l, C.c_void_p))
    return PatternSet(data, lens)


def text(cid: int, start: int = 0, length: int | None = None, threads: int = 0, out=None) -> np.ndarray:
    """Bytes [start, start+length) of config cid's text (default: full size).
    `out` may be a preallocated uint8 buffer (numpy array or a pinned tensor's numpy view)."""
    c = _cfg(cid)
    if length is None:
        length = int(c.text_len) - start
    ps = patterns(cid)
    if out is None:
        out = np.empty(length, dtype=np.uint8)
    assert out.dtype == np.uint8 and out.flags["C_CONTIGUOUS"] and out.size >= length
    rc = _lib().pg_make_text(C.byref(c), ps.data.ctypes.data, ps.lens.ctypes.data, len(ps),
                             start, length, out.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError("pg_make_text failed")
    return out[:length]


def plants(cid: int, chunk_lo: int, chunk_hi: int):
    """Planted (pos, pid) in chunks [chunk_lo, chunk_hi), position order."""
    c = _cfg(cid)
    ps = patterns(cid)
    pp = C.POINTER(C.c_uint64)()
    pq = C.POINTER(C.c_uint32)()
    n = C.c_uint64()
    if _lib().pg_plants(C.byref(c), ps.data.ctypes.data, ps.lens.ctypes.data, len(ps), chunk_lo,
                        chunk_hi, C.byref(pp), C.byref(pq), C.byref(n)) != 0:
        raise RuntimeError("pg_plants failed")
    k = n.value
    pos = np.ctypeslib.as_array(pp, shape=(max(k, 1),))[:k].copy()
    pid = np.ctypeslib.as_array(pq, shape=(max(k, 1),))[:k].copy()
    _lib().pg_free(C.cast(pp, C.c_void_p))
    _lib().pg_free(C.cast(pq, C.c_void_p))
    return pos, pid


def mt64_outputs(seed: int, n: int) -> list[int]:
    m = _MT()
    _lib().pg_mt64_seed(C.byref(m), seed)
    return [_lib().pg_mt64_next(C.byref(m)) for _ in range(n)]


def splitmix64_outputs(state: int, n: int) -> list[int]:
    s = C.c_uint64(state)
    return [_lib().pg_splitmix64_next(C.byref(s)) for _ in range(n)]
