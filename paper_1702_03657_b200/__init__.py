"""paper_1702_03657_b200 -- B200-native PFAC scan over a CSR-compressed trie.

Thin Python binding (argument marshalling only) over the C ABI of
``libpfac.so`` (include/pfac.h).  Every step of the scan runs in the library's
sm_100a kernels; there is no CPU or PyTorch fallback: if the shared library is
missing this module raises on first use, and if no CUDA device is usable the
match calls raise ``PfacError`` (PFAC_ERR_CUDA).  PyTorch is used only for
device memory, streams and (in ``multigpu``) process groups.

    trie = Trie([b"he", b"she", b"his", b"hers"])
    pos, pid = trie.match(torch.frombuffer(bytearray(b"ushers"), dtype=torch.uint8).cuda())
    # pos = [1, 2, 2], pid = [1, 0, 3]   (PAPER.md:62 problem, PAPER.md:76 PFAC)
"""
from __future__ import annotations

import ctypes as C
import functools
import os

import numpy as np

__all__ = ["Trie", "Scanner", "PfacError", "BYTES_KINDS", "lib_path", "launches_per_call", "build_options",
           "plan_options", "PLACEMENTS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("PFAC_LIB") or os.path.join(_HERE, "libpfac.so")  # PFAC_LIB: instrumented build

PFAC_OK = 0
_STATUS = {0: "PFAC_OK", 1: "PFAC_ERR_INVALID_ARG", 2: "PFAC_ERR_LIMIT", 3: "PFAC_ERR_NOMEM",
           4: "PFAC_ERR_CUDA", 5: "PFAC_ERR_CAPACITY"}
BYTES_KINDS = {"device_image": 0, "uncompressed": 1, "dense_stt": 2, "paper_crs": 3, "csr_core": 4, "truncated": 5,
               "merged": 6, "merged_crs": 7, "merged_image": 8, "pipe_trunc": 9, "pipe_merged": 10, "pipe_crs": 11}
FORMS = {"csr_trie": 0, "merged_dag": 1}


class PfacError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {detail}")


class _Stats(C.Structure):
    _fields_ = [("nodes", C.c_uint64), ("edges", C.c_uint64), ("terminals", C.c_uint64),
                ("n_patterns", C.c_uint32), ("max_len", C.c_uint32), ("min_len", C.c_uint32),
                ("filter_gram", C.c_uint32), ("filter_log2_bits", C.c_uint32), ("image_nodes", C.c_uint32),
                ("truncate_depth", C.c_uint32), ("verify_candidates", C.c_uint32)]


class _Matches(C.Structure):
    _fields_ = [("count", C.c_uint64), ("pos", C.POINTER(C.c_uint64)), ("pid", C.POINTER(C.c_uint32))]


class BuildOptions(C.Structure):
    """pfac_build_options (include/pfac.h); fields set from keyword arguments."""
    _fields_ = [("struct_bytes", C.c_uint32), ("filter_kind", C.c_int32), ("pair_bits_per_key", C.c_uint32),
                ("gram8_bits_per_key", C.c_uint32), ("truncate_depth", C.c_uint32), ("merge_suffixes", C.c_uint32),
                ("reserved", C.c_uint32 * 6)]


class PlanOptions(C.Structure):
    """pfac_plan_options (include/pfac.h); fields set from keyword arguments."""
    _fields_ = [("struct_bytes", C.c_uint32), ("placement", C.c_uint32), ("hot_bytes_cap", C.c_uint32),
                ("max_filter_rep_log2", C.c_int32), ("ring_slots", C.c_int32), ("ctg64", C.c_int32),
                ("pool64", C.c_int32), ("stage2", C.c_int32), ("entry", C.c_int32), ("l2_persist", C.c_uint32),
                ("form", C.c_uint32), ("cluster", C.c_uint32), ("reserved", C.c_uint32 * 4)]


class _PlanInfo(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "filter_kind", "ring_slots", "filter_copies", "smem_bytes", "hot_nodes", "image_nodes", "hot_edges",
        "terms_in_smem", "grid", "warps_per_cta", "hit_cap", "stage2", "entry", "kset", "pool_rounds",
        "placement")] + [("rounds_per_cta", C.c_uint64), ("main_rounds", C.c_uint64), ("cluster", C.c_uint32),
                         ("dsm_nodes", C.c_uint32)]


PLACEMENTS = {"auto": 0, "global": 1, "smem": 2, "big_l1": 3, "cluster": 4}


def build_options(**kw) -> BuildOptions:
    o = BuildOptions()
    _lib().pfac_build_options_init(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, int(v))
    return o


def plan_options(**kw) -> PlanOptions:
    o = PlanOptions()
    _lib().pfac_plan_options_init(C.byref(o))
    for k, v in kw.items():
        if isinstance(v, str):
            v = PLACEMENTS[v] if k == "placement" else FORMS[v]
        setattr(o, k, int(v))
    return o


@functools.lru_cache(None)
def _lib():
    if not os.path.exists(lib_path):
        raise RuntimeError(f"{lib_path} is missing: the CUDA library must be built "
                           f"(`make` or __graft_entry__.build()); there is no fallback")
    L = C.CDLL(lib_path)
    vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
    L.pfac_build_concat.argtypes = [vp, vp, u32, C.POINTER(vp)]
    L.pfac_free.argtypes = [vp]
    L.pfac_free.restype = None
    L.pfac_trie_bytes.argtypes = [vp, C.c_int, C.POINTER(u64)]
    L.pfac_trie_stats.argtypes = [vp, C.POINTER(_Stats)]
    L.pfac_image.argtypes = [vp, C.POINTER(vp), C.POINTER(u64)]
    L.pfac_attach.argtypes = [vp, u64, C.c_int, C.POINTER(vp)]
    L.pfac_match.argtypes = [vp, vp, u64, C.POINTER(_Matches)]
    L.pfac_matches_free.argtypes = [C.POINTER(_Matches)]
    L.pfac_matches_free.restype = None
    L.pfac_workspace_bytes.argtypes = [vp, u64, C.POINTER(u64)]
    L.pfac_match_device.argtypes = [vp, C.c_int, vp, u64, u64, u64, vp, vp, u64, vp, vp, u64, vp]
    L.pfac_match_device_ex.argtypes = [vp, C.c_int, vp, u64, u64, u64, vp, vp, u64, vp, vp, u64, vp, vp]
    L.pfac_build_ex.argtypes = [vp, vp, u32, vp, C.POINTER(vp)]
    L.pfac_build_options_init.argtypes = [vp]
    L.pfac_build_options_init.restype = None
    L.pfac_plan_options_init.argtypes = [vp]
    L.pfac_plan_options_init.restype = None
    L.pfac_plan_query.argtypes = [vp, C.c_int, u64, vp, vp]
    L.pfac_launches_per_call.restype = u32
    L.pfac_status_string.restype = C.c_char_p
    L.pfac_last_error.restype = C.c_char_p
    L.pfac_version.restype = C.c_char_p
    return L


def _check(st: int, where: str):
    if st != PFAC_OK:
        raise PfacError(st, where, _lib().pfac_last_error().decode(errors="replace"))


def launches_per_call() -> int:
    return int(_lib().pfac_launches_per_call())


def _concat(patterns):
    if hasattr(patterns, "data") and hasattr(patterns, "lens"):
        return np.ascontiguousarray(patterns.data, np.uint8), np.ascontiguousarray(patterns.lens, np.uint32)
    pats = [bytes(p) for p in patterns]
    data = np.frombuffer(b"".join(pats), dtype=np.uint8).copy() if pats else np.zeros(0, np.uint8)
    return data, np.array([len(p) for p in pats], dtype=np.uint32)


class Trie:
    """Handle over ``pfac_trie`` (immutable; thread-safe for concurrent matches)."""

    def __init__(self, patterns=None, *, _handle=None, **build_kw):
        """build_kw: pfac_build_options fields (filter_kind, pair_bits_per_key,
        gram8_bits_per_key, truncate_depth); none = pfac_build_concat defaults."""
        if _handle is not None:
            self._h = _handle
            return
        data, lens = _concat(patterns if patterns is not None else [])
        h = C.c_void_p()
        dp, lp = (data.ctypes.data if data.size else None), (lens.ctypes.data if lens.size else None)
        if build_kw:
            o = build_options(**build_kw)
            st = _lib().pfac_build_ex(dp, lp, int(lens.size), C.byref(o), C.byref(h))
        else:
            st = _lib().pfac_build_concat(dp, lp, int(lens.size), C.byref(h))
        _check(st, "pfac_build")
        self._h = h

    @classmethod
    def attach(cls, image, device: int = -1) -> "Trie":
        """From a serialised image: bytes / numpy uint8 / torch uint8 tensor (host or CUDA)."""
        keep = image
        if isinstance(image, (bytes, bytearray)):
            keep = np.frombuffer(bytes(image), np.uint8)
        if isinstance(keep, np.ndarray):
            ptr, size = keep.ctypes.data, keep.nbytes
        else:  # torch tensor
            ptr, size = keep.data_ptr(), keep.numel() * keep.element_size()
        h = C.c_void_p()
        _check(_lib().pfac_attach(ptr, size, device, C.byref(h)), "pfac_attach")
        return cls(_handle=h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib().pfac_free(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------ metadata
    def stats(self) -> dict:
        s = _Stats()
        _check(_lib().pfac_trie_stats(self._h, C.byref(s)), "pfac_trie_stats")
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def nbytes(self, kind: str = "device_image") -> int:
        v = C.c_uint64()
        _check(_lib().pfac_trie_bytes(self._h, BYTES_KINDS[kind], C.byref(v)), "pfac_trie_bytes")
        return int(v.value)

    def image(self) -> bytes:
        p, n = C.c_void_p(), C.c_uint64()
        _check(_lib().pfac_image(self._h, C.byref(p), C.byref(n)), "pfac_image")
        return C.string_at(p, n.value)

    def plan(self, n_starts: int, device: int = 0, **plan_kw) -> dict:
        """pfac_plan_query: the plan a scan of n_starts starts would use."""
        o = plan_options(**plan_kw)
        info = _PlanInfo()
        _check(_lib().pfac_plan_query(self._h, device, n_starts, C.byref(o), C.byref(info)), "pfac_plan_query")
        return {f: getattr(info, f) for f, _ in _PlanInfo._fields_}

    def workspace_bytes(self, n_starts: int) -> int:
        v = C.c_uint64()
        _check(_lib().pfac_workspace_bytes(self._h, n_starts, C.byref(v)), "pfac_workspace_bytes")
        return int(v.value)

    # --------------------------------------------------------- host match
    def match_host(self, text):
        """pfac_match: host text in, host (pos uint64, pid uint32) numpy arrays out."""
        t = np.frombuffer(bytes(text), np.uint8) if isinstance(text, (bytes, bytearray)) else \
            np.ascontiguousarray(text, dtype=np.uint8)
        m = _Matches()
        _check(_lib().pfac_match(self._h, t.ctypes.data if t.size else None, t.size, C.byref(m)), "pfac_match")
        n = int(m.count)
        pos = np.ctypeslib.as_array(m.pos, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
        pid = np.ctypeslib.as_array(m.pid, shape=(n,)).copy() if n else np.zeros(0, np.uint32)
        _lib().pfac_matches_free(C.byref(m))
        return pos, pid

    # ------------------------------------------------------- device match
    def match_device(self, d_text, readable_len, n_starts, pos_base, d_pos, d_pid, capacity, d_count,
                     d_ws, ws_bytes, stream=None, device=None, plan=None):
        """Raw pfac_match_device(_ex) on torch tensors / raw pointers (stream-ordered).
        `plan`: a PlanOptions (None = automatic)."""
        import torch
        ptr = (lambda x: x if isinstance(x, int) or x is None else x.data_ptr())
        if device is None:
            device = d_text.device.index if hasattr(d_text, "device") else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        with torch.cuda.device(device):  # the ABI requires `device` to be current
            st = _lib().pfac_match_device_ex(self._h, device, ptr(d_text), readable_len, n_starts, pos_base,
                                             ptr(d_pos), ptr(d_pid), capacity, ptr(d_count), ptr(d_ws), ws_bytes,
                                             C.byref(plan) if plan is not None else None, stream)
        _check(st, "pfac_match_device")

    def match(self, text, readable_len=None, n_starts=None, pos_base=0, capacity=None, **plan_kw):
        """Scan a CUDA uint8 tensor; returns (pos int64, pid int32) CUDA tensors sorted by (pos, pid).
        Count-and-retry when the match count exceeds the first capacity guess.
        plan_kw: pfac_plan_options fields (placement=..., stage2=0, ...)."""
        return Scanner(self, text.device, **plan_kw).match(text, readable_len, n_starts, pos_base, capacity)


class Scanner:
    """Reusable device state for repeated scans on one device: zero-initialised
    workspace, output buffers and a device count (what bench.py times)."""

    def __init__(self, trie: Trie, device, capacity: int = 1 << 16, **plan_kw):
        import torch
        self.torch = torch
        self.trie = trie
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.plan = plan_options(**plan_kw) if plan_kw else None
        self.ws = None
        self.ws_bytes = 0
        with torch.cuda.device(self.device):
            self.count = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.cap = 0
        self._ensure_out(capacity)

    def _ensure_ws(self, n_starts):
        # allocated and zero-filled on the device's current stream; launch()
        # orders a foreign stream after it
        need = self.trie.workspace_bytes(max(n_starts, 1))
        if self.ws is None or need > self.ws_bytes:
            self.ws = self.torch.zeros(need, dtype=self.torch.uint8, device=self.device)
            self.ws_bytes = need

    def _ensure_out(self, cap):
        cap = max(int(cap), 1)
        if cap > self.cap:
            self.pos = self.torch.empty(cap, dtype=self.torch.int64, device=self.device)
            self.pid = self.torch.empty(cap, dtype=self.torch.int32, device=self.device)
            self.cap = cap

    def launch(self, text, readable_len=None, n_starts=None, pos_base=0, stream=None):
        """One stream-ordered scan into the preallocated buffers (no sync).
        `stream` (default: the device's current stream) is ordered after the
        current stream's allocation/zero-fill of the buffers, and the buffers
        are recorded on it so the caching allocator never recycles them early."""
        torch = self.torch
        assert text.dtype == torch.uint8 and text.is_cuda and text.is_contiguous()
        L = text.numel() if readable_len is None else int(readable_len)
        ns = L if n_starts is None else int(n_starts)
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream()
            self._ensure_ws(ns)
            if stream is not None and stream != cur:
                stream.wait_stream(cur)
                for b in (self.ws, self.pos, self.pid, self.count, text):
                    b.record_stream(stream)
            self.trie.match_device(text, L, ns, pos_base, self.pos, self.pid, self.cap, self.count, self.ws,
                                   self.ws_bytes, stream=stream, device=self.device.index, plan=self.plan)

    def match(self, text, readable_len=None, n_starts=None, pos_base=0, capacity=None):
        L = text.numel() if readable_len is None else int(readable_len)
        if capacity is not None:
            self._ensure_out(capacity)
        else:
            self._ensure_out(max(self.cap, L // 512 + 1024))
        self.launch(text, readable_len, n_starts, pos_base)
        n = int(self.count.item())
        if n > self.cap:
            self._ensure_out(n)
            self.launch(text, readable_len, n_starts, pos_base)
            n2 = int(self.count.item())
            assert n2 == n, "match count changed between identical scans"
        return self.pos[:n].clone(), self.pid[:n].clone()
