"""ctypes binding of the C-ABI (include/trilist_b200.h).

This is the thinnest host layer over ``lib/libtrilist_b200.so``: what a
reference-side FFI (ctypes/cffi) would bind.  ``bench.py`` and the C-ABI
parity tests use it; the reference-shaped API is ``paper_2006_11494_b200.trilist``.
The library is required: importing a compute entry point without it raises.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TL_LIB_PATH") or os.path.join(PKG, "lib", "libtrilist_b200.so")

(TL_OK, TL_EINVAL, TL_ERANGE, TL_ELOGIC, TL_ECUDA, TL_ENOMEM, TL_ECAPACITY, TL_ENODEV, TL_EPARSE, TL_ELENGTH,
 TL_EIO, TL_ECANCELED) = range(12)

# tl_batch_fn: int (*)(void* user, const uint32_t* triples, uint64_t count)
BATCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint32), C.c_uint64)

# Every symbol include/trilist_b200.h declares (checked by tests/test_cabi_symbols.py).
EXPORTS = (
    "tl_last_error", "tl_device_count", "tl_version",
    "tl_gen_er", "tl_gen_rmat", "tl_chung_lu_prefix", "tl_gen_chung_lu",
    "tl_graph_from_pairs", "tl_graph_free", "tl_graph_info", "tl_graph_degrees", "tl_graph_csr",
    "tl_graph_from_text", "tl_graph_from_file", "tl_degree_order", "tl_orient", "tl_oriented_from_csr", "tl_oriented_free", "tl_oriented_info",
    "tl_oriented_csr", "tl_cost_model", "tl_aot_count", "tl_aot_hash", "tl_aot_list",
    "tl_run_count", "tl_run_hash", "tl_run_list", "tl_run_list_device", "tl_run_list_batches", "tl_verify", "tl_degeneracy_order", "tl_random_order",
    "tl_brute_force", "tl_multi_create", "tl_multi_free", "tl_multi_count", "tl_multi_hash", "tl_multi_list",
    "tl_fold_parts",
)

# TL_ALGO_* (Algorithm, engine.hpp:18) by the reference's names (engine.cpp:7-15).
ALGO_CODES = {"aot": 0, "cf": 1, "cf-hash": 2, "kclist": 3}


class TlStats(C.Structure):
    _fields_ = [
        ("triangles", C.c_uint64), ("probes", C.c_uint64), ("merge_comparisons", C.c_uint64),
        ("table_builds", C.c_uint64), ("positive_triangles", C.c_uint64), ("negative_triangles", C.c_uint64),
        ("probes_executed", C.c_uint64), ("hash_sum", C.c_uint64), ("hash_xor", C.c_uint64),
        ("tasks", C.c_uint64), ("list_ms", C.c_double), ("prep_ms", C.c_double), ("kernel_launches", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


VERIFY_SAMPLES = 32  # TL_VERIFY_SAMPLES


class TlVerifyResult(C.Structure):
    _fields_ = [("algorithm", C.c_uint32), ("pass_", C.c_uint32), ("unique_triangles", C.c_uint64),
                ("duplicate_emissions", C.c_uint64), ("missing_count", C.c_uint64), ("extra_count", C.c_uint64),
                ("n_missing_samples", C.c_uint32), ("n_extra_samples", C.c_uint32),
                ("missing_samples", C.c_uint32 * (3 * VERIFY_SAMPLES)),
                ("extra_samples", C.c_uint32 * (3 * VERIFY_SAMPLES)), ("stats", TlStats)]

    def as_dict(self) -> dict:
        names = {v: k for k, v in ALGO_CODES.items()}
        ms = [tuple(self.missing_samples[3 * i:3 * i + 3]) for i in range(self.n_missing_samples)]
        es = [tuple(self.extra_samples[3 * i:3 * i + 3]) for i in range(self.n_extra_samples)]
        return {"algorithm": names[self.algorithm], "pass": bool(self.pass_),
                "unique_triangles": self.unique_triangles, "duplicate_emissions": self.duplicate_emissions,
                "missing_count": self.missing_count, "extra_count": self.extra_count,
                "missing_samples": ms, "extra_samples": es, "stats": self.stats.as_dict()}


class TlLoadDiag(C.Structure):
    _fields_ = [("lines_read", C.c_uint64), ("edges_parsed", C.c_uint64), ("self_loops_dropped", C.c_uint64),
                ("duplicates_dropped", C.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class TlRunOptions(C.Structure):
    _fields_ = [("skip_negative_phase", C.c_uint32), ("check_hygiene", C.c_uint32), ("part", C.c_uint32),
                ("nparts", C.c_uint32), ("stream", C.c_void_p), ("algorithm", C.c_uint32),
                ("cf_hash_reuse_last_table", C.c_uint32)]


class TlError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[TL error {code}] {msg}")
        self.code = code


class TlParseError(TlError, ValueError):
    def __init__(self, msg: str, line: int):
        TlError.__init__(self, TL_EPARSE, msg)
        self.line = line


u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


@lru_cache(None)
def lib() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    L.tl_last_error.restype = C.c_char_p
    L.tl_version.restype = C.c_char_p
    L.tl_device_count.argtypes = [C.POINTER(C.c_int)]
    L.tl_gen_er.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, vp, vp]
    L.tl_gen_rmat.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, vp, vp]
    L.tl_chung_lu_prefix.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, u64p]
    L.tl_gen_chung_lu.argtypes = [C.c_uint64, C.c_uint32, u64p, C.c_uint64, vp, vp]
    L.tl_graph_from_pairs.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_int, C.c_int, vp, C.POINTER(vp)]
    L.tl_graph_from_text.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.c_int, C.POINTER(vp),
                                     C.POINTER(TlLoadDiag), u64p]
    L.tl_graph_from_file.argtypes = [C.c_char_p, C.c_uint32, C.c_char_p, C.c_int, C.POINTER(vp),
                                     C.POINTER(TlLoadDiag), u64p]
    L.tl_graph_free.argtypes = [vp]
    L.tl_graph_info.argtypes = [vp, u32p, u64p, u64p, u64p]
    L.tl_graph_degrees.argtypes = [vp, u32p]
    L.tl_graph_csr.argtypes = [vp, u64p, u32p]
    L.tl_degree_order.argtypes = [vp, u32p]
    L.tl_orient.argtypes = [vp, u32p, C.POINTER(vp)]
    L.tl_oriented_from_csr.argtypes = [C.c_uint32, C.c_uint64, vp, vp, vp, C.c_int, vp, C.POINTER(vp)]
    L.tl_oriented_free.argtypes = [vp]
    L.tl_oriented_info.argtypes = [vp, u32p, u64p, u32p]
    L.tl_oriented_csr.argtypes = [vp, u64p, u32p, u64p, u32p, u32p]
    L.tl_cost_model.argtypes = [vp, u64p]
    L.tl_aot_count.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_aot_hash.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_aot_list.argtypes = [vp, C.POINTER(TlRunOptions), u32p, C.c_uint64, C.c_int, C.POINTER(TlStats)]
    L.tl_run_count.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_run_hash.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_run_list.argtypes = [vp, C.POINTER(TlRunOptions), u32p, C.c_uint64, C.c_int, C.POINTER(TlStats)]
    L.tl_run_list_batches.argtypes = [vp, C.POINTER(TlRunOptions), C.c_uint64, C.c_uint32, BATCH_FN, vp,
                                      C.POINTER(TlStats)]
    L.tl_run_list_device.argtypes = [vp, C.POINTER(TlRunOptions), vp, C.c_uint64, C.c_int, C.POINTER(TlStats)]
    L.tl_verify.argtypes = [vp, u32p, C.c_uint32, C.POINTER(TlRunOptions), u32p, C.c_uint64, C.c_int,
                            C.POINTER(TlVerifyResult), u64p]
    L.tl_degeneracy_order.argtypes = [vp, u32p]
    L.tl_random_order.argtypes = [C.c_uint32, C.c_uint64, u32p]
    L.tl_brute_force.argtypes = [vp, C.c_uint32, u32p, C.c_uint64, u64p]
    L.tl_multi_create.argtypes = [vp, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
    L.tl_multi_free.argtypes = [vp]
    L.tl_multi_count.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_multi_hash.argtypes = [vp, C.POINTER(TlRunOptions), C.POINTER(TlStats)]
    L.tl_multi_list.argtypes = [vp, C.POINTER(TlRunOptions), u32p, C.c_uint64, C.POINTER(TlStats)]
    L.tl_fold_parts.argtypes = [C.POINTER(TlStats), C.c_uint32, C.POINTER(TlStats), u64p]
    return L


def _check(rc: int) -> None:
    if rc != TL_OK:
        raise TlError(rc, lib().tl_last_error().decode())


def _p32(a):
    return a.ctypes.data_as(u32p) if a is not None else None


def _p64(a):
    return a.ctypes.data_as(u64p) if a is not None else None


def device_count() -> int:
    c = C.c_int()
    _check(lib().tl_device_count(C.byref(c)))
    return c.value


def version() -> str:
    return lib().tl_version().decode()


# ------------------------------------------------------------- generators
def gen_pairs_device(cfg: dict, d_ptr: int, stream: int = 0) -> None:
    """Writes cfg's 2*npairs uint32 pairs into device memory at d_ptr."""
    kind = cfg["kind"]
    if kind == "er":
        _check(lib().tl_gen_er(cfg["seed"], cfg["n"], cfg["npairs"], d_ptr, stream or None))
    elif kind == "rmat":
        _check(lib().tl_gen_rmat(cfg["seed"], cfg["scale"], cfg["npairs"], d_ptr, stream or None))
    elif kind == "chung_lu":
        pre = chung_lu_prefix(cfg["seed"], cfg["n"], cfg["avg"], cfg["gamma"])
        _check(lib().tl_gen_chung_lu(cfg["seed"], cfg["n"], _p64(pre), cfg["npairs"], d_ptr, stream or None))
    else:
        raise ValueError(kind)


def chung_lu_prefix(seed: int, n: int, avg: float, gamma: float) -> np.ndarray:
    pre = np.empty(n + 1, np.uint64)
    _check(lib().tl_chung_lu_prefix(seed, n, avg, gamma, _p64(pre)))
    return pre


# ------------------------------------------------------------- handles
class DeviceGraph:
    """tl_graph: Graph::from_edges on the device."""

    def __init__(self, handle):
        self._h = handle
        n, m, d, s = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().tl_graph_info(handle, C.byref(n), C.byref(m), C.byref(d), C.byref(s)))
        self.n, self.m, self.duplicates, self.self_loops = n.value, m.value, d.value, s.value

    @classmethod
    def from_pairs(cls, pairs: np.ndarray, min_vertices: int = 0, device: int = 0) -> "DeviceGraph":
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        h = vp()
        _check(lib().tl_graph_from_pairs(pairs.ctypes.data if pairs.size else None, pairs.shape[0], min_vertices,
                                         device, 0, None, C.byref(h)))
        return cls(h)

    @classmethod
    def from_text(cls, text, one_indexed=False, compact_ids=False, comments="#%", device=0):
        """load_edge_list_text on the device: returns (DeviceGraph, diagnostics)."""
        if isinstance(text, str):
            text = text.encode()
        h, diag, line = vp(), TlLoadDiag(), C.c_uint64()
        flags = (1 if one_indexed else 0) | (2 if compact_ids else 0)
        rc = lib().tl_graph_from_text(text, len(text), flags, comments.encode(), device, C.byref(h), C.byref(diag),
                                      C.byref(line))
        if rc == TL_EPARSE:
            raise TlParseError(lib().tl_last_error().decode(), line.value)
        _check(rc)
        return cls(h), diag.as_dict()

    @classmethod
    def from_file(cls, path, one_indexed=False, compact_ids=False, comments="#%", device=0):
        h, diag, line = vp(), TlLoadDiag(), C.c_uint64()
        flags = (1 if one_indexed else 0) | (2 if compact_ids else 0)
        rc = lib().tl_graph_from_file(str(path).encode(), flags, comments.encode(), device, C.byref(h),
                                      C.byref(diag), C.byref(line))
        if rc == TL_EPARSE:
            raise TlParseError(lib().tl_last_error().decode(), line.value)
        _check(rc)
        return cls(h), diag.as_dict()

    @classmethod
    def from_device_pairs(cls, d_ptr: int, npairs: int, min_vertices: int, device: int = 0,
                          stream: int = 0) -> "DeviceGraph":
        h = vp()
        _check(lib().tl_graph_from_pairs(d_ptr, npairs, min_vertices, device, 1, stream or None, C.byref(h)))
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            lib().tl_graph_free(self._h)
            self._h = None

    __del__ = close

    def degrees(self) -> np.ndarray:
        d = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tl_graph_degrees(self._h, _p32(d)))
        return d[: self.n]

    def csr(self):
        off = np.empty(self.n + 1, np.uint64)
        adj = np.empty(max(2 * self.m, 1), np.uint32)
        _check(lib().tl_graph_csr(self._h, _p64(off), _p32(adj)))
        return off, adj[: 2 * self.m]

    def degree_order(self) -> np.ndarray:
        r = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tl_degree_order(self._h, _p32(r)))
        return r[: self.n]

    def degeneracy_order(self) -> np.ndarray:
        r = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tl_degeneracy_order(self._h, _p32(r)))
        return r[: self.n]

    def random_order(self, seed: int) -> np.ndarray:
        r = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tl_random_order(self.n, seed, _p32(r)))
        return r[: self.n]

    def make_order(self, spec: str) -> np.ndarray:
        """make_order(parse_order_spec(spec)) -- ordering.cpp:122-141."""
        if spec == "id":
            return np.arange(self.n, dtype=np.uint32)
        if spec == "degree":
            return self.degree_order()
        if spec == "degeneracy":
            return self.degeneracy_order()
        if spec.startswith("random:"):
            return self.random_order(int(spec[7:]))
        raise ValueError(f"unknown order '{spec}'")

    def orient(self, rank: np.ndarray | None = None) -> "DeviceOriented":
        h = vp()
        if rank is not None:
            rank = np.ascontiguousarray(rank, np.uint32)
        _check(lib().tl_orient(self._h, _p32(rank) if rank is not None else None, C.byref(h)))
        return DeviceOriented(h)

    def brute_force(self, max_vertices: int = 2000) -> np.ndarray:
        cnt = C.c_uint64()
        _check(lib().tl_brute_force(self._h, max_vertices, None, 0, C.byref(cnt)))
        out = np.empty((max(cnt.value, 1), 3), np.uint32)
        _check(lib().tl_brute_force(self._h, max_vertices, _p32(out), cnt.value, C.byref(cnt)))
        return out[: cnt.value]


def run_options(skip_negative=False, part=0, nparts=1, stream=0, algo="aot", reuse=False) -> TlRunOptions:
    return TlRunOptions(int(skip_negative), 0, part, nparts, stream or None, ALGO_CODES[algo], int(reuse))


class DeviceOriented:
    """tl_oriented: the oriented graph in rank space + AOT claims."""

    def __init__(self, handle):
        self._h = handle
        n, m, d = C.c_uint32(), C.c_uint64(), C.c_uint32()
        _check(lib().tl_oriented_info(handle, C.byref(n), C.byref(m), C.byref(d)))
        self.n, self.m, self.max_out_degree = n.value, m.value, d.value

    @classmethod
    def from_csr(cls, n: int, out_offsets: np.ndarray, out: np.ndarray, rank: np.ndarray, device: int = 0,
                 stream: int = 0) -> "DeviceOriented":
        h = vp()
        out_offsets = np.ascontiguousarray(out_offsets, np.uint64)
        out = np.ascontiguousarray(out, np.uint32)
        rank = np.ascontiguousarray(rank, np.uint32)
        _check(lib().tl_oriented_from_csr(n, out.size, out_offsets.ctypes.data, out.ctypes.data if out.size else None,
                                          rank.ctypes.data, device, stream or None, C.byref(h)))
        return cls(h)

    @classmethod
    def from_host_ptrs(cls, n: int, m: int, off_ptr: int, out_ptr: int, rank_ptr: int, device: int = 0,
                       stream: int = 0) -> "DeviceOriented":
        """Same as from_csr over raw host pointers (e.g. pinned torch tensors)."""
        h = vp()
        _check(lib().tl_oriented_from_csr(n, m, off_ptr, out_ptr, rank_ptr, device, stream or None, C.byref(h)))
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            lib().tl_oriented_free(self._h)
            self._h = None

    __del__ = close

    def csr(self) -> dict:
        n1 = self.n + 1
        out_off = np.empty(n1, np.uint64)
        in_off = np.empty(n1, np.uint64)
        out = np.empty(max(self.m, 1), np.uint32)
        inn = np.empty(max(self.m, 1), np.uint32)
        rank = np.empty(max(self.n, 1), np.uint32)
        _check(lib().tl_oriented_csr(self._h, _p64(out_off), _p32(out), _p64(in_off), _p32(inn), _p32(rank)))
        return dict(out_offsets=out_off, out=out[: self.m], in_offsets=in_off, inn=inn[: self.m],
                    rank=rank[: self.n])

    def cost_model(self) -> dict:
        c = np.zeros(3, np.uint64)
        _check(lib().tl_cost_model(self._h, _p64(c)))
        return dict(cf_cost=int(c[0]), kclist_cost=int(c[1]), aot_cost=int(c[2]))

    def verify(self, algos=("cf", "cf-hash", "kclist", "aot"), reference=None, skip_negative=False, reuse=False,
               stream=0):
        """tl_verify: (per-algorithm result dicts, baseline size)."""
        codes = np.array([ALGO_CODES[a] for a in algos], np.uint32)
        res = (TlVerifyResult * max(len(algos), 1))()
        cnt = np.zeros(1, np.uint64)
        o = run_options(skip_negative, 0, 1, stream, "aot", reuse)
        ref = None if reference is None else np.ascontiguousarray(reference, np.uint32).reshape(-1, 3)
        _check(lib().tl_verify(self._h, _p32(codes), len(algos), C.byref(o), _p32(ref) if ref is not None else None,
                               0 if ref is None else ref.shape[0], int(ref is not None), res, _p64(cnt)))
        return [res[i].as_dict() for i in range(len(algos))], int(cnt[0])

    # algo="aot" goes through tl_aot_*, the others through tl_run_* (TL_ALGO_*).
    def count(self, skip_negative=False, part=0, nparts=1, stream=0, algo="aot", reuse=False) -> dict:
        st = TlStats()
        o = run_options(skip_negative, part, nparts, stream, algo, reuse)
        fn = lib().tl_aot_count if algo == "aot" else lib().tl_run_count
        _check(fn(self._h, C.byref(o), C.byref(st)))
        return st.as_dict()

    def hash(self, skip_negative=False, part=0, nparts=1, stream=0, algo="aot", reuse=False) -> dict:
        st = TlStats()
        o = run_options(skip_negative, part, nparts, stream, algo, reuse)
        fn = lib().tl_aot_hash if algo == "aot" else lib().tl_run_hash
        _check(fn(self._h, C.byref(o), C.byref(st)))
        return st.as_dict()

    def list(self, canonical=False, skip_negative=False, part=0, nparts=1, stream=0, algo="aot", reuse=False):
        """Returns (stats, (T, 3) uint32 array)."""
        st = TlStats()
        o = run_options(skip_negative, part, nparts, stream, algo, reuse)
        fn = lib().tl_aot_list if algo == "aot" else lib().tl_run_list
        _check(fn(self._h, C.byref(o), None, 0, int(canonical), C.byref(st)))
        out = np.empty((max(st.triangles, 1), 3), np.uint32)
        _check(fn(self._h, C.byref(o), _p32(out), st.triangles, int(canonical), C.byref(st)))
        return st.as_dict(), out[: st.triangles]

    def list_batches(self, fn, batch_triples=0, host_buffers=0, skip_negative=False, part=0, nparts=1, stream=0,
                     algo="aot", reuse=False) -> dict:
        """tl_run_list_batches: fn((k, 3) uint32 array view, valid during the
        call) per batch; fn returning True stops the run (TL_ECANCELED)."""
        err = []

        def cb(_user, ptr, count):
            try:
                arr = np.ctypeslib.as_array(ptr, shape=(int(count) * 3,)).reshape(-1, 3)
                return 1 if fn(arr) else 0
            except BaseException as e:  # noqa: BLE001 -- re-raised after the run
                err.append(e)
                return 1

        st = TlStats()
        o = run_options(skip_negative, part, nparts, stream, algo, reuse)
        rc = lib().tl_run_list_batches(self._h, C.byref(o), batch_triples, host_buffers, BATCH_FN(cb), None,
                                       C.byref(st))
        if err:
            raise err[0]
        _check(rc)
        return st.as_dict()

    def list_device(self, d_triples: int, cap: int, canonical=False, skip_negative=False, part=0, nparts=1,
                    stream=0, algo="aot", reuse=False) -> dict:
        """tl_run_list_device: one listing pass into device memory d_triples
        (cap uint32 triples on this handle's device); returns the stats."""
        st = TlStats()
        o = run_options(skip_negative, part, nparts, stream, algo, reuse)
        _check(lib().tl_run_list_device(self._h, C.byref(o), C.c_void_p(d_triples), cap, int(canonical),
                                        C.byref(st)))
        return st.as_dict()


def fold_parts(parts) -> tuple[dict, list]:
    """tl_fold_parts: combine per-part stats dicts (sums mod 2^64, xor, the
    slowest part's times) -> (total dict, listing offsets)."""
    arr = (TlStats * max(len(parts), 1))()
    for i, p in enumerate(parts):
        for name, _ in TlStats._fields_:
            if name in p:
                setattr(arr[i], name, p[name])
    out = TlStats()
    offs = np.zeros(max(len(parts), 1), np.uint64)
    _check(lib().tl_fold_parts(arr, len(parts), C.byref(out), _p64(offs)))
    return out.as_dict(), [int(x) for x in offs[: len(parts)]]


class MultiOriented:
    """tl_multi: the oriented graph replicated on a device list (one process),
    each run split over the devices, results combined by NCCL."""

    def __init__(self, oriented: "DeviceOriented", devices):
        self._h = vp()
        import torch  # noqa: F401 -- loads PyTorch's NCCL first; tl_multi then shares it
        devs = (C.c_int * len(devices))(*devices)
        _check(lib().tl_multi_create(oriented._h, devs, len(devices), C.byref(self._h)))
        self._keep = oriented  # borrowed by the replica on its own device

    def close(self):
        if self._h:
            lib().tl_multi_free(self._h)
            self._h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def count(self, algo="aot", skip_negative=False) -> dict:
        st = TlStats()
        o = run_options(skip_negative, 0, 1, 0, algo)
        _check(lib().tl_multi_count(self._h, C.byref(o), C.byref(st)))
        return st.as_dict()

    def hash(self, algo="aot", skip_negative=False) -> dict:
        st = TlStats()
        o = run_options(skip_negative, 0, 1, 0, algo)
        _check(lib().tl_multi_hash(self._h, C.byref(o), C.byref(st)))
        return st.as_dict()

    def list(self, algo="aot", skip_negative=False):
        st = TlStats()
        o = run_options(skip_negative, 0, 1, 0, algo)
        _check(lib().tl_multi_list(self._h, C.byref(o), None, 0, C.byref(st)))
        out = np.empty((max(st.triangles, 1), 3), np.uint32)
        _check(lib().tl_multi_list(self._h, C.byref(o), _p32(out), st.triangles, C.byref(st)))
        return st.as_dict(), out[: st.triangles]
