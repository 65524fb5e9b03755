"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

Two checkers live here:

* ``Oracle*`` wraps ``_build/liboracle.so``, the plain-C restatement of the
  reference AOT path (``trilist_oracle.c``; every function cites the reference
  file:line it restates).
* ``Ref*`` wraps ``_ref/libtrilist_ref.so``: the UNMODIFIED reference library
  compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` together
  with ``ref_shim.cpp`` (which calls only the reference's public API).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker / CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtrilist_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def build(ref: bool = True) -> None:
    """Compile the checkers (make in oracle/).  The reference part needs
    /root/reference, which exists only in the build container."""
    targets = ["_build/liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(u32p)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(u64p)


@lru_cache(None)
def olib() -> C.CDLL:
    if not os.path.exists(ORACLE_SO):
        build(ref=False)
    L = C.CDLL(ORACLE_SO)
    L.or_fmix64.restype = C.c_uint64
    L.or_fmix64.argtypes = [C.c_uint64]
    L.or_draw.restype = C.c_uint64
    L.or_draw.argtypes = [C.c_uint64, C.c_uint64]
    L.or_triangle_hash.restype = C.c_uint64
    L.or_triangle_hash.argtypes = [C.c_uint32] * 3
    L.or_triangle_hash_xor.restype = C.c_uint64
    L.or_triangle_hash_xor.argtypes = [C.c_uint32] * 3
    L.or_vertex_word.restype = C.c_uint64
    L.or_vertex_word.argtypes = [C.c_uint32]
    L.or_permute_id.restype = C.c_uint32
    L.or_permute_id.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
    L.or_gen_er.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, u32p]
    L.or_gen_rmat.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, u32p]
    L.or_chung_lu_prefix.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, u64p]
    L.or_gen_chung_lu.argtypes = [C.c_uint64, C.c_uint32, u64p, C.c_uint64, u32p]
    L.or_gen_gnp.restype = C.c_uint64
    L.or_gen_gnp.argtypes = [C.c_uint32, C.c_double, C.c_uint64, u32p, C.c_uint64]
    L.or_from_edges.restype = C.c_void_p
    L.or_from_edges.argtypes = [C.c_uint32, u32p, C.c_uint64]
    L.or_graph_free.argtypes = [C.c_void_p]
    L.or_graph_n.restype = C.c_uint32
    L.or_graph_n.argtypes = [C.c_void_p]
    L.or_graph_m.restype = C.c_uint64
    L.or_graph_m.argtypes = [C.c_void_p]
    L.or_graph_duplicates.restype = C.c_uint64
    L.or_graph_duplicates.argtypes = [C.c_void_p]
    L.or_graph_csr.argtypes = [C.c_void_p, u64p, u32p]
    L.or_degree_order.argtypes = [C.c_void_p, u32p]
    L.or_orient.restype = C.c_void_p
    L.or_orient.argtypes = [C.c_void_p, u32p]
    L.or_oriented_free.argtypes = [C.c_void_p]
    L.or_oriented_m.restype = C.c_uint64
    L.or_oriented_m.argtypes = [C.c_void_p]
    L.or_oriented_csr.argtypes = [C.c_void_p, u64p, u32p, u64p, u32p, u32p]
    L.or_max_out_degree.restype = C.c_uint32
    L.or_max_out_degree.argtypes = [C.c_void_p]
    L.or_cost_model.argtypes = [C.c_void_p, u64p]
    L.or_aot.restype = C.c_uint64
    L.or_aot.argtypes = [C.c_void_p, C.c_int, u64p, u32p, C.c_uint64]
    L.or_brute_force.restype = C.c_uint64
    L.or_brute_force.argtypes = [C.c_void_p, u32p, C.c_uint64]
    L.or_kernel.restype = C.c_uint64
    L.or_kernel.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, u32p, C.c_uint64]
    L.or_apply_local_order.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
    L.or_degeneracy_order.argtypes = [C.c_void_p, u32p]
    L.or_random_order.argtypes = [C.c_uint32, C.c_uint64, u32p]
    return L


# --------------------------------------------------------------------------
# generators (definitions shared bit-for-bit with the GPU generators)
# --------------------------------------------------------------------------
def fmix64(z: int) -> int:
    return olib().or_fmix64(z)


def triangle_hash(a: int, b: int, c: int) -> int:
    """The triangle's hash_sum term Z(a) Z(b) Z(c) mod 2^64."""
    return olib().or_triangle_hash(a, b, c)


def triangle_hash_xor(a: int, b: int, c: int) -> int:
    """The triangle's hash_xor term Z(a) & Z(b) & Z(c)."""
    return olib().or_triangle_hash_xor(a, b, c)


def vertex_word(v: int) -> int:
    return olib().or_vertex_word(v)


def gen_er(seed: int, n: int, npairs: int) -> np.ndarray:
    out = np.empty((npairs, 2), np.uint32)
    olib().or_gen_er(seed, n, npairs, _p32(out))
    return out


def gen_rmat(seed: int, scale: int, npairs: int) -> np.ndarray:
    out = np.empty((npairs, 2), np.uint32)
    olib().or_gen_rmat(seed, scale, npairs, _p32(out))
    return out


def chung_lu_prefix(seed: int, n: int, avg: float = 32.0, gamma: float = 2.1) -> np.ndarray:
    pre = np.empty(n + 1, np.uint64)
    olib().or_chung_lu_prefix(seed, n, avg, gamma, _p64(pre))
    return pre


def gen_chung_lu(seed: int, n: int, npairs: int, avg: float = 32.0, gamma: float = 2.1) -> np.ndarray:
    pre = chung_lu_prefix(seed, n, avg, gamma)
    out = np.empty((npairs, 2), np.uint32)
    olib().or_gen_chung_lu(seed, n, _p64(pre), npairs, _p32(out))
    return out


def gen_gnp(n: int, p: float, seed: int) -> np.ndarray:
    """testutil.hpp:89-97 restated: returns the (u, v) pair list."""
    cnt = olib().or_gen_gnp(n, p, seed, None, 0)
    out = np.empty((max(cnt, 1), 2), np.uint32)
    olib().or_gen_gnp(n, p, seed, _p32(out), cnt)
    return out[:cnt]


def gen_config(cfg: dict) -> np.ndarray:
    """Pairs for a config dict from paper_2006_11494_b200.configs."""
    kind = cfg["kind"]
    if kind == "er":
        return gen_er(cfg["seed"], cfg["n"], cfg["npairs"])
    if kind == "rmat":
        return gen_rmat(cfg["seed"], cfg["scale"], cfg["npairs"])
    if kind == "chung_lu":
        return gen_chung_lu(cfg["seed"], cfg["n"], cfg["npairs"], cfg["avg"], cfg["gamma"])
    raise ValueError(kind)


def pairs_checksum(pairs: np.ndarray, chunk: int = 1 << 24) -> dict:
    """Order-sensitive checksum of a pair list: sum and xor of
    fmix64((u << 32 | v) ^ i * golden) over the pair index i (chunked)."""
    s, x = 0, 0
    for start in range(0, pairs.shape[0], chunk):
        p = pairs[start:start + chunk].astype(np.uint64)
        idx = np.arange(start, start + p.shape[0], dtype=np.uint64)
        with np.errstate(over="ignore"):
            k = (p[:, 0] << np.uint64(32)) | p[:, 1]
            k = k ^ (idx * np.uint64(0x9E3779B97F4A7C15))
            k = (k ^ (k >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            k = (k ^ (k >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            k = k ^ (k >> np.uint64(31))
            s = (s + int(np.sum(k, dtype=np.uint64))) & ((1 << 64) - 1)
        x ^= int(np.bitwise_xor.reduce(k))
    return {"sum": s, "xor": x}


# --------------------------------------------------------------------------
# fixtures (testutil.hpp:18-77 restated)
# --------------------------------------------------------------------------
def complete_graph(n):
    return n, [(u, v) for u in range(n) for v in range(u + 1, n)]


def star_graph(leaves):
    return leaves + 1, [(0, v) for v in range(1, leaves + 1)]


def path_graph(n):
    return n, [(u, u + 1) for u in range(n - 1)]


def cycle_graph(n):
    return n, [(u, (u + 1) % n) for u in range(n)]


def diamond_graph():
    return 4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]


def paired_hubs_graph():
    return 14, [(0, 6), (1, 9), (2, 7), (3, 10), (4, 8), (5, 11), (6, 9), (7, 10), (8, 11),
                (6, 12), (6, 13), (7, 12), (7, 13), (8, 12), (8, 13), (9, 12), (9, 13),
                (10, 12), (10, 13), (11, 12), (11, 13)]


def as_pairs(edges) -> np.ndarray:
    a = np.asarray(edges, dtype=np.uint32)
    return a.reshape(-1, 2) if a.size else np.zeros((0, 2), np.uint32)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
STAT_KEYS = ("triangles", "probes", "merge_comparisons", "table_builds",
             "positive_triangles", "negative_triangles")


class OracleGraph:
    """Graph::from_edges restated (graph.cpp:158-206)."""

    def __init__(self, min_vertices: int, pairs):
        pairs = np.ascontiguousarray(as_pairs(pairs) if not isinstance(pairs, np.ndarray) else pairs,
                                     dtype=np.uint32)
        self._h = olib().or_from_edges(min_vertices, _p32(pairs), pairs.shape[0])
        self.n = olib().or_graph_n(self._h)
        self.m = olib().or_graph_m(self._h)
        self.duplicates = olib().or_graph_duplicates(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            olib().or_graph_free(self._h)
            self._h = None

    def csr(self):
        off = np.empty(self.n + 1, np.uint64)
        adj = np.empty(max(2 * self.m, 1), np.uint32)
        olib().or_graph_csr(self._h, _p64(off), _p32(adj))
        return off, adj[: 2 * self.m]

    def degree_order(self) -> np.ndarray:
        rank = np.empty(max(self.n, 1), np.uint32)
        olib().or_degree_order(self._h, _p32(rank))
        return rank[: self.n]

    def degeneracy_order(self) -> np.ndarray:
        rank = np.empty(max(self.n, 1), np.uint32)
        olib().or_degeneracy_order(self._h, _p32(rank))
        return rank[: self.n]

    def random_order(self, seed: int) -> np.ndarray:
        rank = np.empty(max(self.n, 1), np.uint32)
        olib().or_random_order(self.n, seed, _p32(rank))
        return rank[: self.n]

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

    def orient(self, rank=None) -> "OracleOriented":
        rank = self.degree_order() if rank is None else np.ascontiguousarray(rank, np.uint32)
        h = olib().or_orient(self._h, _p32(rank))
        if not h:
            raise ValueError("order is not a permutation of the vertex set")
        return OracleOriented(h, self.n)

    def brute_force(self) -> np.ndarray:
        cnt = olib().or_brute_force(self._h, None, 0)
        out = np.empty((max(cnt, 1), 3), np.uint32)
        olib().or_brute_force(self._h, _p32(out), cnt)
        return out[:cnt]


class OracleOriented:
    def __init__(self, h, n):
        self._h = h
        self.n = n
        self.m = olib().or_oriented_m(h)

    def __del__(self):
        if getattr(self, "_h", None):
            olib().or_oriented_free(self._h)
            self._h = None

    def csr(self):
        n1 = self.n + 1
        out_off = np.empty(n1, np.uint64)
        in_off = np.empty(n1, np.uint64)
        out = np.empty(max(self.m, 1), np.uint32)
        inn = np.empty(max(self.m, 1), np.uint32)
        rank = np.empty(max(self.n, 1), np.uint32)
        olib().or_oriented_csr(self._h, _p64(out_off), _p32(out), _p64(in_off), _p32(inn), _p32(rank))
        return dict(out_offsets=out_off, out=out[: self.m], in_offsets=in_off, inn=inn[: self.m],
                    rank=rank[: self.n])

    def max_out_degree(self) -> int:
        return olib().or_max_out_degree(self._h)

    def cost_model(self) -> dict:
        out = np.zeros(3, np.uint64)
        olib().or_cost_model(self._h, _p64(out))
        return dict(cf_cost=int(out[0]), kclist_cost=int(out[1]), aot_cost=int(out[2]))

    def aot(self, skip_negative=False, collect=False):
        """Returns (stats dict incl. hash_sum/hash_xor, raw emissions or None)."""
        st = np.zeros(8, np.uint64)
        if not collect:
            olib().or_aot(self._h, int(skip_negative), _p64(st), None, 0)
            raw = None
        else:
            cnt = olib().or_aot(self._h, int(skip_negative), _p64(st), None, 0)
            raw = np.empty((max(cnt, 1), 3), np.uint32)
            olib().or_aot(self._h, int(skip_negative), _p64(st), _p32(raw), cnt)
            raw = raw[:cnt]
        d = {k: int(st[i]) for i, k in enumerate(STAT_KEYS)}
        d["hash_sum"] = int(st[6])
        d["hash_xor"] = int(st[7])
        return d, raw


    def apply_local_order(self, spec: str) -> None:
        """Rewrites the out-lists in place (ordering.cpp:229-266)."""
        if spec == "rank-asc":
            olib().or_apply_local_order(self._h, 0, 0)
        elif spec == "degree-desc":
            olib().or_apply_local_order(self._h, 1, 0)
        elif spec.startswith("random:"):
            olib().or_apply_local_order(self._h, 2, int(spec[7:]))
        else:
            raise ValueError(f"unknown local order '{spec}'")

    def run(self, algo: str, reuse=False, skip_negative=False, collect=False):
        """Any of the reference's four kernels (engine.hpp:164-304) by name."""
        if algo == "aot":
            return self.aot(skip_negative=skip_negative, collect=collect)
        code = {"cf": 0, "cf-hash": 1, "kclist": 2}[algo]
        st = np.zeros(8, np.uint64)
        cnt = olib().or_kernel(self._h, code, int(reuse), _p64(st), None, 0)
        raw = None
        if collect:
            raw = np.empty((max(cnt, 1), 3), np.uint32)
            olib().or_kernel(self._h, code, int(reuse), _p64(st), _p32(raw), cnt)
            raw = raw[:cnt]
        d = {k: int(st[i]) for i, k in enumerate(STAT_KEYS)}
        d["hash_sum"] = int(st[6])
        d["hash_xor"] = int(st[7])
        return d, raw


def canonical_sorted(raw: np.ndarray) -> np.ndarray:
    """canonicalize_emissions (engine.cpp:51-57) + unique, on numpy arrays."""
    if raw.size == 0:
        return np.zeros((0, 3), np.uint32)
    t = np.sort(raw.astype(np.uint32), axis=1)
    t = t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]
    return t


def hash_of_triples(canon: np.ndarray):
    """(count, sum, xor) of the order-independent hash over canonical triples."""
    a = canon[:, 0].astype(np.uint64)
    b = canon[:, 1].astype(np.uint64)
    c = canon[:, 2].astype(np.uint64)

    def mix(z):
        with np.errstate(over="ignore"):
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

    # Z(v) = fmix64(v + golden); sum of Z(a) Z(b) Z(c) mod 2^64, xor of Z(a) & Z(b) & Z(c)
    with np.errstate(over="ignore"):
        za, zb, zc = (mix(v + np.uint64(0x9E3779B97F4A7C15)) for v in (a, b, c))
        h = za * zb * zc
        s = int(np.sum(h, dtype=np.uint64)) if h.size else 0
    hx = za & zb & zc
    x = int(np.bitwise_xor.reduce(hx)) if hx.size else 0
    return len(h), s, x


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref)
# --------------------------------------------------------------------------
@lru_cache(None)
def rlib() -> C.CDLL:
    if not os.path.exists(REF_SO):
        build(ref=True)
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_hardware_threads.restype = C.c_uint
    L.ref_prepare.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_char_p, C.c_char_p,
                              C.POINTER(C.c_void_p), C.POINTER(C.c_double)]
    L.ref_free.argtypes = [C.c_void_p]
    L.ref_n.restype = C.c_uint32
    L.ref_n.argtypes = [C.c_void_p]
    L.ref_m.restype = C.c_uint64
    L.ref_m.argtypes = [C.c_void_p]
    L.ref_max_out_degree.restype = C.c_uint32
    L.ref_max_out_degree.argtypes = [C.c_void_p]
    L.ref_count.argtypes = [C.c_void_p, C.c_uint, C.c_uint, C.c_int, u64p, C.POINTER(C.c_double)]
    L.ref_hash.argtypes = [C.c_void_p, C.c_uint, C.c_uint, u64p, u64p, C.POINTER(C.c_double)]
    L.ref_collect.argtypes = [C.c_void_p, C.c_uint, C.c_uint, C.c_int, u32p, C.c_uint64, u64p, u64p,
                              C.POINTER(C.c_double)]
    L.ref_cost_model.argtypes = [C.c_void_p, u64p]
    L.ref_run.argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.c_uint, C.c_int, u64p, u64p, C.POINTER(C.c_double)]
    L.ref_collect_algo.argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.c_uint, C.c_int, u32p, C.c_uint64, u64p, u64p,
                                   C.POINTER(C.c_double)]
    L.ref_brute_force.argtypes = [C.c_void_p, C.c_uint32, u32p, C.c_uint64, u64p]
    L.ref_download_oriented.argtypes = [C.c_void_p, u64p, u32p, u64p, u32p, u32p]
    L.ref_download_graph.argtypes = [C.c_void_p, u64p, u32p]
    L.ref_load_text.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p), u64p,
                                u64p]
    L.ref_write_edge_list.restype = C.c_uint64
    L.ref_write_edge_list.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
    return L


def _rcheck(rc):
    if rc != 0:
        raise RuntimeError(rlib().ref_last_error().decode())


def hardware_threads() -> int:
    return int(rlib().ref_hardware_threads())


class RefParseError(ValueError):
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class RefGraph:
    """Graph::from_edges -> make_order -> orient, by the reference library."""

    @classmethod
    def from_text(cls, text: bytes, one_indexed=False, compact=False, comments="#%"):
        """load_edge_list_text (graph.cpp:240-248) + degree order + orient.
        Returns (RefGraph, diagnostics dict); raises RefParseError."""
        if isinstance(text, str):
            text = text.encode()
        h = C.c_void_p()
        diag = np.zeros(4, np.uint64)
        line = np.zeros(1, np.uint64)
        rc = rlib().ref_load_text(text, len(text), int(one_indexed), int(compact), comments.encode(), C.byref(h),
                                  _p64(diag), _p64(line))
        if rc == 2:
            raise RefParseError(rlib().ref_last_error().decode(), int(line[0]))
        _rcheck(rc)
        self = cls.__new__(cls)
        self._h = h
        self.phase_times = {}
        self.n = rlib().ref_n(h)
        self.m = rlib().ref_m(h)
        keys = ("lines_read", "edges_parsed", "self_loops_dropped", "duplicates_dropped")
        return self, {k: int(v) for k, v in zip(keys, diag)}

    def write_edge_list(self) -> bytes:
        size = rlib().ref_write_edge_list(self._h, None, 0)
        buf = C.create_string_buffer(max(size, 1))
        rlib().ref_write_edge_list(self._h, buf, size)
        return buf.raw[:size]

    def __init__(self, min_vertices: int, pairs, order: str = "degree", local: str = "rank-asc"):
        pairs = np.ascontiguousarray(as_pairs(pairs) if not isinstance(pairs, np.ndarray) else pairs,
                                     dtype=np.uint32)
        h = C.c_void_p()
        t = (C.c_double * 3)()
        _rcheck(rlib().ref_prepare(_p32(pairs), pairs.shape[0], min_vertices, order.encode(),
                                   local.encode(), C.byref(h), t))
        self._h = h
        self.phase_times = dict(from_edges=t[0], order=t[1], orient=t[2])
        self.n = rlib().ref_n(h)
        self.m = rlib().ref_m(h)

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_free(self._h)
            self._h = None

    def max_out_degree(self) -> int:
        return rlib().ref_max_out_degree(self._h)

    @staticmethod
    def _stats(st, wall):
        d = {k: int(st[i]) for i, k in enumerate(STAT_KEYS)}
        d["wall_time_s"] = wall.value
        return d

    def count(self, threads=1, chunk=64, skip_negative=False) -> dict:
        st = np.zeros(6, np.uint64)
        wall = C.c_double()
        _rcheck(rlib().ref_count(self._h, threads, chunk, int(skip_negative), _p64(st), C.byref(wall)))
        return self._stats(st, wall)

    def hash(self, threads=1, chunk=64) -> dict:
        st = np.zeros(6, np.uint64)
        hs = np.zeros(3, np.uint64)
        wall = C.c_double()
        _rcheck(rlib().ref_hash(self._h, threads, chunk, _p64(hs), _p64(st), C.byref(wall)))
        d = self._stats(st, wall)
        d["hash_count"], d["hash_sum"], d["hash_xor"] = int(hs[0]), int(hs[1]), int(hs[2])
        return d

    def collect(self, threads=1, chunk=64, skip_negative=False):
        st = np.zeros(6, np.uint64)
        cnt = np.zeros(1, np.uint64)
        wall = C.c_double()
        _rcheck(rlib().ref_collect(self._h, threads, chunk, int(skip_negative), None, 0, _p64(cnt),
                                   _p64(st), C.byref(wall)))
        k = int(cnt[0])
        out = np.empty((max(k, 1), 3), np.uint32)
        _rcheck(rlib().ref_collect(self._h, threads, chunk, int(skip_negative), _p32(out), k, _p64(cnt),
                                   _p64(st), C.byref(wall)))
        return self._stats(st, wall), out[:k]

    def run(self, algo: str, threads=1, chunk=64, skip_negative=False, reuse=False, hash=False) -> dict:
        """run_parallel_count / run_parallel with a hash sink, any kernel."""
        st = np.zeros(6, np.uint64)
        hs = np.zeros(3, np.uint64)
        wall = C.c_double()
        flags = int(skip_negative) | (int(reuse) << 1)
        _rcheck(rlib().ref_run(self._h, algo.encode(), threads, chunk, flags, _p64(hs) if hash else None, _p64(st),
                               C.byref(wall)))
        d = self._stats(st, wall)
        if hash:
            d["hash_count"], d["hash_sum"], d["hash_xor"] = int(hs[0]), int(hs[1]), int(hs[2])
        return d

    def collect_algo(self, algo: str, threads=1, chunk=64, skip_negative=False, reuse=False):
        st = np.zeros(6, np.uint64)
        cnt = np.zeros(1, np.uint64)
        wall = C.c_double()
        flags = int(skip_negative) | (int(reuse) << 1)
        L = rlib()
        _rcheck(L.ref_collect_algo(self._h, algo.encode(), threads, chunk, flags, None, 0, _p64(cnt), _p64(st),
                                   C.byref(wall)))
        k = int(cnt[0])
        out = np.empty((max(k, 1), 3), np.uint32)
        _rcheck(L.ref_collect_algo(self._h, algo.encode(), threads, chunk, flags, _p32(out), k, _p64(cnt), _p64(st),
                                   C.byref(wall)))
        return self._stats(st, wall), out[:k]

    def cost_model(self) -> dict:
        out = np.zeros(3, np.uint64)
        _rcheck(rlib().ref_cost_model(self._h, _p64(out)))
        return dict(cf_cost=int(out[0]), kclist_cost=int(out[1]), aot_cost=int(out[2]))

    def brute_force(self, max_vertices=2000) -> np.ndarray:
        cnt = np.zeros(1, np.uint64)
        _rcheck(rlib().ref_brute_force(self._h, max_vertices, None, 0, _p64(cnt)))
        k = int(cnt[0])
        out = np.empty((max(k, 1), 3), np.uint32)
        _rcheck(rlib().ref_brute_force(self._h, max_vertices, _p32(out), k, _p64(cnt)))
        return out[:k]

    def oriented_csr(self) -> dict:
        n1 = self.n + 1
        out_off = np.empty(n1, np.uint64)
        in_off = np.empty(n1, np.uint64)
        out = np.empty(max(self.m, 1), np.uint32)
        inn = np.empty(max(self.m, 1), np.uint32)
        rank = np.empty(max(self.n, 1), np.uint32)
        _rcheck(rlib().ref_download_oriented(self._h, _p64(out_off), _p32(out), _p64(in_off), _p32(inn),
                                             _p32(rank)))
        return dict(out_offsets=out_off, out=out[: self.m], in_offsets=in_off, inn=inn[: self.m],
                    rank=rank[: self.n])

    def graph_csr(self):
        off = np.empty(self.n + 1, np.uint64)
        adj = np.empty(max(2 * self.m, 1), np.uint32)
        _rcheck(rlib().ref_download_graph(self._h, _p64(off), _p32(adj)))
        return off, adj[: 2 * self.m]
