"""Synthetic inputs at BASELINE scale (native, libgdgen.so): R-MAT, uniform
random, 2-D grid graphs and generate_updates-style streams.  Mirrors the
recipes of the reference's generate.py:15-161 with a counter-based RNG (the
reference's Python generators take ~9 s per 1M edges)."""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgdgen.so")
_lib = None


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i64 = C.c_void_p, C.c_int64
        L.gdgen_rmat.restype = i64
        L.gdgen_rmat.argtypes = [C.c_int, i64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                 i64, vp, vp, vp]
        L.gdgen_uniform.restype = i64
        L.gdgen_uniform.argtypes = [i64, i64, C.c_uint64, C.c_int, C.c_int, i64, vp, vp, vp]
        L.gdgen_grid.restype = i64
        L.gdgen_grid.argtypes = [i64, i64, C.c_uint64, i64, vp, vp, vp]
        L.gdgen_updates.restype = i64
        L.gdgen_updates.argtypes = [vp, vp, i64, i64, i64, i64, i64, C.c_uint64, C.c_int, i64, vp, vp, vp, vp]
        L.gdgen_threads.restype = C.c_int
        L.gdgen_py_rmat.restype = i64
        L.gdgen_py_rmat.argtypes = [C.c_int, i64, C.c_uint64, C.c_int, i64, C.c_double, C.c_double, C.c_double,
                                    C.c_int, vp, vp, vp]
        L.gdgen_py_uniform.restype = i64
        L.gdgen_py_uniform.argtypes = [i64, i64, C.c_uint64, C.c_int, i64, C.c_int, C.c_int, vp, vp, vp]
        L.gdgen_py_updates.restype = i64
        L.gdgen_py_updates.argtypes = [vp, vp, vp, i64, i64, C.c_double, C.c_uint64, C.c_double, C.c_int, vp, vp, vp,
                                       vp]
        L.gdgen_parse_file.restype = vp
        L.gdgen_parse_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(i64), C.POINTER(C.c_int), C.POINTER(i64),
                                       C.POINTER(i64), C.c_char_p, C.c_int]
        L.gdgen_parsed_copy.restype = None
        L.gdgen_parsed_copy.argtypes = [vp, vp, vp, vp, vp]
        L.gdgen_parsed_free.restype = None
        L.gdgen_parsed_free.argtypes = [vp]
        _lib = L
    return _lib


def parse_text_file(path: str, updates: bool):
    """Native parallel parse of an edge (updates=False) or update file:
    returns (kind or None, src, dst, w, weighted, max_id); raises
    MalformedInputError with the first bad line, as the Python loops do."""
    from .errors import MalformedInputError

    L = _L()
    cnt, wtd, mx, eline = C.c_int64(), C.c_int(), C.c_int64(), C.c_int64()
    msg = C.create_string_buffer(512)
    h = L.gdgen_parse_file(os.fsencode(path), int(updates), C.byref(cnt), C.byref(wtd), C.byref(mx),
                           C.byref(eline), msg, 512)
    try:
        if eline.value >= 0:
            text = msg.value.decode(errors="replace")
            if eline.value == 0:
                raise OSError(f"{path}: {text}")
            raise MalformedInputError(text, path=path, line=int(eline.value))
        k = cnt.value
        kind = np.empty(k, dtype=np.uint8) if updates else None
        src = np.empty(k, dtype=np.int64)
        dst = np.empty(k, dtype=np.int64)
        w = np.empty(k, dtype=np.int64)
        L.gdgen_parsed_copy(h, None if kind is None else _p(kind), _p(src), _p(dst), _p(w))
        return kind, src, dst, w, bool(wtd.value), int(mx.value)
    finally:
        L.gdgen_parsed_free(h)


def _p(a):
    return C.c_void_p(a.ctypes.data)


def threads() -> int:
    return _L().gdgen_threads()


def rmat(scale: int, m: int, *, seed: int, weighted: bool = False, max_weight: int = 100, undirected: bool = False,
         a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """R-MAT with distinct pairs and no self-loops: (src, dst, w, node_count)."""
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    w = np.empty(m, dtype=np.int64)
    got = _L().gdgen_rmat(scale, m, seed, a, b, c, int(undirected), int(weighted), max_weight, _p(src), _p(dst), _p(w))
    return src[:got], dst[:got], w[:got], 1 << scale


def uniform(n: int, m: int, *, seed: int, weighted: bool = False, max_weight: int = 100, undirected: bool = False):
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    w = np.empty(m, dtype=np.int64)
    got = _L().gdgen_uniform(n, m, seed, int(undirected), int(weighted), max_weight, _p(src), _p(dst), _p(w))
    return src[:got], dst[:got], w[:got], n


def grid(rows: int, cols: int, *, seed: int, max_weight: int = 100):
    """4-neighbour grid with both arcs per neighbour pair (directed store)."""
    m = 2 * rows * (cols - 1) + 2 * (rows - 1) * cols
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    w = np.empty(m, dtype=np.int64)
    got = _L().gdgen_grid(rows, cols, seed, max_weight, _p(src), _p(dst), _p(w))
    return src[:got], dst[:got], w[:got], rows * cols


def updates(src, dst, n: int, *, percent: float, batches: int = 1, seed: int, add_fraction: float = 0.5,
            undirected: bool = False, max_weight: int = 1):
    """`batches` successive batches of `percent`% of the edge count each
    (ceil, as generate_updates), deletes from edges, adds from non-edges,
    every pair distinct across the whole stream; each batch shuffled.
    Returns (kind uint8, src, dst, w, batch_size)."""
    m = len(src)
    per = math.ceil(percent / 100.0 * m)
    n_add = int(round(per * add_fraction)) * batches
    n_del = min(per * batches - n_add, m)
    total = n_del + n_add
    kind = np.empty(total, dtype=np.uint8)
    us = np.empty(total, dtype=np.int64)
    ud = np.empty(total, dtype=np.int64)
    uw = np.empty(total, dtype=np.int64)
    s = np.ascontiguousarray(src, dtype=np.int64)
    d = np.ascontiguousarray(dst, dtype=np.int64)
    na = _L().gdgen_updates(_p(s), _p(d), m, n, n_del, n_add, per, seed, int(undirected), max_weight, _p(kind),
                            _p(us), _p(ud), _p(uw))
    k = n_del + na
    return kind[:k], us[:k], ud[:k], uw[:k], per


# ---------------------------------------------------------------------------
# Seed-compatible generators: the reference's own recipes (generate.py:15-161)
# drawn from a native restatement of Python's random.Random, so the same seed
# gives the same edges / stream as the reference (checked against it in
# tests/test_pyrand_cpu.py).  Sequential; ~50-100x faster than the Python.


def _seed(seed: int) -> int:
    seed = abs(int(seed))
    if seed >= 1 << 64:
        raise ValueError("seed-compatible generators take seeds below 2**64")
    return seed


def py_rmat_graph(node_count_log2: int, edge_count: int, *, seed: int, weighted: bool = False, max_weight: int = 10,
                  a: float = 0.57, b: float = 0.19, c: float = 0.19, undirected: bool = False):
    """generate.rmat_graph: (src, dst, w, node_count) as int64 arrays."""
    m = max(int(edge_count), 0)
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    w = np.empty(m, dtype=np.int64)
    got = _L().gdgen_py_rmat(node_count_log2, m, _seed(seed), int(weighted), max_weight, a, b, c, int(undirected),
                             _p(src), _p(dst), _p(w))
    return src[:got], dst[:got], w[:got], 1 << node_count_log2


def py_uniform_random_graph(node_count: int, edge_count: int, *, seed: int, weighted: bool = False,
                            max_weight: int = 10, connected: bool = False, undirected: bool = False):
    """generate.uniform_random_graph: (src, dst, w) as int64 arrays."""
    cap = max(int(edge_count), 0) + (node_count if connected else 0)
    src = np.empty(cap, dtype=np.int64)
    dst = np.empty(cap, dtype=np.int64)
    w = np.empty(cap, dtype=np.int64)
    got = _L().gdgen_py_uniform(node_count, max(int(edge_count), 0), _seed(seed), int(weighted), max_weight,
                                int(connected), int(undirected), _p(src), _p(dst), _p(w))
    return src[:got], dst[:got], w[:got]


def py_generate_updates(src, dst, w, node_count: int, percent: float, *, seed: int, add_fraction: float = 0.5,
                        undirected: bool = False):
    """generate.generate_updates: (kind uint8 'a'/'d', src, dst, w) in the
    reference's stream order."""
    from .errors import ContractViolation

    if not (0.0 < percent <= 100.0):
        raise ContractViolation(f"percent must lie in (0, 100], got {percent}")
    if not (0.0 <= add_fraction <= 1.0):
        raise ContractViolation(f"add_fraction must lie in [0, 1], got {add_fraction}")
    s = np.ascontiguousarray(src, dtype=np.int64)
    d = np.ascontiguousarray(dst, dtype=np.int64)
    ww = np.ascontiguousarray(w if w is not None else np.ones(len(s)), dtype=np.int64)
    cap = math.ceil(percent / 100.0 * len(s)) + 1
    kind = np.empty(cap, dtype=np.uint8)
    us = np.empty(cap, dtype=np.int64)
    ud = np.empty(cap, dtype=np.int64)
    uw = np.empty(cap, dtype=np.int64)
    k = _L().gdgen_py_updates(_p(s), _p(d), _p(ww), len(s), node_count, float(percent), _seed(seed),
                              float(add_fraction), int(undirected), _p(kind), _p(us), _p(ud), _p(uw))
    return kind[:k], us[:k], ud[:k], uw[:k]
