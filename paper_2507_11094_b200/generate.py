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
        _lib = L
    return _lib


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
