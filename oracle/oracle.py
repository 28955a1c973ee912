"""ctypes wrapper over the parity checker (oracle/gd_oracle.c) and over the
reference's own compiled OpenMP drivers (oracle/_ref/libgdref.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never by the product package.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libgdref.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def build(force: bool = False) -> None:
    """Compile liboracle.so (and the reference harness when /root/reference exists)."""
    target = "all" if os.path.isdir("/root/reference/pkg") else "oracle"
    subprocess.run(["make", "-s", "-C", HERE, target] + (["-B"] if force else []), check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.or_last_error.restype = C.c_char_p
        L.or_graph_build.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                     C.c_int, C.c_int64, C.POINTER(vp)]
        L.or_graph_free.argtypes = [vp]
        L.or_graph_delete.argtypes = [vp, _i64p, _i64p, C.c_int64, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.c_void_p]
        L.or_graph_add.argtypes = [vp, _i64p, _i64p, C.c_void_p, C.c_int64]
        L.or_graph_merge.argtypes = [vp]
        L.or_graph_live.argtypes = [vp]
        L.or_graph_live.restype = C.c_int64
        L.or_graph_nseg.argtypes = [vp]
        L.or_graph_seg_slots.argtypes = [vp, C.c_int]
        L.or_graph_seg_slots.restype = C.c_int64
        L.or_graph_export_seg.argtypes = [vp, C.c_int, _i64p, _i64p, _i64p]
        L.or_graph_rev_total.argtypes = [vp]
        L.or_graph_rev_total.restype = C.c_int64
        L.or_graph_export_rev.argtypes = [vp, _i64p, _i64p, _i64p]
        L.or_propagate_flags.argtypes = [vp, _u8p]
        L.or_propagate_flags.restype = C.c_int64
        for algo in ("sssp", "pr", "tc"):
            getattr(L, f"or_{algo}_batch").argtypes = [vp, _u8p, _i64p, _i64p, _i64p, C.c_int64, C.c_int64]
            getattr(L, f"or_{algo}_free").argtypes = [vp]
        L.or_sssp_create.argtypes = [vp, C.c_int64, C.POINTER(vp)]
        L.or_sssp_read.argtypes = [vp, _i64p, _i64p]
        L.or_sssp_iters.argtypes = [vp]
        L.or_sssp_iters.restype = C.c_int64
        L.or_pr_create.argtypes = [vp, C.c_double, C.c_double, C.c_int64, C.POINTER(vp)]
        L.or_pr_read.argtypes = [vp, _f64p, _i64p]
        L.or_pr_sweeps.argtypes = [vp]
        L.or_pr_sweeps.restype = C.c_int64
        L.or_tc_create.argtypes = [vp, C.POINTER(vp)]
        L.or_tc_read.argtypes = [vp]
        L.or_tc_read.restype = C.c_int64
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"oracle error {code}: {msg}")


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, lib().or_last_error().decode())


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))


def split_edges(edges: Sequence[Tuple[int, int, int]]):
    arr = np.asarray(list(edges), dtype=np.int64).reshape(-1, 3)
    return _i64(arr[:, 0]), _i64(arr[:, 1]), _i64(arr[:, 2])


def split_records(records):
    """UpdateRecord-like objects (kind, src, dst, weight) -> arrays."""
    recs = list(records)
    kind = np.array([ord(r.kind) for r in recs], dtype=np.uint8)
    s = _i64([r.src for r in recs])
    d = _i64([r.dst for r in recs])
    w = _i64([r.weight for r in recs])
    return kind, s, d, w


class OracleGraph:
    """The reference diff-CSR store restated in C (dynamic.py / graphdyn_rt.h)."""

    def __init__(self, n, src, dst, w=None, *, directed=True, weighted=False, with_reverse=False,
                 merge_interval=1):
        L = lib()
        src, dst = _i64(src), _i64(dst)
        self._w = None if w is None else _i64(w)
        h = C.c_void_p()
        _check(L.or_graph_build(int(n), src, dst,
                                None if self._w is None else self._w.ctypes.data_as(C.c_void_p),
                                len(src), int(directed), int(weighted), int(with_reverse),
                                int(merge_interval), C.byref(h)))
        self.h = h
        self.n = int(n)
        self.directed = directed
        self.weighted = weighted

    @classmethod
    def from_edges(cls, edges, n, **kw):
        if len(edges) == 0:
            z = np.zeros(0, dtype=np.int64)
            return cls(n, z, z, z, **kw)
        s, d, w = split_edges(edges)
        return cls(n, s, d, w, **kw)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_graph_free(self.h)
            self.h = None

    def delete(self, src, dst, with_flags=False):
        src, dst = _i64(src), _i64(dst)
        a, m = C.c_int64(), C.c_int64()
        flags = np.zeros(len(src), dtype=np.uint8)
        _check(lib().or_graph_delete(self.h, src, dst, len(src), C.byref(a), C.byref(m),
                                     flags.ctypes.data_as(C.c_void_p)))
        if with_flags:
            return a.value, m.value, flags
        return a.value, m.value

    def add(self, src, dst, w=None):
        src, dst = _i64(src), _i64(dst)
        ww = None if w is None else _i64(w)
        _check(lib().or_graph_add(self.h, src, dst, None if ww is None else ww.ctypes.data_as(C.c_void_p),
                                  len(src)))

    def merge(self):
        _check(lib().or_graph_merge(self.h))

    @property
    def live(self) -> int:
        return lib().or_graph_live(self.h)

    def segments(self):
        """[(offsets, coords, weights)] exactly as the reference lays them out."""
        L = lib()
        out = []
        for sg in range(L.or_graph_nseg(self.h)):
            m = L.or_graph_seg_slots(self.h, sg)
            off = np.zeros(self.n + 1, dtype=np.int64)
            co = np.zeros(m, dtype=np.int64)
            w = np.zeros(m, dtype=np.int64)
            L.or_graph_export_seg(self.h, sg, off, co, w)
            out.append((off, co, w))
        return out

    def reverse(self):
        """(offsets, src, weight) of the maintained reverse lists, in list order."""
        L = lib()
        t = L.or_graph_rev_total(self.h)
        if t < 0:
            return None
        off = np.zeros(self.n + 1, dtype=np.int64)
        s = np.zeros(t, dtype=np.int64)
        w = np.zeros(t, dtype=np.int64)
        L.or_graph_export_rev(self.h, off, s, w)
        return off, s, w

    def propagate_flags(self, flags) -> Tuple[np.ndarray, int]:
        f = np.ascontiguousarray(np.asarray(flags, dtype=np.uint8))
        rounds = lib().or_propagate_flags(self.h, f)
        return f.astype(bool), rounds


class _Algo:
    name = ""

    def batch(self, kind, s, d, w, batch_index):
        kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
        _check(getattr(lib(), f"or_{self.name}_batch")(self.h, kind, _i64(s), _i64(d), _i64(w), len(kind),
                                                     int(batch_index)))

    def run_stream(self, kind, s, d, w, batch_size):
        kind = np.asarray(kind, dtype=np.uint8)
        k = len(kind)
        for bi, st in enumerate(range(0, k, batch_size)):
            sl = slice(st, st + batch_size)
            self.batch(kind[sl], s[sl], d[sl], w[sl], bi)
        return self

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            getattr(_lib, f"or_{self.name}_free")(self.h)
            self.h = None


class OracleSSSP(_Algo):
    name = "sssp"

    def __init__(self, g: OracleGraph, src: int):
        self.g = g
        h = C.c_void_p()
        _check(lib().or_sssp_create(g.h, int(src), C.byref(h)))
        self.h = h

    def read(self):
        dist = np.zeros(self.g.n, dtype=np.int64)
        par = np.zeros(self.g.n, dtype=np.int64)
        lib().or_sssp_read(self.h, dist, par)
        return dist, par


class OraclePR(_Algo):
    name = "pr"

    def __init__(self, g: OracleGraph, damping=0.85, beta=0.001, maxiter=100):
        self.g = g
        h = C.c_void_p()
        _check(lib().or_pr_create(g.h, float(damping), float(beta), int(maxiter), C.byref(h)))
        self.h = h

    def read(self):
        r = np.zeros(self.g.n, dtype=np.float64)
        od = np.zeros(self.g.n, dtype=np.int64)
        lib().or_pr_read(self.h, r, od)
        return r, od

    @property
    def sweeps(self):
        return lib().or_pr_sweeps(self.h)


class OracleTC(_Algo):
    name = "tc"

    def __init__(self, g: OracleGraph):
        self.g = g
        h = C.c_void_p()
        _check(lib().or_tc_create(g.h, C.byref(h)))
        self.h = h

    def read(self) -> int:
        return lib().or_tc_read(self.h)


# -- the reference's own emitted drivers (oracle/_ref/libgdref.so) ---------------

def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_LIB_PATH} not built (make -C oracle ref needs /root/reference)")
        L = C.CDLL(REF_LIB_PATH)
        vp = C.c_void_p
        L.gdref_run.argtypes = [C.c_int, C.c_int64, _i64p, _i64p, vp, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                _u8p, _i64p, _i64p, _i64p, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                C.c_double, C.c_double, C.c_int64, C.c_int, _f64p, vp, vp, vp]
        _ref = L
    return _ref


def ref_run(algo: str, n, src, dst, w, *, directed=True, weighted=False, merge_interval=1,
            kind=None, us=None, ud=None, uw=None, batch_size=0, threads=1, sssp_src=0,
            damping=0.85, beta=0.001, maxiter=100, skip_t0=False):
    """Run the reference's dynamicSSSP/PR/TC over arrays. Returns (result, times)."""
    a = {"sssp": 0, "pr": 1, "tc": 2}[algo]
    if a == 2:
        threads = 1  # emitted TC crashes with >1 OpenMP thread
    src, dst = _i64(src), _i64(dst)
    ww = None if w is None else _i64(w)
    if kind is None:
        kind = np.zeros(0, dtype=np.uint8)
        us = ud = uw = np.zeros(0, dtype=np.int64)
    kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
    us, ud, uw = _i64(us), _i64(ud), _i64(uw)
    times = np.zeros(2, dtype=np.float64)
    n = int(n)
    o_a = np.zeros(max(n, 1), dtype=np.int64)
    o_b = np.zeros(max(n, 1), dtype=np.int64)
    o_f = np.zeros(max(n, 1), dtype=np.float64)
    ref_lib().gdref_run(a, n, src, dst, None if ww is None else ww.ctypes.data_as(C.c_void_p), len(src),
                        int(directed), int(weighted), int(merge_interval), kind, us, ud, uw, len(kind),
                        int(batch_size), int(threads), int(sssp_src), float(damping), float(beta),
                        int(maxiter), int(skip_t0), times, o_a.ctypes.data_as(C.c_void_p),
                        o_b.ctypes.data_as(C.c_void_p), o_f.ctypes.data_as(C.c_void_p))
    if a == 0:
        res = (o_a[:n], o_b[:n])
    elif a == 1:
        res = o_f[:n]
        ref_run.last_outdeg = o_a[:n]  # live out-degree of the final graph
    else:
        res = int(o_a[0])
    return res, times
