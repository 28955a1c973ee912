"""The GPU-resident dynamic graph, mirroring the reference's store API
(graph/csr.py:17-80, graph/dynamic.py:46-334).

`DynamicGraph` owns a C-ABI store handle (include/gd_capi.h); all structural
work runs in sm_100a kernels.  The host-side accessors the reference's tests
use -- `base`, `deltas`, `segments()`, `neighbors()`, `nodes_to()` -- read a
snapshot exported from the device (cached until the next mutation), so the
reference's store tests read the same arrays they read there.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Dict, Iterator, List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .errors import ConfigurationError, ContractViolation, MalformedInputError
from .updates import ADD, DELETE, RecordArrays, UpdateBatch, UpdateRecord

SENTINEL = np.iinfo(np.int64).max


class Csr:
    """Host snapshot of one segment: offsets + coordinates (+ weights)."""

    __slots__ = ("offsets", "coordinates", "weights")

    def __init__(self, offsets: np.ndarray, coordinates: np.ndarray, weights: Optional[np.ndarray]):
        self.offsets = offsets
        self.coordinates = coordinates
        self.weights = weights

    def slot_range(self, v: int) -> Tuple[int, int]:
        return int(self.offsets[v]), int(self.offsets[v + 1])

    def live_slot_count(self) -> int:
        return int(np.count_nonzero(self.coordinates != SENTINEL))

    def total_slot_count(self) -> int:
        return len(self.coordinates)

    def check_invariants(self, node_count: int) -> None:
        assert len(self.offsets) == node_count + 1
        assert self.offsets[0] == 0
        assert self.offsets[-1] == len(self.coordinates)
        assert np.all(np.diff(self.offsets) >= 0)
        live = self.coordinates[self.coordinates != SENTINEL]
        assert live.size == 0 or (live.min() >= 0 and live.max() < node_count)
        if self.weights is not None:
            assert len(self.weights) == len(self.coordinates)


class DiffCsr(Csr):
    """A delta segment snapshot."""


class EdgeRef(NamedTuple):
    source: int
    target: int
    weight: int
    segment: int
    index: int

    @property
    def slot(self) -> Tuple[int, int]:
        return (self.segment, self.index)


@dataclass
class DeleteReport:
    applied: int = 0
    misses: int = 0
    missed: List[UpdateRecord] = field(default_factory=list)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))


class DynamicGraph:
    """CSR + diff-CSR chain on the GPU with batched structural updates."""

    def __init__(self, handle: C.c_void_p, node_count: int, *, directed: bool, weighted: bool,
                 merge_interval: int, with_reverse: bool, device: int = 0):
        self._h = handle
        self.node_count = node_count
        self.directed = directed
        self.weighted = weighted
        self.merge_interval = merge_interval
        self._with_reverse = with_reverse
        self.device = device
        self.structure_version = 0
        self.merge_epoch = 0
        self._snap_version = -1
        self._segs: List[Csr] = []
        self._rev = None
        self._revl = None
        self._revl_version = -1
        self._mutate_lock = threading.Lock()
        self.comm = None

    # -- construction -----------------------------------------------------------------

    @classmethod
    def from_arrays(cls, node_count: int, src, dst, weight=None, *, directed: bool = True, weighted: bool = False,
                    merge_interval: int = 1, with_reverse: bool = False, device: int = 0,
                    arcs: bool = False, comm=None) -> "DynamicGraph":
        """Columnar DynamicGraph.build.  arcs=True stores the triples as arcs
        as given (no reverse arcs added for undirected graphs), as the
        reference's DynamicGraph constructor does for merged().

        comm (a dist.Communicator): this rank's share of a 1D vertex
        partition (gd_graph_create_dist) -- every rank passes the whole
        edge list and, later, every batch; directed graphs only."""
        if node_count >= SENTINEL:
            raise ContractViolation("node_count collides with the deletion sentinel")
        if merge_interval < 1:
            raise ContractViolation("merge_interval must be >= 1")
        s, d = _i64(src), _i64(dst)
        w = None if weight is None else _i64(weight)
        h = C.c_void_p()
        flags = int(directed) | (2 if arcs else 0)
        if comm is None:
            N.check(N.lib().gd_graph_create(int(node_count), N.ptr(s), N.ptr(d), N.ptr(w), len(s), flags,
                                            int(weighted), int(with_reverse), int(merge_interval), int(device),
                                            C.byref(h)))
        else:
            N.check(N.lib().gd_graph_create_dist(int(node_count), N.ptr(s), N.ptr(d), N.ptr(w), len(s), flags,
                                                 int(weighted), int(with_reverse), int(merge_interval), int(device),
                                                 comm.h, C.byref(h)))
        g = cls(h, int(node_count), directed=directed, weighted=weighted, merge_interval=merge_interval,
                with_reverse=with_reverse, device=device)
        g.comm = comm  # keeps the communicator alive
        return g

    @property
    def owned_range(self) -> Tuple[int, int]:
        """[lo, hi) of the vertices this rank owns (all of them unpartitioned)."""
        lo, hi = C.c_int64(), C.c_int64()
        N.check(N.lib().gd_graph_owned_range(self._h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    @classmethod
    def build(cls, edge_list: Sequence[Tuple[int, int, int]], node_count: int, *, directed: bool = True,
              weighted: bool = False, merge_interval: int = 1, with_reverse: bool = False,
              device: int = 0) -> "DynamicGraph":
        """DynamicGraph.build (graph/dynamic.py:89-120)."""
        if len(edge_list) == 0:
            z = np.zeros(0, dtype=np.int64)
            return cls.from_arrays(node_count, z, z, z, directed=directed, weighted=weighted,
                                   merge_interval=merge_interval, with_reverse=with_reverse, device=device)
        a = np.asarray(edge_list, dtype=np.int64).reshape(-1, 3)
        return cls.from_arrays(node_count, a[:, 0], a[:, 1], a[:, 2], directed=directed, weighted=weighted,
                               merge_interval=merge_interval, with_reverse=with_reverse, device=device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.gd_graph_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- device-side queries --------------------------------------------------------------

    def _stats(self):
        live, nseg, slots = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib().gd_graph_stats(self._h, C.byref(live), C.byref(nseg), C.byref(slots)))
        return live.value, nseg.value, slots.value

    @property
    def live_edge_count(self) -> int:
        return self._stats()[0]

    def total_slot_count(self) -> int:
        return self._stats()[2]

    @property
    def has_reverse(self) -> bool:
        return self._with_reverse

    def device_bytes(self) -> int:
        b = C.c_int64()
        N.check(N.lib().gd_graph_device_bytes(self._h, C.byref(b)))
        return b.value

    # -- host snapshot (export) ----------------------------------------------------------

    def _touch(self) -> None:
        self.structure_version += 1

    def _snapshot(self) -> List[Csr]:
        if self._snap_version != self.structure_version:
            L = N.lib()
            nseg = self._stats()[1]
            segs = []
            for sg in range(nseg):
                m = C.c_int64()
                N.check(L.gd_graph_segment_slots(self._h, sg, C.byref(m)))
                off = np.zeros(self.node_count + 1, dtype=np.int64)
                co = np.zeros(m.value, dtype=np.int64)
                w = np.zeros(m.value, dtype=np.int64)
                N.check(L.gd_graph_export_segment(self._h, sg, N.ptr(off), N.ptr(co), N.ptr(w)))
                cls = Csr if sg == 0 else DiffCsr
                segs.append(cls(off, co, w if self.weighted else None))
            self._segs = segs
            self._rev = None
            self._snap_version = self.structure_version
        return self._segs

    def _reverse_snapshot(self):
        if not self._with_reverse:
            raise ConfigurationError("graph was loaded without reverse-adjacency maintenance")
        self._snapshot()
        if self._rev is None:
            L = N.lib()
            nnz = C.c_int64()
            N.check(L.gd_graph_reverse_nnz(self._h, C.byref(nnz)))
            off = np.zeros(self.node_count + 1, dtype=np.int64)
            s = np.zeros(nnz.value, dtype=np.int64)
            w = np.zeros(nnz.value, dtype=np.int64)
            N.check(L.gd_graph_export_reverse(self._h, N.ptr(off), N.ptr(s), N.ptr(w)))
            self._rev = (off, s, w)
        return self._rev

    @property
    def base(self) -> Csr:
        return self._snapshot()[0]

    @property
    def deltas(self) -> List[DiffCsr]:
        return list(self._snapshot()[1:])

    def segments(self) -> List[Csr]:
        return list(self._snapshot())

    def _check_node(self, v: int) -> None:
        if not (0 <= v < self.node_count):
            raise ContractViolation(f"node id {v} out of range [0, {self.node_count})")

    def neighbors(self, v: int) -> Iterator[EdgeRef]:
        """Live out-edges of v: base slots first, then deltas in creation order."""
        self._check_node(v)
        for seg_id, seg in enumerate(self._snapshot()):
            lo, hi = seg.slot_range(v)
            for i in range(lo, hi):
                dst = seg.coordinates[i]
                if dst != SENTINEL:
                    w = int(seg.weights[i]) if seg.weights is not None else 1
                    yield EdgeRef(v, int(dst), w, seg_id, i)

    def degree(self, v: int) -> int:
        self._check_node(v)
        total = 0
        for seg in self._snapshot():
            lo, hi = seg.slot_range(v)
            total += int(np.count_nonzero(seg.coordinates[lo:hi] != SENTINEL))
        return total

    def _reverse_lists(self):
        """The reference's reverse lists: per node, (src, segment, index,
        weight) in list order (gd_graph_export_reverse_slots)."""
        if not self._with_reverse:
            raise ConfigurationError("graph was loaded without reverse-adjacency maintenance")
        self._snapshot()
        if self._revl is None or self._revl_version != self.structure_version:
            L = N.lib()
            nnz = C.c_int64()
            N.check(L.gd_graph_reverse_nnz(self._h, C.byref(nnz)))
            off = np.zeros(self.node_count + 1, dtype=np.int64)
            cols = [np.zeros(nnz.value, dtype=np.int64) for _ in range(4)]
            N.check(L.gd_graph_export_reverse_slots(self._h, N.ptr(off), *(N.ptr(c) for c in cols)))
            self._revl = (off, *cols)
            self._revl_version = self.structure_version
        return self._revl

    def nodes_to(self, v: int) -> Iterator[EdgeRef]:
        """Live in-edges of v in the reference's reverse-list order, with
        their slot identities (graph/dynamic.py:152-160)."""
        self._check_node(v)
        off, s, sg, ix, w = self._reverse_lists()
        for k in range(int(off[v]), int(off[v + 1])):
            yield EdgeRef(int(s[k]), v, int(w[k]) if self.weighted else 1, int(sg[k]), int(ix[k]))

    def in_degree(self, v: int) -> int:
        self._check_node(v)
        off, _, _ = self._reverse_snapshot()
        return int(off[v + 1] - off[v])

    def live_slot_count(self) -> int:
        return sum(seg.live_slot_count() for seg in self._snapshot())

    def neighbor_multiset(self, v: int) -> Dict[Tuple[int, int], int]:
        out: Dict[Tuple[int, int], int] = {}
        for e in self.neighbors(v):
            key = (e.target, e.weight)
            out[key] = out.get(key, 0) + 1
        return out

    # -- structural updates ------------------------------------------------------------------

    def _arrays_of(self, batch, want: str) -> RecordArrays:
        arr = batch.arrays if hasattr(batch, "arrays") else RecordArrays.from_records(list(batch))
        bad = arr.kind != ord(want)
        if bad.any():
            kind = "delete" if want == DELETE else "add"
            raise ContractViolation(f"update_csr_{'del' if want == DELETE else 'add'} received a non-{kind} record")
        return arr.contiguous()

    def update_csr_del(self, batch, workers: int = 1) -> DeleteReport:
        """Sentinel-mark one matching slot per delete record; misses are counted."""
        arr = self._arrays_of(batch, DELETE)
        k = len(arr)
        applied, misses = C.c_int64(), C.c_int64()
        flags = np.zeros(max(k, 1), dtype=np.uint8)
        with self._mutate_lock:
            N.check(N.lib().gd_graph_apply_deletes(self._h, N.ptr(arr.src), N.ptr(arr.dst), k, C.byref(applied),
                                                   C.byref(misses), N.ptr(flags)))
            self._touch()
        rep = DeleteReport(applied.value, misses.value)
        if misses.value:
            idx = np.flatnonzero(flags[:k])
            rep.missed = [UpdateRecord(DELETE, int(arr.src[i]), int(arr.dst[i])) for i in idx]
        return rep

    def update_csr_add(self, batch, workers: int = 1) -> None:
        """Insert records: reuse vacant slots per source, spill the rest into one new delta."""
        arr = self._arrays_of(batch, ADD)
        with self._mutate_lock:
            N.check(N.lib().gd_graph_apply_adds(self._h, N.ptr(arr.src), N.ptr(arr.dst), N.ptr(arr.weight),
                                                len(arr)))
            self._touch()

    # -- merging ---------------------------------------------------------------------------

    def merged(self) -> "DynamicGraph":
        """A fresh graph with one compacted base: no sentinels, no deltas."""
        segs = self._snapshot()
        rows, cols, wts = [], [], []
        for seg in segs:
            cnt = np.diff(seg.offsets)
            r = np.repeat(np.arange(self.node_count, dtype=np.int64), cnt)
            live = seg.coordinates != SENTINEL
            rows.append(r[live])
            cols.append(seg.coordinates[live])
            wts.append(seg.weights[live] if seg.weights is not None else np.ones(int(live.sum()), dtype=np.int64))
        rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
        wts = np.concatenate(wts) if wts else np.zeros(0, np.int64)
        # neighbors() order: by node, base segment first, then deltas (stable)
        order = np.argsort(rows, kind="stable")
        return DynamicGraph.from_arrays(self.node_count, rows[order], cols[order], wts[order],
                                        directed=self.directed, weighted=self.weighted,
                                        merge_interval=self.merge_interval, with_reverse=self._with_reverse,
                                        device=self.device, arcs=True)

    def merge_deltas(self) -> None:
        """Compact in place; invalidates slot identities."""
        with self._mutate_lock:
            N.check(N.lib().gd_graph_merge(self._h))
            self.merge_epoch += 1
            self._touch()

    def check_invariants(self) -> None:
        for seg in self._snapshot():
            seg.check_invariants(self.node_count)
        assert self.live_edge_count == self.live_slot_count()

    def propagate_flags(self, flags) -> np.ndarray:
        """gview.propagate_flags (engine/interp.py:70-109) on the device."""
        if self.directed and not self._with_reverse:
            raise ConfigurationError("propagateNodeFlags on a directed graph needs reverse adjacency")
        f = np.ascontiguousarray(np.asarray(flags, dtype=np.uint8)).copy()
        rounds = C.c_int64()
        N.check(N.lib().gd_graph_propagate_flags(self._h, N.ptr(f), C.byref(rounds)))
        return f.astype(bool)
