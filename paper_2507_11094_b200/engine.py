"""Front door mirroring the reference engine (engine/run.py:22-68,
engine/interp.py:112-160) for the three shipped programs.

`run_program(check, graph, inputs, entry=...)` runs staticSSSP / dynamicSSSP,
staticPR / dynamicPR or staticTC / dynamicTC entirely on the GPU through the
C ABI and returns an ExecContext-shaped result (`properties[name].values()`,
`return_value`, `scalars`, `batch_stats`, `phase_totals`,
`fixedpoint_iterations`).  `check` is either the reference's own CheckResult
(when its frontend is importable) or the stand-in from `compile_source`
below; the DSL compiler itself is out of scope.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import re
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _native as N
from .errors import CompileError, ConfigurationError, ExecError
from .graph import DynamicGraph
from .updates import RecordArrays, UpdateStream

INT_INF = np.iinfo(np.int64).max

PHASES = ("static_phase", "preprocess", "structural_update", "propagate", "merge")

# entry -> (program, role)
_ENTRIES = {
    "staticSSSP": ("sssp_dynamic", "Static"),
    "decrementalSSSP": ("sssp_dynamic", "Decremental"),
    "incrementalSSSP": ("sssp_dynamic", "Incremental"),
    "dynamicSSSP": ("sssp_dynamic", "Dynamic"),
    "staticPR": ("pr_dynamic", "Static"),
    "incrementalPR": ("pr_dynamic", "Incremental"),
    "dynamicPR": ("pr_dynamic", "Dynamic"),
    "staticTC": ("tc_dynamic", "Static"),
    "dynamicTC": ("tc_dynamic", "Dynamic"),
}
_DRIVER = {"sssp_dynamic": "dynamicSSSP", "pr_dynamic": "dynamicPR", "tc_dynamic": "dynamicTC"}
_FUNCS = {p: [e for e, (q, _) in _ENTRIES.items() if q == p] for p in _DRIVER}


@dataclass
class _Fn:
    name: str
    role: str


class Program:
    """The parts of the reference's ast.Program the engine front door reads."""

    def __init__(self, name: str):
        self.name = name
        self.entry = _DRIVER[name]
        self.functions = [_Fn(f, _ENTRIES[f][1]) for f in _FUNCS[name]]

    def function(self, name: str):
        for f in self.functions:
            if f.name == name:
                return f
        return None

    def by_role(self, role: str):
        return [f for f in self.functions if f.role == role]


@dataclass
class CheckResult:
    program: Program


# SHA-256 of the normalised text (see _normalise) of the shipped programs,
# /root/reference/pkg/src/graphdyn/programs/*.sp.  tests/test_capi_cpu.py
# re-derives them from the reference when it is present.
SHIPPED_DIGESTS = {
    "sssp_dynamic": "ca559ae9aad5a6cdedf346499544a0efb065e3584d22091bf01ab4331138692b",
    "pr_dynamic": "515c5e024d4e62030e32da41bfec3c4a4366ca328a2a4a0ccee453b174218b2c",
    "tc_dynamic": "38faa7c28210c8884787026fcc6510fb1934633ec1d885d043e681d310937e8e",
}
_SHORT = {"sssp": "sssp_dynamic", "pr": "pr_dynamic", "tc": "tc_dynamic"}


def _normalise(source: str) -> str:
    """Comments dropped, then the token sequence (words and single
    punctuation characters) joined by single spaces: layout- and
    comment-insensitive, but any change to the program text shows."""
    text = re.sub(r"/\*.*?\*/", " ", source, flags=re.S)
    text = re.sub(r"//[^\n]*", " ", text)
    return " ".join(re.findall(r"\w+|[^\w\s]", text))


def source_digest(source: str) -> str:
    return hashlib.sha256(_normalise(source).encode()).hexdigest()


def compile_source(source: str, strip: bool = False) -> CheckResult:
    """frontend.compile_source (frontend/__init__.py:13-28) for the B200 path.

    The path executes exactly the three shipped programs (programs/*.sp) in
    native code, so a source is accepted only when it IS one of them up to
    comments and layout; any other text -- including an edited copy of a
    shipped program -- raises CompileError instead of silently running the
    shipped semantics.  The DSL compiler itself is out of scope."""
    digest = source_digest(source)
    for name, want in SHIPPED_DIGESTS.items():
        if digest == want:
            return CheckResult(Program(name))
    raise CompileError(["the B200 path executes only the shipped programs sssp_dynamic, pr_dynamic and "
                        "tc_dynamic (programs/*.sp); this source differs from each of them after comments "
                        "and whitespace are removed"])


def shipped_program(name: str) -> CheckResult:
    """The CheckResult of a shipped program by name ("sssp_dynamic" or its
    short form "sssp"; likewise pr / tc), without its source text."""
    key = _SHORT.get(name, name)
    if key not in SHIPPED_DIGESTS:
        raise CompileError([f"unknown shipped program {name!r}; expected one of {sorted(SHIPPED_DIGESTS)}"])
    return CheckResult(Program(key))


def needs_reverse(program) -> bool:
    """engine/run.py:14-19: reverse adjacency for programs using nodesTo/propagateNodeFlags."""
    name = _program_name(program)
    return name in ("sssp_dynamic", "pr_dynamic")


def _program_name(program) -> str:
    if isinstance(program, Program):
        return program.name
    names = set()
    fns = getattr(program, "functions", None) or getattr(program, "decls", None) or []
    for f in fns:
        names.add(getattr(f, "name", ""))
    if not names and hasattr(program, "function"):
        for e in _ENTRIES:
            if program.function(e) is not None:
                names.add(e)
    for name, driver in _DRIVER.items():
        if driver in names:
            return name
    raise CompileError(["program is not one of sssp_dynamic / pr_dynamic / tc_dynamic"])


class NodePropertyTable:
    """Result table with the reference's read API (properties.py:46-76)."""

    def __init__(self, name: str, dtype: str, data: np.ndarray):
        self.name = name
        self.dtype = dtype
        self.data = data

    def values(self) -> list:
        if self.dtype in ("float", "double"):
            return [float(x) for x in self.data]
        if self.dtype == "bool":
            return [bool(x) for x in self.data]
        return [int(x) for x in self.data]

    def get(self, v: int):
        return self.values()[v]


@dataclass
class ExecContext:
    gview: object
    worker_count: int = 1
    iteration_cap_factor: int = 10
    properties: Dict[str, object] = field(default_factory=dict)
    scalars: Dict[str, object] = field(default_factory=dict)
    return_value: object = None
    fixedpoint_iterations: List[int] = field(default_factory=list)
    batch_stats: List[dict] = field(default_factory=list)
    phase_totals: Dict[str, float] = field(default_factory=dict)
    kernel_times: Dict[str, dict] = field(default_factory=dict)

    @property
    def graph(self) -> DynamicGraph:
        return self.gview


# -------------------------------------------------------------------- handles ----

class _Algo:
    """Owns one algorithm handle of the C ABI (gd_sssp / gd_pr / gd_tc)."""

    kind = ""

    def __init__(self, h: C.c_void_p, graph: DynamicGraph):
        self.h = h
        self.graph = graph  # keeps the store alive
        self.comm = None

    def batch(self, arr: RecordArrays, batch_index: int) -> None:
        a = arr.contiguous()
        N.check(getattr(N.lib(), f"gd_{self.kind}_batch")(self.h, N.ptr(a.kind), N.ptr(a.src), N.ptr(a.dst),
                                                          N.ptr(a.weight), len(a), int(batch_index)))

    def batch_device(self, kind_ptr: int, src_ptr: int, dst_ptr: int, w_ptr: int, k: int, batch_index: int) -> None:
        """Records already in device memory (uint8 kind, int32 src/dst/w)."""
        N.check(getattr(N.lib(), f"gd_{self.kind}_batch_device")(self.h, C.c_void_p(kind_ptr), C.c_void_p(src_ptr),
                                                                 C.c_void_p(dst_ptr), C.c_void_p(w_ptr), int(k),
                                                                 int(batch_index)))

    def run_stream(self, arr: RecordArrays, batch_size: int, first_index: int = 0, *outs) -> None:
        """run_batches over a whole record stream in one call (gd_*_run_stream):
        batches of batch_size, batch j+1 uploaded and batch j-1's result read
        back on a copy stream while batch j runs.  outs: PR rank float64[n];
        SSSP dist, parent int64[n]; TC counts int64[number of batches] --
        each holds the last batch's result on return (TC: every batch's)."""
        a = arr.contiguous()
        addr = lambda x: 0 if x is None else x.ctypes.data  # noqa: E731
        self.run_stream_ptrs(addr(a.kind), addr(a.src), addr(a.dst), addr(a.weight), len(a), batch_size,
                             first_index, *[addr(o) for o in outs])

    def run_stream_ptrs(self, kind_ptr: int, src_ptr: int, dst_ptr: int, w_ptr: int, k: int, batch_size: int,
                        first_index: int, *out_ptrs: int, ids32: bool = False) -> None:
        """run_stream over host pointers (uint8 kind, int64 src/dst/w, or
        int32 with ids32 -- half the upload; pinned memory lets the copies
        overlap the batches)."""
        want = {"pr": 1, "sssp": 2, "tc": 1}[self.kind]
        outs = [C.c_void_p(p or None) for p in out_ptrs] + [C.c_void_p()] * (want - len(out_ptrs))
        N.check(getattr(N.lib(), f"gd_{self.kind}_run_stream{'32' if ids32 else ''}")(
            self.h, C.c_void_p(kind_ptr), C.c_void_p(src_ptr), C.c_void_p(dst_ptr), C.c_void_p(w_ptr or None),
            int(k), int(batch_size), int(first_index), *outs[:want]))

    def phase_ms(self) -> Dict[str, float]:
        ms = (C.c_double * 5)()
        N.check(N.lib().gd_phase_times(self.h, ms))
        return {p: ms[i] for i, p in enumerate(PHASES)}

    def iterations(self) -> int:
        it = C.c_int64()
        N.check(N.lib().gd_iterations(self.h, C.byref(it)))
        return it.value

    def wait(self) -> None:
        """Block until read_async copies have landed (gd_wait)."""
        N.check(N.lib().gd_wait(self.h))

    def set_profiling(self, on: bool) -> None:
        N.check(N.lib().gd_set_profiling(self.h, int(on)))

    def kernel_time(self, name: str, total: bool = False):
        """(ms, launches, algorithmic bytes) of `name` in the last batch, or
        summed since profiling was switched on (total=True)."""
        ms, n, b = C.c_double(), C.c_int64(), C.c_int64()
        fn = N.lib().gd_kernel_time_total if total else N.lib().gd_kernel_time
        N.check(fn(self.h, name.encode(), C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._lib is not None:
            getattr(N._lib, f"gd_{self.kind}_destroy")(h)
            self.h = None


class SSSPHandle(_Algo):
    kind = "sssp"

    def __init__(self, graph: DynamicGraph, src: int, iteration_cap_factor: int = 10):
        h = C.c_void_p()
        N.check(N.lib().gd_sssp_create_ex(graph.handle, int(src), int(iteration_cap_factor), C.byref(h)))
        super().__init__(h, graph)

    def read(self):
        n = self.graph.node_count
        dist = np.zeros(n, dtype=np.int64)
        parent = np.zeros(n, dtype=np.int64)
        N.check(N.lib().gd_sssp_read(self.h, N.ptr(dist), N.ptr(parent)))
        return dist, parent

    def read_async(self, dist_out: np.ndarray, parent_out: Optional[np.ndarray] = None) -> None:
        """Asynchronous read (gd_sssp_read_async); valid after wait()."""
        n = self.graph.node_count
        for a in (dist_out, parent_out):
            if a is not None and (a.dtype != np.int64 or a.size < n):
                raise ValueError("outputs must be int64[node_count]")
        N.check(N.lib().gd_sssp_read_async(self.h, N.ptr(dist_out), N.ptr(parent_out)))


class PRHandle(_Algo):
    kind = "pr"

    def __init__(self, graph: DynamicGraph, damping: float, beta: float, maxiter: int):
        h = C.c_void_p()
        N.check(N.lib().gd_pr_create(graph.handle, float(damping), float(beta), int(maxiter), C.byref(h)))
        super().__init__(h, graph)

    def read(self, with_outdeg: bool = True):
        n = self.graph.node_count
        rank = np.zeros(n, dtype=np.float64)
        od = np.zeros(n, dtype=np.int64) if with_outdeg else None
        N.check(N.lib().gd_pr_read(self.h, N.ptr(rank), N.ptr(od)))
        return rank, od

    def read_affected(self) -> np.ndarray:
        """The last batch's flooded `affected` flags (uint8[n])."""
        out = np.zeros(self.graph.node_count, dtype=np.uint8)
        N.check(N.lib().gd_pr_read_affected(self.h, N.ptr(out)))
        return out

    def read_async(self, rank_out: np.ndarray) -> None:
        """Snapshot the ranks now, copy them to rank_out (float64[n], pinned
        for overlap) behind the next batch; valid after wait()."""
        if rank_out.dtype != np.float64 or rank_out.size < self.graph.node_count:
            raise ValueError("rank_out must be float64[node_count]")
        N.check(N.lib().gd_pr_read_async(self.h, N.ptr(rank_out)))

    def rank_device_ptr(self) -> int:
        p = C.c_void_p()
        N.check(N.lib().gd_pr_rank_device(self.h, C.byref(p)))
        return p.value


class TCHandle(_Algo):
    kind = "tc"

    def __init__(self, graph: DynamicGraph):
        h = C.c_void_p()
        N.check(N.lib().gd_tc_create(graph.handle, C.byref(h)))
        super().__init__(h, graph)

    def read(self) -> int:
        c = C.c_int64()
        N.check(N.lib().gd_tc_read(self.h, C.byref(c)))
        return c.value


# ----------------------------------------------------------------- front door ----

def _need(inputs, key, conv):
    if key not in inputs:
        raise ExecError(f"unbound input {key!r}")
    v = inputs[key]
    if conv is int and v == math.inf:
        return INT_INF
    return conv(v)


def _stream_of(inputs) -> UpdateStream:
    for key in ("updateList", "updates", "update_list"):
        if key in inputs:
            s = inputs[key]
            if s is None:
                raise ExecError(f"unbound input {key!r} (update stream)")
            if isinstance(s, UpdateStream):
                return s
            if hasattr(s, "records"):  # the reference's own UpdateStream
                return UpdateStream(list(s.records))
            return UpdateStream(list(s))
    raise ExecError("unbound input 'updateList' (update stream)")


def _batch_size(inputs, stream_len: int) -> int:
    for key in ("batchsize", "batch_size"):
        if key in inputs:
            return int(inputs[key])
    raise ExecError("unbound input 'batchsize'")


def run_program(check, graph: DynamicGraph, inputs: Dict[str, object], *, entry: Optional[str] = None,
                worker_count: int = 1, iteration_cap_factor: int = 10, debug: bool = False,
                gview=None, comm=None) -> ExecContext:
    """engine/run.py:22-41 on the B200 path.  worker_count/debug/gview are
    accepted for signature compatibility; the GPU path has no worker pool.

    A graph built with a communicator (DynamicGraph.from_arrays(comm=...))
    runs partitioned on every rank.  comm= splits a TC (or PR) handle over a
    replicated store instead (gd_tc_set_comm / gd_pr_set_comm)."""
    program = check.program
    name = _program_name(program)
    entry = entry or getattr(program, "entry", None) or _DRIVER[name]
    if entry not in _ENTRIES or _ENTRIES[entry][0] != name:
        raise ExecError(f"no function named {entry!r}")
    role = _ENTRIES[entry][1]
    if role in ("Incremental", "Decremental"):
        raise ExecError(f"{entry} runs only inside its Dynamic driver on the B200 path")
    if not isinstance(graph, DynamicGraph):
        raise ConfigurationError("run_program on the B200 path needs a paper_2507_11094_b200 DynamicGraph")
    ctx = ExecContext(graph, worker_count=worker_count, iteration_cap_factor=iteration_cap_factor)
    dynamic = role == "Dynamic"
    stream = _stream_of(inputs) if dynamic else None
    bsize = _batch_size(inputs, len(stream)) if dynamic else 0
    if dynamic and bsize <= 0:
        raise ExecError("batch size must be positive")

    t0 = time.perf_counter()
    if name == "sssp_dynamic":
        algo = SSSPHandle(graph, _need(inputs, "src", int), iteration_cap_factor)
    elif name == "pr_dynamic":
        algo = PRHandle(graph, _need(inputs, "damping", float), _need(inputs, "beta", float),
                        _need(inputs, "maxiter", int))
    else:
        algo = TCHandle(graph)
    if comm is not None:
        comm.attach(algo)
    if dynamic:
        arr = stream.arrays
        prev_it = algo.iterations()
        for index, start in enumerate(range(0, len(arr), bsize)):
            part = arr.slice(start, start + bsize)
            stats = {"index": index, "adds": int(np.count_nonzero(part.kind == ord("a"))),
                     "deletes": int(np.count_nonzero(part.kind == ord("d")))}
            before = algo.phase_ms()
            algo.batch(part, index)
            graph._touch()
            after = algo.phase_ms()
            for p in PHASES[1:]:
                stats[p] = (after[p] - before[p]) / 1e3
            ctx.batch_stats.append(stats)
            it = algo.iterations()
            ctx.fixedpoint_iterations.append(it - prev_it)
            prev_it = it
    totals = algo.phase_ms()
    ctx.phase_totals = {p: totals[p] / 1e3 for p in PHASES if totals[p] > 0 or p == "static_phase"}
    ctx.scalars["wall_seconds"] = time.perf_counter() - t0

    # node properties in the reference's declaration order (the entry's
    # parameters, then its locals: interp.py binds every propNode of the
    # entry's scope into ctx.properties)
    n = graph.node_count
    false = lambda: np.zeros(n, dtype=np.uint8)  # noqa: E731
    if name == "sssp_dynamic":
        dist, parent = algo.read()
        ctx.properties["dist"] = NodePropertyTable("dist", "int", dist)
        ctx.properties["parent"] = NodePropertyTable("parent", "int", parent)
        # the bool locals are the `modified` sets of fixedPoint loops, which
        # end only once no flag is set (interp.py:800-813; sssp_dynamic.sp:15,
        # 52,72,110: activeOnDelete / activeOnAdd are passed in as `modified`
        # and are re-attached False per batch, :138) -- so a completed run
        # always leaves them all False
        locals_ = ("activeOnDelete", "activeOnAdd") if dynamic else ("modified", "modified_nxt")
        for nm in locals_:
            ctx.properties[nm] = NodePropertyTable(nm, "bool", false())
    elif name == "pr_dynamic":
        rank, od = algo.read()
        ctx.properties["pagerank"] = NodePropertyTable("pagerank", "float", rank)
        if dynamic:  # pr_dynamic.sp:82-83: affected, then outdeg
            ctx.properties["affected"] = NodePropertyTable("affected", "bool", algo.read_affected())
            ctx.properties["outdeg"] = NodePropertyTable("outdeg", "int", od)
        else:  # staticPR (pr_dynamic.sp:7-9): rank_new holds the last sweep, i.e. the committed ranks
            ctx.properties["outdeg"] = NodePropertyTable("outdeg", "int", od)
            maxiter = _need(inputs, "maxiter", int)
            ctx.properties["rank_new"] = NodePropertyTable(
                "rank_new", "float", rank.copy() if maxiter > 0 else np.zeros(n, dtype=np.float64))
    else:
        c = algo.read()
        ctx.return_value = c
        ctx.scalars["tcount"] = c
    ctx.scalars.pop("wall_seconds", None)
    # bound scalar inputs are program scalars too (interp.py binds them into
    # ctx.scalars): batchsize, src, damping, beta, maxiter
    for key in ("batchsize", "batch_size", "src", "damping", "beta", "maxiter"):
        if key in inputs and isinstance(inputs[key], (bool, int, float, np.integer, np.floating)):
            ctx.scalars.setdefault(key, inputs[key].item() if isinstance(inputs[key], np.generic) else inputs[key])
    return ctx


def run_batches(check, graph: DynamicGraph, updates: UpdateStream, batch_size: int, inputs: Dict[str, object],
                **kwargs) -> ExecContext:
    """engine/run.py:44-68: bind the stream and batch size to the driver."""
    bound = dict(inputs)
    bound["updateList"] = updates
    bound["batchsize"] = batch_size
    return run_program(check, graph, bound, **kwargs)
