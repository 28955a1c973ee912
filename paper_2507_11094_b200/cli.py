"""graphdyn-compatible command line on the B200 path.

Mirrors the reference's cli.py (graphdyn/cli.py:33-635) for the three shipped
programs: `run`, `gen-updates`, `bench` and `oracle`, with the same flags,
CSV / manifest outputs and exit codes (0 ok, 1 usage, 2 compile, 3 runtime,
4 equivalence failure).  Every computation runs on the GPU store; `oracle`
is the static recompute (staticSSSP / staticPR / staticTC) of the replayed
final graph.  `sim --ranks R` runs the program on a real vertex-partitioned
store over R in-process ranks and reports per-rank communication (DESIGN.md
§5).  `emit` (OpenMP code generation) belongs to the reference's compiler
and is out of scope: it exits with a usage error.

Graph and update files may be the reference's text formats or the binary
formats of io.py (detected by magic).

    python -m paper_2507_11094_b200.cli run programs/sssp_dynamic.sp g.txt --updates u.txt --src 0
"""

from __future__ import annotations

import argparse
import csv
import math
import os
import sys
import time
from pathlib import Path
from typing import Dict, List, Optional

import numpy as np

from .engine import INT_INF, NodePropertyTable, compile_source, needs_reverse, run_program, shipped_program
from .errors import CompileError, GraphDynError
from .manifest import build_manifest, write_manifest

EXIT_OK = 0
EXIT_USAGE = 1
EXIT_COMPILE = 2
EXIT_RUNTIME = 3
EXIT_EQUIVALENCE = 4

_PROGRAM_NAMES = {"sssp": "sssp_dynamic", "pr": "pr_dynamic", "tc": "tc_dynamic"}


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage problems exit 1, not argparse's 2 (cli.py:40-44)
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


class UsageError(Exception):
    pass


def _add_common_run_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--updates", help="update stream file (text or GDUPDT01)")
    p.add_argument("--batch", type=int, default=0, help="batch size (0 = whole stream)")
    p.add_argument("--threads", type=int, default=1, help="accepted for compatibility; the GPU has no worker pool")
    p.add_argument("--src", type=int, default=None, help="source node for SSSP")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--merge-interval", type=int, default=1)
    p.add_argument("--undirected", action="store_true")
    p.add_argument("--nodes", type=int, default=None, help="override node count")
    p.add_argument("--damping", type=float, default=0.85)
    p.add_argument("--beta", type=float, default=0.001)
    p.add_argument("--maxiter", type=int, default=100)
    p.add_argument("--iteration-cap-factor", type=int, default=10)
    p.add_argument("--param", action="append", default=[], metavar="NAME=VALUE")
    p.add_argument("--strip", action="store_true", help="accepted for compatibility (no interpreter to strip)")
    p.add_argument("--device", type=int, default=0, help="CUDA device")
    p.add_argument("--out", default="graphdyn_out")


def make_parser() -> _Parser:
    from . import __version__

    parser = _Parser(prog="graphdyn", description="dynamic-graph runtime, B200 backend")
    parser.add_argument("--version", action="version", version=f"graphdyn {__version__} (b200)")
    sub = parser.add_subparsers(dest="command", required=True)

    run = sub.add_parser("run", help="execute a program")
    run.add_argument("program", help="a .sp file of the three shipped programs, or sssp / pr / tc")
    run.add_argument("graph")
    run.add_argument("--mode", choices=("dynamic", "static"), default="dynamic")
    run.add_argument("--entry", help="entry function (defaults per mode)")
    _add_common_run_flags(run)

    gen = sub.add_parser("gen-updates", help="generate a random update stream (seed-compatible)")
    gen.add_argument("graph")
    gen.add_argument("--percent", type=float, required=True)
    gen.add_argument("--add-fraction", type=float, default=0.5)
    gen.add_argument("--seed", type=int, default=0)
    gen.add_argument("--undirected", action="store_true")
    gen.add_argument("--binary", action="store_true", help="write a GDUPDT01 file instead of text")
    gen.add_argument("--out", required=True, help="output update file")

    bench = sub.add_parser("bench", help="static vs dynamic comparison at update percentages")
    bench.add_argument("program")
    bench.add_argument("graph")
    bench.add_argument("--percents", required=True, help="comma list, e.g. 1,5,10,20")
    bench.add_argument("--add-fraction", type=float, default=0.5)
    bench.add_argument("--ranks", type=int, default=1)
    bench.add_argument("--partitioner", choices=("block", "hash"), default="block")
    _add_common_run_flags(bench)

    emit = sub.add_parser("emit", help="(reference compiler; not part of the B200 path)")
    emit.add_argument("program")
    emit.add_argument("--backend", default="omp")
    emit.add_argument("--schedule", default="dynamic")
    emit.add_argument("--out", default="graphdyn_out")

    sim = sub.add_parser("sim", help="run on a vertex-partitioned store over R in-process ranks (one GPU) and "
                                     "report per-rank communication")
    sim.add_argument("program")
    sim.add_argument("graph")
    sim.add_argument("--ranks", type=int, required=True)
    sim.add_argument("--partitioner", default="block")
    sim.add_argument("--entry")
    _add_common_run_flags(sim)

    oracle = sub.add_parser("oracle", help="static recompute of the replayed final graph")
    oracle.add_argument("algo", choices=("sssp", "pr", "tc"))
    oracle.add_argument("graph")
    oracle.add_argument("--updates")
    oracle.add_argument("--src", type=int, default=0)
    oracle.add_argument("--damping", type=float, default=0.85)
    oracle.add_argument("--beta", type=float, default=0.001)
    oracle.add_argument("--maxiter", type=int, default=100)
    oracle.add_argument("--undirected", action="store_true")
    oracle.add_argument("--device", type=int, default=0)
    oracle.add_argument("--out", default="graphdyn_out")
    return parser


# -- inputs ---------------------------------------------------------------------------


def _compile(program: str):
    if program in _PROGRAM_NAMES:  # shorthand: sssp / pr / tc
        return shipped_program(program)
    try:
        text = Path(program).read_text()
    except OSError as exc:
        raise UsageError(f"cannot read program {program!r}: {exc}")
    return compile_source(text)


def _is_binary(path: str, magic: bytes) -> bool:
    with open(path, "rb") as fh:
        return fh.read(8) == magic


def _read_edges(path: str):
    """(src, dst, w, weighted, max_id, node_count_hint, directed_hint)."""
    from .io import _EDGE_MAGIC, load_edges_binary

    if _is_binary(path, _EDGE_MAGIC):
        n, s, d, w, directed = load_edges_binary(path)
        return (np.asarray(s), np.asarray(d), None if w is None else np.asarray(w), w is not None,
                int(max(s.max(), d.max())) if len(s) else -1, n, directed)
    from .io import read_edge_file

    s, d, w, weighted, max_id = read_edge_file(path)
    return s, d, w, weighted, max_id, None, None


def _load_graph(path: str, *, directed: bool, nodes: Optional[int], merge_interval: int, with_reverse: bool,
                device: int):
    from .errors import MalformedInputError
    from .graph import DynamicGraph

    s, d, w, weighted, max_id, n_hint, _ = _read_edges(path)
    n = nodes if nodes is not None else (n_hint if n_hint is not None else max_id + 1)
    if n <= max_id:
        raise MalformedInputError(f"node_count {n} too small for max node id {max_id}", path=path)
    return DynamicGraph.from_arrays(max(n, 0), s, d, w, directed=directed, weighted=weighted,
                                    merge_interval=merge_interval, with_reverse=with_reverse, device=device)


def _load_updates(path: Optional[str]):
    if not path:
        return None
    from .io import _UPD_MAGIC, load_updates_binary
    from .updates import load_update_stream

    return load_updates_binary(path) if _is_binary(path, _UPD_MAGIC) else load_update_stream(path)


def _load_for(check, args, path: str):
    return _load_graph(path, directed=not args.undirected, nodes=args.nodes,
                       merge_interval=getattr(args, "merge_interval", 1),
                       with_reverse=needs_reverse(check.program), device=getattr(args, "device", 0))


def _extra_params(pairs: List[str]) -> Dict[str, str]:
    out = {}
    for pair in pairs:
        if "=" not in pair:
            raise UsageError(f"--param expects NAME=VALUE, got {pair!r}")
        name, value = pair.split("=", 1)
        out[name] = value
    return out


# parameters of the shipped programs' entries (programs/*.sp signatures)
_PARAMS = {
    "dynamicSSSP": ("updateList", "batchsize", "src"),
    "staticSSSP": ("src",),
    "dynamicPR": ("updateList", "batchsize", "damping", "beta", "maxiter"),
    "staticPR": ("damping", "beta", "maxiter"),
    "dynamicTC": ("updateList", "batchsize"),
    "staticTC": (),
}


def _bind_inputs(entry: str, args, updates) -> Dict[str, object]:
    """cli.py:179-220 for the shipped entries."""
    extras = _extra_params(args.param)
    inputs: Dict[str, object] = {}
    if entry not in _PARAMS:
        raise UsageError(f"no function named {entry!r}")
    for p in _PARAMS[entry]:
        if p == "updateList":
            if updates is None:
                raise UsageError(f"program needs --updates for parameter {p!r}")
            inputs[p] = updates
        elif p == "batchsize":
            size = args.batch if args.batch and args.batch > 0 else (len(updates) if updates is not None else 0)
            if size <= 0:
                raise UsageError("--batch must be positive (or provide --updates)")
            inputs[p] = size
        elif p == "src":
            if args.src is None:
                raise UsageError("program needs --src")
            inputs[p] = args.src
        elif p in ("damping", "beta", "maxiter"):
            inputs[p] = getattr(args, p)
        elif p in extras:
            inputs[p] = extras[p]
    return inputs


def _apply_all(graph, updates) -> None:
    """cli.py:232-236: the whole stream as one batch, then merge."""
    batch = updates.as_batch()
    graph.update_csr_del(batch.only_deletes())
    graph.update_csr_add(batch.only_adds())
    graph.merge_deltas()


def _static_entry(check) -> str:
    static = check.program.by_role("Static")
    if not static:
        raise UsageError("program has no Static function for --mode static")
    return static[0].name


# -- outputs ----------------------------------------------------------------------------


def _dump_results(ctx, outdir: str) -> List[str]:
    """cli.py:128-168: one node,value CSV per node property + scalars.csv."""
    out = Path(outdir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    for name, table in ctx.properties.items():
        if not isinstance(table, NodePropertyTable):
            continue
        path = out / f"{name}.csv"
        data = np.asarray(table.data)
        with open(path, "w", newline="") as fh:
            fh.write("node,value\r\n")
            if table.dtype in ("float", "double"):
                fh.writelines(f"{v},{x:.17g}\r\n" for v, x in enumerate(data.tolist()))
            elif table.dtype == "bool":
                fh.writelines(f"{v},{int(x)}\r\n" for v, x in enumerate(data.tolist()))
            else:
                fh.writelines(f"{v},{x}\r\n" for v, x in enumerate(data.tolist()))
        written.append(str(path))
    scalars = {k: v for k, v in ctx.scalars.items() if isinstance(v, (bool, int, float))}
    if ctx.return_value is not None and isinstance(ctx.return_value, (bool, int, float)):
        scalars["return"] = ctx.return_value
    path = out / "scalars.csv"
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["name", "value"])
        for k in sorted(scalars):
            w.writerow([k, scalars[k]])
    written.append(str(path))
    return written


def _values_of(ctx) -> Dict[str, object]:
    out = {}
    for name, table in ctx.properties.items():
        if isinstance(table, NodePropertyTable):
            out[name] = (table.dtype, np.asarray(table.data))
    for name, value in ctx.scalars.items():
        if isinstance(value, (bool, int, float)):
            out[f"scalar:{name}"] = ("scalar", value)
    if isinstance(ctx.return_value, (bool, int, float)):
        out["scalar:return"] = ("scalar", ctx.return_value)
    return out


def _parent_tree_valid(dist, parent, graph, src: Optional[int]):
    """cli.py:322-347, vectorised over the final graph's live arcs."""
    s_all, d_all, w_all = [], [], []
    for seg in graph.segments():
        cnt = np.diff(seg.offsets)
        rows = np.repeat(np.arange(graph.node_count, dtype=np.int64), cnt)
        live = seg.coordinates != np.iinfo(np.int64).max
        s_all.append(rows[live])
        d_all.append(seg.coordinates[live])
        w_all.append(seg.weights[live] if seg.weights is not None else np.ones(int(live.sum()), np.int64))
    s, d, w = np.concatenate(s_all), np.concatenate(d_all), np.concatenate(w_all)
    n = graph.node_count
    v = np.arange(n)
    unreached = dist >= INT_INF
    if src is not None:
        unreached |= v == src
    bad = np.flatnonzero(unreached & (parent != -1))
    if len(bad):
        return False, f"node {int(bad[0])}: expected no parent"
    need = ~unreached & (parent != -1)
    missing = np.flatnonzero(~unreached & (parent == -1))
    if src is not None and len(missing):
        return False, f"node {int(missing[0])}: missing parent"
    key = s * n + d
    order = np.argsort(key, kind="stable")
    ks, ws = key[order], w[order]
    cand = np.flatnonzero(need)
    q = parent[cand] * n + cand
    lo, hi = np.searchsorted(ks, q, "left"), np.searchsorted(ks, q, "right")
    ok = np.zeros(len(cand), dtype=bool)
    for j in range(int((hi - lo).max()) if len(cand) else 0):
        idx = np.minimum(lo + j, max(len(ks) - 1, 0))
        ok |= (lo + j < hi) & (dist[parent[cand]] + ws[idx] == dist[cand])
    if not ok.all():
        b = int(cand[np.flatnonzero(~ok)[0]])
        return False, f"node {b}: parent {int(parent[b])} does not close the distance"
    return True, ""


def _equivalent(dynamic: Dict, static: Dict, *, float_tol: float = 1e-6, final_graph=None,
                src: Optional[int] = None):
    """cli.py:350-393."""
    problems = []
    parent_checked = "dist" in dynamic and "parent" in dynamic and final_graph is not None
    for key in sorted(set(dynamic) & set(static)):
        kind_d, val_d = dynamic[key]
        kind_s, val_s = static[key]
        if kind_d == "scalar":
            if isinstance(val_d, float) or isinstance(val_s, float):
                if abs(val_d - val_s) > float_tol:
                    problems.append(f"{key}: {val_d} vs {val_s}")
            elif val_d != val_s:
                problems.append(f"{key}: {val_d} vs {val_s}")
            continue
        if key == "parent" and parent_checked:
            ok, why = _parent_tree_valid(dynamic["dist"][1], val_d, final_graph, src)
            if not ok:
                problems.append(f"parent: {why}")
            continue
        if kind_d in ("float", "double"):
            worst = float(np.max(np.abs(val_d - val_s))) if len(val_d) else 0.0
            if worst > float_tol:
                problems.append(f"{key}: max |delta| {worst:.3g}")
        elif kind_d in ("int", "long", "node"):
            if not np.array_equal(val_d, val_s):
                problems.append(f"{key}: {int(np.count_nonzero(val_d != val_s))} differing entries")
    return (not problems, "; ".join(problems))


# -- subcommands ------------------------------------------------------------------------


def cmd_run(args) -> int:
    check = _compile(args.program)
    updates = _load_updates(args.updates)
    graph = _load_for(check, args, args.graph)
    if args.mode == "static":
        entry = args.entry or _static_entry(check)
        if updates is not None:
            _apply_all(graph, updates)
        if check.program.function(entry) is None:
            raise UsageError(f"no function named {entry!r}")
        inputs = _bind_inputs(entry, args, None)
    else:
        entry = args.entry or check.program.entry
        if check.program.function(entry) is None:
            raise UsageError(f"no function named {entry!r}")
        inputs = _bind_inputs(entry, args, updates)
    start = time.perf_counter()
    ctx = run_program(check, graph, inputs, entry=entry, worker_count=args.threads,
                      iteration_cap_factor=args.iteration_cap_factor)
    wall = time.perf_counter() - start
    files = _dump_results(ctx, args.out)
    manifest = build_manifest(command="run", args=vars(args), seed=args.seed,
                              input_files={"program": args.program if Path(args.program).is_file() else None,
                                           "graph": args.graph, "updates": args.updates},
                              ctx=ctx, extra={"wall_seconds": wall, "mode": args.mode, "entry": entry,
                                              "results": files})
    write_manifest(manifest, args.out)
    return EXIT_OK


def _generate(args, s, d, w, node_count: int, percent: float):
    from . import generate as G

    return G.py_generate_updates(s, d, w if w is not None else np.ones(len(s), np.int64), node_count, percent,
                                 seed=args.seed, add_fraction=args.add_fraction, undirected=args.undirected)


def _stream(kind, us, ud, uw):
    from .updates import UpdateStream

    return UpdateStream.from_arrays(kind, us, ud, uw)


def cmd_gen_updates(args) -> int:
    """cli.py:283-297; the stream is the reference's own for the same seed."""
    s, d, w, _, max_id, n_hint, _ = _read_edges(args.graph)
    node_count = n_hint if n_hint is not None else max_id + 1
    kind, us, ud, uw = _generate(args, s, d, w, node_count, args.percent)
    if args.binary:
        from .io import save_updates_binary

        save_updates_binary(args.out, kind, us, ud, uw)
    else:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.writelines(f"a {a} {b} {c}\n" if k == ord("a") else f"d {a} {b}\n"
                          for k, a, b, c in zip(kind.tolist(), us.tolist(), ud.tolist(), uw.tolist()))
    print(f"wrote {len(kind)} updates to {args.out}")
    return EXIT_OK


def cmd_bench(args) -> int:
    """cli.py:396-491: per percentage, dynamic batches vs a static recompute
    of the final graph, with the reference's equivalence check."""
    check = _compile(args.program)
    try:
        percents = [float(p) for p in args.percents.split(",") if p.strip()]
    except ValueError:
        raise UsageError(f"bad --percents value {args.percents!r}")
    if not percents:
        raise UsageError("--percents must name at least one percentage")
    if args.ranks > 1:
        raise UsageError("--ranks > 1 uses the reference's partition simulator; the B200 path runs multi-GPU "
                         "under torchrun (bench.py --gpus N)")
    s, d, w, _, max_id, n_hint, _ = _read_edges(args.graph)
    node_count = args.nodes or (n_hint if n_hint is not None else max_id + 1)
    outdir = Path(args.out)
    outdir.mkdir(parents=True, exist_ok=True)
    rows = []
    for percent in percents:
        kind, us, ud, uw = _generate(args, s, d, w, node_count, percent)
        updates = _stream(kind, us, ud, uw)
        with open(outdir / f"updates_p{percent:g}.txt", "w", encoding="utf-8") as fh:
            fh.writelines(f"a {a} {b} {c}\n" if k == ord("a") else f"d {a} {b}\n"
                          for k, a, b, c in zip(kind.tolist(), us.tolist(), ud.tolist(), uw.tolist()))
        g_dyn = _load_for(check, args, args.graph)
        entry = check.program.entry
        inputs = _bind_inputs(entry, args, updates)
        t0 = time.perf_counter()
        ctx_dyn = run_program(check, g_dyn, inputs, worker_count=args.threads,
                              iteration_cap_factor=args.iteration_cap_factor)
        dyn_wall = time.perf_counter() - t0
        dyn_batch = dyn_wall - ctx_dyn.phase_totals.get("static_phase", 0.0)

        g_stat = _load_for(check, args, args.graph)
        _apply_all(g_stat, updates)
        static_entry = _static_entry(check)
        static_inputs = _bind_inputs(static_entry, args, None)
        t0 = time.perf_counter()
        ctx_stat = run_program(check, g_stat, static_inputs, entry=static_entry, worker_count=args.threads,
                               iteration_cap_factor=args.iteration_cap_factor)
        stat_wall = time.perf_counter() - t0
        ok, detail = _equivalent(_values_of(ctx_dyn), _values_of(ctx_stat), final_graph=g_stat, src=args.src)
        row = {"percent": percent, "updates": len(kind), "static_seconds": round(stat_wall, 6),
               "dynamic_seconds": round(dyn_batch, 6), "dynamic_total_seconds": round(dyn_wall, 6),
               "speedup": round(stat_wall / dyn_batch, 3) if dyn_batch > 0 else float("inf"), "equivalent": ok}
        rows.append(row)
        if not ok:
            _write_bench(rows, outdir)
            print(f"equivalence failure at {percent}%: {detail}", file=sys.stderr)
            return EXIT_EQUIVALENCE
        print(f"percent={percent:g} updates={len(kind)} static={stat_wall:.3f}s dynamic={dyn_batch:.3f}s "
              f"speedup={row['speedup']}")
    _write_bench(rows, outdir)
    manifest = build_manifest(command="bench", args=vars(args), seed=args.seed,
                              input_files={"program": args.program if Path(args.program).is_file() else None,
                                           "graph": args.graph}, extra={"rows": rows})
    write_manifest(manifest, str(outdir))
    return EXIT_OK


def _write_bench(rows, outdir: Path) -> None:
    if not rows:
        return
    with open(outdir / "bench.csv", "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
        w.writeheader()
        for row in rows:
            w.writerow(row)


def _replay(graph, updates) -> None:
    """Apply the stream in record order (oracles.py:143-160): consecutive
    records go into one batch until a pair repeats, so every batch's
    deletes-then-adds order equals the stream order."""
    arr = updates.arrays
    n = len(arr)
    if n == 0:
        return
    und = not graph.directed
    a, b = arr.src.astype(np.int64), arr.dst.astype(np.int64)
    if und:
        a, b = np.minimum(a, b), np.maximum(a, b)
    key = a * max(graph.node_count, 1) + b
    start = 0
    seen = set()
    for i, k in enumerate(key.tolist()):
        if k in seen:
            _apply_part(graph, arr.slice(start, i))
            start, seen = i, set()
        seen.add(k)
    _apply_part(graph, arr.slice(start, n))
    graph.merge_deltas()


def _apply_part(graph, part) -> None:
    from .updates import UpdateBatch

    b = UpdateBatch(arrays=part)
    graph.update_csr_del(b.only_deletes())
    graph.update_csr_add(b.only_adds())


def cmd_oracle(args) -> int:
    """cli.py:571-596 on the GPU: the static entry on the replayed graph."""
    check = shipped_program(args.algo)
    graph = _load_graph(args.graph, directed=not args.undirected, nodes=None, merge_interval=1,
                        with_reverse=needs_reverse(check.program), device=args.device)
    updates = _load_updates(args.updates)
    if updates is not None:
        _replay(graph, updates)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    entry = _static_entry(check)
    if args.algo == "sssp":
        ctx = run_program(check, graph, {"src": args.src}, entry=entry)
        dist = np.asarray(ctx.properties["dist"].data)
        with open(out / "dist.csv", "w", newline="") as fh:
            fh.write("node,value\r\n")
            fh.writelines(f"{v},{x}\r\n" for v, x in enumerate(dist.tolist()))
        print(f"wrote {out / 'dist.csv'}")
    elif args.algo == "pr":
        ctx = run_program(check, graph, {"damping": args.damping, "beta": args.beta, "maxiter": args.maxiter},
                          entry=entry)
        rank = np.asarray(ctx.properties["pagerank"].data)
        with open(out / "pagerank.csv", "w", newline="") as fh:
            fh.write("node,value\r\n")
            fh.writelines(f"{v},{x:.17g}\r\n" for v, x in enumerate(rank.tolist()))
        print(f"wrote {out / 'pagerank.csv'}")
    else:
        ctx = run_program(check, graph, {}, entry=entry)
        count = int(ctx.return_value)
        (out / "scalars.csv").write_text(f"name,value\ntcount,{count}\n")
        print(f"triangles: {count}")
    return EXIT_OK


def cmd_sim(args) -> int:
    """cli.py:520-568 on the B200 path: instead of the reference's
    in-process simulation of one-sided windows, the program runs on a REAL
    vertex-partitioned store (gd_graph_create_dist) over `--ranks` ranks of
    an in-process group on one GPU (one host thread per rank, the NCCL call
    sequence with device copies), and commstats.csv reports what each rank
    actually moved.  Directed SSSP / PR partition the store; TC (undirected)
    keeps replicas and splits the records.  Results come from rank 0 (every
    rank holds the same values)."""
    from concurrent.futures import ThreadPoolExecutor

    from .dist import Communicator
    from .graph import DynamicGraph

    if args.partitioner != "block":
        raise UsageError("the B200 path partitions by 1D vertex blocks only (--partitioner block)")
    if args.ranks < 1:
        raise UsageError("--ranks must be >= 1")
    check = _compile(args.program)
    updates = _load_updates(args.updates)
    entry = args.entry or check.program.entry
    if check.program.function(entry) is None:
        raise UsageError(f"no function named {entry!r}")
    inputs = _bind_inputs(entry, args, updates)
    s, d, w, weighted, max_id, n_hint, _ = _read_edges(args.graph)
    n = args.nodes if args.nodes is not None else (n_hint if n_hint is not None else max_id + 1)
    directed = not args.undirected
    name = check.program.name
    partition = directed and name in ("sssp_dynamic", "pr_dynamic")
    if args.ranks > max(n, 1):
        raise UsageError(f"rank_count {args.ranks} exceeds node count {n}")
    comms = Communicator.local_group(args.ranks, device=args.device, group=os.getpid())

    def rank_fn(r):
        g = DynamicGraph.from_arrays(max(n, 0), s, d, w, directed=directed, weighted=weighted,
                                     merge_interval=args.merge_interval, with_reverse=needs_reverse(check.program),
                                     device=args.device, comm=comms[r] if partition else None)
        kw = {}
        if not partition and name == "tc_dynamic":
            kw["comm"] = comms[r]
        ctx = run_program(check, g, inputs, entry=entry, iteration_cap_factor=args.iteration_cap_factor, **kw)
        return ctx, comms[r].stats()

    start = time.perf_counter()
    with ThreadPoolExecutor(args.ranks) as ex:
        res = list(ex.map(rank_fn, range(args.ranks)))
    wall = time.perf_counter() - start
    ctx = res[0][0]
    files = _dump_results(ctx, args.out)
    stats_path = Path(args.out) / "commstats.csv"
    cols = ["rank", "collective_calls", "allgather_bytes", "allreduce_bytes", "alltoall_bytes", "bytes_moved"]
    rows = [{"rank": r, "collective_calls": st["calls"], "allgather_bytes": st["allgather_bytes"],
             "allreduce_bytes": st["allreduce_bytes"], "alltoall_bytes": st["alltoall_bytes"],
             "bytes_moved": st["sent_bytes"]} for r, (_, st) in enumerate(res)]
    with open(stats_path, "w", newline="") as fh:
        wr = csv.DictWriter(fh, fieldnames=cols)
        wr.writeheader()
        for row in rows:
            wr.writerow(row)
    manifest = build_manifest(command="sim", args=vars(args), seed=args.seed,
                              input_files={"program": args.program if Path(args.program).is_file() else None,
                                           "graph": args.graph, "updates": args.updates},
                              ctx=ctx, extra={"wall_seconds": wall, "ranks": args.ranks,
                                              "partitioned_store": partition,
                                              "results": files + [str(stats_path)],
                                              "comm_totals": {c: sum(r[c] for r in rows) for c in cols[1:]}})
    write_manifest(manifest, args.out)
    print(f"per-rank communication stats in {stats_path}")
    return EXIT_OK


def cmd_out_of_scope(args) -> int:
    raise UsageError(f"'{args.command}' belongs to the reference's compiler / simulator and is not part of the "
                     f"B200 path (DESIGN.md §8)")


def main(argv: Optional[List[str]] = None) -> int:
    parser = make_parser()
    args = parser.parse_args(argv)
    handlers = {"run": cmd_run, "gen-updates": cmd_gen_updates, "bench": cmd_bench, "emit": cmd_out_of_scope,
                "sim": cmd_sim, "oracle": cmd_oracle}
    try:
        return handlers[args.command](args)
    except UsageError as exc:
        print(f"graphdyn: usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except CompileError as exc:
        print(f"graphdyn: compile diagnostics:\n{exc}", file=sys.stderr)
        return EXIT_COMPILE
    except GraphDynError as exc:
        print(f"graphdyn: error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
