"""Generate the golden parity fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built):

    make -C oracle all && python tests/golden/make_golden.py

Two sources, both the unmodified reference:
  * the reference Python package (/root/reference/pkg/src/graphdyn): the store
    (DynamicGraph) and the engine (run_batches over the shipped .sp programs);
  * the reference's emitted OpenMP programs (tests/golden/*_omp.cc), run
    through oracle/_ref/libgdref.so for the larger cases.

Fixtures are small .npz files; tests/test_oracle_golden.py pins oracle/ to
them (CPU) and tests/test_gpu_parity.py pins the CUDA path to them (GPU).
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from graphdyn.engine import run_batches, run_program  # noqa: E402
from graphdyn.frontend import compile_source  # noqa: E402
from graphdyn.generate import generate_updates, rmat_graph, uniform_random_graph  # noqa: E402
from graphdyn.graph import ADD, DELETE, SENTINEL, DynamicGraph, UpdateBatch, UpdateRecord, UpdateStream  # noqa: E402

from oracle import oracle as O  # noqa: E402

PROG = "/root/reference/pkg/src/graphdyn/programs"
CHECK = {n: compile_source(open(f"{PROG}/{n}.sp").read()) for n in ("sssp_dynamic", "pr_dynamic", "tc_dynamic")}


def rec_arrays(records):
    kind = np.array([ord(r.kind) for r in records], dtype=np.uint8)
    s = np.array([r.src for r in records], dtype=np.int64)
    d = np.array([r.dst for r in records], dtype=np.int64)
    w = np.array([r.weight for r in records], dtype=np.int64)
    return kind, s, d, w


def edge_arrays(edges):
    if not edges:
        z = np.zeros(0, dtype=np.int64)
        return z, z, z
    a = np.asarray(edges, dtype=np.int64)
    return a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy()


def seg_dump(g: DynamicGraph):
    """Segments exactly as the reference lays them out (SENTINEL kept)."""
    out = []
    for seg in g.segments():
        w = seg.weights if seg.weights is not None else np.ones(len(seg.coordinates), dtype=np.int64)
        out.append((seg.offsets.copy(), seg.coordinates.copy(), np.asarray(w, dtype=np.int64).copy()))
    return out


def rev_dump(g: DynamicGraph, slots=False):
    """Reverse lists (nodes_to) in the reference's own list order; with
    slots=True the EdgeRef slot identities (segment, index) instead."""
    off = [0]
    src, wts = [], []
    for v in range(g.node_count):
        for e in g.nodes_to(v):
            src.append(e.segment if slots else e.source)
            wts.append(e.index if slots else e.weight)
        off.append(len(src))
    return np.array(off, dtype=np.int64), np.array(src, dtype=np.int64), np.array(wts, dtype=np.int64)


# -- store fixtures: the reference's own randomized workload (test_graph_store.py:251-313) ------

def random_workload(seed, n, initial_edges, num_batches, batch_len):
    rng = random.Random(seed)
    weight = lambda u, v: (min(u, v) * 31 + max(u, v)) % 9 + 1  # noqa: E731
    edges = []
    for _ in range(initial_edges):
        u, v = rng.randrange(n), rng.randrange(n)
        edges.append((u, v, weight(u, v)))
    batches = []
    for _ in range(num_batches):
        records = []
        for _ in range(batch_len):
            u, v = rng.randrange(n), rng.randrange(n)
            if rng.random() < 0.45:
                records.append(UpdateRecord(DELETE, u, v))
            else:
                records.append(UpdateRecord(ADD, u, v, weight(u, v)))
        batches.append(records)
    return edges, batches


def store_case(name, n, edges, batches, directed, merge_every, out):
    g = DynamicGraph.build(edges, n, directed=directed, weighted=True, with_reverse=True)
    es, ed, ew = edge_arrays(edges)
    out[f"{name}/meta"] = np.array([n, int(directed), merge_every, len(batches)], dtype=np.int64)
    out[f"{name}/edges"] = np.stack([es, ed, ew]) if len(es) else np.zeros((3, 0), dtype=np.int64)

    def snap(tag):
        # one flat int64 record per snapshot: [nseg, live, (nslots, off, coord, w) * nseg,
        #                                        rev_total, rev_off, rev_src, rev_w]
        segs = seg_dump(g)
        parts = [np.array([len(segs), g.live_edge_count], dtype=np.int64)]
        for o, c, w in segs:
            parts += [np.array([len(c)], dtype=np.int64), o, c, w]
        ro, rs, rw = rev_dump(g)
        parts += [np.array([len(rs)], dtype=np.int64), ro, rs, rw]
        out[f"{name}/{tag}"] = np.concatenate(parts)
        _, rseg, ridx = rev_dump(g, slots=True)
        out[f"{name}/{tag}/revslots"] = np.stack([rseg, ridx]) if len(rseg) else np.zeros((2, 0), np.int64)

    snap("build")
    for i, records in enumerate(batches):
        b = UpdateBatch(records)
        kind, s, d, w = rec_arrays(records)
        out[f"{name}/b{i}/recs"] = np.stack([kind.astype(np.int64), s, d, w]) if len(kind) else np.zeros((4, 0), np.int64)
        rep = g.update_csr_del(b.only_deletes())
        missed = {id(r) for r in rep.missed}
        out[f"{name}/b{i}/report"] = np.array([rep.applied, rep.misses], dtype=np.int64)
        out[f"{name}/b{i}/missflags"] = np.array([1 if id(r) in missed else 0 for r in b.only_deletes().records],
                                                 dtype=np.uint8)
        snap(f"b{i}/del")
        g.update_csr_add(b.only_adds())
        snap(f"b{i}/add")
        if merge_every and (i + 1) % merge_every == 0:
            g.merge_deltas()
            snap(f"b{i}/merge")
    g.check_invariants()


def make_store(path):
    out = {}
    names = []
    # diff-CSR figure walkthrough (test_graph_store.py:22-23,111-138)
    A, B, Cc, D, E, F = range(6)
    fig = [(A, B, 1), (B, Cc, 1), (B, D, 1), (Cc, A, 1), (D, E, 1), (D, F, 1), (F, A, 1)]
    store_case("figure", 6, fig, [[UpdateRecord(DELETE, B, D), UpdateRecord(ADD, E, Cc, 1)],
                                  [UpdateRecord(ADD, B, E, 1)]], True, 0, out)
    names.append("figure")
    store_case("parallel", 3, [(0, 1, 1), (0, 1, 1), (0, 2, 1)],
               [[UpdateRecord(DELETE, 0, 1), UpdateRecord(DELETE, 0, 1), UpdateRecord(DELETE, 0, 1)],
                [UpdateRecord(ADD, 0, 1, 1), UpdateRecord(ADD, 0, 1, 1), UpdateRecord(ADD, 2, 2, 1)]], True, 0, out)
    names.append("parallel")
    for seed in range(0, 240):
        directed = seed < 120
        merge_every = seed % 3
        n = random.Random(seed * 13 + 1).randrange(2, 14)
        edges, batches = random_workload(seed, n, initial_edges=10, num_batches=4, batch_len=6)
        nm = f"rw{seed}"
        store_case(nm, n, edges, batches, directed, merge_every, out)
        names.append(nm)
    for seed in range(1000, 1012):  # larger: n up to 60, denser batches
        directed = seed % 2 == 0
        edges, batches = random_workload(seed, 60, initial_edges=300, num_batches=3, batch_len=80)
        nm = f"rwL{seed}"
        store_case(nm, 60, edges, batches, directed, [0, 1, 2][seed % 3], out)
        names.append(nm)
    out["names"] = np.array(names)
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} store cases")


# -- algorithm fixtures from the reference engine ------------------------------------

BOOL_PROPS = {}  # {prop: uint8[n]} of the last engine_run (filled by engine_run)


def engine_run(algo, edges, n, records, batch, *, directed=True, weighted=False, merge_interval=1,
               src=0, damping=0.85, beta=0.001, maxiter=100, cap=10):
    prog = {"sssp": "sssp_dynamic", "pr": "pr_dynamic", "tc": "tc_dynamic"}[algo]
    g = DynamicGraph.build(edges, n, directed=directed, weighted=weighted, merge_interval=merge_interval,
                           with_reverse=algo != "tc")
    inputs = {"sssp": {"src": src}, "pr": {"damping": damping, "beta": beta, "maxiter": maxiter}, "tc": {}}[algo]
    ctx = run_batches(CHECK[prog], g, UpdateStream(records), batch, inputs, iteration_cap_factor=cap)
    BOOL_PROPS.clear()
    for pname, table in ctx.properties.items():
        if getattr(table, "dtype", None) == "bool" and hasattr(table, "values"):
            BOOL_PROPS[pname] = np.array(table.values(), dtype=np.uint8)
    if algo == "sssp":
        return np.array(ctx.properties["dist"].values(), dtype=np.int64), np.array(
            ctx.properties["parent"].values(), dtype=np.int64)
    if algo == "pr":
        return np.array(ctx.properties["pagerank"].values(), dtype=np.float64)
    return np.array([ctx.return_value], dtype=np.int64)


INF = 2 ** 63 - 1


def put_case(out, names, name, algo, n, edges, records, batch, *, directed, weighted, merge_interval=1,
             src=0, damping=0.85, beta=0.001, maxiter=100, result=None, source="engine"):
    es, ed, ew = edge_arrays(edges)
    kind, s, d, w = rec_arrays(records)
    out[f"{name}/meta"] = np.array([n, int(directed), int(weighted), merge_interval, batch, src, maxiter],
                                   dtype=np.int64)
    out[f"{name}/fmeta"] = np.array([damping, beta], dtype=np.float64)
    out[f"{name}/algo"] = np.array([algo])
    out[f"{name}/source"] = np.array([source])
    out[f"{name}/edges"] = np.stack([es, ed, ew])
    out[f"{name}/recs"] = np.stack([kind.astype(np.int64), s, d, w]) if len(kind) else np.zeros((4, 0), np.int64)
    if source == "engine":
        for pname, vals in BOOL_PROPS.items():
            out[f"{name}/prop/{pname}"] = vals
        out[f"{name}/propnames"] = np.array(list(BOOL_PROPS) or [""])
    if algo == "sssp":
        out[f"{name}/dist"], out[f"{name}/parent"] = result
    elif algo == "pr":
        out[f"{name}/rank"] = result
    else:
        out[f"{name}/count"] = np.asarray(result, dtype=np.int64).reshape(1)
    names.append(name)


def make_algos(path):
    out = {}
    names = []
    # worked example (test_engine.py:15,247-254; test_acceptance.py:47-63)
    ex = [(0, 1, 30), (0, 2, 20), (0, 3, 48), (3, 4, 4), (2, 5, 25), (4, 5, 6)]
    recs = [UpdateRecord(DELETE, 2, 5), UpdateRecord(ADD, 1, 3, 10)]
    r = engine_run("sssp", ex, 6, recs, 2, weighted=True)
    assert list(r[0]) == [0, 30, 20, 40, 44, 50]
    put_case(out, names, "sssp_worked", "sssp", 6, ex, recs, 2, directed=True, weighted=True, result=r)
    # INF saturation [0, INF, 5] (test_engine.py:344-349)
    inf_e = [(0, 2, 5)]
    r = engine_run("sssp", inf_e, 3, [], 1, weighted=True)
    put_case(out, names, "sssp_inf", "sssp", 3, inf_e, [], 1, directed=True, weighted=True, result=r)
    # TC cliques (test_oracles.py:61-75)
    k4 = [(a, b, 1) for a in range(4) for b in range(a + 1, 4)]
    r = engine_run("tc", k4, 4, [UpdateRecord(DELETE, 0, 1), UpdateRecord(ADD, 0, 1, 1)], 1, directed=False)
    put_case(out, names, "tc_k4", "tc", 4, k4, [UpdateRecord(DELETE, 0, 1), UpdateRecord(ADD, 0, 1, 1)], 1,
             directed=False, weighted=False, result=r)
    # PR two-cycle (test_engine.py:29-37)
    r = engine_run("pr", [(0, 1, 1), (1, 0, 1)], 2, [], 1, beta=1e-12, maxiter=500)
    put_case(out, names, "pr_cycle", "pr", 2, [(0, 1, 1), (1, 0, 1)], [], 1, directed=True, weighted=False,
             beta=1e-12, maxiter=500, result=r)

    # random small graphs: uniform + rmat, all three programs, several batch sizes / merge cadences
    case = 0
    for seed in range(30):
        n = [24, 40, 64, 90][seed % 4]
        m = n * [2, 3, 4][seed % 3]
        if seed % 2 == 0:
            edges = uniform_random_graph(n, m, seed=seed, weighted=True, max_weight=9)
        else:
            edges, n = rmat_graph(6 + seed % 2, m, seed=seed, weighted=True, max_weight=9)
        pct = [5, 10, 20][seed % 3]
        records = generate_updates(edges, n, pct, seed=seed + 100)
        batch = [1, 7, max(1, len(records))][seed % 3]
        mi = [1, 1, 2][seed % 3]
        r = engine_run("sssp", edges, n, records, batch, weighted=True, merge_interval=mi, src=seed % n)
        put_case(out, names, f"sssp_r{case}", "sssp", n, edges, records, batch, directed=True, weighted=True,
                 merge_interval=mi, src=seed % n, result=r)
        beta = [1e-3, 1e-10][seed % 2]
        r = engine_run("pr", edges, n, records, batch, merge_interval=mi, beta=beta, maxiter=300)
        put_case(out, names, f"pr_r{case}", "pr", n, edges, records, batch, directed=True, weighted=False,
                 merge_interval=mi, beta=beta, maxiter=300, result=r)
        uedges = uniform_random_graph(n, m, seed=seed + 7, undirected=True)
        urecs = generate_updates(uedges, n, pct, seed=seed + 200, undirected=True)
        r = engine_run("tc", uedges, n, urecs, batch, directed=False, merge_interval=mi)
        put_case(out, names, f"tc_r{case}", "tc", n, uedges, urecs, batch, directed=False, weighted=False,
                 merge_interval=mi, result=r)
        case += 1
    # multigraph / misses / self-loop edge cases straight through the engine
    rng = random.Random(5)
    for j in range(6):
        n = 12
        edges = [(rng.randrange(n), rng.randrange(n), rng.randint(1, 5)) for _ in range(40)]
        records = []
        for _ in range(30):
            u, v = rng.randrange(n), rng.randrange(n)
            if rng.random() < 0.5:
                records.append(UpdateRecord(DELETE, u, v))
            else:
                records.append(UpdateRecord(ADD, u, v, rng.randint(1, 5)))
        bs = [3, 10, 30][j % 3]
        r = engine_run("sssp", edges, n, records, bs, weighted=True, merge_interval=1 + j % 2)
        put_case(out, names, f"sssp_multi{j}", "sssp", n, edges, records, bs, directed=True, weighted=True,
                 merge_interval=1 + j % 2, result=r)
        try:
            r = engine_run("pr", edges, n, records, bs, merge_interval=1 + j % 2, beta=1e-10, maxiter=300)
            put_case(out, names, f"pr_multi{j}", "pr", n, edges, records, bs, directed=True, weighted=False,
                     merge_interval=1 + j % 2, beta=1e-10, maxiter=300, result=r)
        except ZeroDivisionError:
            # a missed delete still decrements outdeg (pr_dynamic.sp:87-92); once an
            # out-degree reaches 0 under a live arc the engine divides by zero
            print(f"pr_multi{j}: reference engine raised ZeroDivisionError; case skipped")
        r = engine_run("tc", edges, n, records, bs, directed=False, merge_interval=1 + j % 2)
        put_case(out, names, f"tc_multi{j}", "tc", n, edges, records, bs, directed=False, weighted=False,
                 merge_interval=1 + j % 2, result=r)

    # undirected and unweighted SSSP: OnAdd relaxes only the record's own
    # direction with the record's own weight, so non-stale distances need not
    # be tight; the decremental repair may change stale nodes only
    # (sssp_dynamic.sp:68-86).  First the advisor's repro.
    rep_e = [(0, 1, 1), (0, 3, 1), (3, 1, 1), (3, 4, 1), (4, 5, 1), (5, 6, 1)]
    rep_r = [UpdateRecord(ADD, 6, 1, 1), UpdateRecord(DELETE, 0, 1)]
    r = engine_run("sssp", rep_e, 7, rep_r, 1, directed=False)
    assert list(r[0]) == [0, 2, INF, 1, 2, 3, 4] and list(r[1]) == [-1, 3, -1, 0, 3, 4, 5]
    put_case(out, names, "sssp_und_repro", "sssp", 7, rep_e, rep_r, 1, directed=False, weighted=False, result=r)
    for j in range(12):
        n = [16, 30, 48, 70][j % 4]
        m = n * [2, 3][j % 2]
        directed = j % 3 == 2
        weighted = j % 2 == 0
        edges = uniform_random_graph(n, m, seed=300 + j, weighted=True, max_weight=7, undirected=not directed)
        if not weighted:
            edges = [(u, v, 1) for u, v, _ in edges]
        recs = generate_updates(edges, n, [10, 20, 30][j % 3], seed=400 + j, undirected=not directed)
        rng = random.Random(500 + j)
        # record weights above 1 on an unweighted store (OnAdd reads them)
        recs = [UpdateRecord(rc.kind, rc.src, rc.dst, rng.randint(1, 6)) if rc.kind == ADD else rc for rc in recs]
        bs = [1, 4, 11, max(1, len(recs))][j % 4]
        mi = [1, 2][j % 2]
        r = engine_run("sssp", edges, n, recs, bs, directed=directed, weighted=weighted, merge_interval=mi,
                       src=j % n)
        put_case(out, names, f"sssp_und{j}", "sssp", n, edges, recs, bs, directed=directed, weighted=weighted,
                 merge_interval=mi, src=j % n, result=r)

    # larger cases from the reference's emitted OpenMP programs (--threads 1)
    for j, (lg, m, pct) in enumerate([(10, 6000, 5), (11, 16000, 10), (12, 40000, 5)]):
        edges, n = rmat_graph(lg, m, seed=40 + j, weighted=True, max_weight=100)
        records = generate_updates(edges, n, pct, seed=50 + j)
        es, ed, ew = edge_arrays(edges)
        kind, s, d, w = rec_arrays(records)
        batch = [len(records), 97, 1000][j]
        res, _ = O.ref_run("sssp", n, es, ed, ew, weighted=True, kind=kind, us=s, ud=d, uw=w,
                           batch_size=batch, threads=1, skip_t0=True)
        put_case(out, names, f"sssp_omp{j}", "sssp", n, edges, records, batch, directed=True, weighted=True,
                 result=res, source="omp")
        res, _ = O.ref_run("pr", n, es, ed, ew, kind=kind, us=s, ud=d, uw=w, batch_size=batch, threads=1,
                           beta=1e-10, maxiter=300, skip_t0=True)
        put_case(out, names, f"pr_omp{j}", "pr", n, edges, records, batch, directed=True, weighted=False,
                 beta=1e-10, maxiter=300, result=res, source="omp")
        ue = uniform_random_graph(1 << lg, m // 2, seed=60 + j, undirected=True)
        ur = generate_updates(ue, 1 << lg, pct, seed=70 + j, undirected=True)
        es, ed, ew = edge_arrays(ue)
        kind, s, d, w = rec_arrays(ur)
        res, _ = O.ref_run("tc", 1 << lg, es, ed, ew, directed=False, kind=kind, us=s, ud=d, uw=w,
                           batch_size=batch, threads=1, skip_t0=True)
        put_case(out, names, f"tc_omp{j}", "tc", 1 << lg, ue, ur, batch, directed=False, weighted=False,
                 result=res, source="omp")
    out["names"] = np.array(names)
    make_caps(out)
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} algorithm cases")


def make_caps(out):
    """iteration_cap_factor -> DivergenceError (interp.py:138-139,800-813):
    for each case, whether the reference raises at each factor."""
    from graphdyn.errors import DivergenceError

    cases = []
    # directed unit path: the static fixpoint needs exactly n body runs
    path = [(i, i + 1, 1) for i in range(9)]
    cases.append(("cap_path", 10, path, [], 1, True, False))
    # the worked example with its batch
    ex = [(0, 1, 30), (0, 2, 20), (0, 3, 48), (3, 4, 4), (2, 5, 25), (4, 5, 6)]
    cases.append(("cap_worked", 6, ex, [UpdateRecord(DELETE, 2, 5), UpdateRecord(ADD, 1, 3, 10)], 2, True, True))
    names = []
    for name, n, edges, recs, bs, directed, weighted in cases:
        factors = [0, 1, 2, 10]
        div = []
        for f in factors:
            try:
                engine_run("sssp", edges, n, recs, bs, directed=directed, weighted=weighted, cap=f)
                div.append(0)
            except DivergenceError:
                div.append(1)
        es, ed, ew = edge_arrays(edges)
        kind, s, d, w = rec_arrays(recs)
        out[f"{name}/meta"] = np.array([n, int(directed), int(weighted), bs], dtype=np.int64)
        out[f"{name}/edges"] = np.stack([es, ed, ew])
        out[f"{name}/recs"] = np.stack([kind.astype(np.int64), s, d, w]) if len(kind) else np.zeros((4, 0), np.int64)
        out[f"{name}/factors"] = np.array(factors, dtype=np.int64)
        out[f"{name}/diverged"] = np.array(div, dtype=np.int64)
        names.append(name)
        print(name, dict(zip(factors, div)))
    out["cap_names"] = np.array(names)


if __name__ == "__main__":
    make_store(os.path.join(HERE, "store_cases.npz"))
    make_algos(os.path.join(HERE, "algo_cases.npz"))
