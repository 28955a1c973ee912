"""Repeat the partitioned / unpartitioned SSSP case of
tests/test_dist_local_gpu.py against the CPU oracle to locate a rare
mismatch (which side, which batch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2507_11094_b200 as gd
from paper_2507_11094_b200 import generate as G
from oracle import oracle as O
from test_dist_local_gpu import run_ranks

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
s, d, w, n = G.rmat(12, 40_000, seed=7, weighted=True, max_weight=100)
kind, us, ud, uw, per = G.updates(s, d, n, percent=5, batches=3, seed=8, max_weight=100)
stream = gd.UpdateStream.from_arrays(kind, us, ud, uw)
og = O.OracleGraph(n, s, d, w, weighted=True, with_reverse=True)
odist, opar = O.OracleSSSP(og, 0).run_stream(kind, us, ud, uw, per).read()
bad = {"single": 0, "w2": 0, "w3": 0}
for it in range(reps):
    ref = gd.run_batches(gd.shipped_program("sssp"),
                         gd.DynamicGraph.from_arrays(n, s, d, w, weighted=True, with_reverse=True), stream, per,
                         {"src": 0})
    dd = np.asarray(ref.properties["dist"].data)
    if not (np.array_equal(dd, odist) and np.array_equal(np.asarray(ref.properties["parent"].data), opar)):
        bad["single"] += 1
        i = np.flatnonzero(dd != odist)
        print(f"rep {it}: SINGLE-GPU mismatch at {i[:5]} got {dd[i[:5]]} want {odist[i[:5]]}", flush=True)
    for world in (2, 3):
        def rank_fn(r, comm):
            g = gd.DynamicGraph.from_arrays(n, s, d, w, weighted=True, with_reverse=True, comm=comm)
            ctx = gd.run_batches(gd.shipped_program("sssp"), g, stream, per, {"src": 0})
            return np.asarray(ctx.properties["dist"].data), np.asarray(ctx.properties["parent"].data)
        for rk, (dist, parent) in enumerate(run_ranks(world, rank_fn)):
            if not (np.array_equal(dist, odist) and np.array_equal(parent, opar)):
                bad[f"w{world}"] += 1
                i = np.flatnonzero(dist != odist)
                j = np.flatnonzero(parent != opar)
                print(f"rep {it}: world {world} rank {rk} mismatch dist at {i[:5]} got {dist[i[:5]]} want "
                      f"{odist[i[:5]]}; parent at {j[:5]}", flush=True)
print("mismatches:", bad, "of", reps)
