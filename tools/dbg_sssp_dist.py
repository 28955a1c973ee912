import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2507_11094_b200 as gd
from paper_2507_11094_b200 import generate as G
from concurrent.futures import ThreadPoolExecutor
from paper_2507_11094_b200.dist import Communicator
s, d, w, n = G.rmat(12, 40_000, seed=7, weighted=True, max_weight=100)
kind, us, ud, uw, per = G.updates(s, d, n, percent=5, batches=3, seed=8, max_weight=100)
for nb in (0, 1, 3):
    stream = gd.UpdateStream.from_arrays(kind[:nb*per], us[:nb*per], ud[:nb*per], uw[:nb*per])
    ref = gd.run_batches(gd.shipped_program("sssp"), gd.DynamicGraph.from_arrays(n, s, d, w, weighted=True, with_reverse=True), stream, per, {"src": 0})
    for world in (2,):
        comms = Communicator.local_group(world, group=100+nb)
        def fn(r):
            g = gd.DynamicGraph.from_arrays(n, s, d, w, weighted=True, with_reverse=True, comm=comms[r])
            ctx = gd.run_batches(gd.shipped_program("sssp"), g, stream, per, {"src": 0})
            return np.asarray(ctx.properties["dist"].data), np.asarray(ctx.properties["parent"].data)
        with ThreadPoolExecutor(world) as ex:
            res = list(ex.map(fn, range(world)))
        rd = np.asarray(ref.properties["dist"].data); rp = np.asarray(ref.properties["parent"].data)
        for r,(dd_, pp) in enumerate(res):
            bad = np.flatnonzero(dd_ != rd)
            print(f"batches={nb} world={world} rank={r}: dist mismatches {len(bad)} parent mismatches {np.count_nonzero(pp != rp)} first {bad[:5]} got {dd_[bad[:5]]} want {rd[bad[:5]]}", flush=True)
