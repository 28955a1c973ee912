"""Per-batch SSSP diagnostics: fixpoint rounds and per-kernel time (GPU box)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2507_11094_b200 as gd
from paper_2507_11094_b200 import generate as G

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if which == "c1":
    s, d, w, n = G.rmat(16, 1_000_000, seed=22, weighted=True, max_weight=100)
else:
    side = int(which[4:]) if which.startswith("grid") and len(which) > 4 else 4899
    s, d, w, n = G.grid(side, side, seed=22)
kind, us, ud, uw, per = G.updates(s, d, n, percent=5, batches=nb, seed=23, max_weight=100)
g = gd.DynamicGraph.from_arrays(n, s, d, w, weighted=True, with_reverse=True)
t = time.time()
h = gd.SSSPHandle(g, 0)
torch.cuda.synchronize()
print(f"{which}: n={n} m={len(s)} static {time.time()-t:.3f}s rounds={h.iterations()}", flush=True)
dk = torch.from_numpy(kind).cuda()
ds = torch.from_numpy(us.astype(np.int32)).cuda()
dd = torch.from_numpy(ud.astype(np.int32)).cuda()
dw = torch.from_numpy(uw.astype(np.int32)).cuda()
h.set_profiling(True)
for i in range(nb):
    a, b = i * per, min((i + 1) * per, len(kind))
    it0 = h.iterations()
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.batch_device(dk.data_ptr() + a, ds.data_ptr() + 4 * a, dd.data_ptr() + 4 * a, dw.data_ptr() + 4 * a, b - a, i)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    ks = {k: h.kernel_time(k) for k in ("sssp_walk", "sssp_pull", "sssp_relax", "sssp_parent", "del_scan_head", "del_scan_tail", "merge_copy")}
    print(f"batch {i}: {el*1e3:.2f} ms rounds={h.iterations()-it0} phases={ {k: round(v, 3) for k, v in h.phase_ms().items()} }")
    print("   ", {k: round(v[0], 3) for k, v in ks.items() if v[1]})
