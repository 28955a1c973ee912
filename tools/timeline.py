"""GPU timeline of a few PR/SSSP/TC batches via torch.profiler (CUPTI sees the
kernels and memcpys our .so launches): busy vs idle per batch and the largest
gaps with the kernels around them.  python tools/timeline.py [pr|sssp|tc] [batches]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import bench

wlname = sys.argv[1] if len(sys.argv) > 1 else "pr"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = bench.WORKLOADS[wlname]
import paper_2507_11094_b200 as gd
n, s, d, w, kind, us, ud, uw, per = bench.make_inputs(wl, nb + 3)
g = gd.DynamicGraph.from_arrays(n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                                weighted=wl["weighted"], with_reverse=wl["algo"] != "tc")
algo = gd.PRHandle(g, 0.85, 1e-3, 100) if wl["algo"] == "pr" else (gd.SSSPHandle(g, 0) if wl["algo"] == "sssp" else gd.TCHandle(g))
dk = torch.from_numpy(kind).cuda(); ds = torch.from_numpy(us.astype(np.int32)).cuda()
dd = torch.from_numpy(ud.astype(np.int32)).cuda(); dw = torch.from_numpy(uw.astype(np.int32)).cuda()
def step(i):
    a, b = i * per, (i + 1) * per
    algo.batch_device(dk.data_ptr() + a, ds.data_ptr() + 4 * a, dd.data_ptr() + 4 * a, dw.data_ptr() + 4 * a, b - a, i)
for i in range(3):
    step(i)
torch.cuda.synchronize()
import time
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(3, 3 + nb):
        torch.cuda.synchronize()
        marks.append(time.perf_counter())
        step(i)
        torch.cuda.synchronize()
out = "gpurun_out/trace.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
# split into batches at gaps > 1 ms? use count: group by cuda sync boundaries: take the whole span
span0, span1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
busy = sum(e["dur"] for e in gpu)
print(f"{wlname}: {nb} batches, GPU span {(span1-span0)/1e3:.2f} ms, busy {busy/1e3:.2f} ms, events {len(gpu)}")
# per-batch: split at the largest nb-1 gaps (the host syncs between batches)
gaps = [(gpu[i+1]["ts"] - (gpu[i]["ts"] + gpu[i]["dur"]), i) for i in range(len(gpu)-1)]
cuts = sorted(i for _, i in sorted(gaps, reverse=True)[:nb-1])
bounds = [0] + [c + 1 for c in cuts] + [len(gpu)]
for b in range(nb):
    seg = gpu[bounds[b]:bounds[b+1]]
    t0, t1 = seg[0]["ts"], seg[-1]["ts"] + seg[-1]["dur"]
    bz = sum(e["dur"] for e in seg)
    print(f" batch {b}: span {(t1-t0)/1e3:.3f} ms busy {bz/1e3:.3f} ms idle {(t1-t0-bz)/1e3:.3f} ms launches {len(seg)}")
seg = gpu[bounds[nb-1]:bounds[nb]]
ig = sorted(((seg[i+1]["ts"] - (seg[i]["ts"] + seg[i]["dur"]), i) for i in range(len(seg)-1)), reverse=True)
print(" largest gaps in the last batch (us):")
for gp, i in ig[:25]:
    print(f"  {gp:8.1f}  after {seg[i]['name'][:60]:60s} before {seg[i+1]['name'][:50]}")
hist = {}
for e in seg:
    k = e["name"][:70]
    hist.setdefault(k, [0, 0.0]); hist[k][0] += 1; hist[k][1] += e["dur"]
print(" kernels in the last batch (us):")
for k, (c, t) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {t:8.1f} {c:3d}  {k}")
