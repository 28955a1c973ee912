"""Where a batch's GPU idle time comes from: the device timeline of a few
batches (torch.profiler / CUPTI: our kernels, memsets, copies) next to the
host's CUDA runtime calls.  For every device gap the host call that was in
progress when the gap began is charged with it (a read-back's sync, a launch
the GPU waited for, an allocation ...).
    python tools/timeline_host.py [pr|sssp|tc] [batches]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_2507_11094_b200 as gd

wlname = sys.argv[1] if len(sys.argv) > 1 else "pr"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = dict(bench.WORKLOADS[wlname])
if len(sys.argv) > 3:
    wl["percent"] = float(sys.argv[3])
n, s, d, w, kind, us, ud, uw, per = bench.make_inputs(wl, nb + 3)
g = gd.DynamicGraph.from_arrays(n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                                weighted=wl["weighted"], with_reverse=wl["algo"] != "tc")
algo = (gd.PRHandle(g, 0.85, 1e-3, 100) if wl["algo"] == "pr" else
        (gd.SSSPHandle(g, 0) if wl["algo"] == "sssp" else gd.TCHandle(g)))
dk = torch.from_numpy(kind).cuda()
ds = torch.from_numpy(us.astype(np.int32)).cuda()
dd = torch.from_numpy(ud.astype(np.int32)).cuda()
dw = torch.from_numpy(uw.astype(np.int32)).cuda()


def step(i):
    a, b = i * per, (i + 1) * per
    algo.batch_device(dk.data_ptr() + a, ds.data_ptr() + 4 * a, dd.data_ptr() + 4 * a, dw.data_ptr() + 4 * a,
                      b - a, i)


for i in range(3):
    step(i)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(3, 3 + nb):
        step(i)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
out = f"gpurun_out/trace_host_{wlname}.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
dev = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
             key=lambda e: e["ts"])
host = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cuda_runtime", "cuda_driver")),
              key=lambda e: e["ts"])
span = dev[-1]["ts"] + dev[-1]["dur"] - dev[0]["ts"]
busy = sum(e["dur"] for e in dev)
print(f"{wlname}: {nb} batches, device span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, "
      f"idle {(span - busy) / 1e3:.3f} ms, {len(dev)} device ops, {len(host)} host API calls")
print(f"per batch: span {span / nb / 1e3:.3f} ms busy {busy / nb / 1e3:.3f} ms ops {len(dev) / nb:.0f}")
api = collections.Counter(e["name"] for e in host)
apit = collections.defaultdict(float)
for e in host:
    apit[e["name"]] += e["dur"]
print("host API calls per batch (count, total us):")
for k, c in api.most_common(20):
    print(f"  {c / nb:7.1f} {apit[k] / nb:9.1f}  {k}")
# charge every device gap to the host call in progress when it began
charge = collections.defaultdict(float)
ncharge = collections.Counter()
hi = 0
for a, b in zip(dev, dev[1:]):
    g0 = a["ts"] + a["dur"]
    gap = b["ts"] - g0
    if gap <= 0:
        continue
    while hi < len(host) and host[hi]["ts"] + host[hi]["dur"] < g0:
        hi += 1
    cur = "none"
    for h in host[hi:hi + 50]:
        if h["ts"] <= g0 <= h["ts"] + h["dur"]:
            cur = h["name"]
            break
        if h["ts"] > g0:
            cur = "host gap before " + h["name"]
            break
    key = f"{cur} | before {b['name'][:40]}"
    charge[key] += gap
    ncharge[key] += 1
tot = sum(charge.values())
kern = collections.defaultdict(float)
for e in dev:
    kern[e["name"][:80]] += e["dur"]
print("device time per batch by kernel (us):")
for k_, v in sorted(kern.items(), key=lambda kv: -kv[1])[:25]:
    print(f"  {v / nb:10.1f}  {k_}")
print(f"device idle {tot / nb:.1f} us per batch, by the host call in progress:")
for k, v in sorted(charge.items(), key=lambda kv: -kv[1])[:30]:
    print(f"  {v / nb:8.1f} us {ncharge[k] / nb:5.1f}x  {k}")
