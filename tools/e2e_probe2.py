"""Where the C2 e2e time goes with gd_pr_run_stream: device-only batches,
run_stream without and with the per-batch rank read-back, and raw copies
(H2D, D2H, both at once, D2H concurrent with device batches)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2507_11094_b200 as gd

wl = bench.WORKLOADS["pr"]
K = 8
n, s, d, w, kind, us, ud, uw, per = bench.make_inputs(wl, 6 + 5 * K)
g = gd.DynamicGraph.from_arrays(n, s, d, with_reverse=True)
pr = gd.PRHandle(g, 0.85, 1e-3, 100)
pin = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for k, a in
       (("kind", kind), ("src", us), ("dst", ud), ("w", uw))}
out = torch.empty(n, dtype=torch.float64).pin_memory()
dk = torch.from_numpy(kind).cuda()
ds = torch.from_numpy(us.astype(np.int32)).cuda()
dd = torch.from_numpy(ud.astype(np.int32)).cuda()
dw = torch.from_numpy(uw.astype(np.int32)).cuda()
nxt = [0]


def dev_steps(k):
    for _ in range(k):
        i = nxt[0]
        a = i * per
        pr.batch_device(dk.data_ptr() + a, ds.data_ptr() + 4 * a, dd.data_ptr() + 4 * a, dw.data_ptr() + 4 * a, per, i)
        nxt[0] += 1


def stream_steps(k, with_out):
    i = nxt[0]
    a = i * per
    pr.run_stream_ptrs(pin["kind"].data_ptr() + a, pin["src"].data_ptr() + 8 * a, pin["dst"].data_ptr() + 8 * a,
                       0, k * per, per, i, *( [out.data_ptr()] if with_out else [0]))
    nxt[0] += k


def timed(label, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t) / K:.3f} ms/step", flush=True)


dev_steps(3)
stream_steps(1, True)
timed("device batches", lambda: dev_steps(K))
timed("run_stream, no read-back", lambda: stream_steps(K, False))
timed("run_stream, rank read-back", lambda: stream_steps(K, True))
side = torch.cuda.Stream()
big = torch.empty(n, dtype=torch.float64, device="cuda")


def dev_with_d2h():
    with torch.cuda.stream(side):
        for _ in range(K):
            out.copy_(big, non_blocking=True)
    dev_steps(K)


timed("device batches + K concurrent 33.5 MB D2H on a side stream", dev_with_d2h)
hbuf = pin["src"].view(torch.uint8)[: per * 17]
dbuf = torch.empty(per * 17, dtype=torch.uint8, device="cuda")
for label, fn in (("H2D 11.4 MB", lambda: dbuf.copy_(hbuf, non_blocking=True)),
                  ("D2H 33.5 MB", lambda: out.copy_(big, non_blocking=True))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t) / 10:.3f} ms", flush=True)
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s2):
        dbuf.copy_(hbuf, non_blocking=True)
    out.copy_(big, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D 11.4 MB and D2H 33.5 MB on two streams: {1e3 * (time.perf_counter() - t) / 10:.3f} ms", flush=True)
