"""Where the e2e step's time goes (C2): host-record batches with and without
the asynchronous rank read-back, and the raw H2D of one batch's records."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2507_11094_b200 as gd
from paper_2507_11094_b200 import _native as N

wl = bench.WORKLOADS["pr"]
n, s, d, w, kind, us, ud, uw, per = bench.make_inputs(wl, 40)
g = gd.DynamicGraph.from_arrays(n, s, d, with_reverse=True)
pr = gd.PRHandle(g, 0.85, 1e-3, 100)
pin = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for k, a in
       (("kind", kind), ("src", us), ("dst", ud), ("w", uw))}
out = torch.empty(n, dtype=torch.float64).pin_memory()
attrs = C.c_int()
print("pinned out ptr", hex(out.data_ptr()))


def batch(i):
    a = i * per
    N.check(N.lib().gd_pr_batch(pr.h, C.c_void_p(pin["kind"].data_ptr() + a), C.c_void_p(pin["src"].data_ptr() + 8 * a),
                                C.c_void_p(pin["dst"].data_ptr() + 8 * a), C.c_void_p(pin["w"].data_ptr() + 8 * a),
                                per, i))


i = 0
for mode in ("batch only", "batch + read_async", "batch + read_async + wait"):
    for _ in range(3):
        batch(i); i += 1
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = 8
    for _ in range(k):
        batch(i); i += 1
        if mode != "batch only":
            N.check(N.lib().gd_pr_read_async(pr.h, C.c_void_p(out.data_ptr())))
        if mode.endswith("wait"):
            N.check(N.lib().gd_wait(pr.h))
    N.check(N.lib().gd_wait(pr.h))
    print(f"{mode}: {1e3 * (time.perf_counter() - t) / k:.3f} ms/step")
# raw H2D of one batch's records
dev = torch.empty(per * 17, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    dev[: per * 8].copy_(pin["src"].view(torch.uint8)[: per * 8], non_blocking=True)
    dev[per * 8: per * 16].copy_(pin["dst"].view(torch.uint8)[: per * 8], non_blocking=True)
    dev[per * 16:].copy_(pin["kind"][:per], non_blocking=True)
torch.cuda.synchronize()
print(f"H2D of {per * 17 / 1e6:.1f} MB: {1e3 * (time.perf_counter() - t) / 10:.3f} ms")
t = time.perf_counter()
for _ in range(10):
    out.copy_(torch.empty(n, dtype=torch.float64, device="cuda"), non_blocking=True)
torch.cuda.synchronize()
print(f"D2H of {n * 8 / 1e6:.1f} MB: {1e3 * (time.perf_counter() - t) / 10:.3f} ms")
