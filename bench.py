#!/usr/bin/env python
"""Benchmark of the B200 dynamic-graph hot path (BASELINE.json).

Default workload = BASELINE configs[1] (the metric's 1-GPU config): dynamic
PageRank on R-MAT scale-22 (4,194,304 V, 2^26 distinct directed edges,
unweighted), successive 1% ΔG batches (671,089 records: 50% deletes drawn
from the edges, 50% adds from non-edges), d=0.85, beta=1e-3, maxiter=100,
merge every batch (the reference default).  One step = one batch: OnDelete/
OnAdd handlers, updateCSRDel/Add on the GPU diff-CSR store, merge, affected
flood, incremental PageRank to convergence.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload pr|sssp|tc|sssp-grid]

Under torchrun (N>1): PR and TC run ONE job over all GPUs -- every rank
holds a replica of the store and applies every batch, PR pulls only its
destination range and all-gathers the rank vector over NCCL each sweep, TC
counts a 1/N slice of the records and all-reduces (strong scaling); SSSP
runs independent replicas (weak scaling).  Timing is the max over ranks.  `--impl reference` times the reference's own emitted OpenMP
driver (oracle/_ref/libgdref.so, compiled from /root/reference) on the host
cores -- rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "per-ΔG-batch time & updated edges/sec for dyn SSSP/PR/TC at 1/2/4/8 B200"
UNIT = "updated edges/s"

WORKLOADS = {
    # BASELINE configs[1]
    "pr": dict(algo="pr", graph="rmat", scale=22, edges=1 << 26, percent=1.0, weighted=False, directed=True,
               desc="dynamic PageRank, R-MAT scale-22 (4,194,304 V, 67,108,864 E), successive 1% batches"),
    # BASELINE configs[0] (the reference's CPU-runnable case)
    "sssp": dict(algo="sssp", graph="rmat", scale=16, edges=1_000_000, percent=5.0, weighted=True, directed=True,
                 desc="dynamic SSSP, R-MAT scale-16 (65,536 V, 1M E, w 1-100), 5% batches"),
    # BASELINE configs[2] at 1%
    # (the reference's emitted TC runs single-threaded -- it crashes with more,
    # so its arm times a 1M-vertex sample of the recipe)
    "tc": dict(algo="tc", graph="uniform", nodes=1 << 24, edges=256_000_000, percent=1.0, weighted=False,
               directed=False, desc="dynamic TC, uniform 16,777,216 V / 256M undirected edges, 1% batches",
               ref_sample=dict(nodes=1 << 20, edges=1 << 24,
                               desc="dynamic TC, uniform 1,048,576 V / 16.8M undirected edges sample, 1% batches")),
    # BASELINE configs[3]
    # north_star target: R-MAT scale-24 (16.8M V, 2^28 edges), 1-20% batches
    "pr-rmat24": dict(algo="pr", graph="rmat", scale=24, edges=1 << 28, percent=1.0, weighted=False, directed=True,
                      desc="dynamic PageRank, R-MAT scale-24 (16,777,216 V, 268,435,456 E), 1% batches",
                      ref_sample=dict(scale=22, edges=1 << 26,
                                      desc="dynamic PageRank, R-MAT scale-22 sample (4.2M V, 67M E), 1% batches")),
    "sssp-rmat24": dict(algo="sssp", graph="rmat", scale=24, edges=1 << 28, percent=1.0, weighted=True,
                        directed=True,
                        desc="dynamic SSSP, R-MAT scale-24 (16,777,216 V, 268,435,456 E, w 1-100), 1% batches",
                        ref_sample=dict(scale=22, edges=1 << 26,
                                        desc="dynamic SSSP, R-MAT scale-22 sample (4.2M V, 67M E), 1% batches")),
    "tc-rmat24": dict(algo="tc", graph="rmat", scale=24, edges=1 << 28, percent=1.0, weighted=False,
                      directed=False,
                      desc="dynamic TC, undirected R-MAT scale-24 (16,777,216 V, 268,435,456 edges), 1% batches",
                      ref_sample=dict(scale=16, edges=1 << 20,
                                      desc="dynamic TC, undirected R-MAT scale-16 sample (65K V, 1M edges), 1% batches")),
    # BASELINE configs[4] (C5) on one GPU: R-MAT scale-26, 2^30 edges.  The
    # reference arm cannot run it in bounded time (its per-batch cost grows
    # with E and the store alone needs ~50 GB of host RAM), so it times the
    # scale-22 sample of the same recipe; its per-record rate overstates the
    # full-size reference.
    "pr-c5": dict(algo="pr", graph="rmat", scale=26, edges=1 << 30, percent=1.0, weighted=False, directed=True,
                  desc="dynamic PageRank, R-MAT scale-26 (67,108,864 V, 1,073,741,824 E), 1% batches",
                  ref_sample=dict(scale=22, edges=1 << 26,
                                  desc="dynamic PageRank, R-MAT scale-22 sample (4.2M V, 67M E), 1% batches")),
    "sssp-c5": dict(algo="sssp", graph="rmat", scale=26, edges=1 << 30, percent=1.0, weighted=True, directed=True,
                    desc="dynamic SSSP, R-MAT scale-26 (67,108,864 V, 1,073,741,824 E, w 1-100), 1% batches",
                    ref_sample=dict(scale=22, edges=1 << 26,
                                    desc="dynamic SSSP, R-MAT scale-22 sample (4.2M V, 67M E), 1% batches")),
    "tc-c5": dict(algo="tc", graph="rmat", scale=26, edges=1 << 30, percent=1.0, weighted=False, directed=False,
                  desc="dynamic TC, undirected R-MAT scale-26 (67,108,864 V, 1,073,741,824 edges), 1% batches",
                  ref_sample=dict(scale=16, edges=1 << 20,
                                  desc="dynamic TC, undirected R-MAT scale-16 sample (65K V, 1M edges), 1% batches")),
    # The reference's fixedPoint sweeps all V per round and needs ~rows+cols
    # rounds, so its CPU time grows ~side^3: its arm runs a 600x600 sample
    # of the same family (per-record rate overstates the full-size reference).
    "sssp-grid": dict(algo="sssp", graph="grid", rows=4899, cols=4899, percent=5.0, weighted=True, directed=True,
                      desc="dynamic SSSP, 4899x4899 grid (24.0M V, 96M arcs), 5% batches, corner source",
                      ref_sample=dict(rows=600, cols=600,
                                      desc="dynamic SSSP, 600x600 grid sample (360K V, 1.44M arcs), 5% batches")),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


GEN = "fast"  # --gen: "fast" (parallel counter-based RNG) or "python" (the reference's own recipes and seeds)


def make_inputs(wl, batches, seed=22):
    from paper_2507_11094_b200 import generate as G

    t = time.time()
    if GEN == "python" and wl["graph"] in ("rmat", "uniform"):
        # generate.py's rmat_graph / uniform_random_graph / generate_updates,
        # draw for draw (seed-compatible); one stream of batches x percent,
        # cut into batches of ceil(percent% of m) as the reference's bench does
        und = not wl["directed"]
        mw = 100 if wl["weighted"] else 10
        if wl["graph"] == "rmat":
            s, d, w, n = G.py_rmat_graph(wl["scale"], wl["edges"], seed=seed, weighted=wl["weighted"], max_weight=mw,
                                         undirected=und)
        else:
            n = wl["nodes"]
            s, d, w = G.py_uniform_random_graph(n, wl["edges"], seed=seed, weighted=wl["weighted"], max_weight=mw,
                                                undirected=und)
        per = math.ceil(wl["percent"] / 100.0 * len(s))
        kind, us, ud, uw = G.py_generate_updates(s, d, w, n, min(100.0, wl["percent"] * batches), seed=seed + 1,
                                                 undirected=und)
        log(f"[bench] inputs (reference generators, seed {seed}): n={n} m={len(s)} records={len(kind)} batch={per} "
            f"gen={time.time() - t:.1f}s")
        return n, s, d, w, kind, us, ud, uw, per
    if wl["graph"] == "rmat":
        s, d, w, n = G.rmat(wl["scale"], wl["edges"], seed=seed, weighted=wl["weighted"],
                            undirected=not wl["directed"])
    elif wl["graph"] == "uniform":
        s, d, w, n = G.uniform(wl["nodes"], wl["edges"], seed=seed, weighted=wl["weighted"],
                               undirected=not wl["directed"])
    else:
        s, d, w, n = G.grid(wl["rows"], wl["cols"], seed=seed)
    kind, us, ud, uw, per = G.updates(s, d, n, percent=wl["percent"], batches=batches, seed=seed + 1,
                                      undirected=not wl["directed"], max_weight=100 if wl["weighted"] else 1)
    log(f"[bench] inputs: n={n} m={len(s)} records={len(kind)} batch={per} gen={time.time() - t:.1f}s "
        f"({G.threads()} threads)")
    return n, s, d, w, kind, us, ud, uw, per


class Clocks:
    """nvidia-smi sampling around the timed region (B200_PROFILING.md clocks
    line); samples are time-stamped and filtered to the timed window."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None
        self.window = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let the sampler come up before the timed region
        except OSError:
            self.p = None

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        import datetime

        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        t0, t1 = self.window or (0, float("inf"))
        inside = [r for r in rows if t0 - 0.02 <= r[0] <= t1 + 0.02]
        note = None
        if not inside:  # region shorter than the sampling period: nearest samples
            inside = sorted(rows, key=lambda r: abs(r[0] - (t0 + t1) / 2))[:3]
            note = "timed region shorter than the sampling period; nearest samples"
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in inside:
            for nm, v in zip(names, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        d = {"sm_mhz": statistics.median([r[1] for r in inside]) if inside else None,
             "sm_max_mhz": inside[0][2] if inside else None, "reasons": sorted(reasons), "samples": len(inside)}
        if note:
            d["note"] = note
        return d


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ reference ----

def reference_run(wl, batches, threads):
    """The reference's own dynamicPR/SSSP/TC (oracle/_ref) on the host cores,
    over `batches` successive batches.  Per-batch time = (T_k - T_0)/k as the
    reference's bench does (cli.py:436-442)."""
    from oracle import oracle as O

    k = max(1, int(batches))
    if "ref_sample" in wl:
        wl = {**wl, **wl["ref_sample"]}
    n, s, d, w, kind, us, ud, uw, per = make_inputs(wl, k)
    total = min(len(kind), k * per)
    t = time.time()
    algo = wl["algo"]
    _, times = O.ref_run(algo, n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                         weighted=wl["weighted"], kind=kind[:total], us=us[:total], ud=ud[:total], uw=uw[:total],
                         batch_size=per, threads=threads, sssp_src=0)
    per_batch = (times[1] - times[0]) / k
    if per_batch <= 0:  # the static run's own jitter exceeded the batches' cost: time twice as many once more
        k *= 2
        n, s, d, w, kind, us, ud, uw, per = make_inputs(wl, k)
        total = min(len(kind), k * per)
        _, times = O.ref_run(algo, n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                             weighted=wl["weighted"], kind=kind[:total], us=us[:total], ud=ud[:total],
                             uw=uw[:total], batch_size=per, threads=threads, sssp_src=0)
        per_batch = (times[1] - times[0]) / k
    if per_batch <= 0:
        raise RuntimeError(f"T_k - T_0 <= 0 over {k} batches (T0={times[0]:.2f}s, Tk={times[1]:.2f}s): "
                           "the batches cost less than the static run's jitter")
    used = 1 if algo == "tc" else threads
    log(f"[reference] T0={times[0]:.2f}s Tk={times[1]:.2f}s k={k} per-batch={per_batch:.3f}s wall={time.time()-t:.1f}s")
    return {"value": per / per_batch, "unit": UNIT, "cores": used, "kind": "reference",
            "per_batch_s": per_batch, "batches": k, "T0_s": float(times[0]), "Tk_s": float(times[1]),
            "sample": (f"{wl['desc']}: the reference's emitted OpenMP driver "
                       f"({algo}_dynamic_omp.cc + graphdyn_rt.h, g++ -O2 -fopenmp) on {k} successive batches of "
                       f"{per} records, (T_k - T_0)/k per batch (cli.py:436-442); "
                       f"{used} OpenMP thread(s){' (emitted TC crashes with >1 thread)' if algo == 'tc' else ''}")}


# ------------------------------------------------------------------------ ours ----

EXTRAS = ("tc", "sssp-grid")  # BASELINE configs[2] and configs[3], timed in the same default run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="pr")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="time only --workload (by default the PR headline also times TC configs[2] and SSSP "
                         "configs[3] in the same run, under the 'extras' key)")
    ap.add_argument("--extra-steps", type=int, default=6, help="timed steps of each extra workload")
    ap.add_argument("--percent", type=float, default=None, help="override the workload's batch percentage")
    ap.add_argument("--force-dist", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--static", action="store_true",
                    help="also time the static alternative per batch: apply the batch, merge, recompute from scratch "
                         "(staticSSSP / staticPR / staticTC), on up to 3 batches")
    ap.add_argument("--gen", choices=("fast", "python"), default="fast",
                    help="input generator: fast (parallel) or python (the reference's generate.py, seed-compatible)")
    ap.add_argument("--ref-batches", type=int, default=3,
                    help="bounded sample for the reference arm: this many successive batches (>= 1)")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.percent is not None:
        wl["percent"] = args.percent
        wl["desc"] = wl["desc"].rsplit(",", 1)[0] + f", {args.percent:g}% batches"
    global GEN
    GEN = args.gen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = os.cpu_count() or 1
        try:
            cb = reference_run(wl, args.ref_batches, threads)
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"impl": "reference", "unavailable": f"{type(exc).__name__}: {exc}"}))
            return 0
        # steps = the batches actually timed (T_k - T_0 over k successive batches)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": cb["batches"], "warmup": 0, "ms_per_step": cb["per_batch_s"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype(wl),
                "data": "synthetic", "config": _config(wl, args, world),
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "reference_timing": {"T0_s": cb["T0_s"], "Tk_s": cb["Tk_s"], "batches": cb["batches"],
                                     "requested_steps": args.steps}}
        print(json.dumps(line))
        return 0

    import torch

    # --force-dist: take the N>1 code path (process group, NCCL communicator,
    # sharded PR / TC) at world size 1, to exercise it on a single GPU
    dist_on = world > 1 or args.force_dist
    torch.cuda.set_device(local)
    if dist_on:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2507_11094_b200 as gd

    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 10))
    res = run_ours(gd, torch, wl, args, args.steps, args.warmup, e2e_steps, world, rank, local, dist_on,
                   static=args.static)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(wl, args.ref_batches)

    extras = None
    if world == 1 and not dist_on and not args.no_extras and args.workload == "pr" and args.percent is None:
        extras = {}
        for name in EXTRAS:
            xwl = dict(WORKLOADS[name])
            try:
                xr = run_ours(gd, torch, xwl, args, args.extra_steps, max(3, min(args.warmup, 3)),
                              max(1, min(args.extra_steps, 4)), world, rank, local, dist_on, static=False)
                xr["config"] = _config(xwl, args, world)
                xr["dtype"] = _dtype(xwl)
                if not args.no_cpu_baseline:
                    xr["cpu_baseline"] = _cpu_baseline(xwl, 3 if xwl["algo"] == "tc" else 1)
                extras[name] = xr
            except Exception as exc:  # noqa: BLE001
                extras[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": res["scaling"], "vs_baseline": None, "dtype": _dtype(wl),
            "data": "synthetic", "config": _config(wl, args, world),
            "e2e": res["e2e"],
            "gpu_launches": res["gpu_launches"],
            "roofline": res["roofline"],
            "kernels": res["kernels"],
            "cpu_baseline": cpu,
            "clocks": res["clocks"],
            "records_per_step": res["records_per_step"],
        }
        if res.get("comm") is not None:
            line["comm"] = res["comm"]
        if res.get("static") is not None:
            line["static"] = res["static"]
        if extras is not None:
            line["extras"] = extras
        print(json.dumps(line))
    if dist_on:
        torch.distributed.destroy_process_group()
    return 0


def _cpu_baseline(wl, batches):
    try:
        cb = reference_run(wl, batches, os.cpu_count() or 1)
        return {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": f"unavailable: {type(exc).__name__}: {exc}"}


def run_ours(gd, torch, wl, args, steps, warmup, e2e_steps, world, rank, local, dist_on, static=False):
    """One workload on the device path: W warm-up steps, K timed steps with
    inputs resident in HBM (CUDA events on the store's stream, max over
    ranks), then e2e steps through the host-buffer C-ABI call."""
    nb = warmup + steps + 1 + e2e_steps  # +1: the untimed e2e warm-up step
    # N > 1 runs ONE job: every rank builds the same graph and stream.  PR and
    # SSSP partition the store by 1D vertex blocks (each rank keeps the arcs
    # of its sources and the in-arcs of its destinations); TC keeps a replica
    # of the undirected graph per rank and counts a slice of the records.
    n, s, d, w, kind, us, ud, uw, per = make_inputs(wl, nb, seed=22)
    records_per_step = per
    comm = None
    if dist_on:
        from paper_2507_11094_b200.dist import Communicator

        comm = Communicator.from_torch_distributed(local)
    partitioned = comm is not None and wl["algo"] in ("pr", "sssp") and wl["directed"]

    t = time.time()
    g = gd.DynamicGraph.from_arrays(n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                                    weighted=wl["weighted"], with_reverse=wl["algo"] != "tc", device=local,
                                    comm=comm if partitioned else None)
    if wl["algo"] == "pr":
        algo = gd.PRHandle(g, 0.85, 1e-3, 100)
    elif wl["algo"] == "sssp":
        algo = gd.SSSPHandle(g, 0)
    else:
        algo = gd.TCHandle(g)
    torch.cuda.synchronize()
    log(f"[bench] {wl['algo']}: store + static pass: {time.time() - t:.1f}s; "
        f"device bytes {g.device_bytes() / 2**30:.2f} GiB")
    sharded = dist_on
    if comm is not None and not partitioned and wl["algo"] in ("pr", "tc"):
        comm.attach(algo)  # replicated store: TC record slices / PR destination ranges

    # records resident in HBM for the device-path steps (int32 ids, uint8 kind)
    dk = torch.from_numpy(kind).to(f"cuda:{local}")
    ds = torch.from_numpy(us.astype(np.int32)).to(f"cuda:{local}")
    dd = torch.from_numpy(ud.astype(np.int32)).to(f"cuda:{local}")
    dw = torch.from_numpy(uw.astype(np.int32)).to(f"cuda:{local}")

    def dev_step(i):
        a, b = i * per, min((i + 1) * per, len(kind))
        algo.batch_device(dk.data_ptr() + a, ds.data_ptr() + 4 * a, dd.data_ptr() + 4 * a, dw.data_ptr() + 4 * a,
                          b - a, i)
        return b - a

    stream = torch.cuda.ExternalStream(_graph_stream(g))
    for i in range(warmup):
        dev_step(i)
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs already in HBM --------------------------------
    algo.set_profiling(os.environ.get("GD_BENCH_NOPROF") is None)
    kstats = {}
    clocks = Clocks(local)
    clocks.start()
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    wall0 = time.time()
    if sharded:
        comm.reset_stats()
    launches0 = gd._native.lib().gd_kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    done = 0
    for i in range(warmup, warmup + steps):
        done += dev_step(i)
    ev1.record(stream)
    torch.cuda.synchronize()
    for name in KERNELS:  # summed over the timed steps by the library
        ms, nl, nb_ = algo.kernel_time(name, total=True)
        if nl:
            kstats[name] = [ms, nl, nb_]
    launches = gd._native.lib().gd_kernel_launches() - launches0
    comm_stats = None
    if sharded:  # CommStats analogue: NCCL traffic of this rank per timed step
        cs = comm.stats()
        comm_stats = {k: v / steps for k, v in cs.items()}
        comm_stats["per"] = "rank and step"
    clocks.mark(wall0, time.time())
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    if dist_on:
        tt = torch.tensor([elapsed_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    algo.set_profiling(False)

    # ---- e2e: host buffers through the public C-ABI call, H2D + D2H inside ----------
    # records as uint8 kinds and int32 ids in pinned memory (gd_*_run_stream32):
    # ids of the B200 layout are < 2^31, and 4-byte ids halve the upload
    pin = {}
    for nm, arr in (("kind", kind), ("src", us.astype(np.int32)), ("dst", ud.astype(np.int32)),
                    ("w", uw.astype(np.int32))):
        t_ = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory()
        pin[nm] = t_
    out_pin = torch.empty((2, n) if wl["algo"] == "sssp" else n,
                          dtype=torch.float64 if wl["algo"] == "pr" else torch.int64).pin_memory()
    # one untimed batch through the same call first (creates the copy stream,
    # its events and the upload slots)
    wi = warmup + steps
    wa, wb = wi * per, min((wi + 1) * per, len(kind))
    if wb > wa:
        _host_stream(algo, wl, pin, wa, wb - wa, per, wi, out_pin)
    # ---- e2e timed region: ONE run_batches call over the e2e steps' records
    # from pinned host memory (gd_*_run_stream): every batch's records go up
    # and every batch's result comes back to host memory inside the region
    e_start = warmup + steps + 1
    a0, b0 = e_start * per, min((e_start + e2e_steps) * per, len(kind))
    e_done = max(b0 - a0, 0)
    nsteps_e = (e_done + per - 1) // per
    h2d = e_done * (1 + 4 + 4 + (4 if (wl["weighted"] or wl["algo"] == "sssp") else 0))  # w not uploaded when unused
    d2h = nsteps_e * {"pr": 8 * n, "sssp": 16 * n, "tc": 8}[wl["algo"]]
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tb0 = time.perf_counter()
    if e_done:
        _host_stream(algo, wl, pin, a0, e_done, per, e_start, out_pin)
    tcall = time.perf_counter() - tb0
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    log(f"[bench] e2e: run_stream over {nsteps_e} batches: {1e3 * tcall:.2f} ms host call, "
        f"{e2e_ms:.2f} ms device events")
    if dist_on:
        tt = torch.tensor([e2e_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = e_done / (e2e_ms / 1e3) if e2e_ms > 0 else None  # one job over all ranks

    stat = _static_compare(gd, torch, wl, args, local, n, s, d, w, kind, us, ud, uw, per) if static else None

    shards = dist_on  # one job over all GPUs
    value = done / (elapsed_ms / 1e3)
    peak, peak_kind = load_peaks()
    dom = max(kstats.items(), key=lambda kv: kv[1][0]) if kstats else None
    roof = None
    if dom:
        name, (ms, nl, nbytes) = dom
        b_per_launch = nbytes / nl
        avg_ms = ms / nl
        ach = (b_per_launch / 1e9) / (avg_ms / 1e3) if b_per_launch else None
        roof = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": _ncu_traffic(wl, name),
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else
                "fallback 6.65 TB/s (B200_PROFILING.md)",
                "bytes_per_launch": b_per_launch, "avg_launch_ms": avg_ms, "launches": nl,
                "share_of_step": ms / elapsed_ms if elapsed_ms else None}
    out = {"value": value, "ms_per_step": elapsed_ms / steps, "steps": steps, "warmup": warmup,
           "scaling": "strong" if shards else "weak",
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // max(nsteps_e, 1),
                   "d2h_bytes_per_step": d2h // max(nsteps_e, 1), "steps": nsteps_e,
                   "ms_per_step": e2e_ms / max(nsteps_e, 1), "api": f"gd_{wl['algo']}_run_stream32"},
           "gpu_launches": int(launches), "roofline": roof,
           "kernels": {k_: {"ms_total": v[0], "launches": v[1], "share": v[0] / elapsed_ms,
                            "gbs": (v[2] / 1e9) / (v[0] / 1e3) if v[2] and v[0] else None}
                       for k_, v in sorted(kstats.items(), key=lambda kv: -kv[1][0])},
           "clocks": clk, "records_per_step": records_per_step, "comm": comm_stats}
    if stat is not None:
        stat["dynamic_speedup"] = stat["ms_per_step"] / (elapsed_ms / steps)
        out["static"] = stat
    del algo, g
    return out


def _static_compare(gd, torch, wl, args, local, n, s, d, w, kind, us, ud, uw, per):
    """The static alternative the reference's `bench` compares against
    (cli.py:396-491): per batch, apply it to the store, merge, and run the
    static entry from scratch.  Same batches as the dynamic timed steps."""
    from paper_2507_11094_b200.updates import RecordArrays, UpdateBatch

    g2 = gd.DynamicGraph.from_arrays(n, s, d, w if wl["weighted"] else None, directed=wl["directed"],
                                     weighted=wl["weighted"], with_reverse=wl["algo"] != "tc", device=local)
    stream = torch.cuda.ExternalStream(_graph_stream(g2))
    k = min(args.steps, 3)
    times = []
    for i in range(args.warmup, args.warmup + k):
        a, b = i * per, min((i + 1) * per, len(kind))
        part = RecordArrays(kind[a:b], us[a:b], ud[a:b], uw[a:b])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        batch = UpdateBatch(arrays=part)
        g2.update_csr_del(batch.only_deletes())
        g2.update_csr_add(batch.only_adds())
        g2.merge_deltas()
        if wl["algo"] == "pr":
            h = gd.PRHandle(g2, 0.85, 1e-3, 100)
        elif wl["algo"] == "sssp":
            h = gd.SSSPHandle(g2, 0)
        else:
            h = gd.TCHandle(g2)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        del h
    ms = sum(times) / len(times)
    return {"ms_per_step": ms, "value": per / (ms / 1e3), "unit": UNIT, "steps": k,
            "what": "apply batch + merge + static recompute from scratch (the reference bench's static column)"}


KERNELS = ("pr_pull", "pr_contrib", "tc_bitmap", "merge_copy", "flood_sample", "flood_rest", "flood_mark", "flood_link", "del_scan_head", "del_scan_tail",
           "add_vacancies", "index_claim", "index_ins_pos", "tc_count", "sssp_relax", "sssp_walk", "sssp_pull",
           "sssp_parent")

def _graph_stream(g):
    import ctypes as C

    from paper_2507_11094_b200 import _native as N

    p = C.c_void_p()
    N.check(N.lib().gd_graph_stream(g.handle, C.byref(p)))
    return p.value


def _host_stream(algo, wl, pin, a, k, per, first, out_pin):
    """run_batches over host records [a, a+k) in batches of `per` through the
    public C-ABI call (gd_*_run_stream), every batch's result read back to
    pinned host memory (PR ranks, SSSP dist + parent, TC counts)."""
    if wl["algo"] == "pr":
        outs = (out_pin.data_ptr(),)
    elif wl["algo"] == "sssp":
        outs = (out_pin[0].data_ptr(), out_pin[1].data_ptr())
    else:
        counts = np.zeros((k + per - 1) // per, dtype=np.int64)
        outs = (counts.ctypes.data,)
    algo.run_stream_ptrs(pin["kind"].data_ptr() + a, pin["src"].data_ptr() + 4 * a, pin["dst"].data_ptr() + 4 * a,
                         pin["w"].data_ptr() + 4 * a, k, per, first, *outs, ids32=True)


def _ncu_traffic(wl, name):
    """Per-launch DRAM bytes of `name` from the committed `ncu --set full`
    capture of this workload (tools/summarize_profiles.py), else None."""
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    key = next((k for k, v in WORKLOADS.items() if v["desc"] == wl["desc"]), None)
    try:
        with open(p) as fh:
            t = json.load(fh)
        return t.get(f"{key}/{name}")
    except Exception:
        return None


def _dtype(wl):
    return {"pr": "f64", "sssp": "int64", "tc": "int64"}[wl["algo"]]


def _config(wl, args, world):
    c = {"workload": wl["desc"], "algo": wl["algo"], "batch_percent": wl["percent"], "merge_interval": 1,
         "parallelism": ("single-gpu" if world == 1 else
                         "1D vertex blocks: partitioned store, owner-routed arcs; PR contrib all-gather + BFS flood "
                         "reduce-scatter per level" if wl["algo"] == "pr" else
                         "1D vertex blocks: partitioned store, owner-routed arcs; SSSP supersteps with owner "
                         "message exchange" if wl["algo"] == "sssp" else
                         "replicated undirected store, TC record slices + NCCL all-reduce"),
         "l2": "inputs larger than L2 (graph store >> 126 MB L2)",
         "generator": ("reference generate.py recipes, seed-compatible" if GEN == "python" and wl["graph"] != "grid"
                       else "parallel counter-based RNG, reference recipes")}
    if wl["algo"] == "pr":
        c.update({"damping": 0.85, "beta": 1e-3, "maxiter": 100})
    return c


if __name__ == "__main__":
    sys.exit(main())
