"""Markdown table of the R-MAT-24 north-star sweep (tools/sweep_rmat24.sh):
    python tools/sweep_table.py gpurun_out/sweep > profiles/round2/sweep_rmat24.md"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
print("# R-MAT scale-24 sweep (north_star target), 1 B200, round 2\n")
print("`tools/sweep_rmat24.sh`: `bench.py --workload {pr,sssp,tc}-rmat24 --percent P --steps 5 --warmup 3 "
      "--e2e-steps 3 --no-cpu-baseline`. R-MAT-24 has 16,777,216 V and 2^28 = 268M edges; TC uses the undirected "
      "graph (536M arcs). Device = records resident in HBM; e2e = one `gd_*_run_stream32` call from pinned host "
      "memory, every batch's upload and result read-back inside the timed region. Batches differ (R-MAT hubs), so "
      "e2e (other batches) can differ from device.\n")
print("| Workload | batch | records / batch | ms / batch (device) | updated edges/s | e2e ms | dominant kernel "
      "(frac of HBM) | top kernels, ms |")
print("|---|---|---|---|---|---|---|---|")
for wl in ("pr-rmat24", "sssp-rmat24", "tc-rmat24"):
    for p in (1, 5, 10, 20):
        f = os.path.join(d, f"{wl}_p{p}.json")
        try:
            j = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:  # noqa: BLE001
            print(f"| {wl} | {p}% | - | (no result) | | | | |")
            continue
        k = j.get("kernels", {})
        s = j["steps"]
        top = ", ".join(f"{n} {v['ms_total'] / s:.2f}" for n, v in list(k.items())[:3])
        r = j.get("roofline") or {}
        frac = f"{r.get('kernel')} ({r['frac']:.2f})" if r.get("frac") else (r.get("kernel") or "")
        print(f"| {wl} | {p}% | {j['records_per_step']:,} | {j['ms_per_step']:.2f} | {j['value']:.2e} | "
              f"{j['e2e']['ms_per_step']:.2f} | {frac} | {top} |")
