"""Key `ncu --set full` metrics of every launch in a report, as markdown:
    python tools/ncu_summary.py gpurun_out/prof_pull_pr.ncu-rep > profiles/round2/x.md"""
import csv, io, subprocess, sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy", "Achieved Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
launches = {}
for r in rows[1:]:
    d = launches.setdefault(r[ii], {"kernel": r[ki].split("(")[0]})
    if r[mi] in KEEP and r[mi] not in d:
        d[r[mi]] = f"{r[vi]} {r[ui]}".strip()
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if rr:
    hh = rr[0]
    for r in rr[2:]:
        d = launches.get(r[hh.index("ID")])
        if d is not None:
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if m in hh:
                    d[m] = f"{r[hh.index(m)]} {rr[1][hh.index(m)]}"
cols = ["kernel"] + KEEP + ["dram__bytes_read.sum", "dram__bytes_write.sum"]
print("| " + " | ".join(cols) + " |")
print("|" + "---|" * len(cols))
for d in launches.values():
    print("| " + " | ".join(d.get(c, "") for c in cols) + " |")
