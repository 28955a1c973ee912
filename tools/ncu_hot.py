"""Top SASS lines by stall samples for one kernel of an ncu report:
python tools/ncu_hot.py gpurun_out/prof.ncu-rep <kernel-regex> [top]"""
import csv, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si] or 0) for r in rows[1:] if len(r) > si and r[si].isdigit())
print("total samples", tot)
best = sorted((r for r in rows[1:] if len(r) > si and r[si].isdigit()), key=lambda r: -int(r[si]))[:top]
for r in best:
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols if (r[i] or "0").isdigit()), reverse=True)[:3]
    print(f"{int(r[si]):6d} {100*int(r[si])/max(tot,1):5.1f}%  {r[1].strip()[:60]:60s} {reasons}")
