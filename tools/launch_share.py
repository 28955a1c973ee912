"""Per-batch device time by kernel from an `ncu --metrics gpu__time_duration.sum`
launch list of bench.py: batches are cut at the staging kernel (one per batch);
the first `skip` batches (warm-up) are dropped.
    python tools/launch_share.py gpurun_out/launches_tc.csv [skip] [nbatches]"""
import collections, csv, sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nb_take = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = [(r[ki], float(r[vi].replace(",", ""))) for r in data]
starts = [i for i, (k, _) in enumerate(seq) if "k_stage_" in k]
a, b = starts[skip], starts[min(skip + nb_take, len(starts) - 1)] if skip + nb_take < len(starts) else len(seq)
nb = min(nb_take, len(starts) - skip)
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in seq[a:b]:
    name = k.split("(")[0].replace("gdb::<unnamed>::", "").replace("void ", "").replace("gdb::", "")
    tot[name] += v
    cnt[name] += 1
allt = sum(tot.values())
unit = "ns" if max(v for _, v in seq) > 1e4 else "us"
scale = 1e3 if unit == "ns" else 1.0
print(f"| kernel | us / batch | launches / batch | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"| `{k[:90]}` | {v / scale / nb:.1f} | {cnt[k] / nb:.1f} | {100 * v / allt:.1f}% |")
print(f"| **total** ({nb} batches) | {allt / scale / nb:.1f} | {sum(cnt.values()) / nb:.1f} | 100% |")
