"""Summarise gpurun_out/ ncu artefacts into profiles/<round>/ (tracked).

  python tools/summarize_profiles.py round1 [--launches] [TAG=path.ncu-rep ...]
writes: launches_per_batch.md (--launches: per-kernel share of one PR batch
from the `gpu__time_duration` launch list), ncu_full_<TAG>.csv (dram bytes,
time, throughput per captured launch from `ncu --set full`), and merges the
per-launch DRAM traffic of the roofline kernels into profiles/ncu_traffic.json
(keyed workload/kernel, read by bench.py for roofline.traffic)."""
import collections, csv, json, os, subprocess, sys

rnd = sys.argv[1]
do_launches = "--launches" in sys.argv[2:]
reps = [a.split("=", 1) for a in sys.argv[2:] if "=" in a]
out = os.path.join("profiles", rnd)
os.makedirs(out, exist_ok=True)

# ---- launch list share
def launch_share():
  rows = list(csv.reader(open("gpurun_out/launches.csv")))
  hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
  hdr, data = rows[hi], rows[hi + 1:]
  ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
  seq = [(r[ki], float(r[vi].replace(",", ""))) for r in data]
  first = next(i for i, (k, _) in enumerate(seq) if "k_pr_onupdate" in k)
  nb = sum(1 for k, _ in seq if "k_pr_onupdate" in k)  # one OnDelete/OnAdd launch per batch
  tot, cnt = collections.defaultdict(float), collections.Counter()
  for k, v in seq[first:]:
      name = k.split("(")[0].replace("gdb::<unnamed>::", "").replace("void ", "")
      tot[name] += v
      cnt[name] += 1
  allt = sum(tot.values())
  with open(os.path.join(out, "launches_per_batch.md"), "w") as fh:
      fh.write(f"# Device time per PR batch (C2), from `ncu --metrics gpu__time_duration.sum` ({nb} batches, "
               f"cold-cache serialised launches: compare shares, not absolutes)\n\n")
      fh.write("| kernel | us / batch | launches / batch | share |\n|---|---|---|---|\n")
      for k, v in sorted(tot.items(), key=lambda x: -x[1]):
          fh.write(f"| `{k[:90]}` | {v / 1e3 / nb:.1f} | {cnt[k] / nb:.1f} | {100 * v / allt:.1f}% |\n")
      fh.write(f"| **total** | {allt / 1e3 / nb:.1f} | {sum(cnt.values()) / nb:.1f} | 100% |\n")

if do_launches:
    launch_share()

# ---- ncu --set full summary (TAG = the bench workload the capture ran)
traffic = collections.defaultdict(list)  # "workload/kernel" -> per-launch DRAM bytes
def full_summary(tag, rep):
  raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                       text=True).stdout.splitlines()
  r = list(csv.reader(raw))
  h, units, d = r[0], r[1], r[2:]
  want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
          "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
  idx = [h.index(x) for x in want if x in h]
  with open(os.path.join(out, f"ncu_full_{tag}.csv"), "w", newline="") as fh:
      w = csv.writer(fh)
      w.writerow([h[i] + (f" [{units[i]}]" if units[i] else "") for i in idx])
      for row in d:
          dur = float(row[h.index("gpu__time_duration.sum")]) * {"usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}.get(
              units[h.index("gpu__time_duration.sum")], 1)
          if dur < 10:  # a queued PR sweep that the device turned into a no-op
              continue
          w.writerow([row[i] for i in idx])
          name = row[h.index("Kernel Name")]
          scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
          rd = float(row[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
          wr = float(row[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
          key = ("pr_pull" if "k_pr_pull" in name else "merge_copy" if "k_edit_base" in name else
                 "del_scan_head" if "k_del_scan_head" in name else "del_scan_tail" if "k_del_scan_tail" in name else "pr_contrib" if "k_pr_contrib" in name else
                 "flood_sample" if "k_aff_sample" in name else "sssp_relax" if "k_fixpoint<0" in name else
               "sssp_walk" if "k_fixpoint<1" in name else "sssp_pull" if "k_fixpoint<2" in name else
               "tc_count" if ("k_tc_count" in name or "k_tc_merge" in name) else name)
          traffic[f"{tag}/{key}"].append(rd + wr)
tpath = os.path.join("profiles", "ncu_traffic.json")
merged = json.load(open(tpath)) if os.path.exists(tpath) else {}
for tag, rep in reps:
    full_summary(tag, rep)
merged.update({k: sum(v) / len(v) for k, v in traffic.items()})
json.dump(merged, open(tpath, "w"), indent=1)
print("wrote", out)
