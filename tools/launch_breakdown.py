"""Summarise an `ncu --csv --metrics gpu__time_duration.sum,...` launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.defaultdict(dict)
for r in data:
    per[(int(r[iID]), r[iK])][r[iM]] = float(r[iV].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, 0.0])
for (i, k), m in sorted(per.items()):
    name = k.split("(")[0][:60]
    a = agg[name]
    t = m.get("gpu__time_duration.sum", 0)
    a[0] += 1
    a[1] += t
    a[2] += t * m.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a[3] += t * m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)
    a[4] += t * m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0)
    a[5] += t * m.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:45s} n={a[0]:3d} time={a[1] / 1e6:8.3f} ms ({a[1] / tot:5.1%}) fma%={a[2] / max(a[1], 1):5.1f} "
          f"issue%={a[3] / max(a[1], 1):5.1f}" + (f" dram%={a[4] / max(a[1], 1):5.1f} fp64%={a[5] / max(a[1], 1):5.1f}"
                                                  if a[4] or a[5] else ""))
print("total", tot / 1e6, "ms")
