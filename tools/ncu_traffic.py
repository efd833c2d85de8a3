#!/usr/bin/env python
"""DRAM bytes per launch of the wavefront kernels from an `ncu --set full` report of one C4 frame
(tools/profile_run.py), as the JSON entries bench.py reads for roofline.traffic
(profiles/ncu_render_kernel.json keys "<config>:<kernel class>"). The first launch of each class
(depth 0 of chunk 0; the secondary scan: the first depth-1 launch) is taken.
Usage: python tools/ncu_traffic.py REPORT.ncu-rep C4 [source-note] > entries.json"""
import csv
import io
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units, data = rows[0], rows[1], rows[2:]
idx = {n: i for i, n in enumerate(head)}
classes = [("camera", "wf_isect_eye2"), ("shade", "wf_shade"), ("shadow", "wf_isect_lt<"), ("accumulate", "wf_accumulate"),
           ("secondary", "wf_isect<1, 0>")]


def val(r, m):
    v = float(r[idx[m]].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1,
                                     "ns": 1e-6, "nsecond": 1e-6}.get(
        units[idx[m]], 1)


out = {}
for key, pat in classes:
    for r in data:
        if pat in r[idx["Kernel Name"]]:
            rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
            out[f"{cfg}:{key}"] = {"kernel": r[idx["Kernel Name"]].split("(")[0], "dram_bytes_per_launch": rd + wr,
                                   "dram_read_bytes": rd, "dram_write_bytes": wr,
                                   "duration_ms_ncu": val(r, "gpu__time_duration.sum"),
                                   "fma_pipe_active_pct": val(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                                   "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                   # active lanes per executed warp instruction / 32
                                   "warp_efficiency_pct": 100.0 / 32.0 * val(
                                       r, "smsp__thread_inst_executed_per_inst_executed.ratio"),
                                   "source": note}
            break
print(json.dumps(out, indent=1))
