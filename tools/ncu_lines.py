#!/usr/bin/env python
"""Top source lines of one kernel in an ncu report by warp-stall samples (ncu --page source
--print-source cuda,sass). Usage: tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
total = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < 7:
        continue
    try:
        allsmp = int(r[4]) if r[4] not in ("-", "") else 0
        notiss = int(r[5]) if r[5] not in ("-", "") else 0
        inst = int(r[7]) if r[7] not in ("-", "") else 0
    except ValueError:
        continue
    total += allsmp
    rows.append((allsmp, notiss, inst, fname, int(r[0]), r[1].strip()[:110]))
rows.sort(reverse=True)
print(f"total stall samples {total}")
for a, b, i, f, ln, src in rows[:n]:
    print(f"{a:7d} {100.0 * a / max(total, 1):5.1f}%  notiss {b:6d}  inst {i:9d}  {f}:{ln}  {src}")
