#!/usr/bin/env python
"""Per-kernel registers / stack / spills from the nvcc -Xptxas -v log (paper_1504_03151_b200/build.log)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1504_03151_b200/build.log").read().splitlines()
cur = None
rows = {}
for ln in log:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        rows[cur].update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    r = rows[n]
    d = re.sub(r"\(.*", "", d)
    tmpl = re.search(r"<.*>", dem[names.index(n)])
    print(f"{r.get('regs', 0):4d} regs  stack {r.get('stack', 0):4d}  spill st/ld {r.get('st', 0):4d}/{r.get('ld', 0):4d}  "
          f"{d}{tmpl.group(0) if tmpl and '<' not in d else ''}")
