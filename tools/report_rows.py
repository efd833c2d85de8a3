"""SURVEY §8(d).8 report rows: runs bench.py per config on this GPU and prints a markdown table
(config | GPUs | Mrays/s | fps | counted TFLOP/s | % FP32 peak | oracle Mrays/s 1 thread / N).
Usage: python tools/report_rows.py C2 C3 C4 C5 > profiles/r02_report_rows.md"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = []
for cfg in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    steps = {"C5": "5"}.get(cfg, "30")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", steps,
                          "--warmup", "3", "--cpu-seconds", "10"], capture_output=True, text=True, timeout=1200)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    r, cb, c = d["roofline"], d["cpu_baseline"], d["config"]
    counted = r.get("whole_frame_counted_tflops", r.get("achieved"))
    dom = r["kernel"].split(" ")[0]
    frac = f"{100 * r['frac']:.0f} % ({r['bound']}, {dom})"
    rows.append(f"| {cfg} | {c['width']}x{c['height']}, {c['spheres']} spheres + {c['planes']} planes, "
                f"{c['lights']} lights, depth {c['max_depth']}, {c['spp']} spp | 1 | {d['value']:.0f} | {d['fps']:.1f} | "
                f"{counted:.1f} | {frac} | {cb['value_1thread']:.2f} / {cb['value']:.1f} ({cb['cores']} cores) | "
                f"{d['e2e']['value']:.0f} |")
print("| config | workload | GPUs | Mrays/s | fps | whole-frame counted TFLOP/s | dominant kernel vs its roofline | oracle Mrays/s 1 thread / all cores | e2e Mrays/s |")
print("|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
