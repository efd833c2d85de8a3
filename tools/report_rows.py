"""SURVEY §8(d).8 report rows: runs bench.py per config on this GPU and prints a markdown table
(config | GPUs | Mrays/s | fps | counted TFLOP/s | dominant kernel vs its roofline | ncu FMA pipe %
and warp efficiency of the dominant kernel (committed captures, profiles/ncu_render_kernel.json)
| oracle Mrays/s 1 thread / N | e2e | parity). --raw FILE keeps each config's bench JSON line.
Usage: python tools/report_rows.py [--raw FILE] C2 C3 C4 C5 > profiles/r02_report_rows.md"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# where each config's frame meets the oracle on the GPU (tests/test_gpu_parity.py)
PARITY = {
    "C1": "full frame, both variants (test_c1_full_frame)",
    "C2": "full frame, both variants (test_c2_full_frame)",
    "C3": "full size, sampled pixels (test_c3_full_size_sampled)",
    "C4": "full size, sampled pixels, both variants (test_c4_full_size_sampled); counts (test_c4_full_size_counts_consistent)",
    "C5": "full size, sampled pixels (test_c5_full_size_sampled)",
}
ap = argparse.ArgumentParser()
ap.add_argument("--raw", default=None)
ap.add_argument("configs", nargs="*", default=["C2", "C3", "C4", "C5"])
args = ap.parse_args()
rows = []
raw = open(args.raw, "w") if args.raw else None
for cfg in args.configs:
    steps = {"C5": "5"}.get(cfg, "30")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", steps,
                          "--warmup", "3", "--cpu-seconds", "10"], capture_output=True, text=True, timeout=1200)
    line = out.stdout.strip().splitlines()[-1]
    if raw:
        raw.write(line + "\n")
    d = json.loads(line)
    r, cb, c = d["roofline"], d["cpu_baseline"], d["config"]
    counted = r.get("whole_frame_counted_tflops", r.get("achieved"))
    dom = r["kernel"].split(" ")[0]
    frac = f"{100 * r['frac']:.0f} % ({r['bound']}, {dom})"
    ks = r.get("kernels") or {}
    ncu = "—"
    if ks:
        top = max(ks.values(), key=lambda v: v.get("share_of_frame", 0.0))
        n = top.get("ncu") or {}
        if n.get("fma_pipe_active_pct") is not None:
            we = n.get("warp_efficiency_pct")
            ncu = f"{n['fma_pipe_active_pct']:.0f} % / " + (f"{we:.1f} %" if we is not None else "—")
    rows.append(f"| {cfg} | {c['width']}x{c['height']}, {c['spheres']} spheres + {c['planes']} planes, "
                f"{c['lights']} lights, depth {c['max_depth']}, {c['spp']} spp | 1 | {d['value']:.0f} | {d['fps']:.1f} | "
                f"{counted:.1f} | {frac} | {ncu} | {cb['value_1thread']:.2f} / {cb['value']:.1f} ({cb['cores']} cores) | "
                f"{d['e2e']['value']:.0f} | {PARITY.get(cfg, '—')} |")
print("| config | workload | GPUs | Mrays/s | fps | whole-frame counted TFLOP/s | dominant kernel vs its roofline "
      "| ncu FMA pipe / warp efficiency (dominant kernel, committed capture) | oracle Mrays/s 1 thread / all cores "
      "| e2e Mrays/s | parity vs the oracle (GPU tests) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
