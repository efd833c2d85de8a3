"""Per-rank work of an N-GPU frame measured on one GPU: every rank's shard of a config for world =
1, 2, 4, 8 (rt_render_shard), each rank rendered repeatedly as its own process would (the first
renders launch stream by stream, later ones replay the captured CUDA graph), timed with CUDA
events (median of the timed repeats). Predicts the strong-scaling efficiency before any
collective: eff(N) = T(1) / (N * max_rank T_rank(N)). Tool only.
Usage: python tools/shard_scaling.py [C4] [--no-graphs] [--variant wavefront|megakernel|auto]
       [--worlds 1,2,4,8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--no-graphs", action="store_true")
ap.add_argument("--variant", default="auto")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--pipeline", type=int, default=0, help="rt_set_pipeline slots (0: library default)")
a = ap.parse_args()
if a.pipeline:
    rt.set_pipeline(a.pipeline)
name = a.config
rt.set_graphs(not a.no_graphs)
rt.set_variant(a.variant)
sc = scenegen.get(name)
rt.load_scene(sc)
W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
base = None
for world in [int(x) for x in a.worlds.split(",")]:
    tpr, sb = rt.shard_layout(W, H, world)
    slab = torch.empty(sb // 4, dtype=torch.float32, device="cuda")
    ts = []
    for rank in range(world):
        for _ in range(3):  # warm-up: plain launches, capture, first replay
            rt.render_shard(W, H, D, S, rank, world, slab)
        reps = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rt.render_shard(W, H, D, S, rank, world, slab)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        ts.append(sorted(reps)[2])
    worst = max(ts)
    if world == 1:
        base = worst
    eff = f"{base / (world * worst):.3f}" if base else "n/a (no world-1 run)"
    print(f"{name} [{a.variant}{f' pipeline {a.pipeline}' if a.pipeline else ''}] world={world}: rank times ms min {min(ts):.3f} max {worst:.3f} -> predicted "
          f"efficiency {eff}", flush=True)
