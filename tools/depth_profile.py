"""Cost of each depth of one rank's shard: the shard rendered with max_depth = 0..D, in order
(rt_set_concurrency(0)) and concurrent; the difference between consecutive max_depth values is
the device time that depth adds. Tool only. Usage: python tools/depth_profile.py [C4] [world]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sc = scenegen.get(name)
rt.load_scene(sc)
W, H, S = sc.width, sc.height, sc.spp
tpr, sb = rt.shard_layout(W, H, world)
slab = torch.empty(sb // 4, dtype=torch.float32, device="cuda")


def timed(D, reps=7):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rt.render_shard(W, H, D, S, 0, world, slab)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], rt.stats()


for conc in (True, False):
    rt.set_concurrency(conc)
    prev = 0.0
    prev_rays = 0
    for D in range(sc.max_depth + 1):
        t, st = timed(D)
        rays = st["primary"] + st["shadow"] + st["secondary"]
        print(f"{name} world={world} conc={int(conc)} max_depth={D}: {t:.3f} ms (+{t - prev:.3f}) rays +{rays - prev_rays} "
              f"secondary={st['secondary']} shadow={st['shadow']} closest={st['isect_closest_ms']:.3f} "
              f"shadow_ms={st['isect_shadow_ms']:.3f} shade={st['shade_ms']:.3f}", flush=True)
        prev, prev_rays = t, rays
rt.set_concurrency(True)
