#!/usr/bin/env python
"""Where the end-to-end step of bench.py goes (N = 1): host wall time of rt_scene_upload,
rt_camera_set and rt_render into a pinned host buffer, each over the same steps, next to the
device-buffer render. Tool only. Usage: python tools/e2e_parts.py [C4] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sc = scenegen.get(name)
W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
prims, mats, lights, env = rt.pack_scene(sc)
rt.set_stream(torch.cuda.current_stream())
rt.load_scene(sc)
host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
dev = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
parts = {"scene_upload": 0.0, "camera_set": 0.0, "render_host": 0.0, "render_device": 0.0}
for it in range(3 + steps):
    t0 = time.perf_counter()
    rt.scene_upload(prims, mats, lights, env)
    t1 = time.perf_counter()
    rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
    t2 = time.perf_counter()
    rt.render(W, H, D, S, host)
    t3 = time.perf_counter()
    rt.render(W, H, D, S, dev)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if it >= 3:
        for k, v in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            parts[k] += v / steps
print(name, {k: round(v * 1e3, 3) for k, v in parts.items()}, "ms per step; graph", rt.stats()["graph"])
