"""Wall-clock breakdown of bench.py's end-to-end step (scene upload, camera, render into pinned
host memory) on C4. Tool only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

sc = scenegen.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
prims, mats, lights, env = rt.pack_scene(sc)
rt.set_stream(torch.cuda.current_stream())
rt.load_scene(sc)
host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
dev = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
for _ in range(3):
    rt.render(W, H, D, S, host)
acc = {"upload": 0.0, "camera": 0.0, "render_host": 0.0, "render_dev+sync": 0.0}
n = 10
for _ in range(n):
    t0 = time.perf_counter(); rt.scene_upload(prims, mats, lights, env)
    t1 = time.perf_counter(); rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
    t2 = time.perf_counter(); rt.render(W, H, D, S, host)
    t3 = time.perf_counter(); rt.render(W, H, D, S, dev); torch.cuda.synchronize()
    t4 = time.perf_counter()
    acc["upload"] += t1 - t0; acc["camera"] += t2 - t1; acc["render_host"] += t3 - t2; acc["render_dev+sync"] += t4 - t3
print({k: round(v / n * 1e3, 3) for k, v in acc.items()}, "ms")
