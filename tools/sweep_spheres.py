"""Time C4 truncated to its first n spheres, per kernel organisation (A/B helper for the AUTO
thresholds in rt_api.cu). Usage: python tools/sweep_spheres.py [variant ...]"""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

variants = sys.argv[1:] or ["wavefront", "megakernel"]
base = scenegen.get("C4")
for n in (32, 64, 128, 256, 384, 512, 768, 1000):
    sc = replace(base, prim_type=base.prim_type[:n], prim_mat=base.prim_mat[:n], prim_p=base.prim_p[:n])
    for var in variants:
        rt.set_variant(var)
        rt.load_scene(sc)
        out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
            st = rt.stats()
            ts.append(st["last_render_ms"])
        rays = st["primary"] + st["shadow"] + st["secondary"]
        print(f"n={n:5d} {var:10s} ms {min(ts):8.3f} Mrays/s {rays / min(ts) / 1e3:8.1f}", flush=True)
