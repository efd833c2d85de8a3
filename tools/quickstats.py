"""Per-kernel-class device times of one wavefront frame (library CUDA events): closest scan,
shadow scan, shade, rest. Usage: python tools/quickstats.py [configs...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

for name in sys.argv[1:] or ["C3", "C4"]:
    sc = scenegen.get(name)
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    best = None
    for _ in range(6):
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
        st = rt.stats()
        if best is None or st["last_render_ms"] < best["last_render_ms"]:
            best = st
    t = best["last_render_ms"]
    c, s, h = best["isect_closest_ms"], best["isect_shadow_ms"], best["shade_ms"]
    print(f"{name}: frame {t:.3f} ms | closest {c:.3f} shadow {s:.3f} shade {h:.3f} rest {t - c - s - h:.3f}")
