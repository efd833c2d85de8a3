"""How much of wf_shade is the light loop: C4 with 8, 1 and 0 point lights (tool only)."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

base = scenegen.get("C4")
for nl in (8, 1, 0):
    sc = replace(base, light_pos=base.light_pos[:nl], light_intensity=base.light_intensity[:nl])
    rt.set_variant("wavefront")
    rt.set_concurrency(False)
    rt.load_scene(sc)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    best = None
    for _ in range(5):
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
        st = rt.stats()
        if best is None or st["last_render_ms"] < best["last_render_ms"]:
            best = st
    print(f"lights={nl}: frame {best['last_render_ms']:.3f} shade {best['shade_ms']:.3f} shadow {best['isect_shadow_ms']:.3f} "
          f"closest {best['isect_closest_ms']:.3f} shadow rays {best['shadow']}", flush=True)
