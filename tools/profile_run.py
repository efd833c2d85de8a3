"""Render N frames of a config through the C ABI (target command for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--progressive", type=int, default=0, help="passes per frame (global + area lights)")
a = ap.parse_args()
sc = scenegen.get(a.config)
rt.set_stream(torch.cuda.current_stream())
rt.load_scene(sc)
out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
if a.progressive:
    rt.set_integrator("global", True)
    acc = torch.zeros((sc.height, sc.width, 3), dtype=torch.float64, device="cuda")
for f in range(a.frames):
    if a.progressive:
        rt.render_passes(sc.width, sc.height, sc.max_depth, f * a.progressive, a.progressive, acc, out)
    else:
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
st = rt.stats()
torch.cuda.synchronize()
print(a.config, st)
