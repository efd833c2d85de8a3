import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, scenegen
from paper_1504_03151_b200 import rt
import sys as _s
variants = _s.argv[1:] or ["wavefront", "megakernel"]
for name in ["C2","C3","C4"]:
  for var in variants:
    rt.set_variant(var)
    sc = scenegen.get(name); rt.load_scene(sc)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out); torch.cuda.synchronize()
    ts=[]
    for _ in range(5):
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out); st = rt.stats(); ts.append(st["last_render_ms"])
    rays = st["primary"]+st["shadow"]+st["secondary"]
    print(name, var, "ms", min(ts), "Mrays/s", rays/min(ts)/1e3, st, "counted TFLOP/s", (19*st["sphere_tests"]+12*st["plane_tests"])/min(ts)/1e9)
