import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, scenegen
from paper_1504_03151_b200 import rt
for name in sys.argv[1:] or ["C4"]:
    sc = scenegen.get(name); rt.set_variant("wavefront"); rt.load_scene(sc)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out); st = rt.stats(); print(name, st, flush=True)
