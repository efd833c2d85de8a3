"""Per-rank work of an N-GPU frame measured on one GPU: rank 0's shard of C4 for world = 1, 2,
4, 8 (rt_render_shard), timed with CUDA events. Predicts the strong-scaling efficiency before any
collective: eff(N) = T(1) / (N * T_rank0(N)). Tool only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
sc = scenegen.get(name)
rt.load_scene(sc)
W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
base = None
for world in (1, 2, 4, 8):
    tpr, sb = rt.shard_layout(W, H, world)
    slab = torch.empty(sb // 4, dtype=torch.float32, device="cuda")
    ts = []
    for r in range(3):
        for rank in ([0] if r < 2 else range(world)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rt.render_shard(W, H, D, S, rank, world, slab)
            e1.record()
            torch.cuda.synchronize()
            if r == 2:
                ts.append(e0.elapsed_time(e1))
    worst = max(ts)
    base = base or worst
    print(f"{name} world={world}: rank times ms min {min(ts):.3f} max {worst:.3f} -> predicted efficiency "
          f"{base / (world * worst):.3f}", flush=True)
