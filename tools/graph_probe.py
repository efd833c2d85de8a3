"""Would CUDA graphs pay? One rank's shard of C4 rendered with stream launches vs the same launch
sequence captured once into a CUDA graph (torch.cuda.graph around rt_render_shard) and replayed.
Checks the replayed slab is bit-identical. Tool only."""
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


def med(fn, reps=21):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for world in (1, 2, 4, 8):
    tpr, sb = rt.shard_layout(W, H, world)
    slab = torch.zeros(sb // 4, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    rt.set_stream(s)
    for _ in range(3):
        rt.render_shard(W, H, D, S, 0, world, slab)
    torch.cuda.synchronize()
    ref = slab.clone()

    def plain():
        rt.render_shard(W, H, D, S, 0, world, slab)

    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        t_plain = med(plain)
    g = torch.cuda.CUDAGraph()
    slab.zero_()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        rt.render_shard(W, H, D, S, 0, world, slab)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    same = torch.equal(slab, ref)
    t_graph = med(g.replay)
    print(f"{name} world={world}: stream launches {t_plain:.3f} ms | graph replay {t_graph:.3f} ms | bit-identical {same}",
          flush=True)
rt.set_stream(None)
