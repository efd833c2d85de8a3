#!/usr/bin/env python
"""Render one rank's shard of a config N times (target command for ncu launch lists of small
shards). Tool only. Usage: python tools/shard_run.py [C4] [world] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sc = scenegen.get(name)
rt.set_stream(torch.cuda.current_stream())
rt.load_scene(sc)
tpr, sb = rt.shard_layout(sc.width, sc.height, world)
slab = torch.empty(sb, dtype=torch.uint8, device="cuda")
for _ in range(frames):
    rt.render_shard(sc.width, sc.height, sc.max_depth, sc.spp, 0, world, slab)
torch.cuda.synchronize()
print(name, world, rt.stats())
