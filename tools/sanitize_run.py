#!/usr/bin/env python
"""Target program for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): renders
small frames through every kernel organisation and mode of the library, each several times so the
CUDA-graph capture and replays run too (VERDICT r1 "race and sync-check evidence").

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Cases: C2 (512x256, wavefront, concurrency + 2-slot pipelining + graphs; in-order; megakernel),
C4 (240x135, 4 spp, the light-origin shadow scans and split scans, 1-4 pipeline slots), 16 lights x
1100 spheres (light-origin scans light by light, forced splits), an
interleaved sphere/plane scene with coloured glass, progressive passes with the global integrator
and area lights, shards of world 3 + assembly, and the tone map. Tool only.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_1504_03151_b200 import rt  # noqa: E402


def frames(sc, n=3, **kw):
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    for _ in range(n):
        rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
    torch.cuda.synchronize()
    return out


def main():
    rt.set_stream(torch.cuda.current_stream())
    c2 = scenegen.get("C2").with_frame(width=512, height=256)
    rt.load_scene(c2)
    for variant in ("wavefront", "megakernel"):
        rt.set_variant(variant)
        frames(c2)
    rt.set_variant("wavefront")
    rt.set_concurrency(False)
    frames(c2)
    rt.set_concurrency(True)
    c4 = scenegen.get("C4").with_frame(width=240, height=135)
    rt.load_scene(c4)
    for slots in (1, 2, 3, 4):
        rt.set_pipeline(slots)
        frames(c4, 2)
    rt.set_pipeline(0)
    for split in (2, 8):
        rt.set_scan_split(split)
        frames(c4, 2)
    rt.set_scan_split(-1)
    many = scenegen.random_tiny(77, n_spheres=1100, n_planes=1, n_lights=16, width=40, height=24, max_depth=3, spp=2)
    rt.load_scene(many)  # light-origin columns beyond 64 KB: the short-list scan works light by light
    for split in (-1, 2, 8):
        rt.set_scan_split(split)
        frames(many, 2)
    rt.set_scan_split(-1)
    tiny = scenegen.random_tiny(20, n_spheres=8, n_planes=2, n_lights=3, width=33, height=17, max_depth=5, spp=2,
                                glass_tint=True, interleave=True)
    rt.load_scene(tiny)
    for variant in ("wavefront", "megakernel"):
        rt.set_variant(variant)
        out = frames(tiny)
        ids = torch.empty((tiny.width * tiny.height, tiny.spp, tiny.max_depth + 1), dtype=torch.int32, device="cuda")
        bn = torch.empty((tiny.width * tiny.height, tiny.spp), dtype=torch.int32, device="cuda")
        rt.render_debug(tiny.width, tiny.height, tiny.max_depth, tiny.spp, out, ids, bn)
    rt.set_variant("auto")
    c0 = scenegen.get("C0").with_frame(width=64, height=48)
    rt.load_scene(c0)
    rt.set_integrator("global", True)
    acc = torch.zeros((c0.height, c0.width, 3), dtype=torch.float64, device="cuda")
    out = torch.empty((c0.height, c0.width, 4), dtype=torch.float32, device="cuda")
    for k in range(3):
        rt.render_passes(c0.width, c0.height, c0.max_depth, 4 * k, 4, acc, out)
    rt.set_integrator("whitted", False)
    rt.load_scene(c2)
    tpr, sb = rt.shard_layout(c2.width, c2.height, 3)
    gathered = torch.zeros(3 * sb, dtype=torch.uint8, device="cuda")
    for r in range(3):
        rt.render_shard(c2.width, c2.height, c2.max_depth, c2.spp, r, 3, gathered[r * sb:(r + 1) * sb])
    full = torch.empty((c2.height, c2.width, 4), dtype=torch.float32, device="cuda")
    rt.assemble_tiles(gathered, c2.width, c2.height, 3, full)
    rgba8 = torch.empty((c2.height, c2.width, 4), dtype=torch.uint8, device="cuda")
    rt.tonemap_rgba8(full, rgba8)
    torch.cuda.synchronize()
    print("sanitize_run: done", rt.stats()["primary"])


if __name__ == "__main__":
    main()
