"""Randomised shapes through both kernel organisations: frame sizes 1..300 px wide, 1..300 spp
(sub-pixel table up to 256, computed offsets beyond), depths 0..8, 0..300 spheres, 0..3 planes, 0..32 point
lights (light-origin scans up to 30), device and host framebuffers (host: the falling-size chunk
plan). The wavefront and megakernel frames must be bit-identical, and so must the statistics."""
import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu


def _cases(n=60):
    g = np.random.default_rng(424242)
    out = []
    for i in range(n):
        out.append(dict(seed=500 + i, n_spheres=int(g.choice([0, 1, 3, 31, 64, 150, 300])),
                        n_planes=int(g.integers(0, 4)), n_lights=int(g.choice([0, 1, 4, 8, 17, 30, 32])),
                        width=int(g.choice([1, 7, 33, 128, 300])), height=int(g.choice([1, 5, 36, 90])),
                        max_depth=int(g.integers(0, 9)), spp=int(g.choice([1, 2, 3, 4, 16, 33, 64, 257, 300])),
                        interleave=bool(g.integers(0, 2)), glass_tint=bool(g.integers(0, 2))))
        if out[-1]["n_spheres"] == 0:  # a scene needs a primitive (and so a material) to upload
            out[-1]["n_planes"] = max(out[-1]["n_planes"], 1)
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"s{c['seed']}")
def test_variants_bit_identical_random_shapes(case):
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.random_tiny(**case)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    res = {}
    try:
        for variant in ("wavefront", "megakernel"):
            rt.set_variant(variant)
            rt.load_scene(sc)
            dev = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
            rt.render(W, H, D, S, dev)
            st = rt.stats()
            host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
            rt.render(W, H, D, S, host)
            torch.cuda.synchronize()
            assert torch.isfinite(dev).all()
            assert torch.equal(dev.cpu(), host), variant
            res[variant] = (dev.cpu(), {k: st[k] for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests")})
    finally:
        rt.set_variant("auto")
    assert torch.equal(res["wavefront"][0], res["megakernel"][0])
    assert res["wavefront"][1] == res["megakernel"][1]
    assert res["wavefront"][1]["primary"] == W * H * S
