"""Helpers for the GPU tests: render through the C-ABI binding into torch CUDA buffers."""
from __future__ import annotations

import numpy as np


def gpu_render(sc, debug=True, width=None, height=None, max_depth=None, spp=None, variant="wavefront", pixels=None,
               integrator="whitted", area_lights=False):
    """Render through the C ABI; with `pixels`, only those pixels' records are copied back
    (indices into the row-major frame) — used at full BASELINE sizes."""
    import torch
    from paper_1504_03151_b200 import rt
    W = sc.width if width is None else width
    H = sc.height if height is None else height
    D = sc.max_depth if max_depth is None else max_depth
    S = sc.spp if spp is None else spp
    rt.set_variant(variant)
    rt.set_integrator(integrator, area_lights)
    rt.load_scene(sc)
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    if debug:
        ids = torch.empty((H * W, S, D + 1), dtype=torch.int32, device="cuda")
        bn = torch.empty((H * W, S), dtype=torch.int32, device="cuda")
        rt.render_debug(W, H, D, S, out, ids, bn)
    else:
        rt.render(W, H, D, S, out)
    st = rt.stats()
    torch.cuda.synchronize()
    sel = slice(None) if pixels is None else torch.as_tensor(np.asarray(pixels), device="cuda", dtype=torch.long)
    rgba = out.reshape(-1, 4)[sel].cpu().numpy()
    res = {"rgba": rgba, "rgb": rgba[:, :3], "stats": st}
    if debug:
        res["ids"] = ids[sel].cpu().numpy()
        res["bounces"] = bn[sel].cpu().numpy()
    return res


def gpu_passes(sc, pass_begin, n_passes, accum=None, debug=True, integrator="global", area_lights=True,
               width=None, height=None, max_depth=None, variant="auto"):
    """Progressive passes through rt_render_passes(_debug); returns host copies."""
    import torch
    from paper_1504_03151_b200 import rt
    W = sc.width if width is None else width
    H = sc.height if height is None else height
    D = sc.max_depth if max_depth is None else max_depth
    rt.set_variant(variant)
    rt.set_integrator(integrator, area_lights)
    rt.load_scene(sc)
    if accum is None:
        accum = torch.zeros((H, W, 3), dtype=torch.float64, device="cuda")
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    res = {}
    if debug:
        ids = torch.empty((H * W, n_passes, D + 1), dtype=torch.int32, device="cuda")
        bn = torch.empty((H * W, n_passes), dtype=torch.int32, device="cuda")
        rt.render_passes_debug(W, H, D, pass_begin, n_passes, accum, out, ids, bn)
    else:
        rt.render_passes(W, H, D, pass_begin, n_passes, accum, out)
    st = rt.stats()
    torch.cuda.synchronize()
    res.update(accum=accum, accum_np=accum.reshape(-1, 3).cpu().numpy(), rgba=out.reshape(-1, 4).cpu().numpy(),
               stats=st)
    if debug:
        res["ids"] = ids.cpu().numpy()
        res["bounces"] = bn.cpu().numpy()
    rt.set_integrator("whitted", False)
    return res
