"""Helpers for the GPU tests: render through the C-ABI binding into torch CUDA buffers."""
from __future__ import annotations

import numpy as np


def gpu_render(sc, debug=True, width=None, height=None, max_depth=None, spp=None, variant="wavefront", pixels=None):
    """Render through the C ABI; with `pixels`, only those pixels' records are copied back
    (indices into the row-major frame) — used at full BASELINE sizes."""
    import torch
    from paper_1504_03151_b200 import rt
    W = sc.width if width is None else width
    H = sc.height if height is None else height
    D = sc.max_depth if max_depth is None else max_depth
    S = sc.spp if spp is None else spp
    rt.set_variant(variant)
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
