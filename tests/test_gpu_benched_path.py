"""The path bench.py times, checked against the path the parity tests check.

The oracle-comparing tests render through rt_render_debug (wf_shade<kDebug = true>, per-sample
hit-id records). bench.py times rt_render: the kDebug = false kernels, CUDA-graph capture and
replay with one kernel per scan chosen from the previous frame's queue lengths, the shadow side
stream, chunk pipelining, host framebuffers copied row-band by row-band while later chunks render.
Here that exact launch configuration (bench.py's: the library bound to torch's current stream,
AUTO variant, concurrency, pipelining and graphs on) renders the full BASELINE.json frames C3, C4
and C5 repeatedly, and every frame must equal the debug render bit for bit, with the same ray and
test counts; the debug render itself is held to the oracle by test_gpu_parity.py. The transitive
chain oracle -> rt_render_debug -> rt_render is then closed at full size.
"""
import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu
COUNTS = ("primary", "shadow", "secondary", "sphere_tests", "plane_tests", "closest_sphere_tests")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    from paper_1504_03151_b200 import rt
    rt.set_stream(torch.cuda.current_stream())
    yield
    rt.set_stream(None)


def _debug_frame(rt, sc):
    import torch
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    ids = torch.empty((H * W, S, D + 1), dtype=torch.int32, device="cuda")
    bn = torch.empty((H * W, S), dtype=torch.int32, device="cuda")
    rt.render_debug(W, H, D, S, out, ids, bn)
    st = rt.stats()
    torch.cuda.synchronize()
    del ids, bn
    return out, st


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_benched_render_equals_debug_render(name):
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(name)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    rt.set_variant("auto")
    rt.set_integrator("whitted", False)
    rt.set_graphs(True)  # empty graph cache: this test's own captures only
    rt.load_scene(sc)
    ref, st_ref = _debug_frame(rt, sc)
    ref_u = ref.view(torch.int32)
    # device framebuffer: plain launches, capture, then replays of the cached graph
    out = torch.empty_like(ref)
    modes, ms = [], []
    for _ in range(4):
        out.fill_(float("nan"))
        rt.render(W, H, D, S, out)
        st = rt.stats()
        torch.cuda.synchronize()
        modes.append(st["graph"])
        ms.append(st["last_render_ms"])
        assert torch.equal(out.view(torch.int32), ref_u), name
        for k in COUNTS:
            assert st[k] == st_ref[k], (name, k)
        assert st["variant"] == st_ref["variant"]
    if st_ref["variant"] == 1:  # wavefront (C4, C5): the timed frames replay a captured graph
        assert modes[0] == 0 and modes[1] == 1 and modes[2:] == [2, 2], modes
        # a replay (kernels chosen from the previous frame's per-chunk queue lengths) is never much
        # slower than the plain launches (round 2 regression: hint-sized grids made C5 36x slower)
        assert max(ms[2:]) <= 1.25 * ms[0], ms
    # pinned host framebuffer (the e2e leg of bench.py): rows copied while later chunks render
    host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
    for _ in range(3):
        host.fill_(float("nan"))
        rt.render(W, H, D, S, host)
        st = rt.stats()
        assert torch.equal(host.view(torch.int32), ref_u.cpu()), name
        for k in COUNTS:
            assert st[k] == st_ref[k], (name, k)
    # in-order timing mode (bench.py's per-kernel timing pass) renders the same frame
    rt.set_concurrency(False)
    try:
        for _ in range(3):
            rt.render(W, H, D, S, out)
            torch.cuda.synchronize()
            assert torch.equal(out.view(torch.int32), ref_u), name
    finally:
        rt.set_concurrency(True)


def test_graph_cache_alternating_buffers():
    """Frames alternating between two output buffers (the multi-GPU double-buffered frame) are
    captured once per buffer and then replayed (the single-key cache never replayed)."""
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C4").with_frame(width=480, height=270)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    rt.set_variant("wavefront")
    rt.set_graphs(True)
    rt.load_scene(sc)
    bufs = [torch.empty((H, W, 4), dtype=torch.float32, device="cuda") for _ in range(2)]
    modes = []
    for i in range(8):
        rt.render(W, H, D, S, bufs[i % 2])
        modes.append(rt.stats()["graph"])
    torch.cuda.synchronize()
    assert modes[:4] == [0, 0, 1, 1] and modes[4:] == [2, 2, 2, 2], modes
    assert torch.equal(bufs[0], bufs[1])
    rt.set_variant("auto")


def test_stale_hints_after_material_change():
    """A captured graph keeps its kernel choices (made from the previous frame's per-chunk queue
    lengths) while the scene's contents change under the same launch key (materials, lights: the
    kernels read them at run time; the camera and the geometry's bounds are kernel arguments, so
    changing them starts a new capture). Turning every sphere into a mirror makes every deep queue
    long where the hints say short: the replay must still render the new scene bit for bit, at a
    cost close to the plain launches (a grid sized from the hints would starve: round 2 regression)."""
    import dataclasses
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C4").with_frame(width=960, height=540)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    mirror = dataclasses.replace(sc, mat_kind=np.full_like(sc.mat_kind, scenegen.SPECULAR),
                                 mat_albedo=np.full_like(sc.mat_albedo, 0.9))
    rt.set_variant("wavefront")
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    for first, second in ((sc, mirror), (mirror, sc)):
        rt.set_graphs(True)  # empties the cache: capture with hints from `first`
        rt.load_scene(first)
        for _ in range(3):
            rt.render(W, H, D, S, out)
        assert rt.stats()["graph"] == 2
        rt.scene_upload(*rt.pack_scene(second))  # same sizes and bounds: the same launch key
        rt.render(W, H, D, S, out)
        st = rt.stats()
        assert st["graph"] == 2, "expected a replay with stale hints"
        stale_ms = st["last_render_ms"]
        torch.cuda.synchronize()
        rep = out.clone()
        rt.set_graphs(False)
        rt.render(W, H, D, S, out)
        plain_ms = rt.stats()["last_render_ms"]
        torch.cuda.synchronize()
        assert torch.equal(out, rep)
        assert stale_ms <= 1.5 * plain_ms + 0.2, (stale_ms, plain_ms)
    rt.set_graphs(True)
    rt.set_variant("auto")
