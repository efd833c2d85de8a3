"""CUDA-graph replay of the wavefront launch sequence (include/rt.h rt_set_graphs): the second
render with the same launch key is captured, later ones are replayed. Replayed frames, shards and
debug records must equal stream-launched ones bit for bit, ray statistics included, and a change
of camera or scene between renders must show up in the next frame (the kernels read them at run
time; the camera basis is a kernel argument and re-keys the graph)."""
import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu

KEYS = ("primary", "shadow", "secondary", "sphere_tests", "plane_tests")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    from paper_1504_03151_b200 import rt
    yield
    rt.set_graphs(True)
    rt.set_variant("auto")


def _frames(sc, graphs, n, W=None, H=None, D=None, S=None, debug=False, between=None):
    import torch
    from paper_1504_03151_b200 import rt
    W = W or sc.width
    H = H or sc.height
    D = sc.max_depth if D is None else D
    S = S or sc.spp
    rt.set_graphs(graphs)
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    ids = torch.empty((H * W, S, D + 1), dtype=torch.int32, device="cuda")
    bn = torch.empty((H * W, S), dtype=torch.int32, device="cuda")
    res = []
    for i in range(n):
        if between is not None:
            between(i)
        out.fill_(-1.0)
        if debug:
            rt.render_debug(W, H, D, S, out, ids, bn)
        else:
            rt.render(W, H, D, S, out)
        st = rt.stats()
        torch.cuda.synchronize()
        res.append((out.cpu().numpy().copy(), ids.cpu().numpy().copy() if debug else None,
                    bn.cpu().numpy().copy() if debug else None, {k: st[k] for k in KEYS}))
    return res


@pytest.mark.parametrize("name,debug", [("C2", False), ("C2", True), ("C3", False)])
def test_replay_equals_stream_launches(name, debug):
    sc = scenegen.get(name)
    if name == "C3":
        sc = sc.with_frame(width=480, height=270)
    ref = _frames(sc, False, 1, debug=debug)[0]
    got = _frames(sc, True, 4, debug=debug)  # plain, capture + launch, replay, replay
    for out, ids, bn, st in got:
        assert np.array_equal(out, ref[0])
        assert st == ref[3]
        if debug:
            assert np.array_equal(ids, ref[1]) and np.array_equal(bn, ref[2])


def test_camera_change_between_replays():
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C2").with_frame(width=256, height=192)
    eyes = [sc.eye, (sc.eye[0] + 1.5, sc.eye[1], sc.eye[2]), (sc.eye[0] + 1.5, sc.eye[1], sc.eye[2])]

    def cam(i):
        rt.camera_set(eyes[i], sc.look_at, sc.up, sc.vfov)

    got = _frames(sc, True, 3, between=cam)
    ref = _frames(sc, False, 3, between=cam)
    for (g, _, _, gs), (r, _, _, rs) in zip(got, ref):
        assert np.array_equal(g, r) and gs == rs
    assert not np.array_equal(got[0][0], got[1][0])


def test_scene_contents_change_between_replays():
    """Same sizes (same launch key), different light intensities: the replay reads the new ones."""
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C2").with_frame(width=200, height=150)
    prims, mats, lights, env = rt.pack_scene(sc)
    brighter = lights.copy()
    brighter["intensity"] *= 2.0

    def upload(i):
        rt.scene_upload(prims, mats, brighter if i == 3 else lights, env)
        rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)

    got = _frames(sc, True, 4, between=upload)
    ref = _frames(sc, False, 4, between=upload)
    for (g, _, _, gs), (r, _, _, rs) in zip(got, ref):
        assert np.array_equal(g, r) and gs == rs
    assert np.array_equal(got[0][0], got[2][0])
    assert not np.array_equal(got[2][0], got[3][0])


@pytest.mark.parametrize("world", [2, 8])
def test_replayed_shards(world):
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C3").with_frame(width=400, height=240, max_depth=4)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    tpr, sb = rt.shard_layout(W, H, world)
    slabs = {}
    for graphs in (False, True):
        rt.set_graphs(graphs)
        slab = torch.empty(sb // 4, dtype=torch.float32, device="cuda")
        outs = []
        for _ in range(3):
            for rank in range(world):
                slab.fill_(-1.0)
                rt.render_shard(W, H, D, S, rank, world, slab)
                st = rt.stats()
                torch.cuda.synchronize()
                outs.append((rank, slab.cpu().numpy().copy(), {k: st[k] for k in KEYS}))
            for rank in (world - 1, world - 1, world - 1):  # same rank in a row: capture + replay
                slab.fill_(-1.0)
                rt.render_shard(W, H, D, S, rank, world, slab)
                st = rt.stats()
                torch.cuda.synchronize()
                outs.append((rank, slab.cpu().numpy().copy(), {k: st[k] for k in KEYS}))
        slabs[graphs] = outs
    for (r0, a, sa), (r1, b, sb_) in zip(slabs[False], slabs[True]):
        assert r0 == r1 and np.array_equal(a, b) and sa == sb_


def test_caller_capture_falls_back_to_plain_launches():
    """A caller capturing its own CUDA graph around rt_render gets the plain launches captured
    (the library never launches its cached graph into a capturing stream)."""
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C2").with_frame(width=160, height=120)
    ref = _frames(sc, False, 1)[0][0]
    rt.set_graphs(True)
    s = torch.cuda.Stream()
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    rt.set_stream(s)
    try:
        for _ in range(3):  # the library's own graph is live when the caller starts capturing
            rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
        out.fill_(-1.0)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)
    finally:
        rt.set_stream(None)
