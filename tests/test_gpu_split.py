"""Split scans: forcing 1, 2, 4 or 8 warps per ray group on every intersection scan
(rt_set_scan_split) must reproduce the default frame bit for bit, debug hit records and ray
statistics included — whatever the queue length, with stream launches and with graph replays
(where each kernel pair is captured as the one kernel the previous frame's queue lengths pick)."""
import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu

KEYS = ("primary", "shadow", "secondary", "sphere_tests", "plane_tests", "closest_sphere_tests")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    from paper_1504_03151_b200 import rt
    yield
    rt.set_scan_split(-1)
    rt.set_graphs(True)
    rt.set_variant("auto")


def _render(sc, split, graphs, reps):
    import torch
    from paper_1504_03151_b200 import rt
    rt.set_variant("wavefront")
    rt.set_graphs(graphs)
    rt.set_scan_split(split)
    rt.load_scene(sc)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    ids = torch.empty((H * W, S, D + 1), dtype=torch.int32, device="cuda")
    bn = torch.empty((H * W, S), dtype=torch.int32, device="cuda")
    res = []
    for _ in range(reps):
        out.fill_(-1.0)
        rt.render_debug(W, H, D, S, out, ids, bn)
        st = rt.stats()
        torch.cuda.synchronize()
        res.append((out.cpu().numpy().copy(), ids.cpu().numpy().copy(), bn.cpu().numpy().copy(),
                    {k: st[k] for k in KEYS}))
    return res


@pytest.mark.parametrize("name,frame", [("C3", dict(width=480, height=270)),
                                        ("C4", dict(width=320, height=180, spp=1)),
                                        ("C5", dict(width=256, height=144, spp=1, max_depth=8))])
def test_forced_split_is_bit_identical(name, frame):
    sc = scenegen.get(name).with_frame(**frame)
    ref = _render(sc, -1, False, 1)[0]
    for split in (1, 2, 4, 8):
        for graphs, reps in ((False, 1), (True, 3)):
            for out, ids, bn, st in _render(sc, split, graphs, reps):
                assert np.array_equal(out, ref[0]), (split, graphs)
                assert np.array_equal(ids, ref[1]) and np.array_equal(bn, ref[2]), (split, graphs)
                assert st == ref[3], (split, graphs)


@pytest.mark.parametrize("name,frame,world", [("C4", dict(width=480, height=270, spp=4), 1),
                                              ("C4", dict(width=960, height=540, spp=4), 8)])
def test_pipeline_slots_bit_identical(name, frame, world):
    """Chunk pipelining over 1..4 buffer-set slots (rt_set_pipeline) renders the same frame / shard
    bit for bit, with the same statistics, launched stream by stream and replayed as a graph."""
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(name).with_frame(**frame)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    tpr, sb = rt.shard_layout(W, H, world)
    ref = None
    try:
        for slots in (1, 2, 3, 4):
            rt.set_pipeline(slots)
            rt.set_graphs(True)
            for rank in (0, world - 1):
                slab = torch.zeros(sb, dtype=torch.uint8, device="cuda")
                outs = []
                for _ in range(3):  # plain, capture, replay
                    rt.render_shard(W, H, D, S, rank, world, slab)
                    st = rt.stats()
                    torch.cuda.synchronize()
                    outs.append((slab.clone(), {k: st[k] for k in KEYS}))
                for o, st in outs:
                    key = (rank,)
                    if ref is None:
                        ref = {}
                    if key not in ref:
                        ref[key] = (o, st)
                    assert torch.equal(o, ref[key][0]), (slots, rank)
                    assert st == ref[key][1], (slots, rank)
        with pytest.raises(rt.RtError):
            rt.set_pipeline(-1)
        with pytest.raises(rt.RtError):
            rt.set_pipeline(5)
    finally:
        rt.set_pipeline(0)


def test_invalid_split_rejected():
    from paper_1504_03151_b200 import rt
    for bad in (0, 3, 16, -2):
        with pytest.raises(rt.RtError):
            rt.set_scan_split(bad)
