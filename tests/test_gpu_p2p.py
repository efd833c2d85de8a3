"""Fused render + gather over peer memory (include/rt.h rt_render_shard_direct; SURVEY §8(e)
ablation): every rank's resolve kernel stores its pixels straight into rank 0's frame.

One process: all shards of a world written into one frame equal rt_render bit for bit, stats
included. Two processes on the one GPU of the test box (gloo for the handle exchange and the
barrier; the two ranks' kernels never wait on each other): rank 1 maps rank 0's frame with CUDA
IPC and stores into it — the same code path as one process per GPU over NVLink."""
import os
import socket

import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    yield


@pytest.mark.parametrize("name,variant", [("C2", "megakernel"), ("C2", "wavefront"), ("C3", "wavefront")])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_direct_shards_fill_the_frame(name, variant, world):
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(name)
    if name == "C3":
        sc = sc.with_frame(width=333, height=201, max_depth=3)
    rt.set_variant(variant)
    rt.load_scene(sc)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    ref = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    rt.render(W, H, D, S, ref)
    st_ref = rt.stats()
    frame = torch.full((H, W, 4), float("nan"), dtype=torch.float32, device="cuda")
    rec = torch.zeros(world * 8, dtype=torch.int64, device="cuda")
    for rank in range(world):
        rt.render_shard_direct(W, H, D, S, rank, world, frame.data_ptr(), rec.data_ptr())
    rt.sum_shard_stats(rec.data_ptr(), world)
    st = rt.stats()
    torch.cuda.synchronize()
    assert torch.equal(frame.view(torch.int32), ref.view(torch.int32))
    for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests", "closest_sphere_tests"):
        assert st[k] == st_ref[k], k
    rt.set_variant("auto")


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    from paper_1504_03151_b200 import rt
    from paper_1504_03151_b200.multigpu import P2PRenderer
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = scenegen.get("C3").with_frame(width=320, height=180, max_depth=3)
    rt.set_stream(torch.cuda.current_stream())
    rt.load_scene(sc)
    rend = P2PRenderer(sc.width, sc.height, sc.max_depth, sc.spp)
    for _ in range(2):
        frame = rend.render()
        if rank == 0:
            ref = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
            rt.render(sc.width, sc.height, sc.max_depth, sc.spp, ref)
            st_ref = rt.stats()
            same = bool(torch.equal(frame.image.view(torch.int32), ref.view(torch.int32)))
            counts = [frame.stats[k] == st_ref[k] for k in ("primary", "shadow", "secondary", "sphere_tests")]
            np.savez(result_path, same=same, counts=np.array(counts))
        rend.release()
    dist.barrier()
    rend.close()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_processes_store_into_one_frame_over_ipc(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "p2p.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    assert bool(r["same"]) and r["counts"].all()
