"""World-size-2 test of the multi-GPU host logic on CPU (gloo): tile layout, per-rank slabs with
their stats record, the single all-gather, slab -> framebuffer assembly order, stats summation.

The per-rank "renderer" here is the oracle (test infrastructure) writing the same slab format the
CUDA library writes; the CUDA slab/assembly kernels themselves are covered on the GPU by
tests/test_gpu_parity.py::test_shards_assemble_bit_identical.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import scenegen
from paper_1504_03151_b200 import multigpu

SCENE = dict(seed=3, n_spheres=5, n_planes=1, n_lights=2, width=21, height=10, max_depth=2, spp=2)


class OracleSlabBackend:
    """Writes slabs in the libb200rt layout from oracle renders (CPU test double)."""

    def __init__(self, sc):
        from oracle import pyoracle
        self.po = pyoracle
        self.sc = sc
        self._stats = None

    def alloc(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def render_shard(self, W, H, D, spp, rank, world, slab):
        tpr, sb = multigpu.shard_layout(W, H, world)
        tiles_x, _ = multigpu.n_tiles(W, H)
        px = slab[: tpr * 32 * 16].view(torch.float32).view(tpr * 32, 4).numpy()
        px[:] = 0
        pix, slots = [], []
        for j, t in enumerate(multigpu.rank_tiles(W, H, rank, world)):
            for i in range(32):
                x = (t % tiles_x) * 8 + i % 8
                y = (t // tiles_x) * 4 + i // 8
                if x < W and y < H:
                    pix.append(y * W + x)
                    slots.append(j * 32 + i)
        r = self.po.render(self.sc, pixels=np.array(pix, np.int64))
        px[slots, :3] = r.rgb.astype(np.float32)
        px[slots, 3] = 1.0
        rec = slab[tpr * 32 * 16:].view(torch.int64).numpy()
        rec[:] = 0
        rec[:5] = [r.counts[k] for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests")]

    def assemble(self, gathered, W, H, world, out):
        tpr, sb = multigpu.shard_layout(W, H, world)
        tiles_x, _ = multigpu.n_tiles(W, H)
        g = gathered.numpy()
        img = out.numpy()
        tot = np.zeros(5, np.int64)
        for r in range(world):
            slab = g[r * sb:(r + 1) * sb]
            px = slab[: tpr * 512].view(np.float32).reshape(tpr * 32, 4)
            for j, t in enumerate(multigpu.rank_tiles(W, H, r, world)):
                for i in range(32):
                    x = (t % tiles_x) * 8 + i % 8
                    y = (t // tiles_x) * 4 + i // 8
                    if x < W and y < H:
                        img[y, x] = px[j * 32 + i]
            tot += slab[tpr * 512:tpr * 512 + 40].view(np.int64)
        self._stats = dict(zip(("primary", "shadow", "secondary", "sphere_tests", "plane_tests"), tot.tolist()))

    def stats(self):
        return self._stats


def _worker(rank, world, port, result_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = scenegen.random_tiny(**SCENE)
    rend = multigpu.ShardedRenderer(OracleSlabBackend(sc), sc.width, sc.height, sc.max_depth, sc.spp)
    frame = rend.render()
    if rank == 0:
        np.savez(result_path, img=frame.image.numpy(), **{k: v for k, v in frame.stats.items()})
    else:
        assert frame.image is None
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_world2_gloo_frame_equals_single_process(world, tmp_path, oracle_lib):
    out = str(tmp_path / "frame.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    sc = scenegen.random_tiny(**SCENE)
    ref = oracle_lib.render(sc)
    img = res["img"].reshape(-1, 4)
    assert (img[:, :3] == ref.rgb.astype(np.float32)).all()
    assert (img[:, 3] == 1.0).all()
    for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests"):
        assert int(res[k]) == ref.counts[k], k


def test_layout_covers_every_tile_once():
    for W, H, world in [(21, 10, 2), (1920, 1080, 8), (13, 7, 3), (8, 4, 5)]:
        _, nt = multigpu.n_tiles(W, H)
        seen = sorted(t for r in range(world) for t in multigpu.rank_tiles(W, H, r, world))
        assert seen == list(range(nt))
        tpr, sb = multigpu.shard_layout(W, H, world)
        assert all(len(multigpu.rank_tiles(W, H, r, world)) <= tpr for r in range(world))
        assert sb == tpr * 512 + 64
