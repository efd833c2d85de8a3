"""Multi-GPU frame driver: image tiles sharded across ranks, one collective per frame.

SURVEY.md §8(e): the image is cut into 8x4-pixel tiles; tile t belongs to rank t % world
(cyclic, spatially interleaved, statistically balanced); inside a rank, persistent CTAs take the
rank's tiles dynamically. Each rank renders its tiles into a dense slab (plus a 64-byte stats
record); ONE all-gather over NCCL (NVLink 5 / NVSwitch) brings the slabs to every rank and rank 0
assembles the row-major framebuffer. The scene is replicated (every rank loads the same seeded
scene), so there is no broadcast. The framebuffer is bit-identical for every world size.

The driver is generic over a `backend` with three calls so that its host logic (layout, buffer
sizes, collective, assembly order) is testable on CPU with gloo; `CudaBackend` is the product
path (C-ABI library), there is no CPU fallback in it.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import rt

TILE_W, TILE_H, TILE_PX = rt.TILE_W, rt.TILE_H, rt.TILE_W * rt.TILE_H
STATS_BYTES = 64


def n_tiles(width: int, height: int) -> tuple[int, int]:
    tx = (width + TILE_W - 1) // TILE_W
    return tx, tx * ((height + TILE_H - 1) // TILE_H)


def shard_layout(width: int, height: int, world: int) -> tuple[int, int]:
    """(tiles_per_rank, slab_bytes) — same contract as rt_shard_layout (include/rt.h)."""
    _, nt = n_tiles(width, height)
    tpr = (nt + world - 1) // world
    return tpr, tpr * TILE_PX * 16 + STATS_BYTES


def rank_tiles(width: int, height: int, rank: int, world: int) -> list[int]:
    """Global tile ids owned by `rank`, in slab order (cyclic assignment)."""
    tpr, _ = shard_layout(width, height, world)
    _, nt = n_tiles(width, height)
    return [j * world + rank for j in range(tpr) if j * world + rank < nt]


class CudaBackend:
    """The product path: libb200rt.so through the ctypes binding."""

    def __init__(self, device: torch.device):
        self.device = device

    def alloc(self, nbytes: int) -> torch.Tensor:
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def render_shard(self, W, H, D, spp, rank, world, slab):
        rt.render_shard(W, H, D, spp, rank, world, slab)

    def assemble(self, gathered, W, H, world, out):
        rt.assemble_tiles(gathered, W, H, world, out)

    def stats(self) -> dict:
        return rt.stats()


@dataclass
class Frame:
    image: torch.Tensor | None   # [H, W, 4] float32 on rank 0, None elsewhere
    stats: dict | None           # summed over ranks, rank 0 only


class ShardedRenderer:
    """Render frames of a fixed size with `world` ranks of the default process group."""

    def __init__(self, backend, width: int, height: int, max_depth: int, spp: int, group=None):
        self.b = backend
        self.W, self.H, self.D, self.spp = width, height, max_depth, spp
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.tpr, self.slab_bytes = shard_layout(width, height, self.world)
        self.slab = backend.alloc(self.slab_bytes)
        self.gathered = backend.alloc(self.slab_bytes * self.world) if self.world > 1 else self.slab
        self.out = None
        if self.rank == 0:
            self.out = torch.empty((height, width, 4), dtype=torch.float32, device=self.slab.device)

    def render(self) -> Frame:
        self.b.render_shard(self.W, self.H, self.D, self.spp, self.rank, self.world, self.slab)
        if self.world > 1:
            # the only collective of the frame: every rank's slab (+ stats record) to all ranks
            dist.all_gather_into_tensor(self.gathered, self.slab, group=self.group)
        if self.rank == 0:
            self.b.assemble(self.gathered, self.W, self.H, self.world, self.out)
            return Frame(self.out, self.b.stats())
        return Frame(None, None)

    @property
    def launches_per_frame(self) -> int:
        """Kernels of ours per frame on this rank: render (+ assemble + stats sum on rank 0)."""
        return 1 + (2 if self.rank == 0 else 0)
