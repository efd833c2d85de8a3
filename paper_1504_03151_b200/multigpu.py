"""Multi-GPU frame driver: image tiles sharded across ranks, one collective per frame.

SURVEY.md §8(e): the image is cut into 8x4-pixel tiles; group j of `world` consecutive tiles gives
rank r its tile j * world + (r + j) % world
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
    tiles = [j * world + (rank + j) % world for j in range(tpr)]  # rank_tile (rt_device.cuh)
    return [t for t in tiles if t < nt]


class P2PRenderer:
    """Fused render + gather over NVLink peer memory (SURVEY §8(e) ablation; include/rt.h
    rt_render_shard_direct). Rank 0 owns the frames and world x 8 uint64 stats-record arrays,
    allocated for CUDA IPC; the handles travel once over the process group and every other rank
    maps them (peer access over NVLink / NVSwitch). Each frame, every rank's resolve kernel
    stores its pixels straight into rank 0's frame — no slab, no all-gather, no assembly kernel.

    Ordering. With NCCL, two stream-ordered all-reduces of a 4-byte token per frame order the
    peer stores, and the host never waits:
      * the frame barrier (after the render): it completes on every rank only after every rank's
        render kernels have completed (their peer stores included), so rank 0's work issued after
        render() returns sees the whole frame;
      * the release barrier (before the render, when the frame reuses a buffer): frame i + nbuf
        stores into frame i's buffer only after rank 0's stream has passed everything rank 0
        issued before that render() call — its reads of frame i included.
    So the image of frame i stays valid for every read rank 0 issues (on its current stream)
    before its next-but-one render() call. With other backends (gloo, the CPU tests) the host
    synchronises its stream and calls dist.barrier() at both points."""

    def __init__(self, width: int, height: int, max_depth: int, spp: int, group=None, buffers: int = 2):
        self.W, self.H, self.D, self.spp = width, height, max_depth, spp
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nbuf = max(1, int(buffers))
        self.frame_ptrs: list = []
        self.rec_ptrs: list = []
        handles = [None] * (2 * self.nbuf)
        if self.rank == 0:
            try:
                for b in range(self.nbuf):
                    fp, hf = rt.ipc_alloc(width * height * 16)
                    self.frame_ptrs.append(fp)
                    rp, hr = rt.ipc_alloc(self.world * 64)
                    self.rec_ptrs.append(rp)
                    handles[2 * b], handles[2 * b + 1] = hf, hr
            except rt.RtError:
                handles = [None] * (2 * self.nbuf)
        if self.world > 1:
            dist.broadcast_object_list(handles, src=0, group=self.group)
        ok = all(h is not None for h in handles)
        if ok and self.rank != 0:
            try:
                for b in range(self.nbuf):
                    self.frame_ptrs.append(rt.ipc_open(handles[2 * b]))
                    self.rec_ptrs.append(rt.ipc_open(handles[2 * b + 1]))
            except rt.RtError:
                ok = False
        self.nccl = self.world > 1 and dist.get_backend(group) == "nccl"
        if self.world > 1:  # every rank agrees, so a failure raises everywhere (no one waits forever)
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda" if self.nccl else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            ok = bool(flag.item())
        if not ok:
            self.close()
            raise RuntimeError("peer-memory frame unavailable (CUDA IPC / peer access failed on some rank)")
        self.token = torch.zeros(1, dtype=torch.int32, device="cuda") if self.nccl else None
        self.images = []
        if self.rank == 0:
            self.images = [torch.as_tensor(rt.DeviceArray(fp, (height, width, 4), "<f4"), device="cuda")
                           for fp in self.frame_ptrs]
        self.image = None
        self.frames = 0

    def _barrier(self):
        if self.world == 1:
            return
        if self.nccl:  # stream-ordered: no host wait
            dist.all_reduce(self.token, group=self.group)
        else:
            torch.cuda.current_stream().synchronize()  # this rank's stores (and stats record) done
            dist.barrier(group=self.group)

    def render(self, want_stats: bool = True) -> Frame:
        """Render this rank's tiles of the next frame into rank 0's buffer. Rank 0 gets the image
        (stream-ordered after every rank's stores) and, with want_stats, the summed statistics
        (a host sync); reads of the image issued before the next-but-one call are safe."""
        b = self.frames % self.nbuf
        if self.frames >= self.nbuf:
            self._barrier()  # release: rank 0's reads of this buffer's previous frame come first
        self.frames += 1
        rt.render_shard_direct(self.W, self.H, self.D, self.spp, self.rank, self.world, self.frame_ptrs[b],
                               self.rec_ptrs[b])
        self._barrier()
        if self.rank == 0:
            rt.sum_shard_stats(self.rec_ptrs[b], self.world)
            self.image = self.images[b]
            return Frame(self.image, rt.stats() if want_stats else None)
        return Frame(None, None)

    def release(self):
        """Nothing to do: the release barrier at the start of the render that reuses a buffer
        orders the new peer stores after rank 0's reads (kept for callers of earlier versions)."""

    def close(self):
        self.image = None
        self.images = []
        for ptr in self.frame_ptrs + self.rec_ptrs:
            if ptr:
                (rt.ipc_free if self.rank == 0 else rt.ipc_close)(ptr)
        self.frame_ptrs, self.rec_ptrs = [], []


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
