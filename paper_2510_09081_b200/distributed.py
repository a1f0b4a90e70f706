"""Multi-GPU sharding of the per-frame path (one process per GPU, torch.distributed).

The path shards in three independent ways; only the first has a data-path
exchange:

1. **Segment-sharded voxelization** -- rank g voxelizes segments ``[bounds[g], bounds[g+1])``
   (the reference's own chunking, lv/voxelizer.py:461-463) into its private packed grid; the grids
   are merged with ONE all-reduce.  A plain sum of packed u32 words would let the 16-bit occupancy
   field carry into the count field, and the reference saturates each field separately
   (lv/voxelizer.py:490-495), so the exchange format is one int64 per voxel,
   ``(count << 32) | occ_q`` -- sum-reducible and exact -- re-packed with per-field saturation
   afterwards.  The result equals the reference's worker-count-invariant grid.
2. **Screen-tile tracing** -- after the merge every rank holds the full pyramid, builds culling /
   A-buffer / shading locally (replicated) and traces only its pixel rectangle; tiles are gathered.
3. **Frame-sharded sequences** -- frames of a dynamic sequence are independent: rank g renders
   frames g, g+G, ...; no communication (this is what ``bench.py --gpus N`` measures).

`merge_partial_grids` is written with device-agnostic torch ops so that the same code runs under
NCCL on GPUs and under gloo in the CPU tests (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

import numpy as np

__all__ = ["shard_bounds", "tile_rects", "frames_for_rank", "widen_packed", "pack_wide",
           "merge_partial_grids", "TiledFrame"]


def shard_bounds(n_segments: int, world: int) -> np.ndarray:
    """lv/voxelizer.py:461-463 `_chunk_bounds`: world+1 ascending bounds covering [0, n)."""
    world = max(1, min(int(world), max(1, int(n_segments))))
    return np.linspace(0, int(n_segments), world + 1).astype(np.int64)


def tile_rects(width: int, height: int, world: int) -> list:
    """Split the image into `world` horizontal strips (x0, y0, x1, y1), rows balanced to +-1.
    Strips keep each rank's pixels contiguous in the (H, W) image, so the gather is a concat."""
    ys = np.linspace(0, int(height), int(world) + 1).astype(np.int64)
    return [(0, int(ys[g]), int(width), int(ys[g + 1])) for g in range(int(world))]


def frames_for_rank(n_frames: int, rank: int, world: int) -> range:
    return range(int(rank), int(n_frames), int(world))


def widen_packed(base_i32):
    """packed (count << 16 | occ_q) int32 bit patterns -> (count << 32) | occ_q as int64."""
    import torch
    w = base_i32.to(torch.int64) & 0xFFFFFFFF
    return ((w >> 16) << 32) | (w & 0xFFFF)


def pack_wide(wide_i64):
    """int64 (count << 32 | occ sum) -> packed int32 bit patterns with per-field saturation
    (lv/voxelizer.py:493-495).  Returns (packed, visited = sum of counts before clamping)."""
    import torch
    cnt = wide_i64 >> 32
    occ = wide_i64 & 0xFFFFFFFF
    visited = int(cnt.sum().item())
    packed = (torch.clamp(cnt, max=0xFFFF) << 16) | torch.clamp(occ, max=0xFFFF)
    # reinterpret the low 32 bits as int32 (values >= 2^31 wrap to negative bit patterns)
    packed = torch.where(packed >= 2 ** 31, packed - 2 ** 32, packed).to(torch.int32)
    return packed, visited


def merge_partial_grids(base_i32, group=None):
    """All-reduce the per-rank packed grids exactly.  `base_i32`: this rank's finalized packed grid
    (int32 bit patterns, any device).  Returns (merged packed int32 grid, total visited)."""
    import torch.distributed as dist
    wide = widen_packed(base_i32)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(wide, op=dist.ReduceOp.SUM, group=group)
    return pack_wide(wide)


class TiledFrame:
    """One frame rendered cooperatively by all ranks: segment-sharded voxelization + all-reduce,
    replicated build, per-rank screen tile, gather to rank 0.  Wraps a FrameEngine."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.engine, self.group = engine, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.tiles = tile_rects(engine.w, engine.h, self.world)

    def _merge(self, eng):
        if eng.use_wide:     # the engine's 64-bit accumulators are sum-reducible as they are; it packs afterwards
            import torch.distributed as dist
            dist.all_reduce(eng.wide, op=dist.ReduceOp.SUM, group=self.group)
            return
        merged, _ = merge_partial_grids(eng.base, self.group)
        eng.base.copy_(merged)

    def run(self, cam, grid, r_world):
        eng = self.engine
        n_seg = eng._segs.numel()
        b = shard_bounds(n_seg, self.world)
        lo, hi = (int(b[self.rank]), int(b[self.rank + 1])) if self.rank < len(b) - 1 else (0, 0)
        return eng.run(cam, grid, r_world, tile=self.tiles[self.rank], seg_range=(lo, hi),
                       after_voxelize=self._merge if self.world > 1 else None)

    def gather_image(self):
        """Rank 0 receives the full sRGB image and hit ids (H, W, 3) u8 / (H, W) i32; others None."""
        import torch
        import torch.distributed as dist
        eng = self.engine
        x0, y0, x1, y1 = self.tiles[self.rank]
        if self.world == 1:
            return eng.srgb, eng.hit_id
        rows = max(t[3] - t[1] for t in self.tiles)
        pad_s = torch.zeros((rows, eng.w, 3), dtype=torch.uint8, device=eng.srgb.device)
        pad_h = torch.zeros((rows, eng.w), dtype=torch.int32, device=eng.srgb.device)
        pad_s[:y1 - y0] = eng.srgb[y0:y1]
        pad_h[:y1 - y0] = eng.hit_id[y0:y1]
        outs = [torch.empty_like(pad_s) for _ in range(self.world)] if self.rank == 0 else None
        outh = [torch.empty_like(pad_h) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(pad_s, outs, dst=0, group=self.group)
        dist.gather(pad_h, outh, dst=0, group=self.group)
        if self.rank != 0:
            return None, None
        srgb = torch.cat([o[:t[3] - t[1]] for o, t in zip(outs, self.tiles)], dim=0)
        hit = torch.cat([o[:t[3] - t[1]] for o, t in zip(outh, self.tiles)], dim=0)
        return srgb, hit
