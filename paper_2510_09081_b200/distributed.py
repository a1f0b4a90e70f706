"""Multi-GPU sharding of the per-frame path (one process per GPU, torch.distributed).

The path shards in three independent ways; only the first has a data-path
exchange:

1. **Segment-sharded voxelization** -- rank g voxelizes segments ``[bounds[g], bounds[g+1])``
   (the reference's own chunking, lv/voxelizer.py:461-463) into its private grid; the grids are
   merged with ONE all-reduce.  A plain sum of packed u32 words would let the 16-bit occupancy
   field carry into the count field, and the reference saturates each field separately
   (lv/voxelizer.py:490-495), so the exchange format is one int64 per voxel,
   ``(count << 32) | occ_q`` -- sum-reducible and exact -- re-packed with per-field saturation
   afterwards.  The result equals the reference's worker-count-invariant grid.
2. **Screen-tile tracing** -- after the merge every rank holds the full pyramid and the full culling
   pyramid (march bits), builds the A-buffer and the shading only for the voxels its own pixel
   rectangle's rays can visit (lvx_tile_owners) and traces that rectangle; tiles are gathered.
3. **Frame-sharded sequences** -- frames of a dynamic sequence are independent: rank g renders
   frames g, g+G, ...; no communication (``bench.py --gpus N`` default).

`TiledFrame` (1 + 2) talks to its peers through a small `Comm` object: `TorchComm` is
torch.distributed (NCCL on GPUs, gloo in the CPU tests), `EmulatedComm` plays one rank of a G-rank
job on a single device -- the peers' contribution to the all-reduce is produced by voxelizing their
segment shards locally -- so that the per-rank work of a G-GPU frame can be tested and timed on
the one GPU this project's runs have.

`merge_partial_grids` is written with device-agnostic torch ops so that the same code runs under
NCCL on GPUs and under gloo in the CPU tests (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

import numpy as np

__all__ = ["shard_bounds", "tile_rects", "balanced_rows", "frames_for_rank", "widen_packed", "pack_wide",
           "field_bounds", "exchange_accumulators",
           "merge_partial_grids", "TiledFrame", "Comm", "TorchComm", "EmulatedComm"]


def shard_bounds(n_segments: int, world: int) -> np.ndarray:
    """lv/voxelizer.py:461-463 `_chunk_bounds`: world+1 ascending bounds covering [0, n)."""
    world = max(1, min(int(world), max(1, int(n_segments))))
    return np.linspace(0, int(n_segments), world + 1).astype(np.int64)


def tile_rects(width: int, height: int, world: int) -> list:
    """Split the image into `world` horizontal strips (x0, y0, x1, y1), rows balanced to +-1.
    Strips keep each rank's pixels contiguous in the (H, W) image, so the gather is a concat."""
    ys = np.linspace(0, int(height), int(world) + 1).astype(np.int64)
    return [(0, int(ys[g]), int(width), int(ys[g + 1])) for g in range(int(world))]


def balanced_rows(bounds, weights, height: int) -> list:
    """New strip boundaries (world+1 ascending row indices, 0 .. height) that equalise the work per strip, given
    the work `weights[r]` measured on the strips `bounds[r] .. bounds[r+1]` of an earlier frame: the work is taken
    to be spread evenly over a strip's rows (a piecewise-constant density) and the cumulative density is cut
    into equal parts.  Every strip keeps at least one row.  Deterministic, so all ranks that feed it the same
    numbers get the same strips."""
    b = [int(x) for x in bounds]
    world = len(b) - 1
    w = [max(float(x), 0.0) for x in weights]
    total = sum(w)
    if world < 2 or total <= 0.0 or b[0] != 0 or b[-1] != int(height):
        return [int(x) for x in np.linspace(0, int(height), world + 1).astype(np.int64)]
    dens = [w[r] / max(b[r + 1] - b[r], 1) for r in range(world)]
    cum = np.zeros(int(height) + 1)
    for r in range(world):
        cum[b[r] + 1:b[r + 1] + 1] = cum[b[r]] + dens[r] * np.arange(1, b[r + 1] - b[r] + 1)
    out = [0]
    for k in range(1, world):
        row = int(np.searchsorted(cum, total * k / world, side="left"))
        row = min(max(row, out[-1] + 1), int(height) - (world - k))
        out.append(row)
    out.append(int(height))
    return out


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


class Comm:
    """What a TiledFrame needs from its peers.  This base class is the single-rank job."""
    rank, world = 0, 1

    def all_reduce_sum(self, t):
        """In-place sum of `t` over all ranks."""

    def gather(self, t):
        """Rank 0 gets [t of rank 0, t of rank 1, ...] (equal shapes); other ranks get None."""
        return [t]

    def barrier(self):
        pass

    def all_gather_value(self, x: float) -> list:
        """[x of rank 0, x of rank 1, ...] on every rank (host numbers; used once per frame for strip balancing)."""
        return [float(x)]


class TorchComm(Comm):
    """torch.distributed: NCCL over NVLink on GPUs, gloo in the CPU tests."""

    def __init__(self, group=None):
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            raise RuntimeError("TorchComm needs an initialised torch.distributed process group")
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def all_reduce_sum(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def gather(self, t):
        import torch
        if self.world == 1:
            return [t]
        outs = [torch.empty_like(t) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(t, outs, dst=0, group=self.group)
        return outs

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def all_gather_value(self, x: float) -> list:
        if self.world == 1:
            return [float(x)]
        out = [None] * self.world
        self.dist.all_gather_object(out, float(x), group=self.group)
        return [float(v) for v in out]


class EmulatedComm(Comm):
    """Rank `rank` of a `world`-rank job played on one device.  The all-reduce of the occupancy
    accumulators is replaced by `peers(t)`, a callback installed by TiledFrame that adds what the
    other ranks would have contributed (their segment shards, voxelized here); `gather` returns only
    this rank's piece.  Every kernel this rank would launch in the real job runs with the same
    arguments; only the NVLink exchange is missing, and its cost is reported as absent, not as zero."""
    emulated = True

    def __init__(self, rank: int, world: int):
        if not 0 <= int(rank) < int(world):
            raise ValueError("rank must be in [0, world)")
        self.rank, self.world = int(rank), int(world)
        self.peers = None

    def all_reduce_sum(self, t):
        if self.world > 1:
            if self.peers is None:
                raise RuntimeError("EmulatedComm has no peer contribution installed")
            self.peers(t)

    def gather(self, t):
        return [t] if self.rank == 0 else None

    def all_gather_value(self, x: float) -> list:
        """The ranks of an emulated job run one after the other, so a rank only learns its own number; the caller
        collects them (bench.py --emulate-world runs a first pass on equal strips for this)."""
        out = [0.0] * self.world
        out[self.rank] = float(x)
        return out


FIELD_LIMIT = 1 << 16      # a 16-bit field of the packed word


def field_bounds(wide_i64, packed_out=None):
    """int64[2] = {largest count, largest occupancy sum} of a rank's accumulators `(count << 32) | occ sum`
    (device kernel on CUDA tensors; torch ops on the CPU tensors of the gloo tests).  `packed_out` (CUDA, V int32):
    the packed words are written in the same pass over the accumulators."""
    import torch
    if wide_i64.is_cuda:
        from . import ops
        out = torch.empty(2, dtype=torch.int64, device=wide_i64.device)
        ops.wide_field_max(wide_i64, out, packed_out)
        return out
    return torch.stack([(wide_i64 >> 32).max(), (wide_i64 & 0xFFFFFFFF).max()])


def exchange_accumulators(wide_i64, comm, packed_scratch=None, widen_back=True):
    """The exchange step of a segment-sharded voxelization.  Returns (bytes every rank contributed, "packed" | "wide").

    The accumulators are 8 bytes per voxel.  Every rank first contributes the two maxima of its own fields to a
    16-byte all-reduce: their sums over the ranks bound every field of the merged grid, and while both bounds stay
    below 2^16 no packed field can carry into its neighbour or saturate -- the ranks then all-reduce the PACKED
    words (4 bytes per voxel, a plain integer sum).  Otherwise the accumulators themselves are
    summed.  All ranks see the same bounds, so they take the same branch; reading them is the one host
    synchronisation of the step (the collective synchronises the ranks anyway).

    "wide": `wide_i64` holds the sum over all ranks.  "packed": `packed_scratch` (CUDA; V int32) holds the merged
    PACKED grid, which is final -- nothing saturates below the bounds, so it is what packing the merged
    accumulators would give -- and, with `widen_back`, `wide_i64` holds the merged accumulators as well."""
    import torch
    n = wide_i64.numel()
    packed = None
    if wide_i64.is_cuda:     # the packed words come out of the same pass as the maxima (unused if the bounds fail)
        packed = packed_scratch if packed_scratch is not None else torch.empty(n, dtype=torch.int32, device=wide_i64.device)
    bounds = field_bounds(wide_i64, packed)
    comm.all_reduce_sum(bounds)
    if bool((bounds < FIELD_LIMIT).all().item()):
        if wide_i64.is_cuda:
            from . import ops
            comm.all_reduce_sum(packed)                      # int32 wraps like the u32 bit patterns it carries
            if widen_back:
                ops.widen(packed, None, wide_i64)
        else:
            packed, _ = pack_wide(wide_i64)
            comm.all_reduce_sum(packed)
            wide_i64.copy_(widen_packed(packed))
        return 4 * n, "packed"
    comm.all_reduce_sum(wide_i64)
    return 8 * n, "wide"


def merge_partial_grids(base_i32, group=None, comm=None):
    """All-reduce the per-rank packed grids exactly.  `base_i32`: this rank's finalized packed grid
    (int32 bit patterns, any device).  Returns (merged packed int32 grid, total visited)."""
    import torch.distributed as dist
    wide = widen_packed(base_i32)
    if comm is not None:
        comm.all_reduce_sum(wide)
    elif dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(wide, op=dist.ReduceOp.SUM, group=group)
    return pack_wide(wide)


class TiledFrame:
    """One frame rendered cooperatively by all ranks: segment-sharded voxelization + all-reduce of the
    occupancy accumulators, per-rank screen tile (tile-restricted A-buffer build and shading), gather
    of the tiles on rank 0.  Wraps a FrameEngine (or anything with its `run` signature and buffers).

    After `run`, `exchange_ms` is the device time of the all-reduce (None under emulation, where the
    time of the locally voxelized peer shards is reported as stage "emulated_peers" instead) and
    `exchange_bytes` the size of the buffer every rank contributed."""

    def __init__(self, engine, group=None, comm=None):
        if comm is None:
            import torch.distributed as dist
            comm = TorchComm(group) if (dist.is_available() and dist.is_initialized()) else Comm()
        self.engine, self.comm = engine, comm
        self.rank, self.world = comm.rank, comm.world
        self.tiles = tile_rects(engine.w, engine.h, self.world)
        self.exchange_ms = None
        self.exchange_bytes = 0
        self.exchange_kind = None        # "packed" (4 B per voxel) | "wide" (8 B per voxel), see exchange_accumulators
        self.packed_exchange = True
        self._ev = None
        if getattr(comm, "emulated", False):
            comm.peers = self._voxelize_peers

    def set_rows(self, bounds):
        """Use the horizontal strips bounds[r] .. bounds[r+1] (world+1 ascending rows, 0 .. height) from now on.
        Every rank of the job must be given the same bounds."""
        b = [int(x) for x in bounds]
        if len(b) != self.world + 1 or b[0] != 0 or b[-1] != self.engine.h or any(b[i + 1] <= b[i] for i in range(self.world)):
            raise ValueError("strip bounds must be world+1 strictly ascending rows from 0 to the image height")
        self.tiles = [(0, b[r], self.engine.w, b[r + 1]) for r in range(self.world)]

    def rows(self) -> list:
        return [t[1] for t in self.tiles] + [self.tiles[-1][3]]

    def rebalance(self, my_work: float):
        """Strip balancing from measured work: every rank contributes the work of its strip in the frame just
        rendered (e.g. the milliseconds of its strip-dependent stages: scan + scatter + shade + trace); the
        numbers are all-gathered (one host number per rank) and the strips of the following frames are cut so
        that each would have held the same share of it (`balanced_rows`).  Returns the new bounds."""
        w = self.comm.all_gather_value(my_work)
        if getattr(self.comm, "emulated", False):
            return self.rows()                   # one rank's number alone cannot rebalance; see bench.py
        b = balanced_rows(self.rows(), w, self.engine.h)
        self.set_rows(b)
        return b

    def seg_range(self):
        b = shard_bounds(self.engine._segs.numel(), self.world)
        return (int(b[self.rank]), int(b[self.rank + 1])) if self.rank < len(b) - 1 else (0, 0)

    def _voxelize_peers(self, wide):
        """EmulatedComm: what the other ranks' shards add to the accumulators (and to the incidence
        count, which the real job all-reduces with the grid)."""
        from . import ops
        eng = self.engine
        b = shard_bounds(eng._segs.numel(), self.world)
        for r in range(len(b) - 1):
            if r != self.rank and b[r + 1] > b[r]:
                ops.voxelize_wide(eng.lines, eng.res, eng.r_min, eng.method, wide, eng.stats, int(b[r]), int(b[r + 1]))

    def _merge(self, eng):
        import torch
        timed = eng.stats.is_cuda
        base_final = False
        if timed:
            if self._ev is None:
                self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            self._ev[0].record()
            self._ev[2].record()
        if eng.use_wide:     # the engine's 64-bit accumulators are sum-reducible as they are; it packs afterwards
            if self.packed_exchange and not getattr(self.comm, "emulated", False):
                # packed 4-byte words when a 16-byte pre-check proves that no field can overflow (exchange_accumulators)
                final = eng.stats.is_cuda and getattr(eng, "base", None) is not None     # a FrameEngine: its `base` receives the merged grid
                self.exchange_bytes, self.exchange_kind = exchange_accumulators(
                    eng.wide, self.comm, packed_scratch=eng.base if final else None, widen_back=not final)
                base_final = final and self.exchange_kind == "packed"
            else:
                self.exchange_bytes, self.exchange_kind = eng.wide.numel() * 8, "wide"
                self.comm.all_reduce_sum(eng.wide)
                if (self.packed_exchange and getattr(self.comm, "emulated", False) and eng.stats.is_cuda
                        and getattr(eng, "base", None) is not None):
                    # Emulation: the peers' shards were voxelized into `wide` above (that time is reported apart).
                    # What THIS rank does locally on the packed path -- the field maxima, the pack pass, an engine
                    # that takes `base` as final -- is run here as in the real job, so that the emulated per-rank
                    # times include it.  (The bounds are taken on the merged grid: at most the real job's.)
                    self._ev[2].record()
                    if bool((field_bounds(eng.wide, eng.base) < FIELD_LIMIT).all().item()):
                        self.exchange_bytes, self.exchange_kind, base_final = eng.wide.numel() * 4, "packed", True
        else:
            self.exchange_bytes = eng.base.numel() * 8
            merged, _ = merge_partial_grids(eng.base, comm=self.comm)
            eng.base.copy_(merged)
        if not getattr(self.comm, "emulated", False):
            from . import _native as N       # Σ incidences over the shards = `visited` of the whole set
            self.comm.all_reduce_sum(eng.stats[N.ST_VISITED:N.ST_VISITED + 1])
        if timed:
            self._ev[1].record()
        return "base_final" if base_final else None       # the engine then skips its pack pass (FrameEngine._stage_voxelize)

    def run(self, cam, grid, r_world):
        """This rank's part of the frame.  Returns the engine's FrameResult; its `stage_ms` gets an
        "exchange" entry (taken out of "voxelize") when the all-reduce was timed."""
        eng = self.engine
        out = eng.run(cam, grid, r_world, tile=self.tiles[self.rank], seg_range=self.seg_range(),
                      after_voxelize=self._merge if self.world > 1 else None)
        self.exchange_ms = None
        if self.world > 1 and self._ev is not None:
            emulated = getattr(self.comm, "emulated", False)
            # emulation: up to event 2 the peers' shards were voxelized here (not this rank's work); what follows it
            # -- the local passes of the packed exchange -- stays in "voxelize"
            ms = self._ev[0].elapsed_time(self._ev[2] if (emulated and self.exchange_kind == "packed") else self._ev[1])
            out.stage_ms["voxelize"] = max(0.0, out.stage_ms["voxelize"] - ms)
            if emulated:
                out.stage_ms["emulated_peers"] = ms
            else:
                out.stage_ms["exchange"] = self.exchange_ms = ms
        return out

    def gather_image(self):
        """Rank 0 receives the full sRGB image and hit ids (H, W, 3) u8 / (H, W) i32; others None."""
        import torch
        eng = self.engine
        x0, y0, x1, y1 = self.tiles[self.rank]
        if self.world == 1:
            return eng.srgb, eng.hit_id
        rows = max(t[3] - t[1] for t in self.tiles)
        pad_s = torch.zeros((rows, eng.w, 3), dtype=torch.uint8, device=eng.srgb.device)
        pad_h = torch.zeros((rows, eng.w), dtype=torch.int32, device=eng.srgb.device)
        pad_s[:y1 - y0] = eng.srgb[y0:y1]
        pad_h[:y1 - y0] = eng.hit_id[y0:y1]
        outs = self.comm.gather(pad_s)        # (strips may differ in height once they are balanced: padded to the tallest)
        outh = self.comm.gather(pad_h)
        if self.rank != 0:
            return None, None
        if getattr(self.comm, "emulated", False):       # only this rank's strip exists
            return pad_s[:y1 - y0], pad_h[:y1 - y0]
        srgb = torch.cat([o[:t[3] - t[1]] for o, t in zip(outs, self.tiles)], dim=0)
        hit = torch.cat([o[:t[3] - t[1]] for o, t in zip(outh, self.tiles)], dim=0)
        return srgb, hit
