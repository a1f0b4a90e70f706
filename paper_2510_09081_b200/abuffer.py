"""GPU A-buffer build with the reference's call surface (lv/abuffer.py:35-45: ``OffsetTable``,
``ABuffer``, ``ABufferError``, ``scan_offsets``, ``build_vsv``, ``build_vcsv``)."""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _native as N
from . import ops
from .culling import occupied_bits
from .voxelizer import METHODS, upload_lineset

__all__ = ["OffsetTable", "ABuffer", "ABufferError", "scan_offsets", "build_vsv", "build_vcsv"]


class ABufferError(RuntimeError):
    pass


class OffsetTable:
    """lv/abuffer.py:97-101.  `offsets_dev` has V+1 u32 entries (exclusive scan + total), so the
    masked count of voxel i is offsets[i+1]-offsets[i]."""

    def __init__(self, offsets_dev, total: int):
        self.offsets_dev, self.total = offsets_dev, int(total)
        self._h = None

    def _host(self):
        if self._h is None:
            self._h = self.offsets_dev.cpu().numpy().view(np.uint32).astype(np.int64)
        return self._h

    @property
    def offsets(self) -> np.ndarray:
        return self._host()[:-1]

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self._host())


def scan_offsets(pyramid, culling=None, capacity=None, _stats=None) -> OffsetTable:
    """lv/abuffer.py:104-114"""
    torch = N.require_cuda()
    base = pyramid.base_dev
    V = base.numel()
    if V >= 2 ** 32:
        raise ABufferError("grid too large")
    dev = base.device
    stats = ops.new_stats(dev) if _stats is None else _stats
    offsets = torch.empty(V + 1, dtype=torch.int32, device=dev)
    scratch = torch.empty(ops.scan_scratch_bytes(V), dtype=torch.uint8, device=dev)
    ops.scan(base, None if culling is None else culling.base_dev, offsets, scratch, stats)
    total = int(stats[N.ST_FRAG_TOTAL].item())
    if capacity is not None and total > capacity:
        raise ABufferError(f"fragment total {total} exceeds capacity {capacity}")
    if total > ops.max_fragments():
        raise ABufferError(f"fragment total {total} exceeds the A-buffer limit of {ops.max_fragments()} fragments")
    return OffsetTable(offsets, total)


class ABuffer:
    """lv/abuffer.py:117-138"""

    def __init__(self, table: OffsetTable, fragments_dev, resolution: int, stats: dict, tight=None,
                 tight_radius: float = -1.0):
        self.table, self.fragments_dev, self.resolution, self.stats = table, fragments_dev, resolution, stats
        # ops.TightIndex: per voxel, the fragments whose capsule of radius <= tight_radius can reach
        # into the voxel (ray-tracer acceleration, csrc/abuffer.cu); not part of the reference's ABuffer
        self.tight, self.tight_radius = tight, float(tight_radius)
        self._frags = None

    @property
    def total(self) -> int:
        return self.table.total

    @property
    def fragments(self) -> np.ndarray:
        if self._frags is None:
            self._frags = self.fragments_dev[:self.total].cpu().numpy().view(np.uint32)
        return self._frags

    def voxel_fragments(self, x: int, y: int, z: int) -> np.ndarray:
        idx = x + self.resolution * (y + self.resolution * z)
        o = self.table.offsets[idx]
        return self.fragments[o:o + self.table.counts[idx]]

    def dump(self, path) -> None:
        """ABUF dump, byte-compatible with lv/abuffer.py:133-138."""
        parts = [b"ABUF", struct.pack("<I", self.resolution ** 3),
                 self.table.offsets.astype("<u8").tobytes(), struct.pack("<I", self.total),
                 self.fragments.astype("<u4").tobytes()]
        Path(path).write_bytes(b"".join(parts))


def _second_pass(ls, cn, g, pyramid, culling, method, r_world):
    """lv/abuffer.py:281-328"""
    if method not in METHODS:
        raise ValueError(f"unknown voxelization method {method!r}")
    torch = N.require_cuda()
    lines = upload_lineset(ls, g, r_world, cn)
    res = g.resolution
    dev = lines.verts.device
    stats = ops.new_stats(dev)
    table = scan_offsets(pyramid, culling, _stats=stats)
    rt = ops.footprint_radius(lines.r, pyramid.r_min)
    frags = torch.empty(max(table.total, 1), dtype=torch.int32, device=dev)
    tight = ops.TightIndex(frags.numel(), res ** 3, dev)
    flat = None if culling is None else culling.flat_dev
    if ops.brick_lists_supported(method, res):     # capsule traversal: per-brick build, no atomics per incidence
        pairs = 6 * lines.n_segments + 1024
        while True:
            scratch = ops.BrickScratch(res, pairs, dev)
            ops.build_lists(lines, rt, res, flat, table.offsets_dev, frags, stats, scratch, tight=tight)
            st = stats.cpu().numpy()
            if int(st[N.ST_BRICK_PAIRS]) <= pairs:
                break
            pairs = int(st[N.ST_BRICK_PAIRS])
    else:
        cursor = torch.empty(res ** 3, dtype=torch.int32, device=dev)
        owners = culling if culling is not None else occupied_bits(pyramid)   # voxels that own fragments
        ops.scatter(lines, rt, res, method, flat, owners.list_dev,
                    table.offsets_dev, cursor, frags, stats, tight=tight)
        st = stats.cpu().numpy()
    if pyramid.saturated == 0 and st[N.ST_MISMATCH]:
        raise ABufferError("fragment count mismatch between passes (nondeterministic traversal?)")
    inc = table.total      # every scanned slot was written exactly once when there is no mismatch
    return ABuffer(table, frags, res, {"incidences": inc, "fragment_touches": 2 * inc,
                                       "fragments": table.total,
                                       "long_lists": int(st[N.ST_LONG_LISTS])},
                   tight=tight, tight_radius=float(lines.r))


def build_vsv(ls, cn, g, pyramid, method="capsule", workers=None, r_world=None) -> ABuffer:
    """lv/abuffer.py:331-334"""
    return _second_pass(ls, cn, g, pyramid, None, method, r_world)


def build_vcsv(ls, cn, g, pyramid, culling, method="capsule", workers=None, r_world=None) -> ABuffer:
    """lv/abuffer.py:337-340"""
    return _second_pass(ls, cn, g, pyramid, culling, method, r_world)
