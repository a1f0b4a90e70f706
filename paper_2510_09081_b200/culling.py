"""GPU camera-visibility culling with the reference's call surface (lv/culling.py:22-23:
``Camera``, ``CullingPyramid``, ``erode``, ``compute_visibility``, ``or_mips``, ``THETA_BLOCK``).

The reference pipeline computes ``eroded = erode(occ_levels[0])`` on the host and hands it to
``compute_visibility``; here erosion is fused with the 0.999 threshold into an integer bit mask
on the device (csrc/cull.cu), so ``erode`` returns a light handle that carries the packed base
words instead of a res^3 f64 field.  ``compute_visibility`` also accepts a plain numpy field
(it is quantised back to the packed representation, which is exact for fields produced by
``OccupancyPyramid.occ_levels[0]``).
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _native as N
from . import ops
from .camera import Camera
from .grid import GridDesc

__all__ = ["Camera", "CullingPyramid", "erode", "compute_visibility", "or_mips", "occupied_bits", "THETA_BLOCK"]

THETA_BLOCK = 0.999   # lv/culling.py:27 (compiled into csrc/cull.cu as occ_q >= 4092)


class CullingPyramid:
    """lv/culling.py:70-100.  `flat_dev`: all levels, u8, level 0 first (== packed())."""

    def __init__(self, flat_dev, resolution: int, list_dev=None):
        self.flat_dev, self._res, self._levels = flat_dev, int(resolution), None
        self.list_dev = list_dev   # compacted indices of the set base bits (include/lvx.h: vis_list)

    @classmethod
    def from_bits(cls, base) -> "CullingPyramid":
        """lv/culling.py:76-78 -- OR-mips of an arbitrary bit volume (numpy or cuda tensor)."""
        torch = N.require_cuda()
        b = base if torch.is_tensor(base) else torch.from_numpy(np.ascontiguousarray(base))
        res = int(b.shape[0])
        dev = torch.device("cuda", torch.cuda.current_device())
        offs = ops.level_offsets(res)
        flat = torch.zeros(int(offs[-1]), dtype=torch.uint8, device=dev)
        flat[:res ** 3] = (b.to(dev) != 0).reshape(-1).to(torch.uint8)
        # reuse the device OR-mip kernels by presenting the bits as counts in packed words
        words = flat[:res ** 3].to(torch.int32) << 16
        vis_list = torch.empty(ops.list_words(res ** 3), dtype=torch.int32, device=dev)
        ops.occupied_pyramid(words, res, flat, vis_list, ops.new_stats(dev))
        return cls(flat, res, vis_list)

    @property
    def resolution(self) -> int:
        return self._res

    @property
    def levels(self) -> list:
        if self._levels is None:
            h = self.flat_dev.cpu().numpy()
            offs = ops.level_offsets(self._res)
            self._levels = [h[offs[l]:offs[l + 1]].reshape((self._res >> l,) * 3)
                            for l in range(len(offs) - 1)]
        return self._levels

    @property
    def base(self) -> np.ndarray:
        return self.levels[0]

    @property
    def base_dev(self):
        return self.flat_dev[:self._res ** 3]

    def packed(self):
        """lv/culling.py:88-95"""
        offs = ops.level_offsets(self._res)
        res = np.array([self._res >> l for l in range(len(offs) - 1)], dtype=np.int64)
        return self.flat_dev.cpu().numpy(), offs, res

    def dump(self, path) -> None:
        """CULP dump, byte-compatible with lv/culling.py:97-100."""
        parts = [b"CULP", struct.pack("<I", self._res)] + [l.tobytes() for l in self.levels]
        Path(path).write_bytes(b"".join(parts))


def occupied_bits(pyramid) -> CullingPyramid:
    """CullingPyramid.from_bits(counts > 0) straight from the packed words on the device
    (lv/raytracer.py:665-668, lv/pipeline.py:115-116); cached on the pyramid."""
    cached = getattr(pyramid, "_occupied_bits", None)
    if cached is None:
        torch = N.require_cuda()
        res, base = pyramid.resolution, pyramid.base_dev
        flat = torch.empty(int(ops.level_offsets(res)[-1]), dtype=torch.uint8, device=base.device)
        vis_list = torch.empty(ops.list_words(res ** 3), dtype=torch.int32, device=base.device)
        ops.occupied_pyramid(base, res, flat, vis_list, ops.new_stats(base.device))
        cached = pyramid._occupied_bits = CullingPyramid(flat, res, vis_list)
    return cached


def or_mips(base) -> list:
    """lv/culling.py:103-109"""
    return CullingPyramid.from_bits(base).levels


class ErodedField:
    """Handle returned by `erode`: the packed base words the fused erode+threshold kernel reads."""

    def __init__(self, base_dev, resolution):
        self.base_dev, self.resolution = base_dev, resolution
        self.shape = (resolution,) * 3
        self.has_counts = True      # False for a plain occupancy field: `occupied` must then be given


def erode(field) -> ErodedField:
    """lv/culling.py:112-127.  Accepts an OccupancyPyramid (preferred, zero copy) or a cubic
    numpy field of clamped occupancies (quantised to 1/4096 like level 0 of the pyramid)."""
    torch = N.require_cuda()
    if hasattr(field, "base_dev"):
        return ErodedField(field.base_dev, field.resolution)
    f = np.asarray(field)
    res = f.shape[0]
    if f.shape != (res, res, res):
        raise ValueError("field must be cubic")
    # Only `eroded >= THETA_BLOCK` is ever consumed (lv/culling.py:186) and erosion (a neighbourhood min)
    # commutes with any monotone quantisation, so an arbitrary field is mapped onto the kernel's integer
    # predicate occ_q >= 4092 exactly: >= 0.999 -> 4096, below -> at most 4091.
    q = np.where(f >= THETA_BLOCK, 4096.0, np.minimum(np.floor(np.clip(f, 0.0, 1.0) * 4096.0), 4091.0)).astype(np.int32)
    dev = torch.device("cuda", torch.cuda.current_device())
    out = ErodedField(torch.from_numpy(q.reshape(-1)).to(dev), res)
    out.has_counts = False
    return out


def compute_visibility(eroded, g: GridDesc, cam: Camera, occupied=None) -> CullingPyramid:
    """lv/culling.py:203-225.  `eroded` is an ErodedField / OccupancyPyramid (the erosion is
    applied inside the kernel).  `occupied` defaults to count > 0 of the same words; a numpy
    bit volume overrides it."""
    torch = N.require_cuda()
    res = g.resolution
    if not isinstance(eroded, ErodedField):
        eroded = erode(eroded)
    if eroded.resolution != res or (occupied is not None and tuple(occupied.shape) != (res,) * 3):
        raise ValueError("field shape does not match grid")
    if occupied is None and not eroded.has_counts:
        raise ValueError("compute_visibility: `occupied` is required when `eroded` is a plain field "
                         "(lv/culling.py:203); only a pyramid handle carries the counts")
    base = eroded.base_dev
    dev = base.device
    if occupied is not None:
        occ = occupied if torch.is_tensor(occupied) else torch.from_numpy(np.ascontiguousarray(occupied))
        occ = (occ.to(dev).reshape(-1) != 0).to(torch.int32)
        base = (base & 0xFFFF) | (occ << 16)
    V = res ** 3
    stats = ops.new_stats(dev)
    solid = torch.empty(ops.cull_scratch_words(res), dtype=torch.int32, device=dev)
    vis = torch.empty(V, dtype=torch.uint8, device=dev)
    flat = torch.empty(int(ops.level_offsets(res)[-1]), dtype=torch.uint8, device=dev)
    vis_list = torch.empty(ops.list_words(V), dtype=torch.int32, device=dev)
    ops.cull(base, res, g.to_voxel(cam.position), solid, vis, flat, vis_list, stats)
    return CullingPyramid(flat, res, vis_list)
