"""Thin, allocation-explicit Python layer over the C ABI (``include/lvx.h``).

Every function takes torch CUDA tensors (device memory is PyTorch's job), enqueues one C-ABI
call on the current CUDA stream and returns without synchronising.  The reference-shaped API
(`voxelizer.py`, `culling.py`, ...) and the per-frame executor (`frame.py`) are built on these.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import check, lib

METHODS = {"dda": 0, "capsule": 1, "aabb": 2}          # lv/voxelizer.py:47


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dbl3(v):
    a = np.ascontiguousarray(v, dtype=np.float64)
    assert a.shape == (3,)
    return a, a.ctypes.data_as(C.c_void_p)


def num_levels(res: int) -> int:
    return int(res).bit_length()


def level_offsets(res: int) -> np.ndarray:
    sizes = [(res >> l) ** 3 for l in range(num_levels(res))]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def new_stats(device):
    import torch
    return torch.zeros(N.STATS_WORDS, dtype=torch.int64, device=device)


def stats_reset(stats):
    check(lib().lvx_stats_reset(_ptr(stats), _stream()), "lvx_stats_reset")


@dataclass
class DeviceLines:
    """A line set resident in HBM in the layout the kernels consume
    (lv/voxelizer.py:435-447 segment_arrays)."""
    verts32: "object"     # (Nv,3) f32 world
    poly_off: "object"    # (P+1,) i64
    verts: "object"       # (Nv,3) f64 voxel units
    verts_f: "object"     # (Nv,3) the same rounded to f32 (renderer pre-test)
    normals: "object"     # (Nv,3) f64 unit tangents, or None
    segs: "object"        # (N,) i32 ascending start-vertex ids
    n_vertices: int
    n_polylines: int
    r: float              # capsule radius, voxel units
    grid: "object"
    r_world: float
    order: "object" = None   # (N,) i32: `segs` grouped by brick (segment_order), the order the kernels process them in

    @property
    def proc_segs(self):
        return self.segs if self.order is None else self.order

    @property
    def n_segments(self) -> int:
        return self.n_vertices - self.n_polylines

    @property
    def use_clip(self) -> bool:
        return self.normals is not None


def upload(verts32, poly_off, grid, r_world, stats, with_normals=True, normals=None) -> DeviceLines:
    """lvx_upload.  verts32: cuda f32 (Nv,3); poly_off: cuda i64 (P+1,).  `normals`, when
    given (cuda f64 (Nv,3)), is used instead of computing tangents on the device."""
    import torch
    nv, npoly = int(verts32.shape[0]), int(poly_off.shape[0]) - 1
    dev = verts32.device
    verts = torch.empty((nv, 3), dtype=torch.float64, device=dev)
    verts_f = torch.empty((nv, 3), dtype=torch.float32, device=dev)
    segs = torch.empty(nv - npoly, dtype=torch.int32, device=dev)
    out_n = None
    if with_normals and normals is None:
        out_n = torch.empty((nv, 3), dtype=torch.float64, device=dev)
    wm, wm_p = _dbl3(grid.world_min)
    check(lib().lvx_upload(_ptr(verts32), _ptr(poly_off), nv, npoly, wm_p, float(grid.voxel_size),
                           _ptr(verts), _ptr(verts_f), _ptr(out_n), _ptr(segs), _ptr(stats), _stream()), "lvx_upload")
    if normals is not None:
        out_n = normals
    return DeviceLines(verts32, poly_off, verts, verts_f, out_n if with_normals else None, segs, nv, npoly,
                       float(r_world) / float(grid.voxel_size), grid, float(r_world))


def aabb(verts32):
    """LineSet.aabb() on the device -> (lo, hi) float64 numpy (synchronises)."""
    import torch
    out = torch.empty(6, dtype=torch.float32, device=verts32.device)
    check(lib().lvx_aabb(_ptr(verts32), int(verts32.shape[0]), _ptr(out), _stream()), "lvx_aabb")
    h = out.cpu().numpy().astype(np.float64)
    return h[:3], h[3:]


def segment_order_scratch_words(n_seg: int, res: int, brick: int) -> int:
    return int(lib().lvx_segment_order_scratch_words(int(n_seg), int(res), int(brick)))


def segment_order(lines: DeviceLines, res: int, brick: int, order, scratch, seg_range=None):
    """Fills `order` (i32, n_segments) with lines.segs grouped by brick and makes it the processing order.
    With `seg_range` = (b, e) only that shard of `segs` is ordered, into order[:e - b], and the whole-set
    processing order is left alone (a multi-GPU rank orders its own voxelization shard)."""
    if seg_range is not None:
        b, e = seg_range
        if e > b:
            check(lib().lvx_segment_order(_ptr(lines.verts), _ptr(lines.segs[b:e]), e - b, int(res), int(brick),
                                          _ptr(order), _ptr(scratch), _stream()), "lvx_segment_order")
        return
    check(lib().lvx_segment_order(_ptr(lines.verts), _ptr(lines.segs), lines.n_segments, int(res), int(brick),
                                  _ptr(order), _ptr(scratch), _stream()), "lvx_segment_order")
    lines.order = order


def footprint_radius(r: float, r_min: float = 0.5) -> float:
    """lv/voxelizer.py:450-458"""
    return max(r, r_min) + 0.5


def clear(t):
    check(lib().lvx_clear(_ptr(t), t.numel() * t.element_size(), _stream()), "lvx_clear")


def _shard_segs(lines: DeviceLines, seg_begin, seg_end):
    """The array a [seg_begin, seg_end) shard indexes.  The brick-grouped processing order is a
    different permutation on every rank (its ranks inside a brick come from atomics), so shards of a
    multi-GPU voxelization are cut from the canonical ascending `segs`; only a whole-set pass uses the
    processing order."""
    whole = seg_begin == 0 and seg_end == lines.n_segments
    return lines.proc_segs if whole else lines.segs


def voxelize(lines: DeviceLines, res, r_min, method, base, occ_sat, stats, seg_begin=0, seg_end=None):
    """lvx_voxelize into zeroed `base` (V i32) / `occ_sat` (V/32 i32)."""
    seg_end = lines.n_segments if seg_end is None else seg_end
    r = lines.r
    check(lib().lvx_voxelize(_ptr(lines.verts), _ptr(lines.normals), _ptr(_shard_segs(lines, seg_begin, seg_end)), seg_begin, seg_end,
                             int(lines.use_clip), r, footprint_radius(r, r_min), float(r_min), res,
                             METHODS[method], _ptr(base), _ptr(occ_sat), _ptr(stats), _stream()),
          "lvx_voxelize")


def voxelize_wide(lines: DeviceLines, res, r_min, method, wide, stats, seg_begin=0, seg_end=None, shard_order=None):
    """`shard_order` (optional i32 tensor): the segments of the shard [seg_begin, seg_end) in the order to process
    them in (segment_order(..., seg_range=...)); the kernel then walks shard_order[0 : seg_end - seg_begin]."""
    seg_end = lines.n_segments if seg_end is None else seg_end
    r = lines.r
    segs = _shard_segs(lines, seg_begin, seg_end)
    if shard_order is not None:
        segs, seg_begin, seg_end = shard_order, 0, seg_end - seg_begin
    check(lib().lvx_voxelize_wide(_ptr(lines.verts), _ptr(lines.normals), _ptr(segs), seg_begin,
                                  seg_end, int(lines.use_clip), r, footprint_radius(r, r_min), float(r_min),
                                  res, METHODS[method], _ptr(wide), _ptr(stats), _stream()),
          "lvx_voxelize_wide")


def widen(base, occ_sat, wide):
    check(lib().lvx_widen(_ptr(base), _ptr(occ_sat), base.numel(), _ptr(wide), _stream()), "lvx_widen")


def wide_field_max(wide, out2, packed=None):
    """out2 (device int64[2]) = {largest count, largest occupancy sum} of the 64-bit accumulators; `packed`
    (optional, V int32) receives the packed words in the same pass."""
    check(lib().lvx_wide_field_max(_ptr(wide), wide.numel(), _ptr(out2), _ptr(packed), _stream()), "lvx_wide_field_max")


def base_mip1(base, res, nz_bits, mips):
    """Level 1 of the pyramid + the non-zero bits from a packed grid (res >= 64); then build_mips_upper."""
    check(lib().lvx_base_mip1(_ptr(base), int(res), _ptr(nz_bits), _ptr(mips), _stream()), "lvx_base_mip1")


def pack_wide(wide, base, stats, nz_bits=None):
    """`nz_bits` (optional i32, V/32): receives one bit per voxel "occupancy non-zero" for `shade`."""
    check(lib().lvx_pack_wide(_ptr(wide), wide.numel(), _ptr(base), _ptr(nz_bits), _ptr(stats), _stream()), "lvx_pack_wide")


def pack_wide_mip1(wide, res, base, stats, nz_bits, mips):
    """pack_wide + level 1 of build_mips in one read of the accumulators (res >= 64); then build_mips_upper."""
    check(lib().lvx_pack_wide_mip1(_ptr(wide), int(res), _ptr(base), _ptr(nz_bits), _ptr(mips), _ptr(stats), _stream()),
          "lvx_pack_wide_mip1")


def build_mips_upper(res, mips):
    check(lib().lvx_build_mips_upper(int(res), _ptr(mips), _stream()), "lvx_build_mips_upper")


def finalize_base(base, occ_sat, stats):
    check(lib().lvx_finalize_base(_ptr(base), _ptr(occ_sat), base.numel(), _ptr(stats), _stream()),
          "lvx_finalize_base")


def build_mips(base, res, mips):
    check(lib().lvx_build_mips(_ptr(base), res, _ptr(mips), _stream()), "lvx_build_mips")


def cull_scratch_words(res: int) -> int:
    return int(lib().lvx_cull_scratch_words(res))


def list_words(n_voxels: int) -> int:
    return int(lib().lvx_list_words(n_voxels))


def cull(base, res, cam_voxel, solid_bits, vis_tmp, cull_flat, vis_list, stats):
    cv, cv_p = _dbl3(cam_voxel)
    check(lib().lvx_cull(_ptr(base), res, cv_p, _ptr(solid_bits), _ptr(vis_tmp), _ptr(cull_flat),
                         _ptr(vis_list), _ptr(stats), _stream()), "lvx_cull")


def occupied_pyramid(base, res, cull_flat, vis_list, stats):
    check(lib().lvx_occupied_pyramid(_ptr(base), res, _ptr(cull_flat), _ptr(vis_list), _ptr(stats),
                                     _stream()), "lvx_occupied_pyramid")


TILE_MARGIN = 1.5 + 1e-3   # voxels: the visited voxel's cube + the 8 trilinear AO/shadow taps of a hit in it


def tile_owners(cull_flat, res, cam_struct, tile, owner_flat, owner_list, stats, margin=TILE_MARGIN):
    """lvx_tile_owners: the visible voxels a rank tracing pixel rect `tile` = (x0, y0, x1, y1) needs."""
    x0, y0, x1, y1 = (int(v) for v in tile)
    check(lib().lvx_tile_owners(_ptr(cull_flat), res, C.byref(cam_struct), x0, y0, x1, y1, float(margin),
                                _ptr(owner_flat), _ptr(owner_list), _ptr(stats), _stream()), "lvx_tile_owners")


def scan_scratch_bytes(n_voxels: int) -> int:
    return int(lib().lvx_scan_scratch_bytes(n_voxels))


def scan(base, cull_base, offsets, scratch, stats, cursor=None):
    """`cursor` (optional, V i32): also written by the scan (pass cursor_ready=True to `scatter`)."""
    check(lib().lvx_scan(_ptr(base), _ptr(cull_base), base.numel(), _ptr(offsets), _ptr(scratch),
                         _ptr(stats), _ptr(cursor), _stream()), "lvx_scan")


TIGHT_MARGIN = 1e-3   # voxels; see csrc/abuffer.cu "Loose bits"


def max_fragments() -> int:
    """Largest fragment total / capacity lvx_scatter accepts (cursor values above it mark culled voxels)."""
    return int(lib().lvx_max_fragments())


class TightIndex:
    """Per-voxel index of the fragments whose capsule can reach into the voxel (csrc/abuffer.cu): the
    ordering pass compacts them to the front of each list's range.  `frags` i32 [capacity],
    `slot` i16 [capacity] (position in the full list), `cnt` i16 [V].  An acceleration structure
    for the ray tracer only; the reference's `fragments` array is untouched."""

    def __init__(self, capacity: int, n_voxels: int, device):
        import torch
        self.capacity = int(capacity)
        self.frags = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=device)
        self.slot = torch.empty(max(self.capacity, 1), dtype=torch.int16, device=device)
        # zeroed once: the tracer fetches cnt[v] together with the march byte of EVERY voxel it steps through
        # and only uses it where the voxel is listed (which the ordering pass has written)
        self.cnt = torch.zeros(int(n_voxels), dtype=torch.int16, device=device)

    def ptrs(self):
        return _ptr(self.frags), _ptr(self.slot), _ptr(self.cnt)


def _tight_ptrs(tight):
    return (None, None, None) if tight is None else tight.ptrs()


def scatter(lines: DeviceLines, rt, res, method, cull_flat, vis_list, offsets, cursor, frags, stats, tight=None,
            cursor_ready=False):
    """`tight` (optional TightIndex with capacity >= frags.numel()) receives the index of the fragments whose
    capsule of radius lines.r can reach into their voxel, for the ray tracer."""
    if tight is not None and tight.capacity < frags.numel():
        raise ValueError("tight index too small for the fragment buffer")
    tf, ts, tc = _tight_ptrs(tight)
    check(lib().lvx_scatter(_ptr(lines.verts), _ptr(lines.proc_segs), lines.n_segments, float(rt),
                            float(lines.r) + TIGHT_MARGIN, res,
                            METHODS[method], _ptr(cull_flat), _ptr(vis_list), _ptr(offsets), _ptr(cursor),
                            _ptr(frags), frags.numel(), tf, ts, tc, int(bool(cursor_ready)), _ptr(stats), _stream()),
          "lvx_scatter")


BRICK = 8     # csrc/bricks.cu


def brick_lists_supported(method, res, builder=None) -> bool:
    """The brick-binned build (lvx_build_lists, csrc/bricks.cu) covers the capsule traversal on grids of at least
    one brick.  It is the OPT-IN builder (`builder="bricks"` / LVX_BUILDER=bricks): same fragments bit for bit, but
    measured slower than the scatter + ordering passes on one B200, which stay the default."""
    import os
    builder = builder or os.environ.get("LVX_BUILDER", "scatter")
    if builder not in ("scatter", "bricks"):
        raise ValueError(f"unknown A-buffer builder {builder!r}")
    return builder == "bricks" and method == "capsule" and res >= BRICK


class BrickScratch:
    """Scratch of lvx_build_lists: per-brick counters and the (segment, brick) pair array."""

    def __init__(self, res: int, pair_capacity: int, device):
        import torch
        self.res, self.capacity = int(res), int(pair_capacity)
        self.words = torch.empty(int(lib().lvx_brick_scratch_words(self.res, self.capacity)), dtype=torch.int32,
                                 device=device)


def build_lists(lines: DeviceLines, rt, res, cull_flat, offsets, frags, stats, scratch: BrickScratch, tight=None):
    """lv/abuffer.py:195-255, 281-328 through per-brick segment lists (csrc/bricks.cu).  The caller checks
    stats[ST_BRICK_PAIRS] <= scratch.capacity (else nothing was built: grow the scratch and call again)."""
    if tight is not None and tight.capacity < frags.numel():
        raise ValueError("tight index too small for the fragment buffer")
    tf, ts, tc = _tight_ptrs(tight)
    check(lib().lvx_build_lists(_ptr(lines.verts), _ptr(lines.proc_segs), lines.n_segments, float(rt),
                                float(lines.r) + TIGHT_MARGIN, res, _ptr(cull_flat), _ptr(offsets),
                                _ptr(frags), frags.numel(), tf, ts, tc, _ptr(scratch.words), scratch.capacity,
                                _ptr(stats), _stream()), "lvx_build_lists")


def march_levels(bits_flat, res, march):
    check(lib().lvx_march_levels(_ptr(bits_flat), res, _ptr(march), _stream()), "lvx_march_levels")


def shade_scratch_bytes(n_voxels: int) -> int:
    return int(lib().lvx_shade_scratch_bytes(n_voxels))


def shade(base, mips, res, vis_list, dirs, tan_ao, light, tan_shadow, ao, shadow, scratch, fill_ones=True, nz_bits=None):
    d = np.ascontiguousarray(dirs, dtype=np.float64)
    l, l_p = _dbl3(light)
    check(lib().lvx_shade(_ptr(base), _ptr(mips), res, _ptr(vis_list), d.ctypes.data_as(C.c_void_p),
                          int(d.shape[0]), float(tan_ao), l_p, float(tan_shadow), _ptr(ao), _ptr(shadow),
                          int(bool(fill_ones)), _ptr(nz_bits), _ptr(scratch), _stream()), "lvx_shade")


def make_camera_struct(cam, grid) -> N.lvx_camera:
    c = N.lvx_camera()
    c.pos[:] = [float(x) for x in grid.to_voxel(cam.position)]       # lv/raytracer.py:690
    c.fwd[:] = [float(x) for x in cam.forward]
    c.right[:] = [float(x) for x in cam.right]
    c.up[:] = [float(x) for x in cam.up]
    c.tan_half_fov = float(np.tan(cam.fov / 2.0))                     # lv/raytracer.py:695
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def render(lines: DeviceLines, offsets, frags, tight, march, res, ao, shadow, cam_struct, params, rgb, srgb,
           hit_id, stats):
    tf, ts, tc = _tight_ptrs(tight)
    check(lib().lvx_render(_ptr(lines.verts), _ptr(lines.verts_f), _ptr(lines.normals), _ptr(offsets), _ptr(frags),
                           tf, ts, tc, _ptr(march), res, _ptr(ao), _ptr(shadow), C.byref(cam_struct), C.byref(params), _ptr(rgb),
                           _ptr(srgb), _ptr(hit_id), _ptr(stats), _stream()), "lvx_render")


def trace_hits(lines: DeviceLines, offsets, frags, tight, march, res, cam_struct, params, hit_t, hit_id, need_bits,
               need_list, stats):
    tf, ts, tc = _tight_ptrs(tight)
    check(lib().lvx_trace_hits(_ptr(lines.verts), _ptr(lines.verts_f), _ptr(lines.normals), _ptr(offsets), _ptr(frags),
                               tf, ts, tc, _ptr(march), res, C.byref(cam_struct), C.byref(params), _ptr(hit_t), _ptr(hit_id),
                               _ptr(need_bits), _ptr(need_list), _ptr(stats), _stream()), "lvx_trace_hits")


def resolve(lines: DeviceLines, march, res, ao, shadow, cam_struct, params, hit_t, hit_id, rgb, srgb):
    check(lib().lvx_resolve(_ptr(lines.verts), _ptr(lines.normals), _ptr(march), res, _ptr(ao), _ptr(shadow),
                            C.byref(cam_struct), C.byref(params), _ptr(hit_t), _ptr(hit_id), _ptr(rgb), _ptr(srgb),
                            _stream()), "lvx_resolve")
