"""FrameEngine: the device-resident, sync-free executor of one frame
(upload -> voxelize -> mips -> cull -> scan -> scatter/order -> shade -> trace).

It is what `ScenePipeline` and `bench.py` run.  All buffers are allocated once and reused;
every stage is enqueued on the current CUDA stream with a CUDA event between stages; the only
host synchronisation is the read-back of the 192-byte stats block (and of the image, when the
caller asks for it) at the end of the frame.  The fragment buffer is sized from the previous
frame's total with head-room; if a frame overflows it (or trips the 16-bit count fallback) the
affected stages are re-run -- exactness is never traded for the fast path.

Stage order and semantics follow lv/pipeline.py:68-136.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from . import ops
from .abuffer import ABufferError
from .grid import GridDesc, fit_grid
from .raytracer import RenderSettings, make_params
from .shading import AO_HALF_ANGLE, SHADOW_HALF_ANGLE, cone_directions

STAGES = ("upload", "voxelize", "mips", "cull", "scan", "scatter", "shade", "trace")


class FrameResult:
    def __init__(self, engine):
        self._e = engine
        self.stats = {}
        self.stage_ms = {}
        self.trace_kernel_ms = None

    @property
    def srgb_dev(self):
        return self._e.srgb

    @property
    def hit_id_dev(self):
        return self._e.hit_id

    @property
    def rgb_dev(self):
        return self._e.rgb


class FrameEngine:
    def __init__(self, res: int, width: int, height: int, strategy="vcsv", mode="opaque", alpha=1.0, k=8,
                 method="capsule", r_min=0.5, light=(-0.5, -0.3, -0.8), clip=True, keep_rgb=False,
                 early_termination=True, background=(0.1, 0.1, 0.12), device=None, frag_capacity=0,
                 shading="auto", builder=None):
        torch = N.require_cuda()
        if strategy not in ("vsv", "vcsv"):
            raise ValueError("strategy must be vsv or vcsv")
        if method not in ops.METHODS:
            raise ValueError(f"unknown voxelization method {method!r}")
        if shading not in ("auto", "demand", "all"):
            raise ValueError("shading must be auto, demand or all")
        # "demand": AO/shadow are cone-traced only for voxels a hit pixel interpolates (opaque mode;
        # identical image, `ao`/`shadow` then hold values only at those voxels).  "all": every
        # visible voxel, like lv/shading.py:170-185.  "auto" = demand for opaque, all for transparent.
        self.shading = ("demand" if mode == "opaque" else "all") if shading == "auto" else shading
        if self.shading == "demand" and mode != "opaque":
            raise ValueError("shading on demand needs opaque mode")
        if int(res) < 4 or int(res) & (int(res) - 1):
            raise ValueError(f"FrameEngine needs a power-of-two grid resolution >= 4, got {res}")
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.res, self.w, self.h = int(res), int(width), int(height)
        self.strategy, self.method, self.r_min, self.clip = strategy, method, float(r_min), bool(clip)
        self.settings = RenderSettings(mode=mode, alpha=alpha, k=k, background=tuple(background),
                                       early_termination=early_termination)
        l = np.asarray(light, dtype=np.float64)
        self.light = l / np.linalg.norm(l)
        self.light = self.light / np.linalg.norm(self.light)      # lv/shading.py:175 normalises again
        self.dirs = cone_directions()
        V = self.V = self.res ** 3
        d, t = self.dev, torch
        n_pyr = int(ops.level_offsets(self.res)[-1])
        self.stats = ops.new_stats(d)
        self.base = t.empty(V, dtype=t.int32, device=d)
        self.occ_sat = t.empty(max(V // 32, 1), dtype=t.int32, device=d)
        self.mips = t.empty(max(n_pyr - V, 1), dtype=t.float64, device=d)
        self.solid = t.empty(ops.cull_scratch_words(self.res), dtype=t.int32, device=d)
        self.vis_tmp = t.empty(V, dtype=t.uint8, device=d)
        self.cull_flat = t.empty(n_pyr, dtype=t.uint8, device=d)
        self.vis_list = t.empty(ops.list_words(V), dtype=t.int32, device=d)
        self.offsets = t.empty(V + 1, dtype=t.int32, device=d)
        self.cursor = t.empty(V, dtype=t.int32, device=d)
        self.scan_scratch = t.empty(ops.scan_scratch_bytes(V), dtype=t.uint8, device=d)
        self.shade_scratch = t.empty(ops.shade_scratch_bytes(V), dtype=t.uint8, device=d)
        self.ao = t.empty(V, dtype=t.float32, device=d)
        self.shadow = t.empty(V, dtype=t.float32, device=d)
        self.rgb = t.empty((self.h, self.w, 3), dtype=t.float64, device=d) if keep_rgb else None
        self.srgb = t.empty((self.h, self.w, 3), dtype=t.uint8, device=d)
        self.hit_id = t.empty((self.h, self.w), dtype=t.int32, device=d)
        self.frags = t.empty(max(int(frag_capacity), 1), dtype=t.int32, device=d)
        self.tight = ops.TightIndex(self.frags.numel(), V, d)
        self.march = t.empty(V, dtype=t.uint8, device=d)
        if self.shading == "demand":
            self.hit_t = t.empty((self.h, self.w), dtype=t.float64, device=d)
            self.need_bits = t.empty(max(V // 32, 1), dtype=t.int32, device=d)
            self.need_list = t.empty(ops.list_words(V), dtype=t.int32, device=d)
        self.wide = None
        self.nz_bits = None          # per-voxel "occupancy non-zero" bits from the pack pass (level-0 shading mask)
        self._nz_valid = False
        self._mip1_done = False
        # Accumulate into 64-bit (count << 32 | occ) words and pack afterwards (lvx_voxelize_wide +
        # lvx_pack_wide) instead of the packed 32-bit word with carry repair (lvx_voxelize).  The wide
        # form never needs the atomic's return value, so it compiles to fire-and-forget RED.64: measured
        # on B200, C2 voxelize 0.81 -> 0.68 ms and C4 12.8 -> 9.5 ms including the clear and the pack.
        # Same result bit for bit (per-field saturation, lv/voxelizer.py:490-495); False selects the packed path.
        self.use_wide = True
        self.lines = None
        self.grid = None
        self._verts32 = self._poly_off = None
        self._ev = [t.cuda.Event(enable_timing=True) for _ in range(len(STAGES) + 3)]
        self.launches_per_frame = 0
        # "all" shading can run beside the A-buffer build on a second stream.  Off by default: measured on
        # C3 (B200) the two only slow each other down (scatter 1.8 -> 4.4 ms, shade 2.9 -> 3.7 ms), the
        # frame time does not change and the per-stage times stop being readable.
        self.overlap_shading = False
        # brick size of the segment processing order (0 = polyline order).  Measured on B200: 8..32 are
        # within 2 % of each other on C2 (256^3), 32 is best on C4 (512^3): res / 16
        import os
        self.order_brick = min(int(os.environ.get("LVX_ORDER_BRICK", str(max(8, self.res // 16)))), self.res)
        self._order_shard = None
        self._stats_host = self._done = self._side = self._ev_side = self._pending = None
        self._geom_stats = self._geom_ms = None
        # tiled frames (`run(..., tile=rect)`): build the A-buffer only for the voxels the tile's rays can
        # visit (see _stage_owners).  False = replicate the whole build on every rank.
        self.tile_build = True
        self._owned = False
        self._sharded = False
        self._base_final = False
        self.owner_flat = self.owner_list = None
        self._overlapped = False
        # A-buffer build through per-brick segment lists (csrc/bricks.cu): opt-in (builder="bricks"), capsule traversal only
        self._bricks = ops.brick_lists_supported(method, self.res, builder)
        self._brick_scratch = None

    def kernel_launches_per_frame(self) -> int:
        """Number of lvx kernels one `run` enqueues (csrc/*.cu), for bench.py's `gpu_launches`."""
        levels = int(self.res).bit_length()

        def pyramid(first):     # one launch per level of more than 16^3 nodes, one for all the levels above
            big = sum(1 for l in range(first, levels) if (self.res >> l) > 16)
            return big + (1 if big < levels - first else 0)
        n = 1 + 1                                   # stats_reset, upload
        n += 3 if self.order_brick > 0 else 0       # processing order: histogram, scan, scatter
        n += 3 if (self.order_brick > 0 and self._sharded) else 0   # ... and the same for a rank's voxelization shard
        n += 2 if not self.use_wide else 2          # voxelize + finalize | voxelize_wide + pack_wide
        n += 1 if (self._base_final and self.res >= 64) else 0   # multi-GPU packed exchange: field maxima + pack, then level 1 + non-empty bits from the merged grid (instead of one fused pack pass)
        n += (0 if (self.use_wide and self.res >= 64) else 1) + pyramid(2)   # mips: level 1 (fused into the pack pass at res >= 64), then the rest
        n += (8 if self.strategy == "vcsv" else 1) + pyramid(1)   # solid, brick flags, super-brick flags, super-brick shadow, visibility, march probe, march, dilate | occupied; or-mips
        n += 1 + pyramid(1) if self._owned else 0   # tile owners + their OR pyramid
        n += 1                                      # scan
        n += (4 if self._bricks else 2) + 1         # bin count, alloc, fill, brick build | scatter, order (cursors from the scan); march table
        n += 1 + pyramid(1) + 1                     # non-empty masks (level 0, the rest), shade
        if self.shading == "demand":
            n += 3                                  # trace_hits, need list, resolve
        else:
            n += 1 + 1                              # shade fill, render
        return n

    # ------------------------------------------------------------------ line set
    def set_topology(self, polyline_offsets: np.ndarray, n_vertices: int):
        """Polyline structure is fixed across an animation; only vertex positions stream in."""
        t = self.torch
        self._poly_off = t.from_numpy(np.ascontiguousarray(polyline_offsets, dtype=np.int64)).to(self.dev)
        self._verts32 = t.empty((int(n_vertices), 3), dtype=t.float32, device=self.dev)
        self._verts64 = t.empty((int(n_vertices), 3), dtype=t.float64, device=self.dev)
        self._vertsf = t.empty((int(n_vertices), 3), dtype=t.float32, device=self.dev)
        self._normals = t.empty((int(n_vertices), 3), dtype=t.float64, device=self.dev) if self.clip else None
        self._segs = t.empty(int(n_vertices) - (len(polyline_offsets) - 1), dtype=t.int32, device=self.dev)
        # processing order of the segments (grouped by brick, csrc/upload.cu); results do not depend on it
        self._order = t.empty_like(self._segs) if self.order_brick > 0 else None
        self._order_scratch = (t.empty(ops.segment_order_scratch_words(self._segs.numel(), self.res, self.order_brick),
                                       dtype=t.int32, device=self.dev) if self.order_brick > 0 else None)

    def load_vertices(self, verts):
        """verts: (N,3) f32 -- pinned host tensor / numpy (H2D on the current stream) or cuda tensor."""
        t = self.torch
        if not t.is_tensor(verts):
            verts = t.from_numpy(np.ascontiguousarray(verts, dtype=np.float32))
        self._verts32.copy_(verts, non_blocking=True)

    def fit(self, radius_voxels=None, radius_world=None):
        """lv/grid.py:51-80 fit_grid with LineSet.aabb() (lv/lineset.py:81-82) reduced on the GPU (one
        24-byte read-back).  Exactly one of `radius_voxels` (the radius is re-derived from the voxel
        size) and `radius_world` (the line set's own radius) must be given."""
        if (radius_voxels is None) == (radius_world is None):
            raise ValueError("fit() needs exactly one of radius_voxels and radius_world")
        lo, hi = ops.aabb(self._verts32)

        class _L:
            radius = radius_world
        return fit_grid(_L, self.res, radius_voxels=radius_voxels, aabb=(lo, hi))

    # ------------------------------------------------------------------ stages
    def _stage_upload(self, grid: GridDesc, r_world: float):
        import ctypes as C
        wm = np.ascontiguousarray(grid.world_min, dtype=np.float64)
        N.check(N.lib().lvx_upload(ops._ptr(self._verts32), ops._ptr(self._poly_off),
                                   int(self._verts32.shape[0]), int(self._poly_off.shape[0]) - 1,
                                   wm.ctypes.data_as(C.c_void_p), float(grid.voxel_size),
                                   ops._ptr(self._verts64), ops._ptr(self._vertsf), ops._ptr(self._normals),
                                   ops._ptr(self._segs),
                                   ops._ptr(self.stats), ops._stream()), "lvx_upload")
        self.lines = ops.DeviceLines(self._verts32, self._poly_off, self._verts64, self._vertsf, self._normals,
                                     self._segs,
                                     int(self._verts32.shape[0]), int(self._poly_off.shape[0]) - 1,
                                     float(r_world) / float(grid.voxel_size), grid, float(r_world))
        self.grid = grid
        if self._order is not None:
            ops.segment_order(self.lines, self.res, self.order_brick, self._order, self._order_scratch)

    def _stage_voxelize(self, seg_range=None, after_voxelize=None):
        """`after_voxelize(engine)`: the multi-GPU exchange hook.  On the 64-bit path it runs between
        accumulation and packing and sums `engine.wide` across ranks (exact: per-field saturation
        comes after the sum, lv/voxelizer.py:490-495); on the packed path it runs on the finished `base`."""
        b, e = (0, self.lines.n_segments) if seg_range is None else seg_range
        self._sharded = self.use_wide and (b, e) != (0, self.lines.n_segments) and e > b
        if self.use_wide:
            if self.wide is None:
                self.wide = self.torch.empty(self.V, dtype=self.torch.int64, device=self.dev)
            ops.clear(self.wide)
            shard_order = None
            if self._order is not None and (b, e) != (0, self.lines.n_segments) and e > b:
                # a multi-GPU rank's shard of the canonical segment list, grouped by brick like the whole set
                if self._order_shard is None:
                    self._order_shard = self.torch.empty_like(self._order)
                ops.segment_order(self.lines, self.res, self.order_brick, self._order_shard, self._order_scratch,
                                  seg_range=(b, e))
                shard_order = self._order_shard
            ops.voxelize_wide(self.lines, self.res, self.r_min, self.method, self.wide, self.stats, b, e,
                              shard_order=shard_order)
            if after_voxelize is not None and after_voxelize(self) == "base_final":
                # the multi-GPU exchange summed PACKED words (no field could overflow): `base` is the merged,
                # final grid already -- no pack pass; level 1 and the non-empty bits come from `base`
                self._base_final = True
                if self.res >= 64:     # level 1 + the non-empty bits in one read of the merged grid
                    if self.nz_bits is None:
                        self.nz_bits = self.torch.empty(self.V // 32, dtype=self.torch.int32, device=self.dev)
                    ops.base_mip1(self.base, self.res, self.nz_bits, self.mips)
                    self._nz_valid = True
                    self._mip1_done = True
                else:
                    self._nz_valid = False
                    self._mip1_done = False
                return
            self._base_final = False
            if self.nz_bits is None and self.res >= 32:
                self.nz_bits = self.torch.empty(self.V // 32, dtype=self.torch.int32, device=self.dev)
            if self.res >= 64:     # pack + level 1 of the pyramid in one read of the accumulators
                ops.pack_wide_mip1(self.wide, self.res, self.base, self.stats, self.nz_bits, self.mips)
                self._mip1_done = True
            else:
                ops.pack_wide(self.wide, self.base, self.stats, self.nz_bits)
            self._nz_valid = self.nz_bits is not None
        else:
            self._nz_valid = False
            self._mip1_done = False
            ops.clear(self.base)
            ops.clear(self.occ_sat)
            ops.voxelize(self.lines, self.res, self.r_min, self.method, self.base, self.occ_sat, self.stats, b, e)
            ops.finalize_base(self.base, self.occ_sat, self.stats)
            if after_voxelize is not None:
                after_voxelize(self)

    def _stage_mips(self):
        if self._mip1_done:
            ops.build_mips_upper(self.res, self.mips)
        else:
            ops.build_mips(self.base, self.res, self.mips)

    def _stage_cull(self, cam):
        if self.strategy == "vcsv":
            ops.cull(self.base, self.res, self.grid.to_voxel(cam.position), self.solid, self.vis_tmp,
                     self.cull_flat, self.vis_list, self.stats)
        else:
            ops.occupied_pyramid(self.base, self.res, self.cull_flat, self.vis_list, self.stats)
        ops.march_levels(self.cull_flat, self.res, self.march)

    def _stage_owners(self, cam, tile):
        """Screen-tile ownership (multi-GPU screen tiles): the A-buffer build and all-voxel shading of
        this frame are restricted to the visible voxels the tile's rays can visit (lvx_tile_owners); the
        march bits stay the full culling pyramid, so the tile's pixels are the single-GPU frame's."""
        full = tile is None or tuple(tile) == (0, 0, self.w, self.h)
        self._owned = self.tile_build and not full
        if not self._owned:
            return
        t = self.torch
        if self.owner_flat is None:
            self.owner_flat = t.empty_like(self.cull_flat)
            self.owner_list = t.empty_like(self.vis_list)
        ops.tile_owners(self.cull_flat, self.res, ops.make_camera_struct(cam, self.grid), tile,
                        self.owner_flat, self.owner_list, self.stats)

    def _owner_bits(self):
        """(pyramid, list) of the voxels that own fragments this frame; pyramid None = every occupied voxel."""
        if self._owned:
            return self.owner_flat, self.owner_list
        return (self.cull_flat if self.strategy == "vcsv" else None), self.vis_list

    def _stage_scan(self):
        flat, _ = self._owner_bits()
        ops.scan(self.base, None if flat is None else flat[:self.V], self.offsets, self.scan_scratch, self.stats,
                 cursor=None if self._bricks else self.cursor)

    def _stage_scatter(self):
        rt = ops.footprint_radius(self.lines.r, self.r_min)
        flat, lst = self._owner_bits()
        if self._bricks:
            if self._brick_scratch is None:
                self._ensure_pairs(6 * self.lines.n_segments + 1024)
            ops.build_lists(self.lines, rt, self.res, flat, self.offsets, self.frags, self.stats,
                            self._brick_scratch, tight=self.tight)
            return
        ops.scatter(self.lines, rt, self.res, self.method, flat, lst,
                    self.offsets, self.cursor, self.frags, self.stats, tight=self.tight, cursor_ready=True)

    def _stage_shade(self):
        demand = self.shading == "demand"
        ops.shade(self.base, self.mips, self.res, self.need_list if demand else self._owner_bits()[1], self.dirs,
                  np.tan(AO_HALF_ANGLE), self.light, np.tan(SHADOW_HALF_ANGLE), self.ao, self.shadow,
                  self.shade_scratch, fill_ones=not demand, nz_bits=self.nz_bits if self._nz_valid else None)

    def _stage_trace(self, cam, tile=None):
        p = make_params(self.settings, self.lines, self.light, tile, self.w, self.h)
        ops.render(self.lines, self.offsets, self.frags, self.tight, self.march, self.res, self.ao, self.shadow,
                   ops.make_camera_struct(cam, self.grid), p, self.rgb, self.srgb, self.hit_id, self.stats)

    def _stage_trace_hits(self, cam, tile=None):
        p = make_params(self.settings, self.lines, self.light, tile, self.w, self.h)
        ops.trace_hits(self.lines, self.offsets, self.frags, self.tight, self.march, self.res,
                       ops.make_camera_struct(cam, self.grid), p, self.hit_t, self.hit_id, self.need_bits,
                       self.need_list, self.stats)

    def _stage_resolve(self, cam, tile=None):
        p = make_params(self.settings, self.lines, self.light, tile, self.w, self.h)
        ops.resolve(self.lines, self.march, self.res, self.ao, self.shadow,
                    ops.make_camera_struct(cam, self.grid), p, self.hit_t, self.hit_id, self.rgb, self.srgb)

    # ------------------------------------------------------------------ frame
    def _ensure_capacity(self, need: int):
        limit = ops.max_fragments()
        if need > limit:
            raise ABufferError(f"fragment total {need} exceeds the A-buffer limit of {limit} fragments")
        if need > self.frags.numel():
            cap = min(int(need * 1.25) + 1024, limit)      # head-room never pushes a valid total over the limit
            self.frags = self.torch.empty(cap, dtype=self.torch.int32, device=self.dev)
            self.tight = ops.TightIndex(cap, self.V, self.dev)

    def _ensure_pairs(self, need: int):
        if self._brick_scratch is None or need > self._brick_scratch.capacity:
            self._brick_scratch = None
            self._brick_scratch = ops.BrickScratch(self.res, int(need * 1.25) + 1024, self.dev)

    def run(self, cam, grid: GridDesc, r_world: float, tile=None, seg_range=None, after_voxelize=None,
            geometry=True):
        """One frame on the already loaded vertices.  `after_voxelize(engine)` is the hook where the
        multi-GPU path all-reduces the occupancy grid (distributed.py).  `geometry=False` keeps the
        grid, pyramid and uploaded line set of the previous frame and redoes only the camera-dependent
        stages (cull -> trace), like lv/pipeline.py:89-136 without cfg.revoxelize.  Returns FrameResult."""
        self.submit(cam, grid, r_world, tile, seg_range, after_voxelize, geometry)
        return self.collect()

    def run_geometry(self, grid: GridDesc, r_world: float, seg_range=None, after_voxelize=None):
        """lv/pipeline.py:68-87 build_geometry on the loaded vertices: upload + voxelize + mips, one
        sync.  Returns {"voxels_visited", "saturated", "upload_ms", "voxelize_ms", "mips_ms"}; later
        `run(..., geometry=False)` frames reuse the result."""
        t = self.torch
        self._prepare_host()
        ev = self._ev
        ops.stats_reset(self.stats)
        ev[0].record()
        self._stage_upload(grid, r_world); ev[1].record()
        self._stage_voxelize(seg_range, after_voxelize); ev[2].record()
        self._stage_mips(); ev[3].record()
        self._stats_host[:N.STATS_WORDS].copy_(self.stats, non_blocking=True)
        self._done.record()
        self._done.synchronize()
        st = self._stats_host.numpy().copy()
        if st[N.ST_NEED_WIDE] and not self.use_wide:
            self.use_wide = True
            return self.run_geometry(grid, r_world, seg_range, after_voxelize)
        self._check_lines(st)
        self._geom_stats = st[:N.STATS_WORDS].copy()
        self._geom_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        return {"voxels_visited": int(st[N.ST_VISITED]), "saturated": int(st[N.ST_SATURATED]),
                "upload_ms": self._geom_ms[0], "voxelize_ms": self._geom_ms[1], "mips_ms": self._geom_ms[2]}

    def _prepare_host(self):
        t = self.torch
        if self._stats_host is None:
            self._stats_host = t.empty(N.STATS_WORDS + 2, dtype=t.int64).pin_memory()
            self._done = t.cuda.Event()
            self._side = t.cuda.Stream(device=self.dev)
            self._ev_side = [t.cuda.Event(enable_timing=True) for _ in range(2)]

    @staticmethod
    def _check_lines(st):
        if st[N.ST_DEGENERATE]:
            from .lineset import LineSetError
            raise LineSetError(f"degenerate polyline {int(st[N.ST_DEGENERATE]) - 1}: all vertices coincide")

    def submit(self, cam, grid: GridDesc, r_world: float, tile=None, seg_range=None, after_voxelize=None,
               geometry=True):
        """Enqueue one frame on the current CUDA stream without waiting for it (`collect` does).
        Two engines on two streams can so keep two frames of a sequence in flight: the stages are
        latency-bound walks that leave issue slots free, and a second frame's kernels fill them."""
        if cam.width != self.w or cam.height != self.h:
            raise ValueError("camera size does not match the engine's image size")
        if not geometry and (self.lines is None or self._geom_stats is None):
            raise ValueError("geometry=False needs a previous run_geometry() / full frame")
        t = self.torch
        self._prepare_host()
        self._pending = (cam, grid, r_world, tile, seg_range, after_voxelize, geometry)
        ev = self._ev
        ops.stats_reset(self.stats)
        if geometry:
            ev[0].record()
            self._stage_upload(grid, r_world); ev[1].record()
            self._stage_voxelize(seg_range, after_voxelize)
            ev[2].record()
            self._stage_mips()
        ev[3].record()
        self._stage_cull(cam)
        self._stage_owners(cam, tile); ev[4].record()
        overlap = self.shading == "all" and self.overlap_shading
        if overlap:
            # cone tracing needs the pyramid and the visible-voxel list only: it runs beside the
            # A-buffer build on a second stream and joins before the trace
            main = t.cuda.current_stream()
            self._side.wait_event(ev[4])
            with t.cuda.stream(self._side):
                self._ev_side[0].record()
                self._stage_shade()
                self._ev_side[1].record()
        self._stage_scan(); ev[5].record()
        if self.frags.numel() <= 1:     # size the fragment buffer once; later frames reuse it with head-room
            self._ensure_capacity(int(self.stats[N.ST_FRAG_TOTAL].item()))
        self._stage_scatter(); ev[6].record()
        if self.shading == "demand":
            self._stage_trace_hits(cam, tile); ev[7].record()
            self._stage_shade(); ev[8].record()
            self._stage_resolve(cam, tile); ev[9].record()
            self._stats_host[N.STATS_WORDS:N.STATS_WORDS + 1].copy_(self.need_list[:2].view(t.int64), non_blocking=True)
        else:
            if overlap:
                main.wait_event(self._ev_side[1])
            else:
                self._stage_shade()
            ev[7].record()
            self._stage_trace(cam, tile); ev[8].record()
        self._stats_host[:N.STATS_WORDS].copy_(self.stats, non_blocking=True)
        self._done.record()
        self._overlapped = overlap

    def collect(self):
        """Wait for the submitted frame, check its status block (re-running the frame on the exact
        wide path or with a larger fragment buffer if it asked for that) and return its FrameResult."""
        ev = self._ev
        for attempt in range(4):
            self._done.synchronize()           # the frame's only mandatory sync
            st = self._stats_host.numpy().copy()
            geometry = self._pending[6]
            if geometry:
                self._geom_stats = st[:N.STATS_WORDS].copy()
            else:       # the voxelize-stage words of the frame that built the geometry
                for w in (N.ST_VISITED, N.ST_SATURATED, N.ST_NEED_WIDE, N.ST_DEGENERATE, N.ST_OCC_SAT):
                    st[w] = self._geom_stats[w]
            if st[N.ST_NEED_WIDE] and not self.use_wide:
                self.use_wide = True               # a 16-bit count wrapped: exact 64-bit path from now on
                self.submit(*self._pending)
                continue
            total = int(st[N.ST_FRAG_TOTAL])
            pairs = int(st[N.ST_BRICK_PAIRS]) if self._bricks else 0
            if total > self.frags.numel() or (self._bricks and pairs > self._brick_scratch.capacity):
                self._ensure_capacity(total)
                if self._bricks:
                    self._ensure_pairs(pairs)
                self.submit(*self._pending)
                continue
            break
        else:
            raise RuntimeError("frame did not converge")
        self._check_lines(st)
        if st[N.ST_MISMATCH] and st[N.ST_SATURATED] == 0:
            raise ABufferError("fragment count mismatch between passes (nondeterministic traversal?)")
        out = FrameResult(self)
        if geometry:
            self._geom_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        out.stage_ms = {s: (ev[i].elapsed_time(ev[i + 1]) if i >= 3 else (self._geom_ms[i] if geometry else 0.0))
                        for i, s in enumerate(STAGES)}
        out.trace_kernel_ms = out.stage_ms["trace"]
        if self.shading == "demand":   # events 6..9 bracket trace_hits, shade, resolve
            out.stage_ms["trace"] = ev[6].elapsed_time(ev[7]) + ev[8].elapsed_time(ev[9])
            out.stage_ms["shade"] = ev[7].elapsed_time(ev[8])
            out.trace_kernel_ms = ev[6].elapsed_time(ev[7])
            shaded = int(st[N.STATS_WORDS])
        else:
            if self._overlapped:   # shade ran beside scan+scatter: its own duration, and the join wait is not a stage
                out.stage_ms["shade"] = self._ev_side[0].elapsed_time(self._ev_side[1])
            shaded = int(st[N.ST_OWNED]) if self._owned else int(st[N.ST_VISIBLE])
        occ = int(st[N.ST_OCCUPIED])
        out.stats = {
            "segments": self.lines.n_segments, "vertices": self.lines.n_vertices, "resolution": self.res,
            "voxels_visited": int(st[N.ST_VISITED]), "saturated": int(st[N.ST_SATURATED]),
            "fragments": total, "fragment_touches": 2 * total, "solid_voxels": int(st[N.ST_SOLID]),
            "occupied_voxels": occ, "visible_voxels": int(st[N.ST_VISIBLE]),
            "culled_fraction": (1.0 - int(st[N.ST_VISIBLE]) / occ) if (self.strategy == "vcsv" and occ) else 0.0,
            "ray_capsule_tests": int(st[N.ST_RAY_TESTS]), "long_lists": int(st[N.ST_LONG_LISTS]),
            "occ_saturated_voxels": int(st[N.ST_OCC_SAT]), "wide_path": bool(self.use_wide),
            "shaded_voxels": shaded, "shading": self.shading,
            "owned_voxels": int(st[N.ST_OWNED]) if self._owned else int(st[N.ST_VISIBLE]),
        }
        out.raw_stats = [int(v) for v in st[:N.STATS_WORDS]]     # incl. the -DLVX_COUNT debug counters (words 11..15)
        return out
