/*
 * lvx.h -- C ABI of liblvx_b200.so: the B200-native (sm_100a) per-frame pipeline of
 * arXiv 2510.09081 (voxel ray tracing of dynamic line sets).
 *
 * The reference package has no FFI; its boundary is the Python function surface re-exported
 * by pkg/src/linevox/__init__.py:9-21, whose hot loops are numba kernels with flat-array,
 * C-style signatures.  Each entry point below replaces one of those kernels (cited as
 * lv/<file>:<line> = /root/reference/pkg/src/linevox/<file>).  INTEGRATION.md shows the
 * ctypes binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless its name ends in `_host`.  The library never
 *    allocates or frees caller-visible memory; scratch is passed in (sizes from the
 *    lvx_*_scratch_bytes helpers).  All work is enqueued on `stream` (a cudaStream_t passed as
 *    void*); nothing synchronises unless stated.
 *  - Volumes are x-fastest: flat index = x + res*(y + res*z)            (lv/grid.py:3-5,46-48)
 *  - Packed base word = (count << 16) | occ_q, occ_q = round(occ*4096)   (lv/voxelizer.py:328-340)
 *  - Pyramids are stored flat, level 0 first: offsets 0, res^3, res^3+(res/2)^3, ...
 *  - Return value: 0 = ok, <0 = error (LVX_E_*).  Data-dependent conditions (count mismatch,
 *    degenerate polyline, 16-bit count overflow) are reported through the `stats` block, which
 *    the caller reads back when it needs them.
 *  - All arithmetic that decides voxel membership is IEEE f64 without FMA contraction, in the
 *    reference's operation order, so integer outputs are bit-identical to the reference.
 */
#ifndef LVX_H
#define LVX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LVX_OK 0
#define LVX_E_ARG (-1)   /* invalid argument (bad method, res not a power of two, ...)      */
#define LVX_E_CUDA (-2)  /* a CUDA runtime call failed; lvx_last_cuda_error() has the text   */

/* indices into the uint64 stats block (device memory, LVX_STATS_WORDS words, zeroed by
 * lvx_stats_reset) */
enum {
    LVX_ST_VISITED = 0,      /* in-grid capsule-voxel incidences (lv/voxelizer.py:492 `visited`) */
    LVX_ST_SATURATED = 1,    /* count increments beyond 0xFFFF (lv/voxelizer.py:333-336), wide path */
    LVX_ST_NEED_WIDE = 2,    /* !=0: a 16-bit count field wrapped in lvx_voxelize; redo with lvx_voxelize_wide */
    LVX_ST_SOLID = 3,        /* voxels whose eroded occupancy >= 0.999 (lv/culling.py:27,186) */
    LVX_ST_FRAG_TOTAL = 4,   /* total fragments = OffsetTable.total (lv/abuffer.py:109) */
    LVX_ST_MISMATCH = 5,     /* !=0: second traversal disagreed with scanned counts (lv/abuffer.py:310-311) */
    LVX_ST_RAY_TESTS = 6,    /* ray-capsule tests (lv/raytracer.py:445,575,706) */
    LVX_ST_LONG_LISTS = 7,   /* voxels whose fragment list needed the block-wide sort */
    LVX_ST_DEGENERATE = 8,   /* !=0: 1 + index of a polyline whose vertices all coincide (lv/lineset.py:237) */
    LVX_ST_VISIBLE = 9,      /* visible voxels = culling.base.sum() */
    LVX_ST_OCCUPIED = 10,    /* voxels with count > 0 */
    LVX_ST_OCC_SAT = 11,     /* voxels whose 16-bit occupancy sum saturated */
    LVX_ST_TILE_CURSOR = 12, /* scratch: pixel-tile queue of the persistent trace kernels (reset by every launch) */
    LVX_ST_OWNED = 13,       /* voxels a screen tile owns (lvx_tile_owners) */
    LVX_ST_BRICK_PAIRS = 16, /* (segment, brick) pairs lvx_build_lists needs; > its pair_capacity: nothing was built, redo */
    LVX_STATS_WORDS = 24
};

typedef struct lvx_camera {
    double pos[3];    /* voxel units: GridDesc.to_voxel(cam.position)  (lv/raytracer.py:690) */
    double fwd[3], right[3], up[3];                                  /* lv/culling.py:53-58 */
    double tan_half_fov;                                             /* lv/raytracer.py:695 */
    int32_t width, height;
} lvx_camera;

typedef struct lvx_render_params {
    int32_t mode;              /* 0 opaque (lv/raytracer.py:459), 1 transparent (518) */
    int32_t k;                 /* transparent k-buffer slots, 1..64 (lv/raytracer.py:64) */
    int32_t early_termination; /* lv/raytracer.py:57 */
    int32_t use_clip;          /* clip planes active (normals given)  */
    double alpha;              /* (0,1] */
    double background[3];      /* lv/raytracer.py:56 */
    double light_to_source[3]; /* = -light_dir (lv/raytracer.py:689) */
    double radius;             /* capsule radius, voxel units (geometric r, lv/raytracer.py:675) */
    int32_t tile_x0, tile_y0, tile_x1, tile_y1; /* pixel rect to trace, [x0,x1) x [y0,y1); multi-GPU screen tiles */
} lvx_render_params;

const char *lvx_last_cuda_error(void);
int lvx_version(void);
int lvx_stats_reset(uint64_t *stats, void *stream);

/* number of pyramid levels (log2(res)+1) and flat size in elements of an all-level pyramid */
int lvx_num_levels(int res);
int64_t lvx_pyramid_elems(int res);

/* ---- line-set upload: lv/voxelizer.py:435-447 segment_arrays, lv/lineset.py:74-79
 * segment_vertex_ids, lv/lineset.py:213-242 compute_clip_normals.
 * verts_f32 (n_verts*3, world), poly_off (n_poly+1).  Outputs: verts (voxel-unit f64,
 * n_verts*3), verts_f (the same rounded to f32, n_verts*3; may be NULL; read only by the renderer's
 * conservative pre-test), normals (unit tangents f64, n_verts*3; may be NULL to skip), segs (start-vertex
 * id of each of the n_verts-n_poly segments, ascending, int32). */
int lvx_upload(const float *verts_f32, const int64_t *poly_off, int64_t n_verts, int64_t n_poly,
               const double *world_min_host, double voxel_size,
               double *verts, float *verts_f, double *normals, int32_t *segs, uint64_t *stats, void *stream);

/* Processing order for lvx_voxelize* / lvx_scatter: `order` = the entries of `segs` grouped by the
 * brick (brick^3 voxels, brick a power of two) of their start vertex.  Both consumers produce the same
 * output for any order of the segments (the reference's results are independent of its chunking,
 * lv/voxelizer.py:461-463); grouping makes neighbouring threads touch the same sectors.
 * scratch: lvx_segment_order_scratch_words(n_seg, res, brick) u32. */
int64_t lvx_segment_order_scratch_words(int64_t n_seg, int res, int brick);
int lvx_segment_order(const double *verts, const int32_t *segs, int64_t n_seg, int res, int brick,
                      int32_t *order, uint32_t *scratch, void *stream);

/* lv/lineset.py:81-82 LineSet.aabb(): out6 = {min xyz, max xyz} as f32 (device). */
int lvx_aabb(const float *verts_f32, int64_t n_verts, float *out6, void *stream);

/* ---- voxelize: lv/voxelizer.py:301-340 _voxelize_kernel (+ the merge at 490-495).
 * method 0 dda / 1 capsule / 2 aabb (lv/voxelizer.py:47).  `base` (V u32) and `occ_sat`
 * (V/32 u32 bit mask) must be zero on entry (lvx_clear does it).  seg_begin/seg_end select a
 * contiguous shard of `segs` (multi-GPU segment sharding; lv/voxelizer.py:461-463). */
int lvx_clear(void *ptr, int64_t bytes, void *stream);
int lvx_voxelize(const double *verts, const double *normals, const int32_t *segs,
                 int64_t seg_begin, int64_t seg_end, int use_clip, double r, double rt, double r_min,
                 int res, int method, uint32_t *base, uint32_t *occ_sat, uint64_t *stats, void *stream);
/* exact 64-bit accumulators ((count << 32) | occ_sum per voxel); used when LVX_ST_NEED_WIDE is
 * raised and as the multi-GPU exchange format (sum-reducible). */
int lvx_voxelize_wide(const double *verts, const double *normals, const int32_t *segs,
                      int64_t seg_begin, int64_t seg_end, int use_clip, double r, double rt, double r_min,
                      int res, int method, uint64_t *wide, uint64_t *stats, void *stream);
/* packed (+occ_sat) -> wide, so that per-GPU partial grids can be all-reduced with a plain sum */
int lvx_widen(const uint32_t *base, const uint32_t *occ_sat, int64_t n_voxels, uint64_t *wide, void *stream);
/* out2 (device, 2 x u64) = {largest count, largest occupancy sum} of the accumulators.  Multi-GPU exchange: the
 * sums of these maxima over the ranks bound every field of the merged grid; while both stay below 65536 the ranks
 * can all-reduce the PACKED words (lvx_pack_wide, 4 bytes per voxel: no field can carry into the other or saturate)
 * instead of the accumulators (8 bytes per voxel), and lvx_widen the sum back. */
int lvx_wide_field_max(const uint64_t *wide, int64_t n_voxels, uint64_t *out2,
                       uint32_t *packed /* may be NULL; n_voxels u32: also receives the packed words, same pass */,
                       void *stream);
/* level 1 of the pyramid (at the start of `mips`, as lvx_build_mips writes it) and the "occupancy non-zero" bits
 * from a PACKED grid -- lvx_pack_wide_mip1 without the pack, for a grid that arrives packed (the merged grid of a
 * packed multi-GPU exchange).  res >= 64; follow with lvx_build_mips_upper. */
int lvx_base_mip1(const uint32_t *base, int res, uint32_t *nz_bits /* may be NULL */, double *mips, void *stream);
/* wide -> packed with per-field saturation (lv/voxelizer.py:493-495); adds to LVX_ST_SATURATED */
int lvx_pack_wide(const uint64_t *wide, int64_t n_voxels, uint32_t *base,
                  uint32_t *nz_bits /* may be NULL; n_voxels/32 u32: bit = occupancy field non-zero, for lvx_shade */,
                  uint64_t *stats, void *stream);
/* lvx_pack_wide and level 1 of lvx_build_mips in one read of the accumulators (res >= 64, else LVX_E_ARG):
 * `mips` receives level 1 at its start, exactly as lvx_build_mips writes it; follow with lvx_build_mips_upper. */
int lvx_pack_wide_mip1(const uint64_t *wide, int res, uint32_t *base, uint32_t *nz_bits /* may be NULL */,
                       double *mips, uint64_t *stats, void *stream);
/* applies occ_sat to `base` in place (occ field := 0xFFFF where flagged) */
int lvx_finalize_base(uint32_t *base, const uint32_t *occ_sat, int64_t n_voxels, uint64_t *stats, void *stream);

/* ---- occupancy pyramid: lv/voxelizer.py:422-432 build_mips.  Level 0 is implied by `base`
 * (min(occ_q,4096)/4096); `mips` receives levels 1.. as f64, flat, level 1 first
 * (lvx_pyramid_elems(res) - res^3 elements).  Values are exact dyadic rationals. */
int lvx_build_mips(const uint32_t *base, int res, double *mips, void *stream);
/* levels 2.. from a level 1 that is already in `mips` (lvx_pack_wide_mip1) */
int lvx_build_mips_upper(int res, double *mips, void *stream);

/* ---- culling: lv/culling.py:112-127 erode, 143-200 _march_blocked/_visibility_kernel,
 * 130-140 dilate_bits, 103-109 or_mips.  cull_flat (lvx_pyramid_elems(res) bytes) receives the
 * u8 visibility pyramid (CullingPyramid.packed()).  solid_bits: lvx_cull_scratch_words(res) u32
 * of scratch (per-voxel solid bits + coarse brick flags); vis_tmp: V bytes scratch.  cam_voxel_host = GridDesc.to_voxel(cam.position). */
int64_t lvx_cull_scratch_words(int res);
int lvx_cull(const uint32_t *base, int res, const double *cam_voxel_host,
             uint32_t *solid_bits, uint8_t *vis_tmp, uint8_t *cull_flat, uint32_t *vis_list,
             uint64_t *stats, void *stream);
/* march bits for the un-culled strategy: CullingPyramid.from_bits(counts > 0)
 * (lv/raytracer.py:665-668, lv/pipeline.py:115-116) */
int lvx_occupied_pyramid(const uint32_t *base, int res, uint8_t *cull_flat, uint32_t *vis_list,
                         uint64_t *stats, void *stream);
/* Both calls also emit `vis_list`: lvx_list_words(V) u32 words -- word 0..1 = number of set base
 * bits (u64), entries (flat voxel indices, unordered) from word 16.  The A-buffer ordering pass
 * and the shading kernel iterate this list instead of the whole volume. */
int64_t lvx_list_words(int64_t n_voxels);

/* ---- screen-tile ownership (multi-GPU screen tiles; no counterpart in the reference, whose only
 * decomposition is by segment chunk, lv/voxelizer.py:461-463).  owner_flat (lvx_pyramid_elems(res) u8,
 * all levels) / owner_list (lvx_list_words(V)) = the set bits of cull_flat's level 0 whose voxel cube,
 * grown by `margin` voxels, meets the sub-frustum of the pixel rect [x0,x1) x [y0,y1) of `cam`
 * (conservative).  A rank that traces only this rect passes them to lvx_scan / lvx_scatter / lvx_shade
 * in place of the culling pyramid and keeps the FULL pyramid for lvx_march_levels: its rays then step
 * exactly as on one GPU and find the reference's fragment lists in every voxel they visit.  margin
 * >= 1.5 also covers the 8 trilinear AO/shadow taps of any hit (lv/raytracer.py:368-390). */
int lvx_tile_owners(const uint8_t *cull_flat, int res, const lvx_camera *cam_host, int tile_x0, int tile_y0,
                    int tile_x1, int tile_y1, double margin, uint8_t *owner_flat, uint32_t *owner_list,
                    uint64_t *stats, void *stream);

/* ---- A-buffer: lv/abuffer.py:104-114 scan_offsets; 195-255 _chunk_count_kernel/_write_kernel.
 * offsets has V+1 entries (u32): offsets[i] = exclusive scan of the culling-masked counts,
 * offsets[V] = total, so count(i) = offsets[i+1]-offsets[i].  cull_base may be NULL (VSV).
 * The total is also written to stats[LVX_ST_FRAG_TOTAL].  cursor (V u32, may be NULL): when given, the scan
 * also writes lvx_scatter's cursors in the same pass (list start per visible voxel, a parking value per
 * culled one); pass cursor_ready = 1 to lvx_scatter then. */
int64_t lvx_scan_scratch_bytes(int64_t n_voxels);
int lvx_scan(const uint32_t *base, const uint8_t *cull_base, int64_t n_voxels,
             uint32_t *offsets, void *scratch, uint64_t *stats, uint32_t *cursor, void *stream);
/* second traversal: cursor (V u32 scratch) is initialised from offsets (unless cursor_ready != 0: lvx_scan
 * with the same culling mask has already written it); fragments of each
 * voxel end up in ascending segment order (lv/abuffer.py:313-317 semantics) after the
 * ordering pass, which walks vis_list (the voxels that own fragments).
 * Tight index (optional; pass all three arrays or none): tight_frags (frag_capacity u32),
 * tight_slot (frag_capacity u16), tight_cnt (V u16).  A fragment is "tight" unless its capsule
 * (radius r_tight = r + 1e-3, voxel units) provably does not reach into the voxel that lists it --
 * then no ray hit can be accepted for it there (lv/raytracer.py:446-452).  For every listed voxel v
 * the ordering pass writes tight_cnt[v] and, at offsets[v] + 0 .. tight_cnt[v], the tight
 * fragments' segment ids and their slots in the full list.  Acceleration only: `frags`, offsets and
 * the ray-test counts are the reference's. */
/* largest frag_capacity (and fragment total) lvx_scatter accepts; larger -> LVX_E_ARG */
int64_t lvx_max_fragments(void);
int lvx_scatter(const double *verts, const int32_t *segs, int64_t n_seg, double rt, double r_tight, int res, int method,
                const uint8_t *cull_flat /* NULL = no culling */, const uint32_t *vis_list,
                const uint32_t *offsets, uint32_t *cursor, uint32_t *frags, int64_t frag_capacity,
                uint32_t *tight_frags, uint16_t *tight_slot, uint16_t *tight_cnt /* may be NULL */,
                int cursor_ready, uint64_t *stats, void *stream);

/* The same second traversal for the capsule method (method 1), without per-incidence global atomics and without
 * an ordering pass (csrc/bricks.cu): the segments are binned into 8^3-voxel bricks, one CTA per brick sorts the
 * brick's segment ids and builds the lists of its voxels in ascending order in shared memory.  Same `frags` as
 * lvx_scatter bit for bit (the reference's array, lv/abuffer.py:313-317); the tight index may list a few more
 * fragments (cube grown by r_tight in the maximum norm instead of the Euclidean one), it stays conservative.
 * res >= 8.  scratch: lvx_brick_scratch_words(res, pair_capacity) u32; pair_capacity = (segment, brick) pairs the
 * scratch can hold (a segment overlaps ~3-5 bricks).  stats[LVX_ST_BRICK_PAIRS] receives the number needed: if
 * it exceeds pair_capacity nothing was built and the call must be repeated with a larger scratch.  No cursor, no
 * vis_list. */
int64_t lvx_brick_scratch_words(int res, int64_t pair_capacity);
int lvx_build_lists(const double *verts, const int32_t *segs, int64_t n_seg, double rt, double r_tight, int res,
                    const uint8_t *cull_flat /* NULL = no culling */, const uint32_t *offsets,
                    uint32_t *frags, int64_t frag_capacity,
                    uint32_t *tight_frags, uint16_t *tight_slot, uint16_t *tight_cnt /* may be NULL */,
                    uint32_t *scratch, int64_t pair_capacity, uint64_t *stats, void *stream);

/* ---- shading: lv/shading.py:72-155 _trilinear/_cone_trace/_shading_kernel, 170-185.
 * dirs_host: n_dirs*3 unit vectors (lv/shading.py:32-40); light_host: unit light direction.
 * ao/shadow: V f32; with fill_ones != 0 every voxel not in vis_list is set to 1.0 (the reference's
 * volumes), with 0 only listed voxels are written (shading on demand, see lvx_trace_hits).  n_dirs <= 15.  scratch: lvx_shade_scratch_bytes(V)
 * (per-level non-empty masks).  nz_bits: the per-voxel bits from lvx_pack_wide, or NULL (the level-0
 * mask is then derived from `base`). */
int64_t lvx_shade_scratch_bytes(int64_t n_voxels);
int lvx_shade(const uint32_t *base, const double *mips, int res, const uint32_t *vis_list,
              const double *dirs_host, int n_dirs, double tan_ao, const double *light_host,
              double tan_shadow, float *ao, float *shadow, int fill_ones, const uint32_t *nz_bits,
              void *scratch, void *stream);

/* ---- march table: lv/raytracer.py:316-326 _empty_level evaluated once per voxel.  march[i] (V u8) =
 * 255 where bits_flat's level-0 bit is set, else the level _empty_level returns there; the ray
 * tracer's DDA then needs one byte per step.  bits_flat = the pyramid from lvx_cull or
 * lvx_occupied_pyramid (CullingPyramid.packed(), lv/culling.py:88-95).  res >= 4. */
int lvx_march_levels(const uint8_t *bits_flat, int res, uint8_t *march, void *stream);

/* ---- render: lv/raytracer.py:459-515 _opaque_kernel, 518-645 _transparent_kernel, 94-97 _to_srgb.
 * rgb: h*w*3 f64 linear (may be NULL), srgb: h*w*3 u8 (may be NULL), hit_id: h*w i32.
 * tight_*: the tight index from lvx_scatter, or NULL; valid only if it was built with r_tight >= params.radius. */
int lvx_render(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
               const uint32_t *tight_frags, const uint16_t *tight_slot, const uint16_t *tight_cnt,
               const uint8_t *march, int res, const float *ao, const float *shadow,
               const lvx_camera *cam_host, const lvx_render_params *params_host,
               double *rgb, uint8_t *srgb, int32_t *hit_id, uint64_t *stats, void *stream);

/* ---- shading on demand (opaque mode).  Same image as lvx_shade(all visible) + lvx_render, but AO and
 * shadow are cone-traced only for the voxels some pixel's hit actually interpolates:
 *   lvx_trace_hits  first hit per pixel (hit_t f64 h*w, < 0 = miss; hit_id) + need_list = visible
 *                   voxels among the 8 trilinear taps of every hit (lv/raytracer.py:368-390);
 *                   need_bits: V/32 u32 scratch; need_list: lvx_list_words(V) u32
 *   lvx_shade       with vis_list = need_list, fill_ones = 0
 *   lvx_resolve     normal + colour per hit pixel (lv/raytracer.py:486-502), reading ao/shadow only
 *                   where march marks the voxel visible (1.0 elsewhere, lv/shading.py:177-178) */
int lvx_trace_hits(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
                   const uint32_t *tight_frags, const uint16_t *tight_slot, const uint16_t *tight_cnt,
                   const uint8_t *march, int res, const lvx_camera *cam_host,
                   const lvx_render_params *params_host, double *hit_t, int32_t *hit_id, uint32_t *need_bits,
                   uint32_t *need_list, uint64_t *stats, void *stream);
int lvx_resolve(const double *verts, const double *normals, const uint8_t *march, int res, const float *ao,
                const float *shadow, const lvx_camera *cam_host, const lvx_render_params *params_host,
                const double *hit_t, const int32_t *hit_id, double *rgb, uint8_t *srgb, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LVX_H */
