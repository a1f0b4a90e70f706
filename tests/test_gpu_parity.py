"""GPU parity tests (run on the B200 box): the CUDA path, called through the C ABI, against the
CPU oracle on the same seeded inputs and against the committed golden fixtures.

Bars (BASELINE.json north_star): bit-exact counts, culling masks, offsets, fragment lists;
occupancy max-abs <= 1e-4 (in practice bit-exact); pixels <= 1/255 on >= 99.9 % of pixels.
"""
import numpy as np
import pytest

from helpers import SCENES, Scene, h

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lvx():
    import paper_2510_09081_b200 as m
    return m


def gpu_frame(lvx, sc, method="capsule"):
    cn = lvx.compute_clip_normals(sc.ls)
    pyr = lvx.voxelize(sc.ls, cn, sc.g, method=method, r_min=sc.r_min, r_world=sc.r_world)
    culling = None
    if sc.strategy == "vcsv":
        culling = lvx.compute_visibility(lvx.erode(pyr), sc.g, sc.cam)
        abuf = lvx.build_vcsv(sc.ls, cn, sc.g, pyr, culling, method=method, r_world=sc.r_world)
    else:
        abuf = lvx.build_vsv(sc.ls, cn, sc.g, pyr, method=method, r_world=sc.r_world)
    scene = lvx.RenderScene(sc.ls, cn, sc.g, pyr, abuf, None, culling=culling, r_world=sc.r_world)
    scene.shading = lvx.compute_shading(pyr, scene.march_bits(), sc.g, sc.light)
    img = lvx.render(scene, sc.cam, lvx.RenderSettings(mode=sc.mode, alpha=sc.alpha, k=sc.k))
    return cn, pyr, culling, abuf, scene, img


@pytest.fixture(scope="module", params=SCENES)
def both(request, lvx, oracle):
    sc = Scene(request.param)
    ref = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                           alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    return sc, ref, gpu_frame(lvx, sc)


def test_upload(both, lvx):
    sc, ref, (cn, *_rest) = both
    verts, segs, normals, use_clip, r = lvx.segment_arrays(sc.ls, cn, sc.g, sc.r_world)
    assert h(verts.cpu().numpy()) == sc.hash["verts_voxel_f64"]
    assert h(normals.cpu().numpy()) == sc.hash["normals_f64"]
    assert h(segs.cpu().numpy().astype(np.int64)) == sc.hash["segs_i64"]
    assert float(r).hex() == sc.meta["r_voxel"] and use_clip


def test_base_bit_exact(both):
    sc, ref, (_, pyr, *_r) = both
    assert np.array_equal(pyr.base, ref.pyramid.base)
    assert h(pyr.base) == sc.hash["base_u32"]
    assert pyr.visited == sc.stats["visited"] and pyr.saturated == sc.stats["saturated"]
    # stated tolerance on occupancy: max-abs <= 1e-4 (holds trivially when the words are equal)
    assert np.abs(pyr.occupancy() - (ref.pyramid.base & 0xFFFF) / 4096.0).max() <= 1e-4


def test_mips(both):
    sc, ref, (_, pyr, *_r) = both
    assert [h(l) for l in pyr.occ_levels] == sc.hash["occ_levels_f64"]


def test_culling_masks(both):
    sc, ref, (_, _p, culling, *_r) = both
    if culling is None:
        pytest.skip("vsv")
    assert [h(l) for l in culling.levels] == sc.hash["cull_levels_u8"]
    assert np.array_equal(np.packbits(culling.base.ravel(), bitorder="little"), sc.arr["cull_base_bits"])


def test_abuffer_bit_exact(both):
    sc, ref, (_, _p, _c, abuf, *_r) = both
    assert abuf.total == sc.stats["fragments"]
    assert np.array_equal(abuf.table.offsets, ref.abuf.table.offsets)
    assert np.array_equal(abuf.table.counts, ref.abuf.table.counts)
    assert np.array_equal(abuf.fragments, ref.abuf.fragments)
    assert h(abuf.table.offsets) == sc.hash["offsets_i64"]
    assert h(abuf.table.counts) == sc.hash["counts_i64"]
    assert h(abuf.fragments) == sc.hash["fragments_u32"]


def test_shading(both):
    sc, ref, (*_a, scene, _img) = both
    assert np.array_equal(scene.shading.ao, ref.shading.ao)
    assert np.array_equal(scene.shading.shadow, ref.shading.shadow)
    assert h(scene.shading.ao) == sc.hash["ao_f32"] and h(scene.shading.shadow) == sc.hash["shadow_f32"]


def test_image(both):
    sc, ref, (*_a, img) = both
    assert img.stats["ray_capsule_tests"] == sc.stats["ray_capsule_tests"]
    assert np.array_equal(img.hit_id, sc.arr["hit_id"])
    srgb = np.frombuffer(img.srgb_bytes(), np.uint8).reshape(sc.arr["srgb"].shape)
    d = np.abs(srgb.astype(int) - sc.arr["srgb"].astype(int))
    assert (d <= 1).all(axis=2).mean() >= 0.999      # <= 1/255 per channel on >= 99.9 % of pixels
    assert d.max() <= 1
    assert np.abs(img.rgb - ref.image.rgb).max() <= 1e-12
    assert h(img.rgb) == sc.hash["rgb_f64"]          # f64 path without FMA: bit-identical in practice


@pytest.mark.parametrize("method", ["dda", "aabb"])
def test_other_traversals(lvx, oracle, method):
    sc = Scene("walk32_inside_cam")
    cn = oracle.compute_clip_normals(sc.ls)
    rp = oracle.voxelize(sc.ls, cn, sc.g, method=method, r_min=sc.r_min, r_world=sc.r_world)
    ra = oracle.build_vsv(sc.ls, cn, sc.g, rp, method=method, r_world=sc.r_world)
    gp = lvx.voxelize(sc.ls, cn, sc.g, method=method, r_min=sc.r_min, r_world=sc.r_world)
    ga = lvx.build_vsv(sc.ls, cn, sc.g, gp, method=method, r_world=sc.r_world)
    assert np.array_equal(gp.base, rp.base) and gp.visited == rp.visited
    assert np.array_equal(ga.fragments, ra.fragments)
    assert np.array_equal(ga.table.offsets, ra.table.offsets)


def test_no_clip_normals(lvx, oracle):
    sc = Scene("helix32_vsv")
    rp = oracle.voxelize(sc.ls, None, sc.g, r_min=sc.r_min, r_world=sc.r_world)
    gp = lvx.voxelize(sc.ls, None, sc.g, r_min=sc.r_min, r_world=sc.r_world)
    assert np.array_equal(gp.base, rp.base)


@pytest.mark.parametrize("seed,res,r", [(1, 16, 0.2), (2, 32, 0.7), (5, 64, 0.2), (7, 64, 1.1), (11, 128, 0.3)])
def test_random_scenes_vs_oracle(lvx, oracle, seed, res, r):
    ls = lvx.generate("random_streamlines", seed=seed, polylines=60, verts_per_line=40)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=r)
    cfg = lvx.PipelineConfig(res=res, width=96, height=80, strategy="vcsv", cam_azimuth=10.0 * seed)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")
    eng = lvx.FrameEngine(res, 96, 80, strategy="vcsv", keep_rgb=True, shading="all")
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    out = eng.run(cam, g, r_world)
    assert np.array_equal(eng.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    assert np.array_equal(eng.cull_flat.cpu().numpy(), ref.culling.flat)
    n = out.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(eng.offsets.cpu().numpy().view(np.uint32)[:-1].astype(np.int64), ref.abuf.table.offsets)
    assert np.array_equal(eng.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(eng.ao.cpu().numpy().reshape(res, res, res), ref.shading.ao)
    assert np.array_equal(eng.shadow.cpu().numpy().reshape(res, res, res), ref.shading.shadow)
    assert np.array_equal(eng.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(eng.rgb.cpu().numpy(), ref.image.rgb)
    assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
    assert out.stats["voxels_visited"] == ref.pyramid.visited


@pytest.mark.parametrize("seed,res,r,strategy", [(3, 32, 0.4, "vcsv"), (6, 64, 0.2, "vsv"), (9, 64, 0.9, "vcsv")])
def test_shading_on_demand_same_image(lvx, oracle, seed, res, r, strategy):
    """FrameEngine's default for opaque frames: AO/shadow only where a hit pixel reads them."""
    ls = lvx.generate("random_streamlines", seed=seed, polylines=50, verts_per_line=40)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=r)
    cfg = lvx.PipelineConfig(res=res, width=112, height=72, strategy=strategy, cam_elevation=5.0 * seed)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy)
    eng = lvx.FrameEngine(res, 112, 72, strategy=strategy, keep_rgb=True)
    assert eng.shading == "demand"
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    out = eng.run(cam, g, r_world)
    assert np.array_equal(eng.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(eng.rgb.cpu().numpy(), ref.image.rgb)
    assert np.array_equal(eng.srgb.cpu().numpy(), ref.image.srgb)
    assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
    # the requested voxels carry the oracle's values; fewer voxels were shaded than are visible
    n = out.stats["shaded_voxels"]
    idx = eng.need_list.cpu().numpy().view(np.uint32)[16:16 + n].astype(np.int64)
    assert len(np.unique(idx)) == n and 0 < n <= out.stats["visible_voxels"]
    assert np.array_equal(eng.ao.cpu().numpy()[idx], ref.shading.ao.ravel()[idx])
    assert np.array_equal(eng.shadow.cpu().numpy()[idx], ref.shading.shadow.ravel()[idx])


def test_transparent_engine_vs_oracle(lvx, oracle):
    ls = lvx.generate("random_streamlines", seed=4, polylines=80, verts_per_line=30)
    g, r_world = lvx.fit_grid(ls, 32, radius_voxels=0.5)
    cfg = lvx.PipelineConfig(res=32, width=80, height=64, strategy="vsv", mode="transparent", alpha=0.25, k=3)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vsv", mode="transparent",
                           alpha=0.25, k=3)
    eng = lvx.FrameEngine(32, 80, 64, strategy="vsv", mode="transparent", alpha=0.25, k=3, keep_rgb=True)
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    out = eng.run(cam, g, r_world)
    assert np.array_equal(eng.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(eng.rgb.cpu().numpy(), ref.image.rgb)
    assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]


def test_count_overflow_takes_wide_path(lvx, oracle):
    """> 65535 segments through one voxel: the 16-bit count saturates (lv/voxelizer.py:333-336)."""
    n = 70000
    rng = np.random.default_rng(0)
    a = 3.5 + 0.2 * rng.uniform(-1, 1, size=(n, 3))
    v = np.empty((2 * n, 3), np.float32)
    v[0::2] = a
    v[1::2] = a + 0.05
    ls = lvx.LineSet(v, np.arange(n + 1, dtype=np.int64) * 2, 0.1)
    g = lvx.GridDesc(8, np.zeros(3), 1.0)
    rp = oracle.voxelize(ls, None, g, r_world=0.1)
    gp = lvx.voxelize(ls, None, g, r_world=0.1)
    assert rp.saturated > 0
    assert np.array_equal(gp.base, rp.base)
    assert gp.visited == rp.visited and gp.saturated == rp.saturated


def test_empty_and_tiny_inputs(lvx, oracle):
    # a single 2-vertex polyline, zero-length segment included
    v = np.array([[1.5, 1.5, 1.5], [1.5, 1.5, 1.5], [2.5, 2.0, 1.0]], np.float32)
    ls = lvx.LineSet(v, np.array([0, 3]), 0.3)
    g = lvx.GridDesc(4, np.zeros(3), 1.0)
    cn = oracle.compute_clip_normals(ls)
    rp = oracle.voxelize(ls, cn, g)
    gp = lvx.voxelize(ls, cn, g)
    assert np.array_equal(gp.base, rp.base)
    ra = oracle.build_vsv(ls, cn, g, rp)
    ga = lvx.build_vsv(ls, cn, g, gp)
    assert np.array_equal(ga.fragments, ra.fragments)
    # geometry entirely outside the grid -> empty structures
    g2 = lvx.GridDesc(4, np.array([100.0, 100.0, 100.0]), 1.0)
    gp2 = lvx.voxelize(ls, cn, g2)
    assert gp2.visited == 0 and not gp2.base.any()
    ga2 = lvx.build_vsv(ls, cn, g2, gp2)
    assert ga2.total == 0


def test_long_lists_sorted(lvx, oracle):
    """Lists longer than the per-lane insertion-sort limit go through the warp bitonic sort."""
    n = 3000
    rng = np.random.default_rng(1)
    a = 2.0 + 4.0 * rng.uniform(0, 1, size=(n, 3))
    v = np.empty((2 * n, 3), np.float32)
    v[0::2] = a
    v[1::2] = a + rng.normal(scale=0.6, size=(n, 3))
    ls = lvx.LineSet(v, np.arange(n + 1, dtype=np.int64) * 2, 0.3)
    g = lvx.GridDesc(8, np.zeros(3), 1.0)
    rp = oracle.voxelize(ls, None, g)
    ra = oracle.build_vsv(ls, None, g, rp)
    gp = lvx.voxelize(ls, None, g)
    ga = lvx.build_vsv(ls, None, g, gp)
    assert ga.stats["long_lists"] > 0
    assert np.array_equal(ga.fragments, ra.fragments)


def _segment_box_distance(a, b, lo):
    """Distance between segments a->b and unit cubes [lo, lo+1] (rows), by ternary search on the convex
    function t -> dist(a + t (b - a), cube).  numpy, f64."""
    t0 = np.zeros(len(a)); t1 = np.ones(len(a))

    def f(t):
        p = a + t[:, None] * (b - a)
        d = np.maximum(np.maximum(lo - p, p - (lo + 1.0)), 0.0)
        return np.sqrt((d * d).sum(axis=1))
    for _ in range(70):
        m1 = t0 + (t1 - t0) / 3.0; m2 = t1 - (t1 - t0) / 3.0
        left = f(m1) <= f(m2)
        t1 = np.where(left, m2, t1); t0 = np.where(left, t0, m1)
    return f(0.5 * (t0 + t1))


@pytest.mark.parametrize("name", ["c1_vcsv", "diag32_thick_vsv", "walk32_transp_k2"])
def test_tight_index(lvx, name):
    """The ray tracer's acceleration index (csrc/abuffer.cu): per listed voxel the first tcnt entries
    of tfrags/tslot at the list's offset are a subset of the list in list order, and every
    fragment left out has its capsule provably outside the voxel (so it can never yield an accepted
    hit there, lv/raytracer.py:446-452)."""
    sc = Scene(name)
    cn, pyr, culling, abuf, scene, img = gpu_frame(lvx, sc)
    assert abuf.tight is not None
    res = sc.g.resolution
    off = abuf.table.offsets.astype(np.int64)
    cnt = abuf.table.counts.astype(np.int64)
    frags = abuf.fragments.astype(np.int64)
    tfr = abuf.tight.frags.cpu().numpy().view(np.uint32).astype(np.int64)
    tsl = abuf.tight.slot.cpu().numpy().view(np.uint16).astype(np.int64)
    tcn = abuf.tight.cnt.cpu().numpy().view(np.uint16).astype(np.int64)
    listed = np.nonzero(cnt > 0)[0]
    assert np.all(tcn[listed] <= cnt[listed])
    # expand (voxel, j) for j < tcnt
    reps = tcn[listed]
    vox_t = np.repeat(listed, reps)
    j = np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps)
    pos = off[vox_t] + j
    slot = tsl[pos]
    assert np.all(slot < cnt[vox_t])
    assert np.array_equal(frags[off[vox_t] + slot], tfr[pos])          # slot = position in the full list
    same = vox_t[1:] == vox_t[:-1]
    assert np.all(slot[1:][same] > slot[:-1][same])                    # list order kept (ascending ids)
    # fragments left out: capsule of radius r farther than r from the voxel cube
    is_tight = np.zeros(len(frags), dtype=bool)
    is_tight[off[vox_t] + slot] = True
    vox_all = np.repeat(listed, cnt[listed])
    loose = ~is_tight
    assert loose.sum() > 0
    verts = (sc.ls.vertices.astype(np.float64) - sc.g.world_min) / sc.g.voxel_size       # lv/voxelizer.py:440
    a = verts[frags[loose]]; b = verts[frags[loose] + 1]      # a fragment is its segment's start-vertex index
    v = vox_all[loose]
    lo = np.stack([v % res, (v // res) % res, v // (res * res)], axis=1).astype(np.float64)
    d = _segment_box_distance(a, b, lo)
    r = sc.r_world / sc.g.voxel_size
    assert d.min() > r + 5e-4, f"a loose fragment comes within {d.min() - r:.2e} of its voxel"
    if r < 0.5:
        assert is_tight.mean() < 0.6      # the index is worth having for thin lines


def test_engine_variants_identical(lvx, oracle):
    """FrameEngine's internal choices -- segment processing order (brick-sorted vs polyline order), 64-bit
    vs packed accumulation, frames submitted to two engines on two streams -- never change an output."""
    import torch
    ls = lvx.generate("random_streamlines", seed=12, polylines=120, verts_per_line=50)
    res = 64
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.3)
    cfg = lvx.PipelineConfig(res=res, width=160, height=96, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")

    def engine(order_brick, wide):
        e = lvx.FrameEngine(res, 160, 96, strategy="vcsv", keep_rgb=True)
        e.order_brick, e.use_wide = order_brick, wide
        e.set_topology(ls.polyline_offsets, ls.n_vertices)
        return e

    outs = []
    for order_brick, wide in [(0, False), (8, True), (16, False), (4, True)]:
        e = engine(order_brick, wide)
        e.load_vertices(ls.vertices)
        out = e.run(cam, g, r_world)
        n = out.stats["fragments"]
        assert np.array_equal(e.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
        assert n == ref.abuf.total
        assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
        assert np.array_equal(e.cull_flat.cpu().numpy(), ref.culling.flat)
        assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)
        assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
        assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
        assert out.stats["voxels_visited"] == ref.pyramid.visited
        if order_brick:
            order = e._order.cpu().numpy()
            assert np.array_equal(np.sort(order), e._segs.cpu().numpy())          # a permutation of segs
            v = e._verts64.cpu().numpy()[order]
            nb = res // order_brick
            c = np.clip(np.floor(v), 0, res - 1).astype(np.int64) // order_brick
            key = c[:, 0] + nb * (c[:, 1] + nb * c[:, 2])
            assert np.all(np.diff(key) >= 0)                                      # grouped by brick
        outs.append(e)
    # two frames in flight on two streams (submit/collect)
    ea, eb = engine(8, True), engine(8, True)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(sa):
        ea.load_vertices(ls.vertices); ea.submit(cam, g, r_world)
    with torch.cuda.stream(sb):
        eb.load_vertices(ls.vertices); eb.submit(cam, g, r_world)
    with torch.cuda.stream(sa):
        ra = ea.collect()
    with torch.cuda.stream(sb):
        rb = eb.collect()
    torch.cuda.synchronize()
    for e, r in ((ea, ra), (eb, rb)):
        assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
        assert r.stats["fragments"] == ref.abuf.total


def test_segment_shards_merge_on_engine(lvx, oracle):
    """Multi-GPU voxelization emulated on one GPU: two engines accumulate disjoint segment shards, the
    `after_voxelize` hook sums the 64-bit accumulators (what TiledFrame's all-reduce does) and the rest
    of the frame runs replicated -- the result is the single-GPU frame, bit for bit."""
    from paper_2510_09081_b200 import distributed as D
    ls = lvx.generate("grid_diagonals", count=300, length=14.0, domain=20.0)
    ls = lvx.LineSet(ls.vertices, ls.polyline_offsets, 1.1)
    res = 32
    g, r_world = lvx.fit_grid(ls, res)
    cfg = lvx.PipelineConfig(res=res, width=96, height=64, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")
    b = D.shard_bounds(ls.n_segments, 2)
    partial = {}

    def engine():
        e = lvx.FrameEngine(res, 96, 64, strategy="vcsv", keep_rgb=True)
        e.set_topology(ls.polyline_offsets, ls.n_vertices)
        e.load_vertices(ls.vertices)
        return e

    from paper_2510_09081_b200 import ops
    for rank in range(2):       # what each rank accumulates on its own (upload + voxelize stages only)
        e = engine()
        assert e.use_wide
        ops.stats_reset(e.stats)
        e._stage_upload(g, r_world)
        e._stage_voxelize((int(b[rank]), int(b[rank + 1])),
                          lambda eng, rank=rank: partial.__setitem__(rank, eng.wide.clone()))
    e = engine()
    out = e.run(cam, g, r_world, seg_range=(int(b[0]), int(b[1])),
                after_voxelize=lambda eng: eng.wide.copy_(partial[0] + partial[1]))
    assert np.array_equal(e.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    n = out.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.cull_flat.cpu().numpy(), ref.culling.flat)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
    assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)


@pytest.mark.parametrize("mode", ["opaque", "transparent"])
def test_screen_tiles_make_the_full_image(lvx, oracle, mode):
    """Screen-tile sharding (lvx_render_params.tile_*): tracing the tiles of a 3-way split one after the
    other fills exactly the image of a single full-frame trace, and the test counts add up."""
    from paper_2510_09081_b200 import distributed as D
    ls = lvx.generate("random_streamlines", seed=21, polylines=90, verts_per_line=40)
    res, w, h = 32, 150, 101          # sizes that are not multiples of the 8x4 warp tile
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.35)
    strategy = "vcsv" if mode == "opaque" else "vsv"
    cfg = lvx.PipelineConfig(res=res, width=w, height=h, strategy=strategy, mode=mode, alpha=0.4)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy, mode=mode, alpha=0.4)
    e = lvx.FrameEngine(res, w, h, strategy=strategy, mode=mode, alpha=0.4, keep_rgb=True)
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    full = e.run(cam, g, r_world)
    for tile_build in (True, False):
        e.tile_build = tile_build
        rgb = np.zeros((h, w, 3)); hit = np.full((h, w), -7, np.int32); tests = 0; frag_sum = 0
        for (x0, y0, x1, y1) in D.tile_rects(w, h, 3):
            out = e.run(cam, g, r_world, tile=(x0, y0, x1, y1))
            rgb[y0:y1, x0:x1] = e.rgb.cpu().numpy()[y0:y1, x0:x1]
            hit[y0:y1, x0:x1] = e.hit_id.cpu().numpy()[y0:y1, x0:x1]
            tests += out.stats["ray_capsule_tests"]
            frag_sum += out.stats["fragments"]
            if tile_build:      # the build of a tile is restricted to the voxels its rays can visit
                assert out.stats["owned_voxels"] < full.stats["visible_voxels"]
                assert out.stats["fragments"] < full.stats["fragments"]
            else:
                assert out.stats["fragments"] == full.stats["fragments"]
        assert np.array_equal(hit, ref.image.hit_id)
        assert np.array_equal(rgb, ref.image.rgb)
        assert tests == ref.image.stats["ray_capsule_tests"]
        if tile_build:
            assert frag_sum < 2 * full.stats["fragments"]       # three tiles together: little more than one full build


@pytest.mark.parametrize("mode,inside", [("opaque", False), ("opaque", True), ("transparent", False), ("transparent", True)])
def test_tile_owner_build_is_exact_on_rect_tiles(lvx, oracle, mode, inside):
    """lvx_tile_owners on a 3 x 2 grid of pixel rects (all four frustum planes in play), camera outside and
    inside the grid: per tile, the owners' lists are the reference's lists, every voxel the full frame's
    rays of that tile hit is owned, and the assembled image is the oracle's."""
    ls = lvx.generate("random_streamlines", seed=33, polylines=70, verts_per_line=50)
    res, w, h = 64, 133, 94
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.45)
    strategy = "vcsv" if mode == "opaque" else "vsv"
    cfg = lvx.PipelineConfig(res=res, width=w, height=h, strategy=strategy, mode=mode, alpha=0.35)
    cam = lvx.make_camera(cfg, g)
    if inside:
        centre = np.asarray(g.world_min) + 0.5 * res * g.voxel_size
        cam = lvx.Camera(centre + np.array([1.3, -2.1, 0.7]) * g.voxel_size, np.array([0.3, 1.0, -0.2]),
                         np.array([0.0, 0.0, 1.0]), np.deg2rad(70.0), w, h)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy, mode=mode, alpha=0.35)
    e = lvx.FrameEngine(res, w, h, strategy=strategy, mode=mode, alpha=0.35, keep_rgb=True)
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    xs, ys = [0, 40, 41, w], [0, 50, h]       # one tile is a single pixel column
    rgb = np.zeros((h, w, 3)); hit = np.full((h, w), -7, np.int32); tests = 0
    ref_off = ref.abuf.table.offsets; ref_cnt = ref.abuf.table.counts
    V = res ** 3
    for y0, y1 in zip(ys[:-1], ys[1:]):
        for x0, x1 in zip(xs[:-1], xs[1:]):
            out = e.run(cam, g, r_world, tile=(x0, y0, x1, y1))
            rgb[y0:y1, x0:x1] = e.rgb.cpu().numpy()[y0:y1, x0:x1]
            hit[y0:y1, x0:x1] = e.hit_id.cpu().numpy()[y0:y1, x0:x1]
            tests += out.stats["ray_capsule_tests"]
            own = e.owner_flat[:V].cpu().numpy() != 0
            assert own.sum() == out.stats["owned_voxels"]
            vis = ref.culling.flat[:V] != 0 if ref.culling is not None else ref_cnt > 0
            assert not (own & ~vis).any()                                    # owners are visible voxels
            # the owners' lists are the reference's lists
            offs = e.offsets.cpu().numpy().view(np.uint32).astype(np.int64)
            cnt = np.diff(offs)
            assert np.array_equal(cnt, np.where(own, ref_cnt, 0))
            fr = e.frags[:out.stats["fragments"]].cpu().numpy().view(np.uint32)
            idx = np.nonzero(own & (ref_cnt > 0))[0]
            pick = idx[:: max(1, len(idx) // 400)]
            for v in pick:
                assert np.array_equal(fr[offs[v]:offs[v] + cnt[v]], ref.abuf.fragments[ref_off[v]:ref_off[v] + ref_cnt[v]])
            # the OR pyramid above the owners
            lv = oracle.culling_from_bits(own.reshape(res, res, res).astype(np.uint8))
            assert np.array_equal(e.owner_flat.cpu().numpy(), lv.flat)
    assert np.array_equal(hit, ref.image.hit_id)
    assert np.array_equal(rgb, ref.image.rgb)
    assert tests == ref.image.stats["ray_capsule_tests"]


@pytest.mark.parametrize("kind,mode", [("walk", "opaque"), ("walk", "transparent"), ("diag", "opaque")])
def test_tiled_frame_emulated_ranks_make_the_frame(lvx, oracle, kind, mode):
    """Every rank of a 3-rank TiledFrame job, played one after the other on this GPU (EmulatedComm: the
    peers' shards are voxelized locally in place of the all-reduce; everything else is what the rank runs in
    the real job): each rank ends up with the whole-set grid and incidence count, builds only its tile's
    voxels, and the gathered strips are the oracle's image.  `diag` saturates the 16-bit occupancy field, so
    the per-field saturation after the sum is exercised."""
    from paper_2510_09081_b200 import distributed as D
    if kind == "walk":
        ls = lvx.generate("random_streamlines", seed=44, polylines=80, verts_per_line=45)
        res, w, h = 64, 150, 101
        g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.4)
    else:
        ls = lvx.generate("grid_diagonals", count=300, length=14.0, domain=20.0)
        ls = lvx.LineSet(ls.vertices, ls.polyline_offsets, 1.1)
        res, w, h = 32, 96, 64
        g, r_world = lvx.fit_grid(ls, res)
    strategy = "vcsv" if mode == "opaque" else "vsv"
    cfg = lvx.PipelineConfig(res=res, width=w, height=h, strategy=strategy, mode=mode, alpha=0.3)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy, mode=mode, alpha=0.3)
    if kind == "diag":
        assert (ref.pyramid.base & 0xFFFF).max() == 0xFFFF
    world = 3
    srgb = np.zeros((h, w, 3), np.uint8); hit = np.full((h, w), -7, np.int32); tests = 0; frags = 0
    for rank in range(world):
        e = lvx.FrameEngine(res, w, h, strategy=strategy, mode=mode, alpha=0.3)
        e.set_topology(ls.polyline_offsets, ls.n_vertices)
        e.load_vertices(ls.vertices)
        tf = D.TiledFrame(e, comm=D.EmulatedComm(rank, world))
        if kind == "diag":      # strips of unequal height, as strip balancing produces them
            tf.set_rows([0, 7, 50, h])
        lo, hi = tf.seg_range()
        assert hi - lo in (ls.n_segments // world, ls.n_segments // world + 1)
        out = tf.run(cam, g, r_world)
        # thin lines: the packed exchange (4 bytes per voxel, `base` arrives final); `diag` saturates a field: 8 bytes
        assert tf.exchange_kind == ("wide" if kind == "diag" else "packed") and e._base_final == (kind != "diag")
        assert tf.exchange_ms is None and tf.exchange_bytes == (8 if kind == "diag" else 4) * res ** 3
        assert np.array_equal(e.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
        assert out.stats["voxels_visited"] == ref.pyramid.visited
        if ref.culling is not None:
            assert np.array_equal(e.cull_flat.cpu().numpy(), ref.culling.flat)
        assert out.stats["fragments"] <= ref.abuf.total          # (a tall strip may own every visible voxel)
        s, hh = tf.gather_image()
        x0, y0, x1, y1 = tf.tiles[rank]
        if rank == 0:
            assert s.shape == (y1 - y0, w, 3)
        else:
            assert s is None and hh is None
        srgb[y0:y1] = e.srgb.cpu().numpy()[y0:y1]
        hit[y0:y1] = e.hit_id.cpu().numpy()[y0:y1]
        tests += out.stats["ray_capsule_tests"]
        frags += out.stats["fragments"]
    assert np.array_equal(hit, ref.image.hit_id)
    assert np.array_equal(srgb, ref.image.srgb)
    assert tests == ref.image.stats["ray_capsule_tests"]
    assert frags < 2 * ref.abuf.total


@pytest.mark.parametrize("res,mode", [(4, "opaque"), (8, "transparent"), (16, "opaque")])
def test_engine_tiny_inputs(lvx, oracle, res, mode):
    """FrameEngine at the small end: one or two segments, grids below the brick / bit-mask granularity
    (res < 32), images smaller than one 8x4 warp tile."""
    v = np.array([[0.1, 0.2, 0.3], [0.9, 0.8, 0.6], [0.5, 0.1, 0.9]], np.float32)
    ls = lvx.LineSet(v, np.array([0, 3], np.int64), 0.05)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.3) if res > 4 else (lvx.GridDesc(4, np.array([-0.5, -0.5, -0.5]), 0.5), 0.1)
    strategy = "vcsv" if mode == "opaque" else "vsv"
    cfg = lvx.PipelineConfig(res=res, width=5, height=3, strategy=strategy, mode=mode, alpha=0.5)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy, mode=mode, alpha=0.5)
    e = lvx.FrameEngine(res, 5, 3, strategy=strategy, mode=mode, alpha=0.5, keep_rgb=True)
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    out = e.run(cam, g, r_world)
    assert np.array_equal(e.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    n = out.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
    assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]


@pytest.mark.parametrize("kind,kw,res,r,az,lo,hi", [
    ("bundles", dict(seed=2, n_bundles=2, fibers=40, verts=41, domain=40.0), 64, 0.6, 35.0, 0, 1024),
    ("bundles", dict(seed=5, n_bundles=3, fibers=30, verts=41, domain=40.0), 64, 0.7, 35.0, 0, 1024),
    ("bundles", dict(seed=5, n_bundles=3, fibers=30, verts=41, domain=40.0), 64, 0.7, 200.0, 0, 1024),
    ("grid_diagonals", dict(count=6, length=20, domain=26), 64, 1.6, 35.0, 0, 1024),
    ("grid_diagonals", dict(count=12, length=14, domain=26), 32, 1.6, 120.0, 0, 1024),
    # 1025..16384 solid voxels: super-bricks with a short row use it, the others walk the brick flags
    ("grid_diagonals", dict(count=60, length=20, domain=26), 64, 1.5, 35.0, 1024, 16384),
    ("random_streamlines", dict(seed=4, polylines=60, verts_per_line=40), 64, 1.8, 35.0, 1024, 16384),
    ("bundles", dict(seed=2, n_bundles=3, fibers=60, verts=41, domain=40.0), 64, 0.6, 300.0, 1024, 16384),
])
def test_culling_with_few_solid_voxels(lvx, oracle, kind, kw, res, r, az, lo, hi):
    """1..16384 solid voxels: every super-brick keeps the solid voxels that shadow it and each occupied
    voxel is decided against them in closed form (blocked / visible / undecided -> literal march,
    csrc/cull.cu listed_solid_blocks).  The masks must equal the oracle's literal march bit for bit."""
    ls = lvx.generate(kind, **kw)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=r)
    cfg = lvx.PipelineConfig(res=res, width=64, height=64, strategy="vcsv", cam_azimuth=az)
    cam = lvx.make_camera(cfg, g)
    cn = oracle.compute_clip_normals(ls)
    pyr = oracle.voxelize(ls, cn, g, r_world=r_world)
    er = oracle.erode(pyr.occ_levels[0])
    n_solid = int((er >= 0.999).sum())
    assert lo < n_solid <= hi                        # the listed-solid path, not the all-walk fallback
    ref = oracle.compute_visibility(er, g, cam, pyr.counts() > 0)
    gp = lvx.voxelize(ls, lvx.compute_clip_normals(ls), g, r_world=r_world)
    got = lvx.compute_visibility(lvx.erode(gp), g, cam)
    occupied = int((pyr.counts() > 0).sum())
    visible = int((ref.flat[:res ** 3] != 0).sum())
    assert visible < occupied                        # something is really culled
    for a, b in zip(got.levels, ref.levels):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    # the same through the engine, from a camera inside the grid as well
    for position in (None, "inside"):
        c = cam
        if position == "inside":
            centre = np.asarray(g.world_min) + 0.5 * g.resolution * g.voxel_size
            c = lvx.Camera(centre + np.array([0.13, -0.21, 0.07]) * g.voxel_size, cam.forward, cam.up, cam.fov,
                           cam.width, cam.height)
            ref_c = oracle.compute_visibility(er, g, c, pyr.counts() > 0)
        else:
            ref_c = ref
        eng = lvx.FrameEngine(res, 64, 64, strategy="vcsv")
        eng.set_topology(ls.polyline_offsets, ls.n_vertices)
        eng.load_vertices(ls.vertices)
        out = eng.run(c, g, r_world)
        assert out.stats["solid_voxels"] == n_solid
        assert np.array_equal(eng.cull_flat.cpu().numpy(), ref_c.flat)


@pytest.mark.parametrize("res,strategy,mode", [(64, "vcsv", "opaque"), (256, "vcsv", "opaque"), (64, "vsv", "transparent")])
def test_launch_count_is_what_the_engine_claims(lvx, res, strategy, mode):
    """bench.py's `gpu_launches` comes from FrameEngine.kernel_launches_per_frame(); CUPTI (torch.profiler)
    counts the lvx kernels one frame really launches."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    ls = lvx.generate("random_streamlines", seed=8, polylines=60, verts_per_line=40)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.3)
    cfg = lvx.PipelineConfig(res=res, width=96, height=64, strategy=strategy, mode=mode, alpha=0.4)
    cam = lvx.make_camera(cfg, g)
    eng = lvx.FrameEngine(res, 96, 64, strategy=strategy, mode=mode, alpha=0.4)
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    eng.run(cam, g, r_world)                       # sizes the fragment buffer
    torch.cuda.synchronize()
    try:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            eng.run(cam, g, r_world)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if "lvx::" in e.name]
    except Exception as e:                         # no CUPTI in this environment
        pytest.skip(f"torch.profiler unavailable: {e}")
    if not names:
        pytest.skip("the profiler recorded no device activity")
    assert len(names) == eng.kernel_launches_per_frame(), sorted(names)


@pytest.mark.parametrize("r", [0.3, 1.7])
def test_zero_length_segments_through_the_engine(lvx, oracle, r):
    """Repeated vertices (zero-length segments take the AABB traversal, lv/voxelizer.py:155-156) mixed with
    ordinary ones, some of them at the grid boundary: the row-pooled scatter's state machine has its own form
    of that branch (RowGen box mode), so grid, lists and image are compared with the oracle."""
    rng = np.random.default_rng(17)
    polys, off = [], [0]
    for _ in range(40):
        n = int(rng.integers(3, 9))
        p = rng.uniform(2.0, 29.0, size=(n, 3))
        for k in rng.choice(n - 1, size=max(1, n // 3), replace=False):
            p[k + 1] = p[k]                      # a zero-length segment
        polys.append(p)
        off.append(off[-1] + n)
    polys.append(np.array([[0.2, 0.3, 31.6], [0.2, 0.3, 31.6], [0.2, 0.3, 31.6]]))   # all in one corner voxel
    off.append(off[-1] + 3)
    v = np.concatenate(polys).astype(np.float32)
    v[-3:] += np.array([[0, 0, 0], [0, 0, 0], [0.4, 0.0, -0.3]], np.float32)          # (not fully degenerate)
    ls = lvx.LineSet(v, np.array(off, dtype=np.int64), 0.25)
    res = 32
    g = lvx.GridDesc(res, np.zeros(3), 1.0)
    r_world = r
    cfg = lvx.PipelineConfig(res=res, width=80, height=60, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")
    e = lvx.FrameEngine(res, 80, 60, strategy="vcsv", keep_rgb=True)
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    out = e.run(cam, g, r_world)
    assert np.array_equal(e.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    n = out.stats["fragments"]
    assert n == ref.abuf.total and out.stats["voxels_visited"] == ref.pyramid.visited
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
