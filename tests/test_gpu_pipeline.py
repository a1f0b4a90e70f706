"""GPU parity, second set (run on the B200 box): the drop-in frame entry (`ScenePipeline`, `run_once`,
dump files), the device AABB / grid fit, the reference's own edge-case grids (alpha x k, culling safety
over random poses, k-independence, early termination) and the culling paths beyond the listed-solid
limit -- all against the CPU oracle and the committed fixtures of the live reference.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import GOLDEN, Scene

pytestmark = pytest.mark.gpu

DUMPS = json.load(open(os.path.join(GOLDEN, "dumps.json")))


@pytest.fixture(scope="module")
def lvx():
    import paper_2510_09081_b200 as m
    return m


def sha(path):
    b = open(path, "rb").read()
    return {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}


# ----------------------------------------------------------------------------- frame entry (a22, f2, f3)

@pytest.mark.parametrize("name", sorted(DUMPS))
def test_scene_pipeline_is_the_reference_frame(lvx, name, tmp_path):
    """lv/pipeline.py:50-156 on the GPU: `ScenePipeline(cfg).render_frame()` and `run_once(cfg)` from the
    golden scene's own config -- image, hit ids, every non-timing `stats` value, the set of `stats` keys
    and the VOXP / CULP / ABUF / PPM / HITI files equal what the live reference produced."""
    sc = Scene(name)
    want = DUMPS[name]
    cfg = lvx.PipelineConfig(**sc.meta["cfg"])
    pipe = lvx.ScenePipeline(cfg)
    assert pipe.stats["voxels_visited"] == want["stats"]["voxels_visited"]        # build_geometry ran in __post_init__
    img = pipe.render_frame()
    assert np.array_equal(img.hit_id, sc.arr["hit_id"])
    assert img.srgb_bytes() == sc.arr["srgb"].tobytes()
    assert hashlib.sha256(np.ascontiguousarray(img.rgb).tobytes()).hexdigest()[:16] == sc.hash["rgb_f64"]
    assert sorted(pipe.stats) == want["stats_keys"]
    for k, v in want["stats"].items():
        got = pipe.stats[k]
        assert (float(got).hex() if k == "culled_fraction" else got) == v, k
    for k in want["stats_keys"]:
        if k.endswith("_ms"):
            assert pipe.stats[k] >= 0.0
    # grid, radius and camera are the reference's
    assert [float(x).hex() for x in pipe.g.world_min] == sc.meta["grid"]["world_min"]
    assert float(pipe.g.voxel_size).hex() == sc.meta["grid"]["voxel_size"]
    assert float(pipe.r_world).hex() == sc.meta["r_world"]
    # dump_intermediates + image files (lv/cli.py:64-77)
    pre = str(tmp_path / "f")
    pipe.dump_intermediates(pre)
    img.save_ppm(pre + ".ppm")
    img.save_hit_ids(pre + ".hiti")
    for ext, meta in want["files"].items():
        assert sha(f"{pre}.{ext}") == meta, ext
    assert os.path.exists(pre + ".culp") == ("culp" in want["files"])
    # intermediates hang off the pipeline like in the reference
    scene, cam = pipe._last
    assert hashlib.sha256(pipe.pyramid.base.tobytes()).hexdigest()[:16] == sc.hash["base_u32"]
    assert hashlib.sha256(scene.abuf.fragments.tobytes()).hexdigest()[:16] == sc.hash["fragments_u32"]
    assert hashlib.sha256(scene.abuf.table.offsets.tobytes()).hexdigest()[:16] == sc.hash["offsets_i64"]
    x, y, z = (int(v) for v in np.argwhere(pipe.pyramid.counts() > 0)[0][::-1])
    lst = scene.abuf.voxel_fragments(x, y, z)
    if scene.culling is None or scene.culling.base[z, y, x]:
        assert len(lst) == pipe.pyramid.counts()[z, y, x] and np.all(np.diff(lst.astype(np.int64)) > 0)
    # the returned image owns its pixels: a second frame must not change it
    before = img.srgb_bytes()
    cam2 = lvx.Camera.orbit((pipe.g.world_min + pipe.g.world_max) / 2, 1.1 * float(pipe.g.world_max[0] - pipe.g.world_min[0]),
                            1.0, 0.3, width=cfg.width, height=cfg.height)
    pipe.render_frame(cam2)
    assert img.srgb_bytes() == before
    # run_once: same image, same stats
    img2, stats2 = lvx.run_once(cfg)
    assert img2.srgb_bytes() == sc.arr["srgb"].tobytes() and np.array_equal(img2.hit_id, sc.arr["hit_id"])
    assert sorted(stats2) == want["stats_keys"]
    assert stats2["fragments"] == want["stats"]["fragments"]


def test_scene_pipeline_poses_revoxelize_and_streamed_vertices(lvx, oracle):
    """Per-pose frames reuse the geometry (lv/pipeline.py:89-93); cfg.revoxelize rebuilds it; the dynamic
    line-set additions (`update_vertices`, `set_lineset`) rebuild from the new vertices; a camera of another
    size is accepted.  Every frame equals the oracle's."""
    cfg = lvx.PipelineConfig(input="gen:random_streamlines?polylines=40&verts_per_line=30", res=32, r=0.4,
                             width=72, height=56, strategy="vcsv", seed=5)
    pipe = lvx.ScenePipeline(cfg)
    ls, g, rw = pipe.ls, pipe.g, pipe.r_world

    def check(img, ls_, g_, rw_, cam):
        ref = oracle.run_frame(ls_, g_, rw_, cam, cfg.light_vector(), strategy="vcsv")
        assert np.array_equal(img.hit_id, ref.image.hit_id)
        assert np.array_equal(img.rgb, ref.image.rgb)
        assert img.srgb_bytes() == ref.image.srgb.tobytes()
        assert pipe.stats["fragments"] == ref.abuf.total
        assert pipe.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
        assert pipe.stats["voxels_visited"] == ref.pyramid.visited

    centre = (g.world_min + g.world_max) / 2
    ext = float(g.world_max[0] - g.world_min[0])
    for az, el, dist in [(0.3, 0.2, 1.3), (2.0, -0.7, 0.9), (4.4, 1.0, 1.7)]:
        cam = lvx.Camera.orbit(centre, dist * ext, az, el, width=72, height=56)
        check(pipe.render_frame(cam), ls, g, rw, cam)
    cam_big = lvx.Camera.orbit(centre, 1.2 * ext, 0.9, 0.1, width=100, height=40)      # another image size
    check(pipe.render_frame(cam_big), ls, g, rw, cam_big)
    # streamed vertices: same topology, new positions -> refit + rebuild
    v2 = (ls.vertices * np.float32(1.07) + np.float32(0.3) * np.sin(ls.vertices[:, ::-1])).astype(np.float32)
    pipe.update_vertices(v2)
    img = pipe.render_frame()
    ls2 = lvx.LineSet(v2, ls.polyline_offsets, ls.radius)
    g2, rw2 = lvx.fit_grid(ls2, 32, radius_voxels=0.4)
    assert np.array_equal(pipe.g.world_min, g2.world_min) and pipe.g.voxel_size == g2.voxel_size and pipe.r_world == rw2
    check(img, ls2, g2, rw2, lvx.make_camera(cfg, g2))
    # a different line set altogether
    ls3 = lvx.generate("helix", turns=2.0, verts=50)
    pipe.set_lineset(ls3)
    img = pipe.render_frame()
    g3, rw3 = lvx.fit_grid(ls3, 32, radius_voxels=0.4)
    check(img, ls3, g3, rw3, lvx.make_camera(cfg, g3))
    # cfg.revoxelize: geometry rebuilt every frame (from cfg.input / the override)
    cfg.revoxelize = True
    img = pipe.render_frame()
    check(img, ls3, g3, rw3, lvx.make_camera(cfg, g3))
    assert pipe.stats["voxelize_ms"] > 0.0


def test_scene_pipeline_errors(lvx):
    with pytest.raises(lvx.ConfigError):
        lvx.ScenePipeline(lvx.PipelineConfig(strategy="vcsv", mode="transparent"))
    with pytest.raises(ValueError):
        lvx.ScenePipeline(lvx.PipelineConfig(strategy="vss", res=32))
    with pytest.raises(ValueError):
        lvx.FrameEngine(2, 8, 8)
    e = lvx.FrameEngine(16, 8, 8)
    e.set_topology(np.array([0, 2]), 2)
    e.load_vertices(np.array([[0, 0, 0], [1, 1, 1]], np.float32))
    with pytest.raises(ValueError):
        e.fit()
    with pytest.raises(ValueError):
        e.fit(radius_voxels=0.2, radius_world=0.1)


# ----------------------------------------------------------------------------- device AABB / fit (a3, f1)

@pytest.mark.parametrize("kind,kw,res,rv", [
    ("helix", dict(turns=3.0, verts=120), 64, 0.2),
    ("random_streamlines", dict(seed=0, polylines=100, verts_per_line=101), 64, 0.2),
    ("grid_diagonals", dict(count=400, length=20, domain=26), 64, 1.5),
    ("bundles", dict(seed=3, n_bundles=4, fibers=50, verts=61), 128, None),
    ("random_streamlines", dict(seed=9, polylines=3, verts_per_line=2), 16, None),
])
def test_engine_fit_is_fit_grid_of_the_host_aabb(lvx, kind, kw, res, rv):
    """`FrameEngine.fit` (AABB by `lvx_aabb`, run every bench frame) == fit_grid(ls) with LineSet.aabb()
    (lv/lineset.py:81-82, lv/grid.py:51-80), bit for bit."""
    import torch
    from paper_2510_09081_b200 import ops
    ls = lvx.generate(kind, **kw)
    lo, hi = ops.aabb(torch.from_numpy(ls.vertices).cuda())
    wlo, whi = ls.aabb()
    assert np.array_equal(lo, wlo) and np.array_equal(hi, whi)
    eng = lvx.FrameEngine(res, 8, 8)
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    g, rw = eng.fit(radius_voxels=rv) if rv is not None else eng.fit(radius_world=ls.radius)
    g0, rw0 = lvx.fit_grid(ls, res, radius_voxels=rv)
    assert np.array_equal(g.world_min, g0.world_min) and g.voxel_size == g0.voxel_size and rw == rw0


def test_engine_fit_golden_and_odd_sizes(lvx):
    import torch
    from paper_2510_09081_b200 import ops
    for name in ("c1_vcsv", "diag_vcsv", "helix64_vcsv"):
        sc = Scene(name)
        eng = lvx.FrameEngine(sc.g.resolution, 8, 8)
        eng.set_topology(sc.ls.polyline_offsets, sc.ls.n_vertices)
        eng.load_vertices(sc.ls.vertices)
        cfg = sc.meta["cfg"]
        g, rw = eng.fit(radius_voxels=cfg.get("r", 0.2))
        assert [float(x).hex() for x in g.world_min] == sc.meta["grid"]["world_min"]
        assert float(g.voxel_size).hex() == sc.meta["grid"]["voxel_size"] and float(rw).hex() == sc.meta["r_world"]
    rng = np.random.default_rng(3)
    for n in (1, 2, 31, 33, 1023, 4097, 100_003):       # sizes around the reduction's block boundaries
        v = (rng.normal(size=(n, 3)) * [1.0, 50.0, 1e-3] + [7.0, -3.0, 0.0]).astype(np.float32)
        lo, hi = ops.aabb(torch.from_numpy(v).cuda())
        assert np.array_equal(lo, v.min(axis=0).astype(np.float64)) and np.array_equal(hi, v.max(axis=0).astype(np.float64))


# ----------------------------------------------------------------------------- transparency grids (a20)

def _stage_scene(lvx, oracle, ls, g, r_world, light):
    cn = oracle.compute_clip_normals(ls)
    rp = oracle.voxelize(ls, cn, g, r_world=r_world)
    ra = oracle.build_vsv(ls, cn, g, rp, r_world=r_world)
    bits = oracle.culling_from_bits((rp.counts() > 0).astype(np.uint8))
    rs = oracle.compute_shading(rp, bits, g, light)
    gcn = lvx.compute_clip_normals(ls)
    gp = lvx.voxelize(ls, gcn, g, r_world=r_world)
    ga = lvx.build_vsv(ls, gcn, g, gp, r_world=r_world)
    scene = lvx.RenderScene(ls, gcn, g, gp, ga, None, r_world=r_world)
    scene.shading = lvx.compute_shading(gp, scene.march_bits(), g, light)
    return (cn, rp, ra, rs), scene


@pytest.mark.parametrize("spec,res,r,size", [
    ("gen:helix?turns=3&verts=120", 64, 0.2, 96),                                    # the reference's fixture
    ("gen:random_streamlines?polylines=60&verts_per_line=40", 32, 0.5, 80),          # many hits per voxel: re-scans at small k
])
def test_transparency_alpha_k_grid(lvx, oracle, spec, res, r, size):
    """pkg/tests/test_acceptance.py:187-204 on the GPU path: alpha in {0.1, 0.5, 1.0} x k in {1, 8, 32, 64}
    (k = 64 is the k-buffer's maximum) against the oracle, bit for bit; alpha = 1 transparent == opaque."""
    cfg = lvx.PipelineConfig(input=spec, res=res, r=r, width=size, height=size)
    ls = lvx.pipeline.load_input(cfg)
    g, rw = lvx.fit_grid(ls, res, radius_voxels=r)
    cam = lvx.make_camera(cfg, g)
    light = cfg.light_vector()
    (cn, rp, ra, rs), scene = _stage_scene(lvx, oracle, ls, g, rw, light)
    tests = {}
    for alpha in (0.1, 0.5, 1.0):
        for k in (1, 8, 32, 64):
            ref = oracle.render(ls, cn, g, rp, ra, rs, None, cam, mode="transparent", alpha=alpha, k=k, r_world=rw)
            img = lvx.render(scene, cam, lvx.RenderSettings(mode="transparent", alpha=alpha, k=k))
            assert np.array_equal(img.hit_id, ref.hit_id), (alpha, k)
            assert np.array_equal(img.rgb, ref.rgb), (alpha, k)
            assert img.srgb_bytes() == ref.srgb.tobytes(), (alpha, k)
            assert img.stats["ray_capsule_tests"] == ref.stats["ray_capsule_tests"], (alpha, k)
            tests[(alpha, k)] = img.stats["ray_capsule_tests"]
    assert tests[(0.1, 1)] > tests[(0.1, 64)] or "helix" in spec       # small k re-scans voxels (lv/raytracer.py:630-634)
    assert tests[(0.1, 8)] >= tests[(1.0, 8)]                           # more transparency, more tests
    op = lvx.render(scene, cam, lvx.RenderSettings(mode="opaque"))
    tr = lvx.render(scene, cam, lvx.RenderSettings(mode="transparent", alpha=1.0, k=8))
    assert op.srgb_bytes() == tr.srgb_bytes() and np.array_equal(op.hit_id, tr.hit_id)
    # the same through the engine (what the bench runs) at the extremes
    for alpha, k in ((0.1, 1), (0.1, 64), (1.0, 32)):
        ref = oracle.render(ls, cn, g, rp, ra, rs, None, cam, mode="transparent", alpha=alpha, k=k, r_world=rw)
        eng = lvx.FrameEngine(res, size, size, strategy="vsv", mode="transparent", alpha=alpha, k=k, keep_rgb=True)
        eng.set_topology(ls.polyline_offsets, ls.n_vertices)
        eng.load_vertices(ls.vertices)
        out = eng.run(cam, g, rw)
        assert np.array_equal(eng.rgb.cpu().numpy(), ref.rgb) and np.array_equal(eng.hit_id.cpu().numpy(), ref.hit_id)
        assert out.stats["ray_capsule_tests"] == ref.stats["ray_capsule_tests"]


def test_k_independence_and_early_termination(lvx, oracle):
    """pkg/tests/test_raytracer.py:208-222: the image does not depend on k (<= 1/255) and early
    termination is a no-op (<= 1/255); each variant equals the oracle bit for bit."""
    cfg = lvx.PipelineConfig(input="gen:helix?turns=3&verts=120", res=32, width=64, height=64)
    ls = lvx.pipeline.load_input(cfg)
    g, rw = lvx.fit_grid(ls, 32, radius_voxels=0.2)
    cam = lvx.make_camera(cfg, g)
    (cn, rp, ra, rs), scene = _stage_scene(lvx, oracle, ls, g, rw, cfg.light_vector())

    def both(**kw):
        ref = oracle.render(ls, cn, g, rp, ra, rs, None, cam, mode="transparent", r_world=rw, **kw)
        img = lvx.render(scene, cam, lvx.RenderSettings(mode="transparent", **kw))
        assert np.array_equal(img.rgb, ref.rgb) and np.array_equal(img.hit_id, ref.hit_id), kw
        return np.frombuffer(img.srgb_bytes(), np.uint8).astype(int)
    imgs = [both(alpha=0.4, k=k) for k in (1, 2, 8, 32)]
    for im in imgs[:-1]:
        assert np.abs(im - imgs[-1]).max() <= 1
    a = both(alpha=0.7, k=8, early_termination=True)
    b = both(alpha=0.7, k=8, early_termination=False)
    assert np.abs(a - b).max() <= 1


# ----------------------------------------------------------------------------- culling (a9)

@pytest.mark.parametrize("spec,radius", [
    ("gen:helix?turns=3&verts=120", 0.2),
    ("gen:random_streamlines?polylines=25&verts_per_line=25", 0.2),
    ("gen:grid_diagonals?count=400&length=20&domain=26", 1.5),      # interior voxels saturate and really occlude
])
def test_culling_safety_over_random_poses(lvx, oracle, spec, radius):
    """pkg/tests/test_acceptance.py:151-184: 20 random poses per fixture; opaque VCSV hit ids == VSV hit
    ids, and the VCSV culling pyramid, fragment total and hit ids equal the oracle's at every pose."""
    cfg_v = lvx.PipelineConfig(input=spec, res=64, width=96, height=96, r=radius)
    cfg_c = lvx.PipelineConfig(input=spec, res=64, width=96, height=96, r=radius, strategy="vcsv")
    vsv, vcsv = lvx.ScenePipeline(cfg_v), lvx.ScenePipeline(cfg_c)
    ls, g, rw = vsv.ls, vsv.g, vsv.r_world
    cn = oracle.compute_clip_normals(ls)
    rp = oracle.voxelize(ls, cn, g, r_world=rw)
    er = oracle.erode(rp.occ_levels[0])
    occupied = rp.counts() > 0
    centre = g.world_min + g.resolution * g.voxel_size / 2
    extent = g.resolution * g.voxel_size
    rng = np.random.default_rng(99)
    culled_some = False
    for _ in range(20):
        cam = lvx.Camera.orbit(centre, extent * rng.uniform(0.9, 1.8), azimuth=rng.uniform(0, 2 * np.pi),
                               elevation=rng.uniform(-1.2, 1.2), width=96, height=96)
        a = vsv.render_frame(cam)
        b = vcsv.render_frame(cam)
        assert np.array_equal(a.hit_id, b.hit_id)
        rc = oracle.compute_visibility(er, g, cam, occupied)
        scene, _ = vcsv._last
        assert np.array_equal(scene.culling.flat_dev.cpu().numpy(), rc.flat)
        assert vcsv.stats["fragments"] == int(rp.counts()[rc.base != 0].sum())
        culled_some |= vcsv.stats["fragments"] < vsv.stats["fragments"]
    # one full oracle frame at the last pose (image + fragments)
    ra = oracle.build_vcsv(ls, cn, g, rp, rc, r_world=rw)
    assert np.array_equal(scene.abuf.fragments, ra.fragments)
    rs = oracle.compute_shading(rp, rc, g, cfg_c.light_vector())
    ri = oracle.render(ls, cn, g, rp, ra, rs, rc, cam, r_world=rw)
    assert np.array_equal(b.hit_id, ri.hit_id) and np.array_equal(b.rgb, ri.rgb)
    if radius > 1.0:
        assert culled_some


@pytest.mark.parametrize("kind,kw,res,r", [
    ("random_streamlines", dict(seed=4, polylines=60, verts_per_line=40), 64, 3.0),      # 64 852 solid voxels
    ("grid_diagonals", dict(count=400, length=20, domain=26), 128, 3.0),                 # 51 078
    ("grid_diagonals", dict(count=400, length=20, domain=26), 64, 2.5),                  # 7 975: listed path, for the far / near cameras
])
def test_culling_beyond_the_listed_solid_limit(lvx, oracle, kind, kw, res, r):
    """More than LVX_SOLID_CAP = 16 384 solid voxels: every warp takes the brick-flag walk and the literal
    march with its early stop (csrc/cull.cu `t_stop`); the masks must equal the oracle's full-length march
    from cameras outside, inside, just outside and very far from the grid (f32-coarse parameters)."""
    ls = lvx.generate(kind, **kw)
    g, rw = lvx.fit_grid(ls, res, radius_voxels=r)
    cn = oracle.compute_clip_normals(ls)
    rp = oracle.voxelize(ls, cn, g, r_world=rw)
    er = oracle.erode(rp.occ_levels[0])
    occupied = rp.counts() > 0
    n_solid = int((er >= 0.999).sum())
    if res == 64 and r == 2.5:
        assert 1024 < n_solid <= 16384
    else:
        assert n_solid > 16384
    eng = lvx.FrameEngine(res, 32, 32, strategy="vcsv")
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    centre = np.asarray(g.world_min) + 0.5 * res * g.voxel_size
    ext = res * g.voxel_size
    fwd, up = np.array([0.0, 0.0, -1.0]), np.array([0.0, 1.0, 0.0])
    positions = {
        "orbit": lvx.make_camera(lvx.PipelineConfig(res=res, width=32, height=32, strategy="vcsv"), g).position,
        "inside": centre + np.array([0.13, -0.21, 0.07]) * g.voxel_size,
        "inside_solid": None,
        "near": centre + np.array([0.5 * ext + 0.3 * g.voxel_size, 0.11 * ext, -0.2 * ext]),
        "far": centre + np.array([0.3, -0.5, 0.8]) * 1e5 * g.voxel_size,
        "axis": centre + np.array([0.0, 0.0, 3.0 * ext]),                    # rays parallel to grid planes: tie steps
    }
    solid_idx = np.argwhere(er >= 0.999)
    z, y, x = solid_idx[len(solid_idx) // 2]
    positions["inside_solid"] = np.asarray(g.world_min) + (np.array([x, y, z]) + 0.4) * g.voxel_size
    some_culled = False
    for label, pos in positions.items():
        cam = lvx.Camera(np.asarray(pos, dtype=np.float64), fwd, up, np.deg2rad(45.0), 32, 32)
        ref = oracle.compute_visibility(er, g, cam, occupied)
        out = eng.run(cam, g, rw)
        assert out.stats["solid_voxels"] == n_solid
        got = eng.cull_flat.cpu().numpy()
        assert np.array_equal(got, ref.flat), f"{label}: {(got != ref.flat).sum()} mask bytes differ"
        assert out.stats["visible_voxels"] == int((ref.base != 0).sum())
        some_culled |= out.stats["visible_voxels"] < out.stats["occupied_voxels"]
        # the stage function is the same kernel sequence
        gp = lvx.voxelize(ls, lvx.compute_clip_normals(ls), g, r_world=rw) if label == "orbit" else gp
        cp = lvx.compute_visibility(lvx.erode(gp), g, cam)
        assert np.array_equal(cp.flat_dev.cpu().numpy(), ref.flat), label
    assert some_culled


def test_compute_visibility_on_plain_fields(lvx, oracle):
    """`erode` / `compute_visibility` on a numpy field (the reference's calling convention,
    lv/culling.py:112, 203): values just below THETA_BLOCK must not block; `occupied` is required."""
    res = 16
    g = lvx.GridDesc(res, np.zeros(3), 1.0)
    f = np.zeros((res, res, res))
    f[6:9, 4:12, 4:12] = 1.0             # (z, y, x): a slab normal to z
    f[7, 4:12, 4:12] = 0.99895          # in [4091.5/4096, 0.999): rounds to 4092 but is NOT >= 0.999
    occ = np.zeros((res, res, res), np.uint8)
    occ[2:14, 2:14, 2:14] = 1
    cam = lvx.Camera(np.array([8.0, 8.0, 40.0]), np.array([0.0, 0.0, -1.0]), np.array([0.0, 1.0, 0.0]), 0.8, 8, 8)
    ref = oracle.compute_visibility(oracle.erode(f), g, cam, occ)
    got = lvx.compute_visibility(lvx.erode(f), g, cam, occ)
    assert np.array_equal(got.flat_dev.cpu().numpy(), ref.flat)
    f[7, 4:12, 4:12] = 1.0              # now the slab is solid through and through and blocks
    ref2 = oracle.compute_visibility(oracle.erode(f), g, cam, occ)
    got2 = lvx.compute_visibility(lvx.erode(f), g, cam, occ)
    assert np.array_equal(got2.flat_dev.cpu().numpy(), ref2.flat)
    assert ref2.base.sum() < ref.base.sum()
    with pytest.raises(ValueError):
        lvx.compute_visibility(lvx.erode(f), g, cam)


def test_upload_cache_sees_in_place_edits(lvx, oracle):
    """The device copy of a LineSet is keyed on the content of its vertices: an in-place edit between two
    stage calls must be seen (the reference recomputes segment_arrays every call, lv/voxelizer.py:480)."""
    ls = lvx.generate("random_streamlines", seed=2, polylines=20, verts_per_line=20)
    g, rw = lvx.fit_grid(ls, 32, radius_voxels=0.4)
    p1 = lvx.voxelize(ls, None, g, r_world=rw)
    assert np.array_equal(p1.base, oracle.voxelize(ls, None, g, r_world=rw).base)
    ls.vertices[:, 0] += np.float32(0.37 * g.voxel_size)
    p2 = lvx.voxelize(ls, None, g, r_world=rw)
    assert np.array_equal(p2.base, oracle.voxelize(ls, None, g, r_world=rw).base)
    assert not np.array_equal(p1.base, p2.base)
    cn = oracle.compute_clip_normals(ls)
    p3 = lvx.voxelize(ls, cn, g, r_world=rw)
    cn[:] = cn[::-1].copy()             # same array object, new content
    p4 = lvx.voxelize(ls, cn, g, r_world=rw)
    assert np.array_equal(p4.base, oracle.voxelize(ls, cn, g, r_world=rw).base)
    assert not np.array_equal(p3.base, p4.base)


def test_fragment_buffer_overflow_is_redone_exactly(lvx, oracle):
    """A frame whose fragment total exceeds the buffer sized by earlier frames: the overflowing attempt's
    tracer must not follow stale tight counts past the buffer, and the redone frame equals the oracle."""
    ls = lvx.generate("random_streamlines", seed=17, polylines=60, verts_per_line=40)
    res = 32
    g, rw = lvx.fit_grid(ls, res, radius_voxels=0.2)
    cfg = lvx.PipelineConfig(res=res, width=64, height=48, strategy="vsv")
    cam = lvx.make_camera(cfg, g)
    eng = lvx.FrameEngine(res, 64, 48, strategy="vsv", keep_rgb=True)
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)
    small = eng.run(cam, g, rw)
    cap = eng.frags.numel()
    # the same lines four times as thick (same grid): far more incidences than the buffer holds
    big = eng.run(cam, g, 6.0 * rw)
    assert big.stats["fragments"] > cap > small.stats["fragments"] and eng.frags.numel() >= big.stats["fragments"]
    ref = oracle.run_frame(ls, g, 6.0 * rw, cam, cfg.light_vector(), strategy="vsv")
    n = big.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(eng.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(eng.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(eng.rgb.cpu().numpy(), ref.image.rgb)
    # and back: the thin frame after the thick one (stale tight counts of voxels that lost fragments)
    again = eng.run(cam, g, rw)
    ref0 = oracle.run_frame(ls, g, rw, cam, cfg.light_vector(), strategy="vsv")
    assert again.stats["fragments"] == ref0.abuf.total
    assert np.array_equal(eng.rgb.cpu().numpy(), ref0.image.rgb)


@pytest.mark.parametrize("res,r", [(64, 0.3), (128, 1.4), (32, 0.5)])
def test_engine_fused_pack_and_level1(lvx, oracle, res, r):
    """FrameEngine packs the 64-bit accumulators and builds pyramid level 1 in one kernel at res >= 64
    (lvx_pack_wide_mip1), then the upper levels (lvx_build_mips_upper), and lets the scan write the scatter
    cursors: grid, every pyramid level, the non-zero bits handed to the cone tracer, saturation count and the
    fragment lists must be what the separate passes / the oracle give."""
    ls = lvx.generate("grid_diagonals", count=220, length=16.0, domain=24.0)
    g, rw = lvx.fit_grid(ls, res, radius_voxels=r)
    cfg = lvx.PipelineConfig(res=res, width=48, height=40, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, rw, cam, cfg.light_vector(), strategy="vcsv")
    e = lvx.FrameEngine(res, 48, 40, strategy="vcsv", keep_rgb=True)
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    out = e.run(cam, g, rw)
    assert e._mip1_done == (res >= 64)
    base = e.base.cpu().numpy().view(np.uint32).reshape(res, res, res)
    assert np.array_equal(base, ref.pyramid.base)
    assert out.stats["saturated"] == ref.pyramid.saturated
    mips = e.mips.cpu().numpy()
    off = 0
    for l, lvl in enumerate(ref.pyramid.occ_levels[1:], 1):
        n = lvl.size
        assert np.array_equal(mips[off:off + n], lvl.ravel()), f"pyramid level {l}"
        off += n
    nz = np.unpackbits(e.nz_bits.cpu().numpy().view(np.uint8), bitorder="little").astype(bool)
    assert np.array_equal(nz, (ref.pyramid.base.ravel() & 0xFFFF) != 0)
    n = out.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)


def test_packed_exchange_of_two_shards_equals_the_whole_grid(lvx, oracle):
    """Multi-GPU exchange on the device (distributed.exchange_accumulators): the accumulators of two
    segment shards, merged through the 16-byte pre-check + PACKED 4-byte words (lvx_wide_field_max, lvx_pack_wide,
    int32 sum, lvx_widen), equal the accumulators of the whole set; a set whose fields can overflow takes the
    8-byte path; the packed base of the merged grid is the oracle's."""
    import torch
    from paper_2510_09081_b200 import distributed as D, ops
    ls = lvx.generate("random_streamlines", seed=8, polylines=80, verts_per_line=60)
    res = 64
    dev = torch.device("cuda")

    class Peer(D.Comm):
        rank, world = 0, 2

        def __init__(self, peer):
            self.peer, self.reduced = peer, []

        def all_reduce_sum(self, t):
            if t.numel() == 2 and t.dtype == torch.int64:
                t += D.field_bounds(self.peer); self.reduced.append("bounds")
            elif t.dtype == torch.int32:
                p = torch.empty_like(t)
                ops.pack_wide(self.peer, p, ops.new_stats(dev))
                t += p; self.reduced.append("packed")
            else:
                t += self.peer; self.reduced.append("wide")

    dense = lvx.generate("random_streamlines", seed=9, polylines=600, verts_per_line=60, domain=16.0)
    for ls, rv, want in ((ls, 0.3, "packed"), (dense, 3.0, "wide")):   # thin lines | a crowd of fat tubes (occupancy sums beyond 2^16)
        g, r_world = lvx.fit_grid(ls, res, radius_voxels=rv)
        eng = lvx.FrameEngine(res, 64, 48, strategy="vsv")
        eng.set_topology(ls.polyline_offsets, ls.n_vertices)
        eng.load_vertices(ls.vertices)
        eng._prepare_host()
        ops.stats_reset(eng.stats)
        eng._stage_upload(g, r_world)
        n = eng.lines.n_segments
        b = D.shard_bounds(n, 2)
        V = res ** 3
        parts = []
        for r in range(2):
            w = torch.zeros(V, dtype=torch.int64, device=dev)
            ops.voxelize_wide(eng.lines, res, eng.r_min, eng.method, w, eng.stats, int(b[r]), int(b[r + 1]))
            parts.append(w)
        whole = torch.zeros(V, dtype=torch.int64, device=dev)
        ops.voxelize_wide(eng.lines, res, eng.r_min, eng.method, whole, eng.stats, 0, n)
        bounds = D.field_bounds(whole).cpu().numpy()
        assert bounds[0] == int((whole >> 32).max().item()) and bounds[1] == int((whole & 0xFFFFFFFF).max().item())
        assert (bounds[1] >= 65536) == (want == "wide")
        mine = parts[0].clone()
        comm = Peer(parts[1])
        nbytes, kind = D.exchange_accumulators(mine, comm, packed_scratch=torch.empty(V, dtype=torch.int32, device=dev))
        assert kind == want and nbytes == (4 if want == "packed" else 8) * V and comm.reduced == ["bounds", want]
        assert torch.equal(mine, whole)
        base = torch.empty(V, dtype=torch.int32, device=dev)
        ops.pack_wide(mine, base, ops.new_stats(dev))
        ref = oracle.voxelize(ls, oracle.compute_clip_normals(ls), g, r_world=r_world)
        assert np.array_equal(base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.base)


@pytest.mark.parametrize("rank", [0, 1])
def test_tiled_frame_with_packed_exchange_on_the_engine(lvx, oracle, rank):
    """TiledFrame.run on the real FrameEngine as one rank of a 2-rank job whose peer is played by a Comm that adds
    what the other rank would contribute to each of the three collectives (bounds, packed words, incidence count):
    the exchange takes the packed 4-byte path, the engine skips its pack pass (`base` arrives final), and grid,
    lists and the rank's strip of the image are the oracle's."""
    import torch
    from paper_2510_09081_b200 import distributed as D, ops
    ls = lvx.generate("random_streamlines", seed=12, polylines=70, verts_per_line=50)
    res = 64
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.3)
    cfg = lvx.PipelineConfig(res=res, width=96, height=64, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")
    eng = lvx.FrameEngine(res, 96, 64, strategy="vcsv", keep_rgb=True)
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    eng.load_vertices(ls.vertices)

    class PeerComm(D.Comm):
        world = 2

        def __init__(self, rank):
            self.rank, self.kinds, self._peer = rank, [], None

        def peer_wide(self):
            if self._peer is None:        # the other rank's shard, voxelized here (its incidences go to eng.stats too)
                b = D.shard_bounds(eng.lines.n_segments, 2)
                o = 1 - self.rank
                self._peer = torch.zeros(eng.V, dtype=torch.int64, device=eng.dev)
                ops.voxelize_wide(eng.lines, res, eng.r_min, eng.method, self._peer, eng.stats, int(b[o]), int(b[o + 1]))
            return self._peer

        def all_reduce_sum(self, t):
            if t.dtype == torch.int32:
                p = torch.empty_like(t)
                ops.pack_wide(self.peer_wide(), p, ops.new_stats(eng.dev))
                t += p; self.kinds.append("packed")
            elif t.numel() == 2:
                t += D.field_bounds(self.peer_wide()); self.kinds.append("bounds")
            elif t.numel() == 1:
                self.kinds.append("count")            # (added by peer_wide's voxelization above)
            else:
                t += self.peer_wide(); self.kinds.append("wide")

        def gather(self, t):
            return [t] if self.rank == 0 else None

    comm = PeerComm(rank)
    tf = D.TiledFrame(eng, comm=comm)
    out = tf.run(cam, g, r_world)
    assert tf.exchange_kind == "packed" and tf.exchange_bytes == 4 * res ** 3 and comm.kinds == ["bounds", "packed", "count"]
    assert eng._base_final
    assert np.array_equal(eng.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    assert out.stats["voxels_visited"] == ref.pyramid.visited
    assert np.array_equal(eng.cull_flat.cpu().numpy(), ref.culling.flat)
    x0, y0, x1, y1 = tf.tiles[rank]
    assert np.array_equal(eng.hit_id.cpu().numpy()[y0:y1, x0:x1], ref.image.hit_id[y0:y1, x0:x1])
    assert np.array_equal(eng.rgb.cpu().numpy()[y0:y1, x0:x1], ref.image.rgb[y0:y1, x0:x1])
    # the same rank with the packed exchange switched off: the 8-byte path, the same frame
    comm2 = PeerComm(rank)
    tf2 = D.TiledFrame(eng, comm=comm2)
    tf2.packed_exchange = False
    tf2.run(cam, g, r_world)
    assert tf2.exchange_kind == "wide" and comm2.kinds == ["wide", "count"] and not eng._base_final
    assert np.array_equal(eng.base.cpu().numpy().view(np.uint32).reshape(res, res, res), ref.pyramid.base)
    assert np.array_equal(eng.hit_id.cpu().numpy()[y0:y1, x0:x1], ref.image.hit_id[y0:y1, x0:x1])


def test_base_mip1_equals_the_fused_pack_pass(lvx):
    """lvx_base_mip1 (level 1 of the pyramid + non-empty bits from a PACKED grid, used after a packed multi-GPU
    exchange) against lvx_pack_wide_mip1 on the same accumulators; lvx_wide_field_max's packed words against
    lvx_pack_wide's."""
    import torch
    from paper_2510_09081_b200 import ops
    res = 64
    V = res ** 3
    dev = torch.device("cuda")
    g = torch.Generator(device="cpu").manual_seed(5)
    cnt = torch.randint(0, 70000, (V,), generator=g)          # some counts and sums beyond the 16-bit fields
    occ = torch.randint(0, 90000, (V,), generator=g) * (torch.rand(V, generator=g) < 0.3)
    wide = ((cnt << 32) | occ).to(dev)
    n_mip = int(ops.level_offsets(res)[-1]) - V
    base_a = torch.empty(V, dtype=torch.int32, device=dev); nz_a = torch.zeros(V // 32, dtype=torch.int32, device=dev)
    mips_a = torch.zeros(n_mip, dtype=torch.float64, device=dev)
    ops.pack_wide_mip1(wide, res, base_a, ops.new_stats(dev), nz_a, mips_a)
    out2 = torch.empty(2, dtype=torch.int64, device=dev)
    base_b = torch.empty(V, dtype=torch.int32, device=dev)
    ops.wide_field_max(wide, out2, base_b)
    assert out2.tolist() == [int(cnt.max()), int(occ.max())]
    assert torch.equal(base_a, base_b)
    base_c = torch.empty(V, dtype=torch.int32, device=dev)
    ops.pack_wide(wide, base_c, ops.new_stats(dev))
    assert torch.equal(base_a, base_c)
    nz_b = torch.zeros(V // 32, dtype=torch.int32, device=dev); mips_b = torch.zeros(n_mip, dtype=torch.float64, device=dev)
    ops.base_mip1(base_b, res, nz_b, mips_b)
    n1 = (res // 2) ** 3
    assert torch.equal(nz_a, nz_b)
    assert torch.equal(mips_a[:n1], mips_b[:n1])
