"""GPU tests of the opt-in A-buffer builder (csrc/bricks.cu, lvx_build_lists): per-brick segment lists, no global
atomic and no sort per incidence.  Same `fragments` as the reference (lv/abuffer.py:313-317) and as the default
scatter + ordering passes, bit for bit; its tight index is conservative (a superset of the default one's)."""
import numpy as np
import pytest

from helpers import Scene
from test_gpu_parity import _segment_box_distance, gpu_frame

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lvx():
    import paper_2510_09081_b200 as m
    return m


@pytest.fixture()
def bricks(monkeypatch):
    monkeypatch.setenv("LVX_BUILDER", "bricks")


@pytest.mark.parametrize("name", ["c1_vcsv", "diag32_thick_vsv", "walk32_transp_k2"])
def test_stage_function_vs_oracle(lvx, oracle, bricks, name):
    """build_vsv / build_vcsv through the brick builder: fragments and image equal the oracle's; every fragment
    the tight index leaves out is provably out of reach of its voxel."""
    sc = Scene(name)
    ref = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                           alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    cn, pyr, culling, abuf, scene, img = gpu_frame(lvx, sc)
    assert abuf.total == ref.abuf.total
    assert np.array_equal(abuf.fragments, ref.abuf.fragments)
    assert np.array_equal(img.hit_id, ref.image.hit_id)
    assert np.array_equal(img.rgb, ref.image.rgb)
    assert img.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
    res = sc.g.resolution
    off = abuf.table.offsets.astype(np.int64)
    cnt = abuf.table.counts.astype(np.int64)
    frags = abuf.fragments.astype(np.int64)
    tfr = abuf.tight.frags.cpu().numpy().view(np.uint32).astype(np.int64)
    tsl = abuf.tight.slot.cpu().numpy().view(np.uint16).astype(np.int64)
    tcn = abuf.tight.cnt.cpu().numpy().view(np.uint16).astype(np.int64)
    listed = np.nonzero(cnt > 0)[0]
    assert np.all(tcn[listed] <= cnt[listed])
    reps = tcn[listed]
    vox_t = np.repeat(listed, reps)
    j = np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps)
    pos = off[vox_t] + j
    slot = tsl[pos]
    assert np.all(slot < cnt[vox_t])
    assert np.array_equal(frags[off[vox_t] + slot], tfr[pos])
    same = vox_t[1:] == vox_t[:-1]
    assert np.all(slot[1:][same] > slot[:-1][same])
    is_tight = np.zeros(len(frags), dtype=bool)
    is_tight[off[vox_t] + slot] = True
    loose = ~is_tight
    assert loose.sum() > 0
    vox_all = np.repeat(listed, cnt[listed])
    verts = (sc.ls.vertices.astype(np.float64) - sc.g.world_min) / sc.g.voxel_size
    a = verts[frags[loose]]; b = verts[frags[loose] + 1]
    v = vox_all[loose]
    lo = np.stack([v % res, (v // res) % res, v // (res * res)], axis=1).astype(np.float64)
    r = sc.r_world / sc.g.voxel_size
    assert _segment_box_distance(a, b, lo).min() > r + 5e-4


@pytest.mark.parametrize("seed,res,r,strategy,mode", [(1, 16, 0.2, "vcsv", "opaque"), (2, 32, 0.7, "vsv", "transparent"),
                                                      (5, 64, 0.2, "vcsv", "opaque"), (7, 64, 1.1, "vcsv", "opaque"),
                                                      (11, 128, 0.3, "vsv", "opaque")])
def test_engine_equals_default_builder_and_oracle(lvx, oracle, seed, res, r, strategy, mode):
    """FrameEngine(builder="bricks") against the default engine and the oracle on random scenes: offsets, fragments,
    hit ids and f64 colours identical; the two tight indices differ only in fragments that are out of reach."""
    ls = lvx.generate("random_streamlines", seed=seed, polylines=60, verts_per_line=40)
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=r)
    cfg = lvx.PipelineConfig(res=res, width=96, height=80, strategy=strategy, mode=mode, alpha=0.4, cam_azimuth=10.0 * seed)
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strategy, mode=mode, alpha=0.4)
    outs = []
    for builder in ("scatter", "bricks"):
        e = lvx.FrameEngine(res, 96, 80, strategy=strategy, mode=mode, alpha=0.4, keep_rgb=True, builder=builder)
        e.set_topology(ls.polyline_offsets, ls.n_vertices)
        e.load_vertices(ls.vertices)
        out = e.run(cam, g, r_world)
        n = out.stats["fragments"]
        assert n == ref.abuf.total
        assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
        assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)
        assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)
        assert out.stats["ray_capsule_tests"] == ref.image.stats["ray_capsule_tests"]
        outs.append((e, n))
    (es, n), (eb, _) = outs
    off = es.offsets.cpu().numpy().view(np.uint32).astype(np.int64)
    cnt = np.diff(off)
    listed = np.nonzero(cnt > 0)[0]

    def tight_set(e):
        tc = e.tight.cnt.cpu().numpy().view(np.uint16).astype(np.int64)[listed]
        tf = e.tight.frags.cpu().numpy().view(np.uint32).astype(np.int64)
        vox = np.repeat(listed, tc)
        j = np.arange(tc.sum()) - np.repeat(np.cumsum(tc) - tc, tc)
        return set(zip(vox.tolist(), tf[off[vox] + j].tolist()))
    # Both indices are conservative supersets of "the capsule reaches the voxel" (neither contains the other: one
    # bounds the distance to the cube from below with a separating direction, the other grows the cube in the
    # maximum norm); every fragment either of them leaves out must be out of reach, and the sizes are comparable.
    ts, tb = tight_set(es), tight_set(eb)
    verts = (ls.vertices.astype(np.float64) - g.world_min) / g.voxel_size
    rv = r_world / g.voxel_size
    for left_out in (ts - tb, tb - ts):
        if left_out:
            vox = np.array([p[0] for p in left_out]); seg = np.array([p[1] for p in left_out])
            lo = np.stack([vox % res, (vox // res) % res, vox // (res * res)], axis=1).astype(np.float64)
            assert _segment_box_distance(verts[seg], verts[seg + 1], lo).min() > rv + 5e-4
    assert len(tb) <= 1.6 * len(ts) + 16          # (thick tubes: the box has corners the rounded cube has not)


def test_pair_scratch_grows(lvx, oracle):
    """A pair array that is too small is reported (ST_BRICK_PAIRS) and the frame is redone with a larger one."""
    ls = lvx.generate("random_streamlines", seed=4, polylines=80, verts_per_line=50)
    res = 64
    g, r_world = lvx.fit_grid(ls, res, radius_voxels=0.3)
    cfg = lvx.PipelineConfig(res=res, width=64, height=48, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy="vcsv")
    e = lvx.FrameEngine(res, 64, 48, strategy="vcsv", keep_rgb=True, builder="bricks")
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    from paper_2510_09081_b200 import ops
    e._brick_scratch = ops.BrickScratch(res, 16, e.dev)       # far too small
    out = e.run(cam, g, r_world)
    assert e._brick_scratch.capacity > 16
    n = out.stats["fragments"]
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)


@pytest.mark.parametrize("r", [0.3, 1.7])
def test_zero_length_and_boundary_segments(lvx, oracle, r):
    """Zero-length segments (box traversal, lv/voxelizer.py:155-156) and segments at the grid boundary through
    the box mode of SlabPlan / slab_at."""
    rng = np.random.default_rng(17)
    polys, off = [], [0]
    for _ in range(40):
        n = int(rng.integers(3, 9))
        p = rng.uniform(-1.0, 33.0, size=(n, 3))          # some vertices outside the grid
        for k in rng.choice(n - 1, size=max(1, n // 3), replace=False):
            p[k + 1] = p[k]
        polys.append(p)
        off.append(off[-1] + n)
    v = np.concatenate(polys).astype(np.float32)
    ls = lvx.LineSet(v, np.array(off, dtype=np.int64), 0.25)
    res = 32
    g = lvx.GridDesc(res, np.zeros(3), 1.0)
    cfg = lvx.PipelineConfig(res=res, width=80, height=60, strategy="vcsv")
    cam = lvx.make_camera(cfg, g)
    ref = oracle.run_frame(ls, g, r, cam, cfg.light_vector(), strategy="vcsv")
    e = lvx.FrameEngine(res, 80, 60, strategy="vcsv", keep_rgb=True, builder="bricks")
    e.set_topology(ls.polyline_offsets, ls.n_vertices)
    e.load_vertices(ls.vertices)
    out = e.run(cam, g, r)
    n = out.stats["fragments"]
    assert n == ref.abuf.total
    assert np.array_equal(e.frags[:n].cpu().numpy().view(np.uint32), ref.abuf.fragments)
    assert np.array_equal(e.hit_id.cpu().numpy(), ref.image.hit_id)
    assert np.array_equal(e.rgb.cpu().numpy(), ref.image.rgb)


def test_long_brick_lists(lvx, oracle, bricks):
    """More segments in one brick than the shared-memory sort holds (> 1024): the in-place sort path."""
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
