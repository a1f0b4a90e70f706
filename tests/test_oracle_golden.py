"""Pins the C oracle (oracle/) against fixtures generated from the LIVE reference package
(tests/golden/make_golden.py).  CPU only; this is the gate that lets the GPU parity tests
trust the oracle on the GPU box, where /root/reference does not exist."""
import ctypes as C

import numpy as np
import pytest

from helpers import FULL_SCENES, GOLDEN, SCENES, Scene, h


@pytest.fixture(scope="module", params=SCENES)
def run(request, oracle):
    sc = Scene(request.param)
    out = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy,
                           mode=sc.mode, alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    return sc, out


def test_upload_arrays(run, oracle):
    sc, out = run
    verts, segs, normals, use_clip, r = oracle.segment_arrays(sc.ls, out.cn, sc.g, sc.r_world)
    assert h(verts) == sc.hash["verts_voxel_f64"]
    assert h(segs) == sc.hash["segs_i64"]
    assert h(normals) == sc.hash["normals_f64"]
    assert float(r).hex() == sc.meta["r_voxel"]


def test_voxelize_and_mips(run):
    sc, out = run
    assert h(out.pyramid.base) == sc.hash["base_u32"]
    assert out.pyramid.visited == sc.stats["visited"]
    assert out.pyramid.saturated == sc.stats["saturated"]
    assert [h(l) for l in out.pyramid.occ_levels] == sc.hash["occ_levels_f64"]


def test_culling(run):
    sc, out = run
    if sc.strategy != "vcsv":
        pytest.skip("no culling for vsv")
    assert [h(l) for l in out.culling.levels] == sc.hash["cull_levels_u8"]
    assert int(out.culling.base.sum()) == sc.stats["visible"]


def test_abuffer(run):
    sc, out = run
    assert out.abuf.total == sc.stats["fragments"]
    assert h(out.abuf.table.offsets) == sc.hash["offsets_i64"]
    assert h(out.abuf.table.counts) == sc.hash["counts_i64"]
    assert h(out.abuf.fragments) == sc.hash["fragments_u32"]


def test_shading(run):
    sc, out = run
    assert h(out.shading.ao) == sc.hash["ao_f32"]
    assert h(out.shading.shadow) == sc.hash["shadow_f32"]


def test_render(run):
    sc, out = run
    img = out.image
    assert img.stats["ray_capsule_tests"] == sc.stats["ray_capsule_tests"]
    assert h(img.hit_id) == sc.hash["hit_id_i32"]
    assert np.array_equal(img.hit_id, sc.arr["hit_id"])
    assert np.array_equal(img.srgb, sc.arr["srgb"])
    assert h(img.rgb) == sc.hash["rgb_f64"]


@pytest.mark.parametrize("name", FULL_SCENES)
def test_full_arrays(name, oracle):
    sc = Scene(name)
    out = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy,
                           mode=sc.mode, alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    a = sc.arr
    assert np.array_equal(out.pyramid.base, a["base"])
    assert np.array_equal(out.abuf.fragments, a["fragments"])
    assert np.array_equal(out.abuf.table.offsets, a["offsets"])
    assert np.array_equal(out.shading.ao, a["ao"])
    assert np.array_equal(out.shading.shadow, a["shadow"])
    assert np.array_equal(out.image.rgb, a["rgb"])
    for i, lvl in enumerate(out.pyramid.occ_levels[1:], 1):
        assert np.array_equal(lvl, a[f"occ_level{i}"])


def test_unit_vectors(oracle):
    """Scalar known answers from the reference's own device functions."""
    u = np.load(GOLDEN + "/unit_vectors.npz")
    lib = oracle.lib()
    d = lambda x: C.c_double(float(x))
    n = len(u["r"])
    cells = np.empty((1 << 16, 3), dtype=np.int64)
    for i in range(n):
        a, b, n0, n1, p, r, o, dr = (u[k][i] for k in ("a", "b", "n0", "n1", "p", "r", "o", "d"))
        for c in (0, 1):
            args = [d(x) for x in (*p, *a, *b, *n0, *n1)]
            assert lib.orc_sdf(*args, d(r), C.c_int(c)) == u["sdf"][i, c]
            assert lib.orc_occupancy(*args, d(r), d(0.5), C.c_int(c)) == u["occ"][i, c]
            P = lambda v: np.ascontiguousarray(v, dtype=np.float64).ctypes.data_as(C.c_void_p)
            t = lib.orc_ray_capsule(P(o), P(dr), P(a), P(b), P(n0), P(n1), d(r), C.c_int(c))
            assert t == u["t"][i, c]
            if t >= 0:
                hp = np.ascontiguousarray(o + dr * t)
                nn = np.zeros(3)
                lib.orc_capsule_normal(P(hp), P(a), P(b), P(n0), P(n1), d(r), C.c_int(c), P(nn))
                assert np.array_equal(nn, u["normal"][i, c])
        a64, b64 = np.ascontiguousarray(a), np.ascontiguousarray(b)
        m = lib.orc_capsule_cells(a64.ctypes.data_as(C.c_void_p), b64.ctypes.data_as(C.c_void_p), d(r),
                                  cells.ctypes.data_as(C.c_void_p), C.c_int64(len(cells)))
        assert m == u["cells_n"][i]
        cl = cells[:m]
        key = np.sort((cl[:, 0] + 1000) + 4096 * ((cl[:, 1] + 1000) + 4096 * (cl[:, 2] + 1000)))
        assert h(key) == str(u["cells_hash"][i])
