"""Host-side logic (no GPU): generators, grid fit and camera reproduce the reference bit for bit
(checked against the golden fixtures made from the live reference), configuration rules, .lns I/O."""
import numpy as np
import os
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import paper_2510_09081_b200 as lvx
from helpers import SCENES, Scene, h


@pytest.mark.parametrize("name", SCENES)
def test_generators_grid_and_camera_match_reference(name):
    sc = Scene(name)
    cfg = lvx.PipelineConfig(**sc.meta["cfg"])
    ls = lvx.pipeline.load_input(cfg)
    assert h(ls.vertices) == sc.hash["vertices_f32"]
    assert np.array_equal(ls.polyline_offsets, sc.arr["polyline_offsets"])
    g, r_world = lvx.fit_grid(ls, cfg.res, radius_voxels=cfg.r if cfg.r > 0 else None)
    assert [float(x).hex() for x in g.world_min] == sc.meta["grid"]["world_min"]
    assert float(g.voxel_size).hex() == sc.meta["grid"]["voxel_size"]
    assert float(r_world).hex() == sc.meta["r_world"]
    cam = lvx.make_camera(cfg, g)
    c = sc.meta["camera"]
    assert [float(x).hex() for x in cam.position] == c["position"]
    assert [float(x).hex() for x in cam.forward] == c["forward"]
    assert [float(x).hex() for x in cam.up] == c["up"]
    assert [float(x).hex() for x in cfg.light_vector()] == sc.meta["light"]


def test_config_rules():
    C = lvx.PipelineConfig
    C().validate()
    for bad in (dict(res=100), dict(method="x"), dict(strategy="y"), dict(mode="z"), dict(alpha=0.0),
                dict(alpha=1.5), dict(k=0), dict(k=65), dict(r=-1.0), dict(r_min=0.0), dict(workers=-1),
                dict(width=0), dict(cam_fov=180.0), dict(light="0,0,0"), dict(light="a,b"),
                dict(strategy="vcsv", mode="transparent")):
        with pytest.raises(lvx.ConfigError):
            C(**bad).validate()


def test_config_sources(tmp_path):
    f = tmp_path / "c.cfg"
    f.write_text("# comment\nres = 64\nmode=transparent\ndump = yes\n")
    cfg = lvx.PipelineConfig.from_sources(str(f), {"res": 32, "alpha": None})
    assert cfg.res == 32 and cfg.mode == "transparent" and cfg.dump is True
    f.write_text("nonsense\n")
    with pytest.raises(lvx.ConfigError):
        lvx.PipelineConfig.from_sources(str(f))
    with pytest.raises(lvx.ConfigError):
        lvx.PipelineConfig.from_sources(None, {"nope": 1})


def test_lineset_validation_and_segments():
    v = np.zeros((5, 3), np.float32)
    v[:, 0] = np.arange(5)
    ls = lvx.LineSet(v, [0, 2, 5], 0.1)
    assert ls.n_segments == 3 and ls.segment_vertex_ids().tolist() == [0, 2, 3]
    for off in ([0, 1, 5], [1, 5], [0, 4]):
        with pytest.raises(lvx.LineSetError):
            lvx.LineSet(v, off, 0.1)
    with pytest.raises(lvx.LineSetError):
        lvx.LineSet(v, [0, 5], 0.0)


@pytest.mark.parametrize("fmt", ["lns-binary", "lns-text"])
def test_lns_roundtrip(tmp_path, fmt):
    ls = lvx.generate("random_streamlines", seed=5, polylines=4, verts_per_line=6)
    p = tmp_path / "a.lns"
    lvx.save_lineset(ls, p, fmt)
    back = lvx.load_lineset(p)
    assert np.array_equal(back.vertices, ls.vertices) and np.array_equal(back.polyline_offsets, ls.polyline_offsets)
    assert back.radius == pytest.approx(ls.radius)
    p.write_bytes(b"LNS1\x00")
    with pytest.raises(lvx.ParseError):
        lvx.load_lineset(p)


def test_decimate_keeps_ends():
    ls = lvx.generate("helix", verts=11)
    d = lvx.decimate(ls, 4)
    assert d.n_vertices == 4 and np.array_equal(d.vertices[-1], ls.vertices[-1])


def test_bundles_generator_shape():
    ls = lvx.generate("bundles", seed=0, n_bundles=2, fibers=5, verts=11)
    assert ls.n_polylines == 10 and ls.n_segments == 100


def test_grid_desc_rules():
    with pytest.raises(ValueError):
        lvx.GridDesc(48, np.zeros(3), 1.0)
    g = lvx.GridDesc(64, np.array([1.0, 2.0, 3.0]), 0.5)
    assert g.n_levels == 7 and g.flat_index(1, 2, 3) == 1 + 64 * (2 + 64 * 3)
    assert np.allclose(g.to_world(g.to_voxel([2.0, 3.0, 4.0])), [2.0, 3.0, 4.0])


def test_shards_index_the_canonical_segment_array():
    """A multi-GPU shard [b, e) must mean the same segments on every rank: the brick-grouped processing
    order is a per-rank permutation, so only a whole-set pass may use it (ops._shard_segs)."""
    from paper_2510_09081_b200 import ops
    lines = ops.DeviceLines(None, None, None, None, None, "SEGS", 110, 10, 0.2, None, 0.1, order="ORDER")
    assert lines.n_segments == 100
    assert ops._shard_segs(lines, 0, 100) == "ORDER"
    assert ops._shard_segs(lines, 0, 50) == "SEGS"
    assert ops._shard_segs(lines, 50, 100) == "SEGS"
    lines.order = None
    assert ops._shard_segs(lines, 0, 100) == "SEGS"


def test_bench_traffic_is_refused_when_stale(tmp_path, monkeypatch):
    """bench.py reads roofline.traffic from the committed ncu capture only if it was taken on these kernel
    sources (tools/ncu_summary.py stores the hash of csrc/)."""
    import json
    import sys
    sys.path.insert(0, ROOT)
    import bench
    prof = tmp_path / "profiles"
    prof.mkdir()
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "csrc_sha16", lambda: "abc")
    (prof / "ncu_traffic.json").write_text(json.dumps({"c2": {"k_a": 5, "k_b": 7}, "_csrc_sha16": {"c2": "abc"}}))
    v, src = bench.load_traffic("c2", "k_a+k_b")
    assert v == 12 and "csrc abc" in src
    (prof / "ncu_traffic.json").write_text(json.dumps({"c2": {"k_a": 5}, "_csrc_sha16": {"c2": "old"}}))
    v, src = bench.load_traffic("c2", "k_a")
    assert v is None and src.startswith("stale")
    v, src = bench.load_traffic("c3", "k_a")
    assert v is None and "no capture" in src


def test_bench_config_is_the_same_in_both_arms():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import paper_2510_09081_b200 as lvx
    ls = lvx.generate("random_streamlines", seed=0, polylines=100, verts_per_line=101)
    c = bench.workload_config("c1", ls)
    assert set(c) == {"workload", "segments", "grid", "image", "l2"} and c["segments"] == 10000
    assert "10000 segments" in c["workload"] and "r=0.2" in c["workload"]
    assert "r=0.6" in bench.describe("c2thick", ls)


def test_lns_files_written_by_the_reference():
    """tests/golden/walk6*.lns were written by the reference's save_lineset (make_golden.py lns_files): our
    loader reads both formats to the reference's arrays, our writer reproduces the files byte for byte, and
    decimate / segment_vertex_ids agree with the reference on the same set."""
    import tempfile
    g = os.path.join(ROOT, "tests", "golden")
    want = np.load(os.path.join(g, "walk6_lns.npz"))
    for name, fmt in (("walk6.lns", "lns-binary"), ("walk6_text.lns", "lns-text")):
        ls = lvx.load_lineset(os.path.join(g, name))          # format sniffed from the first bytes
        assert ls.vertices.dtype == np.float32 and np.array_equal(ls.vertices, want["vertices"])
        assert np.array_equal(ls.polyline_offsets, want["polyline_offsets"])
        assert ls.radius == float(want["radius"])
        with tempfile.TemporaryDirectory() as d:
            out = os.path.join(d, "o.lns")
            lvx.save_lineset(ls, out, fmt)
            assert open(out, "rb").read() == open(os.path.join(g, name), "rb").read(), f"{fmt} bytes differ"
    dec = lvx.decimate(ls, 3)
    assert np.array_equal(dec.vertices, want["dec_vertices"]) and np.array_equal(dec.polyline_offsets, want["dec_offsets"])
    assert np.array_equal(ls.segment_vertex_ids(), want["segment_vertex_ids"])


@pytest.mark.parametrize("kw", [dict(polylines=100, verts_per_line=101, seed=0),
                                dict(polylines=257, verts_per_line=33, seed=9, domain=128.0, curl=0.3),
                                dict(polylines=64, verts_per_line=2, seed=2, seg_length=9.0, domain=12.0)])
def test_vectorised_streamlines_are_the_reference_walks(kw):
    """random_streamlines advances all walks together for large sets (C5's 2 M-segment time steps in 0.5 s instead
    of 20 s); vertex for vertex it must be the sequential walk of lv/lineset.py:288-314 (same random stream, same
    rounding, reflections included)."""
    from paper_2510_09081_b200 import lineset as L
    k = dict(seg_length=1.0, domain=32.0, curl=0.6)
    k.update(kw)
    lo, hi = 0.2 * k["domain"], 0.8 * k["domain"]
    rng = np.random.default_rng(k["seed"])
    slow = np.concatenate([L._walk(rng, k["verts_per_line"], lo, hi, k["seg_length"], k["curl"]) for _ in range(k["polylines"])])
    fast = L._walks_vectorised(np.random.default_rng(k["seed"]), k["polylines"], k["verts_per_line"], lo, hi, k["seg_length"], k["curl"])
    assert np.array_equal(slow, fast)
    assert ((slow == lo) | (slow == hi)).any() or kw["verts_per_line"] < 5      # some walk was reflected at the domain wall
    ls = lvx.generate("random_streamlines", **kw)
    assert np.array_equal(ls.vertices, slow.astype(np.float32))
