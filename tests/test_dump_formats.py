"""On-disk formats either side of the path, CPU part: the package's writers
(`OccupancyPyramid.dump` VOXP, `CullingPyramid.dump` CULP, `ABuffer.dump` ABUF, `Image.save_ppm` /
`save_hit_ids`) are fed the ORACLE's arrays as CPU tensors and must produce the bytes the live
reference's writers produced (`tests/golden/dumps.json`, made by `make_golden.py dumps` from
lv/voxelizer.py:414-419, lv/culling.py:97-100, lv/abuffer.py:133-138, lv/raytracer.py:85-91).
The GPU part (the same files written from device tensors by `ScenePipeline`) is in
tests/test_gpu_pipeline.py."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from helpers import GOLDEN, Scene

DUMPS = json.load(open(os.path.join(GOLDEN, "dumps.json")))


def sha(path):
    b = open(path, "rb").read()
    return {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}


@pytest.mark.parametrize("name", sorted(DUMPS))
def test_writers_reproduce_reference_files(name, oracle, tmp_path):
    from paper_2510_09081_b200.abuffer import ABuffer, OffsetTable
    from paper_2510_09081_b200.culling import CullingPyramid
    from paper_2510_09081_b200.raytracer import Image
    from paper_2510_09081_b200.voxelizer import OccupancyPyramid
    sc = Scene(name)
    want = DUMPS[name]["files"]
    ref = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                           alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    res = sc.g.resolution
    V = res ** 3
    base = torch.from_numpy(ref.pyramid.base.reshape(-1).view(np.int32).copy())
    mips = torch.from_numpy(ref.pyramid.occ_flat[V:].copy())
    pyr = OccupancyPyramid(base, mips, sc.g, sc.r_min, ref.pyramid.saturated, ref.pyramid.visited)
    pyr.dump(tmp_path / "f.voxp")
    assert sha(tmp_path / "f.voxp") == want["voxp"]
    offs = np.concatenate([ref.abuf.table.offsets, [ref.abuf.total]]).astype(np.uint32)
    table = OffsetTable(torch.from_numpy(offs.view(np.int32).copy()), ref.abuf.total)
    frags = torch.from_numpy(ref.abuf.fragments.view(np.int32).copy())
    ABuffer(table, frags, res, {}).dump(tmp_path / "f.abuf")
    assert sha(tmp_path / "f.abuf") == want["abuf"]
    if ref.culling is not None:
        CullingPyramid(torch.from_numpy(ref.culling.flat.copy()), res).dump(tmp_path / "f.culp")
        assert sha(tmp_path / "f.culp") == want["culp"]
    else:
        assert "culp" not in want
    img = Image(torch.from_numpy(ref.image.rgb), torch.from_numpy(ref.image.srgb), torch.from_numpy(ref.image.hit_id))
    img.save_ppm(tmp_path / "f.ppm")
    img.save_hit_ids(tmp_path / "f.hiti")
    assert sha(tmp_path / "f.ppm") == want["ppm"]
    assert sha(tmp_path / "f.hiti") == want["hiti"]
    # the host sRGB conversion (used when only the f64 image was kept) gives the same bytes
    assert Image(torch.from_numpy(ref.image.rgb), None, torch.from_numpy(ref.image.hit_id)).srgb_bytes() == \
        ref.image.srgb.tobytes()


@pytest.mark.parametrize("name", sorted(DUMPS))
def test_oracle_frame_stats_match_run_once(name, oracle):
    """The non-timing `stats` of the reference's frame entry (lv/pipeline.py:78-86, 124-133)."""
    sc = Scene(name)
    st = DUMPS[name]["stats"]
    ref = oracle.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                           alpha=sc.alpha, k=sc.k, r_min=sc.r_min)
    assert ref.pyramid.visited == st["voxels_visited"]
    assert ref.abuf.total == st["fragments"] and ref.abuf.stats["fragment_touches"] == st["fragment_touches"]
    assert ref.image.stats["ray_capsule_tests"] == st["ray_capsule_tests"]
    assert sc.ls.n_segments == st["segments"] and sc.ls.n_vertices == st["vertices"]
    occ = int((ref.pyramid.counts() > 0).sum())
    cf = 0.0 if ref.culling is None else 1.0 - int((ref.culling.base != 0).sum()) / occ
    assert float(cf).hex() == st["culled_fraction"]
    lo, hi = sc.ls.aabb()
    assert [float(x).hex() for x in lo] == DUMPS[name]["aabb"]["lo"]
    assert [float(x).hex() for x in hi] == DUMPS[name]["aabb"]["hi"]
