#!/usr/bin/env python3
"""Generate golden fixtures from the LIVE reference package (linevox, numba CPU).

Runs only in the build container where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every scene it stores the *inputs* (f32 vertices, polyline offsets, radius, grid,
camera, light, settings) and the reference's *outputs*: sha256 of every intermediate
array (base, mips, culling levels, offsets, counts, fragments, ao, shadow, rgb, hit_id,
srgb bytes), the sRGB image and hit ids in full, and -- for the small scenes -- all
arrays in full.  The fixtures are what the C oracle (oracle/) is pinned against; the
CUDA path is then compared with the oracle on the GPU box where the reference
package is not available.
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import linevox as lv  # noqa: E402
from linevox.voxelizer import segment_arrays  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


SCENES = {
    # name: (cfg kwargs, store_full)
    "helix32_vsv": (dict(input="gen:helix?turns=2&verts=60", res=32, width=64, height=64), True),
    "helix64_vcsv": (dict(input="gen:helix?turns=3&verts=120", res=64, width=64, height=64,
                          strategy="vcsv"), False),
    "c1_vcsv": (dict(input="gen:random_streamlines?polylines=100&verts_per_line=101", res=64,
                     width=256, height=256, strategy="vcsv"), False),
    "c1_vsv_transparent": (dict(input="gen:random_streamlines?polylines=100&verts_per_line=101",
                                res=64, width=256, height=256, strategy="vsv",
                                mode="transparent", alpha=0.3, k=8), False),
    "diag_vcsv": (dict(input="gen:grid_diagonals?count=400&length=20&domain=26", res=64, r=1.5,
                       width=96, height=96, strategy="vcsv"), False),
    "walk32_transp_k2": (dict(input="gen:random_streamlines?polylines=30&verts_per_line=25",
                              res=32, r=0.5, width=64, height=64, strategy="vsv",
                              mode="transparent", alpha=0.2, k=2), True),
    "walk32_inside_cam": (dict(input="gen:random_streamlines?polylines=20&verts_per_line=20",
                               res=32, r=0.4, width=48, height=48, strategy="vcsv",
                               cam_distance=3.0, cam_azimuth=10.0, cam_elevation=5.0), True),
    "diag32_thick_vsv": (dict(input="gen:grid_diagonals?count=60&length=8&domain=14", res=32,
                              r=1.2, width=48, height=48, strategy="vsv"), True),
}


def run_scene(name, kw, full):
    cfg = lv.PipelineConfig(**kw)
    pipe = lv.ScenePipeline(cfg)
    img = pipe.render_frame()
    scene, cam = pipe._last
    ls, cn, g, pyr = pipe.ls, pipe.cn, pipe.g, pipe.pyramid
    verts, segs, normals, use_clip, r = segment_arrays(ls, cn, g, pipe.r_world)
    ab = scene.abuf
    cull = scene.culling
    sh = scene.shading
    srgb = np.frombuffer(img.srgb_bytes(), dtype=np.uint8).reshape(img.height, img.width, 3)

    meta = {
        "cfg": kw,
        "grid": {"res": int(g.resolution), "world_min": [float(x).hex() for x in g.world_min],
                 "voxel_size": float(g.voxel_size).hex()},
        "r_world": float(pipe.r_world).hex(),
        "r_voxel": float(r).hex(),
        "r_min": float(cfg.r_min).hex(),
        "camera": {"position": [float(x).hex() for x in cam.position],
                   "forward": [float(x).hex() for x in cam.forward],
                   "up": [float(x).hex() for x in cam.up],
                   "fov": float(cam.fov).hex(), "width": cam.width, "height": cam.height},
        "light": [float(x).hex() for x in cfg.light_vector()],
        "settings": {"mode": cfg.mode, "alpha": float(cfg.alpha).hex(), "k": cfg.k},
        "strategy": cfg.strategy,
        "stats": {"visited": int(pyr.visited), "saturated": int(pyr.saturated),
                  "fragments": int(ab.total),
                  "ray_capsule_tests": int(img.stats["ray_capsule_tests"]),
                  "hits": int((img.hit_id >= 0).sum()),
                  "occ_q_sum": int((pyr.base & 0xFFFF).astype(np.int64).sum()),
                  "visible": int((cull.base != 0).sum()) if cull is not None else -1},
        "hash": {
            "vertices_f32": h(ls.vertices), "verts_voxel_f64": h(verts), "normals_f64": h(normals),
            "segs_i64": h(segs),
            "base_u32": h(pyr.base),
            "occ_levels_f64": [h(l) for l in pyr.occ_levels],
            "cull_levels_u8": [h(l) for l in cull.levels] if cull is not None else None,
            "offsets_i64": h(ab.table.offsets), "counts_i64": h(ab.table.counts),
            "fragments_u32": h(ab.fragments),
            "ao_f32": h(sh.ao), "shadow_f32": h(sh.shadow),
            "rgb_f64": h(img.rgb), "hit_id_i32": h(img.hit_id), "srgb_u8": h(srgb),
        },
    }
    arrays = {
        "vertices": ls.vertices, "polyline_offsets": ls.polyline_offsets,
        "radius": np.float64(ls.radius),
        "srgb": srgb, "hit_id": img.hit_id,
    }
    if cull is not None:
        arrays["cull_base_bits"] = np.packbits(cull.base.ravel(), bitorder="little")
    if full:
        arrays.update({
            "normals": normals, "base": pyr.base, "offsets": ab.table.offsets,
            "counts": ab.table.counts, "fragments": ab.fragments,
            "ao": sh.ao, "shadow": sh.shadow, "rgb": img.rgb,
        })
        for i, l in enumerate(pyr.occ_levels[1:], 1):
            arrays[f"occ_level{i}"] = l
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(name, meta["stats"], flush=True)


def unit_vectors():
    """Scalar known-answer vectors for the device functions (sdf, occupancy, ray-capsule,
    traversal cell lists, cone trace) on seeded random inputs."""
    from linevox.voxelizer import _sdf, _occupancy, capsule_cells
    from linevox.raytracer import _ray_capsule, _capsule_normal
    rng = np.random.default_rng(777)
    n = 400
    a = rng.uniform(2, 12, (n, 3)); b = a + rng.uniform(-4, 4, (n, 3))
    n0 = rng.normal(size=(n, 3)); n0 /= np.linalg.norm(n0, axis=1, keepdims=True)
    n1 = rng.normal(size=(n, 3)); n1 /= np.linalg.norm(n1, axis=1, keepdims=True)
    p = a + rng.uniform(-2, 2, (n, 3))
    r = rng.uniform(0.1, 1.5, n)
    o = rng.uniform(-5, 20, (n, 3)); d = (a + b) / 2 + rng.normal(scale=0.6, size=(n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    b[::50] = a[::50]  # zero-length capsules
    sdf = np.empty((n, 2)); occ = np.empty((n, 2)); tt = np.empty((n, 2)); nrm = np.zeros((n, 2, 3))
    cells_n = np.empty(n, np.int64); cells_hash = []
    for i in range(n):
        for c in (0, 1):
            sdf[i, c] = _sdf(*p[i], *a[i], *b[i], *n0[i], *n1[i], r[i], bool(c))
            occ[i, c] = _occupancy(*p[i], *a[i], *b[i], *n0[i], *n1[i], r[i], 0.5, bool(c))
            tt[i, c] = _ray_capsule(*o[i], *d[i], *a[i], *b[i], *n0[i], *n1[i], r[i], bool(c))
            if tt[i, c] >= 0:
                hp = o[i] + d[i] * tt[i, c]
                nrm[i, c] = _capsule_normal(*hp, *a[i], *b[i], *n0[i], *n1[i], r[i], bool(c))
        cl = capsule_cells(a[i], b[i], r[i])
        cells_n[i] = len(cl)
        # order-independent digest of the cell set
        key = np.sort((cl[:, 0] + 1000) + 4096 * ((cl[:, 1] + 1000) + 4096 * (cl[:, 2] + 1000)))
        cells_hash.append(h(key))
    np.savez_compressed(os.path.join(OUT, "unit_vectors.npz"), a=a, b=b, n0=n0, n1=n1, p=p, r=r,
                        o=o, d=d, sdf=sdf, occ=occ, t=tt, normal=nrm, cells_n=cells_n,
                        cells_hash=np.array(cells_hash))
    print("unit_vectors", n, flush=True)


def dumps_and_stats():
    """On-disk formats either side of the path and the frame entry's `stats`:
    the reference's own writers (VOXP lv/voxelizer.py:414-419, CULP lv/culling.py:97-100, ABUF
    lv/abuffer.py:133-138, PPM/HITI lv/raytracer.py:85-91) are run on golden scenes and the sha256 + size
    of every file is committed, together with the non-timing `stats` of `run_once` (lv/pipeline.py:153-156)
    and `LineSet.aabb()` (lv/lineset.py:81-82)."""
    import tempfile
    out = {}
    for name in ("helix32_vsv", "walk32_inside_cam", "diag32_thick_vsv", "walk32_transp_k2", "helix64_vcsv", "diag_vcsv"):
        kw, _ = SCENES[name]
        pipe = lv.ScenePipeline(lv.PipelineConfig(**kw))
        img = pipe.render_frame()
        files = {}
        with tempfile.TemporaryDirectory() as d:
            pre = os.path.join(d, "f")
            pipe.dump_intermediates(pre)
            img.save_ppm(pre + ".ppm")
            img.save_hit_ids(pre + ".hiti")
            for ext in ("voxp", "culp", "abuf", "ppm", "hiti"):
                if os.path.exists(f"{pre}.{ext}"):
                    b = open(f"{pre}.{ext}", "rb").read()
                    files[ext] = {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}
        lo, hi = pipe.ls.aabb()
        stats = {k: v for k, v in pipe.stats.items() if not k.endswith("_ms")}
        stats["culled_fraction"] = float(stats["culled_fraction"]).hex()
        out[name] = {"files": files, "stats": stats, "stats_keys": sorted(pipe.stats),
                     "aabb": {"lo": [float(x).hex() for x in lo], "hi": [float(x).hex() for x in hi]}}
        print("dumps", name, {k: v["bytes"] for k, v in files.items()}, stats, flush=True)
    with open(os.path.join(OUT, "dumps.json"), "w") as f:
        json.dump(out, f, indent=1)


def lns_files():
    """Line-set files written by the reference's own writer (lv/lineset.py:191-210), both formats, committed as
    fixtures: the GPU package's loader must read them to the same arrays and its writer reproduce their bytes.
    `decimate` (lv/lineset.py:245-263) and `compute_clip_normals` (213-242) of the same set ride along."""
    ls = lv.generate("random_streamlines", seed=5, polylines=6, verts_per_line=9)
    ls = lv.LineSet(ls.vertices, ls.polyline_offsets, 0.3125)
    lv.save_lineset(ls, os.path.join(OUT, "walk6.lns"), "lns-binary")
    lv.save_lineset(ls, os.path.join(OUT, "walk6_text.lns"), "lns-text")
    dec = lv.decimate(ls, 3)
    np.savez_compressed(os.path.join(OUT, "walk6_lns.npz"), vertices=ls.vertices, polyline_offsets=ls.polyline_offsets,
                        radius=np.float64(ls.radius), dec_vertices=dec.vertices, dec_offsets=dec.polyline_offsets,
                        clip_normals=lv.compute_clip_normals(ls), segment_vertex_ids=ls.segment_vertex_ids())
    print("lns", ls.n_polylines, ls.n_vertices, flush=True)


if __name__ == "__main__":
    only = sys.argv[1:]
    if not only or "lns" in only:
        lns_files()
    if only == ["lns"]:
        sys.exit(0)
    if not only or "unit" in only:
        unit_vectors()
    if not only or "dumps" in only:
        dumps_and_stats()
    for name, (kw, full) in SCENES.items():
        if only and name not in only:
            continue
        run_scene(name, kw, full)
