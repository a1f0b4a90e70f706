"""CPU ORACLE -- test infrastructure, not the product.

numpy/ctypes front end of ``oracle/lvx_oracle.c`` (a plain-C f64 restatement of the
reference package ``linevox``, file:line citations in the C source).  The function names
and result fields mirror the reference (`pkg/src/linevox/__init__.py:9-21`) so that parity
tests read like the reference's own tests.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module; the product
package ``paper_2510_09081_b200`` never does.

Parity status: PINNED -- ``tests/test_oracle_golden.py`` checks every stage of this oracle
against fixtures generated from the live reference (``tests/golden/make_golden.py``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblvx_oracle.so")
_lib = None

OCC_SCALE = 4096
THETA_BLOCK = 0.999
AO_HALF_ANGLE = float(np.arccos(1.0 - 2.0 / 12.0))      # shading.py:25
SHADOW_HALF_ANGLE = float(np.deg2rad(5.0))              # shading.py:26
METHODS = {"dda": 0, "capsule": 1, "aabb": 2}


class OracleABufferError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "lvx_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", _HERE, "-B", "liblvx_oracle.so"],
                              stdout=subprocess.DEVNULL)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = C.CDLL(_SO)
        _lib.orc_sdf.restype = C.c_double
        _lib.orc_occupancy.restype = C.c_double
        _lib.orc_ray_capsule.restype = C.c_double
        _lib.orc_cone_trace.restype = C.c_double
        for f in ("orc_segment_ids", "orc_clip_normals", "orc_capsule_cells", "orc_pyramid_size",
                  "orc_scan_offsets"):
            getattr(_lib, f).restype = C.c_int64
        _lib.orc_second_pass.restype = C.c_int
        _lib.orc_max_threads.restype = C.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _d(x):
    return C.c_double(float(x))


def set_threads(n: int) -> None:
    lib().orc_set_threads(C.c_int(int(n)))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ----------------------------------------------------------------------------- upload

def compute_clip_normals(ls) -> np.ndarray:
    out = np.zeros((ls.n_vertices, 3), dtype=np.float64)
    rc = lib().orc_clip_normals(_p(ls.vertices), _p(ls.polyline_offsets),
                                C.c_int64(ls.n_polylines), _p(out))
    if rc < 0:
        raise ValueError(f"degenerate polyline {-rc - 1}: all vertices coincide")
    return out


def segment_arrays(ls, cn, g, r_world=None):
    """voxelizer.py:435-447"""
    verts = np.empty((ls.n_vertices, 3), dtype=np.float64)
    wmin = np.ascontiguousarray(g.world_min, dtype=np.float64)
    lib().orc_to_voxel(_p(ls.vertices), C.c_int64(ls.n_vertices), _p(wmin), _d(g.voxel_size), _p(verts))
    segs = np.empty(ls.n_segments, dtype=np.int64)
    n = lib().orc_segment_ids(_p(ls.polyline_offsets), C.c_int64(ls.n_polylines), _p(segs))
    assert n == ls.n_segments
    if cn is None:
        normals = np.zeros((ls.n_vertices, 3), dtype=np.float64)
        use_clip = False
    else:
        normals = np.ascontiguousarray(cn, dtype=np.float64)
        use_clip = True
    r = (ls.radius if r_world is None else r_world) / g.voxel_size
    return verts, segs, normals, use_clip, r


def footprint_radius(r, r_min=0.5):
    return max(r, r_min) + 0.5


def level_offsets(res: int) -> np.ndarray:
    sizes = []
    r = res
    while r >= 1:
        sizes.append(r ** 3)
        r >>= 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def _split_levels(flat, res):
    offs = level_offsets(res)
    out = []
    r = res
    for l in range(len(offs) - 1):
        out.append(flat[offs[l]:offs[l + 1]].reshape(r, r, r))
        r >>= 1
    return out


# ----------------------------------------------------------------------------- stages

def voxelize(ls, cn, g, method="capsule", r_min=0.5, workers=None, r_world=None, seg_range=None):
    """voxelizer.py:466-498 -> namespace(base, occ_levels, occ_flat, grid, r_min, saturated, visited).
    `seg_range=(lo, hi)` voxelizes only segments segs[lo:hi] (one chunk of voxelizer.py:461-463)."""
    if method not in METHODS:
        raise ValueError(f"unknown voxelization method {method!r}")
    if not r_min > 0:
        raise ValueError("r_min must be positive")
    res = g.resolution
    verts, segs, normals, use_clip, r = segment_arrays(ls, cn, g, r_world)
    if seg_range is not None:
        segs = np.ascontiguousarray(segs[seg_range[0]:seg_range[1]])
    base = np.zeros((res, res, res), dtype=np.uint32)
    visited = C.c_int64(0)
    sat = C.c_int64(0)
    lib().orc_voxelize(_p(verts), _p(segs), C.c_int64(len(segs)), _p(normals), C.c_int(use_clip),
                       _d(r), _d(footprint_radius(r, r_min)), _d(r_min), C.c_int(res),
                       C.c_int(METHODS[method]), _p(base), C.byref(visited), C.byref(sat))
    flat = np.empty(int(lib().orc_pyramid_size(C.c_int(res))), dtype=np.float64)
    lib().orc_build_mips(_p(base), C.c_int(res), _p(flat))
    return SimpleNamespace(base=base, occ_flat=flat, occ_levels=_split_levels(flat, res), grid=g,
                           r_min=r_min, saturated=int(sat.value), visited=int(visited.value),
                           resolution=res, counts=lambda: (base >> np.uint32(16)).astype(np.int64))


def erode(field: np.ndarray) -> np.ndarray:
    res = field.shape[0]
    if field.shape != (res, res, res):
        raise ValueError("field must be cubic")
    f = np.ascontiguousarray(field, dtype=np.float64)
    out = np.empty_like(f)
    lib().orc_erode(_p(f), C.c_int(res), _p(out))
    return out


def compute_visibility(eroded, g, cam, occupied):
    """culling.py:203-225 -> namespace(levels, base, flat)"""
    res = g.resolution
    if eroded.shape != (res, res, res) or occupied.shape != (res, res, res):
        raise ValueError("field shape does not match grid")
    cv = g.to_voxel(cam.position)
    occ = np.ascontiguousarray(occupied != 0, dtype=np.uint8)
    er = np.ascontiguousarray(eroded, dtype=np.float64)
    vis = np.empty((res, res, res), dtype=np.uint8)
    lib().orc_visibility(_p(er), _p(occ), C.c_int(res), _d(cv[0]), _d(cv[1]), _d(cv[2]),
                         _d(THETA_BLOCK), _p(vis))
    offs = level_offsets(res)
    flat = np.zeros(int(offs[-1]), dtype=np.uint8)
    lib().orc_dilate_and(_p(vis), _p(occ), C.c_int(res), _p(flat))
    return culling_from_bits(flat[:res ** 3].reshape(res, res, res), _flat=flat)


def culling_from_bits(base, _flat=None):
    """culling.py:76-78, 103-109"""
    res = base.shape[0]
    offs = level_offsets(res)
    if _flat is None:
        _flat = np.zeros(int(offs[-1]), dtype=np.uint8)
        _flat[:res ** 3] = (base != 0).ravel()
    lib().orc_or_mips(_p(_flat), C.c_int(res))
    levels = _split_levels(_flat, res)
    return SimpleNamespace(levels=levels, base=levels[0], flat=_flat, offs=offs, resolution=res)


def scan_offsets(pyramid, culling=None, capacity=None):
    """abuffer.py:104-114"""
    V = pyramid.base.size
    offsets = np.empty(V, dtype=np.int64)
    counts = np.empty(V, dtype=np.int64)
    cb = None if culling is None else np.ascontiguousarray(culling.base.ravel())
    total = int(lib().orc_scan_offsets(_p(pyramid.base), _p(cb), C.c_int64(V), _p(offsets), _p(counts)))
    if capacity is not None and total > capacity:
        raise OracleABufferError(f"fragment total {total} exceeds capacity {capacity}")
    return SimpleNamespace(offsets=offsets, counts=counts, total=total)


def _second_pass(ls, cn, g, pyramid, culling, method, r_world):
    verts, segs, _, _, r = segment_arrays(ls, cn, g, r_world)
    rt = footprint_radius(r, pyramid.r_min)
    res = g.resolution
    table = scan_offsets(pyramid, culling)
    use_cull = culling is not None
    if use_cull:
        cull_flat, cull_offs, n_levels = culling.flat, culling.offs, len(culling.levels)
    else:
        cull_flat, cull_offs, n_levels = np.zeros(1, np.uint8), np.zeros(2, np.int64), 1
    frags = np.zeros(table.total, dtype=np.uint32)
    inc = C.c_int64(0)
    rc = lib().orc_second_pass(_p(verts), _p(segs), C.c_int64(len(segs)), _d(rt), C.c_int(res),
                               C.c_int(METHODS[method]), C.c_int(use_cull), _p(cull_flat), _p(cull_offs),
                               C.c_int(n_levels), _p(table.offsets), _p(table.counts),
                               C.c_int64(table.total), C.c_int(pyramid.saturated == 0), _p(frags),
                               C.byref(inc))
    if rc != 0:
        raise OracleABufferError("fragment count mismatch between passes")
    stats = {"incidences": int(inc.value), "fragment_touches": 2 * int(inc.value),
             "fragments": table.total}
    return SimpleNamespace(table=table, fragments=frags, resolution=res, stats=stats, total=table.total)


def build_vsv(ls, cn, g, pyramid, method="capsule", workers=None, r_world=None):
    return _second_pass(ls, cn, g, pyramid, None, method, r_world)


def build_vcsv(ls, cn, g, pyramid, culling, method="capsule", workers=None, r_world=None):
    return _second_pass(ls, cn, g, pyramid, culling, method, r_world)


def cone_directions() -> np.ndarray:
    """shading.py:32-40 (same numpy expression so the bits match)"""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    dirs = []
    for a in (-1.0, 1.0):
        for b in (-phi, phi):
            dirs += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    d = np.array(dirs)
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def compute_shading(pyramid, culling, g, light_dir):
    """shading.py:170-185"""
    res = g.resolution
    light = np.asarray(light_dir, dtype=np.float64)
    light = light / np.linalg.norm(light)
    ao = np.empty((res, res, res), dtype=np.float32)
    sh = np.empty((res, res, res), dtype=np.float32)
    dirs = np.ascontiguousarray(cone_directions())
    vis = np.ascontiguousarray(culling.base)
    lib().orc_shading(_p(pyramid.occ_flat), C.c_int(res), _p(vis), _p(dirs), C.c_int(len(dirs)),
                      _d(np.tan(AO_HALF_ANGLE)), _d(light[0]), _d(light[1]), _d(light[2]),
                      _d(np.tan(SHADOW_HALF_ANGLE)), _p(ao), _p(sh))
    return SimpleNamespace(ao=ao, shadow=sh, light_dir=light)


def to_srgb(linear: np.ndarray) -> np.ndarray:
    """raytracer.py:94-97"""
    c = np.clip(linear, 0.0, 1.0)
    s = np.where(c <= 0.0031308, 12.92 * c, 1.055 * np.power(c, 1.0 / 2.4) - 0.055)
    return np.rint(s * 255.0).astype(np.uint8)


def render(ls, cn, g, pyramid, abuf, shading, culling, cam, mode="opaque", alpha=1.0, k=8,
           background=(0.1, 0.1, 0.12), early_termination=True, r_world=None):
    """raytracer.py:671-706"""
    res = g.resolution
    verts, _, normals, use_clip, r = segment_arrays(ls, cn, g, r_world)
    bits = culling if culling is not None else \
        culling_from_bits((pyramid.counts() > 0).astype(np.uint8))
    if shading is not None:
        ao, sh = np.ascontiguousarray(shading.ao), np.ascontiguousarray(shading.shadow)
        light = np.asarray(shading.light_dir, dtype=np.float64)
    else:
        ao = sh = None
        light = np.array([0.0, 0.0, -1.0])
    to_src = np.ascontiguousarray(-light)
    pos = np.ascontiguousarray(g.to_voxel(cam.position))
    w, h = cam.width, cam.height
    rgb = np.zeros((h, w, 3), dtype=np.float64)
    hit = np.zeros((h, w), dtype=np.int32)
    tests = np.zeros((h, w), dtype=np.int64)
    fwd, right, up = (np.ascontiguousarray(v, dtype=np.float64) for v in (cam.forward, cam.right, cam.up))
    bg = np.asarray(background, dtype=np.float64)
    lib().orc_render(_p(verts), _p(normals), C.c_int(use_clip), _d(r), _p(abuf.table.offsets),
                     _p(abuf.table.counts), _p(abuf.fragments), _p(bits.flat), C.c_int(res),
                     _p(ao), _p(sh), _p(to_src), _p(pos), _p(fwd), _p(right), _p(up),
                     _d(np.tan(cam.fov / 2.0)), C.c_int(0 if mode == "opaque" else 1), _d(alpha),
                     C.c_int(k), C.c_int(bool(early_termination)), _p(bg), C.c_int(w), C.c_int(h),
                     _p(rgb), _p(hit), _p(tests))
    return SimpleNamespace(rgb=rgb, hit_id=hit, stats={"ray_capsule_tests": int(tests.sum())},
                           srgb=to_srgb(rgb), width=w, height=h)


def run_frame(ls, g, r_world, cam, light, strategy="vcsv", mode="opaque", alpha=1.0, k=8,
              r_min=0.5, method="capsule", cn="auto", timings=None):
    """pipeline.py:68-136 in one call; returns every intermediate.  `timings` (dict) receives
    per-stage wall ms with the reference's stat keys."""
    import time
    t = [time.perf_counter()]

    def tick():
        t.append(time.perf_counter())
        return 1e3 * (t[-1] - t[-2])
    if isinstance(cn, str):
        cn = compute_clip_normals(ls)
    ms = {"normals_ms": tick()}
    pyr = voxelize(ls, cn, g, method=method, r_min=r_min, r_world=r_world)
    ms["voxelize_ms"] = tick()
    culling = None
    if strategy == "vcsv":
        eroded = erode(pyr.occ_levels[0])
        culling = compute_visibility(eroded, g, cam, pyr.counts() > 0)
    ms["cull_ms"] = tick()
    if strategy == "vsv":
        abuf = build_vsv(ls, cn, g, pyr, method=method, r_world=r_world)
    else:
        abuf = build_vcsv(ls, cn, g, pyr, culling, method=method, r_world=r_world)
    ms["abuffer_ms"] = tick()
    shade_bits = culling if culling is not None else \
        culling_from_bits((pyr.counts() > 0).astype(np.uint8))
    shading = compute_shading(pyr, shade_bits, g, light)
    ms["shading_ms"] = tick()
    img = render(ls, cn, g, pyr, abuf, shading, culling, cam, mode=mode, alpha=alpha, k=k, r_world=r_world)
    ms["render_ms"] = tick()
    if timings is not None:
        timings.update(ms)
    return SimpleNamespace(cn=cn, pyramid=pyr, culling=culling, shade_bits=shade_bits, abuf=abuf,
                           shading=shading, image=img)
