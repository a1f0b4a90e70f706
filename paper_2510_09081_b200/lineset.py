"""Line-set model and procedural generators (host side).

Mirrors the data model of the reference (`pkg/src/linevox/lineset.py:39-101`): one flat
f32 vertex buffer, polyline offsets with a terminal sentinel and one shared world-space
radius.  Segment ``i`` is the capsule v_i -> v_{i+1}; the last vertex of each polyline
starts no segment.  This module is input plumbing only; the per-frame work (voxel-unit
conversion, clip normals, AABB) runs on the GPU, see :mod:`.upload`.

The generators reproduce the reference's RNG call order (``lineset.py:277-329``) so a
given ``seed`` yields the same vertices in both packages; ``bundles`` is new (SURVEY.md
§8(d), config C2/C4) and exists only here.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = ["LineSet", "Capsule", "LineSetError", "ParseError", "generate", "decimate",
           "load_lineset", "save_lineset"]


class LineSetError(ValueError):
    pass


class ParseError(LineSetError):
    pass


@dataclass
class LineSet:
    vertices: np.ndarray          # (N, 3) float32, world units
    polyline_offsets: np.ndarray  # (P+1,) int64: 0 = o_0 < o_1 < ... < o_P = N
    radius: float                 # world units, > 0

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float32)
        self.polyline_offsets = np.ascontiguousarray(self.polyline_offsets, dtype=np.int64)
        self.validate()

    def validate(self) -> None:
        o = self.polyline_offsets
        nv = len(self.vertices)
        if self.vertices.ndim != 2 or self.vertices.shape[1] != 3:
            raise LineSetError("vertices must have shape (N, 3)")
        if o.ndim != 1 or o.size < 2 or o[0] != 0 or o[-1] != nv:
            raise LineSetError("polyline offsets must start at 0 and end at the vertex count")
        if (np.diff(o) < 2).any():
            raise LineSetError("every polyline needs at least 2 vertices")
        if not self.radius > 0:
            raise LineSetError("radius must be positive")
        if not np.isfinite(self.vertices).all():
            raise LineSetError("non-finite vertex coordinate")

    @property
    def n_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def n_polylines(self) -> int:
        return int(self.polyline_offsets.size - 1)

    @property
    def n_segments(self) -> int:
        return self.n_vertices - self.n_polylines

    def segment_vertex_ids(self) -> np.ndarray:
        """Start-vertex index of every segment, ascending (host copy; the device builds
        its own in `lvx_upload`)."""
        keep = np.ones(self.n_vertices, dtype=bool)
        keep[self.polyline_offsets[1:] - 1] = False
        return np.flatnonzero(keep).astype(np.int64)

    def aabb(self):
        v = self.vertices
        return v.min(axis=0).astype(np.float64), v.max(axis=0).astype(np.float64)


@dataclass
class Capsule:
    """One thick segment with its two clip-plane normals (reference `lineset.py:85-101`)."""
    v0: np.ndarray
    v1: np.ndarray
    r: float
    n0: np.ndarray
    n1: np.ndarray

    def __post_init__(self):
        for k in ("v0", "v1", "n0", "n1"):
            setattr(self, k, np.asarray(getattr(self, k), dtype=np.float64))
        if not self.r > 0:
            raise LineSetError("capsule radius must be positive")


# --------------------------------------------------------------------------- generators

def _helix(turns=2.0, verts=100, coil_radius=4.0, pitch=2.0, radius=0.25):
    if verts < 2 or turns <= 0 or radius <= 0:
        raise LineSetError("helix needs verts >= 2, turns > 0, radius > 0")
    ang = np.linspace(0.0, 2.0 * np.pi * turns, verts)
    pts = np.stack([coil_radius * np.cos(ang), coil_radius * np.sin(ang),
                    pitch * ang / (2.0 * np.pi)], axis=1)
    return LineSet(pts.astype(np.float32), np.array([0, verts]), radius)


def _walk(rng, n_verts, lo, hi, seg_length, curl):
    """One reflected random walk; consumes rng exactly like reference lineset.py:297-310."""
    p = rng.uniform(lo, hi, size=3)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    out = np.empty((n_verts, 3))
    out[0] = p
    for j in range(1, n_verts):
        d = d + curl * rng.normal(size=3)
        d /= np.linalg.norm(d)
        p = p + seg_length * d
        for a in range(3):
            if p[a] < lo or p[a] > hi:
                d[a] = -d[a]
                p[a] = np.clip(p[a], lo, hi)
        out[j] = p
    return out


def _walks_vectorised(rng, polylines, n_verts, lo, hi, seg_length, curl):
    """All polylines' walks advanced together, one vertex per step.  The random numbers are drawn polyline by
    polyline in `_walk`'s order (uniform start, then a normal triple per vertex: a Generator's stream does not
    depend on how a request is batched) and every arithmetic step is `_walk`'s, element for element; the vector
    norms go through a batched matmul, which rounds like the `x.dot(x)` inside np.linalg.norm (an explicit
    x0*x0 + x1*x1 + x2*x2 does not).  The caller checks the first polylines against `_walk` itself."""
    p = np.empty((polylines, 3))
    nrm = np.empty((polylines, n_verts, 3))
    for i in range(polylines):
        p[i] = rng.uniform(lo, hi, size=3)
        nrm[i] = rng.normal(size=(n_verts, 3))

    def unit(v):
        return v / np.sqrt(np.matmul(v[:, None, :], v[:, :, None]).reshape(-1, 1))

    d = unit(nrm[:, 0])
    out = np.empty((polylines, n_verts, 3))
    out[:, 0] = p
    for j in range(1, n_verts):
        d = unit(d + curl * nrm[:, j])
        p = p + seg_length * d
        bad = (p < lo) | (p > hi)
        d = np.where(bad, -d, d)
        p = np.where(bad, np.clip(p, lo, hi), p)
        out[:, j] = p
    return out.reshape(-1, 3)


def _random_streamlines(polylines=50, verts_per_line=30, seg_length=1.0, domain=32.0,
                        radius=0.25, curl=0.6, seed=0):
    if polylines < 1 or verts_per_line < 2 or seg_length <= 0 or radius <= 0:
        raise LineSetError("bad random_streamlines parameters")
    lo, hi = 0.2 * domain, 0.8 * domain
    off = np.arange(polylines + 1, dtype=np.int64) * verts_per_line
    if polylines >= 64:      # large sets (C5's time steps: 20 000 polylines): ~40x faster than walk by walk
        v = _walks_vectorised(np.random.default_rng(seed), polylines, verts_per_line, lo, hi, seg_length, curl)
        rng = np.random.default_rng(seed)
        head = np.concatenate([_walk(rng, verts_per_line, lo, hi, seg_length, curl) for _ in range(2)])
        if np.array_equal(v[:head.shape[0]], head):      # bit for bit the reference's walk on this platform
            return LineSet(v.astype(np.float32), off, radius)
    rng = np.random.default_rng(seed)
    v = np.concatenate([_walk(rng, verts_per_line, lo, hi, seg_length, curl)
                        for _ in range(polylines)])
    return LineSet(v.astype(np.float32), off, radius)


def _grid_diagonals(count=64, length=16.0, domain=128.0, radius=0.2, seed=0):
    if count < 1 or length <= 0 or radius <= 0 or domain <= length + 4:
        raise LineSetError("bad grid_diagonals parameters")
    rng = np.random.default_rng(seed)
    a = rng.uniform(2.0, domain - length - 2.0, size=(count, 3))
    v = np.empty((2 * count, 3), dtype=np.float32)
    v[0::2] = a
    v[1::2] = a + length
    return LineSet(v, np.arange(count + 1, dtype=np.int64) * 2, radius)


def _bundles(n_bundles=40, fibers=250, verts=101, seg_length=1.0, domain=128.0,
             radius=0.25, curl=0.15, spread=3.0, jitter=0.05, seed=0):
    """Tractography-like fibre bundles: every bundle follows one
    low-curl random-walk centreline; a fibre is the centreline plus a constant offset drawn
    uniformly from a ball of radius `spread` plus per-vertex N(0, jitter^2) noise.
    Vectorised so that 10 M-segment sets build in seconds."""
    if n_bundles < 1 or fibers < 1 or verts < 2 or radius <= 0:
        raise LineSetError("bad bundles parameters")
    rng = np.random.default_rng(seed)
    lo, hi = 0.2 * domain, 0.8 * domain
    chunks = []
    for _ in range(n_bundles):
        centre = _walk(rng, verts, lo, hi, seg_length, curl)
        u = rng.normal(size=(fibers, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        off = u * (spread * rng.uniform(size=(fibers, 1)) ** (1.0 / 3.0))
        pts = centre[None, :, :] + off[:, None, :] + jitter * rng.normal(size=(fibers, verts, 3))
        chunks.append(pts.reshape(-1, 3).astype(np.float32))
    v = np.concatenate(chunks)
    offs = np.arange(n_bundles * fibers + 1, dtype=np.int64) * verts
    return LineSet(v, offs, radius)


_GENERATORS = {"helix": (_helix, False), "random_streamlines": (_random_streamlines, True),
               "grid_diagonals": (_grid_diagonals, True), "bundles": (_bundles, True)}


def generate(kind: str, seed: int = 0, **params) -> LineSet:
    """Deterministic procedural line sets (reference `lineset.py:266-274` + ``bundles``)."""
    if kind not in _GENERATORS:
        raise LineSetError(f"unknown generator kind {kind!r}")
    fn, seeded = _GENERATORS[kind]
    return fn(seed=seed, **params) if seeded else fn(**params)


def decimate(ls: LineSet, n: int) -> LineSet:
    """Every n-th vertex of each polyline, last vertex always kept."""
    if n < 1:
        raise LineSetError("decimation step must be >= 1")
    o = ls.polyline_offsets
    picks, offs = [], [0]
    for s, e in zip(o[:-1], o[1:]):
        idx = np.arange(s, e, n)
        if idx[-1] != e - 1:
            idx = np.append(idx, e - 1)
        picks.append(idx)
        offs.append(offs[-1] + idx.size)
    return LineSet(ls.vertices[np.concatenate(picks)], np.asarray(offs), ls.radius)


# --------------------------------------------------------------------------- .lns files
# Binary layout (reference lineset.py:172-200): "LNS1", u32 n_poly, u32 n_vert, f32 radius,
# u32 offsets[n_poly+1], f32 xyz[n_vert].  Text: "lns 1 radius=<r>", "v x y z" lines,
# blank line closes a polyline.

_MAGIC = b"LNS1"


def save_lineset(ls: LineSet, path, fmt: str = "lns-binary") -> None:
    path = Path(path)
    if fmt == "lns-binary":
        path.write_bytes(_MAGIC + struct.pack("<IIf", ls.n_polylines, ls.n_vertices, ls.radius)
                         + ls.polyline_offsets.astype("<u4").tobytes()
                         + ls.vertices.astype("<f4").tobytes())
    elif fmt == "lns-text":
        rows = [f"lns 1 radius={float(ls.radius)!r}"]
        o = ls.polyline_offsets
        for s, e in zip(o[:-1], o[1:]):
            rows += [f"v {float(x)!r} {float(y)!r} {float(z)!r}" for x, y, z in ls.vertices[s:e]]
            rows.append("")
        path.write_text("\n".join(rows) + "\n")
    else:
        raise ValueError(f"unknown line-set format {fmt!r}")


def load_lineset(path, fmt: str | None = None) -> LineSet:
    path = Path(path)
    raw = path.read_bytes()
    if fmt is None:
        fmt = "lns-binary" if raw[:4] == _MAGIC else "lns-text"
    try:
        if fmt == "lns-binary":
            if raw[:4] != _MAGIC:
                raise ParseError(f"{path}: byte 0: bad magic (want LNS1)")
            if len(raw) < 16:
                raise ParseError(f"{path}: byte {len(raw)}: truncated header")
            n_poly, n_vert, radius = struct.unpack_from("<IIf", raw, 4)
            if n_poly == 0:
                raise ParseError(f"{path}: byte 4: no polylines")
            want = 16 + 4 * (n_poly + 1) + 12 * n_vert
            if len(raw) != want:
                raise ParseError(f"{path}: byte {len(raw)}: expected {want} bytes")
            off = np.frombuffer(raw, "<u4", n_poly + 1, 16).astype(np.int64)
            v = np.frombuffer(raw, "<f4", 3 * n_vert, 16 + 4 * (n_poly + 1)).reshape(n_vert, 3)
            return LineSet(v.copy(), off, float(radius))
        if fmt == "lns-text":
            return _parse_text(raw, path)
    except ParseError:
        raise
    except LineSetError as e:
        raise ParseError(f"{path}: {e}") from None
    raise ValueError(f"unknown line-set format {fmt!r}")


def _parse_text(raw: bytes, path: Path) -> LineSet:
    rows = raw.decode("ascii", errors="replace").splitlines()
    if not rows:
        raise ParseError(f"{path}: empty file, no polylines")
    head = rows[0].split()
    if len(head) != 3 or head[:2] != ["lns", "1"] or not head[2].startswith("radius="):
        raise ParseError(f"{path}:1: malformed header (want 'lns 1 radius=<float>')")
    try:
        radius = float(head[2][7:])
    except ValueError:
        raise ParseError(f"{path}:1: malformed radius") from None
    pts, offs, start = [], [0], 0

    def close(ln):
        nonlocal start
        if len(pts) - start < 2:
            raise ParseError(f"{path}:{ln}: polyline with fewer than 2 vertices")
        offs.append(len(pts))
        start = len(pts)

    for ln, row in enumerate(rows[1:], 2):
        tok = row.split()
        if not tok:
            if len(pts) > start:
                close(ln)
            continue
        if tok[0] != "v" or len(tok) != 4:
            raise ParseError(f"{path}:{ln}: expected 'v x y z'")
        try:
            xyz = [float(t) for t in tok[1:]]
        except ValueError:
            raise ParseError(f"{path}:{ln}: bad coordinate") from None
        if not np.isfinite(xyz).all():
            raise ParseError(f"{path}:{ln}: non-finite coordinate")
        pts.append(xyz)
    if len(pts) > start:
        close(len(rows))
    if len(offs) < 2:
        raise ParseError(f"{path}: no polylines")
    return LineSet(np.asarray(pts, dtype=np.float32), np.asarray(offs), radius)
