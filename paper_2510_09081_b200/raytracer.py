"""GPU image-order renderer with the reference's call surface (lv/raytracer.py:26-27:
``RenderSettings``, ``Image``, ``RenderScene``, ``render``, ``tangent_color``, ``AMBIENT``,
``DIFFUSE``)."""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from . import ops
from .camera import Camera
from .culling import CullingPyramid
from .voxelizer import upload_lineset

__all__ = ["RenderSettings", "Image", "RenderScene", "render", "tangent_color", "AMBIENT", "DIFFUSE"]

AMBIENT = 0.4    # lv/raytracer.py:29-30 (compiled into csrc/render.cu)
DIFFUSE = 0.6


@dataclass
class RenderSettings:
    """lv/raytracer.py:51-65"""
    mode: str = "opaque"
    alpha: float = 1.0
    k: int = 8
    background: tuple = (0.1, 0.1, 0.12)
    early_termination: bool = True

    def __post_init__(self):
        if self.mode not in ("opaque", "transparent"):
            raise ValueError(f"unknown render mode {self.mode!r}")
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError("alpha must be in (0, 1]")
        if not 1 <= self.k <= 64:
            raise ValueError("k must be in [1, 64]")


def _to_srgb(linear: np.ndarray) -> np.ndarray:
    """lv/raytracer.py:94-97 (host version, used when only the f64 image was kept)"""
    c = np.clip(linear, 0.0, 1.0)
    s = np.where(c <= 0.0031308, 12.92 * c, 1.055 * np.power(c, 1.0 / 2.4) - 0.055)
    return np.rint(s * 255.0).astype(np.uint8)


class Image:
    """lv/raytracer.py:68-91.  `rgb_dev` (H,W,3) f64 linear, `srgb_dev` (H,W,3) u8 (converted in
    the render kernel), `hit_id_dev` (H,W) i32."""

    def __init__(self, rgb_dev, srgb_dev, hit_id_dev, stats=None):
        self.rgb_dev, self.srgb_dev, self.hit_id_dev = rgb_dev, srgb_dev, hit_id_dev
        self.stats = stats or {}
        self._rgb = self._hit = None

    @property
    def rgb(self) -> np.ndarray:
        if self._rgb is None:
            self._rgb = self.rgb_dev.cpu().numpy()
        return self._rgb

    @property
    def hit_id(self) -> np.ndarray:
        if self._hit is None:
            self._hit = self.hit_id_dev.cpu().numpy()
        return self._hit

    @property
    def width(self) -> int:
        return int(self.hit_id_dev.shape[1])

    @property
    def height(self) -> int:
        return int(self.hit_id_dev.shape[0])

    def srgb_bytes(self) -> bytes:
        if self.srgb_dev is not None:
            return self.srgb_dev.cpu().numpy().tobytes()
        return _to_srgb(self.rgb).tobytes()

    def save_ppm(self, path) -> None:
        Path(path).write_bytes(f"P6\n{self.width} {self.height}\n255\n".encode() + self.srgb_bytes())

    def save_hit_ids(self, path) -> None:
        Path(path).write_bytes(b"HITI" + struct.pack("<II", self.width, self.height)
                               + self.hit_id.astype("<i4").tobytes())


def tangent_color(d) -> np.ndarray:
    """lv/raytracer.py:100-106"""
    d = np.asarray(d, dtype=np.float64)
    n = np.linalg.norm(d)
    return np.array([0.5, 0.5, 0.5]) if n == 0 else np.abs(d) / n


@dataclass
class RenderScene:
    """lv/raytracer.py:652-668"""
    ls: "object"
    cn: "object"
    g: "object"
    pyramid: "object"
    abuf: "object"
    shading: "object"
    culling: "object" = None
    r_world: float = None
    _march: "object" = field(default=None, repr=False)

    def march_bits(self) -> CullingPyramid:
        if self.culling is not None:
            return self.culling
        if self._march is None:
            from .culling import occupied_bits
            self._march = occupied_bits(self.pyramid)
        return self._march


def make_params(settings: RenderSettings, lines, light_dir, tile=None, width=None, height=None):
    p = N.lvx_render_params()
    p.mode = 0 if settings.mode == "opaque" else 1
    p.k = int(settings.k)
    p.early_termination = int(bool(settings.early_termination))
    p.use_clip = int(lines.use_clip)
    p.alpha = float(settings.alpha)
    p.background[:] = [float(x) for x in settings.background]
    p.light_to_source[:] = [-float(x) for x in light_dir]             # lv/raytracer.py:689
    p.radius = float(lines.r)
    x0, y0, x1, y1 = tile if tile is not None else (0, 0, width, height)
    p.tile_x0, p.tile_y0, p.tile_x1, p.tile_y1 = int(x0), int(y0), int(x1), int(y1)
    return p


def render(scene: RenderScene, cam: Camera, settings: RenderSettings, tile=None, keep_rgb=True) -> Image:
    """lv/raytracer.py:671-706.  `tile` = (x0, y0, x1, y1) restricts tracing to a pixel rect
    (multi-GPU screen tiles); pixels outside are left zero."""
    torch = N.require_cuda()
    g = scene.g
    res = g.resolution
    lines = upload_lineset(scene.ls, g, scene.r_world, scene.cn)
    dev = lines.verts.device
    bits = scene.march_bits()
    if scene.shading is not None:
        ao, sh, light = scene.shading.ao_dev, scene.shading.shadow_dev, scene.shading.light_dir
    else:
        ao = sh = None                                                # all-ones volumes, 685-688
        light = np.array([0.0, 0.0, -1.0])
    w, h = cam.width, cam.height
    rgb = torch.zeros((h, w, 3), dtype=torch.float64, device=dev) if keep_rgb else None
    srgb = torch.zeros((h, w, 3), dtype=torch.uint8, device=dev)
    hit = torch.zeros((h, w), dtype=torch.int32, device=dev)
    stats = ops.new_stats(dev)
    march = torch.empty(res ** 3, dtype=torch.uint8, device=dev)
    ops.march_levels(bits.flat_dev, res, march)
    abuf = scene.abuf
    # the tight index is valid for capsules no thicker than the radius it was built with
    tight = abuf.tight if getattr(abuf, "tight", None) is not None and lines.r <= abuf.tight_radius else None
    ops.render(lines, abuf.table.offsets_dev, abuf.fragments_dev, tight, march, res, ao, sh,
               ops.make_camera_struct(cam, g), make_params(settings, lines, light, tile, w, h),
               rgb, srgb, hit, stats)
    return Image(rgb, srgb, hit, stats={"ray_capsule_tests": int(stats[N.ST_RAY_TESTS].item())})
