"""GPU cone-traced AO + directional shadow with the reference's call surface
(lv/shading.py:21-22: ``ConeSet``, ``ShadingVolume``, ``cone_directions``, ``compute_shading``)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import ops

__all__ = ["ConeSet", "ShadingVolume", "cone_directions", "compute_shading", "AO_HALF_ANGLE",
           "SHADOW_HALF_ANGLE"]

AO_HALF_ANGLE = float(np.arccos(1.0 - 2.0 / 12.0))   # lv/shading.py:25
SHADOW_HALF_ANGLE = float(np.deg2rad(5.0))           # lv/shading.py:26


def cone_directions() -> np.ndarray:
    """The 12 icosahedron vertex directions (lv/shading.py:32-40), in the reference's order:
    for a in (-1,1), b in (-phi,phi): (0,a,b), (a,b,0), (b,0,a)."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    rows = [v for a in (-1.0, 1.0) for b in (-phi, phi) for v in ((0.0, a, b), (a, b, 0.0), (b, 0.0, a))]
    d = np.array(rows)
    return d / np.linalg.norm(d, axis=1, keepdims=True)


@dataclass(frozen=True)
class ConeSet:
    directions: np.ndarray
    half_angle: float

    @property
    def weight(self) -> float:
        return 1.0 / len(self.directions)

    @classmethod
    def ambient(cls) -> "ConeSet":
        return cls(cone_directions(), AO_HALF_ANGLE)


class ShadingVolume:
    """lv/shading.py:57-61; `ao_dev` / `shadow_dev` are (V,) f32 on the GPU."""

    def __init__(self, ao_dev, shadow_dev, light_dir, resolution):
        self.ao_dev, self.shadow_dev, self.light_dir, self._res = ao_dev, shadow_dev, light_dir, resolution

    @property
    def ao(self) -> np.ndarray:
        return self.ao_dev.cpu().numpy().reshape((self._res,) * 3)

    @property
    def shadow(self) -> np.ndarray:
        return self.shadow_dev.cpu().numpy().reshape((self._res,) * 3)


def compute_shading(pyramid, culling, g, light_dir) -> ShadingVolume:
    """lv/shading.py:170-185"""
    torch = N.require_cuda()
    res = g.resolution
    light = np.asarray(light_dir, dtype=np.float64)
    light = light / np.linalg.norm(light)
    dev = pyramid.base_dev.device
    V = res ** 3
    ao = torch.empty(V, dtype=torch.float32, device=dev)
    sh = torch.empty(V, dtype=torch.float32, device=dev)
    scratch = torch.empty(ops.shade_scratch_bytes(V), dtype=torch.uint8, device=dev)
    if culling.list_dev is None:
        from .culling import CullingPyramid
        culling = CullingPyramid.from_bits(culling.base_dev.reshape(res, res, res))
    ops.shade(pyramid.base_dev, pyramid.mips_dev, res, culling.list_dev, cone_directions(),
              np.tan(AO_HALF_ANGLE), light, np.tan(SHADOW_HALF_ANGLE), ao, sh, scratch)
    return ShadingVolume(ao, sh, light, res)
