"""Pinhole camera (reference `pkg/src/linevox/culling.py:30-67`)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Camera"]


@dataclass
class Camera:
    position: np.ndarray
    forward: np.ndarray
    up: np.ndarray
    fov: float = float(np.deg2rad(45.0))  # vertical, radians
    width: int = 256
    height: int = 256

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        if not 0.0 < self.fov < np.pi:
            raise ValueError("fov must be in (0, pi)")
        f = np.asarray(self.forward, dtype=np.float64)
        fl = np.linalg.norm(f)
        if fl == 0:
            raise ValueError("forward must be nonzero")
        f = f / fl
        u = np.asarray(self.up, dtype=np.float64)
        u = u - (u @ f) * f
        ul = np.linalg.norm(u)
        if ul == 0:
            raise ValueError("up must not be parallel to forward")
        self.forward = f
        self.up = u / ul

    @property
    def right(self) -> np.ndarray:
        return np.cross(self.forward, self.up)

    @classmethod
    def orbit(cls, target, distance, azimuth, elevation, fov=float(np.deg2rad(45.0)),
              width=256, height=256) -> "Camera":
        target = np.asarray(target, dtype=np.float64)
        ce = np.cos(elevation)
        pos = target + distance * np.array([ce * np.cos(azimuth), ce * np.sin(azimuth),
                                            np.sin(elevation)])
        return cls(pos, target - pos, np.array([0.0, 0.0, 1.0]), fov, width, height)
