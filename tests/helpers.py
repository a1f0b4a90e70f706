"""Shared test helpers: golden-scene loading and hashing (no reference import)."""
import hashlib
import json
import os

import numpy as np

from paper_2510_09081_b200.camera import Camera
from paper_2510_09081_b200.grid import GridDesc
from paper_2510_09081_b200.lineset import LineSet

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = ["helix32_vsv", "helix64_vcsv", "c1_vcsv", "c1_vsv_transparent", "diag_vcsv",
          "walk32_transp_k2", "walk32_inside_cam", "diag32_thick_vsv"]
FULL_SCENES = ["helix32_vsv", "walk32_transp_k2", "walk32_inside_cam", "diag32_thick_vsv"]


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def fh(s) -> float:
    return float.fromhex(s)


class Scene:
    def __init__(self, name):
        self.name = name
        with open(os.path.join(GOLDEN, name + ".json")) as f:
            self.meta = json.load(f)
        self.arr = np.load(os.path.join(GOLDEN, name + ".npz"))
        m = self.meta
        self.ls = LineSet(self.arr["vertices"], self.arr["polyline_offsets"], float(self.arr["radius"]))
        self.g = GridDesc(m["grid"]["res"], np.array([fh(x) for x in m["grid"]["world_min"]]),
                          fh(m["grid"]["voxel_size"]))
        self.r_world = fh(m["r_world"])
        self.r_min = fh(m["r_min"])
        c = m["camera"]
        self.cam = Camera(np.array([fh(x) for x in c["position"]]), np.array([fh(x) for x in c["forward"]]),
                          np.array([fh(x) for x in c["up"]]), fh(c["fov"]), c["width"], c["height"])
        # Camera.__post_init__ re-normalises; that is not idempotent to the last bit, so put
        # the reference's exact basis back (the fixture stores the post-init values).
        self.cam.forward = np.array([fh(x) for x in c["forward"]])
        self.cam.up = np.array([fh(x) for x in c["up"]])
        self.light = np.array([fh(x) for x in m["light"]])
        self.mode = m["settings"]["mode"]
        self.alpha = fh(m["settings"]["alpha"])
        self.k = m["settings"]["k"]
        self.strategy = m["strategy"]
        self.hash = m["hash"]
        self.stats = m["stats"]
