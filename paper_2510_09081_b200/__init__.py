"""linevox-b200: the per-frame pipeline of arXiv 2510.09081 (voxel ray tracing of dynamic line
sets) as hand-written sm_100a CUDA kernels behind the reference package's Python API.

Importing the package never touches the GPU; calling any stage without a CUDA device or without
the built `liblvx_b200.so` raises (there is no CPU fallback).  Names mirror
`pkg/src/linevox/__init__.py:9-21` of the reference.
"""
from .abuffer import ABuffer, ABufferError, OffsetTable, build_vcsv, build_vsv, scan_offsets
from .camera import Camera
from .config import ConfigError, PipelineConfig
from .culling import CullingPyramid, compute_visibility, erode
from .frame import FrameEngine
from .grid import GridDesc, fit_grid
from .lineset import (Capsule, LineSet, LineSetError, ParseError, decimate, generate, load_lineset,
                      save_lineset)
from .pipeline import ScenePipeline, make_camera, run_once
from .raytracer import Image, RenderScene, RenderSettings, render, tangent_color
from .shading import ConeSet, ShadingVolume, compute_shading, cone_directions
from .voxelizer import (OccupancyPyramid, compute_clip_normals, footprint_radius, segment_arrays,
                        upload_lineset, voxelize)

__version__ = "0.1.0"
