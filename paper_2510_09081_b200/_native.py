"""ctypes binding of ``liblvx_b200.so`` (the C ABI declared in ``include/lvx.h``).

There is no CPU fallback: if the shared library is missing, or no CUDA device is present when a
kernel is requested, the call raises.  The library is built in-tree by
``paper_2510_09081_b200/csrc/build.sh`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LVX_LIB selects an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("LVX_LIB") or os.path.join(_HERE, "liblvx_b200.so")

# stats block indices (include/lvx.h)
ST_VISITED, ST_SATURATED, ST_NEED_WIDE, ST_SOLID, ST_FRAG_TOTAL, ST_MISMATCH, ST_RAY_TESTS, \
    ST_LONG_LISTS, ST_DEGENERATE, ST_VISIBLE, ST_OCCUPIED, ST_OCC_SAT = range(12)
ST_OWNED = 13
ST_BRICK_PAIRS = 16
STATS_WORDS = 24


class lvx_camera(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("fwd", C.c_double * 3), ("right", C.c_double * 3),
                ("up", C.c_double * 3), ("tan_half_fov", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class lvx_render_params(C.Structure):
    _fields_ = [("mode", C.c_int32), ("k", C.c_int32), ("early_termination", C.c_int32),
                ("use_clip", C.c_int32), ("alpha", C.c_double), ("background", C.c_double * 3),
                ("light_to_source", C.c_double * 3), ("radius", C.c_double),
                ("tile_x0", C.c_int32), ("tile_y0", C.c_int32), ("tile_x1", C.c_int32),
                ("tile_y1", C.c_int32)]


_P, _I, _L, _D = C.c_void_p, C.c_int, C.c_int64, C.c_double

# name -> (restype, argtypes); mirrors include/lvx.h one to one
SIGNATURES = {
    "lvx_last_cuda_error": (C.c_char_p, []),
    "lvx_version": (_I, []),
    "lvx_stats_reset": (_I, [_P, _P]),
    "lvx_num_levels": (_I, [_I]),
    "lvx_pyramid_elems": (_L, [_I]),
    "lvx_upload": (_I, [_P, _P, _L, _L, _P, _D, _P, _P, _P, _P, _P, _P]),
    "lvx_aabb": (_I, [_P, _L, _P, _P]),
    "lvx_clear": (_I, [_P, _L, _P]),
    "lvx_voxelize": (_I, [_P, _P, _P, _L, _L, _I, _D, _D, _D, _I, _I, _P, _P, _P, _P]),
    "lvx_voxelize_wide": (_I, [_P, _P, _P, _L, _L, _I, _D, _D, _D, _I, _I, _P, _P, _P]),
    "lvx_widen": (_I, [_P, _P, _L, _P, _P]),
    "lvx_wide_field_max": (_I, [_P, _L, _P, _P, _P]),
    "lvx_base_mip1": (_I, [_P, _I, _P, _P, _P]),
    "lvx_pack_wide": (_I, [_P, _L, _P, _P, _P, _P]),
    "lvx_pack_wide_mip1": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "lvx_finalize_base": (_I, [_P, _P, _L, _P, _P]),
    "lvx_build_mips": (_I, [_P, _I, _P, _P]),
    "lvx_build_mips_upper": (_I, [_I, _P, _P]),
    "lvx_cull_scratch_words": (_L, [_I]),
    "lvx_cull": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "lvx_occupied_pyramid": (_I, [_P, _I, _P, _P, _P, _P]),
    "lvx_list_words": (_L, [_L]),
    "lvx_tile_owners": (_I, [_P, _I, _P, _I, _I, _I, _I, _D, _P, _P, _P, _P]),
    "lvx_scan_scratch_bytes": (_L, [_L]),
    "lvx_scan": (_I, [_P, _P, _L, _P, _P, _P, _P, _P]),
    "lvx_max_fragments": (_L, []),
    "lvx_segment_order_scratch_words": (_L, [_L, _I, _I]),
    "lvx_segment_order": (_I, [_P, _P, _L, _I, _I, _P, _P, _P]),
    "lvx_scatter": (_I, [_P, _P, _L, _D, _D, _I, _I, _P, _P, _P, _P, _P, _L, _P, _P, _P, _I, _P, _P]),
    "lvx_brick_scratch_words": (_L, [_I, _L]),
    "lvx_build_lists": (_I, [_P, _P, _L, _D, _D, _I, _P, _P, _P, _L, _P, _P, _P, _P, _L, _P, _P]),
    "lvx_march_levels": (_I, [_P, _I, _P, _P]),
    "lvx_shade_scratch_bytes": (_L, [_L]),
    "lvx_shade": (_I, [_P, _P, _I, _P, _P, _I, _D, _P, _D, _P, _P, _I, _P, _P, _P]),
    "lvx_trace_hits": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lvx_resolve": (_I, [_P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lvx_render": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
}

_lib = None


class LvxError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """The loaded library; raises LvxError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LvxError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(paper_2510_09081_b200/csrc/build.sh); there is no CPU fallback")
        l = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc == -2:
        raise LvxError(f"{what}: CUDA error: {lib().lvx_last_cuda_error().decode()}")
    raise LvxError(f"{what}: invalid argument (status {rc})")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise LvxError("no CUDA device: the B200 path has no CPU fallback")
    lib()
    return torch
