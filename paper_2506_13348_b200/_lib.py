"""ctypes binding of libtsb.so (include/tsb.h).

The library is built in-tree by paper_2506_13348_b200/csrc/Makefile (see
__graft_entry__.build()). There is no fallback: if the shared library is
missing or fails to load, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TSB_LIB", str(_HERE / "libtsb.so")))

TSB_OK = 0
TSB_ERR_VALUE = -1
TSB_ERR_LOOKUP = -2
TSB_ERR_CUDA = -3
TSB_ERR_CAPACITY = -4

MODE_HW = 0
MODE_VERIFY = 1
MODE_FLAT = 2

TEXEL_RGBA32F = 0
TEXEL_RGBA16F = 1

ENV_MAX_LEVELS = 16


class Camera_t(C.Structure):
    _fields_ = [("world_to_view", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("near_z", C.c_double),
                ("far_z", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class Scene_t(C.Structure):
    _fields_ = [("num_splats", C.c_int32), ("sh_degree", C.c_int32),
                ("positions", C.c_void_p), ("tangent_u", C.c_void_p),
                ("tangent_v", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("sh", C.c_void_p), ("record_slot", C.c_void_p)]


class Atlas_t(C.Structure):
    _fields_ = [("resolution", C.c_int32), ("page_w", C.c_int32), ("page_h", C.c_int32),
                ("pages", C.c_int32), ("entries", C.c_void_p), ("family_a", C.c_void_p),
                ("family_b", C.c_void_p), ("flat_attrs", C.c_void_p), ("tex", C.c_void_p),
                ("texel_stride", C.c_int32)]


class Environment_t(C.Structure):
    _fields_ = [("levels", C.c_int32), ("spec_mips", C.c_void_p * ENV_MAX_LEVELS),
                ("mip_h", C.c_int32 * ENV_MAX_LEVELS), ("mip_w", C.c_int32 * ENV_MAX_LEVELS),
                ("diffuse", C.c_void_p), ("diff_h", C.c_int32), ("diff_w", C.c_int32),
                ("lut", C.c_void_p), ("lut_res", C.c_int32)]


class PixelState_t(C.Structure):
    _fields_ = [("n_contrib", C.c_void_p), ("last_entry", C.c_void_p),
                ("final_T", C.c_void_p), ("T_last", C.c_void_p), ("splat_touched", C.c_void_p)]


class SceneGrads_t(C.Structure):
    _fields_ = [("positions", C.c_void_p), ("tangent_u", C.c_void_p),
                ("tangent_v", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("sh", C.c_void_p), ("texels", C.c_void_p),
                ("texel_layout", C.c_int32)]


TEXELS_COMBINED = 0
TEXELS_INTERLEAVED = 1

ADAM_MAX_GROUPS = 24
F32, F64, F32_TEX87 = 0, 1, 2
CLAMP_NONE, CLAMP_UNIT, CLAMP_FLOOR = 0, 1, 2


class RowBuffer_t(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("row_bytes", C.c_int64)]


class AdamGroup_t(C.Structure):
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p),
                ("v", C.c_void_p), ("count", C.c_int64), ("lr", C.c_double),
                ("floor", C.c_double), ("dtype", C.c_int32), ("clamp", C.c_int32)]


class EnvGrads_t(C.Structure):
    _fields_ = [("spec_mips", C.c_void_p * ENV_MAX_LEVELS), ("diffuse", C.c_void_p)]


_P = C.c_void_p
_SIGNATURES = {
    "tsb_frame_workspace_size": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                 C.POINTER(C.c_uint64)],
    "tsb_frame_workspace_max_needed_offset": [C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int64, C.POINTER(C.c_uint64)],
    "tsb_render_forward": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                           C.c_int32, C.c_int32, _P, C.c_uint64, C.c_int64, _P,
                           C.POINTER(PixelState_t), _P, _P],
    "tsb_render_binning": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                           C.c_int32, C.c_int32, _P, C.c_uint64, C.c_int64, _P, _P],
    "tsb_render_composite": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                             C.c_int32, C.c_int32, _P, C.c_uint64, C.c_int64, _P,
                             C.POINTER(PixelState_t), _P],
    "tsb_frame_export": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _P, _P, _P,
                         _P, _P, _P],
    "tsb_shade_forward": [_P, C.POINTER(Camera_t), C.POINTER(Environment_t), _P, _P, _P, _P, _P],
    "tsb_atlas_tex_create": [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                             C.POINTER(C.c_void_p), _P],
    "tsb_atlas_tex_destroy": [_P],
    "tsb_tex_probe": [_P, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P],
    "tsb_red_probe": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P],
    "tsb_debug_red_count": [C.c_int32, C.POINTER(C.c_ulonglong)],
    "tsb_shade_backward": [_P, C.POINTER(Camera_t), C.POINTER(Environment_t), _P, _P, _P,
                           C.POINTER(EnvGrads_t), _P, C.c_uint64, _P],
    "tsb_shade_backward_scratch_size": [C.POINTER(Environment_t), C.POINTER(C.c_uint64)],
    "tsb_render_backward": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                            C.c_int32, _P, C.c_uint64, C.c_int64, C.POINTER(PixelState_t), _P,
                            _P, C.POINTER(SceneGrads_t), _P],
    "tsb_render_backward_ex": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                               C.c_int32, _P, C.c_uint64, C.c_int64, C.POINTER(PixelState_t),
                               _P, _P, C.POINTER(SceneGrads_t), C.c_int32, _P, C.c_uint64, _P],
    "tsb_backward_scratch_size": [C.c_int32, C.POINTER(C.c_uint64)],
    "tsb_backward_det_scratch_size": [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)],
    "tsb_loss_scratch_size": [C.c_int32, C.c_int32, C.POINTER(C.c_uint64)],
    "tsb_loss_image": [_P, _P, C.c_int32, C.c_int32, C.c_float, _P, _P, _P, C.c_uint64, _P],
    "tsb_loss_regularizers": [_P, _P, C.POINTER(Camera_t), C.c_float, C.c_float, _P, _P, _P],
    "tsb_adam_step": [C.POINTER(AdamGroup_t), C.c_int32, C.c_int32, C.c_double, C.c_double,
                      C.c_double, _P],
    "tsb_orthonormalize_tangents": [C.c_int32, _P, _P, _P],
    "tsb_orthonormalize_tangents_ex": [C.c_int32, _P, _P, _P, _P],
    "tsb_adam_step_ex": [C.POINTER(AdamGroup_t), C.c_int32, C.c_int32, C.c_double, C.c_double,
                         C.c_double, _P, _P],
    "tsb_guard_finite": [_P, C.c_int32, _P, _P],
    "tsb_broadcast_texels": [C.c_int32, C.c_int32, C.c_int32, _P, _P, _P],
    "tsb_prune_scratch_size": [C.c_int32, C.POINTER(C.c_uint64)],
    "tsb_prune_rows": [C.c_int32, _P, C.c_double, C.POINTER(RowBuffer_t), C.c_int32, _P, _P,
                       C.c_uint64, _P],
    "tsb_frame_graph_create": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                               C.c_int32, C.c_int32, _P, C.c_uint64, C.c_int64, _P,
                               C.POINTER(PixelState_t), _P, C.POINTER(Environment_t), _P, _P,
                               _P, _P, C.POINTER(C.c_void_p)],
    "tsb_frame_graph_create_ev": [C.POINTER(Scene_t), C.POINTER(Camera_t), C.POINTER(Atlas_t),
                                  C.c_int32, C.c_int32, _P, C.c_uint64, C.c_int64, _P,
                                  C.POINTER(PixelState_t), _P, C.POINTER(Environment_t), _P, _P,
                                  _P, _P, _P, C.POINTER(C.c_void_p)],
    "tsb_frame_graph_launch": [_P, C.POINTER(Camera_t), _P, _P],
    "tsb_frame_graph_destroy": [_P],
    "tsb_env_scratch_size": [C.c_int32, C.c_int32, C.POINTER(C.c_uint64)],
    "tsb_env_prefilter": [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), _P, C.c_int32, C.c_int32,
                          _P, C.c_uint64, _P],
    "tsb_brdf_lut": [C.c_int32, C.c_int32, _P, _P],
    "tsb_decompose": [_P, _P, _P, _P, C.c_int32, C.c_int32, _P, _P],
}

_lib = None


class TsbError(RuntimeError):
    pass


def lib():
    """Load libtsb.so once; raise loudly if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise TsbError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(make -C paper_2506_13348_b200/csrc). There is no CPU fallback.")
    h = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, args in _SIGNATURES.items():
        fn = getattr(h, name, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = C.c_int
    h.tsb_last_error.restype = C.c_char_p
    h.tsb_version.restype = C.c_char_p
    _lib = h
    return h


def exported_symbols():
    """Names of every entry point declared in include/tsb.h."""
    import re
    hdr = (_HERE.parent / "include" / "tsb.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void|const char\s*\*)\s+(tsb_[a-z0-9_]+)\s*\(",
                                  hdr, re.M)))


def check(rc: int, what: str):
    """Map a libtsb return code to the reference's exception types."""
    if rc == TSB_OK:
        return
    msg = lib().tsb_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == TSB_ERR_VALUE:
        raise ValueError(text)
    if rc == TSB_ERR_LOOKUP:
        raise LookupError(text)
    if rc == TSB_ERR_CAPACITY:
        raise MemoryError(text)
    raise TsbError(text)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def camera_struct(cam) -> Camera_t:
    c = Camera_t()
    w2v = [float(v) for v in __import__("numpy").asarray(cam.world_to_view, dtype="f8").ravel()]
    c.world_to_view[:] = w2v
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near_z, c.far_z = float(cam.near), float(cam.far)
    c.width, c.height = int(cam.width), int(cam.height)
    return c
