"""Deferred split-sum shading behind the reference's shading API.

Mirrors /root/reference/pkg/src/texsplat/shading.py:
    shade_gbuffer(gbuf, camera, env, lut, mesh=None, background=None)  (:126-183)
    ShadeResult (:41-48)
The per-pixel work is k_shade in libtsb (tsb_shade_forward). Mesh
visibility (visibility.py) is out of scope (no BASELINE
config has a mesh), so mesh must be None.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, resident
from .device import DeviceEnvironment

COS_MIN = 1e-4
COVER_EPS = 1e-8


@dataclass
class ShadeResult:
    """Linear radiance (H, W, 3) float32 on the GPU; diffuse/specular are
    coverage-weighted (alpha * L_d, alpha * L_s)."""

    color: torch.Tensor
    diffuse: torch.Tensor
    specular: torch.Tensor
    cache: tuple = None


def device_environment(env, lut, device=None) -> DeviceEnvironment:
    """The environment + LUT in HBM, cached per (env, lut) host objects."""
    if isinstance(env, DeviceEnvironment):
        return env
    if env is None:
        raise ValueError("shading needs an environment")
    return resident.cached("env", env, (id(lut), str(device)), resident.env_arrays(env, lut),
                           lambda: DeviceEnvironment(env, lut, device))


def shade_planar(planar: torch.Tensor, camera, denv: DeviceEnvironment, background=None, *,
                 color=None, diffuse=None, specular=None, want_split=True, stream=None):
    H, W = int(camera.height), int(camera.width)
    if tuple(planar.shape) != (13, H, W):
        raise ValueError("G-buffer shape does not match the camera")
    dev = planar.device
    color = color if color is not None else torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    if want_split:
        diffuse = diffuse if diffuse is not None else torch.empty_like(color)
        specular = specular if specular is not None else torch.empty_like(color)
    bg = (C.c_float * 3)(*([0.0] * 3 if background is None else
                           [float(v) for v in np.asarray(background, np.float64)]))
    cam = _lib.camera_struct(camera)
    env = denv.struct()
    _lib.check(_lib.lib().tsb_shade_forward(_lib.ptr(planar), C.byref(cam), C.byref(env), bg,
                                            _lib.ptr(color), _lib.ptr(diffuse),
                                            _lib.ptr(specular), _lib.stream_handle(stream)),
               "tsb_shade_forward")
    return color, diffuse, specular


def shade_gbuffer(gbuf, camera, env, lut, mesh=None, background=None) -> ShadeResult:
    """Shade a G-buffer into final linear radiance (shading.py:126-183)."""
    if mesh is not None:
        raise NotImplementedError("mesh visibility is outside the B200 render path")
    planar = gbuf.planar if hasattr(gbuf, "planar") else _to_planar(gbuf)
    denv = device_environment(env, lut, planar.device)
    color, diffuse, specular = shade_planar(planar, camera, denv, background)
    bg = np.zeros(3) if background is None else np.asarray(background, np.float64)
    return ShadeResult(color, diffuse, specular, cache=(planar, denv, bg))


def _to_planar(gbuf) -> torch.Tensor:
    data = gbuf.data if hasattr(gbuf, "data") else gbuf
    t = torch.as_tensor(np.asarray(data, dtype=np.float32)) if not torch.is_tensor(data) else data
    if not t.is_cuda:
        t = t.cuda()
    return t.float().permute(2, 0, 1).contiguous()
