"""Training backward behind the reference's API.

Mirrors /root/reference/pkg/src/texsplat:
    splat_backward(scene, camera, prep, tape, dbuf) -> SceneGrads   (rasterize.py:472-593)
    shade_backward(result, camera, env, lut, dcolor) -> (dgbuf, EnvGrads)  (shading.py:186-228)
    SceneGrads (rasterize.py:441-469), EnvGrads (environment.py:198-206)
The adjoints run in libtsb (K7 k_shade_bwd, K8 k_raster_bwd, K9
k_finish_grads). Gradients are float64 for the float64 scene parameters
and float32 for texels/environment grids, on the GPU. Float atomics make
the low bits order-dependent (the reference is bitwise deterministic);
parity is held to the tolerance stated in DESIGN.md.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .environment import EnvGrads
from .rasterize import NUM_CHANNELS, Tape
from .shading import ShadeResult, device_environment


@dataclass
class SceneGrads:
    """Gradients on every learnable splat parameter (GPU tensors)."""

    positions: torch.Tensor   # (P, 3) float64
    tangent_u: torch.Tensor   # (P, 3) float64
    tangent_v: torch.Tensor   # (P, 3) float64
    scales: torch.Tensor      # (P, 2) float64
    opacities: torch.Tensor   # (P,) float64
    sh: torch.Tensor          # (P, K, 3) float64
    texels_dense: torch.Tensor  # (P, T, T, 7) float32, combined order (or (P, T, T, 8)
    #                             interleaved atlas order when texel_layout == 1)
    texel_layout: int = 0

    @staticmethod
    def zeros(P, K, T, device):
        f64 = dict(dtype=torch.float64, device=device)
        return SceneGrads(torch.zeros((P, 3), **f64), torch.zeros((P, 3), **f64),
                          torch.zeros((P, 3), **f64), torch.zeros((P, 2), **f64),
                          torch.zeros((P,), **f64), torch.zeros((P, K, 3), **f64),
                          torch.zeros((P, T, T, 7), dtype=torch.float32, device=device))

    @property
    def texels(self):
        """Reference-style list: (T, T, 7) per splat, None if untouched."""
        t = self.texels_dense
        if self.texel_layout == _lib.TEXELS_INTERLEAVED:
            t = t[..., [0, 1, 2, 3, 6, 4, 5]]
        t = t.cpu().numpy().astype(np.float64)
        touched = np.any(t != 0, axis=(1, 2, 3))
        return [t[k] if touched[k] else None for k in range(t.shape[0])]

    def struct(self) -> _lib.SceneGrads_t:
        s = _lib.SceneGrads_t()
        s.positions = _lib.ptr(self.positions)
        s.tangent_u = _lib.ptr(self.tangent_u)
        s.tangent_v = _lib.ptr(self.tangent_v)
        s.scales = _lib.ptr(self.scales)
        s.opacities = _lib.ptr(self.opacities)
        s.sh = _lib.ptr(self.sh)
        s.texels = _lib.ptr(self.texels_dense)
        s.texel_layout = self.texel_layout
        return s

    def flat(self) -> list:
        return [self.positions, self.tangent_u, self.tangent_v, self.scales, self.opacities,
                self.sh, self.texels_dense]


def _planar(dbuf, H, W, device) -> torch.Tensor:
    """(13, H, W) float32 device tensor from an (H, W, 13) array/tensor or a
    planar tensor."""
    t = dbuf if torch.is_tensor(dbuf) else torch.from_numpy(np.asarray(dbuf))
    if tuple(t.shape) == (H, W, NUM_CHANNELS):
        t = t.permute(2, 0, 1)
    if tuple(t.shape) != (NUM_CHANNELS, H, W):
        raise ValueError("dbuf must be (H, W, 13) or (13, H, W)")
    return t.to(device=device, dtype=torch.float32).contiguous()


def splat_backward(scene, camera, prep, tape: Tape, dbuf, *, grads: SceneGrads = None,
                   scratch: torch.Tensor = None, deterministic: bool = False) -> SceneGrads:
    """Backpropagate a G-buffer gradient to splat parameters.

    `tape` is the second return of render_forward(..., with_tape=True) in
    texture_mode "perprim" (fp32 software sampling), as in the reference
    (rasterize.py:482-483 raises ValueError otherwise). `scene` and `prep`
    are accepted for signature parity; the frame state lives in the tape.
    deterministic=True: bitwise-repeatable gradients (int64 fixed-point
    accumulation, tsb_render_backward_ex) like the reference's fixed-order
    reduction (rasterize.py:494, :646); the default float atomics are faster.
    """
    del scene
    if tape.mode != _lib.MODE_VERIFY or tape.prep.texture_mode == "flat":
        raise ValueError("gradients require the per-primitive texture path")
    tape.check_current()
    prep = prep if prep is not None else tape.prep
    dev = tape.gbuf.device
    H, W = int(camera.height), int(camera.width)
    dplanar = _planar(dbuf, H, W, dev)
    ds = prep.scene
    P = ds.num_splats
    K = (ds.sh_degree + 1) ** 2
    T = ds.texture_resolution
    if grads is None:
        grads = SceneGrads.zeros(P, K, T, dev)
    L = _lib.lib()
    if scratch is None:
        nb = C.c_uint64()
        _lib.check(L.tsb_backward_scratch_size(P, C.byref(nb)), "tsb_backward_scratch_size")
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
    sc, at, cam = ds.struct(), prep.atlas.struct(), _lib.camera_struct(camera)
    pst = tape.pixels.struct()
    gs = grads.struct()
    det = None
    if deterministic:
        nb = C.c_uint64()
        _lib.check(L.tsb_backward_det_scratch_size(P, T, grads.texel_layout, C.byref(nb)),
                   "tsb_backward_det_scratch_size")
        det = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
    _lib.check(L.tsb_render_backward_ex(C.byref(sc), C.byref(cam), C.byref(at), tape.tile,
                                        _lib.ptr(tape.workspace), tape.workspace_bytes,
                                        tape.capacity, C.byref(pst), _lib.ptr(dplanar),
                                        _lib.ptr(scratch), C.byref(gs), 1 if deterministic else 0,
                                        _lib.ptr(det), 0 if det is None else det.numel(),
                                        _lib.stream_handle()),
               "tsb_render_backward")
    return grads


@dataclass
class DeviceEnvGrads:
    spec_mips: list
    diffuse: torch.Tensor

    def struct(self) -> _lib.EnvGrads_t:
        e = _lib.EnvGrads_t()
        for i, m in enumerate(self.spec_mips):
            e.spec_mips[i] = _lib.ptr(m)
        e.diffuse = _lib.ptr(self.diffuse)
        return e

    def numpy(self) -> EnvGrads:
        return EnvGrads([m.double().cpu().numpy() for m in self.spec_mips],
                        self.diffuse.double().cpu().numpy())


def shade_backward(result: ShadeResult, camera, env, lut, dcolor, *, env_grads=None,
                   dgbuf=None):
    """Backpropagate a gradient on ShadeResult.color (shading.py:186-228).

    Returns (dgbuf planar (13, H, W) float32, DeviceEnvGrads). `env_grads`
    (a DeviceEnvGrads) and `dgbuf` may be preallocated; env gradients are
    accumulated into them."""
    planar, denv_cached, bg = result.cache
    denv = denv_cached if env is None else device_environment(env, lut, planar.device)
    H, W = int(camera.height), int(camera.width)
    dev = planar.device
    dc = dcolor if torch.is_tensor(dcolor) else torch.from_numpy(np.asarray(dcolor))
    dc = dc.to(device=dev, dtype=torch.float32).contiguous()
    if tuple(dc.shape) != (H, W, 3):
        raise ValueError("dcolor must be (H, W, 3)")
    if dgbuf is None:
        dgbuf = torch.empty((NUM_CHANNELS, H, W), dtype=torch.float32, device=dev)
    eg = env_grads if env_grads is not None else DeviceEnvGrads(
        [torch.zeros_like(m) for m in denv.mips], torch.zeros_like(denv.diffuse))
    bgc = (C.c_float * 3)(*[float(v) for v in np.asarray(bg, np.float64)])
    cam = _lib.camera_struct(camera)
    es = denv.struct()
    egs = eg.struct()
    L = _lib.lib()
    nb = C.c_uint64()
    _lib.check(L.tsb_shade_backward_scratch_size(C.byref(es), C.byref(nb)),
               "tsb_shade_backward_scratch_size")
    scratch = getattr(denv, "_bwd_scratch", None)
    if scratch is None or scratch.numel() < nb.value:
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
        denv._bwd_scratch = scratch
    _lib.check(L.tsb_shade_backward(_lib.ptr(planar), C.byref(cam), C.byref(es), bgc,
                                    _lib.ptr(dc), _lib.ptr(dgbuf), C.byref(egs),
                                    _lib.ptr(scratch), int(scratch.numel()),
                                    _lib.stream_handle()), "tsb_shade_backward")
    return dgbuf, eg
