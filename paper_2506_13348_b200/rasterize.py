"""Forward render path behind the reference's rasterize API.

Mirrors /root/reference/pkg/src/texsplat/rasterize.py:
    prepare(scene, camera, texture_mode, atlas_set)          (:172-243)
    render_forward(scene, camera, texture_mode, atlas_set,
                   threads, tile, with_tape, prep)           (:395-438)
    GBuffer (:62-95), NUM_CHANNELS and the channel map (:52-59)
Every frame runs in libtsb (tsb_render_forward: K1-K5 on sm_100a); there is
no CPU path. Differences from the reference, by design:
  * G-buffers are float32 torch tensors on the GPU, stored planar
    (13, H, W); GBuffer.data is the (H, W, 13) view the reference exposes.
  * `threads` is accepted and ignored (the GPU is the thread pool); `tile`
    (8/16/32) selects the CTA tile and, as in the reference, never changes
    the result.
  * The tape is an opaque Tape (workspace + per-pixel state) consumed by
    splat_backward, not a list of per-tile Python records.
  * texture_mode="perprim" packs the charts into an atlas internally and
    samples it with the fp32 software-bilinear verify sampler (bit-identical
    to per-primitive sampling, as atlas.py:184-211 guarantees);
    texture_mode="atlas" samples with the texture units (sampler="hw",
    bilinear, 8-bit fractional weights) unless sampler="verify".
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, resident
from .device import DeviceAtlas, DeviceScene, FrameWorkspace
from .scene import scene_texels

TILE = 16
NUM_CHANNELS = 13
CH_ALBEDO = slice(0, 3)
CH_METALLIC = 3
CH_ROUGHNESS = 4
CH_NORMAL = slice(5, 8)
CH_INDIRECT = slice(8, 11)
CH_DEPTH = 11
CH_ALPHA = 12

_MODES = {"hw": _lib.MODE_HW, "verify": _lib.MODE_VERIFY, "flat": _lib.MODE_FLAT}


@dataclass
class PixelState:
    n_contrib: torch.Tensor   # (H, W) int32
    last_entry: torch.Tensor  # (H, W) int32
    final_T: torch.Tensor     # (H, W) float32
    T_last: torch.Tensor      # (H, W) float32

    @staticmethod
    def empty(H, W, device):
        return PixelState(torch.empty((H, W), dtype=torch.int32, device=device),
                          torch.empty((H, W), dtype=torch.int32, device=device),
                          torch.empty((H, W), dtype=torch.float32, device=device),
                          torch.empty((H, W), dtype=torch.float32, device=device))

    def struct(self, touched: torch.Tensor = None) -> _lib.PixelState_t:
        s = _lib.PixelState_t()
        s.n_contrib = _lib.ptr(self.n_contrib)
        s.last_entry = _lib.ptr(self.last_entry)
        s.final_T = _lib.ptr(self.final_T)
        s.T_last = _lib.ptr(self.T_last)
        s.splat_touched = _lib.ptr(touched)
        return s


class GBuffer:
    """Blended attribute buffers; all channels coverage-premultiplied."""

    def __init__(self, planar, pixels: PixelState = None):
        """`planar`: a (13, H, W) float32 device tensor, or — like the
        reference's GBuffer(data) (rasterize.py:62-67) — an (H, W, 13) array
        (numpy or tensor), uploaded to the current device as planar float32."""
        if not (torch.is_tensor(planar) and planar.is_cuda and planar.dim() == 3
                and planar.shape[0] == NUM_CHANNELS and planar.dtype == torch.float32):
            t = planar if torch.is_tensor(planar) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(planar), dtype=np.float32))
            if t.dim() != 3 or t.shape[-1] != NUM_CHANNELS:
                raise ValueError(f"G-buffer data must be (H, W, {NUM_CHANNELS})")
            planar = t.to(device="cuda", dtype=torch.float32).permute(2, 0, 1).contiguous()
        self.planar = planar          # (13, H, W) float32
        self.pixels = pixels

    @property
    def data(self) -> torch.Tensor:
        return self.planar.permute(1, 2, 0)

    @property
    def fragment_count(self) -> int:
        if self.pixels is None:
            return 0
        return int(self.pixels.n_contrib.sum(dtype=torch.int64).item())

    @property
    def albedo(self):
        return self.data[..., CH_ALBEDO]

    @property
    def metallic(self):
        return self.data[..., CH_METALLIC]

    @property
    def roughness(self):
        return self.data[..., CH_ROUGHNESS]

    @property
    def normal(self):
        return self.data[..., CH_NORMAL]

    @property
    def indirect(self):
        return self.data[..., CH_INDIRECT]

    @property
    def depth(self):
        return self.data[..., CH_DEPTH]

    @property
    def alpha(self):
        return self.data[..., CH_ALPHA]

    def numpy(self) -> np.ndarray:
        """(H, W, 13) float64 host copy, the reference's GBuffer.data layout."""
        return self.data.double().cpu().numpy()


@dataclass
class PreparedScene:
    """Device-side inputs of one (scene, camera, texture mode) — the analogue
    of the reference's PreparedScene (rasterize.py:106-124); the per-splat
    quantities themselves are computed on the GPU inside every frame."""

    scene: DeviceScene
    atlas: DeviceAtlas
    texture_mode: str
    sampler: str
    host_scene: object = None
    workspace: FrameWorkspace = None


@dataclass
class Tape:
    """Forward state that splat_backward replays (workspace + pixel state)."""

    prep: PreparedScene
    camera: object
    tile: int
    capacity: int
    workspace: torch.Tensor
    workspace_bytes: int
    pixels: PixelState
    gbuf: torch.Tensor
    mode: int = 0
    extra: dict = field(default_factory=dict)
    generation: int = 0  # the workspace's frame counter when this tape was taken

    def check_current(self):
        """The tape's tile lists and records live in the shared frame
        workspace; a later frame rendered into it invalidates them."""
        ws = self.prep.workspace
        if ws is None or ws.generation != self.generation or ws.buf is not self.workspace:
            raise RuntimeError("stale tape: another frame was rendered into this prepared "
                               "scene's workspace after it (render again with_tape=True, or "
                               "use a separate prepare() per pending backward)")


def _resolve_sampler(texture_mode, sampler):
    if texture_mode == "flat":
        return "flat"
    if sampler is None:
        return "hw" if texture_mode == "atlas" else "verify"
    if sampler not in ("hw", "verify"):
        raise ValueError(f"unknown sampler {sampler!r}")
    return sampler


def prepare(scene, camera=None, texture_mode: str = "perprim", atlas_set=None, *,
            sampler: str = None, texel_format: str = "rgba32f", device=None) -> PreparedScene:
    """Upload the scene and its texture source for `texture_mode`.

    Raises ValueError like rasterize.py:175-176 (unknown mode), :220-221
    (atlas mode without atlas_set) and :223-224 (resolution mismatch).
    """
    if texture_mode not in ("flat", "perprim", "atlas"):
        raise ValueError(f"unknown texture mode {texture_mode!r}")
    smp = _resolve_sampler(texture_mode, sampler)
    dkey = (str(device),)
    # device copies are cached per host object (resident.py): repeated calls
    # with the same scene / atlas objects upload nothing
    if isinstance(scene, DeviceScene):
        dscene = scene
    else:
        geo = resident.scene_arrays(scene)[:6]
        dscene = resident.cached("scene", scene, dkey, geo, lambda: DeviceScene(scene, device))
    T = dscene.texture_resolution
    if texture_mode == "flat":
        datlas = resident.cached("flat", scene, dkey, resident.scene_arrays(scene)[6:],
                                 lambda: DeviceAtlas.flat_only(scene_texels(scene), device))
    elif texture_mode == "perprim":
        datlas = resident.cached(
            "perprim", scene, dkey + (smp, texel_format), resident.scene_arrays(scene)[6:],
            lambda: DeviceAtlas(texels=scene_texels(scene), linear=(smp == "verify"),
                                hw=(smp == "hw"), texel_format=texel_format, device=device))
    else:
        if atlas_set is None:
            raise ValueError("atlas mode needs a packed atlas_set")
        if isinstance(atlas_set, DeviceAtlas):
            datlas = atlas_set
        else:
            if atlas_set.resolution != T:
                raise ValueError("atlas resolution mismatch with scene")
            datlas = resident.cached(
                "atlas", atlas_set, dkey + (smp, texel_format), resident.atlas_arrays(atlas_set),
                lambda: DeviceAtlas(atlas_set, linear=(smp == "verify"), hw=(smp == "hw"),
                                    texel_format=texel_format, device=device))
        if datlas.resolution != T:
            raise ValueError("atlas resolution mismatch with scene")
    if texture_mode != "flat" and datlas.num_entries < dscene.num_splats:
        raise LookupError("atlas has fewer indirection entries than splats")
    return PreparedScene(dscene, datlas, texture_mode, smp, host_scene=scene,
                         workspace=FrameWorkspace(dscene.device))


def render_prepared(prep: PreparedScene, camera, tile: int = TILE, *, out=None,
                    pixels: PixelState = None, check: bool = True, stream=None):
    """One frame K1-K5 into a planar G-buffer. Returns (GBuffer, Tape)."""
    if tile not in (8, 16, 32):
        raise ValueError("tile must be 8, 16 or 32")
    L = _lib.lib()
    dev = prep.scene.device
    W, H = int(camera.width), int(camera.height)
    P = prep.scene.num_splats
    ws = prep.workspace
    if ws.key != (P, W, H, tile):
        ws.ensure(P, W, H, tile, FrameWorkspace.initial_capacity(P, W, H, tile))
    ws.generation += 1
    gbuf = out if out is not None else torch.empty((NUM_CHANNELS, H, W), dtype=torch.float32,
                                                   device=dev)
    px = pixels if pixels is not None else PixelState.empty(H, W, dev)
    cam = _lib.camera_struct(camera)
    sc = prep.scene.struct()
    at = prep.atlas.struct()
    mode = _MODES[prep.sampler]
    st = _lib.stream_handle(stream)
    for _ in range(3):
        pst = px.struct()
        _lib.check(L.tsb_render_forward(C.byref(sc), C.byref(cam), C.byref(at), mode, tile,
                                        _lib.ptr(ws.buf), ws.nbytes, ws.capacity,
                                        _lib.ptr(gbuf), C.byref(pst), _lib.ptr(ws.needed), st),
                   "tsb_render_forward")
        if not check:
            break
        needed = int(ws.needed.item())
        if needed <= ws.capacity:
            break
        ws.ensure(P, W, H, tile, int(needed * 1.25) + 1024)
        ws.generation += 1
    tape = Tape(prep, camera, tile, ws.capacity, ws.buf, ws.nbytes, px, gbuf, mode,
                generation=ws.generation)
    return GBuffer(gbuf, px), tape


def render_forward(scene, camera, texture_mode: str = "perprim", atlas_set=None,
                   threads: int = 1, tile: int = TILE, with_tape: bool = False,
                   prep: PreparedScene = None, *, sampler: str = None,
                   texel_format: str = "rgba32f"):
    """Rasterize the scene into a G-buffer (rasterize.py:395-438).

    Returns GBuffer, or (GBuffer, Tape) when with_tape.
    """
    del threads  # the reference's tile thread pool; the GPU replaces it
    if prep is None:
        prep = prepare(scene, camera, texture_mode, atlas_set, sampler=sampler,
                       texel_format=texel_format)
        if not with_tape:
            # no tape outlives the call: the scene's cached workspace serves
            # every such frame on the calling stream (a tape gets its own, as
            # the reference's tapes are independent objects). One workspace
            # per stream, so concurrent renders on different streams never
            # share one (concurrent cameras over one scene).
            pool = getattr(prep.scene, "_shared_workspaces", None)
            if pool is None:
                pool = prep.scene._shared_workspaces = {}
            key = _lib.stream_handle(None) or 0
            shared = pool.get(key)
            if shared is None:
                shared = pool[key] = prep.workspace
            prep.workspace = shared
    gbuf, tape = render_prepared(prep, camera, tile)
    return (gbuf, tape) if with_tape else gbuf


def frame_structure(tape: Tape):
    """Sorted ids, (tile << 32 | rank) keys, tile ranges and rects of a frame
    (parity checks against the oracle)."""
    L = _lib.lib()
    P = tape.prep.scene.num_splats
    W, H = int(tape.camera.width), int(tape.camera.height)
    dev = tape.gbuf.device
    tiles = ((W + tape.tile - 1) // tape.tile) * ((H + tape.tile - 1) // tape.tile)
    sorted_ids = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    keys = torch.empty(max(tape.capacity, 1), dtype=torch.int64, device=dev)
    ranges = torch.empty((tiles, 2), dtype=torch.int32, device=dev)
    rects = torch.empty((max(P, 1), 4), dtype=torch.int32, device=dev)
    _lib.check(L.tsb_frame_export(P, W, H, tape.tile, tape.capacity, _lib.ptr(tape.workspace),
                                  _lib.ptr(sorted_ids), _lib.ptr(keys), _lib.ptr(ranges),
                                  _lib.ptr(rects), _lib.stream_handle()), "tsb_frame_export")
    keys = keys.cpu().numpy()
    return {"sorted_ids": sorted_ids.cpu().numpy()[:P], "keys": keys[keys >= 0],
            "ranges": ranges.cpu().numpy(), "rects": rects.cpu().numpy()[:P]}


def render_normal_map(scene, camera, **kw):
    gbuf = render_forward(scene, camera, **kw)
    n = gbuf.normal
    norm = torch.linalg.norm(n, dim=-1, keepdim=True)
    covered = gbuf.alpha[..., None] > 1e-8
    unit = torch.where(covered & (norm > 1e-12), n / norm.clamp_min(1e-30),
                       torch.zeros_like(n))
    return 0.5 * (unit + 1.0)


def render_depth_map(scene, camera, **kw):
    gbuf = render_forward(scene, camera, **kw)
    a = gbuf.alpha
    return torch.where(a > 1e-8, gbuf.depth / a.clamp_min(1e-30), torch.zeros_like(a))
