"""render(camera, gaussians, atlas, envmap): the composed hot path.

The reference composes it in cmd_render's per-view body (cli.py:63-68):
render_forward(scene, cam, "atlas", atlas_set) then shade_gbuffer(...).
Renderer keeps the scene, atlas and environment resident in HBM and renders
views with two library calls (tsb_render_forward + tsb_shade_forward) and no
host synchronisation, so a view batch (cfg3) streams back to back.
"""

from __future__ import annotations

import torch

from .device import DeviceAtlas, DeviceEnvironment, DeviceScene, FrameWorkspace
from .rasterize import NUM_CHANNELS, TILE, GBuffer, PixelState, PreparedScene, prepare, render_prepared
from .shading import ShadeResult, shade_planar


class Renderer:
    """Device-resident scene + atlas + environment for repeated views."""

    def __init__(self, scene, atlas_set=None, environment=None, lut=None, *,
                 texture_mode: str = "atlas", sampler: str = None, texel_format: str = "rgba32f",
                 tile: int = TILE, device=None, background=None):
        if texture_mode == "atlas" and atlas_set is None:
            from .atlas import pack_atlases
            atlas_set = pack_atlases(scene)
        self.prep: PreparedScene = prepare(scene, None, texture_mode, atlas_set, sampler=sampler,
                                           texel_format=texel_format, device=device)
        env = environment if environment is not None else getattr(scene, "environment", None)
        if env is None:
            raise ValueError("Renderer needs an environment")
        if lut is None and not isinstance(env, DeviceEnvironment):
            from .environment import BrdfLut
            lut = BrdfLut.build()
        self.env = env if isinstance(env, DeviceEnvironment) else DeviceEnvironment(
            env, lut, self.prep.scene.device)
        self.tile = tile
        self.background = background if background is not None else getattr(
            scene, "background", None)
        self._bufs = {}

    @property
    def device(self):
        return self.prep.scene.device

    def _buffers(self, W, H):
        key = (W, H)
        if key not in self._bufs:
            dev = self.device
            self._bufs[key] = (
                torch.empty((NUM_CHANNELS, H, W), dtype=torch.float32, device=dev),
                PixelState.empty(H, W, dev),
                torch.empty((H, W, 3), dtype=torch.float32, device=dev),
                torch.empty((H, W, 3), dtype=torch.float32, device=dev),
                torch.empty((H, W, 3), dtype=torch.float32, device=dev),
            )
        return self._bufs[key]

    def reserve(self, camera, entries: int):
        """Pre-size the frame workspace (no per-frame capacity sync needed)."""
        ws = self.prep.workspace
        ws.ensure(self.prep.scene.num_splats, int(camera.width), int(camera.height), self.tile,
                  entries)

    def entries_needed(self) -> int:
        return int(self.prep.workspace.needed.item())

    def render(self, camera, *, check: bool = True, want_split: bool = False, stream=None):
        """Forward + shade one view. Returns (color (H,W,3), GBuffer), both on
        the GPU; buffers are reused across calls of the same size."""
        W, H = int(camera.width), int(camera.height)
        gb, px, col, dif, spe = self._buffers(W, H)
        gbuf, _ = render_prepared(self.prep, camera, self.tile, out=gb, pixels=px, check=check,
                                  stream=stream)
        shade_planar(gb, camera, self.env, self.background, color=col,
                     diffuse=dif if want_split else None, specular=spe if want_split else None,
                     want_split=want_split, stream=stream)
        return col, gbuf

    def shade(self, gbuf: GBuffer, camera) -> ShadeResult:
        c, d, s = shade_planar(gbuf.planar, camera, self.env, self.background)
        return ShadeResult(c, d, s)


def render(camera, gaussians, atlas=None, envmap=None, lut=None, background=None,
           mode: str = "hw", tile: int = TILE):
    """One-shot render(camera, gaussians, atlas, envmap) -> (color, GBuffer).

    mode: "hw" (texture units), "verify" (fp32 software bilinear) or "flat".
    For many views build a Renderer once instead.
    """
    texture_mode = "flat" if mode == "flat" else "atlas"
    sampler = None if mode == "flat" else mode
    r = Renderer(gaussians, atlas, envmap, lut, texture_mode=texture_mode, sampler=sampler,
                 tile=tile, background=background)
    return r.render(camera)
