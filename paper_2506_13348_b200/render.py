"""render(camera, gaussians, atlas, envmap): the composed hot path.

The reference composes it in cmd_render's per-view body (cli.py:63-68):
render_forward(scene, cam, "atlas", atlas_set) then shade_gbuffer(...).
Renderer keeps the scene, atlas and environment resident in HBM and renders
views with two library calls (tsb_render_forward + tsb_shade_forward) and no
host synchronisation, so a view batch (cfg3) streams back to back.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
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
        self._graphs = {}           # (W, H) -> (key, handle)
        self.use_graph = True

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
                  entries, exact=True)
        ws.shrink_to = None

    def entries_needed(self) -> int:
        return int(self.prep.workspace.needed.item())

    def _graph(self, camera, W, H, binned_event=None):
        """CUDA graph of this view size over the current buffers (rebuilt if
        the workspace was reallocated). `binned_event`: a torch.cuda.Event the
        graph records between binning and rasterisation on every replay."""
        ws = self.prep.workspace
        gb, px, col, _, _ = self._buffers(W, H)
        ev = None if binned_event is None else binned_event.cuda_event
        key = (_lib.ptr(ws.buf), ws.capacity, ws.nbytes, ev)
        cur = self._graphs.get((W, H, ev))
        if cur is not None and cur[0] == key:
            return cur[1], col
        if cur is not None:
            _lib.lib().tsb_frame_graph_destroy(cur[1])
            del self._graphs[(W, H, ev)]
        L = _lib.lib()
        sc, at, cam = self.prep.scene.struct(), self.prep.atlas.struct(), _lib.camera_struct(camera)
        pst = px.struct()
        env = self.env.struct()
        bg = (C.c_float * 3)(*([0.0] * 3 if self.background is None else
                               [float(v) for v in np.asarray(self.background, np.float64)]))
        from .rasterize import _MODES
        h = C.c_void_p()
        _lib.check(L.tsb_frame_graph_create_ev(
            C.byref(sc), C.byref(cam), C.byref(at), _MODES[self.prep.sampler], self.tile,
            _lib.ptr(ws.buf), ws.nbytes, ws.capacity, _lib.ptr(gb), C.byref(pst),
            _lib.ptr(ws.needed), C.byref(env), bg, _lib.ptr(col), None, None,
            C.c_void_p(ev) if ev else None, C.byref(h)), "tsb_frame_graph_create_ev")
        self._graphs[(W, H, ev)] = (key, h)
        return h, col

    def close(self):
        for _, h in self._graphs.values():
            _lib.lib().tsb_frame_graph_destroy(h)
        self._graphs = {}

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass

    def _graph_ready(self, W, H) -> bool:
        ws = self.prep.workspace
        return (self.use_graph and ws.buf is not None
                and ws.key == (self.prep.scene.num_splats, W, H, self.tile))

    def render(self, camera, *, check: bool = True, want_split: bool = False, stream=None,
               color=None, binned_event=None):
        """Forward + shade one view. Returns (color (H,W,3), GBuffer), both on
        the GPU; buffers are reused across calls of the same size (pass
        `color` to shade into a caller-owned buffer instead). With
        check=False (workspace already reserved) the view replays a CUDA
        graph of the whole frame (tsb_frame_graph_*), which records
        `binned_event` (if given) once the frame's tile lists are built."""
        W, H = int(camera.width), int(camera.height)
        if not check and not want_split and self._graph_ready(W, H):
            h, col = self._graph(camera, W, H, binned_event)
            out = color if color is not None else col
            cam = _lib.camera_struct(camera)
            _lib.check(_lib.lib().tsb_frame_graph_launch(h, C.byref(cam), _lib.ptr(out),
                                                         _lib.stream_handle(stream)),
                       "tsb_frame_graph_launch")
            gb, px = self._buffers(W, H)[:2]
            return out, GBuffer(gb, px)
        gb, px, col, dif, spe = self._buffers(W, H)
        if color is not None:
            col = color
        gbuf, _ = render_prepared(self.prep, camera, self.tile, out=gb, pixels=px, check=check,
                                  stream=stream)
        shade_planar(gb, camera, self.env, self.background, color=col,
                     diffuse=dif if want_split else None, specular=spe if want_split else None,
                     want_split=want_split, stream=stream)
        return col, gbuf

    def stream_views(self, cameras, host_out=None, depth: int = 2):
        """Render a sequence of views and read each colour image back to
        pinned host memory (`depth` rotating output buffers, a dedicated copy
        stream). Frame i's device->host copy starts once frame i+1's tile
        lists are built (an event recorded inside the frame graph), so it
        overlaps frame i+1's rasteriser rather than its latency-bound
        binning. Yields (index, host colour tensor) in order as each copy
        completes; a host buffer is reused `depth` frames later."""
        cams = list(cameras)
        if not cams:
            return
        W, H = int(cams[0].width), int(cams[0].height)
        dev = self.device
        depth = max(2, int(depth))
        key = ("stream", W, H, depth)
        if key not in self._bufs:  # pinned buffers, copy stream, events: allocated once
            binned = torch.cuda.Event()
            binned.record()  # materialise the CUDA event before it is captured
            self._bufs[key] = (
                [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(depth)],
                [torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True)
                 for _ in range(depth)],
                torch.cuda.Stream(dev), binned)
        dcol, hcol_cached, copy, binned = self._bufs[key]
        hcol = host_out or hcol_cached
        compute = torch.cuda.current_stream(dev)
        done = [torch.cuda.Event() for _ in range(depth)]
        ready = torch.cuda.Event()
        use_ev = self._graph_ready(W, H)

        def queue_copy(j, after):
            b = j % depth
            copy.wait_event(after)
            with torch.cuda.stream(copy):
                hcol[b].copy_(dcol[b], non_blocking=True)
            done[b].record(copy)

        for i, cam in enumerate(cams):
            b = i % depth
            if i >= depth:
                compute.wait_event(done[b])     # device buffer b copied out
            self.render(cam, check=False, stream=compute, color=dcol[b],
                        binned_event=binned if use_ev else None)
            if i >= 1:
                if use_ev:
                    queue_copy(i - 1, binned)   # frame i-1 done, frame i binned
                else:
                    ready.record(compute)       # no graph: after frame i
                    queue_copy(i - 1, ready)
            if i >= 2:
                done[(i - 2) % depth].synchronize()
                yield i - 2, hcol[(i - 2) % depth]
        n = len(cams)
        ready.record(compute)
        queue_copy(n - 1, ready)
        for j in range(max(0, n - 2), n):
            done[j % depth].synchronize()
            yield j, hcol[j % depth]

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
