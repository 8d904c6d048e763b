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

from . import _lib, resident
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
            lut = BrdfLut.build(device=self.prep.scene.device)  # K16 on the GPU
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
        """Pre-size the frame workspace (no per-frame capacity sync needed).
        Frames replayed with check=False are validated afterwards with
        check_capacity() (or automatically by stream_views)."""
        ws = self.prep.workspace
        ws.ensure(self.prep.scene.num_splats, int(camera.width), int(camera.height), self.tile,
                  entries, exact=True)

    def entries_needed(self) -> int:
        """Entry count of the last binned frame."""
        return int(self.prep.workspace.needed.item())

    def max_entries_needed(self) -> int:
        """Largest entry count of any frame since the last reset (host sync)."""
        return self.prep.workspace.max_needed_value()

    def check_capacity(self, reset: bool = True):
        """Raise if any frame rendered since the last check outgrew the
        workspace (such a frame has empty tile lists: background only). The
        running maximum lives on the device (k_ranges), so graph replays need
        no per-frame host sync."""
        ws = self.prep.workspace
        need = ws.max_needed_value()
        if reset:
            ws.reset_max()
        if need > ws.capacity:
            raise RuntimeError(f"frame workspace overflow: a frame needed {need} tile entries, "
                               f"capacity {ws.capacity}; reserve() more and re-render")

    def _slot(self, W, H, slot):
        """(workspace, buffers) of frame slot `slot`: slot 0 is the prepared
        scene's own workspace; further slots (pipelined views, see
        stream_views) get their own workspace of the same capacity."""
        if slot == 0:
            return self.prep.workspace, self._buffers(W, H)
        key = ("slot", W, H, slot)
        ws0 = self.prep.workspace
        if key not in self._bufs:
            self._bufs[key] = (FrameWorkspace(self.device), None)
        ws = self._bufs[key][0]
        if ws0.key is not None and (ws.key != ws0.key or ws.capacity != ws0.capacity):
            ws.ensure(*ws0.key, ws0.capacity, exact=True)
        bkey = ("slotbuf", W, H, slot)
        if bkey not in self._bufs:
            dev = self.device
            self._bufs[bkey] = (
                torch.empty((NUM_CHANNELS, H, W), dtype=torch.float32, device=dev),
                PixelState.empty(H, W, dev),
                torch.empty((H, W, 3), dtype=torch.float32, device=dev), None, None)
        return ws, self._bufs[bkey]

    def _graph(self, camera, W, H, binned_event=None, slot: int = 0):
        """CUDA graph of this view size over the current buffers (rebuilt if
        the workspace was reallocated). `binned_event`: a torch.cuda.Event the
        graph records between binning and rasterisation on every replay.
        `slot`: an independent workspace + buffer set (pipelined views)."""
        ws, bufs = self._slot(W, H, slot)
        gb, px, col = bufs[0], bufs[1], bufs[2]
        ev = None if binned_event is None else binned_event.cuda_event
        key = (_lib.ptr(ws.buf), ws.capacity, ws.nbytes, ev)
        cur = self._graphs.get((W, H, ev, slot))
        if cur is not None and cur[0] == key:
            return cur[1], col
        if cur is not None:
            _lib.lib().tsb_frame_graph_destroy(cur[1])
            del self._graphs[(W, H, ev, slot)]
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
        self._graphs[(W, H, ev, slot)] = (key, h)
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

    def _stream_pipelined(self, cams, host_out, depth, n):
        """stream_views with `n` frames in flight: frame i renders in slot
        i % n (its own workspace and buffers) on that slot's stream, so the
        latency-bound binning of one view overlaps the rasteriser tail of the
        previous; colour goes to a ring of `depth` device buffers (no frame
        waits for an earlier frame's copy unless the ring wraps) and is copied
        out on a copy stream once its frame is done. Yields (i, host image)
        in order, or (i, None) at the first frame whose slot reported a
        tile-entry overflow (the caller grows and resumes)."""
        W, H = int(cams[0].width), int(cams[0].height)
        dev = self.device
        depth = max(n + 2, int(depth))
        key = ("pipe", W, H, n, depth)
        if key not in self._bufs:
            self._bufs[key] = (
                [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(depth)],
                [torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True)
                 for _ in range(depth)],
                [torch.cuda.Stream(dev) for _ in range(n)], torch.cuda.Stream(dev),
                torch.zeros((depth,), dtype=torch.int64, pin_memory=True))
        dcol, hcol_cached, streams, copy, hmax = self._bufs[key]
        hcol = host_out or hcol_cached
        graphs = [self._graph(cams[0], W, H, slot=j)[0] for j in range(n)]
        wss = [self._slot(W, H, j)[0] for j in range(n)]
        cur = torch.cuda.current_stream(dev)
        start = torch.cuda.Event()
        for ws in wss:
            ws.reset_max()
        start.record(cur)
        for st in streams:
            st.wait_event(start)
        cdone = [None] * len(cams)

        def emit(i):
            b = i % depth
            cdone[i].synchronize()
            return i, (hcol[b] if int(hmax[b]) <= wss[i % n].capacity else None)

        lag = depth - 1  # frames in flight beyond the one being consumed
        for i, cam in enumerate(cams):
            j, b = i % n, i % depth
            st = streams[j]
            if i >= depth:  # ring buffer b: the copy of frame i - depth is done
                st.wait_event(cdone[i - depth])
            cs = _lib.camera_struct(cam)
            _lib.check(_lib.lib().tsb_frame_graph_launch(graphs[j], C.byref(cs),
                                                         _lib.ptr(dcol[b]),
                                                         _lib.stream_handle(st)),
                       "tsb_frame_graph_launch")
            fdone = torch.cuda.Event()
            fdone.record(st)
            copy.wait_event(fdone)
            with torch.cuda.stream(copy):
                hcol[b].copy_(dcol[b], non_blocking=True)
                hmax[b:b + 1].copy_(wss[j].max_needed, non_blocking=True)
            cdone[i] = torch.cuda.Event()
            cdone[i].record(copy)
            if i >= lag:  # host buffer b is rewritten `depth` frames later
                k, img = emit(i - lag)
                yield k, img
                if img is None:
                    return
        for k in range(max(0, len(cams) - lag), len(cams)):
            kk, img = emit(k)
            yield kk, img
            if img is None:
                return
        for st in streams:
            end = torch.cuda.Event()
            end.record(st)
            cur.wait_event(end)

    def stream_views(self, cameras, host_out=None, depth: int = 2, pipeline: int = 3):
        """Render a sequence of views and read each colour image back to
        pinned host memory (`depth` rotating output buffers, a dedicated copy
        stream). Frame i's device->host copy starts once frame i+1's tile
        lists are built (an event recorded inside the frame graph), so it
        overlaps frame i+1's rasteriser rather than its latency-bound
        binning. Yields (index, host colour tensor) in order as each copy
        completes; a host buffer is reused `depth` frames later. pipeline > 1:
        that many frames in flight in independent workspaces on their own
        streams (_stream_pipelined).

        Capacity: with every image the device's running maximum of the
        frames' entry counts comes back too. A frame is yielded only once it
        is known to have fitted the workspace; on an overflow the workspace
        grows and the stream resumes from the first unverified frame."""
        cams = list(cameras)
        start = 0
        while start < len(cams):
            resume = None
            W, H = int(cams[0].width), int(cams[0].height)
            gen = (self._stream_pipelined(cams[start:], host_out, depth, pipeline)
                   if pipeline > 1 and self._graph_ready(W, H)
                   else self._stream(cams[start:], host_out, depth))
            for i, img in gen:
                if img is None:       # overflow detected: frames >= i unverified
                    resume = start + i
                    break
                yield start + i, img
            if resume is None:
                return
            torch.cuda.synchronize(self.device)
            ws = self.prep.workspace
            need = max([ws.max_needed_value()] + [
                v[0].max_needed_value() for k, v in self._bufs.items()
                if isinstance(k, tuple) and k[0] == "slot"])
            c = cams[resume]
            ws.ensure(self.prep.scene.num_splats, int(c.width), int(c.height), self.tile,
                      int(need * 1.25) + 4096)
            start = resume

    def _stream(self, cams, host_out, depth):
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
                torch.cuda.Stream(dev), binned,
                torch.zeros((depth,), dtype=torch.int64, pin_memory=True))
        dcol, hcol_cached, copy, binned, hmax = self._bufs[key]
        hcol = host_out or hcol_cached
        ws = self.prep.workspace
        compute = torch.cuda.current_stream(dev)
        done = [torch.cuda.Event() for _ in range(depth)]
        ready = torch.cuda.Event()
        use_ev = self._graph_ready(W, H)
        if ws.max_needed is not None:
            ws.reset_max()            # (on the compute stream, before the first frame)
        verified = -1                 # frames <= verified fitted the workspace

        def queue_copy(j, after):
            b = j % depth
            copy.wait_event(after)
            with torch.cuda.stream(copy):
                hcol[b].copy_(dcol[b], non_blocking=True)
                if ws.max_needed is not None:  # running max incl. the frames binned so far
                    hmax[b:b + 1].copy_(ws.max_needed, non_blocking=True)
            done[b].record(copy)

        def emit(j):
            """(j, image) if frame j is known to fit, else (j, None)."""
            nonlocal verified
            b = j % depth
            done[b].synchronize()
            if ws.max_needed is None or int(hmax[b]) <= ws.capacity:
                # this read covers every frame binned before the copy started:
                # frame j + 1 too, except for the last frame
                verified = max(verified, j + 1 if j + 1 < len(cams) else j)
                return j, hcol[b]
            return j, (hcol[b] if j <= verified else None)

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
                j, img = emit(i - 2)
                yield j, img
                if img is None:
                    return
                if j + 1 > verified:            # the next frame is already known bad
                    yield j + 1, None
                    return
        n = len(cams)
        ready.record(compute)
        queue_copy(n - 1, ready)
        for j in range(max(0, n - 2), n):
            jj, img = emit(j)
            yield jj, img
            if img is None:
                return
            if jj + 1 < n and jj + 1 > verified:
                yield jj + 1, None
                return

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
    env = envmap if envmap is not None else getattr(gaussians, "environment", None)
    # one Renderer per (scene, atlas, environment, LUT) objects (resident.py):
    # repeated calls re-upload nothing and reuse the frame workspace
    key = (id(atlas), id(env), id(lut), mode, tile, None if background is None
           else tuple(float(v) for v in np.asarray(background, np.float64)))
    r = resident.cached(
        "renderer", gaussians, key,
        resident.scene_arrays(gaussians) + resident.env_arrays(env, lut)
        + (resident.atlas_arrays(atlas) if atlas is not None else []),
        lambda: Renderer(gaussians, atlas, envmap, lut, texture_mode=texture_mode,
                         sampler=sampler, tile=tile, background=background))
    return r.render(camera)
