"""Device-resident inputs and frame workspace for libtsb.

PyTorch owns every device buffer (plumbing only); libtsb receives raw
pointers. Layouts:
  DeviceScene        float64 SoA: positions/t_u/t_v (P,3), scales (P,2),
                     opacities (P,), sh (P,K,3)       — scene.py:52-77
  DeviceAtlas        family A/B pages (pages, page_h, page_w, 4) float32,
                     indirection (P,3) int32, flat attrs (P,5) float32, and
                     the layered texture objects (RGBA32F or RGBA16F)
  DeviceEnvironment  spec mips (h_l, w_l, 3), diffuse (h, w, 3), LUT (r, r, 2), float32
  FrameWorkspace     one byte buffer carved by tsb_frame_workspace_size()
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .atlas import AtlasSet, pack_texels
from .scene import flat_attrs, scene_texels


def _dev(device):
    if device is None:
        if not torch.cuda.is_available():
            raise _lib.TsbError("libtsb needs a CUDA device (no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def morton_order(positions: np.ndarray, bits: int = 10) -> np.ndarray:
    """Splat indices sorted by the Morton (Z-order) code of their positions."""
    p = np.asarray(positions, np.float64)
    if len(p) == 0:
        return np.zeros(0, np.int64)
    lo, ext = p.min(0), max(float(np.ptp(p, axis=0).max()), 1e-300)
    q = np.clip(((p - lo) / ext * ((1 << bits) - 1)).astype(np.int64), 0, (1 << bits) - 1)
    code = np.zeros(len(q), np.int64)
    for b in range(bits):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return np.argsort(code, kind="stable")


class DeviceScene:
    """Splat parameters resident in HBM (float64, the reference's dtype)."""

    def __init__(self, scene, device=None):
        dev = _dev(device)
        self.device = dev
        self.num_splats = int(scene.positions.shape[0])
        self.sh_degree = int(scene.sh_degree)
        if not 0 <= self.sh_degree <= 3:
            raise ValueError("SH degree must be in [0, 3]")

        def up(a, shape):
            a = np.ascontiguousarray(a, dtype=np.float64).reshape(shape)
            return torch.from_numpy(a).to(dev, non_blocking=False)

        P = self.num_splats
        K = (self.sh_degree + 1) ** 2
        self.positions = up(scene.positions, (P, 3))
        self.tangent_u = up(scene.tangent_u, (P, 3))
        self.tangent_v = up(scene.tangent_v, (P, 3))
        self.scales = up(scene.scales, (P, 2))
        self.opacities = up(scene.opacities, (P,))
        self.sh = up(scene.sh, (P, K, 3))
        self.texture_resolution = int(scene.texture_config.resolution)
        # per-frame records stored in Morton order of position: splats that
        # share a tile sit close in memory when the rasteriser stages them
        self.record_slot = None
        if P > 1:
            order = morton_order(scene.positions)
            slot = np.empty(P, np.int32)
            slot[order] = np.arange(P, dtype=np.int32)
            self.record_slot = torch.from_numpy(slot).to(dev)

    @staticmethod
    def from_tensors(positions, tangent_u, tangent_v, scales, opacities, sh, sh_degree,
                     texture_resolution):
        self = DeviceScene.__new__(DeviceScene)
        self.device = positions.device
        self.num_splats = int(positions.shape[0])
        self.sh_degree = int(sh_degree)
        self.positions, self.tangent_u, self.tangent_v = positions, tangent_u, tangent_v
        self.scales, self.opacities, self.sh = scales, opacities, sh
        self.texture_resolution = int(texture_resolution)
        self.record_slot = None
        return self

    def struct(self) -> _lib.Scene_t:
        s = _lib.Scene_t()
        s.num_splats = self.num_splats
        s.sh_degree = self.sh_degree
        s.positions = _lib.ptr(self.positions)
        s.tangent_u = _lib.ptr(self.tangent_u)
        s.tangent_v = _lib.ptr(self.tangent_v)
        s.scales = _lib.ptr(self.scales)
        s.opacities = _lib.ptr(self.opacities)
        s.sh = _lib.ptr(self.sh)
        s.record_slot = _lib.ptr(getattr(self, "record_slot", None))
        return s


_FORMATS = {"rgba32f": _lib.TEXEL_RGBA32F, "rgba16f": _lib.TEXEL_RGBA16F}


class DeviceAtlas:
    """Atlas pages in HBM: linear copies (verify mode) and/or layered
    texture objects (HW mode), plus flat-mode per-splat means."""

    def __init__(self, atlas_set: AtlasSet = None, *, texels=None, linear=True, hw=True,
                 texel_format="rgba32f", flat=False, device=None):
        dev = _dev(device)
        self.device = dev
        if atlas_set is None:
            if texels is None:
                raise ValueError("DeviceAtlas needs an atlas_set or texels")
            atlas_set = pack_texels(texels)
        ind = atlas_set.indirection
        ind.validate()
        self.resolution = int(atlas_set.resolution)
        p0 = atlas_set.family_a[0].texels
        self.pages, self.page_h, self.page_w = len(atlas_set.family_a), int(p0.shape[0]), int(p0.shape[1])
        if self.pages * self.page_h * self.page_w >= 2 ** 31:
            raise ValueError("atlas larger than 2^31 texels per family")
        self.entries = torch.from_numpy(np.ascontiguousarray(ind.entries, np.int32)).to(dev)
        self.num_entries = int(ind.entries.shape[0])
        # page by page into one device tensor per family (no host-side stack:
        # a cfg5 atlas is 2 x 8.3 GB)
        shape = (self.pages, self.page_h, self.page_w, 4)
        fa = torch.empty(shape, dtype=torch.float32, device=dev)
        fb = torch.empty(shape, dtype=torch.float32, device=dev)
        for i, (qa, qb) in enumerate(zip(atlas_set.family_a, atlas_set.family_b)):
            fa[i].copy_(torch.from_numpy(np.ascontiguousarray(qa.texels, np.float32)))
            fb[i].copy_(torch.from_numpy(np.ascontiguousarray(qb.texels, np.float32)))
        self.family_a = fa if linear else None
        self.family_b = fb if linear else None
        self.texel_format = texel_format
        self.tex = None
        if hw:
            if texel_format not in _FORMATS:
                raise ValueError(f"unknown texel format {texel_format!r}")
            h = C.c_void_p()
            _lib.check(_lib.lib().tsb_atlas_tex_create(
                _lib.ptr(fa), _lib.ptr(fb), self.page_w, self.page_h, self.pages,
                _FORMATS[texel_format], C.byref(h), _lib.stream_handle()),
                "tsb_atlas_tex_create")
            torch.cuda.current_stream().synchronize()
            self.tex = h
        self.flat = None
        if flat is not False:
            fl = flat if isinstance(flat, np.ndarray) else None
            if fl is None:
                raise ValueError("flat=True needs the (P, 5) flat attribute array")
            self.flat = torch.from_numpy(np.ascontiguousarray(fl, np.float32)).to(dev)

    @staticmethod
    def interleaved(texels8: torch.Tensor) -> "DeviceAtlas":
        """Verify-mode atlas over a device tensor (P, T, T, 8) holding, per
        texel, family A (albedo rgb, roughness) then family B (normal a, b,
        metallic, 0) — the reference's 8-channel page order
        (rasterize.py:231-233). Chart k is row k of a single T-wide page,
        so the tensor can be a live training parameter (no repacking)."""
        if texels8.dim() != 4 or texels8.shape[-1] != 8 or texels8.dtype != torch.float32:
            raise ValueError("interleaved texels must be (P, T, T, 8) float32")
        if not texels8.is_contiguous():
            raise ValueError("interleaved texels must be contiguous")
        self = DeviceAtlas.__new__(DeviceAtlas)
        P, T = int(texels8.shape[0]), int(texels8.shape[1])
        self.device = texels8.device
        self.resolution = T
        self.pages, self.page_h, self.page_w = 1, P * T, T
        k = torch.arange(P, dtype=torch.int32, device=texels8.device)
        self.entries = torch.stack([torch.zeros_like(k), k, torch.zeros_like(k)], 1).contiguous()
        self.num_entries = P
        self.storage = texels8
        self.family_a = texels8
        self.family_b = texels8.view(-1)[4:]
        self.texel_stride = 2
        self.texel_format = None
        self.tex = None
        self.flat = None
        return self

    @staticmethod
    def flat_only(texels, device=None) -> "DeviceAtlas":
        self = DeviceAtlas.__new__(DeviceAtlas)
        dev = _dev(device)
        self.device = dev
        self.resolution = int(texels.shape[1])
        self.pages = self.page_h = self.page_w = 0
        self.entries = None
        self.num_entries = int(texels.shape[0])
        self.family_a = self.family_b = None
        self.texel_format = None
        self.tex = None
        self.flat = torch.from_numpy(flat_attrs(texels)).to(dev)
        return self

    def struct(self) -> _lib.Atlas_t:
        a = _lib.Atlas_t()
        a.resolution = self.resolution
        a.page_w, a.page_h, a.pages = self.page_w, self.page_h, self.pages
        a.entries = _lib.ptr(self.entries)
        a.family_a = _lib.ptr(self.family_a)
        a.family_b = _lib.ptr(self.family_b)
        a.flat_attrs = _lib.ptr(self.flat)
        a.tex = self.tex.value if self.tex is not None else None
        a.texel_stride = getattr(self, "texel_stride", 1)
        return a

    def close(self):
        if self.tex is not None and self.tex.value:
            _lib.lib().tsb_atlas_tex_destroy(self.tex)
            self.tex = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceEnvironment:
    """Environment mips, irradiance map and split-sum LUT in HBM (float32)."""

    def __init__(self, env, lut, device=None):
        dev = _dev(device)
        self.device = dev
        if env.levels < 1 or env.levels > _lib.ENV_MAX_LEVELS:
            raise ValueError(f"environment needs 1..{_lib.ENV_MAX_LEVELS} levels")
        self.mips = [torch.from_numpy(np.ascontiguousarray(m, np.float32)).to(dev)
                     for m in env.spec_mips]
        self.diffuse = torch.from_numpy(np.ascontiguousarray(env.diffuse, np.float32)).to(dev)
        table = np.ascontiguousarray(lut.table, np.float32)
        self.lut = torch.from_numpy(table).to(dev)
        self.lut_res = int(table.shape[0])

    @staticmethod
    def from_tensors(mips, diffuse, lut):
        self = DeviceEnvironment.__new__(DeviceEnvironment)
        self.device = diffuse.device
        self.mips, self.diffuse, self.lut = list(mips), diffuse, lut
        self.lut_res = int(lut.shape[0])
        return self

    @property
    def levels(self) -> int:
        return len(self.mips)

    def struct(self) -> _lib.Environment_t:
        e = _lib.Environment_t()
        e.levels = len(self.mips)
        for i, m in enumerate(self.mips):
            e.spec_mips[i] = _lib.ptr(m)
            e.mip_h[i] = int(m.shape[0])
            e.mip_w[i] = int(m.shape[1])
        e.diffuse = _lib.ptr(self.diffuse)
        e.diff_h, e.diff_w = int(self.diffuse.shape[0]), int(self.diffuse.shape[1])
        e.lut = _lib.ptr(self.lut)
        e.lut_res = self.lut_res
        return e


class FrameWorkspace:
    """Frame workspace (sort buffers, per-splat records, tile lists) sized for
    `capacity` splat x tile entries; grown when a frame needs more.

    `needed` (device int64) receives each frame's entry count; `max_needed`
    is the device-side running maximum over every frame binned since the
    last `reset_max()` (tsb_frame_workspace_max_needed_offset), so frames
    replayed without a host check can be validated afterwards. `generation`
    counts the frames rendered into the workspace (a Tape remembers its own)."""

    def __init__(self, device=None):
        self.device = _dev(device)
        self.key = None
        self.capacity = 0
        self.buf = None
        self.nbytes = 0
        self.needed = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.max_needed = None
        self.generation = 0
        self.shrink_to = None

    def ensure(self, P, W, H, tile, capacity, exact: bool = False):
        """Make room for `capacity` entries (`exact=True` also shrinks)."""
        key = (P, W, H, tile)
        if self.key == key and (self.capacity == capacity or
                                (not exact and self.capacity >= capacity)):
            return
        cap = max(int(capacity), 1)
        nb, off = C.c_uint64(), C.c_uint64()
        L = _lib.lib()
        _lib.check(L.tsb_frame_workspace_size(P, W, H, tile, cap, C.byref(nb)),
                   "tsb_frame_workspace_size")
        _lib.check(L.tsb_frame_workspace_max_needed_offset(P, W, H, tile, cap, C.byref(off)),
                   "tsb_frame_workspace_max_needed_offset")
        self.buf = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        self.nbytes = int(nb.value)
        o = int(off.value)
        self.max_needed = self.buf[o:o + 8].view(torch.int64)
        self.max_needed.zero_()
        self.capacity = cap
        self.key = key
        self.generation += 1

    def reset_max(self):
        if self.max_needed is not None:
            self.max_needed.zero_()

    def max_needed_value(self) -> int:
        """Largest entry count of any frame since reset_max() (host sync)."""
        return 0 if self.max_needed is None else int(self.max_needed.item())

    def overflowed(self) -> bool:
        return self.max_needed_value() > self.capacity

    @staticmethod
    def initial_capacity(P, W, H, tile):
        return int(16 * P + 4 * ((W + tile - 1) // tile) * ((H + tile - 1) // tile) + 4096)
