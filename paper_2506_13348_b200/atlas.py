"""Texture-atlas packing (mirrors texsplat.atlas).

Reference: atlas.py:31-211. Charts are packed in splat-id order, row-major
within a page, in two RGBA families:
    family A = [albedo.r, albedo.g, albedo.b, roughness]
    family B = [normal.a, normal.b, metallic, 0]
The packing here is vectorised over splats (one reshape per page) instead of
the reference's per-splat Python loop; the resulting pages and indirection
entries are identical.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .scene import scene_texels

FAMILY_A = "albedo_roughness"
FAMILY_B = "normal_metallic"


@dataclass
class TextureAtlas:
    texels: np.ndarray  # (charts_y*T, charts_x*T, 4) float32
    family: str
    page_index: int
    charts_x: int
    charts_y: int
    resolution: int


@dataclass
class IndirectionBuffer:
    entries: np.ndarray  # (P, 3) int32 (chart_x, chart_y, page)
    charts_x: int
    charts_y: int
    pages: int

    def lookup(self, splat_id: int):
        if not 0 <= splat_id < self.entries.shape[0]:
            raise LookupError(f"splat id {splat_id} has no atlas entry")
        cx, cy, page = self.entries[splat_id]
        return int(cx), int(cy), int(page)

    def validate(self):
        if self.entries.ndim != 2 or self.entries.shape[1] != 3:
            raise ValueError("indirection entries must be (P, 3)")
        cx, cy, pg = self.entries[:, 0], self.entries[:, 1], self.entries[:, 2]
        if cx.size and (cx.min() < 0 or cx.max() >= self.charts_x):
            raise ValueError("chart_x out of range")
        if cy.size and (cy.min() < 0 or cy.max() >= self.charts_y):
            raise ValueError("chart_y out of range")
        if pg.size and (pg.min() < 0 or pg.max() >= self.pages):
            raise ValueError("page index out of range")


@dataclass
class AtlasSet:
    family_a: list
    family_b: list
    indirection: IndirectionBuffer
    resolution: int

    @property
    def atlases(self):
        return list(self.family_a) + list(self.family_b)


def chart_grid(num_splats: int, resolution: int, max_dim: int):
    """(charts_x, charts_y, pages) for P splats (atlas.py:108-124)."""
    if resolution > max_dim:
        raise ValueError("texture resolution exceeds the atlas dimension")
    if num_splats < 1:
        raise ValueError("need at least one splat to pack")
    charts_x = max_dim // resolution
    rows_needed = -(-num_splats // charts_x)
    charts_y = min(max_dim // resolution, rows_needed)
    per_page = charts_x * charts_y
    pages = -(-num_splats // per_page)
    return charts_x, charts_y, pages


def pack_texels(texels: np.ndarray, max_dim: int = 4096) -> AtlasSet:
    """Pack a (P, T, T, 7) combined texel array into atlas pages."""
    texels = np.ascontiguousarray(texels, dtype=np.float32)
    if texels.ndim != 4 or texels.shape[0] == 0:
        raise ValueError("no texture sets to pack")
    P, T = texels.shape[0], texels.shape[1]
    charts_x, charts_y, pages = chart_grid(P, T, max_dim)
    per_page = charts_x * charts_y
    ids = np.arange(P)
    page, idx = np.divmod(ids, per_page)
    cy, cx = np.divmod(idx, charts_x)
    entries = np.stack([cx, cy, page], axis=1).astype(np.int32)
    fam_a, fam_b = [], []
    for pg in range(pages):
        lo, hi = pg * per_page, min(P, (pg + 1) * per_page)
        n = hi - lo
        block = np.zeros((per_page, T, T, 7), dtype=np.float32)
        block[:n] = texels[lo:hi]
        # (charts_y, charts_x, T, T, 7) -> (charts_y*T, charts_x*T, 7)
        grid = block.reshape(charts_y, charts_x, T, T, 7).transpose(0, 2, 1, 3, 4)
        grid = grid.reshape(charts_y * T, charts_x * T, 7)
        a = np.empty(grid.shape[:2] + (4,), dtype=np.float32)
        b = np.zeros(grid.shape[:2] + (4,), dtype=np.float32)
        a[..., 0:3] = grid[..., 0:3]
        a[..., 3] = grid[..., 3]
        b[..., 0:2] = grid[..., 5:7]
        b[..., 2] = grid[..., 4]
        fam_a.append(TextureAtlas(a, FAMILY_A, pg, charts_x, charts_y, T))
        fam_b.append(TextureAtlas(b, FAMILY_B, pg, charts_x, charts_y, T))
    ind = IndirectionBuffer(entries, charts_x, charts_y, pages)
    return AtlasSet(fam_a, fam_b, ind, T)


def pack_atlases(sets, max_dim: int = 4096) -> AtlasSet:
    """pack_atlases(sets) of the reference (atlas.py:127-167). `sets` may be
    a list of MaterialTextureSet, a (P, T, T, 7) array, or a Scene."""
    if isinstance(sets, np.ndarray):
        return pack_texels(sets, max_dim)
    if hasattr(sets, "positions"):
        return pack_texels(scene_texels(sets), max_dim)
    if not sets:
        raise ValueError("no texture sets to pack")
    T = sets[0].resolution
    for s in sets:
        if s.resolution != T:
            raise ValueError("texture sets must share one resolution")
    return pack_texels(np.stack([s.combined() for s in sets]), max_dim)


def atlas_coords(chart_x, chart_y, s, t, resolution: int, charts_x: int, charts_y: int):
    """Normalised atlas coordinates of chart-local (s, t) (atlas.py:170-181)."""
    T = float(resolution)
    s_a = (np.asarray(chart_x) * T + np.asarray(s, dtype=np.float64) * T) / (charts_x * T)
    t_a = (np.asarray(chart_y) * T + np.asarray(t, dtype=np.float64) * T) / (charts_y * T)
    return s_a, t_a
