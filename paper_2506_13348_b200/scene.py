"""Scene container (mirrors texsplat.scene.Scene / texsplat.textures).

Reference: scene.py:52-151, textures.py:28-149. The reference keeps one
MaterialTextureSet object per splat; at 100k-2M splats that list dominates
host time, so this Scene stores every chart in one (P, T, T, 7) float32
array in the reference's combined channel order (textures.py:28-30:
albedo.rgb, roughness, metallic, tangent-normal a, b) and materialises
MaterialTextureSet objects only on request. Reference Scene objects are
accepted everywhere a Scene is (duck typing on the same field names).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

COMBINED_CHANNELS = 7


@dataclass
class TextureConfig:
    """Chart parameters shared by every map of a splat (textures.py:41-52)."""

    resolution: int = 4
    support: float = 3.0

    def __post_init__(self):
        if self.resolution < 1:
            raise ValueError("texture resolution must be >= 1")
        if self.support <= 0:
            raise ValueError("support must be positive")


class _Map:
    """Minimal TextureMap view: `.data` (T, T, C) float32 (textures.py:55-81)."""

    def __init__(self, data, semantic):
        self.data = np.ascontiguousarray(data, dtype=np.float32)
        self.semantic = semantic

    @property
    def resolution(self) -> int:
        return self.data.shape[0]


class MaterialTextureSet:
    """The four material maps of one splat (textures.py:84-149)."""

    def __init__(self, albedo, roughness, metallic, tangent_normal):
        self.albedo = albedo
        self.roughness = roughness
        self.metallic = metallic
        self.tangent_normal = tangent_normal

    @property
    def resolution(self) -> int:
        return self.albedo.data.shape[0]

    def combined(self) -> np.ndarray:
        return np.concatenate([self.albedo.data, self.roughness.data, self.metallic.data,
                               self.tangent_normal.data], axis=2)

    @staticmethod
    def from_combined(block) -> "MaterialTextureSet":
        block = np.ascontiguousarray(block, dtype=np.float32)
        if block.ndim != 3 or block.shape[2] != COMBINED_CHANNELS:
            raise ValueError("combined block must be (T, T, 7)")
        return MaterialTextureSet(_Map(block[:, :, 0:3], "albedo"),
                                  _Map(block[:, :, 3:4], "roughness"),
                                  _Map(block[:, :, 4:5], "metallic"),
                                  _Map(block[:, :, 5:7], "tangent_normal"))

    @staticmethod
    def constant(albedo, roughness, metallic, normal=(0.5, 0.5), resolution: int = 4):
        T = resolution
        block = np.empty((T, T, 7), dtype=np.float32)
        block[..., 0:3] = np.asarray(np.atleast_1d(albedo), dtype=np.float32)
        block[..., 3] = np.float32(roughness)
        block[..., 4] = np.float32(metallic)
        block[..., 5:7] = np.asarray(normal, dtype=np.float32)
        return MaterialTextureSet.from_combined(block)


@dataclass
class Scene:
    """Splat parameters (float64) plus texel charts and lighting."""

    positions: np.ndarray    # (P, 3)
    tangent_u: np.ndarray    # (P, 3)
    tangent_v: np.ndarray    # (P, 3)
    scales: np.ndarray       # (P, 2)
    opacities: np.ndarray    # (P,)
    sh: np.ndarray           # (P, K, 3)
    sh_degree: int
    texels: np.ndarray       # (P, T, T, 7) float32, combined order
    texture_config: TextureConfig = field(default_factory=TextureConfig)
    environment: object = None
    mesh: object = None
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64)
        self.tangent_u = np.ascontiguousarray(self.tangent_u, dtype=np.float64)
        self.tangent_v = np.ascontiguousarray(self.tangent_v, dtype=np.float64)
        self.scales = np.ascontiguousarray(self.scales, dtype=np.float64)
        self.opacities = np.ascontiguousarray(self.opacities, dtype=np.float64)
        self.sh = np.ascontiguousarray(self.sh, dtype=np.float64)
        self.texels = np.ascontiguousarray(self.texels, dtype=np.float32)
        self.background = np.asarray(self.background, dtype=np.float64)

    @property
    def num_splats(self) -> int:
        return self.positions.shape[0]

    @property
    def textures(self):
        """Reference-style list of MaterialTextureSet (built on demand)."""
        return [MaterialTextureSet.from_combined(b) for b in self.texels]

    def copy(self) -> "Scene":
        env = self.environment
        return Scene(self.positions.copy(), self.tangent_u.copy(), self.tangent_v.copy(),
                     self.scales.copy(), self.opacities.copy(), self.sh.copy(),
                     self.sh_degree, self.texels.copy(),
                     TextureConfig(self.texture_config.resolution,
                                   self.texture_config.support),
                     None if env is None else env.copy(), self.mesh,
                     self.background.copy())

    @staticmethod
    def from_reference(ref) -> "Scene":
        """Convert a texsplat.scene.Scene (or any object with its fields)."""
        return Scene(ref.positions, ref.tangent_u, ref.tangent_v, ref.scales, ref.opacities,
                     ref.sh, ref.sh_degree, scene_texels(ref),
                     TextureConfig(ref.texture_config.resolution,
                                   ref.texture_config.support),
                     getattr(ref, "environment", None), getattr(ref, "mesh", None),
                     getattr(ref, "background", np.zeros(3)))


def scene_texels(scene) -> np.ndarray:
    """(P, T, T, 7) float32 charts of a Scene or a reference Scene."""
    tex = getattr(scene, "texels", None)
    if isinstance(tex, np.ndarray):
        return tex
    sets = scene.textures
    if not sets:
        T = scene.texture_config.resolution
        return np.zeros((0, T, T, 7), dtype=np.float32)
    return np.stack([s.combined() for s in sets]).astype(np.float32, copy=False)


def flat_attrs(texels: np.ndarray) -> np.ndarray:
    """Per-splat mean texels for flat mode, (P, 5) float32: albedo rgb,
    metallic, roughness — the same numpy float32 means as rasterize.py:205-207."""
    P, T = texels.shape[0], texels.shape[1]
    out = np.zeros((P, 5), dtype=np.float32)
    for k in range(P):
        b = texels[k]
        out[k, 0:3] = np.ascontiguousarray(b[:, :, 0:3]).reshape(-1, 3).mean(axis=0)
        out[k, 3] = np.ascontiguousarray(b[:, :, 4:5]).mean()
        out[k, 4] = np.ascontiguousarray(b[:, :, 3:4]).mean()
    return out
