"""B200-native (sm_100a) textured 2D-Gaussian-splat render path.

A drop-in for the hot path of the TextureSplat reference renderer
(texsplat, /root/reference/pkg/src/texsplat): per-splat preprocess,
fp64-depth-rank + tile radix sort, per-tile textured compositing into the
13-channel G-buffer, deferred split-sum shading, and the training backward.
The compute runs in libtsb.so (hand-written CUDA for sm_100a, C ABI in
include/tsb.h); this package is the host layer with the reference's names.
"""

from .atlas import (AtlasSet, IndirectionBuffer, TextureAtlas, atlas_coords, chart_grid,
                    pack_atlases, pack_texels)
from .device import DeviceAtlas, DeviceEnvironment, DeviceScene, FrameWorkspace
from .environment import BrdfLut, EnvGrads, EnvironmentLight
from .rasterize import (NUM_CHANNELS, TILE, GBuffer, PreparedScene, Tape, frame_structure,
                        prepare, render_depth_map, render_forward, render_normal_map)
from .render import Renderer, render
from .scene import MaterialTextureSet, Scene, TextureConfig
from .shading import ShadeResult, shade_gbuffer
from .splats import ALPHA_CUTOFF, DENOM_EPS, SUPPORT_SIGMA, Camera
# the rest of texsplat's hot-path surface under the same top-level names
# (texsplat/__init__.py:10-36): adjoints, the training step and loop, formats
from .backward import SceneGrads, shade_backward, splat_backward
from .environment import (diffuse_irradiance, equirect_dirs, equirect_solid_angles,
                          prefilter_specular)
from .formats import (MissingReferenceError, SchemaError, VersionError, load_atlases,
                      load_manifest, load_scene, save_atlases, save_manifest, save_scene)
from .training import (LossWeights, TrainConfig, compute_step, linear_to_display, train)

__version__ = "0.1.0"

__all__ = [
    "AtlasSet", "IndirectionBuffer", "TextureAtlas", "atlas_coords", "chart_grid",
    "pack_atlases", "pack_texels", "DeviceAtlas", "DeviceEnvironment", "DeviceScene",
    "FrameWorkspace", "BrdfLut", "EnvGrads", "EnvironmentLight", "NUM_CHANNELS", "TILE",
    "GBuffer", "PreparedScene", "Tape", "frame_structure", "prepare", "render_depth_map",
    "render_forward", "render_normal_map", "Renderer", "render", "MaterialTextureSet", "Scene",
    "TextureConfig", "ShadeResult", "shade_gbuffer", "ALPHA_CUTOFF", "DENOM_EPS",
    "SUPPORT_SIGMA", "Camera", "SceneGrads", "shade_backward", "splat_backward",
    "diffuse_irradiance", "equirect_dirs", "equirect_solid_angles", "prefilter_specular",
    "MissingReferenceError", "SchemaError", "VersionError", "load_atlases", "load_manifest",
    "load_scene", "save_atlases", "save_manifest", "save_scene", "LossWeights", "TrainConfig",
    "compute_step", "linear_to_display", "train", "__version__",
]
