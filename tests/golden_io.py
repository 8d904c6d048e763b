"""Load the golden fixtures (tests/golden/*.npz) into package objects."""
from __future__ import annotations

import numpy as np

from paper_2506_13348_b200.environment import BrdfLut, EnvironmentLight
from paper_2506_13348_b200.scene import Scene, TextureConfig
from paper_2506_13348_b200.splats import Camera

from conftest import GOLDEN


def load(name):
    return np.load(GOLDEN / f"{name}.npz")


def camera(g, pre="cam_"):
    intr = g[pre + "intr"]
    W, H = (int(v) for v in g[pre + "size"])
    return Camera(g[pre + "w2v"], float(intr[0]), float(intr[1]), float(intr[2]),
                  float(intr[3]), W, H, float(intr[4]), float(intr[5]))


def environment(g, pre=""):
    if pre + "env_levels" not in g:
        return None
    L = int(g[pre + "env_levels"])
    return EnvironmentLight([g[f"{pre}env_mip{i}"] for i in range(L)], g[pre + "env_diffuse"])


def scene(g, pre=""):
    tex = g[pre + "texels"]
    return Scene(g[pre + "positions"], g[pre + "tangent_u"], g[pre + "tangent_v"],
                 g[pre + "scales"], g[pre + "opacities"], g[pre + "sh"],
                 int(g[pre + "sh_degree"]), tex, TextureConfig(int(tex.shape[1])),
                 environment=environment(g, pre), background=g[pre + "background"])


def lut():
    return BrdfLut(load("lut")["table"])


def cfg2_scene():
    """The 100k-splat shell scene, regenerated (bit-exact, see test_synth)."""
    from paper_2506_13348_b200 import synth
    return synth.make_shell_scene(100_000, 8, seed=3, with_environment=True)
