"""Render a few cfg2 frames for ncu (no timing; use under ncu only after a
plain run of the same command exited 0)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2506_13348_b200 import Renderer, pack_atlases, synth  # noqa: E402
from paper_2506_13348_b200.environment import BrdfLut  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--splats", type=int, default=100_000)
ap.add_argument("--texture-res", type=int, default=8)
ap.add_argument("--width", type=int, default=800)
ap.add_argument("--height", type=int, default=800)
ap.add_argument("--sampler", default="hw")
ap.add_argument("--texel-format", default="rgba32f")
a = ap.parse_args()
scene = synth.make_shell_scene(a.splats, a.texture_res, seed=3, with_environment=True)
cams = synth.bench_cameras(256, a.width, a.height)
mode = "flat" if a.sampler == "flat" else "atlas"
r = Renderer(scene, pack_atlases(scene) if mode == "atlas" else None, scene.environment,
             BrdfLut.build(), texture_mode=mode, sampler=None if mode == "flat" else a.sampler,
             texel_format=a.texel_format)
r.render(cams[0], check=True)
r.reserve(cams[0], int(r.entries_needed() * 1.25) + 4096)  # as bench.py sizes it
for i in range(a.frames):
    r.render(cams[i], check=(i == 0))
torch.cuda.synchronize()
print("frames ok", r.entries_needed())
